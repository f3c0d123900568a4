#!/bin/bash
# r02 batch B: full gpu test list, config4 sweep ncu capture, config4 launch list
O=gpurun_out/r02b; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
PDG_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 30 -c 1 \
  -o $O/sweep_c4 python scripts/c4_probe.py 1 config4 > $O/ncu_sweep.log 2>&1; echo "rc=$?" >> $O/ncu_sweep.log
PDG_NO_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 1500 --csv \
  --log-file $O/launches_c4.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_bench.log 2>&1; echo "rc=$?" >> $O/ncu_bench.log
