#!/bin/bash
# r02 batch G: new defaults (MD >= 2M dofs, even-row panels, 128 KB units): tests, bench, probes, ncu
O=gpurun_out/r02g; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
run() { local name=$1 cfg=$2; shift 2; env "$@" timeout 600 python scripts/c4_probe.py 2 $cfg > $O/$name.txt 2>&1; }
run c4_u192 config4 PDG_UNIT_MAX_KB=192
run c4_u256 config4 PDG_UNIT_MAX_KB=256
run c2 config2
run c5p2 config5:2
run c5p4 config5:4
run c3p4s64 config3:4:64
PDG_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 30 -c 1 \
  -o $O/sweep_c4 python scripts/c4_probe.py 1 config4 > $O/ncu_sweep.log 2>&1
PDG_NO_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 1500 --csv \
  --log-file $O/launches_c4.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_bench.log 2>&1
