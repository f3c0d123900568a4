#!/bin/bash
# r02 batch AH: evidence on HEAD — GPU suite, smoke, bench (both arms), ncu full capture of the sweep, launch list, probes
O=gpurun_out/r02ah; mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "rc=$?" >> $O/bench_ref.err
PDG_BOTTOM_KB=0 timeout 900 python bench.py --no-cpu-baseline > $O/bench_off.json 2> $O/bench_off.err
PDG_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 30 -c 1 \
  -o $O/sweep_c4 python scripts/c4_probe.py 1 config4 > $O/ncu_sweep.log 2>&1
PDG_NO_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 1500 --csv \
  --log-file $O/launches_c4.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_bench.log 2>&1
run() { local name=$1 cfg=$2; shift 2; env PDG_SETUP_TIMES=1 "$@" timeout 600 python scripts/c4_probe.py 3 $cfg > $O/$name.txt 2>&1; echo "rc=$?" >> $O/$name.txt; }
run c4 config4
run c5p4 config5:4
run c5p2 config5:2
run c5p2_off config5:2 PDG_BOTTOM_KB=0
run c2 config2
timeout 500 python scripts/chunk_trace.py config4 > $O/trace_c4.txt 2>&1
timeout 900 python scripts/c5_probe.py 2 > $O/c5_probe_p2.txt 2>&1
