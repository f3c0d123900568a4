#!/bin/bash
# r02 batch P: persistent vector kernels A/B + GPU suite
O=gpurun_out/r02p; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
run() { local name=$1 cfg=$2; shift 2; env "$@" timeout 600 python scripts/c4_probe.py 3 $cfg > $O/$name.txt 2>&1; }
run c4 config4
run c4_np config4 PDG_PERSIST=0
run c2 config2
run c2_np config2 PDG_PERSIST=0
run c5p4 config5:4
run c5p4_np config5:4 PDG_PERSIST=0
timeout 900 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err
PDG_PERSIST=0 timeout 900 python bench.py --no-cpu-baseline > $O/bench_np.json 2> $O/bench_np.err
timeout 1200 python scripts/c3_study.py $O/c3 > $O/c3_study.log 2>&1
