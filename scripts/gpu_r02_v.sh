#!/bin/bash
# r02 batch V: bottom levels on by default (b >= 10, >= 2M dofs): full GPU suite + probes
O=gpurun_out/r02v; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
run() { local name=$1 cfg=$2; shift 2; env PDG_SETUP_TIMES=1 "$@" timeout 600 python scripts/c4_probe.py 3 $cfg > $O/$name.txt 2>&1; echo "rc=$?" >> $O/$name.txt; }
run c4 config4
run c4_off config4 PDG_BOTTOM_KB=0
run c5p4 config5:4
run c5p4_off config5:4 PDG_BOTTOM_KB=0
run c5p2 config5:2
run c2 config2
timeout 500 python scripts/chunk_trace.py config4 > $O/trace_c4.txt 2>&1
