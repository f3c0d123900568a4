#!/bin/bash
# r02 batch AJ: chunk tiles dealt to the warps longest first
O=gpurun_out/r02aj; mkdir -p $O
PDG_BOTTOM_KB=64 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_tuning_knobs.py -m gpu -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
run() { local name=$1 cfg=$2; shift 2; env PDG_SETUP_TIMES=1 "$@" timeout 600 python scripts/c4_probe.py 3 $cfg > $O/$name.txt 2>&1; echo "rc=$?" >> $O/$name.txt; }
run c4 config4
run c5p4 config5:4
run c5p2 config5:2
timeout 500 python scripts/chunk_trace.py config4 > $O/trace_c4.txt 2>&1
