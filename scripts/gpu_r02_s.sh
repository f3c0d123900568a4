#!/bin/bash
# r02 batch S: bottom levels as column-streamed level chunks (PDG_BOTTOM_KB / _LEVELS, PDG_CHUNK_KB, PDG_MD_RELAX) + parity
O=gpurun_out/r02s; mkdir -p $O
PDG_BOTTOM_KB=64 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > $O/pytest_parity.log 2>&1; echo "rc=$?" >> $O/pytest_parity.log
run() { local name=$1 cfg=$2; shift 2; env PDG_SETUP_TIMES=1 "$@" timeout 600 python scripts/c4_probe.py 2 $cfg > $O/$name.txt 2>&1; echo "rc=$?" >> $O/$name.txt; }
run c4_off config4 PDG_BOTTOM_KB=0
run c4_r8 config4
run c4_r2 config4 PDG_MD_RELAX=2
run c4_r1 config4 PDG_MD_RELAX=1
run c4_r1_l4 config4 PDG_MD_RELAX=1 PDG_BOTTOM_LEVELS=4
run c4_r1_l10 config4 PDG_MD_RELAX=1 PDG_BOTTOM_LEVELS=10
run c4_r1_c128 config4 PDG_MD_RELAX=1 PDG_CHUNK_KB=128
run c4_r1_b256 config4 PDG_MD_RELAX=1 PDG_BOTTOM_KB=256
PDG_MD_RELAX=1 timeout 500 python scripts/chunk_trace.py config4 > $O/trace_r1.txt 2>&1
run c2_b96 config2 PDG_BOTTOM_KB=96
