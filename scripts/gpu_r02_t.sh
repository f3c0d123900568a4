#!/bin/bash
# r02 batch T: bottom levels as level chunks with the lean per-tile kernel (PDG_BOTTOM_KB / _LEVELS, PDG_CHUNK_KB, PDG_MD_RELAX) + parity
O=gpurun_out/r02t; mkdir -p $O
PDG_BOTTOM_KB=64 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > $O/pytest_parity.log 2>&1; echo "rc=$?" >> $O/pytest_parity.log
run() { local name=$1 cfg=$2; shift 2; env PDG_SETUP_TIMES=1 "$@" timeout 600 python scripts/c4_probe.py 2 $cfg > $O/$name.txt 2>&1; echo "rc=$?" >> $O/$name.txt; }
run c4_off config4 PDG_BOTTOM_KB=0
run c4_r8 config4
run c4_r2 config4 PDG_MD_RELAX=2
run c4_r1 config4 PDG_MD_RELAX=1
run c4_r1_l4 config4 PDG_MD_RELAX=1 PDG_BOTTOM_LEVELS=4
run c4_r1_l10 config4 PDG_MD_RELAX=1 PDG_BOTTOM_LEVELS=10
run c4_r1_c32 config4 PDG_MD_RELAX=1 PDG_CHUNK_KB=32
run c4_r1_c128 config4 PDG_MD_RELAX=1 PDG_CHUNK_KB=128
PDG_MD_RELAX=1 timeout 500 python scripts/chunk_trace.py config4 > $O/trace_r1.txt 2>&1
