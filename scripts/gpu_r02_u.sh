#!/bin/bash
# r02 batch U: level chunks, tuned kernel; ordering variants (PDG_MD_RELAX, PDG_RELAX_MIN_SUBTREE), bottom size
O=gpurun_out/r02u; mkdir -p $O
PDG_BOTTOM_KB=64 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > $O/pytest_parity.log 2>&1; echo "rc=$?" >> $O/pytest_parity.log
run() { local name=$1 cfg=$2; shift 2; env PDG_SETUP_TIMES=1 "$@" timeout 600 python scripts/c4_probe.py 2 $cfg > $O/$name.txt 2>&1; echo "rc=$?" >> $O/$name.txt; }
run c4_off config4 PDG_BOTTOM_KB=0
run c4_r2 config4 PDG_MD_RELAX=2
run c4_r1 config4 PDG_MD_RELAX=1
run c4_r8_m12 config4 PDG_RELAX_MIN_SUBTREE=12
run c4_r8_m20 config4 PDG_RELAX_MIN_SUBTREE=20
run c4_r8_m32 config4 PDG_RELAX_MIN_SUBTREE=32
run c4_r8_m20_b160 config4 PDG_RELAX_MIN_SUBTREE=20 PDG_BOTTOM_KB=160
run c4_r1_b48 config4 PDG_MD_RELAX=1 PDG_BOTTOM_KB=48
run c4_r1_b160_l8 config4 PDG_MD_RELAX=1 PDG_BOTTOM_KB=160 PDG_BOTTOM_LEVELS=8
PDG_MD_RELAX=1 timeout 500 python scripts/chunk_trace.py config4 > $O/trace_r1.txt 2>&1
run c5p2_off config5:2 PDG_BOTTOM_KB=0
run c5p2_r1 config5:2 PDG_MD_RELAX=1
run c5p4_off config5:4 PDG_BOTTOM_KB=0
run c5p4_r1 config5:4 PDG_MD_RELAX=1
