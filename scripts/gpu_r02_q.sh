#!/bin/bash
# r02 batch Q: subtree bundles A/B (PDG_BUNDLE_KB, PDG_MD_RELAX) + parity
O=gpurun_out/r02q2; mkdir -p $O
PDG_BUNDLE_KB=64 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > $O/pytest_parity.log 2>&1; echo "rc=$?" >> $O/pytest_parity.log
run() { local name=$1 cfg=$2; shift 2; env PDG_SETUP_TIMES=1 "$@" timeout 600 python scripts/c4_probe.py 2 $cfg > $O/$name.txt 2>&1; echo "rc=$?" >> $O/$name.txt; }
run c4_off config4 PDG_BUNDLE_KB=0
run c4_b96_r8 config4
run c4_b96_r2 config4 PDG_MD_RELAX=2
run c4_b96_r1 config4 PDG_MD_RELAX=1
run c4_b48_r1 config4 PDG_MD_RELAX=1 PDG_BUNDLE_KB=48
run c4_b32_r2 config4 PDG_MD_RELAX=2 PDG_BUNDLE_KB=32
run c4_b96_r1_t64 config4 PDG_MD_RELAX=1 PDG_SWEEP_THREADS=64
run c2_b96 config2 PDG_BUNDLE_KB=96
