#!/bin/bash
# r02 batch Y: level chunks in subdomain groups for the lowest levels (PDG_BOTTOM_GROUP_MB / _GROUP_LEVELS / _INTERLEAVE)
O=gpurun_out/r02y2; mkdir -p $O
PDG_BOTTOM_KB=64 PDG_BOTTOM_GROUP_MB=1 PDG_BOTTOM_GROUP_LEVELS=2 PDG_BOTTOM_INTERLEAVE=2 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > $O/pytest_parity.log 2>&1; echo "rc=$?" >> $O/pytest_parity.log
run() { local name=$1 cfg=$2; shift 2; env PDG_SETUP_TIMES=1 "$@" timeout 600 python scripts/c4_probe.py 2 $cfg > $O/$name.txt 2>&1; echo "rc=$?" >> $O/$name.txt; }
run c4_def config4
run c4_gl0 config4 PDG_BOTTOM_GROUP_LEVELS=0
run c4_gl2 config4 PDG_BOTTOM_GROUP_LEVELS=2
run c4_gl1 config4 PDG_BOTTOM_GROUP_LEVELS=1
run c4_gl2_i8 config4 PDG_BOTTOM_GROUP_LEVELS=2 PDG_BOTTOM_INTERLEAVE=8
run c4_gl3_i8 config4 PDG_BOTTOM_INTERLEAVE=8
run c4_gl2_g64_i4 config4 PDG_BOTTOM_GROUP_LEVELS=2 PDG_BOTTOM_GROUP_MB=64
run c4_gl2_g16_i8 config4 PDG_BOTTOM_GROUP_LEVELS=2 PDG_BOTTOM_GROUP_MB=16 PDG_BOTTOM_INTERLEAVE=8
timeout 500 python scripts/chunk_trace.py config4 > $O/trace_c4.txt 2>&1
