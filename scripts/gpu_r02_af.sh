#!/bin/bash
# r02 batch AF: level chunks in subdomain groups, skewed order (group g's level l runs one step after its level l-1)
O=gpurun_out/r02af; mkdir -p $O
PDG_BOTTOM_KB=64 PDG_BOTTOM_GROUP_MB=1 PDG_BOTTOM_GROUP_LEVELS=99 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > $O/pytest_parity.log 2>&1; echo "rc=$?" >> $O/pytest_parity.log
run() { local name=$1 cfg=$2; shift 2; env PDG_SETUP_TIMES=1 "$@" timeout 600 python scripts/c4_probe.py 2 $cfg > $O/$name.txt 2>&1; echo "rc=$?" >> $O/$name.txt; }
run c4_global config4
run c4_g64_all config4 PDG_BOTTOM_GROUP_MB=64 PDG_BOTTOM_GROUP_LEVELS=99
run c4_g96_all config4 PDG_BOTTOM_GROUP_MB=96 PDG_BOTTOM_GROUP_LEVELS=99
run c4_g128_all config4 PDG_BOTTOM_GROUP_MB=128 PDG_BOTTOM_GROUP_LEVELS=99
run c4_g192_all config4 PDG_BOTTOM_GROUP_MB=192 PDG_BOTTOM_GROUP_LEVELS=99
run c4_g96_l3 config4 PDG_BOTTOM_GROUP_MB=96 PDG_BOTTOM_GROUP_LEVELS=3
run c4_g128_l4 config4 PDG_BOTTOM_GROUP_MB=128 PDG_BOTTOM_GROUP_LEVELS=4
PDG_BOTTOM_GROUP_MB=96 PDG_BOTTOM_GROUP_LEVELS=99 timeout 500 python scripts/chunk_trace.py config4 > $O/trace_g96_all.txt 2>&1
