#!/bin/bash
# r02 batch AG: skewed grouped order, group size
O=gpurun_out/r02ag; mkdir -p $O
run() { local name=$1 cfg=$2; shift 2; env PDG_SETUP_TIMES=1 "$@" timeout 600 python scripts/c4_probe.py 3 $cfg > $O/$name.txt 2>&1; echo "rc=$?" >> $O/$name.txt; }
run c4_g160 config4 PDG_BOTTOM_GROUP_MB=160 PDG_BOTTOM_GROUP_LEVELS=99
run c4_g256 config4 PDG_BOTTOM_GROUP_MB=256 PDG_BOTTOM_GROUP_LEVELS=99
run c4_global config4
run c5p4_g160 config5:4 PDG_BOTTOM_GROUP_MB=160 PDG_BOTTOM_GROUP_LEVELS=99
run c5p4_g256 config5:4 PDG_BOTTOM_GROUP_MB=256 PDG_BOTTOM_GROUP_LEVELS=99
run c5p4_global config5:4
run c5p2_g160 config5:2 PDG_BOTTOM_GROUP_MB=160 PDG_BOTTOM_GROUP_LEVELS=99
run c5p2_global config5:2
