#!/bin/bash
# r02 batch AI: chunk / bottom size under the grouped order
O=gpurun_out/r02ai; mkdir -p $O
run() { local name=$1 cfg=$2; shift 2; env PDG_SETUP_TIMES=1 "$@" timeout 600 python scripts/c4_probe.py 3 $cfg > $O/$name.txt 2>&1; echo "rc=$?" >> $O/$name.txt; }
run c4_def config4
run c4_c96 config4 PDG_CHUNK_KB=96
run c4_c48 config4 PDG_CHUNK_KB=48
run c4_b320_l12 config4 PDG_BOTTOM_KB=320 PDG_BOTTOM_LEVELS=12
run c4_b96_l6 config4 PDG_BOTTOM_KB=96 PDG_BOTTOM_LEVELS=6
run c4_x2048 config4 PDG_CHUNK_X=2048 PDG_CHUNK_KB=80
