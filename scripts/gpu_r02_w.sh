#!/bin/bash
# r02 batch W: level chunks: CTA size and chunk size
O=gpurun_out/r02w; mkdir -p $O
run() { local name=$1 cfg=$2; shift 2; env PDG_SETUP_TIMES=1 "$@" timeout 600 python scripts/c4_probe.py 2 $cfg > $O/$name.txt 2>&1; echo "rc=$?" >> $O/$name.txt; }
run c4 config4
run c4_t64 config4 PDG_SWEEP_THREADS=64
run c4_c32 config4 PDG_CHUNK_KB=32
run c4_c48 config4 PDG_CHUNK_KB=48
run c4_c96 config4 PDG_CHUNK_KB=96
run c4_t64_c32 config4 PDG_SWEEP_THREADS=64 PDG_CHUNK_KB=32
run c4_b320_l12 config4 PDG_BOTTOM_KB=320 PDG_BOTTOM_LEVELS=12
run c4_u64 config4 PDG_UNIT_MAX_KB=64
