#!/bin/bash
# r02 batch O: runtime CTA size (64 for large small-block problems) check + config2 sweep-shape scan
O=gpurun_out/r02o; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
run() { local name=$1 cfg=$2; shift 2; env "$@" timeout 600 python scripts/c4_probe.py 3 $cfg > $O/$name.txt 2>&1; }
run c5p2 config5:2
run c5p2_t128 config5:2 PDG_SWEEP_THREADS=128
run c3p2s256 config3:2:256
run c3p2s256_t64 config3:2:256 PDG_SWEEP_THREADS=64
run c2 config2
for leaf in 4 8 12; do run c2_leaf$leaf config2 PDG_ND_LEAF=$leaf; done
for mg in 1 3; do run c2_merge$mg config2 PDG_ND_MERGE=$mg; done
for kb in 16 24 32; do run c2_u$kb config2 PDG_UNIT_KB=$kb PDG_LEAF_KB=$kb; done
run c2_leafkb16 config2 PDG_LEAF_KB=16
run c2_ro8 config2 PDG_ROW_ALIGN=8
