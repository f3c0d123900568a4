#!/bin/bash
# r02 batch AE: bottom levels at mid sizes (config 3 rows, 65,536 cells)
O=gpurun_out/r02ae; mkdir -p $O
run() { local name=$1 cfg=$2; shift 2; env PDG_SETUP_TIMES=1 "$@" timeout 300 python scripts/c4_probe.py 5 $cfg > $O/$name.txt 2>&1; echo "rc=$?" >> $O/$name.txt; }
for c in 3:64 3:256 4:64 4:256 2:64; do
  n=c3_${c/:/_}
  run ${n}_off config3:$c
  run ${n}_nd_b64 config3:$c PDG_BOTTOM_KB=64
  run ${n}_md1_b160 config3:$c PDG_BOTTOM_KB=160 PDG_ORDER=md PDG_MD_RELAX=1
  run ${n}_md2_b160 config3:$c PDG_BOTTOM_KB=160 PDG_ORDER=md PDG_MD_RELAX=2
  run ${n}_md8_off config3:$c PDG_ORDER=md
done
