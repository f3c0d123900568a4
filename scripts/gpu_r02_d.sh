#!/bin/bash
# r02 batch D: config4 sweep L2 policy A/B (prefetch bits) x ordering (ND vs MD relaxed)
O=gpurun_out/r02d; mkdir -p $O
run() {  # name, env...
  local name=$1; shift
  env "$@" timeout 600 python scripts/c4_probe.py 2 config4 > $O/c4_$name.txt 2>&1; echo "rc=$?" >> $O/c4_$name.txt
  env "$@" PDG_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum \
     --clock-control none -k regex:sweep_kernel -s 20 -c 1 --csv python scripts/c4_probe.py 1 config4 > $O/ncu_$name.csv 2>&1
}
run nd_pf1 PDG_SWEEP_PREFETCH=1
run nd_pf3 PDG_SWEEP_PREFETCH=3
run nd_pf7 PDG_SWEEP_PREFETCH=7
run nd_pf2 PDG_SWEEP_PREFETCH=2
M="PDG_ORDER=md PDG_MD_RELAX=8 PDG_RELAX_Z=0.5"
run md8_pf1 $M PDG_SWEEP_PREFETCH=1
run md8_pf3 $M PDG_SWEEP_PREFETCH=3
run md8_pf7 $M PDG_SWEEP_PREFETCH=7
run md12z5_pf3 PDG_ORDER=md PDG_MD_RELAX=12 PDG_RELAX_Z=0.5 PDG_SWEEP_PREFETCH=3
run md8z4_pf3 PDG_ORDER=md PDG_MD_RELAX=8 PDG_RELAX_Z=0.4 PDG_SWEEP_PREFETCH=3
run md16z4_pf3 PDG_ORDER=md PDG_MD_RELAX=16 PDG_RELAX_Z=0.4 PDG_SWEEP_PREFETCH=3
