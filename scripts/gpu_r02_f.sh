#!/bin/bash
# r02 batch F: warp-worker sweep (PDG_SWEEP=warp): correctness, then config4/config2 timings by ordering and unit size
O=gpurun_out/r02f; mkdir -p $O
PDG_SWEEP=warp PDG_ORDER=md PDG_MD_RELAX=2 PDG_RELAX_Z=0.3 timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu_warp.log 2>&1; echo "rc=$?" >> $O/pytest_gpu_warp.log
run() {  # name, config, env...
  local name=$1 cfg=$2; shift 2
  env "$@" timeout 600 python scripts/c4_probe.py 2 $cfg > $O/$name.txt 2>&1; echo "rc=$?" >> $O/$name.txt
}
W="PDG_SWEEP=warp PDG_ORDER=md"
run c4_w_r1 config4 $W PDG_MD_RELAX=1 PDG_RELAX_Z=0.3
run c4_w_r2z3 config4 $W PDG_MD_RELAX=2 PDG_RELAX_Z=0.3
run c4_w_r4z3 config4 $W PDG_MD_RELAX=4 PDG_RELAX_Z=0.3
run c4_w_r8z5 config4 $W PDG_MD_RELAX=8 PDG_RELAX_Z=0.5
run c4_w_r4z3_u8 config4 $W PDG_MD_RELAX=4 PDG_RELAX_Z=0.3 PDG_UNIT_KB=8
run c4_w_r4z3_u32 config4 $W PDG_MD_RELAX=4 PDG_RELAX_Z=0.3 PDG_UNIT_KB=32
run c4_w_nd config4 PDG_SWEEP=warp
run c2_w_r2z3 config2 $W PDG_MD_RELAX=2 PDG_RELAX_Z=0.3
run c2_w_r4z3 config2 $W PDG_MD_RELAX=4 PDG_RELAX_Z=0.3
run c2_w_r4z3_u8 config2 $W PDG_MD_RELAX=4 PDG_RELAX_Z=0.3 PDG_UNIT_KB=8
run c2_w_nd config2 PDG_SWEEP=warp
PDG_SWEEP=warp PDG_ORDER=md PDG_MD_RELAX=4 PDG_RELAX_Z=0.3 PDG_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__warps_active.avg.pct_of_peak_sustained_active \
   --clock-control none -k regex:sweep_warp_kernel -s 20 -c 1 --csv python scripts/c4_probe.py 1 config4 > $O/ncu_c4_w_r4z3.csv 2>&1
