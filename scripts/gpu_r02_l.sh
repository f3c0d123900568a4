#!/bin/bash
# r02 batch L: sweep CTA size (build knob PDG_SWEEP_THREADS=64) x MD amalgamation (config4, config2, config5 p=2)
O=gpurun_out/r02l; mkdir -p $O
R=$(pwd)
T=64
rm -rf /tmp/v$T; mkdir -p /tmp/v$T; cp -r paper_2512_19536_b200 scripts tests include /tmp/v$T/
(cd /tmp/v$T && make -C paper_2512_19536_b200/csrc -j16 BUILD=/tmp/v$T/build/csrc EXTRA_NVFLAGS=-DPDG_SWEEP_THREADS=$T > $R/$O/build_$T.log 2>&1; echo "build rc=$?" >> $R/$O/build_$T.log)
grep -A2 sweep_kernel /tmp/v$T/build/csrc/sweep.ptxas.log >> $R/$O/build_$T.log
run() { local dir=$1 name=$2 cfg=$3; shift 3; (cd $dir && env "$@" timeout 600 python scripts/c4_probe.py 2 $cfg > $R/$O/$name.txt 2>&1); }
for v in "$R 128" "/tmp/v64 64"; do
  set -- $v; D=$1; T=$2
  run $D t${T}_c4 config4
  run $D t${T}_c4_md4z4 config4 PDG_MD_RELAX=4 PDG_RELAX_Z=0.4
  run $D t${T}_c4_md2z3 config4 PDG_MD_RELAX=2 PDG_RELAX_Z=0.3
  run $D t${T}_c4_md4z4_u64 config4 PDG_MD_RELAX=4 PDG_RELAX_Z=0.4 PDG_UNIT_KB=64
  run $D t${T}_c2 config2
  run $D t${T}_c5p2 config5:2
done
# per-unit trace with the batched forward gather (compare trace_c4 of r02j: gather|ready 3.16 us)
(cd $R && timeout 900 python scripts/sweep_trace.py config4 > $R/$O/trace_c4.txt 2>&1)
# list-schedule cost model calibrated to the traced unit times (fixed ~7 us, ~10 GB/s per CTA, publish ~1.3 us)
run $R sched_c4_a config4 PDG_SCHED_COST=7000,10,1300
run $R sched_c4_b config4 PDG_SCHED_COST=4000,15,1000
run $R sched_c2_a config2 PDG_SCHED_COST=7000,10,1300
run $R sched_c2_b config2 PDG_SCHED_COST=4000,15,1000
(cd $R && timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $R/$O/smoke.log 2>&1; echo "smoke rc=$?" >> $R/$O/smoke.log)
