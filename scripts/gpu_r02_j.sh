#!/bin/bash
# r02 batch J: sweep CTA size (64 / 128 / 256 threads, build knob) x MD amalgamation at config4 and config2
O=gpurun_out/r02j; mkdir -p $O
R=$(pwd)
for T in 64 256; do
  rm -rf /tmp/v$T; mkdir -p /tmp/v$T; cp -r paper_2512_19536_b200 scripts tests /tmp/v$T/ 2>/dev/null
  (cd /tmp/v$T && rm -rf build && make -C paper_2512_19536_b200/csrc -j16 BUILD=/tmp/v$T/build/csrc EXTRA_NVFLAGS=-DPDG_SWEEP_THREADS=$T > $R/$O/build_$T.log 2>&1)
done
run() { local dir=$1 name=$2 cfg=$3; shift 3; (cd $dir && env "$@" timeout 600 python scripts/c4_probe.py 2 $cfg > $R/$O/$name.txt 2>&1); }
for T in 64 128 256; do
  D=$R; [ $T != 128 ] && D=/tmp/v$T
  run $D t${T}_c4 config4
  run $D t${T}_c4_md4z4 config4 PDG_MD_RELAX=4 PDG_RELAX_Z=0.4
  run $D t${T}_c4_md6z5 config4 PDG_MD_RELAX=6 PDG_RELAX_Z=0.5
  run $D t${T}_c2 config2
  run $D t${T}_c5p2 config5:2
done
# lookahead-unit L2 prefetch (bit 8) on top of the default (3), and instead of it (10)
run $R pf11_c2 config2 PDG_SWEEP_PREFETCH=11
run $R pf10_c2 config2 PDG_SWEEP_PREFETCH=10
run $R pf11_c4 config4 PDG_SWEEP_PREFETCH=11
run $R pf10_c4 config4 PDG_SWEEP_PREFETCH=10
run $R pf11_c3p3 config3:3:64 PDG_SWEEP_PREFETCH=11
run $R pf3_c3p3 config3:3:64
# per-unit phase trace of one config4 sweep (HEAD defaults)
(cd $R && timeout 900 python scripts/sweep_trace.py config4 > $R/$O/trace_c4.txt 2>&1)
# SpMV kernel choice at config4 (warp-per-row forced)
run $R spmvwarp_c4 config4 PDG_SPMV_WARP=1
