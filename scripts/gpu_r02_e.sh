#!/bin/bash
# r02 batch E: ordering / amalgamation / row-alignment sweep with evict-first panel loads (default now)
O=gpurun_out/r02e; mkdir -p $O
run() {  # name, config, env...
  local name=$1 cfg=$2; shift 2
  env "$@" timeout 600 python scripts/c4_probe.py 2 $cfg > $O/$name.txt 2>&1; echo "rc=$?" >> $O/$name.txt
}
run c4_md8z5 config4 PDG_ORDER=md PDG_MD_RELAX=8 PDG_RELAX_Z=0.5
run c4_md8z5_a2 config4 PDG_ORDER=md PDG_MD_RELAX=8 PDG_RELAX_Z=0.5 PDG_ROW_ALIGN=2
run c4_md8z5_a4 config4 PDG_ORDER=md PDG_MD_RELAX=8 PDG_RELAX_Z=0.5 PDG_ROW_ALIGN=4
run c4_md6z4 config4 PDG_ORDER=md PDG_MD_RELAX=6 PDG_RELAX_Z=0.4
run c4_md10z5 config4 PDG_ORDER=md PDG_MD_RELAX=10 PDG_RELAX_Z=0.5
run c4_md8z3 config4 PDG_ORDER=md PDG_MD_RELAX=8 PDG_RELAX_Z=0.3
run c4_md12z3 config4 PDG_ORDER=md PDG_MD_RELAX=12 PDG_RELAX_Z=0.3
run c4_md8z5_u64 config4 PDG_ORDER=md PDG_MD_RELAX=8 PDG_RELAX_Z=0.5 PDG_UNIT_KB=64
run c4_md8z5_u128 config4 PDG_ORDER=md PDG_MD_RELAX=8 PDG_RELAX_Z=0.5 PDG_UNIT_MAX_KB=128 PDG_UNIT_KB=128
run c2_nd config2
run c2_md4z3 config2 PDG_ORDER=md PDG_MD_RELAX=4 PDG_RELAX_Z=0.3
run c2_md8z5 config2 PDG_ORDER=md PDG_MD_RELAX=8 PDG_RELAX_Z=0.5
run c2_md12z5 config2 PDG_ORDER=md PDG_MD_RELAX=12 PDG_RELAX_Z=0.5
run c2_md16z6 config2 PDG_ORDER=md PDG_MD_RELAX=16 PDG_RELAX_Z=0.6
run c5p2_nd config5:2
run c5p2_md8z5 config5:2 PDG_ORDER=md PDG_MD_RELAX=8 PDG_RELAX_Z=0.5
run c5p2_md12z5 config5:2 PDG_ORDER=md PDG_MD_RELAX=12 PDG_RELAX_Z=0.5
run c5p4_nd config5:4
run c5p4_md8z5 config5:4 PDG_ORDER=md PDG_MD_RELAX=8 PDG_RELAX_Z=0.5
run c3p3s64_nd config3:3:64
run c3p3s64_md8z5 config3:3:64 PDG_ORDER=md PDG_MD_RELAX=8 PDG_RELAX_Z=0.5
run c3p1s256_nd config3:1:256
run c3p1s256_md8z5 config3:1:256 PDG_ORDER=md PDG_MD_RELAX=8 PDG_RELAX_Z=0.5
