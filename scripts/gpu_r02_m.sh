#!/bin/bash
# r02 batch M: pipelined warp-specialised sweep (PDG_SWEEP=pipe): correctness, then config4/2/5 A/B
O=gpurun_out/r02m; mkdir -p $O
PDG_SWEEP=pipe timeout 900 python -m pytest tests -m gpu -q -x -k "not knob" > $O/pytest_gpu_pipe.log 2>&1; echo "rc=$?" >> $O/pytest_gpu_pipe.log
run() { local name=$1 cfg=$2; shift 2; env "$@" timeout 600 python scripts/c4_probe.py 2 $cfg > $O/$name.txt 2>&1; echo "rc=$?" >> $O/$name.txt; }
run cta_c4 config4
run pipe_c4 config4 PDG_SWEEP=pipe
run pipe_c4_u64 config4 PDG_SWEEP=pipe PDG_UNIT_KB=64
run pipe_c4_md4z4 config4 PDG_SWEEP=pipe PDG_MD_RELAX=4 PDG_RELAX_Z=0.4
run pipe_c4_md4z4_u64 config4 PDG_SWEEP=pipe PDG_MD_RELAX=4 PDG_RELAX_Z=0.4 PDG_UNIT_KB=64
run pipe_c4_md2z3 config4 PDG_SWEEP=pipe PDG_MD_RELAX=2 PDG_RELAX_Z=0.3
run pipe_c4_md2z3_u48 config4 PDG_SWEEP=pipe PDG_MD_RELAX=2 PDG_RELAX_Z=0.3 PDG_UNIT_KB=48
run cta_c2 config2
run pipe_c2 config2 PDG_SWEEP=pipe
run cta_c5p2 config5:2
run pipe_c5p2 config5:2 PDG_SWEEP=pipe
