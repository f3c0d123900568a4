#!/bin/bash
# r02 batch AA: lookahead fetch beside the gather; b = 6 variants; config-5 probes with the coarse solve's span
O=gpurun_out/r02aa; mkdir -p $O
PDG_BOTTOM_KB=64 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_tuning_knobs.py -m gpu -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
run() { local name=$1 cfg=$2; shift 2; env PDG_SETUP_TIMES=1 "$@" timeout 600 python scripts/c4_probe.py 3 $cfg > $O/$name.txt 2>&1; echo "rc=$?" >> $O/$name.txt; }
run c4 config4
timeout 500 python scripts/chunk_trace.py config4 > $O/trace_c4.txt 2>&1
run c5p4 config5:4
run c5p2_off config5:2
run c5p2_r1_t128 config5:2 PDG_BOTTOM_KB=160 PDG_MD_RELAX=1 PDG_SWEEP_THREADS=128
run c5p2_r1_t64 config5:2 PDG_BOTTOM_KB=160 PDG_MD_RELAX=1
run c5p2_r2_t128 config5:2 PDG_BOTTOM_KB=160 PDG_MD_RELAX=2 PDG_SWEEP_THREADS=128
timeout 900 python scripts/c5_probe.py 2 > $O/c5_probe_p2.txt 2>&1
timeout 900 python scripts/c5_probe.py 4 > $O/c5_probe_p4.txt 2>&1
