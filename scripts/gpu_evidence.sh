# Fresh evidence across the BASELINE configs on one B200 (each run bounded by
# its own timeout):  bash scripts/gpu_evidence.sh TAG
tag=${1:-r01}
mkdir -p gpurun_out/$tag
nproc > gpurun_out/$tag/nproc.txt
PDG_SETUP_TIMES=1 timeout 900 python scripts/c5_probe.py 2 > gpurun_out/$tag/config5_p2_probe.txt 2>&1; echo c5p2=$?
PDG_SETUP_TIMES=1 timeout 1200 python scripts/c5_probe.py 4 > gpurun_out/$tag/config5_p4_probe.txt 2>&1; echo c5p4=$?
timeout 1500 python scripts/c3_study.py gpurun_out/$tag/config3 > gpurun_out/$tag/config3_study.txt 2>&1; echo c3=$?
timeout 1500 python scripts/parity_full.py config1 > gpurun_out/$tag/parity_config1_full.txt 2>&1; echo parity1=$?
timeout 2400 python scripts/parity_full.py config2 > gpurun_out/$tag/parity_config2_full.txt 2>&1; echo parity2=$?
