# One round of GPU evidence: tests, the bench line, a sweep trace, the ncu
# launch list and full captures of the top kernels (each ncu pass only after
# the same command ran clean without ncu).   bash scripts/gpu_round.sh TAG
set -x
tag=${1:-r01}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$tag.log 2>&1; echo pytest=$?
timeout 600 python bench.py > gpurun_out/bench_$tag.log 2> gpurun_out/bench_$tag.err; echo bench=$?
timeout 200 python scripts/sweep_trace.py > gpurun_out/sweep_trace_$tag.log 2>&1; echo trace=$?
PDG_NO_GRAPH=1 timeout 200 python scripts/profile_step.py config2 2 > gpurun_out/plain_$tag.log 2>&1; echo plain=$?
PDG_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_$tag.csv python scripts/profile_step.py config2 2 > gpurun_out/ncu1_$tag.log 2>&1; echo ncu1=$?
for k in sweep spmv_warp update_restrict prolong; do
  PDG_NO_GRAPH=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 20 -c 1 -o gpurun_out/${k}_$tag python scripts/profile_step.py config2 2 > gpurun_out/ncu_${k}_$tag.log 2>&1; echo ncu_$k=$?
done
