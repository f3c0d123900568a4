set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_e.log 2>&1; echo pytest=$?
python bench.py > gpurun_out/bench_e.log 2> gpurun_out/bench_e.err; echo bench=$?
PDG_NO_GRAPH=1 python scripts/profile_step.py config2 2 > gpurun_out/plain_e.log 2>&1; echo plain=$?
PDG_NO_GRAPH=1 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_r01e.csv python scripts/profile_step.py config2 2 > gpurun_out/ncu_e1.log 2>&1; echo ncu1=$?
PDG_NO_GRAPH=1 ncu --set full --clock-control none --import-source on -k regex:sweep -s 20 -c 1 -o gpurun_out/sweep_r01e python scripts/profile_step.py config2 2 > gpurun_out/ncu_e2.log 2>&1; echo ncu2=$?
PDG_NO_GRAPH=1 ncu --set full --clock-control none --import-source on -k regex:spmv -s 20 -c 1 -o gpurun_out/spmv_r01e python scripts/profile_step.py config2 2 > gpurun_out/ncu_e3.log 2>&1; echo ncu3=$?
