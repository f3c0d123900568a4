# A/B of sweep variants: bench (no CPU leg) + sweep trace per env setting.
# usage: bash scripts/gpu_cmp.sh TAG "ENV1" "ENV2" ...
mkdir -p gpurun_out
tag=$1; shift
python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo pytest=$?
for e in "$@"; do
  n=$(echo "$e" | tr ' =' '__')
  env $e python bench.py --steps 100 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_bench_$n.log 2>&1; echo "$e bench=$?"
  env $e python scripts/sweep_trace.py config2 > gpurun_out/${tag}_trace_$n.log 2>&1; echo "$e trace=$?"
done
