# bench-only sweep over env settings (no traces): bash scripts/gpu_bench_env.sh TAG "ENV1" "ENV2" ...
mkdir -p gpurun_out
tag=$1; shift
for e in "$@"; do
  n=$(echo "$e" | tr ' =' '__')
  env $e python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_bench_$n.log 2>&1
  python - "$e" gpurun_out/${tag}_bench_$n.log <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1]); r = d["roofline"]
    print(f"{sys.argv[1]:60s} value {d['value']:.4g} sweep_us {r['launch_ms']*1e3:.1f} GB/s {r['kernels']['sweep']['GB/s']:.0f} update_us {r['kernels']['update']['ms']*1e3:.1f} prolong_us {r['kernels']['prolong_dot']['ms']*1e3:.1f}")
except Exception as ex:
    print(sys.argv[1], "FAILED", ex)
PY
done
