# Factor-ordering knobs on the GPU: C2 bench + C3 (p=3, S=64) probe per env.
#   bash scripts/gpu_order_env.sh TAG "ENV1" "ENV2" ...
mkdir -p gpurun_out
tag=$1; shift
for e in "$@"; do
  n=$(echo "$e" | tr ' =' '__')
  env $e timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_bench_$n.log 2>&1
  env $e timeout 300 python scripts/c4_probe.py 8 config3:3:64 > gpurun_out/${tag}_c3_$n.log 2>&1
  python - "$e" gpurun_out/${tag}_bench_$n.log gpurun_out/${tag}_c3_$n.log <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1]); r = d["roofline"]
    c = [json.loads(l) for l in open(sys.argv[3]).read().strip().splitlines()]
    print(f"{sys.argv[1]:40s} C2 {d['value']:.4g} sweep_us {r['launch_ms']*1e3:.1f} GB/s {r['kernels']['sweep']['GB/s']:.0f} | C3p3 factor_gb {c[0]['factor_gb']} tasks {c[0]['tasks']} its {c[-1]['iterations'][-1]} DOF-it/s {c[-1]['dof_iter_per_s']:.4g} sweep_ms {c[-1]['sweep_live_ms']} GB/s {c[-1]['sweep_GBs']}")
except Exception as ex:
    print(sys.argv[1], "FAILED", ex)
PY
done
