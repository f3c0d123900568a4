# Probe one config under several env settings (scripts/c4_probe.py summary per env).
#   bash scripts/gpu_probe_env.sh TAG CONFIG STEPS "ENV1" "ENV2" ...   (CONFIG e.g. config3:3:64)
mkdir -p gpurun_out
tag=$1; cfg=$2; steps=$3; shift 3
for e in "$@"; do
  n=$(echo "$e $cfg" | tr ' =:' '___')
  env $e timeout 900 python scripts/c4_probe.py $steps $cfg > gpurun_out/${tag}_$n.log 2>&1
  python - "$e" "$cfg" gpurun_out/${tag}_$n.log <<'PY'
import json, sys
try:
    c = [json.loads(l) for l in open(sys.argv[3]).read().strip().splitlines() if l.startswith("{")]
    print(f"{sys.argv[2]:14s} {sys.argv[1]:32s} setup {c[0]['setup_s']}s factor_gb {c[0]['factor_gb']} its {c[-1]['iterations']} DOF-it/s {c[-1]['dof_iter_per_s']:.4g} sweep_ms {c[-1]['sweep_live_ms']} GB/s {c[-1]['sweep_GBs']}", flush=True)
except Exception as ex:
    print(sys.argv[1], sys.argv[2], "FAILED", ex, open(sys.argv[3]).read()[-500:])
PY
done
