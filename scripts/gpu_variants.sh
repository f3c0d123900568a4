# A/B of prebuilt library variants (variants/NAME/libpolydg_b200.so, built with
# EXTRA_NVFLAGS): C2 bench + one probe config per variant.
#   bash scripts/gpu_variants.sh TAG CONFIG STEPS base NAME1 NAME2 ...
mkdir -p gpurun_out
tag=$1; cfg=$2; steps=$3; shift 3
cp paper_2512_19536_b200/libpolydg_b200.so /tmp/base_lib.so
for v in "$@"; do
  if [ "$v" = base ]; then cp /tmp/base_lib.so paper_2512_19536_b200/libpolydg_b200.so; else cp variants/$v/libpolydg_b200.so paper_2512_19536_b200/libpolydg_b200.so; fi
  timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_bench_$v.log 2>&1
  python -c "
import json,sys
try:
    d=json.loads(open('gpurun_out/${tag}_bench_$v.log').read().strip().splitlines()[-1]); r=d['roofline']
    print('$v', 'C2', '%.4g' % d['value'], 'sweep_us %.1f' % (r['launch_ms']*1e3), 'GB/s %.0f' % r['kernels']['sweep']['GB/s'], flush=True)
except Exception as e: print('$v C2 FAILED', e)
"
  bash scripts/gpu_probe_env.sh ${tag}_$v $cfg $steps "V=$v"
done
cp /tmp/base_lib.so paper_2512_19536_b200/libpolydg_b200.so
