# bench alternative builds of the library: bash scripts/gpu_bench_libs.sh TAG lib1.so lib2.so ...
tag=$1; shift
cp paper_2512_19536_b200/libpolydg_b200.so /tmp/lib_orig.so
for l in "$@"; do
  cp "$l" paper_2512_19536_b200/libpolydg_b200.so
  n=$(basename "$l" .so)
  python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_bench_$n.log 2>&1
  python - "$n" gpurun_out/${tag}_bench_$n.log <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1]); r = d["roofline"]
    print(f"LIB {sys.argv[1]:30s} value {d['value']:.4g} sweep_us {r['launch_ms']*1e3:.1f} GB/s {r['kernels']['sweep']['GB/s']:.0f}")
except Exception as ex:
    print(sys.argv[1], "FAILED", ex)
PY
done
cp /tmp/lib_orig.so paper_2512_19536_b200/libpolydg_b200.so
