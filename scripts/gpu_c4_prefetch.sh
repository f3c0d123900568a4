# config4 sweep: L2 prefetch and unit size A/B (ncu showed DRAM reads 1.27x the panel bytes)
mkdir -p gpurun_out/r01v
for v in "1 0" "0 0" "1 44" "0 44" "1 0"; do
  set -- $v
  if [ "$2" = "0" ]; then unset PDG_UNIT_KB; else export PDG_UNIT_KB=$2; fi
  PDG_SWEEP_PREFETCH=$1 timeout 600 python scripts/c4_probe.py 2 config4 > gpurun_out/r01v/c4_pf$1_kb$2.txt 2>&1
  echo "prefetch=$1 unit_kb=$2 rc=$? $(tail -1 gpurun_out/r01v/c4_pf$1_kb$2.txt)"
done
