#!/bin/bash
# r02 batch 1: config4 bench (both arms) + large-config parity runs
set -x
mkdir -p gpurun_out/r02b1
python bench.py --steps 3 --warmup 3 > gpurun_out/r02b1/bench_c4.json 2> gpurun_out/r02b1/bench_c4.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02b1/bench_ref_c4.json 2> gpurun_out/r02b1/bench_ref_c4.err
export PARITY_OUT=gpurun_out/r02b1/parity.jsonl
python scripts/parity_large.py c4 3 > gpurun_out/r02b1/par_c4.log 2>&1
python scripts/parity_large.py c5 4 > gpurun_out/r02b1/par_c5p4.log 2>&1
for p in 1 2 3 4; do for S in 64 256; do
  [ "$p$S" = "164" ] && continue
  python scripts/parity_large.py c3 $p $S > gpurun_out/r02b1/par_c3_p${p}_S${S}.log 2>&1
done; done
