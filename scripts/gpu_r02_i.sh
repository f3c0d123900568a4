#!/bin/bash
# r02 batch I: config3 parity against the CPU oracle, all 8 (p, S) rows over the full 50 CN steps
O=gpurun_out/r02i; mkdir -p $O
export PARITY_OUT=$O/parity.jsonl
for p in 1 2 3 4; do for S in 64 256; do
  timeout 1500 python scripts/parity_large.py c3 $p $S > $O/par_c3_p${p}_S${S}.log 2>&1; echo "rc=$?" >> $O/par_c3_p${p}_S${S}.log
done; done
