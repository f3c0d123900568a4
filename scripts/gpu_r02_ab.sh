#!/bin/bash
# r02 batch AB (bottom levels on by default): large-config parity against the CPU oracle (config4 3 CN steps, config5 p=2 / p=4 one solve)
O=gpurun_out/r02ab; mkdir -p $O
export PARITY_OUT=$O/parity.jsonl
nproc > $O/nproc.txt; free -g > $O/free.txt
timeout 2700 python scripts/parity_large.py c4 3 > $O/par_c4.log 2>&1; echo "rc=$?" >> $O/par_c4.log
timeout 1500 python scripts/parity_large.py c5 2 > $O/par_c5p2.log 2>&1; echo "rc=$?" >> $O/par_c5p2.log
timeout 2700 python scripts/parity_large.py c5 4 > $O/par_c5p4.log 2>&1; echo "rc=$?" >> $O/par_c5p4.log
