#!/bin/bash
# r02 batch K: full GPU suite (device assembly + knobs), bench with device assembly, setup timing
O=gpurun_out/r02k; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
PDG_SETUP_TIMES=1 timeout 600 python scripts/c4_probe.py 1 config4 > $O/c4_setup.txt 2>&1
