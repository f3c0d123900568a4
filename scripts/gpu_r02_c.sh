#!/bin/bash
# r02 batch C: ordering A/B at config4 (ND vs minimum degree), prefetch A/B, DRAM bytes per sweep
O=gpurun_out/r02c; mkdir -p $O
PDG_ORDER=md timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu_md.log 2>&1; echo "pytest md rc=$?" >> $O/pytest_gpu_md.log
run() {  # name, env...
  local name=$1; shift
  env "$@" timeout 600 python scripts/c4_probe.py 2 config4 > $O/c4_$name.txt 2>&1; echo "rc=$?" >> $O/c4_$name.txt
  env "$@" PDG_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_ltcfabric.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum \
     --clock-control none -k regex:sweep_kernel -s 20 -c 3 --csv python scripts/c4_probe.py 1 config4 > $O/ncu_$name.csv 2>&1
}
run nd
run nd_nopf PDG_SWEEP_PREFETCH=0
run md PDG_ORDER=md
run md_nopf PDG_ORDER=md PDG_SWEEP_PREFETCH=0
run md_r4 PDG_ORDER=md PDG_MD_RELAX=4
run md_r8z5 PDG_ORDER=md PDG_MD_RELAX=8 PDG_RELAX_Z=0.5
