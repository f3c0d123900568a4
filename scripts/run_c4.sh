# config 4 (1,048,576 cells, p=3, 512 subdomains) on one GPU: setup time, memory, steps
mkdir -p gpurun_out
free -g | head -2; nproc
timeout 2400 python scripts/c4_probe.py ${1:-5} config4 > gpurun_out/c4_probe.log 2>&1
echo probe=$?
tail -12 gpurun_out/c4_probe.log
