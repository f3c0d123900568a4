# config 4 (1,048,576 cells, p=3, 512 subdomains) on one GPU: setup time, memory, bench line
mkdir -p gpurun_out
free -g; nproc; nvidia-smi --query-gpu=memory.total --format=csv
/usr/bin/time -v timeout 2000 python bench.py --config config4 --steps 10 --warmup 2 --no-cpu-baseline > gpurun_out/c4_bench.log 2> gpurun_out/c4_bench.err
echo bench=$?
tail -25 gpurun_out/c4_bench.err
