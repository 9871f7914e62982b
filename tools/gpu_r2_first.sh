set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python bench.py --workload c5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c5_bench0.json 2> gpurun_out/c5_bench0.err
echo rc=$?
timeout 300 python bench.py --workload c2 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/c2_bench0.json 2> gpurun_out/c2_bench0.err
echo rc=$?
