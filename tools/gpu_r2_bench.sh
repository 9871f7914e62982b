nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python bench.py --workload c5 --steps 5 --warmup 3 > gpurun_out/c5_bench.json 2> gpurun_out/c5_bench.err; echo c5 rc=$?
timeout 300 python bench.py --workload c2 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/c2_bench.json 2> gpurun_out/c2_bench.err; echo c2 rc=$?
timeout 600 python bench.py --workload c5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/c5_plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python bench.py --workload c5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c5.log 2>&1; echo ncu rc=$?
