set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --workload c5 --steps 5 --warmup 3 > gpurun_out/c5_bench.json 2> gpurun_out/c5_bench.err; echo c5 rc=$?
timeout 300 python bench.py --workload c2 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/c2_bench.json 2> gpurun_out/c2_bench.err; echo c2 rc=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref_bench.json 2> gpurun_out/ref_bench.err; echo ref rc=$?
