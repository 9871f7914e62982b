# build-measure iteration: GPU parity suite, then per-level contraction timings
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
FC_BENCH_REPS=5 timeout 300 python tools/bench_level.py c2 2>&1 | tail -3
FC_MODE=baseline FC_BENCH_REPS=3 timeout 300 python tools/bench_level.py c2 2>&1 | tail -3
FC_MODE=baseline FC_PATH=exact FC_BENCH_REPS=2 timeout 300 python tools/bench_level.py c2 2>&1 | tail -3
FC_BENCH_REPS=2 timeout 300 python tools/bench_level.py c5 2:65536 2>&1 | tail -1
