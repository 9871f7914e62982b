python __graft_entry__.py
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
FC_FIX_FUSED=0 timeout 900 python -m pytest tests -m gpu -q -x -k "encode_c2 or matcher or levelwise" 2>&1 | tail -1
for v in 1 0 1 0; do FC_FIX_FUSED=$v TAG="fused=$v" timeout 300 python tools/step_time.py c2 150 2>&1 | tail -1; done
timeout 300 python tools/bench_level.py c2 2>&1 | tail -3
FC_BENCH_REPS=3 timeout 600 python tools/bench_level.py c4 1:16384 2:64360 3:14796 2>&1 | tail -3
