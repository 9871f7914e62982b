python __graft_entry__.py
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
FC_PATH=tensor FC_REPS=2 timeout 300 python tools/time_encode.py c1 c2 c4 c5 > gpurun_out/time_tc.log 2>&1; echo "time rc=$?"
cat gpurun_out/time_tc.log | tail -30
