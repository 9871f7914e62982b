python __graft_entry__.py
timeout 900 python -m pytest tests -m gpu -q -k "not tensor" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python tools/time_exact.py c1 c2 c4 > gpurun_out/time_exact.log 2>&1; echo "time rc=$?"
cat gpurun_out/time_exact.log
