python __graft_entry__.py
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -20 gpurun_out/smoke.log
timeout 600 python -m pytest tests -m gpu -q -x -k "tensor" > gpurun_out/pytest_tc.log 2>&1; echo "pytest tc rc=$?"
tail -30 gpurun_out/pytest_tc.log
FC_PATH=tensor timeout 300 python tools/time_encode.py c1 c2 c4 > gpurun_out/time_tc.log 2>&1; echo "time rc=$?"
cat gpurun_out/time_tc.log | tail -20
