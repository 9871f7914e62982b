python __graft_entry__.py
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
FC_PATH=tensor FC_REPS=2 timeout 300 python tools/time_encode.py c2 c4 c5 > gpurun_out/time_tc.log 2>&1; echo "time rc=$?"
cat gpurun_out/time_tc.log | tail -30
timeout 300 python tools/prof_tc.py c4 > gpurun_out/prof_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_scan -s 1 -c 1 -o gpurun_out/prof_tc_c4_v12 python tools/prof_tc.py c4 > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/ncu.log
