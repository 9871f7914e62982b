# One development iteration on the GPU box: parity tests, timings, launch list.
python __graft_entry__.py
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log | grep -v "^$"
FC_REPS=3 timeout 300 python tools/time_encode.py ${FC_WL:-c2 c4 c5} 2>&1 | grep -E "it2|phases|level"
timeout 300 python tools/prof_c2.py c2 > gpurun_out/prof_c2_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/prof_c2.py c2 > gpurun_out/ncu_c2.log 2>&1; echo "ncu rc=$?"
