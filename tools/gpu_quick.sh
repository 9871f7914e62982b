# Parity tests, per-level timings (c2, c4, c5 L2) and the c2 launch list.
python __graft_entry__.py
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python tools/bench_level.py c2 2>&1 | tail -3
FC_BENCH_REPS=3 timeout 300 python tools/bench_level.py c4 1:16384 2:64360 3:14796 2>&1 | tail -3
FC_BENCH_REPS=3 timeout 600 python tools/bench_level.py c5 2:65536 2>&1 | tail -1
timeout 300 python tools/prof_c2.py c2 > /dev/null 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/prof_c2.py c2 > /dev/null 2>&1; echo "ncu rc=$?"
