FC_BENCH_REPS=3 timeout 300 python tools/bench_level.py c5 2:65536 2>&1 | tail -1
FC_BENCH_REPS=5 timeout 300 python tools/bench_level.py c2 2>&1 | tail -3
