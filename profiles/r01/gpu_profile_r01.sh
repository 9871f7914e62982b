# Round-1 evidence: bench line + reference arm, launch lists, full ncu of the contraction,
python __graft_entry__.py
# per-level timings and the encode timeline.
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench=$?
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>/dev/null; echo ref=$?
timeout 300 python tools/bench_level.py c2 > gpurun_out/levels_c2.txt 2>&1
FC_BENCH_REPS=3 timeout 600 python tools/bench_level.py c4 1:16384 2:64360 3:14796 > gpurun_out/levels_c4.txt 2>&1
FC_BENCH_REPS=3 timeout 600 python tools/bench_level.py c5 2:65536 > gpurun_out/levels_c5.txt 2>&1
FC_TRACE=1 FC_REPS=3 timeout 300 python tools/time_encode.py c2 > gpurun_out/trace_c2.txt 2>&1
FC_TRACE=2 FC_REPS=4 timeout 300 python tools/time_encode.py c2 > gpurun_out/trace2_c2.txt 2>&1
FC_REPS=2 timeout 600 python tools/time_encode.py c1 c2 c3 c4 c5 > gpurun_out/encode_all.txt 2>&1
timeout 600 python tools/prof_c2.py c2 > /dev/null 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/prof_c2.py c2 > /dev/null 2>&1; echo l=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_c2.csv python bench.py --steps 3 --warmup 3 > /dev/null 2>&1; echo lb=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tc_scan_kernel --launch-skip 6 -c 3 -o gpurun_out/tc_scan_c2_full python tools/prof_c2.py c2 > /dev/null 2>&1; echo f=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:entropy_all_kernel --launch-skip 2 -c 1 -o gpurun_out/entropy_c2_full python tools/prof_c2.py c2 > /dev/null 2>&1; echo f2=$?
