# ncu --set full (source) of the c4 level-2 contraction (steady state epilogue).
python __graft_entry__.py
FC_BENCH_REPS=1 timeout 300 python tools/bench_level.py c4 2:64360 > /dev/null 2>&1 || echo "plain failed"
FC_BENCH_REPS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:tc_scan_kernel -s 0 -c 1 -o gpurun_out/tc_c4l2 python tools/bench_level.py c4 2:64360 > gpurun_out/ncu_c4l2.log 2>&1; echo "ncu rc=$?"
