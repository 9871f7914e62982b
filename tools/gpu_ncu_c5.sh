export FC_BENCH_REPS=1
OUT=${1:-tc_scan_c5_full}
timeout 300 python tools/bench_level.py c5 2:65536 > gpurun_out/c5_level.txt 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:tc_scan_kernel -c 1 -f -o gpurun_out/$OUT python tools/bench_level.py c5 2:65536 > gpurun_out/ncu_c5_full.log 2>&1; echo ncu rc=$?
cat gpurun_out/c5_level.txt
