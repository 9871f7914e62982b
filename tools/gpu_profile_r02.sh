# round-2 evidence: c5 tc_scan full capture, bench launch list (c5), c2 launch list
export FC_BENCH_REPS=1
timeout 300 python tools/bench_level.py c5 2:65536 > gpurun_out/c5_level.txt 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:tc_scan_kernel -c 1 -f -o gpurun_out/tc_scan_c5_r02 python tools/bench_level.py c5 2:65536 > gpurun_out/ncu_c5_r02.log 2>&1; echo "ncu c5 rc=$?"
timeout 600 python bench.py --workload c5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/c5_plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_c5.csv python bench.py --workload c5 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "launches c5 rc=$?"
timeout 300 python bench.py --workload c2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/c2_plain.json 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_c2.csv python bench.py --workload c2 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "launches c2 rc=$?"
