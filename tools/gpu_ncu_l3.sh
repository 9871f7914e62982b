# ncu --set full (with source) of one contraction launch per level of c2.
export FC_BENCH_REPS=2
timeout 300 python tools/bench_level.py c2 3:2420 2:1884 > /dev/null 2>&1 || echo "plain run failed"
for L in ${FC_NCU_LEVELS:-3:2420 2:1884}; do
  n=${L%%:*}
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:tc_scan_kernel -s 1 -c 1 -o gpurun_out/tc_L${n} python tools/bench_level.py c2 $L > gpurun_out/ncu_L${n}.log 2>&1; echo "ncu L$n rc=$?"
done
