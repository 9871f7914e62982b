# ncu --set full of one level-3 contraction launch: current tree vs _ab_old.
export FC_BENCH_REPS=2
timeout 300 python tools/bench_level.py c2 3:2420 > /dev/null 2>&1 || echo "plain run failed"
timeout 600 ncu --set full --clock-control none -k regex:tc_scan_kernel -s 1 -c 1 -o gpurun_out/tc_L3_new python tools/bench_level.py c2 3:2420 > gpurun_out/ncu_new.log 2>&1; echo "ncu new rc=$?"
(cd _ab_old && timeout 600 ncu --set full --clock-control none -k regex:tc_scan_kernel -s 1 -c 1 -o ../gpurun_out/tc_L3_old python tools/bench_level.py c2 3:2420 > ../gpurun_out/ncu_old.log 2>&1; echo "ncu old rc=$?")
