# ncu --set full (source) of two kernels (regex $1, $2) of a c2 encode -> gpurun_out/one*.ncu-rep
python __graft_entry__.py
timeout 300 python tools/prof_c2.py c2 > /dev/null 2>&1 || echo "plain failed"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$1" -s ${3:-1} -c 1 -o gpurun_out/one1 python tools/prof_c2.py c2 > gpurun_out/ncu_one1.log 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$2" -s ${4:-3} -c 1 -o gpurun_out/one2 python tools/prof_c2.py c2 > gpurun_out/ncu_one2.log 2>&1; echo "ncu2 rc=$?"
