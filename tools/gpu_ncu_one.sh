# ncu --set full (source) of one kernel (regex $1) in a c2 encode; report -> gpurun_out/one.ncu-rep
python __graft_entry__.py
timeout 300 python tools/prof_c2.py c2 > /dev/null 2>&1 || echo "plain failed"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$1" -s ${2:-0} -c 1 -o gpurun_out/one python tools/prof_c2.py c2 > gpurun_out/ncu_one.log 2>&1; echo "ncu rc=$?"
