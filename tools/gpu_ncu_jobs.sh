# ncu --set full (source) of the clamp-correction jobs kernels of one c2 encode.
python __graft_entry__.py
timeout 300 python tools/prof_c2.py c2 > /dev/null 2>&1 || echo "plain failed"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"fix_pairs" -s 6 -c 3 -o gpurun_out/jobs python tools/prof_c2.py c2 > gpurun_out/ncu_jobs.log 2>&1; echo "ncu rc=$?"
