# ncu --set full of the mid-size kernels of one c2 encode (one launch each).
python __graft_entry__.py
timeout 300 python tools/prof_c2.py c2 > /dev/null 2>&1 || echo "plain failed"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"survivors_all|gather_build|build_b|chunk_sort|qprep_multi|reach_scatter|scan_jobs|classify|chunk_pair" -s 40 -c 14 -o gpurun_out/small python tools/prof_c2.py c2 > gpurun_out/ncu_small.log 2>&1; echo "ncu rc=$?"
