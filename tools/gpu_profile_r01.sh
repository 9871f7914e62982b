# Full ncu captures of the dominant kernels of the c2 encode (third encode of prof_c2.py).
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tc_scan_kernel --launch-skip 6 -c 3 -o gpurun_out/tc_scan_c2_full python tools/prof_c2.py c2 > gpurun_out/ncu_tc_full.log 2>&1; echo full_rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:entropy_all_kernel --launch-skip 2 -c 1 -o gpurun_out/entropy_c2_full python tools/prof_c2.py c2 > gpurun_out/ncu_ent_full.log 2>&1; echo full2_rc=$?
