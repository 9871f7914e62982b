timeout 300 python tools/shist_once.py c2 > gpurun_out/shist_once.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tc_scan_kernel -s 1 -c 1 -f -o gpurun_out/tc_real_c2 python tools/shist_once.py c2 > gpurun_out/ncu_real.log 2>&1; echo "ncu rc=$?"
