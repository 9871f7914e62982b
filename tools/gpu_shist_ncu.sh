timeout 300 python tools/shist_once.py c2 > gpurun_out/shist_once.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_shist_tc.csv python tools/shist_once.py c2 > /dev/null 2>&1
FC_REAL_CUDA_CORES=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_shist_dp4a.csv python tools/shist_once.py c2 > /dev/null 2>&1
echo done
