timeout 120 tools/microbench/tmem_bw > gpurun_out/tmem_bw.log 2>&1; echo "tmem rc=$?"; cat gpurun_out/tmem_bw.log
timeout 120 tools/microbench/mma_rate > gpurun_out/mma_rate.log 2>&1; echo "mma rc=$?"; cat gpurun_out/mma_rate.log
