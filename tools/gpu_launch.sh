python __graft_entry__.py
timeout 300 python tools/prof_c2.py c2 > gpurun_out/prof_c2_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/prof_c2.py c2 > gpurun_out/ncu_c2.log 2>&1; echo "ncu rc=$?"
cat gpurun_out/prof_c2_plain.log
