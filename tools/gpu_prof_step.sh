# Step breakdown: FC_TRACE timeline of c2 encodes and the ncu launch list of three encodes.
python __graft_entry__.py
FC_TRACE=1 FC_REPS=3 timeout 300 python tools/time_encode.py c2 > gpurun_out/trace_c2.txt 2>&1; echo "trace rc=$?"
timeout 300 python tools/prof_c2.py c2 > gpurun_out/prof_c2_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/prof_c2.py c2 > gpurun_out/ncu_c2.log 2>&1; echo "ncu rc=$?"
