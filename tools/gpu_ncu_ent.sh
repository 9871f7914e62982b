# ncu --set full (source) of the entropy kernel in one c2 encode.
python __graft_entry__.py
timeout 600 ncu --set full --import-source on --clock-control none -k regex:entropy_all -s 1 -c 1 -o gpurun_out/ent python tools/prof_c2.py c2 > gpurun_out/ncu_ent.log 2>&1; echo "ncu rc=$?"
