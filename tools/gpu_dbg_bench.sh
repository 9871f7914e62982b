timeout 300 python -X faulthandler bench.py --workload c2 --steps 2 --warmup 3 --no-cpu-baseline --shard images > gpurun_out/dbg_img.json 2> gpurun_out/dbg_img.err; echo img rc=$?
timeout 300 python -X faulthandler bench.py --workload c2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/dbg_rng.json 2> gpurun_out/dbg_rng.err; echo rng rc=$?
tail -40 gpurun_out/dbg_img.err gpurun_out/dbg_rng.err
