for m in 0 1 2; do echo "debug_mode=$m"; FC_TC_DEBUG_MODE=$m timeout 120 python tools/bench_level.py 10; done
