python __graft_entry__.py
FC_REPS=3 timeout 300 python tools/time_encode.py c2 c1 2>&1 | grep -E "it2|phases"
