python __graft_entry__.py
FC_PATH=tensor FC_REPS=2 timeout 300 python tools/time_encode.py c5 2>&1 | grep "'level': 2"
FC_TC_DEBUG_MODE=1 FC_PATH=tensor FC_REPS=2 timeout 300 python tools/time_encode.py c5 2>&1 | grep "'level': 2"
