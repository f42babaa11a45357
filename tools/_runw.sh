python tools/c2_trace.py 3 2>&1 | tail -1
CTD_FILTER_TRACE=1 python tools/c2_trace.py 1 2>&1 | grep "cycles/cand"
CTD_NO_WPANEL=1 python tools/c2_trace.py 3 2>&1 | tail -1
CTD_NO_WPANEL=1 CTD_FILTER_TRACE=1 python tools/c2_trace.py 1 2>&1 | grep "cycles/cand"
