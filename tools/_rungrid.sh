for g in "$@"; do
  echo "== grid $g"
  CTD_FILTER_GRID=$g python tools/c2_trace.py 2 2>&1 | tail -1
  CTD_FILTER_GRID=$g CTD_FILTER_TRACE=1 python tools/c2_trace.py 1 2>&1 | grep -E "cycles/cand|cand 1264" | cut -c1-300
done
