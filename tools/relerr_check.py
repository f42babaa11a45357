"""Compare the GPU error pass (W panel and two panels) with the reference's relative_error."""
import os, subprocess, sys, time
sys.path.insert(0, '.')
import numpy as np
from paper_1710_03608_b200 import datagen as g

CASES = [("traffic_1k", lambda: g.traffic([1000, 1000, 40], 150000, 21), 400),
         ("traffic_2k", lambda: g.traffic([2000, 2000, 50], 400000, 22), 800),
         ("c4", lambda: g.c4(seed=4, scale_j=300, scale_k=30), 300)]
which = sys.argv[1] if len(sys.argv) > 1 else "all"
if which == "ref":
    from oracle.bindings import Ref
    R = Ref()
    for name, mk, s in CASES:
        x = mk()
        t = R.tensor(x.shape, x.flat_idx(), x.val)
        t0 = time.time()
        fe = R.ctd_s(t, 0, s, 1e-6, 42, error=True)
        print(name, "ref", repr(fe.extra["relative_error"]), "kept", len(fe.kept_flat), "%.1fs" % (time.time() - t0), flush=True)
else:
    import paper_1710_03608_b200 as ctd
    ctx = ctd.Context(0)
    for name, mk, s in CASES:
        x = mk()
        f = ctd.ctd_s(ctd.SparseTensor.from_datagen(x), 0, s, 1e-6, 42, with_error=True, ctx=ctx)
        print(name, os.environ.get("CTD_RELERR_TWO_PANELS", "W"), repr(f.relative_error), "kept", f.kept_count(), flush=True)
