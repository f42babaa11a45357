"""Pin the relative error at BASELINE sizes: run the C restatement's front end
(oracle/ctd_oracle.c, itself pinned bit for bit to the compiled reference by
tests/test_oracle_pin.py) on the full C2 and C4 tensors, then evaluate
relative_error (evaluation.cpp:88-122) in double-double with
oracle/relerr_dd.c (cto_relerr_dd_full: |X|^2 - <U, N> + tr((U G - I) U N)).

    python tests/golden/make_relerr_golden.py [c2 c4 ...]

Writes tests/golden/relerr_golden.json: per case the input/factor hashes the
GPU test checks first (so the value is known to belong to the same R and U)
and the double-double numerator and |X|^2.  The reference's own relative_error
cannot run at these sizes (O(nnz(C) I_alpha)); relerr_dd.c is
checked against it on smaller cases by tests/test_relerr_oracle.py.
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.bindings import Port  # noqa: E402
from paper_1710_03608_b200 import datagen as g  # noqa: E402

CASES = {
    # name: (generator, c, eps, seed) -- the bench.py / BASELINE.json configs
    "c2": (lambda: g.traffic([10000, 10000, 1000], 10_000_000, 2), 2000, 1e-6, 42),
    "c4": (lambda: g.c4(seed=4), 5000, 1e-6, 42),
    "c2x0.1": (lambda: g.c2(seed=2, scale=0.1), 2000, 1e-6, 42),
}
OUT = os.path.join(HERE, "relerr_golden.json")


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main(names):
    P = Port()
    out = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for name in names:
        make, s, eps, seed = CASES[name]
        x = make()
        t0 = time.time()
        fe = P.frontend(x.shape, x.flat_idx(), x.val, 0, s, eps, seed)
        t1 = time.time()
        xm = P.matricize(x.shape, x.flat_idx(), x.val, 0)
        v = P.relerr_dd_full(xm, fe.R, fe.U)
        t2 = time.time()
        out[name] = {
            "shape": list(map(int, x.shape)), "nnz": int(x.nnz), "c": s, "eps": eps, "seed": seed, "mode": 0,
            "input_sha": sha(np.concatenate([x.flat_idx().astype(np.int64).view(np.uint8),
                                             x.val.astype(np.float64).view(np.uint8)])),
            "kept": int(len(fe.kept_flat)), "kept_sha": sha(fe.kept_flat.astype(np.int64)),
            "U_sha": sha(fe.U.astype(np.float64)),
            "relative_error": v,
            "how": "oracle/relerr_dd.c cto_relerr_dd_full (double-double) on the C restatement's R, U",
            "seconds": {"front_end": round(t1 - t0, 1), "relerr_dd": round(t2 - t1, 1)},
        }
        print(name, out[name], flush=True)
        with open(OUT, "w") as f:
            json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1:] or list(CASES))
