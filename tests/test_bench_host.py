"""Host-side pieces of bench.py (no GPU): the algorithmic byte model and the
filter's dependency floor, on hand-computed cases."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def test_chain_floor_hand_case():
    # accept {0,1}; accept {1,2}; reject; accept {1}
    acc = np.array([1, 1, 0, 1], bool)
    ptr = np.array([0, 2, 4, 5])
    rows = np.array([0, 1, 1, 2, 1])
    # steps: (0+0) + (1+1) + (2+2) + (2+2) = 10
    assert bench.chain_floor_cycles(acc, ptr, rows, 3) == 8.2 * 10
    assert bench.chain_floor_cycles(np.zeros(0, bool), np.array([0]), np.zeros(0, np.int64), 3) == 0.0


def test_phase_bytes():
    acc = np.array([1, 0, 1], bool)
    pb = bench.phase_bytes(nnz=100, F=10, kept_seq=acc, r_lens=np.array([3, 4]))
    assert pb["matricize"] == 32 * 100 + 24 * 10
    assert pb["law"] == 24 * 10
    # cand 0: K=0 -> 0 + accept 8*1; cand 1: K=1 -> 8 + 12*3; cand 2: K=1 -> 8 + 36 + accept 8*4
    assert pb["filter"] == 8 + (8 + 36) + (8 + 36 + 32)
