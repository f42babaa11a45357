"""Factor bundle I/O (factor_io.hpp, factor_io.cpp:56-232): the reference's
on-disk format, byte for byte.

    manifest.txt  "ctd-factors 1", shape, mode (1-based), epsilon (%.17g),
                  seed, kept count, kept fiber ids (1-based)
    R.tsv         row col value (1-based), columns in acceptance order
    C.tsv         the folded core's index tuple (1-based) + value, in
                  lexicographic entry order (SparseTensor order)
    U.tsv         dense rows, tab-separated

Host code over an ``LRFactors`` (the factors are copied off the device by
``ctd_s`` / ``StreamState.factors``); load_factors(save_factors(f)) == f bit for
bit.  Errors raise ``IoError`` (ErrorClass io = 7, error.hpp:11-19).
"""
from __future__ import annotations

import os

import numpy as np

from . import ctd as api

MAGIC = "ctd-factors"
VERSION = 1


class IoError(api.CtdError):
    error_class = 7


def _fmt(v: float) -> str:
    return "%.17g" % v


def _core_entries(f: api.LRFactors):
    """The folded core C (fold, tensor_ops.cpp:137-170) as lexicographically
    sorted (indices [nnz, order], values)."""
    order = len(f.shape)
    if f.C_col is None:
        return np.zeros((0, order), np.int64), np.zeros(0)
    others = [k for k in range(order) if k != f.mode]
    cnt = np.diff(np.asarray(f.C_ptr, np.int64))
    cols = np.repeat(np.asarray(f.C_col, np.int64), cnt)
    idx = np.zeros((cols.shape[0], order), np.int64)
    rem = cols.copy()
    for k in others:
        idx[:, k] = rem % f.shape[k]
        rem //= f.shape[k]
    idx[:, f.mode] = np.asarray(f.C_row, np.int64)
    perm = np.lexsort(tuple(idx[:, k] for k in range(order - 1, -1, -1))) if idx.shape[0] else np.zeros(0, int)
    return idx[perm], np.asarray(f.C_val, np.float64)[perm]


def save_factors(f: api.LRFactors, directory: str) -> None:
    """save_factors (factor_io.cpp:56-105)."""
    try:
        os.makedirs(directory, exist_ok=True)
    except OSError as e:
        raise IoError(f"cannot create '{directory}'") from e
    K = f.kept_count()
    lines = [f"{MAGIC} {VERSION}", "shape" + "".join(f" {int(e)}" for e in f.shape), f"mode {f.mode + 1}",
             f"epsilon {_fmt(f.epsilon)}", f"seed {int(f.seed)}", f"kept {K}",
             "fibers" + "".join(f" {int(j) + 1}" for j in f.kept_flat)]
    _write(os.path.join(directory, "manifest.txt"), "\n".join(lines) + "\n")
    cp = np.asarray(f.R_col_ptr, np.int64)
    out = []
    for j in range(K):
        for t in range(cp[j], cp[j + 1]):
            out.append(f"{int(f.R_row[t]) + 1}\t{j + 1}\t{_fmt(float(f.R_val[t]))}\n")
    _write(os.path.join(directory, "R.tsv"), "".join(out))
    idx, val = _core_entries(f)
    out = ["".join(f"{int(i) + 1}\t" for i in idx[e]) + _fmt(float(val[e])) + "\n" for e in range(val.shape[0])]
    _write(os.path.join(directory, "C.tsv"), "".join(out))
    U = np.asarray(f.U, np.float64).reshape(K, K)
    _write(os.path.join(directory, "U.tsv"), "".join("\t".join(_fmt(float(v)) for v in U[r]) + "\n"
                                                       for r in range(K)))


def _write(path, text):
    try:
        with open(path, "w") as fh:
            fh.write(text)
    except OSError as e:
        raise IoError(f"cannot write '{path}'") from e


def _read(path):
    try:
        with open(path) as fh:
            return fh.read()
    except OSError as e:
        raise IoError(f"missing bundle file '{path}'") from e


def _parse_double(tok, what):
    try:
        if tok.strip() != tok or not tok:
            raise ValueError
        return float(tok)
    except ValueError:
        raise IoError(f"malformed {what} '{tok}'") from None


def _parse_index(tok, what):
    try:
        return int(tok, 10)
    except ValueError:
        raise IoError(f"malformed {what} '{tok}'") from None


def load_factors(directory: str) -> api.LRFactors:
    """load_factors (factor_io.cpp:107-232): IoError on a missing member, bad
    magic, unsupported version or inconsistent dimensions."""
    toks = _read(os.path.join(directory, "manifest.txt")).split("\n")
    words = " ".join(toks).split()
    if len(words) < 2 or words[0] != MAGIC:
        raise IoError("not a factor bundle (bad magic)")
    if _parse_index(words[1], "version") != VERSION:
        raise IoError(f"unsupported bundle version {words[1]}")
    shape, mode, eps, seed, kept, fibers = [], None, 0.0, 0, 0, []
    for line in toks:
        parts = line.split()
        if not parts or parts[0] == MAGIC:
            continue
        key, rest = parts[0], parts[1:]
        if key == "shape":
            shape = [_parse_index(t, "shape") for t in rest]
        elif key == "mode":
            mode = _parse_index(rest[0], "mode") - 1 if rest else None
        elif key == "epsilon":
            eps = _parse_double(rest[0] if rest else "", "epsilon")
        elif key == "seed":
            seed = _parse_index(rest[0], "seed")
        elif key == "kept":
            kept = _parse_index(rest[0], "kept")
        elif key == "fibers":
            fibers = [_parse_index(t, "fiber id") - 1 for t in rest]
        else:
            raise IoError(f"unknown manifest key '{key}'")
    if not shape:
        raise IoError("manifest shape missing")
    if mode is None or mode < 0 or mode >= len(shape):
        raise IoError("manifest mode out of range")
    if len(fibers) != kept:
        raise IoError("manifest fiber ids disagree with kept count")
    for j in fibers:
        api.make_fiber_id(shape, mode, j)
    # R: (row, col, value) triples -> CSC in (col, row) order
    rt = _read(os.path.join(directory, "R.tsv")).split()
    if len(rt) % 3:
        raise IoError("R.tsv inconsistent: truncated triple")
    rows = np.array([_parse_index(t, "R row") - 1 for t in rt[0::3]], np.int64)
    cols = np.array([_parse_index(t, "R column") - 1 for t in rt[1::3]], np.int64)
    vals = np.array([_parse_double(t, "R value") for t in rt[2::3]], np.float64)
    dim = shape[mode]
    if rows.size and (rows.min() < 0 or rows.max() >= dim or cols.min() < 0 or cols.max() >= kept):
        raise IoError("R.tsv inconsistent: index out of range")
    o = np.lexsort((rows, cols))
    rows, cols, vals = rows[o], cols[o], vals[o]
    cp = np.zeros(kept + 1, np.int64)
    np.add.at(cp, cols + 1, 1)
    cp = np.cumsum(cp)
    # C: folded entries -> matricized CSC over the nonempty columns
    order = len(shape)
    cidx, cval = [], []
    for n, line in enumerate(_read(os.path.join(directory, "C.tsv")).split("\n"), 1):
        t = line.split()
        if not t:
            continue
        if len(t) != order + 1:
            raise IoError(f"C.tsv line {n}: wrong field count")
        cidx.append([_parse_index(x, "C index") - 1 for x in t[:order]])
        cval.append(_parse_double(t[-1], "C value"))
    f_c = [None] * 4
    if cidx:
        ci = np.array(cidx, np.int64)
        cv = np.array(cval, np.float64)
        cshape = list(shape)
        cshape[mode] = kept
        if (ci < 0).any() or (ci >= np.array(cshape)).any():
            raise IoError("C.tsv inconsistent: index out of range")
        j = np.zeros(ci.shape[0], np.int64)
        stride = 1
        for k in range(order):
            if k != mode:
                j += ci[:, k] * stride
                stride *= shape[k]
        o = np.lexsort((ci[:, mode], j))
        j, r, cv = j[o], ci[o, mode], cv[o]
        ucol, start = np.unique(j, return_index=True)
        f_c = [ucol, np.append(start, j.shape[0]).astype(np.int64), r, cv]
    # U: K rows of K values
    ul = [ln.split() for ln in _read(os.path.join(directory, "U.tsv")).split("\n") if ln.split()]
    if len(ul) != kept or any(len(r) != kept for r in ul):
        raise IoError("U.tsv dimensions disagree with kept count")
    U = np.array([[_parse_double(x, "U value") for x in r] for r in ul], np.float64).reshape(kept, kept)
    f = api.LRFactors(mode, shape, eps, seed, np.array(fibers, np.int64), U, cp, rows, vals)
    f.C_col, f.C_ptr, f.C_row, f.C_val = f_c
    return f
