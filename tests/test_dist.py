"""Sharded CTD-S (paper_1710_03608_b200.dist) with world_size 2.

CPU: two gloo ranks run the sharded host logic (fiber-range shards, all-gather
of candidate payloads, the sampling law chained rank to rank, replicated filter, all-reduced error
partials) with oracle-backed per-rank kernels; the replicated result must equal
the single-process oracle bit for bit (kept ids, decisions, U) and the error
within 1e-9.  GPU: the same with the C-ABI kernels (two ranks on one device,
host-side gloo collectives) against the single-process GPU ctd_s.
"""
import os
import socket

import numpy as np
import pytest

from paper_1710_03608_b200 import datagen, dist

CASES = {
    "c1": lambda: datagen.c1(),
    "cp": lambda: datagen.low_rank([30, 25, 12], 3, 0.3, 11) if hasattr(datagen, "low_rank") else datagen.c1(),
    "traffic": lambda: datagen.traffic([80, 80, 30], 6000, 5),
}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, mode, s, backend, out):
    import torch.distributed as tdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x = CASES[case]()
        bounds = dist.fiber_range_bounds(x.shape, mode, x.idx, world)
        il, vl = dist.shard(x.shape, x.idx, x.val, mode, bounds, rank)
        if backend == "oracle":
            from oracle.bindings import Port
            from dist_oracle_kernels import OracleKernels
            k = OracleKernels(Port())
        else:
            k = dist.GpuKernels()
        r = dist.ctd_s_sharded(x.shape, (il, vl), mode, s, 1e-6, 42, comm=dist.Comm(), kernels=k,
                               with_error=True, with_core=True)
        cc, cptr, crow, cval = r.core
        np.savez(os.path.join(out, f"r{rank}.npz"), kept=r.kept_flat, U=r.U, acc=r.accepted, deg=r.degenerate,
                 delta=r.delta, unique=r.unique, rel=r.relative_error, total=r.total_sq_norm,
                 cp=r.R_col_ptr, rr=r.R_row, rv=r.R_val, ccol=cc, cptr=cptr, crow=crow, cval=cval,
                 cnnz=r.core_nnz, mem=r.memory_usage)
    finally:
        tdist.destroy_process_group()


def _run(case, mode, s, backend, tmp_path, world=2):
    import torch.multiprocessing as mp
    mp.spawn(_worker, args=(world, _free_port(), case, mode, s, backend, str(tmp_path)), nprocs=world, join=True)
    return [dict(np.load(tmp_path / f"r{r}.npz")) for r in range(world)]


def test_fiber_ids_match_matricize_order(port):
    x = datagen.c1()
    for mode in range(3):
        m = port.matricize(x.shape, x.idx.reshape(-1), x.val, mode)
        j = dist.fiber_ids(x.shape, mode, x.idx)
        cols = np.nonzero(np.diff(m.col_ptr) > 0)[0]
        assert np.array_equal(np.unique(j), cols)


def test_bounds_partition_everything():
    x = datagen.traffic([80, 80, 30], 6000, 5)
    for world in (1, 2, 3, 8):
        b = dist.fiber_range_bounds(x.shape, 0, x.idx, world)
        assert b[0] == 0 and b[-1] == 80 * 30 and np.all(np.diff(b) >= 0)
        n = sum(dist.shard(x.shape, x.idx, x.val, 0, b, r)[1].shape[0] for r in range(world))
        assert n == x.nnz


@pytest.mark.parametrize("case,mode,s", [("c1", 0, 200), ("c1", 2, 150), ("traffic", 0, 300), ("cp", 1, 120)])
def test_sharded_equals_single_process_oracle(case, mode, s, port, tmp_path):
    res = _run(case, mode, s, "oracle", tmp_path)
    x = CASES[case]()
    fe = port.frontend(x.shape, x.idx.reshape(-1), x.val, mode, s, 1e-6, 42)
    for r in res:  # every rank holds the same replicated result
        assert np.array_equal(r["unique"], fe.unique)
        assert np.array_equal(r["acc"], fe.accepted)
        assert np.array_equal(r["deg"], fe.degenerate)
        assert np.array_equal(r["delta"].view(np.int64), fe.delta.view(np.int64))
        assert np.array_equal(r["kept"], fe.kept_flat)
        assert np.array_equal(r["U"].view(np.int64), fe.U.view(np.int64))
        assert np.array_equal(r["cp"], fe.R.col_ptr) and np.array_equal(r["rr"], fe.R.row)
        assert r["total"] == fe.total
    # the error partials combine to the single-process value of the same formula
    # (|X|^2 - sum_j x_j^T R U R^T x_j) / |X|^2 ...
    want = _gram_identity_error(port, x, mode, fe.R, fe.U)
    for r in res:
        assert abs(float(r["rel"]) - want) <= 1e-9 * max(1.0, abs(want))
    # ... which is the reference's relative_error when U is well conditioned
    fe2, core, rel = port.ctd_s_error(x.shape, x.idx.reshape(-1), x.val, mode, s, 1e-6, 42)
    if 0.0 <= rel <= 1.0:
        assert abs(want - rel) <= 1e-9 * max(1.0, abs(rel))


def _merged_core(res):
    """The ranks' column shards of C concatenated in rank order (their fiber
    ranges ascend): (col ids, col_ptr, rows, vals)."""
    cols, rows, vals, ptr = [], [], [], [0]
    for r in res:
        cols.append(r["ccol"])
        rows.append(r["crow"])
        vals.append(r["cval"])
        ptr.extend((np.asarray(r["cptr"][1:]) + ptr[-1]).tolist())
    return (np.concatenate(cols), np.asarray(ptr, np.int64), np.concatenate(rows), np.concatenate(vals))


def _nonempty_cols(c):
    counts = np.diff(c.col_ptr)
    cols = np.nonzero(counts > 0)[0]
    sel = np.concatenate([np.arange(c.col_ptr[j], c.col_ptr[j + 1]) for j in cols]) if cols.size else \
        np.zeros(0, np.int64)
    return cols, np.concatenate([[0], np.cumsum(counts[cols])]), np.asarray(c.row)[sel], np.asarray(c.val)[sel]


@pytest.mark.parametrize("case,mode,s", [("c1", 0, 200), ("traffic", 0, 300)])
def test_sharded_core_equals_single_process_oracle(case, mode, s, port, tmp_path):
    """compute_core over fiber-range shards (gloo, two ranks, oracle kernels):
    the ranks' column shards of C, in rank order, are the single-process core
    bit for bit, and every rank reports the same global nnz(C) / memory_usage."""
    res = _run(case, mode, s, "oracle", tmp_path)
    x = CASES[case]()
    fe, core, _ = port.ctd_s_error(x.shape, x.idx.reshape(-1), x.val, mode, s, 1e-6, 42)
    want = _nonempty_cols(core)
    got = _merged_core(res)
    assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])
    assert np.array_equal(got[2], want[2]) and np.array_equal(got[3].view(np.int64), want[3].view(np.int64))
    for r in res:
        assert int(r["cnnz"]) == core.nnz
        assert float(r["mem"]) == (core.nnz + np.count_nonzero(fe.U) + fe.R.nnz) / x.nnz


def _gram_identity_error(port, x, mode, R, U):
    m = port.matricize(x.shape, x.idx.reshape(-1), x.val, mode)
    K = U.shape[0]
    Rd = np.zeros((m.rows, K))
    for k in range(K):
        Rd[R.row[R.col_ptr[k]:R.col_ptr[k + 1]], k] = R.val[R.col_ptr[k]:R.col_ptr[k + 1]]
    xs = float(np.sum(m.val * m.val))
    cross = 0.0
    for c in range(m.cols):
        a, b = m.col_ptr[c], m.col_ptr[c + 1]
        if b > a:
            g = Rd[m.row[a:b]].T @ m.val[a:b]
            cross += float(g @ (U @ g))
    return 1.0 if K == 0 else (xs - cross) / xs


@pytest.mark.gpu
@pytest.mark.parametrize("case,mode,s", [("c1", 0, 200), ("traffic", 0, 300)])
def test_sharded_gpu_two_ranks_equal_single_gpu(case, mode, s, tmp_path):
    from paper_1710_03608_b200 import ctd
    res = _run(case, mode, s, "gpu", tmp_path)
    x = CASES[case]()
    f = ctd.ctd_s(ctd.SparseTensor.from_datagen(x), mode, s, 1e-6, 42, with_error=True)
    for r in res:
        assert np.array_equal(r["kept"], f.kept_flat)
        assert np.array_equal(r["U"].view(np.int64), f.U.view(np.int64))
        assert abs(float(r["rel"]) - f.relative_error) <= 1e-9 * max(1.0, abs(f.relative_error))
    # the core, column-sharded: the ranks' shards in rank order are the single-GPU core
    fc = ctd.ctd_s(ctd.SparseTensor.from_datagen(x), mode, s, 1e-6, 42, with_core=True)
    got = _merged_core(res)
    assert np.array_equal(got[0], fc.C_col) and np.array_equal(got[1], fc.C_ptr)
    assert np.array_equal(got[2], fc.C_row) and np.array_equal(got[3].view(np.int64), fc.C_val.view(np.int64))


def _stream_worker(rank, world, port, backend, out):
    import torch.distributed as tdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x = datagen.c3_stream(seed=5, n_steps=3, slices_per_step=3, draws_per_slice=2500, n=300, planted_step=2,
                              block=20)
        hist = x.time_slab(0, 3)
        if backend == "oracle":
            from oracle.bindings import Port
            from dist_oracle_kernels import OracleKernels
            k = OracleKernels(Port())
        else:
            k = dist.GpuKernels()
        comm = dist.Comm()
        hb = dist.fiber_range_bounds(hist.shape, 0, hist.idx, world)
        st = dist.ShardedStream(hist.shape, dist.shard(hist.shape, hist.idx, hist.val, 0, hb, rank), 0, 120, 1e-6,
                                7, comm=comm, kernels=k, with_core=True)
        kept = [np.array(st.kept_flat, np.int64)]
        for t in range(3, x.shape[2]):
            sl = x.time_slab(t, t + 1)
            sb = dist.fiber_range_bounds(sl.shape, 0, sl.idx, world)
            st.step(dist.shard(sl.shape, sl.idx, sl.val, 0, sb, rank), 40)
            kept.append(np.array(st.kept_flat, np.int64))
        cc, cptr, crow, cval = st.core_columns()
        np.savez(os.path.join(out, f"s{rank}.npz"), U=st.U(), t=st.t, ccol=cc, cptr=cptr, crow=crow, cval=cval,
                 **{f"k{i}": k_ for i, k_ in enumerate(kept)})
        st.close()
    finally:
        tdist.destroy_process_group()


def _run_stream(backend, tmp_path, world=2):
    import torch.multiprocessing as mp
    mp.spawn(_stream_worker, args=(world, _free_port(), backend, str(tmp_path)), nprocs=world, join=True)
    return [dict(np.load(tmp_path / f"s{r}.npz")) for r in range(world)]


def test_sharded_stream_equals_single_process(port, tmp_path):
    """CTD-D with every slab split by fiber range over two ranks (gloo, CPU
    kernels): kept ids after every step and U equal the single-process
    restatement's stream, and the ranks' column shards of the Eq. 13 core, in
    rank order per slab, are its core bit for bit."""
    res = _run_stream("oracle", tmp_path)
    x = datagen.c3_stream(seed=5, n_steps=3, slices_per_step=3, draws_per_slice=2500, n=300, planted_step=2, block=20)
    hist = x.time_slab(0, 3)
    ps = port.stream(hist.shape, hist.flat_idx(), hist.val, 0, 120, 1e-6, 7, core=True)
    want = [ps.kept_flat()]
    for t in range(3, x.shape[2]):
        sl = x.time_slab(t, t + 1)
        ps.step(sl.shape, sl.flat_idx(), sl.val, 40)
        want.append(ps.kept_flat())
    for r in res:
        for i, w in enumerate(want):
            assert np.array_equal(r[f"k{i}"], w), i
        assert int(r["t"]) == x.shape[2]
        assert np.array_equal(r["U"].view(np.int64), ps.U().view(np.int64))
    _check_sharded_stream_core(res, ps.core())


def _check_sharded_stream_core(res, core):
    """Every core column is held by exactly one rank; together they are the
    single-process core (nonempty columns), bit for bit."""
    want = _nonempty_cols(core)
    cols = np.concatenate([r["ccol"] for r in res])
    assert np.unique(cols).shape[0] == cols.shape[0]
    order = np.argsort(cols, kind="stable")
    got_rows, got_vals, ptr = [], [], [0]
    flat = [(r, q) for r in res for q in range(r["ccol"].shape[0])]
    for o in order:
        r, q = flat[o]
        a, b = r["cptr"][q], r["cptr"][q + 1]
        got_rows.append(r["crow"][a:b])
        got_vals.append(r["cval"][a:b])
        ptr.append(ptr[-1] + (b - a))
    assert np.array_equal(cols[order], want[0])
    assert np.array_equal(np.asarray(ptr), want[1])
    assert np.array_equal(np.concatenate(got_rows), want[2])
    assert np.array_equal(np.concatenate(got_vals).view(np.int64), want[3].view(np.int64))
    # the bottom-left block (chain_product) was exercised: some history column
    # holds a row of a fiber kept after init_stream
    k0 = res[0]["k0"].shape[0]
    hist_cols = want[0] < 3 * 300  # the 3 history slices (slab columns: 300 dst ids)
    rows_of = [want[2][want[1][q]:want[1][q + 1]] for q in np.nonzero(hist_cols)[0]]
    assert any((rr >= k0).any() for rr in rows_of)


@pytest.mark.gpu
def test_sharded_stream_gpu_two_ranks(port, tmp_path):
    res = _run_stream("gpu", tmp_path)
    x = datagen.c3_stream(seed=5, n_steps=3, slices_per_step=3, draws_per_slice=2500, n=300, planted_step=2, block=20)
    hist = x.time_slab(0, 3)
    ps = port.stream(hist.shape, hist.flat_idx(), hist.val, 0, 120, 1e-6, 7, core=True)
    for t in range(3, x.shape[2]):
        sl = x.time_slab(t, t + 1)
        ps.step(sl.shape, sl.flat_idx(), sl.val, 40)
    for r in res:
        assert np.array_equal(r[f"k{x.shape[2] - 3}"], ps.kept_flat())
        assert np.array_equal(r["U"].view(np.int64), ps.U().view(np.int64))
    _check_sharded_stream_core(res, ps.core())


@pytest.mark.gpu
def test_device_candidates_match_host_path(port):
    """The device-plane entry points (ctd_gpu_shard_gather_device,
    ctd_gpu_basis_append_batch_device) give the host path's decisions and U
    bit for bit, and run the host path's input checks on the device."""
    from paper_1710_03608_b200 import ctd as api

    k = dist.GpuKernels()
    x = datagen.random_sparse([40, 30, 20], 0.05, 33)
    sh = k.shard((x.shape, x.idx, x.val), 0)
    cols = sh.col[::7][:40]
    ptr_h, rows_h, vals_h = sh.gather(cols)
    ptr_d, rows_d, vals_d = sh.gather_device(cols)
    assert np.array_equal(ptr_h, ptr_d)
    assert np.array_equal(rows_h, rows_d.cpu().numpy().astype(np.int64))
    assert np.array_equal(vals_h, vals_d.cpu().numpy())
    Bh, Bd = k.basis(40), k.basis(40)
    a_h = Bh.append_batch(ptr_h, rows_h, vals_h, 1e-6)
    a_d = Bd.append_batch_device(ptr_d, rows_d, vals_d, 1e-6)
    for u, v in zip(a_h, a_d):
        assert np.array_equal(np.asarray(u).view(np.int64) if u.dtype == np.float64 else u,
                              np.asarray(v).view(np.int64) if v.dtype == np.float64 else v)
    assert np.array_equal(Bh.u().view(np.int64), Bd.u().view(np.int64))
    # checks: a row outside [0, dim) and rows that do not ascend
    bad = rows_d.clone()
    bad[0] = 40
    with pytest.raises(api.ShapeError):
        k.basis(40).append_batch_device(ptr_d, bad, vals_d, 1e-6)
    j = int(np.argmax(np.diff(ptr_d) >= 2))
    bad = rows_d.clone()
    bad[ptr_d[j] + 1] = bad[ptr_d[j]]
    with pytest.raises(api.ArgumentError):
        k.basis(40).append_batch_device(ptr_d, bad, vals_d, 1e-6)
    for b in (Bh, Bd):
        b.close()
    sh.close()
