"""Sharded CTD-S with the host orchestration inside the library
(`ctd_gpu_ctd_s_sharded`, csrc/dist.cu).

GPU: two ranks sharing one device over the host-callback communicator (gloo
underneath) must give the single-GPU ctd_s bit for bit (kept ids, decisions,
delta, U, R; the core columns merged in rank order) and the error within
1e-9; one rank over the library's own NCCL communicator must do the same.
CPU: the NCCL loader and the communicator's argument checks (no GPU needed).
"""
import ctypes as C
import os
import socket

import numpy as np
import pytest

from paper_1710_03608_b200 import datagen, dist

CASES = {
    "c1": lambda: datagen.c1(),
    "traffic": lambda: datagen.traffic([80, 80, 30], 6000, 5),
}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, mode, s, backend, out):
    import torch
    import torch.distributed as tdist
    from paper_1710_03608_b200 import ctd as api
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x = CASES[case]()
        bounds = dist.fiber_range_bounds(x.shape, mode, x.idx, world)
        il, vl = dist.shard(x.shape, x.idx, x.val, mode, bounds, rank)
        ctx = api.Context(0)
        local = api.DeviceTensor(api.SparseTensor(list(x.shape), il, vl), ctx)
        comm = dist.NativeComm(ctx, backend)
        r = dist.ctd_s_sharded_native(local, mode, s, 1e-6, 42, comm=comm, with_error=True, with_core=True)
        cc, cptr, crow, cval = r.core
        np.savez(os.path.join(out, f"r{rank}.npz"), kept=r.kept_flat, U=r.U, acc=r.accepted, deg=r.degenerate,
                 delta=r.delta, unique=r.unique, rel=r.relative_error, total=r.total_sq_norm,
                 cp=r.R_col_ptr, rr=r.R_row, rv=r.R_val, ccol=cc, cptr=cptr, crow=crow, cval=cval,
                 nf=r.n_fibers)
        comm.close()
    finally:
        tdist.destroy_process_group()


def _run(case, mode, s, backend, tmp_path, world):
    import torch.multiprocessing as mp
    mp.spawn(_worker, args=(world, _free_port(), case, mode, s, backend, str(tmp_path)), nprocs=world, join=True)
    return [dict(np.load(tmp_path / f"r{r}.npz")) for r in range(world)]


def _merged_core(res):
    cols, ptrs, rows, vals = [], [0], [], []
    for r in res:
        cols.append(r["ccol"])
        ptrs.extend((r["cptr"][1:] + ptrs[-1]).tolist())
        rows.append(r["crow"])
        vals.append(r["cval"])
    return np.concatenate(cols), np.array(ptrs, np.int64), np.concatenate(rows), np.concatenate(vals)


def _check_equal_single(res, case, mode, s):
    from paper_1710_03608_b200 import ctd
    x = CASES[case]()
    f = ctd.ctd_s(ctd.SparseTensor.from_datagen(x), mode, s, 1e-6, 42, with_error=True)
    for r in res:
        assert np.array_equal(r["kept"], f.kept_flat)
        assert np.array_equal(r["U"].view(np.int64), f.U.view(np.int64))
        assert np.array_equal(r["cp"], f.R_col_ptr) and np.array_equal(r["rr"], f.R_row)
        assert np.array_equal(r["rv"].view(np.int64), f.R_val.view(np.int64))
        assert abs(float(r["rel"]) - f.relative_error) <= 1e-9 * max(1.0, abs(f.relative_error))
        assert float(r["total"]) == f.total_sq_norm
    for a, b in zip(res, res[1:]):  # replicated: identical bits on every rank
        for k in ("kept", "unique", "acc", "deg", "delta", "U", "rel"):
            assert np.asarray(a[k]).tobytes() == np.asarray(b[k]).tobytes()
    fc = ctd.ctd_s(ctd.SparseTensor.from_datagen(x), mode, s, 1e-6, 42, with_core=True)
    got = _merged_core(res)
    assert np.array_equal(got[0], fc.C_col) and np.array_equal(got[1], fc.C_ptr)
    assert np.array_equal(got[2], fc.C_row) and np.array_equal(got[3].view(np.int64), fc.C_val.view(np.int64))


@pytest.mark.gpu
@pytest.mark.parametrize("case,mode,s", [("c1", 0, 200), ("traffic", 0, 300), ("traffic", 1, 250)])
def test_native_two_ranks_host_comm_equal_single_gpu(case, mode, s, tmp_path):
    _check_equal_single(_run(case, mode, s, "host", tmp_path, 2), case, mode, s)


@pytest.mark.gpu
def test_native_three_ranks_host_comm(tmp_path):
    """Three ranks (one may hold few fibers): the chained law and the slot
    exchanges do not depend on the rank count."""
    _check_equal_single(_run("traffic", 0, 300, "host", tmp_path, 3), "traffic", 0, 300)


@pytest.mark.gpu
def test_native_nccl_one_rank_equal_single_gpu(tmp_path):
    """The library's own NCCL communicator (dlopen'ed libnccl, ncclAllReduce on
    the context stream); one rank is all a one-GPU box can run."""
    _check_equal_single(_run("traffic", 0, 300, "nccl", tmp_path, 1), "traffic", 0, 300)


@pytest.mark.gpu
def test_native_sharded_errors():
    import torch.distributed as tdist
    from paper_1710_03608_b200 import ctd as api
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    tdist.init_process_group("gloo", rank=0, world_size=1)
    try:
        x = CASES["c1"]()
        ctx = api.Context(0)
        local = api.DeviceTensor(api.SparseTensor.from_datagen(x), ctx)
        comm = dist.NativeComm(ctx, "host")
        with pytest.raises(api.ArgumentError):
            dist.ctd_s_sharded_native(local, 0, 0, 1e-6, 42, comm=comm)
        with pytest.raises(api.ArgumentError):
            dist.ctd_s_sharded_native(local, 0, 10, 0.0, 42, comm=comm)
        with pytest.raises(api.ArgumentError):
            dist.ctd_s_sharded_native(local, 5, 10, 1e-6, 42, comm=comm)
        other = api.Context(0)
        h = C.c_void_p()
        st = comm.L.ctd_gpu_ctd_s_sharded(other.h, comm.h, local.h, 0, 10, C.c_double(1e-6), C.c_uint64(42), 0,
                                          C.byref(h))
        assert st == 1  # ArgumentError: communicator of another context
        comm.close()
    finally:
        tdist.destroy_process_group()


def test_comm_argument_checks_without_gpu():
    """Communicator entry points reject bad arguments before touching a device."""
    from paper_1710_03608_b200 import _lib
    L = _lib.load()
    h = C.c_void_p()
    assert L.ctd_gpu_comm_host_create(None, 2, 0, _lib.ALLREDUCE_FN(lambda *a: 0), None, C.byref(h)) == 1
    assert L.ctd_gpu_comm_nccl_create(None, 2, 0, (C.c_ubyte * 128)(), C.byref(h)) == 1
    assert L.ctd_gpu_comm_destroy(None) == 0
    assert L.ctd_gpu_sharded_destroy(None) == 0
    assert L.ctd_gpu_sharded_basis(None) is None
