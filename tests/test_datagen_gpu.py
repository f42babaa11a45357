"""The device traffic generator (C5 input) against the host generator: identical
bytes on shared sizes (torch CPU tensors here; the same code runs on CUDA)."""
import numpy as np
import pytest

from paper_1710_03608_b200 import datagen

torch = pytest.importorskip("torch")


@pytest.mark.parametrize("shape,nnz,seed,batch,parts", [
    ([500, 500, 20], 20000, 11, 1 << 12, 4),
    ([10000, 10000, 30], 300000, 2, 1 << 16, 8),
    ([300, 200, 7], 5000, 3, 1 << 20, 1),
])
def test_device_generator_matches_host(shape, nnz, seed, batch, parts):
    from paper_1710_03608_b200 import datagen_gpu
    x = datagen.traffic(shape, nnz, seed)
    idx, val, meta = datagen_gpu.traffic(shape, nnz, seed, device="cpu", batch=batch, parts=parts)
    assert meta["draws"] == x.meta["draws"]
    assert np.array_equal(idx.numpy().T.astype(np.int64), x.idx)
    assert np.array_equal(val.numpy(), x.val)


def test_uniform_bits_match():
    from paper_1710_03608_b200 import datagen_gpu
    for seed, stream, start in [(0, 0, 0), (42, 3, 10**9), (2**40 + 3, 7, 123)]:
        a = datagen.uniform(seed, stream, start, 4096)
        b = datagen_gpu.uniform(seed, stream, start, 4096, "cpu").numpy()
        assert np.array_equal(a, b)


@pytest.mark.gpu
def test_device_generator_cuda_matches_host():
    from paper_1710_03608_b200 import datagen_gpu
    x = datagen.traffic([10000, 10000, 30], 300000, 2)
    idx, val, meta = datagen_gpu.traffic([10000, 10000, 30], 300000, 2, device="cuda", batch=1 << 16,
                                         parts=8)
    assert np.array_equal(idx.cpu().numpy().T.astype(np.int64), x.idx)
    assert np.array_equal(val.cpu().numpy(), x.val)
