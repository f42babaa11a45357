"""The C-ABI library loads on a CPU-only host and exports every symbol that
include/ctd_gpu.h declares; the Python binding table covers the header
exactly.  No compute calls (no GPU here)."""
import ctypes
import os
import re

from paper_1710_03608_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ctd_gpu.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ctd_gpu_\w+)\s*\(", src)))


def test_header_declares_entry_points():
    names = declared()
    for must in ("ctd_gpu_ctd_s", "ctd_gpu_stream_init", "ctd_gpu_stream_step",
                 "ctd_gpu_relative_error", "ctd_gpu_basis_try_append",
                 "ctd_gpu_column_distribution", "ctd_gpu_sample_with_replacement",
                 "ctd_gpu_unique_first_occurrence", "ctd_gpu_matricize"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_table_matches_header():
    bound = sorted(n for n, _, _ in _lib.SIGNATURES)
    assert bound == declared()


def test_load_binds_all_and_version():
    L = _lib.load()
    assert L.ctd_gpu_version().startswith(b"ctd_gpu")


def test_missing_library_fails_loudly(tmp_path):
    import pytest
    with pytest.raises(ImportError):
        _lib.load(str(tmp_path / "nope.so"))


def test_context_without_gpu_reports_device_error():
    """On a host without a GPU the API raises (no CPU fallback)."""
    import torch
    if torch.cuda.is_available():
        return
    import pytest
    import paper_1710_03608_b200 as ctd
    with pytest.raises(ctd.CtdError):
        ctd.Context(0)
