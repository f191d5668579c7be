"""CPU-side checks of the C ABI boundary: the library builds/loads and exports
every entry point declared in include/rtec.h (no compute without a GPU)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
HEADER = os.path.join(ROOT, "include", "rtec.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|size_t|void|const char\*)\s+(rtec_\w+)\s*\(", text, re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2603_20622_b200 import _lib

    if not os.path.exists(_lib.LIB_PATH):
        import __graft_entry__

        __graft_entry__.build()
    return _lib.load(require_cuda=False)


def test_header_declares_entry_points():
    syms = declared_symbols()
    for s in ("rtec_batch_apply", "rtec_frontier_layer", "rtec_layer_incremental", "rtec_layer_full", "rtec_query"):
        assert s in syms


def test_library_exports_every_declared_symbol(lib):
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_binding_covers_header(lib):
    from paper_2603_20622_b200 import _lib

    assert set(declared_symbols()) == set(_lib.EXPORTED)


def test_pure_host_entry_points(lib):
    assert lib.rtec_version().startswith(b"rtec-b200")
    assert lib.rtec_workspace_bytes(1000, 100, 10000, 128) > 1000 * 128 * 4
    assert lib.rtec_build_workspace_bytes(1000, 10000) > 10000 * 12


def test_struct_layouts_match_header(lib):
    from paper_2603_20622_b200 import _lib

    sizes = (ctypes.c_int64 * 7)()
    lib.rtec_struct_sizes(sizes)
    mirror = [_lib.Adj, _lib.Graph, _lib.Batch, _lib.Frontier, _lib.Layer, _lib.State, _lib.Shard]
    assert list(sizes) == [ctypes.sizeof(t) for t in mirror]
    assert ctypes.sizeof(_lib.Adj) == 8 * 7
    assert ctypes.sizeof(_lib.Graph) == 8 + 2 * 56 + 5 * 8 + 8 + 8  # + part_rank / part_count
    assert ctypes.sizeof(_lib.Batch) == 8 * 20  # + apply_ctr
    assert ctypes.sizeof(_lib.Frontier) == 8 * 11
    assert ctypes.sizeof(_lib.Layer) == 6 * 4 + 9 * 8 + 8  # + Wp, bp, scalar, d_k
    assert ctypes.sizeof(_lib.State) == 15 * 8 + 16


def test_sass_is_sm100a(lib):
    from paper_2603_20622_b200 import _lib
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_cpu_import_fails_loudly_without_gpu():
    import torch

    from paper_2603_20622_b200 import _lib, errors

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(errors.NativeError):
        _lib.load(require_cuda=True)
