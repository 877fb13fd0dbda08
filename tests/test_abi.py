"""C-ABI checks that need no GPU: the library loads, exports every symbol
include/hs.h declares, and rejects bad arguments on the host before any CUDA
call (include/hs.h "Validation happens before any launch")."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_2003_01216_b200 as hs
from paper_2003_01216_b200 import _build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
INVALID, UNSUPPORTED = 1, 2
FAKE = 0x10000  # never dereferenced: validation fails first


@pytest.fixture(scope="module")
def lib():
    _build.build()
    return hs.load()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "hs.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hs_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_paper_entry_points():
    syms = declared_symbols()
    for s in ("hs_msd_partition", "hs_sort_chunks", "hs_merge", "hs_sort", "hs_status_string"):
        assert s in syms
    assert set(syms) == set(hs.EXPORTED_SYMBOLS)


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", _build.SO], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\sT\s(\w+)$", out, flags=re.M))
    for s in declared_symbols():
        assert s in exported, s
        assert getattr(lib, s) is not None


def test_library_is_sm100a(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", _build.SO], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_abi_version_and_strings(lib):
    assert hs.abi_version() == 1
    names = [lib.hs_status_string(i).decode() for i in range(5)]
    assert names == ["HS_OK", "HS_ERR_INVALID_VALUE", "HS_ERR_UNSUPPORTED_DTYPE", "HS_ERR_OUT_OF_MEMORY", "HS_ERR_CUDA"]
    assert hs.tile_keys(0, 0) > 0 and hs.tile_keys(1, 2) > 0


def err(lib):
    return lib.hs_last_error_message().decode()


@pytest.mark.parametrize("args,code", [
    ((FAKE, -1, 0, 6, 8, None), INVALID),            # n < 0
    ((FAKE, 1 << 31, 0, 6, 8, None), INVALID),       # n >= 2^31
    ((FAKE, 10, 7, 6, 8, None), UNSUPPORTED),        # dtype
    ((FAKE, 10, 0, 0, 8, None), INVALID),            # D < 1
    ((FAKE, 10, 0, 11, 8, None), INVALID),           # D > 10 for int32
    ((FAKE, 10, 1, 20, 8, None), INVALID),           # D > 19 for int64
    ((FAKE, 10, 0, 6, 3, None), INVALID),            # c not a power of two
    ((FAKE, 10, 0, 6, 0, None), INVALID),            # c = 0
    ((FAKE, 10, 0, 6, 1 << 17, None), INVALID),      # c > 65536
    ((None, 10, 0, 6, 8, None), INVALID),            # NULL keys
    ((FAKE + 2, 10, 0, 6, 8, None), INVALID),        # misaligned int32
    ((FAKE + 4, 10, 1, 6, 8, None), INVALID),        # misaligned int64
])
def test_hs_sort_rejects(lib, args, code):
    assert lib.hs_sort(*args) == code
    assert err(lib)


def test_hs_sort_empty_is_ok_without_device(lib):
    assert lib.hs_sort(None, 0, 0, 6, 8, None) == 0
    assert hs.last_launch_count() == 0


def test_msd_partition_rejects(lib):
    assert lib.hs_msd_partition(FAKE, 10, 0, 3, FAKE + 4096, FAKE, None) == INVALID        # keys == out
    assert lib.hs_msd_partition(FAKE, 10, 0, 3, FAKE + 4096, FAKE + 8, None) == INVALID    # overlap
    assert lib.hs_msd_partition(FAKE, 10, 0, 3, None, FAKE + 4096, None) == INVALID        # no offsets
    assert lib.hs_msd_partition(FAKE, 10, 0, 3, FAKE + 4092, FAKE + 4096, None) == INVALID  # offsets misaligned
    assert lib.hs_msd_partition(FAKE, 10, 0, 12, FAKE + 8192, FAKE + 4096, None) == INVALID
    assert lib.hs_msd_partition(FAKE, 10, 3, 3, FAKE + 8192, FAKE + 4096, None) == UNSUPPORTED
    lib.hs_msd_partition(FAKE, 10, 0, 3, FAKE + 4096, FAKE + 8, None)
    assert "overlap" in err(lib)


@pytest.mark.parametrize("fn", ["hs_sort_chunks", "hs_merge"])
def test_chunks_merge_reject(lib, fn):
    f = getattr(lib, fn)
    assert f(FAKE, FAKE + 8, 10, 0, FAKE + 4096, 8, None) == INVALID          # partial overlap
    assert f(FAKE, FAKE + 4096, 10, 0, None, 8, None) == INVALID              # no offsets
    assert f(FAKE, FAKE + 4096, 10, 0, FAKE + 8192, 6, None) == INVALID       # c not pow2
    assert f(FAKE, FAKE + 4096, 10, 9, FAKE + 8192, 8, None) == UNSUPPORTED
    assert f(None, FAKE + 4096, 10, 0, FAKE + 8192, 8, None) == INVALID
    assert f(FAKE, FAKE, 0, 0, FAKE + 8192, 8, None) == 0                     # n = 0: no work


def test_python_binding_refuses_cpu_tensors():
    import torch
    with pytest.raises(ValueError):
        hs.hs_sort(torch.arange(10, dtype=torch.int32), 3)
    with pytest.raises((TypeError, ValueError)):
        hs.hs_sort(torch.arange(10, dtype=torch.float32), 3)


def test_missing_library_fails_loudly(tmp_path):
    with pytest.raises(RuntimeError):
        hs.load(str(tmp_path / "nope.so"))


class _FakeTensor:
    """Just the attributes the binding's argument checks read (no device needed)."""

    def __init__(self, dtype, numel, device="cuda:0"):
        import torch
        self.dtype, self._n, self.device, self.is_cuda = dtype, numel, torch.device(device), True

    def numel(self):
        return self._n

    def is_contiguous(self):
        return True


def test_binding_rejects_short_or_mismatched_out():
    """hs_sort_chunks / hs_merge write n * itemsize bytes into out (the C ABI takes n from x):
    the binding must refuse an out that is shorter, of another dtype or on another device."""
    import torch
    x = _FakeTensor(torch.int32, 1000)
    off = _FakeTensor(torch.int64, 11)
    hs._check_out(x, _FakeTensor(torch.int32, 1000), off)  # matching: accepted
    for bad in (_FakeTensor(torch.int32, 999), _FakeTensor(torch.int64, 1000), _FakeTensor(torch.int32, 1000, "cuda:1")):
        with pytest.raises(ValueError, match="out must match"):
            hs._check_out(x, bad, off)
    with pytest.raises(ValueError, match="bucket_offsets"):
        hs._check_out(x, _FakeTensor(torch.int32, 1000), _FakeTensor(torch.int64, 11, "cuda:1"))
    with pytest.raises(ValueError, match="bucket_offsets"):
        hs._check_out(x, _FakeTensor(torch.int32, 1000), _FakeTensor(torch.int32, 11))


def test_library_has_no_runtime_switches():
    """The C ABI's behaviour depends on its arguments only: no environment variable picks a path."""
    csrc = os.path.join(ROOT, "paper_2003_01216_b200", "csrc")
    for f in os.listdir(csrc):
        src = open(os.path.join(csrc, f)).read()
        assert "getenv" not in src, f  # (the statically linked cudart reads CUDA_* variables itself)
