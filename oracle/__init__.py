"""CPU oracle of the hybrid-sort hot path (arXiv 2003.01216) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  It shares no code with the
CUDA path (``paper_2003_01216_b200``) and never imports it.

The arithmetic lives in ``oracle/oracle.c`` (plain C, each function citing the
paper passage it follows); this module only marshals numpy arrays.  Keys are
widened to int64 before every call, and narrowed back for int32 callers.

Parity status: all functions pinned (tests/test_oracle.py); none unpinned.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import time

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_SO = os.path.join(_HERE, "liboracle.so")
_SO_OMP = os.path.join(_HERE, "liboracle_omp.so")

OK, ERR_KEY_OUT_OF_RANGE, ERR_BAD_DIGITS, ERR_NOT_POW2, ERR_NOMEM = 0, 1, 2, 3, 4


class KeyOutOfRange(ValueError):
    """a key outside [0, 10^D) in strict mode."""

    def __init__(self, index: int):
        super().__init__(f"key at index {index} is outside [0, 10^D)")
        self.index = index


def build(force: bool = False) -> None:
    """gcc -O2 builds of the oracle: plain (the oracle) and -fopenmp (timing)."""
    for so, extra in ((_SO, []), (_SO_OMP, ["-fopenmp"])):
        if force or not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(_SRC):
            subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", *extra, "-o", so, _SRC])


_libs: dict = {}


def _lib(openmp: bool = False):
    key = bool(openmp)
    if key not in _libs:
        build()
        lib = ctypes.CDLL(_SO_OMP if openmp else _SO)
        i64, vp, ci = ctypes.c_int64, ctypes.c_void_p, ctypes.c_int
        lib.oracle_digit.argtypes = [i64, ci, ci, ctypes.POINTER(ci)]
        lib.oracle_digit.restype = ci
        lib.oracle_msd_partition.argtypes = [vp, i64, ci, ci, vp, vp, ctypes.POINTER(i64)]
        lib.oracle_msd_partition.restype = ci
        lib.oracle_partition_even.argtypes = [i64, i64, vp]
        lib.oracle_partition_even.restype = ci
        lib.oracle_merge_schedule.argtypes = [i64, vp]
        lib.oracle_merge_schedule.restype = i64
        lib.oracle_quicksort.argtypes = [vp, i64]
        lib.oracle_quicksort.restype = None
        lib.oracle_merge_runs.argtypes = [vp, i64, vp, i64, vp]
        lib.oracle_merge_runs.restype = None
        lib.oracle_sort_chunks.argtypes = [vp, vp, i64, vp, i64]
        lib.oracle_sort_chunks.restype = ci
        lib.oracle_merge.argtypes = [vp, vp, i64, vp, i64]
        lib.oracle_merge.restype = ci
        lib.oracle_sort.argtypes = [vp, i64, ci, i64, ci, ctypes.POINTER(i64)]
        lib.oracle_sort.restype = ci
        lib.oracle_msd_partition_pairs.argtypes = [vp, vp, i64, ci, vp, vp, vp]
        lib.oracle_msd_partition_pairs.restype = ci
        lib.oracle_sort_pairs.argtypes = [vp, vp, i64, ci, i64]
        lib.oracle_sort_pairs.restype = ci
        lib.oracle_sort_chunks_pairs.argtypes = [vp, vp, i64, vp, i64]
        lib.oracle_sort_chunks_pairs.restype = ci
        lib.oracle_merge_pairs.argtypes = [vp, vp, i64, vp, i64]
        lib.oracle_merge_pairs.restype = ci
        lib.oracle_sort_shared.argtypes = [vp, i64, i64]
        lib.oracle_sort_shared.restype = ci
        lib.oracle_openmp_threads.argtypes = []
        lib.oracle_openmp_threads.restype = ci
        _libs[key] = lib
    return _libs[key]


def _w(a) -> np.ndarray:
    """Widen to a fresh contiguous int64 array."""
    return np.ascontiguousarray(np.asarray(a), dtype=np.int64).copy()


def _p(a: np.ndarray) -> int:
    return a.ctypes.data


def _check(rc: int, bad: int | None = None) -> None:
    if rc == OK:
        return
    if rc == ERR_KEY_OUT_OF_RANGE:
        raise KeyOutOfRange(bad if bad is not None else -1)
    if rc == ERR_BAD_DIGITS:
        raise ValueError("num_digits outside [1, 19]")
    if rc == ERR_NOT_POW2:
        raise ValueError("worker/chunk count must be a power of two (P:80)")
    raise MemoryError("oracle allocation failed")


def max_digits(dtype) -> int:
    """D limit per dtype: 10 for int32, 19 for int64 (keys < 10^D must fit)."""
    return 10 if np.dtype(dtype) == np.int32 else 19


def digit(key: int, num_digits: int, strict: bool = False) -> int:
    d = ctypes.c_int(-1)
    _check(_lib().oracle_digit(int(key), num_digits, int(strict), ctypes.byref(d)), 0)
    return d.value


def msd_partition(keys, num_digits: int, strict: bool = False):
    """(out, offsets[11]) of the stable one-step MSD partition."""
    src = np.asarray(keys)
    k = _w(src)
    out = np.empty_like(k)
    off = np.zeros(11, dtype=np.int64)
    bad = ctypes.c_int64(-1)
    _check(_lib().oracle_msd_partition(_p(k), k.size, num_digits, int(strict), _p(off), _p(out), ctypes.byref(bad)), bad.value)
    return out.astype(src.dtype if src.size else np.int64), off


def histogram(keys, num_digits: int) -> np.ndarray:
    _, off = msd_partition(keys, num_digits)
    return np.diff(off)


def partition_even(m: int, p: int) -> list[int]:
    lens = np.zeros(max(p, 1), dtype=np.int64)
    _check(_lib().oracle_partition_even(m, p, _p(lens)))
    return lens.tolist()


def merge_schedule(p: int) -> list[tuple[int, int, int]]:
    k = _lib().oracle_merge_schedule(p, None)
    if k < 0:
        raise ValueError("p must be a power of two (P:58)")
    t = np.zeros(3 * k + 1, dtype=np.int64)
    _lib().oracle_merge_schedule(p, _p(t))
    return [tuple(int(x) for x in t[3 * i:3 * i + 3]) for i in range(k)]


def quicksort(keys) -> np.ndarray:
    src = np.asarray(keys)
    k = _w(src)
    _lib().oracle_quicksort(_p(k), k.size)
    return k.astype(src.dtype) if src.size else k


def merge_runs(left, right) -> np.ndarray:
    a, b = _w(left), _w(right)
    out = np.empty(a.size + b.size, dtype=np.int64)
    _lib().oracle_merge_runs(_p(a), a.size, _p(b), b.size, _p(out))
    return out


def sort_chunks(x, offsets, chunks: int, openmp: bool = False) -> np.ndarray:
    src = np.asarray(x)
    k = _w(src)
    off = _w(offsets)
    _check(_lib(openmp).oracle_sort_chunks(_p(k), _p(k), k.size, _p(off), chunks))
    return k.astype(src.dtype)


def merge(x, offsets, chunks: int, openmp: bool = False) -> np.ndarray:
    src = np.asarray(x)
    k = _w(src)
    off = _w(offsets)
    _check(_lib(openmp).oracle_merge(_p(k), _p(k), k.size, _p(off), chunks))
    return k.astype(src.dtype)


def sort(keys, num_digits: int, chunks: int = 8, strict: bool = False, openmp: bool = False) -> np.ndarray:
    """Whole path (P:76-84 with one node): partition -> chunk quicksort -> tree merge."""
    src = np.asarray(keys)
    k = _w(src)
    bad = ctypes.c_int64(-1)
    _check(_lib(openmp).oracle_sort(_p(k), k.size, num_digits, chunks, int(strict), ctypes.byref(bad)), bad.value)
    return k.astype(src.dtype)


def sort_shared(keys, chunks: int = 8, openmp: bool = False) -> np.ndarray:
    """No-MSD ablation: chunk quicksort + tree merge of the whole array."""
    src = np.asarray(keys)
    k = _w(src)
    _check(_lib(openmp).oracle_sort_shared(_p(k), k.size, chunks))
    return k.astype(src.dtype)


def msd_partition_pairs(keys, tags, num_digits: int):
    """f3: stable MSD partition of (key, tag) items.  Returns (out_keys, out_tags, offsets11)."""
    src = np.asarray(keys)
    k = _w(src)
    t = np.ascontiguousarray(np.asarray(tags).astype(np.uint64))
    ok = np.empty_like(k)
    ot = np.empty_like(t)
    off = np.zeros(11, dtype=np.int64)
    _check(_lib().oracle_msd_partition_pairs(_p(k), _p(t), k.size, num_digits, _p(off), _p(ok), _p(ot)))
    return ok.astype(src.dtype), ot, off


def sort_pairs(keys, tags, num_digits: int, chunks: int = 8):
    """f3: stable sort of (key, tag) items: MSD partition -> Fig 1b merge sort per chunk -> tree merge."""
    src = np.asarray(keys)
    k = _w(src)
    t = np.ascontiguousarray(np.asarray(tags).astype(np.uint64)).copy()
    _check(_lib().oracle_sort_pairs(_p(k), _p(t), k.size, num_digits, chunks))
    return k.astype(src.dtype), t


def sort_chunks_pairs(keys, tags, offsets, chunks: int):
    """f3, a5 on items: each chunk sorted stably (Fig 1b merge sort).  Returns (keys, tags)."""
    src = np.asarray(keys)
    k = _w(src)
    t = np.ascontiguousarray(np.asarray(tags).astype(np.uint64)).copy()
    off = _w(offsets)
    _check(_lib().oracle_sort_chunks_pairs(_p(k), _p(t), k.size, _p(off), chunks))
    return k.astype(src.dtype), t


def merge_pairs(keys, tags, offsets, chunks: int):
    """f3, a6 on items: tree merge of each bucket's chunk runs, stable-left.  Returns (keys, tags)."""
    src = np.asarray(keys)
    k = _w(src)
    t = np.ascontiguousarray(np.asarray(tags).astype(np.uint64)).copy()
    off = _w(offsets)
    _check(_lib().oracle_merge_pairs(_p(k), _p(t), k.size, _p(off), chunks))
    return k.astype(src.dtype), t


def timed_sort(keys, num_digits: int, chunks: int = 8, openmp: bool = False):
    """(sorted, seconds, threads): wall time of the oracle sort call only."""
    src = np.asarray(keys)
    k = _w(src)
    bad = ctypes.c_int64(-1)
    lib = _lib(openmp)
    t0 = time.perf_counter()
    rc = lib.oracle_sort(_p(k), k.size, num_digits, chunks, 0, ctypes.byref(bad))
    dt = time.perf_counter() - t0
    _check(rc, bad.value)
    return k.astype(src.dtype), dt, int(lib.oracle_openmp_threads())
