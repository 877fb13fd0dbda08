"""Seeded synthetic inputs for the hybrid-sort hot path (tests and bench only).

Holds none of the sort method's arithmetic; it only produces keys.  The recipe
is SURVEY.md §8(d) (a counter-form splitmix64, with a
multiply-high range map), standing in for the paper's "data ... generated
randomly" (§4.2).  There is no public dataset in the paper.

Two independent implementations are kept and cross-checked in
tests/test_workload.py:
  * ``libworkload.so`` (workload/gen.c, OpenMP) -- fast, used for big configs;
  * ``*_np`` numpy twins -- used to pin the C code on prefixes.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libworkload.so")
_SRC = os.path.join(_HERE, "gen.c")

GOLDEN = 0x9E3779B97F4A7C15
M64 = (1 << 64) - 1


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    dtype: str          # "int32" | "int64"
    seed: int
    kind: str           # "uniform" | "mixture"
    value_range: int    # uniform keys in [0, value_range)
    num_digits: int     # D: MSD digit = floor(k / 10^(D-1))
    chunks: int         # chunks per bucket (paper's threads per node)
    value_lo: int = 0   # uniform keys are value_lo + [0, value_range)


# BASELINE.json configs[0..4]; D per SURVEY §8(c) reading #2, c = 8 per reading #6.
CONFIGS = {
    "C1": Config("C1", 1_048_576, "int32", 1, "uniform", 10**6, 6, 8),
    "C2": Config("C2", 16_777_216, "int32", 2, "uniform", 10**9, 9, 8),
    "C3": Config("C3", 268_435_456, "int32", 3, "uniform", 10**9, 9, 8),
    "C4": Config("C4", 67_108_864, "int32", 4, "mixture", 10**9, 9, 8),
    "C5": Config("C5", 536_870_912, "int64", 5, "uniform", 10**18, 18, 8),
    # SURVEY §8(f) f4, the paper's own workload: "each number consists of three
    # digits", i.e. [100, 999], n up to 1e7; 900 distinct
    # values, bucket 0 empty.  Not a BASELINE.json config.
    "P3": Config("P3", 10_000_000, "int32", 6, "uniform", 900, 3, 8, value_lo=100),
}


def build(force: bool = False) -> str:
    """Compile libworkload.so with gcc -O2 -fopenmp (host code only)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", _SO, _SRC])
    return _SO


_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        u64, i64, vp = ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p
        lib.wl_splitmix_output.restype = u64
        lib.wl_splitmix_output.argtypes = [u64, u64]
        lib.wl_mix64.restype = u64
        lib.wl_mix64.argtypes = [u64]
        lib.wl_uniform_i32.argtypes = [vp, u64, u64, i64, i64]
        lib.wl_uniform_i64.argtypes = [vp, u64, u64, i64, i64]
        lib.wl_mixture_i32.argtypes = [vp, u64, i64, i64, i64]
        lib.wl_mixture_table.argtypes = [u64, i64, vp]
        _lib = lib
    return _lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def generate(cfg: Config | str, start: int = 0, count: int | None = None, out: np.ndarray | None = None) -> np.ndarray:
    """Keys [start, start+count) of config ``cfg`` (C implementation)."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    if count is None:
        count = cfg.n - start
    lib = _load()
    dt = np.int32 if cfg.dtype == "int32" else np.int64
    if out is None:
        out = np.empty(count, dtype=dt)
    assert out.dtype == dt and out.flags.c_contiguous and out.size >= count
    if cfg.kind == "uniform":
        fn = lib.wl_uniform_i32 if cfg.dtype == "int32" else lib.wl_uniform_i64
        fn(_ptr(out), cfg.seed, cfg.value_range, start, count)
        if cfg.value_lo:
            out[:count] += cfg.value_lo
    else:
        assert cfg.dtype == "int32"
        lib.wl_mixture_i32(_ptr(out), cfg.seed, cfg.n, start, count)
    return out


def uniform(n: int, seed: int, value_range: int, dtype=np.int32) -> np.ndarray:
    """Ad-hoc uniform keys in [0, value_range) (C implementation)."""
    lib = _load()
    out = np.empty(n, dtype=dtype)
    fn = lib.wl_uniform_i32 if out.dtype == np.int32 else lib.wl_uniform_i64
    fn(_ptr(out), seed, value_range, 0, n)
    return out


def splitmix_output(seed: int, j: int) -> int:
    return int(_load().wl_splitmix_output(seed, j))


def mixture_table(cfg: Config | str) -> np.ndarray:
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    t = np.empty(1024, dtype=np.int64)
    _load().wl_mixture_table(cfg.seed, cfg.n, _ptr(t))
    return t


# ---------------------------------------------------------------- numpy twin
def mix_np(z: np.ndarray) -> np.ndarray:
    z = z.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        z ^= z >> np.uint64(30)
        z *= np.uint64(0xBF58476D1CE4E5B9)
        z ^= z >> np.uint64(27)
        z *= np.uint64(0x94D049BB133111EB)
        z ^= z >> np.uint64(31)
    return z


def out_np(seed: int, j: np.ndarray) -> np.ndarray:
    j = np.asarray(j, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return mix_np(np.uint64(seed) + (j + np.uint64(1)) * np.uint64(GOLDEN))


def mulhi_np(x: np.ndarray, r: int) -> np.ndarray:
    """floor(x * r / 2^64) for uint64 arrays, via 32-bit limbs."""
    x = np.asarray(x, dtype=np.uint64)
    m = np.uint64(0xFFFFFFFF)
    s = np.uint64(32)
    xl, xh = x & m, x >> s
    rl, rh = np.uint64(r & 0xFFFFFFFF), np.uint64(r >> 32)
    with np.errstate(over="ignore"):
        ll = xl * rl
        hl = xh * rl
        lh = xl * rh
        hh = xh * rh
        cross = (ll >> s) + (hl & m) + lh
        return hh + (hl >> s) + (cross >> s)


def generate_np(cfg: Config | str, start: int = 0, count: int | None = None) -> np.ndarray:
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    if count is None:
        count = cfg.n - start
    dt = np.int32 if cfg.dtype == "int32" else np.int64
    idx = np.arange(start, start + count, dtype=np.uint64)
    if cfg.kind == "uniform":
        return (mulhi_np(out_np(cfg.seed, idx), cfg.value_range).astype(np.int64) + cfg.value_lo).astype(dt)
    table = mulhi_np(out_np(cfg.seed, np.uint64(8 * cfg.n) + np.arange(1024, dtype=np.uint64)), 10**9).astype(np.int64)
    w = [out_np(cfg.seed, np.uint64(8) * idx + np.uint64(j)) for j in range(8)]
    sel = mulhi_np(w[0], 100)
    s = np.zeros(count, dtype=np.uint64)
    for j in range(1, 7):
        s += (w[j] >> np.uint64(32)) + (w[j] & np.uint64(0xFFFFFFFF))
    z = s.astype(np.int64) - np.int64(6 << 32)
    normal = np.clip(300_000_000 + ((z * 20_000_000) >> 32), 0, 999_999_999)
    from_table = table[(w[7] >> np.uint64(54)).astype(np.int64)]
    unif = mulhi_np(w[7], 10**9).astype(np.int64)
    v = np.where(sel < 70, normal, np.where(sel < 90, from_table, unif))
    return v.astype(dt)


def fingerprint(keys: np.ndarray) -> dict:
    """Multiset fingerprint over u64(k): count, sum64, xor64, mix64."""
    u = keys.astype(np.int64).view(np.uint64)
    with np.errstate(over="ignore"):
        s = int(np.sum(u, dtype=np.uint64))
        m = int(np.sum(mix_np(u), dtype=np.uint64))
    x = int(np.bitwise_xor.reduce(u)) if u.size else 0
    return {"count": int(keys.size), "sum64": s, "xor64": x, "mix64": m}
