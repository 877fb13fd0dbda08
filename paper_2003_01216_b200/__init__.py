"""paper_2003_01216_b200 -- B200-native hot path of the hybrid MSD-radix /
quicksort / merge sort of arXiv 2003.01216 (§3.4).

A thin ctypes binding over libhybridsort.so (C ABI: include/hs.h).  This
module only marshals arguments: tensors -> device pointers, the current torch
CUDA stream -> cudaStream_t, status codes -> exceptions.  Every step of the
method runs in the library's sm_100a kernels.  There is no CPU fallback: if
the library is missing, or a tensor is not on a CUDA device, calls raise.

Names follow the C ABI (hs_msd_partition, hs_sort_chunks, hs_merge,
hs_sort); msd_partition / sort_chunks / merge / sort are aliases.
"""
from __future__ import annotations

import ctypes
import os

from . import _build

__all__ = [
    "HS_INT32", "HS_INT64", "HybridSortError", "library_path", "load",
    "hs_msd_partition", "hs_sort_chunks", "hs_merge", "hs_sort", "hs_sort_shared", "hs_sort_plan", "hs_sort_buckets", "hs_sort_host",
    "msd_partition", "sort_chunks", "merge", "sort", "sort_shared", "sort_host",
    "hs_msd_partition_pairs", "hs_sort_pairs", "msd_partition_pairs", "sort_pairs",
    "hs_sort_chunks_pairs", "hs_merge_pairs", "sort_chunks_pairs", "merge_pairs",
    "abi_version", "tile_keys", "last_launch_count", "EXPORTED_SYMBOLS", "HostSortPipeline", "PartitionPlan", "SortGraph",
]

HS_INT32, HS_INT64 = 0, 1
STATUS = {0: "HS_OK", 1: "HS_ERR_INVALID_VALUE", 2: "HS_ERR_UNSUPPORTED_DTYPE", 3: "HS_ERR_OUT_OF_MEMORY", 4: "HS_ERR_CUDA"}
EXPORTED_SYMBOLS = (
    "hs_msd_partition", "hs_sort_chunks", "hs_merge", "hs_sort", "hs_sort_shared", "hs_status_string",
    "hs_last_error_message", "hs_abi_version", "hs_last_launch_count", "hs_tile_keys",
    "hs_profile_enable", "hs_profile_read", "hs_profile_kind_name", "hs_plan_levels", "hs_assign_buckets",
    "hs_msd_partition_pairs", "hs_sort_pairs",
    "hs_partition_plan_create", "hs_partition_scatter", "hs_partition_plan_destroy", "hs_sort_plan",
    "hs_sort_buckets", "hs_sort_pairs64", "hs_msd_partition_pairs64", "hs_sort_chunks_pairs", "hs_merge_pairs",
)
PROFILE_KINDS = ("tile_hist", "tile_scan", "scatter", "plan", "tile_sort", "merge_partition", "merge_level", "copy",
                 "split_count", "split_scatter")


class HybridSortError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{STATUS.get(status, status)}: {message}")
        self.status = status


def library_path() -> str:
    return _build.SO


_LIB = None


def load(path: str | None = None):
    """Load libhybridsort.so (raises if it has not been built)."""
    global _LIB
    if _LIB is not None and path is None:
        return _LIB
    p = path or _build.SO
    if not os.path.exists(p):
        raise RuntimeError(f"{p} is missing: build it with `python -m paper_2003_01216_b200._build` "
                           "or __graft_entry__.build(); there is no CPU fallback")
    lib = ctypes.CDLL(p)
    vp, i64, ci = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
    lib.hs_msd_partition.argtypes = [vp, i64, ci, ci, vp, vp, vp]
    lib.hs_sort_chunks.argtypes = [vp, vp, i64, ci, vp, ci, vp]
    lib.hs_merge.argtypes = [vp, vp, i64, ci, vp, ci, vp]
    lib.hs_sort.argtypes = [vp, i64, ci, ci, ci, vp]
    lib.hs_sort_shared.argtypes = [vp, i64, ci, ci, vp]
    lib.hs_sort_plan.argtypes = [vp, i64, ci, ci, ci, vp, vp, vp, vp]
    lib.hs_sort_buckets.argtypes = [vp, i64, ci, ci, vp, ci, vp]
    lib.hs_msd_partition_pairs.argtypes = [vp, vp, i64, ci, vp, vp, vp, vp]
    lib.hs_sort_pairs.argtypes = [vp, vp, i64, ci, ci, vp]
    lib.hs_sort_pairs64.argtypes = [vp, vp, i64, ci, ci, vp]
    lib.hs_msd_partition_pairs64.argtypes = [vp, vp, i64, ci, vp, vp, vp, vp]
    lib.hs_sort_chunks_pairs.argtypes = [vp, vp, vp, vp, i64, ci, vp, ci, vp]
    lib.hs_merge_pairs.argtypes = [vp, vp, vp, vp, i64, ci, vp, ci, vp]
    for f in ("hs_msd_partition", "hs_sort_chunks", "hs_merge", "hs_sort", "hs_sort_shared",
              "hs_msd_partition_pairs", "hs_sort_pairs", "hs_sort_plan", "hs_sort_buckets", "hs_sort_pairs64",
              "hs_msd_partition_pairs64", "hs_sort_chunks_pairs", "hs_merge_pairs"):
        getattr(lib, f).restype = ci
    lib.hs_status_string.argtypes = [ci]
    lib.hs_status_string.restype = ctypes.c_char_p
    lib.hs_last_error_message.argtypes = []
    lib.hs_last_error_message.restype = ctypes.c_char_p
    lib.hs_abi_version.restype = ci
    lib.hs_last_launch_count.restype = ci
    lib.hs_tile_keys.argtypes = [ci, ci]
    lib.hs_tile_keys.restype = ci
    lib.hs_profile_enable.argtypes = [ci]
    lib.hs_profile_enable.restype = ci
    lib.hs_profile_read.argtypes = [vp, vp, ci]
    lib.hs_profile_read.restype = ci
    lib.hs_profile_kind_name.argtypes = [ci]
    lib.hs_profile_kind_name.restype = ctypes.c_char_p
    lib.hs_plan_levels.argtypes = [vp, ci, ci, ci, vp, vp]
    lib.hs_plan_levels.restype = ci
    lib.hs_assign_buckets.argtypes = [vp, ci, vp, vp]
    lib.hs_assign_buckets.restype = ci
    lib.hs_partition_plan_create.argtypes = [vp, i64, ci, ci, vp, ctypes.POINTER(vp), vp]
    lib.hs_partition_plan_create.restype = ci
    lib.hs_partition_scatter.argtypes = [vp, ctypes.POINTER(vp), vp]
    lib.hs_partition_scatter.restype = ci
    lib.hs_partition_plan_destroy.argtypes = [vp, vp]
    lib.hs_partition_plan_destroy.restype = ci
    if path is None:
        _LIB = lib
    return lib


def _check(rc: int) -> None:
    if rc != 0:
        msg = load().hs_last_error_message().decode(errors="replace")
        raise HybridSortError(rc, msg)


def abi_version() -> int:
    return int(load().hs_abi_version())


def last_launch_count() -> int:
    """Kernel launches enqueued by the last successful call on this thread."""
    return int(load().hs_last_launch_count())


def tile_keys(dtype_code: int, which: int) -> int:
    return int(load().hs_tile_keys(dtype_code, which))


def profile_enable(on: bool = True) -> None:
    """Bracket every library kernel with CUDA events on its stream (this thread)."""
    load().hs_profile_enable(1 if on else 0)


def profile_read() -> dict:
    """{kind: (total_ms, launches)} since the last read (synchronises)."""
    import numpy as np
    n = len(PROFILE_KINDS)
    ms = np.zeros(n, dtype=np.float64)
    cnt = np.zeros(n, dtype=np.int32)
    if load().hs_profile_read(ms.ctypes.data, cnt.ctypes.data, n) != 0:
        raise HybridSortError(4, "event timing failed")
    return {PROFILE_KINDS[i]: (float(ms[i]), int(cnt[i])) for i in range(n)}


def plan_levels(bucket_offsets_host, dtype_code: int, chunks: int, mode: int = 0):
    """(levels[10], tile_levels[10]) of the device plan, computed on the host."""
    import numpy as np
    off = np.ascontiguousarray(np.asarray(bucket_offsets_host, dtype=np.int64))
    L = np.zeros(10, dtype=np.int32)
    k = np.zeros(10, dtype=np.int32)
    if load().hs_plan_levels(off.ctypes.data, dtype_code, chunks, mode, L.ctypes.data, k.ctypes.data) < 0:
        raise ValueError("bad plan arguments")
    return L.tolist(), k.tolist()


def assign_buckets(bucket_sizes, nodes: int):
    """Contiguous digit groups for `nodes` nodes: (group_start[nodes+1], max_load)."""
    import numpy as np
    sizes = np.ascontiguousarray(np.asarray(bucket_sizes, dtype=np.int64))
    if sizes.size != 10:
        raise ValueError("bucket_sizes must have 10 entries")
    gs = np.zeros(nodes + 1 if 1 <= nodes <= 10 else 1, dtype=np.int32)
    ml = np.zeros(1, dtype=np.int64)
    _check(load().hs_assign_buckets(sizes.ctypes.data, nodes, gs.ctypes.data, ml.ctypes.data))
    return gs.tolist(), int(ml[0])


# ------------------------------------------------------------ tensor glue
def _torch():
    import torch
    return torch


def _dtype_code(t) -> int:
    torch = _torch()
    if t.dtype == torch.int32:
        return HS_INT32
    if t.dtype == torch.int64:
        return HS_INT64
    raise TypeError(f"keys must be torch.int32 or torch.int64, got {t.dtype}")


def _check_tensor(t, name: str) -> None:
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


def _stream(stream) -> int:
    torch = _torch()
    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream) if hasattr(stream, "cuda_stream") else int(stream)


def _validate_range(keys, num_digits: int) -> None:
    """SPEC S:294 KeyOutOfRange: optional check that 0 <= k < 10^D (reading #3)."""
    torch = _torch()
    hi = 10 ** num_digits
    bad = (keys < 0) | (keys >= hi) if hi <= torch.iinfo(keys.dtype).max else (keys < 0)
    if bool(bad.any()):
        idx = int(torch.nonzero(bad)[0, 0])
        raise ValueError(f"key at index {idx} ({int(keys[idx])}) is outside [0, 10^{num_digits})")


def hs_msd_partition(keys, num_digits: int, out=None, bucket_offsets=None, stream=None, validate: bool = False):
    """Stable one-step MSD partition.  Returns (out, bucket_offsets[11])."""
    torch = _torch()
    _check_tensor(keys, "keys")
    dt = _dtype_code(keys)
    if validate:
        _validate_range(keys, num_digits)
    if out is None:
        out = torch.empty_like(keys)
    if bucket_offsets is None:
        bucket_offsets = torch.empty(11, dtype=torch.int64, device=keys.device)
    _check_tensor(out, "out")
    _check_tensor(bucket_offsets, "bucket_offsets")
    if out.dtype != keys.dtype or out.numel() != keys.numel() or out.device != keys.device:
        raise ValueError("out must match keys in dtype, size and device")
    if bucket_offsets.dtype != torch.int64 or bucket_offsets.numel() != 11 or bucket_offsets.device != keys.device:
        raise ValueError("bucket_offsets must be an int64 tensor of 11 elements on the keys' device")
    with torch.cuda.device(keys.device):
        _check(load().hs_msd_partition(keys.data_ptr(), keys.numel(), dt, num_digits, bucket_offsets.data_ptr(),
                                       out.data_ptr(), _stream(stream)))
    return out, bucket_offsets


def _check_out(x, out, bucket_offsets) -> None:
    """out must match x in dtype, size and device (the library writes n * itemsize bytes
    into it); bucket_offsets must be int64[11] on x's device (the kernels read it)."""
    torch = _torch()
    _check_tensor(out, "out")
    _check_tensor(bucket_offsets, "bucket_offsets")
    if out.dtype != x.dtype or out.numel() != x.numel() or out.device != x.device:
        raise ValueError(f"out must match x in dtype, size and device: got {out.dtype}[{out.numel()}] on "
                         f"{out.device} for {x.dtype}[{x.numel()}] on {x.device}")
    if bucket_offsets.dtype != torch.int64 or bucket_offsets.numel() != 11 or bucket_offsets.device != x.device:
        raise ValueError("bucket_offsets must be an int64 tensor of 11 elements on x's device")


def hs_sort_chunks(x, bucket_offsets, chunks_per_bucket: int = 8, out=None, stream=None):
    """Sort every chunk of every bucket.  out=x sorts in place."""
    torch = _torch()
    _check_tensor(x, "x")
    dt = _dtype_code(x)
    if out is None:
        out = torch.empty_like(x)
    _check_out(x, out, bucket_offsets)
    with torch.cuda.device(x.device):
        _check(load().hs_sort_chunks(x.data_ptr(), out.data_ptr(), x.numel(), dt, bucket_offsets.data_ptr(),
                                     chunks_per_bucket, _stream(stream)))
    return out


def hs_merge(x, bucket_offsets, chunks_per_bucket: int = 8, out=None, stream=None):
    """Binary-tree merge of each bucket's sorted chunks.  out=x merges in place."""
    torch = _torch()
    _check_tensor(x, "x")
    dt = _dtype_code(x)
    if out is None:
        out = torch.empty_like(x)
    _check_out(x, out, bucket_offsets)
    with torch.cuda.device(x.device):
        _check(load().hs_merge(x.data_ptr(), out.data_ptr(), x.numel(), dt, bucket_offsets.data_ptr(),
                               chunks_per_bucket, _stream(stream)))
    return out


def hs_sort(keys, num_digits: int, chunks_per_bucket: int = 8, stream=None, validate: bool = False):
    """Whole path in place: partition -> chunk sort -> tree merge.  Returns keys."""
    torch = _torch()
    _check_tensor(keys, "keys")
    dt = _dtype_code(keys)
    if validate:
        _validate_range(keys, num_digits)
    with torch.cuda.device(keys.device):
        _check(load().hs_sort(keys.data_ptr(), keys.numel(), dt, num_digits, chunks_per_bucket, _stream(stream)))
    return keys


def hs_sort_buckets(keys, bucket_offsets, num_digits: int, chunks_per_bucket: int = 8, stream=None):
    """Sort every bucket of an already digit-partitioned array in place (a4-a7 of hs_sort
    without the partition; the f2 receive side).  bucket_offsets: device int64[11]."""
    torch = _torch()
    _check_tensor(keys, "keys")
    dt = _dtype_code(keys)
    if bucket_offsets.dtype != torch.int64 or bucket_offsets.numel() != 11 or bucket_offsets.device != keys.device:
        raise ValueError("bucket_offsets must be an int64 tensor of 11 entries on the keys' device")
    off = bucket_offsets.contiguous()
    with torch.cuda.device(keys.device):
        _check(load().hs_sort_buckets(keys.data_ptr(), keys.numel(), dt, num_digits, off.data_ptr(),
                                      chunks_per_bucket, _stream(stream)))
    return keys


def hs_sort_plan(keys, num_digits: int, chunks_per_bucket: int = 8, stream=None):
    """The plan hs_sort would run on keys (keys unchanged): dict of per-bucket
    merge levels, K5a split flags (and whether the split used the padded
    layout) and tile-sort leaves per chunk."""
    import numpy as np
    torch = _torch()
    _check_tensor(keys, "keys")
    dt = _dtype_code(keys)
    L = np.zeros(10, dtype=np.int32)
    sp = np.zeros(10, dtype=np.int32)
    lv = np.zeros(10, dtype=np.int32)
    with torch.cuda.device(keys.device):
        _check(load().hs_sort_plan(keys.data_ptr(), keys.numel(), dt, num_digits, chunks_per_bucket,
                                   L.ctypes.data, sp.ctypes.data, lv.ctypes.data, _stream(stream)))
    return {"levels": L.tolist(), "split": [int(v != 0) for v in sp.tolist()],
            "padded": [int(v == 2) for v in sp.tolist()], "leaves": lv.tolist()}


def hs_sort_shared(keys, chunks: int = 8, stream=None):
    """No-MSD ablation: the paper's Shared-Parallel Hybrid
    Quicksort + Merge Sort (§3.2) on the whole array, in place."""
    torch = _torch()
    _check_tensor(keys, "keys")
    dt = _dtype_code(keys)
    with torch.cuda.device(keys.device):
        _check(load().hs_sort_shared(keys.data_ptr(), keys.numel(), dt, chunks, _stream(stream)))
    return keys


def _check_pairs(keys, tags, int32_only: bool = False):
    torch = _torch()
    _check_tensor(keys, "keys")
    _check_tensor(tags, "tags")
    if int32_only and keys.dtype != torch.int32:
        raise TypeError("keys must be torch.int32 here")
    if keys.dtype not in (torch.int32, torch.int64):
        raise TypeError(f"keys must be torch.int32 or torch.int64, got {keys.dtype}")
    if tags.element_size() != 8 or tags.numel() != keys.numel() or tags.device != keys.device:
        raise ValueError("tags must be a 64-bit tensor with one tag per key, on the keys' device")


def hs_msd_partition_pairs(keys, tags, num_digits: int, stream=None):
    """f3: stable MSD partition of (key, tag) items: within a bucket items keep
    their input order.  int32 keys: (key << 32 | index) items; int64 keys: the KV item path
    (hs_msd_partition_pairs64).  Returns (out_keys, out_tags, bucket_offsets)."""
    torch = _torch()
    _check_pairs(keys, tags)
    out_k = torch.empty_like(keys)
    out_t = torch.empty_like(tags)
    off = torch.empty(11, dtype=torch.int64, device=keys.device)
    fn = load().hs_msd_partition_pairs if keys.dtype == torch.int32 else load().hs_msd_partition_pairs64
    with torch.cuda.device(keys.device):
        _check(fn(keys.data_ptr(), tags.data_ptr(), keys.numel(), num_digits, off.data_ptr(), out_k.data_ptr(),
                  out_t.data_ptr(), _stream(stream)))
    return out_k, out_t, off


def hs_sort_pairs(keys, tags, num_digits: int, chunks_per_bucket: int = 8, stream=None):
    """f3: stable sort of (key, tag) items in place (ties keep input order).  int32 keys go
    through the keys path as (key << 32 | index) items (K5a split included) and the tags follow
    their index; int64 keys through the stable KV item path (hs_sort_pairs64: tags travel with
    their keys).  Returns (keys, tags)."""
    torch = _torch()
    _check_pairs(keys, tags)
    fn = load().hs_sort_pairs if keys.dtype == torch.int32 else load().hs_sort_pairs64
    with torch.cuda.device(keys.device):
        _check(fn(keys.data_ptr(), tags.data_ptr(), keys.numel(), num_digits, chunks_per_bucket, _stream(stream)))
    return keys, tags


def _pairs_outputs(keys, tags, bucket_offsets, out_keys, out_tags):
    torch = _torch()
    _check_pairs(keys, tags)
    if out_keys is None:
        out_keys = torch.empty_like(keys)
    if out_tags is None:
        out_tags = torch.empty_like(tags)
    _check_pairs(out_keys, out_tags)
    _check_out(keys, out_keys, bucket_offsets)
    if out_tags.numel() != tags.numel() or out_tags.device != tags.device:
        raise ValueError("out_tags must match tags in size and device")
    return out_keys, out_tags


def hs_sort_chunks_pairs(keys, tags, bucket_offsets, chunks_per_bucket: int = 8, out_keys=None, out_tags=None,
                         stream=None):
    """f3, a5 on items: every chunk of every bucket sorted stably (KV item path).  In place when
    out_keys / out_tags are keys / tags.  Returns (out_keys, out_tags)."""
    torch = _torch()
    out_keys, out_tags = _pairs_outputs(keys, tags, bucket_offsets, out_keys, out_tags)
    with torch.cuda.device(keys.device):
        _check(load().hs_sort_chunks_pairs(keys.data_ptr(), tags.data_ptr(), out_keys.data_ptr(), out_tags.data_ptr(),
                                           keys.numel(), _dtype_code(keys), bucket_offsets.data_ptr(),
                                           chunks_per_bucket, _stream(stream)))
    return out_keys, out_tags


def hs_merge_pairs(keys, tags, bucket_offsets, chunks_per_bucket: int = 8, out_keys=None, out_tags=None,
                   stream=None):
    """f3, a6 on items: the tree merge of each bucket's chunk-sorted runs of (key, tag) items with a
    key-only comparator, ties taking the left run.  Returns (out_keys, out_tags)."""
    torch = _torch()
    out_keys, out_tags = _pairs_outputs(keys, tags, bucket_offsets, out_keys, out_tags)
    with torch.cuda.device(keys.device):
        _check(load().hs_merge_pairs(keys.data_ptr(), tags.data_ptr(), out_keys.data_ptr(), out_tags.data_ptr(),
                                     keys.numel(), _dtype_code(keys), bucket_offsets.data_ptr(), chunks_per_bucket,
                                     _stream(stream)))
    return out_keys, out_tags


class SortGraph:
    """hs_sort of one fixed device buffer captured once in a CUDA graph and
    replayed: for launch-bound sizes (the ~30 kernel launches and the
    stream-ordered scratch allocation of one call become one graph launch).
    The library never synchronises the host inside a call, so the whole call
    is capturable; scratch comes from graph memory nodes.

        g = SortGraph(buf, num_digits=6)   # buf: CUDA tensor, sorted in place on every replay()
        buf.copy_(new_keys); g.replay()
    """

    def __init__(self, keys, num_digits: int, chunks_per_bucket: int = 8):
        torch = _torch()
        _check_tensor(keys, "keys")
        self.keys = keys
        self.stream = torch.cuda.Stream(keys.device)
        self.graph = torch.cuda.CUDAGraph()
        self.stream.wait_stream(torch.cuda.current_stream(keys.device))
        # one uncaptured call on a scratch copy first: the library's one-time
        # per-device setup (kernel attributes, occupancy queries, memory pool
        # threshold) must not run inside a capture
        warm = keys.clone()
        with torch.cuda.stream(self.stream):
            hs_sort(warm, num_digits, chunks_per_bucket, stream=self.stream)
        self.stream.synchronize()
        del warm
        with torch.cuda.graph(self.graph, stream=self.stream):
            hs_sort(keys, num_digits, chunks_per_bucket, stream=self.stream)

    def replay(self) -> None:
        self.graph.replay()


class PartitionPlan:
    """a1-a2 now, a3 later into caller-chosen (possibly peer-GPU) destinations:
    hs_partition_plan_create / hs_partition_scatter / hs_partition_plan_destroy
    (the bucket exchange fused into the scatter)."""

    def __init__(self, keys, num_digits: int, stream=None):
        torch = _torch()
        _check_tensor(keys, "keys")
        self.keys = keys  # must stay alive and unchanged until scatter()
        self.dt = _dtype_code(keys)
        self.stream = stream
        self.offsets = torch.empty(11, dtype=torch.int64, device=keys.device)
        self.handle = ctypes.c_void_p()
        with torch.cuda.device(keys.device):
            _check(load().hs_partition_plan_create(keys.data_ptr(), keys.numel(), self.dt, num_digits,
                                                   self.offsets.data_ptr(), ctypes.byref(self.handle),
                                                   _stream(stream)))

    def scatter(self, dst_ptrs) -> None:
        """dst_ptrs: 10 device addresses (ints; 0 for empty buckets)."""
        torch = _torch()
        arr = (ctypes.c_void_p * 10)(*[int(p) if p else None for p in dst_ptrs])
        with torch.cuda.device(self.keys.device):
            _check(load().hs_partition_scatter(self.handle, arr, _stream(self.stream)))

    def close(self) -> None:
        if self.handle:
            load().hs_partition_plan_destroy(self.handle, _stream(self.stream))
            self.handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def hs_sort_host(host_keys, num_digits: int, chunks_per_bucket: int = 8, device=None, out=None):
    """End-to-end convenience: pinned host keys -> H2D -> hs_sort -> D2H.

    host_keys is a (preferably pinned) CPU torch tensor; the sorted keys are
    copied into ``out`` (a CPU tensor, default: a new pinned one)."""
    torch = _torch()
    dev = torch.device(device or "cuda")
    d = host_keys.to(dev, non_blocking=True)
    hs_sort(d, num_digits, chunks_per_bucket)
    if out is None:
        out = torch.empty_like(host_keys, pin_memory=True)
    out.copy_(d, non_blocking=True)
    torch.cuda.current_stream(dev).synchronize()
    return out


class HostSortPipeline:
    """End-to-end sorting of a stream of host batches through hs_sort.

    Each batch goes pinned host -> H2D -> hs_sort -> D2H.  ``slots`` device
    buffers (default 3) and three CUDA streams (H2D copy, compute, D2H copy) let
    the H2D of batch i+1 and the D2H of batch i-1 run on the two copy engines
    (opposite PCIe directions, concurrently) while batch i is sorted, so a long
    stream of batches is bounded by the slowest of the three stages instead of
    their sum.  With 2 slots the H2D of batch i+1 would wait for the D2H of
    batch i-1 and the copies would serialise; 3 keep both directions busy.
    Ordering is kept with CUDA events only (no host synchronisation except in
    ``finish``).

        pipe = HostSortPipeline(n, torch.int32, num_digits=9, chunks=8)
        for h_in, h_out in batches:      # pinned CPU tensors of n keys
            pipe.submit(h_in, h_out)     # h_out holds the sorted keys once finish() returns
        pipe.finish()
    """

    def __init__(self, n: int, dtype, num_digits: int, chunks: int = 8, device=None, slots: int = 3):
        torch = _torch()
        if slots < 1:
            raise ValueError("slots must be >= 1")
        self.dev = torch.device(device or "cuda")
        self.n, self.num_digits, self.chunks = n, num_digits, chunks
        self.bufs = [torch.empty(n, dtype=dtype, device=self.dev) for _ in range(slots)]
        self.s_in = torch.cuda.Stream(self.dev)
        self.s_cmp = torch.cuda.Stream(self.dev)
        self.s_out = torch.cuda.Stream(self.dev)
        self.out_done = [None] * slots  # event: slot's D2H finished (slot free again)
        self.i = 0

    def submit(self, h_in, h_out) -> None:
        torch = _torch()
        slot = self.i % len(self.bufs)
        buf = self.bufs[slot]
        ev_free = self.out_done[slot]
        with torch.cuda.stream(self.s_in):
            if ev_free is not None:
                self.s_in.wait_event(ev_free)
            buf.copy_(h_in, non_blocking=True)
            ev_in = torch.cuda.Event()
            ev_in.record(self.s_in)
        with torch.cuda.stream(self.s_cmp):
            self.s_cmp.wait_event(ev_in)
            hs_sort(buf, self.num_digits, self.chunks, stream=self.s_cmp)
            ev_cmp = torch.cuda.Event()
            ev_cmp.record(self.s_cmp)
        with torch.cuda.stream(self.s_out):
            self.s_out.wait_event(ev_cmp)
            h_out.copy_(buf, non_blocking=True)
            ev_out = torch.cuda.Event()
            ev_out.record(self.s_out)
        for t in (buf,):  # keep the caching allocator from recycling across streams
            t.record_stream(self.s_in)
            t.record_stream(self.s_cmp)
            t.record_stream(self.s_out)
        self.out_done[slot] = ev_out
        self.i += 1

    def finish(self) -> None:
        for ev in self.out_done:
            if ev is not None:
                ev.synchronize()


msd_partition = hs_msd_partition
sort_chunks = hs_sort_chunks
merge = hs_merge
sort = hs_sort
sort_shared = hs_sort_shared
sort_pairs = hs_sort_pairs
msd_partition_pairs = hs_msd_partition_pairs
sort_chunks_pairs = hs_sort_chunks_pairs
merge_pairs = hs_merge_pairs
sort_host = hs_sort_host
