"""Runs every C-ABI entry point of libhybridsort_debug.so (-DHS_DEBUG device
invariant checks) on a spread of small inputs and checks each result against
the oracle.  Exit 0 = all bit-exact and no device assert fired.  Used by
tests/test_debug_build.py (in a subprocess: a fired __trap() poisons the CUDA
context of the process)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle as O
import workload as W
from paper_2003_01216_b200 import _build


def main():
    lib = ctypes.CDLL(os.environ.get("HS_DEBUG_LIB", _build.SO_DEBUG))
    vp, i64, ci = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
    lib.hs_sort.argtypes = [vp, i64, ci, ci, ci, vp]
    lib.hs_msd_partition.argtypes = [vp, i64, ci, ci, vp, vp, vp]
    lib.hs_sort_chunks.argtypes = [vp, vp, i64, ci, vp, ci, vp]
    lib.hs_merge.argtypes = [vp, vp, i64, ci, vp, ci, vp]
    lib.hs_sort_shared.argtypes = [vp, i64, ci, ci, vp]
    lib.hs_sort_pairs.argtypes = [vp, vp, i64, ci, ci, vp]
    lib.hs_sort_pairs64.argtypes = [vp, vp, i64, ci, ci, vp]
    lib.hs_merge_pairs.argtypes = [vp, vp, vp, vp, i64, ci, vp, ci, vp]
    st = torch.cuda.current_stream().cuda_stream
    dev = "cuda:0"
    cases = 0

    def ok(rc):
        assert rc == 0, rc

    rng = np.random.default_rng(1234)
    sizes = [1, 2, 31, 2047, 2049, 27_135, 27_137, 100_003, 400_001]
    for n in sizes:
        for dt, D, hi in [(np.int32, 9, 10**9), (np.int32, 3, 1000), (np.int64, 18, 10**18)]:
            keys = W.uniform(n, 7 + n % 13, hi, dtype=dt)
            if n > 10:
                keys[rng.integers(0, n, 5)] = np.iinfo(dt).max
            code = 0 if dt == np.int32 else 1
            for c in (1, 8, 64):
                d = torch.from_numpy(keys).to(dev)
                ok(lib.hs_sort(d.data_ptr(), n, code, D, c, st))
                torch.cuda.synchronize()
                assert np.array_equal(d.cpu().numpy(), O.sort(keys, D, c)), ("sort", n, dt, c)
                cases += 1
            src = torch.from_numpy(keys).to(dev)
            out = torch.empty_like(src)
            off = torch.empty(11, dtype=torch.int64, device=dev)
            ok(lib.hs_msd_partition(src.data_ptr(), n, code, D, off.data_ptr(), out.data_ptr(), st))
            ro, roff = O.msd_partition(keys, D)
            torch.cuda.synchronize()
            assert np.array_equal(out.cpu().numpy(), ro) and np.array_equal(off.cpu().numpy(), roff)
            sc = torch.empty_like(src)
            ok(lib.hs_sort_chunks(out.data_ptr(), sc.data_ptr(), n, code, off.data_ptr(), 4, st))
            mg = torch.empty_like(src)
            ok(lib.hs_merge(sc.data_ptr(), mg.data_ptr(), n, code, off.data_ptr(), 4, st))
            torch.cuda.synchronize()
            assert np.array_equal(mg.cpu().numpy(), O.sort(keys, D, 4)), ("chunks+merge", n, dt)
            sh = torch.from_numpy(keys).to(dev)
            ok(lib.hs_sort_shared(sh.data_ptr(), n, code, 8, st))
            torch.cuda.synchronize()
            assert np.array_equal(sh.cpu().numpy(), np.sort(keys)), ("shared", n, dt)
            cases += 3
        keys = W.uniform(n, 99, 1000, dtype=np.int32)
        tags = np.arange(n, dtype=np.int64)
        dk, dtg = torch.from_numpy(keys).to(dev), torch.from_numpy(tags).to(dev)
        ok(lib.hs_sort_pairs(dk.data_ptr(), dtg.data_ptr(), n, 3, 8, st))
        torch.cuda.synchronize()
        rk, rt = O.sort_pairs(keys, tags.astype(np.uint64), 3, 8)
        assert np.array_equal(dk.cpu().numpy(), rk) and np.array_equal(dtg.cpu().numpy().view(np.uint64), rt)
        cases += 1
        # f3 stable item path (k_kv.cu): int64 keys with ties, then a merge of chunk-sorted item runs
        k64 = W.uniform(n, 5, 1000, dtype=np.int64) * 10**15
        dk, dtg = torch.from_numpy(k64).to(dev), torch.from_numpy(tags).to(dev)
        ok(lib.hs_sort_pairs64(dk.data_ptr(), dtg.data_ptr(), n, 18, 8, st))
        torch.cuda.synchronize()
        rk, rt = O.sort_pairs(k64, tags.astype(np.uint64), 18, 8)
        assert np.array_equal(dk.cpu().numpy(), rk) and np.array_equal(dtg.cpu().numpy().view(np.uint64), rt)
        pk, pt, poff = O.msd_partition_pairs(k64, tags.astype(np.uint64), 18)
        ck, ct = O.sort_chunks_pairs(pk, pt, poff, 4)
        dk, dtg, doff = (torch.from_numpy(ck).to(dev), torch.from_numpy(ct.view(np.int64)).to(dev),
                         torch.from_numpy(poff).to(dev))
        ok(lib.hs_merge_pairs(dk.data_ptr(), dtg.data_ptr(), dk.data_ptr(), dtg.data_ptr(), n, 1, doff.data_ptr(), 4,
                              st))
        torch.cuda.synchronize()
        mk, mt = O.merge_pairs(ck, ct, poff, 4)
        assert np.array_equal(dk.cpu().numpy(), mk) and np.array_equal(dtg.cpu().numpy().view(np.uint64), mt)
        cases += 2
    # big pieces (1-4 tiles: a dense value range) and constant pieces (one value, ~6 tiles per chunk)
    t = 27_136
    for c in (2, 8):
        keys = W.uniform(c * 12 * t, 5 + c, 10**9, dtype=np.int32)
        keys[: int(2.5 * t) * c] = 500_000_000 + rng.integers(0, 3 * t, size=int(2.5 * t) * c)
        keys[int(2.5 * t) * c: int(8.5 * t) * c] = 300_000_777
        rng.shuffle(keys)
        d = torch.from_numpy(keys).to(dev)
        ok(lib.hs_sort(d.data_ptr(), keys.size, 0, 9, c, st))
        torch.cuda.synchronize()
        assert np.array_equal(d.cpu().numpy(), np.sort(keys)), ("big/constant pieces", c)
        cases += 1
    # one full-size config through the debug checks
    keys = W.generate("C2")
    d = torch.from_numpy(keys).to(dev)
    ok(lib.hs_sort(d.data_ptr(), keys.size, 0, 9, 8, st))
    torch.cuda.synchronize()
    assert np.array_equal(d.cpu().numpy(), np.sort(keys))
    print(f"debug build: {cases + 1} calls bit-exact, no device assert fired")


if __name__ == "__main__":
    main()
