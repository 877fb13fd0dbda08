"""SURVEY §8(f) rows built this round.

f1  No-MSD ablation: ``hs_sort_shared`` = the paper's
    Shared-Parallel Hybrid Quicksort + Merge Sort on the whole array.
f3  Key + tag items, sorted stably (SPEC SortItem S:31-37; "merge sort
    is a stable sort"): ``hs_sort_pairs`` / ``hs_msd_partition_pairs`` against
    the oracle's stable path (Fig 1b merge sort per chunk) -- the tie order is
    observable through the tags.
f4  The paper's own workload: config P3, 10^7 three-digit keys
    in [100, 999] -- 900 distinct values, bucket 0 empty.

CPU tests pin the oracle's ``sort_shared`` and the P3 generator against
things other than themselves (brute force, np.sort, the numpy twin); the
``gpu`` tests compare the CUDA path with the oracle element by element.
"""
import numpy as np
import pytest

import oracle as O
import workload as W

rng = np.random.default_rng(62)


def insertion_sort(xs):
    a = list(xs)
    for i in range(1, len(a)):
        v, j = a[i], i - 1
        while j >= 0 and a[j] > v:
            a[j + 1] = a[j]
            j -= 1
        a[j + 1] = v
    return a


# ------------------------------------------------------ oracle pins (CPU)
def test_sort_shared_bruteforce():
    for _ in range(300):
        n = int(rng.integers(0, 200))
        c = int(2 ** rng.integers(0, 6))
        keys = rng.integers(-50, 50, size=n).astype(np.int64)
        assert O.sort_shared(keys, c).tolist() == insertion_sort(keys.tolist())


def test_sort_shared_npsort_and_special_cases():
    k = W.uniform(300_007, 9, 10**9, dtype=np.int32)
    for c in (1, 2, 8, 64):
        assert np.array_equal(O.sort_shared(k, c), np.sort(k))
    # c = 1: no merge rounds -- the whole array is one quicksorted part (Fig 1c)
    assert np.array_equal(O.sort_shared(k, 1), O.quicksort(k))
    # equals the MSD path (both are the unique ascending order)
    assert np.array_equal(O.sort_shared(k, 8), O.sort(k, 9, 8))
    with pytest.raises(Exception):
        O.sort_shared(k, 6)  # threads must be a power of two


def test_p3_workload_shape():
    cfg = W.CONFIGS["P3"]
    k = W.generate("P3")
    assert k.size == 10_000_000 and k.dtype == np.int32
    assert k.min() >= 100 and k.max() <= 999          # "three digits"
    assert np.unique(k).size == 900
    assert np.array_equal(k[:4096], W.generate_np("P3", 0, 4096))
    assert np.array_equal(k[-777:], W.generate_np("P3", cfg.n - 777, 777))
    hist = O.histogram(k[:1_000_000], 3)
    assert hist[0] == 0 and hist[1:].min() > 0        # bucket 0 empty


def test_p3_oracle_npsort():
    k = W.generate("P3")[:2_000_000]
    assert np.array_equal(O.sort(k, 3, 8), np.sort(k))
    assert np.array_equal(O.sort_shared(k, 8), np.sort(k))


# ------------------------------------------------------ GPU parity
def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2003_01216_b200 as hs
    hs.load()
    return torch, hs


def _run_shared(keys, c):
    torch, hs = _gpu()
    d = torch.from_numpy(np.ascontiguousarray(keys)).to("cuda:0")
    hs.hs_sort_shared(d, c)
    torch.cuda.synchronize()
    return d.cpu().numpy()


@pytest.mark.gpu
@pytest.mark.parametrize("n", [0, 1, 2, 1000, 13_823, 13_825, 100_003, 1 << 20, 3_000_017])
def test_sort_shared_sizes(n):
    keys = W.uniform(n, 70 + n % 97, 10**9, dtype=np.int32)
    got = _run_shared(keys, 8)
    assert np.array_equal(got, O.sort_shared(keys, 8))


@pytest.mark.gpu
@pytest.mark.parametrize("c", [1, 2, 4, 16, 64])
def test_sort_shared_chunks(c):
    keys = W.uniform(777_777, 80 + c, 10**6, dtype=np.int32)
    assert np.array_equal(_run_shared(keys, c), O.sort_shared(keys, c))


@pytest.mark.gpu
def test_sort_shared_int64_and_degenerate():
    k64 = W.uniform(600_001, 91, 10**18, dtype=np.int64)
    k64[::31] = np.iinfo(np.int64).max
    assert np.array_equal(_run_shared(k64, 8), O.sort_shared(k64, 8))
    eq = np.full(400_000, 123, dtype=np.int32)
    assert np.array_equal(_run_shared(eq, 8), eq)
    rev = np.arange(500_000, dtype=np.int32)[::-1].copy()
    assert np.array_equal(_run_shared(rev, 16), np.arange(500_000, dtype=np.int32))


@pytest.mark.gpu
def test_sort_shared_rejects_bad_chunks():
    torch, hs = _gpu()
    d = torch.zeros(10, dtype=torch.int32, device="cuda:0")
    with pytest.raises(hs.HybridSortError):
        hs.hs_sort_shared(d, 6)


@pytest.mark.gpu
def test_p3_full_bitexact():
    """f4: the paper's 3-digit workload at its largest size, both paths."""
    torch, hs = _gpu()
    keys = W.generate("P3")
    ref = O.sort(keys, 3, 8)
    d = torch.from_numpy(keys).to("cuda:0")
    hs.hs_sort(d, 3, 8)
    torch.cuda.synchronize()
    assert np.array_equal(d.cpu().numpy(), ref)
    out, off = hs.hs_msd_partition(torch.from_numpy(keys).to("cuda:0"), 3)
    ref_out, ref_off = O.msd_partition(keys, 3)
    assert np.array_equal(off.cpu().numpy(), ref_off) and np.array_equal(out.cpu().numpy(), ref_out)
    assert int(ref_off[1]) == 0  # bucket 0 empty
    assert np.array_equal(_run_shared(keys, 8), O.sort_shared(keys, 8))


# ------------------------------------------------------ f3: key + tag items
def stable_ref(keys, tags):
    """Python's sorted() is stable: the unique stable order of (key, tag) items by key."""
    items = sorted(zip(np.asarray(keys).tolist(), np.asarray(tags).tolist()), key=lambda kv: kv[0])
    return (np.array([k for k, _ in items], dtype=np.asarray(keys).dtype),
            np.array([t for _, t in items], dtype=np.uint64))


def test_sort_pairs_oracle_bruteforce():
    for _ in range(300):
        n = int(rng.integers(0, 300))
        c = int(2 ** rng.integers(0, 5))
        keys = rng.integers(0, 40, size=n).astype(np.int32)       # many ties
        tags = rng.permutation(n).astype(np.uint64)
        k, t = O.sort_pairs(keys, tags, 2, c)
        rk, rt = stable_ref(keys, tags)
        assert np.array_equal(k, rk) and np.array_equal(t, rt)


def test_sort_pairs_oracle_npsort_stable_and_partition():
    keys = W.generate("C4")[:400_000]                             # heavy duplicates (1024-value table)
    tags = np.arange(keys.size, dtype=np.uint64)
    k, t = O.sort_pairs(keys, tags, 9, 8)
    order = np.argsort(keys, kind="stable")                        # library stable sort
    assert np.array_equal(k, keys[order]) and np.array_equal(t, tags[order])
    pk, pt, off = O.msd_partition_pairs(keys, tags, 9)
    d = np.clip(keys.astype(np.int64) // 10**8, 0, 9)
    order = np.argsort(d, kind="stable")
    assert np.array_equal(pk, keys[order]) and np.array_equal(pt, tags[order])
    assert np.array_equal(off, np.concatenate([[0], np.cumsum(np.bincount(d, minlength=10))]))


def _run_pairs(keys, tags, D, c):
    torch, hs = _gpu()
    dk = torch.from_numpy(np.ascontiguousarray(keys)).to("cuda:0")
    dt = torch.from_numpy(np.ascontiguousarray(tags).view(np.int64)).to("cuda:0")
    hs.hs_sort_pairs(dk, dt, D, c)
    torch.cuda.synchronize()
    return dk.cpu().numpy(), dt.cpu().numpy().view(np.uint64)


@pytest.mark.gpu
@pytest.mark.parametrize("name,n", [("C1", None), ("C4", 3_000_000), ("P3", 2_000_000)])
def test_sort_pairs_parity(name, n):
    cfg = W.CONFIGS[name]
    keys = W.generate(name, 0, n)
    tags = W.uniform(keys.size, 77, 2**62, dtype=np.int64).astype(np.uint64)
    k, t = _run_pairs(keys, tags, cfg.num_digits, 8)
    rk, rt = O.sort_pairs(keys, tags, cfg.num_digits, 8)
    assert np.array_equal(k, rk)
    assert np.array_equal(t, rt)    # ties in input order: only a stable path matches


@pytest.mark.gpu
@pytest.mark.parametrize("n", [0, 1, 5, 13_825, 100_003])
def test_sort_pairs_edges(n):
    keys = W.uniform(n, 91, 2**31 - 1, dtype=np.int32) - 2**30    # negative and clamped keys
    if n > 3:
        keys[::3] = np.iinfo(np.int32).max
        keys[1::7] = np.iinfo(np.int32).min
    tags = np.arange(n, dtype=np.uint64) * 3 + 1
    k, t = _run_pairs(keys, tags, 6, 4)
    rk, rt = stable_ref(keys, tags)
    assert np.array_equal(k, rk) and np.array_equal(t, rt)


@pytest.mark.gpu
def test_msd_partition_pairs_parity():
    torch, hs = _gpu()
    keys = W.generate("C4", 0, 1_000_003)
    tags = np.arange(keys.size, dtype=np.uint64)[::-1].copy()
    ok, ot, off = hs.hs_msd_partition_pairs(torch.from_numpy(keys).cuda(),
                                            torch.from_numpy(tags.view(np.int64)).cuda(), 9)
    rk, rt, roff = O.msd_partition_pairs(keys, tags, 9)
    assert np.array_equal(off.cpu().numpy(), roff)
    assert np.array_equal(ok.cpu().numpy(), rk)
    assert np.array_equal(ot.cpu().numpy().view(np.uint64), rt)
