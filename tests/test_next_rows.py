"""SURVEY §8(f) rows built this round.

f1  No-MSD ablation: ``hs_sort_shared`` = the paper's
    Shared-Parallel Hybrid Quicksort + Merge Sort on the whole array.
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
