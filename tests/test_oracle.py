"""Pins for the CPU oracle (oracle/oracle.c) against things other than itself.

Each pin is chosen so a plausible slip in the oracle (a dropped term, a wrong
sign or index, a non-stable scatter, a wrong chunk rule, a transposed merge
operand) fails at least one test:

* worked examples -- SPEC.md's stated examples and SURVEY §8(c) W2, held in
  tests/golden/worked_examples.json with their citations;
* closed forms -- numpy floor division, np.bincount, stable argsort;
* brute force on tiny inputs -- pure-Python insertion sort and an O(n^2)
  rank-count permutation;
* library special cases -- np.sort (keys-only ascending sort is unique);
* invariants -- range disjointness, conservation, multiset
  fingerprints of SURVEY Appendix A.
"""
import numpy as np
import pytest

import oracle as O
import workload as W

rng_master = np.random.default_rng(20030121)


# ----------------------------------------------------------------- helpers
def insertion_sort(xs):
    a = list(xs)
    for i in range(1, len(a)):
        v, j = a[i], i - 1
        while j >= 0 and a[j] > v:
            a[j + 1] = a[j]
            j -= 1
        a[j + 1] = v
    return a


def rank_sort(a):
    """Brute-force O(n^2) stable sort: position_i = #{j: a_j < a_i} + #{j < i: a_j == a_i}."""
    a = np.asarray(a, dtype=np.int64)
    n = a.size
    if n == 0:
        return a
    lt = (a[None, :] < a[:, None]).sum(axis=1)
    eq_before = np.tril(a[None, :] == a[:, None], k=-1).sum(axis=1)
    out = np.empty_like(a)
    out[lt + eq_before] = a
    return out


def np_digit(keys, D):
    k = np.asarray(keys, dtype=np.int64)
    return np.clip(np.where(k < 0, 0, k // 10 ** (D - 1)), 0, 9)


def chunk_bounds(offsets, c):
    """partition_even bounds per S:138, written out independently of the oracle."""
    bounds = []
    for b in range(10):
        lo, m = int(offsets[b]), int(offsets[b + 1] - offsets[b])
        q, r = divmod(m, c)
        s = lo
        for i in range(c):
            ln = q + (1 if i < r else 0)
            bounds.append((s, s + ln))
            s += ln
    return bounds


# ------------------------------------------------------------------ digit
def test_digit_golden(golden):
    for k, D, d in golden["digit"]["cases"]:
        assert O.digit(k, D) == d, (k, D)


def test_digit_vs_floor_division():
    rng = np.random.default_rng(1)
    for D in range(1, 19):
        hi = 10**D
        keys = rng.integers(0, hi, size=2000, dtype=np.int64)
        # boundary keys d*10^(D-1) and d*10^(D-1)-1
        b = np.array([d * 10 ** (D - 1) + e for d in range(1, 10) for e in (-1, 0)], dtype=np.int64)
        keys = np.concatenate([keys, b, [0, hi - 1]])
        got = [O.digit(int(k), D) for k in keys]
        assert got == np_digit(keys, D).tolist(), D


def test_digit_clamp_and_strict():
    assert O.digit(-5, 3) == 0 and O.digit(1000, 3) == 9 and O.digit(2**62, 3) == 9
    assert O.digit(-(2**63), 18) == 0
    with pytest.raises(O.KeyOutOfRange):
        O.digit(1000, 3, strict=True)
    with pytest.raises(O.KeyOutOfRange):
        O.digit(-1, 3, strict=True)
    with pytest.raises(ValueError):
        O.digit(5, 0)
    with pytest.raises(ValueError):
        O.digit(5, 20)


# ---------------------------------------------------------- msd_partition
def test_msd_partition_golden(golden):
    for ex in golden["msd_partition"]:
        out, off = O.msd_partition(np.array(ex["keys"], dtype=np.int64), ex["D"])
        assert off.tolist() == ex["offsets"]
        assert np.diff(off).tolist() == ex["hist"]
        assert out.tolist() == ex["partitioned"]


@pytest.mark.parametrize("D,hi,n", [(1, 10, 5000), (3, 1000, 777), (6, 10**6, 40000), (9, 10**9, 30001), (18, 10**18, 5000)])
def test_msd_partition_vs_stable_argsort(D, hi, n):
    rng = np.random.default_rng(D)
    dt = np.int64 if hi > 2**31 else np.int32
    keys = rng.integers(0, hi, size=n).astype(dt)
    out, off = O.msd_partition(keys, D)
    d = np_digit(keys, D)
    np.testing.assert_array_equal(off, np.concatenate([[0], np.cumsum(np.bincount(d, minlength=10))]))
    np.testing.assert_array_equal(out, keys[np.argsort(d, kind="stable")])
    assert out.dtype == keys.dtype


def test_msd_partition_list_filter_and_disjoint():
    rng = np.random.default_rng(7)
    keys = rng.integers(0, 1000, size=3000)
    out, off = O.msd_partition(keys, 3)
    for b in range(10):
        expect = [int(x) for x in keys if int(x) // 100 == b]  # S:305 bucket semantics
        assert out[off[b]:off[b + 1]].tolist() == expect
    # range disjointness: max(bucket b) < min(bucket b+1) when both non-empty
    nonempty = [out[off[b]:off[b + 1]] for b in range(10) if off[b + 1] > off[b]]
    for x, y in zip(nonempty, nonempty[1:]):
        assert x.max() < y.min()
    assert off[10] == keys.size


def test_msd_partition_strict():
    keys = np.array([5, 17, 1000, 3, -1])
    with pytest.raises(O.KeyOutOfRange) as e:
        O.msd_partition(keys, 3, strict=True)
    assert e.value.index == 2
    out, off = O.msd_partition(keys, 3)  # clamp mode (reading #3)
    assert out.tolist() == [5, 17, 3, -1, 1000] and off.tolist() == [0, 4, 4, 4, 4, 4, 4, 4, 4, 4, 5]


def test_msd_partition_appendix_a_c1(golden):
    keys = W.generate("C1")
    _, off = O.msd_partition(keys, 6)
    assert np.diff(off).tolist() == [104610, 104628, 104662, 105231, 104383, 104944, 104446, 105373, 104770, 105529]


# --------------------------------------------------------- partition_even
def test_partition_even_golden(golden):
    for m, p, lens in golden["partition_even"]["cases"]:
        assert O.partition_even(m, p) == lens


def test_partition_even_properties():
    for m in [0, 1, 5, 63, 64, 65, 1000, 123457]:
        for p in [1, 2, 4, 8, 16, 64]:
            lens = O.partition_even(m, p)
            assert sum(lens) == m and len(lens) == p
            assert max(lens) - min(lens) <= 1
            assert lens == sorted(lens, reverse=True)  # the ceil parts come first
    for bad in (0, 3, 6, 12):
        with pytest.raises(ValueError):
            O.partition_even(10, bad)


# --------------------------------------------------------- merge_schedule
def test_merge_schedule_golden(golden):
    for p, triples in golden["merge_schedule"]["cases"]:
        assert [list(t) for t in O.merge_schedule(p)] == triples


def test_merge_schedule_ownership():
    # after round r every active worker i owns exactly [i, i+2^r)
    for p in [1, 2, 4, 8, 16, 32]:
        owns = {i: {i} for i in range(p)}
        sched = O.merge_schedule(p)
        assert len(sched) == p - 1
        for r, i, j in sched:
            assert i % (1 << r) == 0 and j == i + (1 << (r - 1))
            owns[i] |= owns.pop(j)
        assert owns == {0: set(range(p))}
    with pytest.raises(ValueError):
        O.merge_schedule(6)


# -------------------------------------------------------------- quicksort
def test_quicksort_insertion_bruteforce():
    rng = np.random.default_rng(11)
    for _ in range(150):
        n = int(rng.integers(0, 200))
        hi = int(rng.choice([3, 50, 1000, 10**9]))
        a = rng.integers(0, hi, size=n)
        assert O.quicksort(a).tolist() == insertion_sort(a.tolist())


def test_quicksort_rank_bruteforce_1000():
    # 1000 instances, n in [0, 512]
    rng = np.random.default_rng(12)
    for _ in range(1000):
        n = int(rng.integers(0, 513))
        hi = int(rng.choice([2, 10, 1000, 10**6]))
        a = rng.integers(0, hi, size=n)
        np.testing.assert_array_equal(O.quicksort(a), rank_sort(a))


def test_quicksort_adversarial():
    n = 100_000
    asc = np.arange(n)
    np.testing.assert_array_equal(O.quicksort(asc), asc)          # S:80 sorted input, no depth failure
    np.testing.assert_array_equal(O.quicksort(asc[::-1]), asc)
    np.testing.assert_array_equal(O.quicksort(np.full(n, 7)), np.full(n, 7))
    organ = np.concatenate([np.arange(n // 2), np.arange(n // 2)[::-1]])
    np.testing.assert_array_equal(O.quicksort(organ), np.sort(organ))
    big = W.uniform(1_000_000, 99, 10**9)
    np.testing.assert_array_equal(O.quicksort(big), np.sort(big))


# ------------------------------------------------------------- merge_runs
def test_merge_runs_golden(golden):
    for left, right, out in golden["merge_runs"]["cases"]:
        assert O.merge_runs(left, right).tolist() == out


def test_merge_runs_random():
    rng = np.random.default_rng(13)
    for _ in range(300):
        a = np.sort(rng.integers(0, 20, size=int(rng.integers(0, 50))))
        b = np.sort(rng.integers(0, 20, size=int(rng.integers(0, 50))))
        np.testing.assert_array_equal(O.merge_runs(a, b), np.sort(np.concatenate([a, b])))


def test_merge_runs_all_equal():
    # Stable-left is unobservable for keys-only data (reading #10);
    # what is observable is that ties lose no element and add none.
    assert O.merge_runs([5, 5, 5], [5, 5]).tolist() == [5] * 5
    assert O.merge_runs([1, 5, 5], [5, 9]).tolist() == [1, 5, 5, 5, 9]


# ------------------------------------------------------ sort_chunks, merge
def test_sort_chunks_and_merge_golden(golden):
    for ex in golden["sort_chunks"]:
        x = np.array(ex["partitioned"], dtype=np.int64)
        cs = O.sort_chunks(x, ex["offsets"], ex["c"])
        assert cs.tolist() == ex["chunk_sorted"]
        assert O.merge(cs, ex["offsets"], ex["c"]).tolist() == ex["merged"]


@pytest.mark.parametrize("c", [1, 2, 4, 8, 16, 64])
def test_sort_chunks_per_chunk_npsort(c):
    rng = np.random.default_rng(c)
    keys = rng.integers(0, 10**6, size=20011).astype(np.int32)
    part, off = O.msd_partition(keys, 6)
    cs = O.sort_chunks(part, off, c)
    for lo, hi in chunk_bounds(off, c):
        np.testing.assert_array_equal(cs[lo:hi], np.sort(part[lo:hi]))
    m = O.merge(cs, off, c)
    for b in range(10):
        np.testing.assert_array_equal(m[off[b]:off[b + 1]], np.sort(part[off[b]:off[b + 1]]))
    np.testing.assert_array_equal(m, np.sort(keys))


def test_merge_c1_identity_and_small_buckets():
    x = np.array([3, 1, 2, 9, 8], dtype=np.int64)
    off = [0, 3, 3, 3, 3, 3, 3, 3, 3, 3, 5]
    assert O.merge(x, off, 1).tolist() == [3, 1, 2, 9, 8]   # c = 1: zero rounds
    # m_b < c: empty chunks are legal
    assert O.sort_chunks(x, off, 8).tolist() == [3, 1, 2, 9, 8]
    assert O.merge(x, off, 8).tolist() == [1, 2, 3, 8, 9]


# ------------------------------------------------------------------- sort
def test_sort_bruteforce_small():
    rng = np.random.default_rng(14)
    for _ in range(300):
        n = int(rng.integers(0, 300))
        D = int(rng.integers(1, 7))
        a = rng.integers(0, 10**D, size=n)
        c = int(rng.choice([1, 2, 4, 8]))
        np.testing.assert_array_equal(O.sort(a, D, c), rank_sort(a))


def test_sort_special_cases():
    for n in (0, 1, 2, 3):
        a = np.arange(n)[::-1].copy()
        assert O.sort(a, 1, 8).tolist() == sorted(a.tolist())
    # D = 1 with keys < 10 is a counting sort
    a = np.random.default_rng(3).integers(0, 10, size=5000)
    np.testing.assert_array_equal(O.sort(a, 1, 4), np.repeat(np.arange(10), np.bincount(a, minlength=10)))
    # all-equal, negatives and >= 10^D keys (clamp is order-preserving, reading #3)
    b = np.array([-7, 10**4, 3, -1, 999, 10**9, 0])
    assert O.sort(b, 3, 2).tolist() == sorted(b.tolist())
    with pytest.raises(O.KeyOutOfRange):
        O.sort(b, 3, 2, strict=True)
    with pytest.raises(ValueError):
        O.sort(b, 3, 3)


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_sort_configs_npsort_and_appendix(name):
    cfg = W.CONFIGS[name]
    keys = W.generate(name)
    out = O.sort(keys, cfg.num_digits, cfg.chunks)
    np.testing.assert_array_equal(out, np.sort(keys))
    fp_in, fp_out = W.fingerprint(keys), W.fingerprint(out)
    assert fp_in == fp_out
    assert np.all(out[1:] >= out[:-1])
    app = {"C1": (0, 500766, 999997), "C2": (64, 499982710, 999999883)}[name]
    assert (out[0], out[cfg.n // 2], out[-1]) == app


def test_openmp_build_identical():
    keys = W.generate("C1")
    a = O.sort(keys, 6, 8)
    b = O.sort(keys, 6, 8, openmp=True)
    np.testing.assert_array_equal(a, b)
