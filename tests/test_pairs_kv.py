"""SURVEY §8(f) f3 on the stable item path (k_kv.cu): SPEC's SortItem
-- a key plus a 64-bit tag that never influences order -- sorted STABLY (P:29:
"Merge sort is a stable sort"), with the tag carried through every pass.

CPU (-m "not gpu"): the oracle's item phases (``sort_chunks_pairs``,
``merge_pairs``, and ``sort_pairs`` on int64 keys) pinned to Python's stable
``sorted`` -- the unique stable order -- with chunk bounds from an
independently written partition_even.

GPU: ``hs_sort_pairs`` on int64 keys, ``hs_msd_partition_pairs`` on int64
keys, ``hs_sort_chunks_pairs`` and ``hs_merge_pairs`` (int32 and int64 keys)
element by element against the oracle, keys AND tags -- the order of equal
keys is observable through the tags, so only a stable path matches.  The
merge tests put equal keys into every chunk of a bucket: K6's stable-left tie
rule ("on equal keys, left first") is exercised on real ties.
"""
import numpy as np
import pytest

import oracle as O
import workload as W

rng = np.random.default_rng(3137)


def chunk_bounds(m, c):
    """partition_even, written out here: the first m % c chunks get one more key."""
    q, r = divmod(m, c)
    b = [0]
    for i in range(c):
        b.append(b[-1] + q + (1 if i < r else 0))
    return b


def stable_sorted(keys, tags):
    items = sorted(zip(np.asarray(keys).tolist(), np.asarray(tags).tolist()), key=lambda kv: kv[0])
    return [k for k, _ in items], [t for _, t in items]


def bucketed(n, D, distinct, seed, dtype):
    """n keys already partitioned by leading digit (bucket order), heavy ties, and offsets[11]."""
    g = np.random.default_rng(seed)
    div = 10 ** (D - 1)
    sizes = g.multinomial(n, [0.1] * 10)
    parts = []
    for b, m in enumerate(sizes):
        vals = g.integers(b * div, (b + 1) * div, size=distinct)
        parts.append(vals[g.integers(0, distinct, size=m)])
    keys = np.concatenate(parts).astype(dtype)
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    return keys, off


# ---------------------------------------------------------------- oracle pins (CPU)
@pytest.mark.parametrize("dtype,D", [(np.int32, 4), (np.int64, 18)])
def test_oracle_sort_chunks_pairs_is_stable_per_chunk(dtype, D):
    for trial in range(40):
        n = int(rng.integers(0, 400))
        c = int(2 ** rng.integers(0, 4))
        keys, off = bucketed(n, D, 7, 100 + trial, dtype)
        tags = rng.permutation(n).astype(np.uint64)
        k, t = O.sort_chunks_pairs(keys, tags, off, c)
        ek, et = keys.copy(), tags.copy()
        for b in range(10):
            lo = int(off[b])
            cb = chunk_bounds(int(off[b + 1] - off[b]), c)
            for i in range(c):
                s, e = lo + cb[i], lo + cb[i + 1]
                sk, st = stable_sorted(keys[s:e], tags[s:e])
                ek[s:e], et[s:e] = sk, st
        assert np.array_equal(k, ek) and np.array_equal(t, et)


@pytest.mark.parametrize("dtype,D", [(np.int32, 4), (np.int64, 18)])
def test_oracle_merge_pairs_equals_stable_sort_of_chunk_runs(dtype, D):
    """The stable-left tree merge of a bucket's chunk-sorted runs, laid out chunk by chunk, is the
    stable sort of that sequence (ties: lower chunk first, then position)."""
    for trial in range(40):
        n = int(rng.integers(0, 400))
        c = int(2 ** rng.integers(0, 4))
        keys, off = bucketed(n, D, 5, 200 + trial, dtype)
        tags = rng.permutation(n).astype(np.uint64)
        ck, ct = keys.copy(), tags.copy()
        for b in range(10):   # make every chunk sorted (stably), independently of the oracle
            lo = int(off[b])
            cb = chunk_bounds(int(off[b + 1] - off[b]), c)
            for i in range(c):
                s, e = lo + cb[i], lo + cb[i + 1]
                ck[s:e], ct[s:e] = stable_sorted(ck[s:e], ct[s:e])
        k, t = O.merge_pairs(ck, ct, off, c)
        ek, et = ck.copy(), ct.copy()
        for b in range(10):
            s, e = int(off[b]), int(off[b + 1])
            ek[s:e], et[s:e] = stable_sorted(ck[s:e], ct[s:e])
        assert np.array_equal(k, ek) and np.array_equal(t, et)


def test_oracle_sort_pairs_int64_bruteforce():
    for trial in range(100):
        n = int(rng.integers(0, 300))
        c = int(2 ** rng.integers(0, 4))
        keys = rng.integers(0, 30, size=n).astype(np.int64) * (10**16 + 12345)   # ties, all 18-digit buckets
        tags = rng.permutation(n).astype(np.uint64)
        k, t = O.sort_pairs(keys, tags, 18, c)
        rk, rt = stable_sorted(keys, tags)
        assert k.tolist() == rk and t.tolist() == rt


# ---------------------------------------------------------------- GPU parity
def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2003_01216_b200 as hs
    hs.load()
    return torch, hs


def _dev(torch, a):
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint64:
        a = a.view(np.int64)
    return torch.from_numpy(a).to("cuda:0")


def _tags(t):
    return t.cpu().numpy().view(np.uint64)


def assert_same(got, ref, what):
    if not np.array_equal(got, ref):
        bad = np.nonzero(got != ref)[0]
        raise AssertionError(f"{what}: {bad.size} mismatches, first at {bad[0]}: got {got[bad[0]]} want {ref[bad[0]]}")


@pytest.mark.gpu
@pytest.mark.parametrize("n,distinct,c", [(0, 1, 8), (1, 1, 8), (5, 2, 2), ("T-1", 40, 1), ("T+1", 40, 1),
                                          ("8T+3", 40, 8), (100_003, 1000, 8), (400_001, 50, 16),
                                          (1_000_003, 10**9, 8), (300_007, 3, 1)])
def test_sort_pairs64_parity(n, distinct, c):
    torch, hs = _gpu()
    if isinstance(n, str):  # around the item tile size (K5kv leaves)
        t = hs.tile_keys(1, 3)
        n = {"T-1": t - 1, "T+1": t + 1, "8T+3": 8 * t + 3}[n]
    g = np.random.default_rng(n + distinct)
    vals = g.integers(0, 10**18, size=min(distinct, 10**6), dtype=np.int64)
    keys = vals[g.integers(0, vals.size, size=n)] if distinct < 10**9 else g.integers(0, 10**18, size=n)
    keys = keys.astype(np.int64)
    tags = g.integers(0, 2**63, size=n, dtype=np.int64).astype(np.uint64)
    dk, dt = _dev(torch, keys), _dev(torch, tags)
    hs.hs_sort_pairs(dk, dt, 18, c)
    rk, rt = O.sort_pairs(keys, tags, 18, c)
    assert_same(dk.cpu().numpy(), rk, "keys")
    assert_same(_tags(dt), rt, "tags")


@pytest.mark.gpu
def test_sort_pairs64_clamped_and_extreme_keys():
    """Negative keys and keys >= 10^D clamp into buckets 0 / 9 (reading #3); INT64_MIN / INT64_MAX
    included (INT64_MAX equals the item path's pad key: pads must stay behind real keys)."""
    torch, hs = _gpu()
    g = np.random.default_rng(9)
    n = 200_003
    keys = g.integers(-2**62, 2**62, size=n, dtype=np.int64)
    keys[::5] = np.iinfo(np.int64).max
    keys[1::11] = np.iinfo(np.int64).min
    tags = np.arange(n, dtype=np.uint64)
    dk, dt = _dev(torch, keys), _dev(torch, tags)
    hs.hs_sort_pairs(dk, dt, 12, 8)
    rk, rt = O.sort_pairs(keys, tags, 12, 8)
    assert_same(dk.cpu().numpy(), rk, "keys")
    assert_same(_tags(dt), rt, "tags")


@pytest.mark.gpu
def test_sort_pairs64_c5_sample():
    torch, hs = _gpu()
    cfg = W.CONFIGS["C5"]
    keys = W.generate("C5", 0, 2_000_000)
    tags = W.uniform(keys.size, 55, 2**62, dtype=np.int64).astype(np.uint64)
    dk, dt = _dev(torch, keys), _dev(torch, tags)
    hs.hs_sort_pairs(dk, dt, cfg.num_digits, cfg.chunks)
    rk, rt = O.sort_pairs(keys, tags, cfg.num_digits, cfg.chunks)
    assert_same(dk.cpu().numpy(), rk, "keys")
    assert_same(_tags(dt), rt, "tags")


@pytest.mark.gpu
def test_msd_partition_pairs64_parity():
    torch, hs = _gpu()
    g = np.random.default_rng(17)
    n = 500_009
    keys = g.integers(0, 10**18, size=n, dtype=np.int64)
    keys[::3] = keys[0]
    tags = np.arange(n, dtype=np.uint64)[::-1].copy()
    ok, ot, off = hs.hs_msd_partition_pairs(_dev(torch, keys), _dev(torch, tags), 18)
    rk, rt, roff = O.msd_partition_pairs(keys, tags, 18)
    assert_same(off.cpu().numpy(), roff, "offsets")
    assert_same(ok.cpu().numpy(), rk, "keys")
    assert_same(_tags(ot), rt, "tags")


@pytest.mark.gpu
@pytest.mark.parametrize("dtype,D", [(np.int32, 9), (np.int64, 18)])
@pytest.mark.parametrize("c", [2, 8])
def test_merge_pairs_stable_left_on_real_ties(dtype, D, c):
    """K6 on items with a key-only comparator: every chunk of every bucket holds copies of the same
    few keys, each chunk's tags record (chunk index, position).  The merged bucket must list equal
    keys left run first -- here: by chunk index, then by position -- exactly as the oracle's
    stable-left tree merge does."""
    torch, hs = _gpu()
    keys, off = bucketed(300_000, D, 6, 31 + c, dtype)
    ck = keys.copy()
    tags = np.zeros(keys.size, dtype=np.uint64)
    for b in range(10):   # sort each chunk (np.sort: keys only), tag = chunk << 32 | position
        lo = int(off[b])
        cb = chunk_bounds(int(off[b + 1] - off[b]), c)
        for i in range(c):
            s, e = lo + cb[i], lo + cb[i + 1]
            ck[s:e] = np.sort(ck[s:e])
            tags[s:e] = (np.uint64(i) << np.uint64(32)) | np.arange(e - s, dtype=np.uint64)
    mk, mt = hs.hs_merge_pairs(_dev(torch, ck), _dev(torch, tags), _dev(torch, off), c)
    rk, rt = O.merge_pairs(ck, tags, off, c)
    assert_same(mk.cpu().numpy(), rk, "keys")
    got_t = _tags(mt)
    assert_same(got_t, rt, "tags")
    # the tie rule itself: within a run of equal keys, (chunk, position) tags ascend
    gk = mk.cpu().numpy()
    same = gk[1:] == gk[:-1]
    assert same.sum() > keys.size // 2
    assert np.all(got_t[1:][same] > got_t[:-1][same])


@pytest.mark.gpu
@pytest.mark.parametrize("dtype,D", [(np.int32, 9), (np.int64, 18)])
def test_sort_chunks_pairs_then_merge_pairs(dtype, D):
    """a5 then a6 on items (in place) equals the whole stable path, and each equals the oracle."""
    torch, hs = _gpu()
    g = np.random.default_rng(77)
    n = 700_001
    vals = g.integers(0, 10 ** D, size=5000).astype(dtype)
    keys = vals[g.integers(0, vals.size, size=n)]
    tags = g.integers(0, 2**63, size=n, dtype=np.int64).astype(np.uint64)
    pk, pt, off = O.msd_partition_pairs(keys, tags, D)
    pk = pk.astype(dtype)
    dk, dt, doff = _dev(torch, pk), _dev(torch, pt), _dev(torch, off)
    hs.hs_sort_chunks_pairs(dk, dt, doff, 8, out_keys=dk, out_tags=dt)
    ck, ct = O.sort_chunks_pairs(pk, pt, off, 8)
    assert_same(dk.cpu().numpy(), ck, "chunks keys")
    assert_same(_tags(dt), ct, "chunks tags")
    hs.hs_merge_pairs(dk, dt, doff, 8, out_keys=dk, out_tags=dt)
    mk, mt = O.merge_pairs(ck, ct, off, 8)
    assert_same(dk.cpu().numpy(), mk, "merged keys")
    assert_same(_tags(dt), mt, "merged tags")
    sk, st = O.sort_pairs(keys, tags, D, 8)
    assert_same(mk, sk, "composition keys")
    assert_same(mt, st, "composition tags")
