"""K5a value split of the chunks (hs_sort): parity on inputs built to take
the split, to fall back from it, and to mix both within one call.

A bucket is split when its chunks exceed one tile (T keys); a split bucket
whose equal-width value sub-ranges overflow a tile (skew, heavy duplicates,
clamped keys piling into the first / last sub-range) falls back to tile sort
+ in-chunk merge levels.  Either way hs_sort must return the unique
ascending array, so every case compares with the oracle element by element;
``hs_sort_plan`` shows which path each bucket took, so the cases provably
cover both.
"""
import numpy as np
import pytest

import oracle as O
import workload as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2003_01216_b200 as hs  # noqa: E402

DEV = "cuda:0"


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    hs.load()


def T(code):
    return hs.tile_keys(code, 1)


def run(keys, D, c):
    d = torch.from_numpy(np.ascontiguousarray(keys)).to(DEV)
    plan = hs.hs_sort_plan(d, D, c)
    before = d.clone()
    hs.hs_sort(d, D, c)
    torch.cuda.synchronize()
    return d.cpu().numpy(), plan, before


def check(keys, D, c):
    got, plan, _ = run(keys, D, c)
    ref = O.sort(keys, D, c)
    if not np.array_equal(got, ref):
        bad = np.nonzero(got != ref)[0]
        raise AssertionError(f"{bad.size} mismatches, first at {bad[0]}: got {got[bad[0]]} want {ref[bad[0]]}")
    return plan


def buckets(per_bucket, D, seed, dtype=np.int32, lo_frac=0.0, hi_frac=1.0):
    """per_bucket[b] keys uniform over [lo_frac, hi_frac) of digit b's range, shuffled."""
    div = 10 ** (D - 1)
    rng = np.random.default_rng(seed)
    parts = []
    for b, m in enumerate(per_bucket):
        lo = b * div + int(lo_frac * div)
        hi = b * div + max(int(hi_frac * div), int(lo_frac * div) + 1)
        parts.append(rng.integers(lo, hi, size=m, dtype=np.int64))
    k = np.concatenate(parts).astype(dtype)
    rng.shuffle(k)
    return k


@pytest.mark.parametrize("c", [1, 2, 8, 64])
def test_split_uniform_all_buckets(c):
    t = T(0)
    keys = buckets([c * 3 * t + 17 * b for b in range(10)], 9, 11 + c)
    plan = check(keys, 9, c)
    lg = c.bit_length() - 1
    assert plan["split"] == [1] * 10
    assert plan["padded"] == [1] * 10           # uniform buckets: padded layout, no count pass
    assert plan["levels"] == [lg] * 10          # only the paper's chunk tree remains
    assert all(lv >= 2 for lv in plan["leaves"])


def test_split_just_over_one_tile():
    t = T(0)
    keys = buckets([t + 1 + b for b in range(10)], 6, 5)   # c = 1: every chunk = T + 1 + b keys -> 2 sub-ranges
    plan = check(keys, 6, 1)
    assert plan["split"] == [1] * 10 and plan["leaves"] == [2] * 10


def test_split_mixed_with_fallback_buckets():
    """Buckets 1, 4, 7 split (equal width), 6 splits through the sampled map (a narrow normal peak),
    9 (clamped keys pile into the last sub-range: 2.5 tiles per chunk) splits with a big piece (K5's
    in-CTA tiles + merges), 2 (one value, 4.5 tiles per chunk) splits with a constant piece (filled,
    not sorted); 5 (three values, 4.5 tiles per chunk in one sub-range: over the big-piece limit and
    not constant) falls back; 0, 3 fit a tile."""
    t, D, c = T(0), 7, 2
    div = 10 ** (D - 1)
    rng = np.random.default_rng(3)
    m = 5 * t
    parts = [
        rng.integers(0, div, size=t // 3),                     # bucket 0: small, no split needed
        rng.integers(div, 2 * div, size=m),                    # bucket 1: split
        np.full(9 * t, 2 * div + 12345),                       # bucket 2: constant -> sub-range over 4 tiles
        rng.integers(3 * div, 4 * div, size=t // 2),           # bucket 3: small
        rng.integers(4 * div, 5 * div, size=m + 999),          # bucket 4: split
        5 * div + rng.integers(0, 3, size=9 * t),              # bucket 5: three values, 1.5 T copies each per chunk
        np.clip(rng.normal(6.5 * div, div / 40, size=m), 6 * div, 7 * div - 1).astype(np.int64),  # bucket 6: peak
        rng.integers(7 * div, 8 * div, size=m - 5),            # bucket 7: split
        rng.integers(10 * div, 2**31 - 1, size=m),             # bucket 9: clamped (>= 10^D): last sub-range
    ]
    keys = np.concatenate(parts).astype(np.int32)
    rng.shuffle(keys)
    plan = check(keys, D, c)
    assert [plan["split"][b] for b in (1, 2, 4, 6, 7, 9)] == [1] * 6
    assert [plan["split"][b] for b in (0, 3, 5)] == [0] * 3
    assert plan["levels"][1] == 1 and plan["levels"][5] > 1    # fallback keeps its in-chunk levels


def test_split_clamped_and_negative_inside_split_buckets():
    """A few clamped keys (negative -> bucket 0, >= 10^D -> bucket 9) land in the edge sub-ranges."""
    t, D, c = T(0), 8, 2
    keys = buckets([c * 4 * t] * 10, D, 21)
    rng = np.random.default_rng(22)
    idx = rng.choice(keys.size, 4000, replace=False)
    keys[idx[:2000]] = -rng.integers(1, 2**31 - 1, size=2000)
    keys[idx[2000:]] = rng.integers(10**D, 2**31 - 1, size=2000)
    keys[idx[:5]] = np.iinfo(np.int32).min
    keys[idx[-5:]] = np.iinfo(np.int32).max
    plan = check(keys, D, c)
    assert plan["split"][0] == 1 and plan["split"][9] == 1


def test_split_sorted_and_reversed_input():
    """Sorted input: every chunk covers its own slice of the bucket's value range, so equal-width
    sub-ranges of the bucket overflow; the per-chunk sampled maps split every chunk anyway."""
    t = T(0)
    n = 10 * 2 * 3 * t
    for keys in (np.arange(n, dtype=np.int32) * 13, (np.arange(n, dtype=np.int32) * 13)[::-1].copy()):
        D = len(str(int(keys.max())))
        plan = check(keys, D, 2)
        off = np.concatenate([[0], np.cumsum(np.bincount(np.minimum(keys // 10 ** (D - 1), 9), minlength=10))])
        for b in range(10):
            if off[b + 1] - off[b] > 2 * t:     # chunks larger than a tile
                assert plan["split"][b] == 1, (b, plan)


def test_split_sorted_runs_c8():
    """Nearly sorted data with c = 8 (per-chunk maps for every chunk of a large bucket)."""
    t = T(0)
    rng = np.random.default_rng(91)
    n = 8 * 4 * t * 3
    keys = (np.sort(rng.integers(0, 3 * 10**7, size=n)) + rng.integers(0, 50, size=n)).astype(np.int32)
    plan = check(keys, 8, 8)
    assert plan["split"][0] == 1 and plan["split"][1] == 1 and plan["split"][2] == 1


def test_split_duplicates_half_the_keys():
    t, c = T(0), 4
    keys = buckets([c * 3 * t] * 10, 9, 31)
    keys[::2] = 123_456_789      # half of everything is one value in bucket 1
    plan = check(keys, 9, c)
    assert plan["split"][1] == 0 and plan["split"][5] == 1


def test_split_int64():
    t, D, c = T(1), 18, 2
    keys = buckets([c * 3 * t + b for b in range(10)], D, 41, dtype=np.int64)
    keys[::97] = np.iinfo(np.int64).max    # clamped into bucket 9's last sub-range
    keys[1::89] = np.iinfo(np.int64).min   # clamped into bucket 0's first sub-range
    plan = check(keys, D, c)
    assert sum(plan["split"]) >= 8


def test_split_pairs_stable():
    """hs_sort_pairs items (key << 32 | index) go through the split with shift 32: still stable."""
    t64, c = T(1), 4
    keys = buckets([c * 3 * t64] * 10, 6, 51)
    keys[::3] = 345_678                                   # many ties
    tags = np.random.default_rng(52).integers(0, 2**62, size=keys.size, dtype=np.int64).astype(np.uint64)
    dk = torch.from_numpy(keys).to(DEV)
    dt = torch.from_numpy(tags.view(np.int64)).to(DEV)
    hs.hs_sort_pairs(dk, dt, 6, c)
    torch.cuda.synchronize()
    rk, rt = O.sort_pairs(keys, tags, 6, c)
    assert np.array_equal(dk.cpu().numpy(), rk)
    assert np.array_equal(dt.cpu().numpy().view(np.uint64), rt)


def test_sort_plan_leaves_keys_and_matches_nonsplit_levels():
    t = T(0)
    keys = buckets([2 * 3 * t] * 10, 9, 61)
    d = torch.from_numpy(keys).to(DEV)
    plan = hs.hs_sort_plan(d, 9, 2)
    assert np.array_equal(d.cpu().numpy(), keys)          # inspection does not modify keys
    off = np.concatenate([[0], np.cumsum([2 * 3 * t] * 10)]).astype(np.int64)
    L_host, k_host = hs.plan_levels(off, 0, 2, 0)
    for b in range(10):
        if plan["split"][b]:
            assert plan["levels"][b] == 1
        else:
            assert plan["levels"][b] == L_host[b] and plan["leaves"][b] == 1 << k_host[b]
    empty = hs.hs_sort_plan(torch.empty(0, dtype=torch.int32, device=DEV), 9, 2)
    assert empty["split"] == [0] * 10 and empty["levels"] == [0] * 10


def test_split_skewed_mixture_uses_sampled_map():
    """C4's mixture (70% one normal peak across buckets 2-3, 20% from a 1024-value table, 10% uniform):
    equal-width sub-ranges of the peak buckets would overflow a tile; the sampled map splits them."""
    keys = W.generate("C4", 0, 6_000_000)
    plan = check(keys, 9, 8)
    assert plan["split"][2] == 1 and plan["split"][3] == 1
    assert plan["levels"][2] == 3 and plan["levels"][3] == 3


def test_split_sampled_map_int64_and_pairs():
    """The sampled map on int64 keys (a peak in bucket 4) and on hs_sort_pairs items (shift 32)."""
    rng = np.random.default_rng(71)
    D, n = 18, 10 * 2 * 4 * T(1)
    div = 10 ** (D - 1)
    k64 = rng.integers(0, 10 * div, size=n, dtype=np.int64)
    k64[: n // 2] = np.clip(rng.normal(4.3 * div, div / 100, size=n // 2), 4 * div, 5 * div - 1).astype(np.int64)
    rng.shuffle(k64)
    plan = check(k64, D, 2)
    assert plan["split"][4] == 1
    t64 = T(1)
    keys = buckets([4 * 3 * t64] * 10, 6, 72)
    keys[::2] = np.clip(rng.normal(3.5e5, 2e3, size=keys[::2].size), 3e5, 4e5 - 1).astype(np.int32)
    tags = rng.integers(0, 2**62, size=keys.size, dtype=np.int64).astype(np.uint64)
    dk = torch.from_numpy(keys).to(DEV)
    dt = torch.from_numpy(tags.view(np.int64)).to(DEV)
    hs.hs_sort_pairs(dk, dt, 6, 4)
    torch.cuda.synchronize()
    rk, rt = O.sort_pairs(keys, tags, 6, 4)
    assert np.array_equal(dk.cpu().numpy(), rk)
    assert np.array_equal(dt.cpu().numpy().view(np.uint64), rt)


@pytest.mark.parametrize("name,n,c", [("C1", None, 8), ("C4", 3_000_000, 8), ("C2", 4_000_000, 2), ("C5", 2_000_001, 4)])
def test_sort_buckets_after_partition(name, n, c):
    """hs_sort_buckets (a4-a7 on a digit-partitioned array, the f2 receive side) == oracle sort of
    the keys == hs_merge(hs_sort_chunks(.)) on the same partition."""
    cfg = W.CONFIGS[name]
    keys = W.generate(name, 0, n)
    part, off = hs.hs_msd_partition(torch.from_numpy(keys).to(DEV), cfg.num_digits)
    ref_cm = hs.hs_merge(hs.hs_sort_chunks(part.clone(), off, c), off, c)
    hs.hs_sort_buckets(part, off, cfg.num_digits, c)
    torch.cuda.synchronize()
    got = part.cpu().numpy()
    assert np.array_equal(got, O.sort(keys, cfg.num_digits, c))
    assert np.array_equal(got, ref_cm.cpu().numpy())


def test_sort_buckets_misaligned_and_empty():
    t = T(0)
    keys = buckets([3 * t + b for b in range(10)], 8, 81)
    base = torch.from_numpy(np.concatenate([[7], keys, [9]]).astype(np.int32)).to(DEV)
    part, off = hs.hs_msd_partition(base[1:-1].clone(), 8)
    view = base[1:-1]
    view.copy_(part)
    hs.hs_sort_buckets(view, off, 8, 1)
    torch.cuda.synchronize()
    got = base.cpu().numpy()
    assert got[0] == 7 and got[-1] == 9
    assert np.array_equal(got[1:-1], np.sort(keys))
    e = torch.empty(0, dtype=torch.int32, device=DEV)
    hs.hs_sort_buckets(e, torch.zeros(11, dtype=torch.int64, device=DEV), 8, 8)


def test_split_half_sorted_bucket():
    """Chunks 0-3 of each bucket sorted, chunks 4-7 random: the sorted chunks put the bucket in map
    mode, the random ones use equal-width groups of fine bins."""
    t = T(0)
    rng = np.random.default_rng(93)
    D, c = 9, 8
    div = 10 ** (D - 1)
    parts = []
    for b in range(10):
        m = c * 3 * t
        half = np.sort(rng.integers(b * div, (b + 1) * div, size=m // 2))
        rest = rng.integers(b * div, (b + 1) * div, size=m - m // 2)
        parts.append(np.concatenate([half, rest]))
    keys = np.concatenate(parts).astype(np.int32)   # already bucket-major: the stable partition keeps it
    plan = check(keys, D, c)
    assert sum(plan["split"]) >= 8


def test_split_many_chunks_bucket_map():
    """c = 128 > kMapChunksMax: one sampled map per bucket (not per chunk); a skewed bucket still splits."""
    t, D, c = T(0), 9, 128
    div = 10 ** (D - 1)
    rng = np.random.default_rng(97)
    m = c * 2 * t
    peak = np.clip(rng.normal(3.4 * div, div / 30, size=m), 3 * div, 4 * div - 1).astype(np.int64)
    other = rng.integers(0, 10 * div, size=200_000)
    keys = np.concatenate([peak, other]).astype(np.int32)
    rng.shuffle(keys)
    plan = check(keys, D, c)
    assert plan["split"][3] == 1 and plan["levels"][3] == 7


def test_split_density_ramp():
    """Keys with a 1:3 linear density ramp inside every bucket: equal-width sub-ranges of 0.9 T would
    overflow at the dense end (~1.35 x the mean); the coarse skew test sends the buckets to the map."""
    t, D, c = T(0), 9, 8
    div = 10 ** (D - 1)
    rng = np.random.default_rng(101)
    m = c * 3 * t
    parts = []
    for b in range(10):
        u = rng.random(m)
        x = (np.sqrt(u * 8 + 1) - 1) / 2          # density rising linearly from 1 to 3 over [0, 1)
        parts.append(b * div + np.minimum((x * div).astype(np.int64), div - 1))
    keys = np.concatenate(parts).astype(np.int32)
    rng.shuffle(keys)
    plan = check(keys, D, c)
    assert sum(plan["split"]) == 10, plan


@pytest.mark.parametrize("c", [2, 8])
def test_split_big_pieces_int64_and_items(c):
    """The big-piece path (1-4 tiles per sub-range piece) on int64 keys and on hs_sort_pairs items
    (the int64 path with key = item >> 32): a dense value range inside one sub-range per chunk."""
    t, D = T(1), 18
    div = 10 ** (D - 1)
    rng = np.random.default_rng(77 + c)
    m = c * 3 * t
    parts = [rng.integers(b * div, (b + 1) * div, size=m) for b in range(10)]
    parts.append(rng.integers(5 * div + 10**9, 5 * div + 10**9 + 5 * t, size=int(2.5 * t) * c))
    keys = np.concatenate(parts).astype(np.int64)
    rng.shuffle(keys)
    plan = check(keys, D, c)
    assert plan["split"][5] == 1, plan
    k32 = (rng.integers(0, 10**9, size=c * 4 * T(1) * 10) // 1).astype(np.int32)
    k32[: int(2.5 * T(1)) * c * 3] = 500_000_123 + rng.integers(0, 2000, size=int(2.5 * T(1)) * c * 3)
    tags = rng.permutation(k32.size).astype(np.uint64)
    dk, dt = torch.from_numpy(k32).to(DEV), torch.from_numpy(tags.view(np.int64)).to(DEV)
    hs.hs_sort_pairs(dk, dt, 9, c)
    rk, rt = O.sort_pairs(k32, tags, 9, c)
    assert np.array_equal(dk.cpu().numpy(), rk) and np.array_equal(dt.cpu().numpy().view(np.uint64), rt)


def test_split_big_pieces_sorted_in_cta():
    """Sub-range pieces of 1-4 tiles (values with ~2.2 T copies per chunk, plus a narrow
    non-constant peak): the bucket keeps the split -- such a piece is sorted by its CTA as tiles +
    CTA-level merges (K5 big-piece path) instead of sending the bucket to the fallback."""
    t, D, c = T(0), 9, 8
    div = 10 ** (D - 1)
    rng = np.random.default_rng(2024)
    m = c * 3 * t
    parts = [rng.integers(b * div, (b + 1) * div, size=m) for b in range(10)]
    heavy = rng.integers(4 * div, 5 * div, size=5)
    parts.append(np.repeat(heavy, int(2.2 * t) * c))                          # bucket 4: five heavy values
    parts.append(rng.integers(7 * div + 1000, 7 * div + 1000 + 3 * t, size=int(2.5 * t) * c))  # bucket 7: dense
    keys = np.concatenate(parts).astype(np.int32)
    rng.shuffle(keys)
    plan = check(keys, D, c)
    assert plan["split"][4] == 1 and plan["split"][7] == 1, plan


@pytest.mark.parametrize("dtype,D", [(np.int32, 9), (np.int64, 18)])
def test_split_constant_pieces(dtype, D):
    """All keys of bucket 3 equal, and bucket 6 made of four values with ~6 tiles of copies per chunk
    each (far apart: one value per sub-range): every over-full piece is constant, so both buckets keep
    the split -- the pieces are filled from the count pass's min == max, not sorted."""
    t, c = T(0 if dtype == np.int32 else 1), 8
    div = 10 ** (D - 1)
    rng = np.random.default_rng(606)
    m = c * 3 * t
    parts = [rng.integers(b * div, (b + 1) * div, size=m) for b in range(10) if b not in (3, 6)]
    parts.append(np.full(c * 7 * t, 3 * div + 777))
    vals = 6 * div + np.array([1, 3, 5, 7]) * (div // 9)
    parts.append(np.repeat(vals, 6 * t * c))
    keys = np.concatenate(parts).astype(dtype)
    rng.shuffle(keys)
    plan = check(keys, D, c)
    assert plan["split"][3] == 1 and plan["split"][6] == 1, plan


def test_split_constant_piece_in_a_bucket_that_falls_back():
    """Bucket 3, c = 2: chunk 0's heavy sub-range piece is one value (6 tiles: constant, legal), chunk
    1's is the same value plus other keys of that sub-range (6.1 tiles, not constant: the bucket falls
    back).  The constant piece must then NOT be filled (the fill would overwrite the fallback's
    partitioned keys); exact either way."""
    t, D, c = T(0), 9, 2
    div = 10 ** (D - 1)
    rng = np.random.default_rng(4321)
    heavy = 3 * div + 777
    others = lambda m: rng.integers(3 * div + div // 8, 4 * div, size=m)   # outside the heavy sub-range
    chunk0 = np.concatenate([np.full(6 * t, heavy), others(2 * t)])
    chunk1 = np.concatenate([np.full(6 * t, heavy), rng.integers(3 * div, 3 * div + 1000, size=t // 10),
                             others(2 * t - t // 10)])
    rest = np.concatenate([rng.integers(b * div, (b + 1) * div, size=3 * t) for b in range(10) if b != 3])
    keys = np.concatenate([chunk0, chunk1, rest]).astype(np.int32)   # bucket 3 in this order: chunk 0 then 1
    plan = check(keys, D, c)
    assert plan["split"][3] == 0, plan


def _hidden_cluster(n, D, dtype, seed):
    """One bucket, one chunk (c = 1): every position K5a's phase-1 sample reads
    ((r n) >> 15 for r = 0, 8, ..., 32760; k_split_sample_map) holds a uniform key of
    digit 1, every other position a key of one narrow value range -- the sample sees a
    uniform bucket, so the bucket takes the padded layout (no count pass), and one
    region overflows: k_split_pad_plan must send the bucket back to the leaf plan."""
    div = 10 ** (D - 1)
    rng = np.random.default_rng(seed)
    keys = (div + div // 2 + rng.integers(0, 1000, n)).astype(dtype)   # the hidden cluster
    pos = (np.arange(0, 1 << 15, 8, dtype=np.int64) * n) >> 15
    keys[pos] = (div + rng.integers(0, div, pos.size)).astype(dtype)
    return keys


@pytest.mark.parametrize("dtype,D", [(np.int32, 9), (np.int64, 18)])
def test_split_padded_region_overflow_falls_back(dtype, D):
    n = 1 << 20
    keys = _hidden_cluster(n, D, dtype, 77)
    plan = check(keys, D, 1)
    assert plan["split"][1] == 0, plan          # the overflow was caught after the scatter


@pytest.mark.parametrize("dtype,D", [(np.int32, 9), (np.int64, 18)])
def test_split_padded_next_to_counted_buckets(dtype, D):
    """Padded (uniform) buckets beside a counted one (a dense core: constant tracking, sampled
    map) and a bucket whose padded region overflows -- each path in one call."""
    t, c = T(0 if dtype == np.int32 else 1), 4
    div = 10 ** (D - 1)
    rng = np.random.default_rng(5)
    uni = buckets([c * 3 * t] * 10, D, 61, dtype=dtype)
    core = (5 * div + rng.integers(0, 1000, c * 3 * t)).astype(dtype)   # bucket 5: dense core
    hid = _hidden_cluster(c * 6 * t, D, dtype, 62)                       # bucket 1: hidden cluster
    keys = np.concatenate([uni, core, hid])
    plan = check(keys, D, c)
    assert sum(plan["split"][b] for b in (0, 2, 3, 4, 6, 7, 8, 9)) == 8, plan
    assert sum(plan["padded"][b] for b in (0, 2, 3, 4, 6, 7, 8, 9)) == 8, plan
    assert plan["padded"][5] == 0, plan         # the dense core is counted (constant tracking)


@pytest.mark.parametrize("kind", ["uniform", "fallback"])
def test_graph_replay_gates_extra_levels(kind):
    """SortGraph (CUDA-graph capture of hs_sort): the merge levels past the log2 c tree levels sit
    behind a conditional node the device plan opens.  A uniform input skips them; a padded bucket
    that overflows (fallback: k in-chunk levels) needs them -- both must replay to the oracle's
    result, twice (the gate is re-evaluated on every replay)."""
    t = T(0)
    if kind == "uniform":
        keys = buckets([2 * 3 * t] * 10, 9, 71)
        c = 2
    else:
        keys = _hidden_cluster(1 << 20, 9, np.int32, 72)
        c = 1
    d = torch.from_numpy(np.ascontiguousarray(keys)).to(DEV)
    plan = hs.hs_sort_plan(d, 9, c)
    if kind == "fallback":
        assert plan["split"][1] == 0 and plan["levels"][1] > 0, plan
    buf = torch.empty_like(d)
    g = hs.SortGraph(buf, 9, c)
    ref = O.sort(keys, 9, c)
    for _ in range(2):
        buf.copy_(d)
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(buf.cpu().numpy(), ref)


@pytest.mark.parametrize("power", [4, 12])
def test_tile_rebucket_steep_density(power):
    """Leaves whose keys crowd one end of their range (density ~ x^(1/p - 1)): the tile sort's
    equal-width buckets overflow there, and the tile re-buckets by an equal-count map interpolated
    from its first-pass histogram (or, if that still overflows, takes the merge rounds) -- bit-exact
    either way, through hs_sort (chunks of one tile: no split) and hs_sort_chunks."""
    t, c = T(0), 8
    rng = np.random.default_rng(90 + power)
    n = c * (t - 1000)
    u = rng.random(n)
    keys = (10**8 + np.floor(u ** power * (10**8 - 1))).astype(np.int32)
    check(keys, 9, c)
    d = torch.from_numpy(keys).to(DEV)
    out, off = hs.hs_msd_partition(d, 9)
    chunks = torch.empty_like(out)
    hs.hs_sort_chunks(out, off, c, out=chunks)
    torch.cuda.synchronize()
    p_ref, off_ref = O.msd_partition(keys, 9)
    ref = O.sort_chunks(p_ref, off_ref, c)
    assert np.array_equal(chunks.cpu().numpy(), ref)
