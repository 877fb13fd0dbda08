"""The paper's chunk tree (a6) run on chip in one HBM pass (k_tree.cu)
for buckets whose chunks K5a split into equal-width sub-ranges: parity with the
oracle on inputs that take it (c = 2, 8: odd log2 c <= 3), that cannot take it
(c = 4, 16, 32), and that fall back from it to the merge levels (a fine key bin
with more copies than a segment can hold), plus int64 keys, key + tag items,
clamped keys, misaligned views and pre-partitioned buckets.  ``hs_sort_plan``
reports which path every bucket takes (split 2 = on-chip tree), so the cases
provably cover each one."""
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


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def assert_same(got, ref, what=""):
    assert got.shape == ref.shape, (what, got.shape, ref.shape)
    if not np.array_equal(got, ref):
        bad = np.nonzero(got != ref)[0]
        raise AssertionError(f"{what}: {bad.size} mismatches, first at {bad[0]}: got {got[bad[0]]} want {ref[bad[0]]}")


def sort_and_plan(keys, D, c):
    d = dev(keys)
    plan = hs.hs_sort_plan(d, D, c)
    hs.hs_sort(d, D, c)
    torch.cuda.synchronize()
    got = d.cpu().numpy()
    assert_same(got, O.sort(keys, D, c), f"hs_sort c={c}")
    return plan


def uniform_buckets(per_bucket, D, seed, dtype=np.int32):
    div = 10 ** (D - 1)
    rng = np.random.default_rng(seed)
    k = np.concatenate([rng.integers(b * div, (b + 1) * div, size=per_bucket, dtype=np.int64) for b in range(10)])
    rng.shuffle(k)
    return k.astype(dtype)


@pytest.mark.parametrize("c", [2, 8])
def test_tree_uniform_takes_the_on_chip_tree(c):
    T = hs.tile_keys(0, 1)
    keys = uniform_buckets(3 * T * c + 12_345, 9, 1000 + c)
    plan = sort_and_plan(keys, 9, c)
    assert plan["split"] == [1] * 10 and plan["tree"] == [1] * 10, plan


@pytest.mark.parametrize("c", [4, 16, 32])
def test_tree_even_rounds_keep_the_levels(c):
    T = hs.tile_keys(0, 1)
    keys = uniform_buckets(2 * T * c + 777, 9, 2000 + c)
    plan = sort_and_plan(keys, 9, c)
    assert plan["split"] == [1] * 10 and plan["tree"] == [0] * 10, plan


def test_tree_heavy_duplicates_fall_back_per_bucket():
    """Bucket 3: 70% of its keys are 100 values with ~4.6k copies each (~570 per chunk, so every
    sub-range piece still fits a tile) -- some key segment of 32 fine bins then holds more keys
    than the tree merge takes, the tree check marks the bucket and its merge levels run instead;
    the other buckets keep the on-chip tree.  Both exact."""
    T = hs.tile_keys(0, 1)
    c = 8
    m = 3 * T * c
    rng = np.random.default_rng(77)
    div = 10**8
    parts = []
    for b in range(10):
        if b == 3:
            vals = rng.integers(3 * div, 4 * div, size=100)
            dup = vals[rng.integers(0, 100, size=int(0.7 * m))]
            parts.append(np.concatenate([dup, rng.integers(3 * div, 4 * div, size=m - dup.size)]))
        else:
            parts.append(rng.integers(b * div, (b + 1) * div, size=m))
    keys = np.concatenate(parts)
    rng.shuffle(keys)
    keys = keys.astype(np.int32)
    plan = sort_and_plan(keys, 9, c)
    assert plan["split"][3] == 1 and plan["tree"][3] == 0, plan
    assert all(plan["tree"][b] == 1 for b in range(10) if b != 3), plan


def test_tree_int64():
    T = hs.tile_keys(1, 1)
    keys = uniform_buckets(3 * T * 8 + 99, 18, 31, dtype=np.int64)
    plan = sort_and_plan(keys, 18, 8)
    assert plan["tree"] == [1] * 10, plan


def test_tree_clamped_and_extreme_keys():
    """Negative keys clamp into bucket 0's first sub-range, keys >= 10^D into bucket 9's last:
    the tree map sends them to the first / last fine bin (still monotone)."""
    T = hs.tile_keys(0, 1)
    keys = uniform_buckets(3 * T * 8, 9, 5)
    rng = np.random.default_rng(6)
    idx = rng.choice(keys.size, 3000, replace=False)
    keys[idx[:1000]] = rng.integers(-2**31, 0, size=1000)
    keys[idx[1000:2000]] = rng.integers(10**9, 2**31 - 1, size=1000)
    keys[idx[2000]] = -2**31
    keys[idx[2001]] = 2**31 - 1
    sort_and_plan(keys, 9, 8)


def test_tree_pairs_stable():
    """Key + tag items (hs_sort_pairs) through the on-chip tree: keys sorted, ties in input order."""
    T = hs.tile_keys(1, 1)  # items travel through the int64 path
    keys = uniform_buckets(3 * T * 8, 9, 8)
    keys[::7] = keys[0]  # many ties
    tags = np.arange(keys.size, dtype=np.uint64) * np.uint64(2654435761)
    dk, dt = dev(keys), dev(tags.view(np.int64))
    hs.hs_sort_pairs(dk, dt, 9, 8)
    rk, rt = O.sort_pairs(keys, tags, 9, 8)
    assert_same(dk.cpu().numpy(), rk, "keys")
    assert_same(dt.cpu().numpy().view(np.uint64), rt, "tags")


@pytest.mark.parametrize("shift", [1, 2, 3])
def test_tree_misaligned_view(shift):
    T = hs.tile_keys(0, 1)
    keys = uniform_buckets(3 * T * 2 + 5, 9, 40 + shift)
    n = keys.size
    full = dev(np.concatenate([np.full(shift, 7, np.int32), keys, np.full(5, 9, np.int32)]))
    view = full[shift:shift + n]
    hs.hs_sort(view, 9, 2)
    got = full.cpu().numpy()
    assert np.all(got[:shift] == 7) and np.all(got[shift + n:] == 9)
    assert_same(got[shift:shift + n], O.sort(keys, 9, 2), "view")


def test_tree_sort_buckets_after_partition():
    cfg = W.CONFIGS["C2"]
    keys = W.generate("C2")
    part, off = O.msd_partition(keys, cfg.num_digits)
    d = dev(part.astype(keys.dtype))
    hs.hs_sort_buckets(d, dev(off), cfg.num_digits, 8)
    assert_same(d.cpu().numpy(), O.sort(keys, cfg.num_digits, 8), "hs_sort_buckets C2")


@pytest.mark.parametrize("name", ["C2", "C4"])
def test_tree_plan_on_configs(name):
    """C2 (uniform): every bucket on chip; C4 (skewed mixture): the peak buckets take sampled
    maps (no common key interval across chunks: levels), the 1024-value table's duplicates
    push some uniform buckets back to the levels; all exact."""
    cfg = W.CONFIGS[name]
    keys = W.generate(name)
    plan = sort_and_plan(keys, cfg.num_digits, cfg.chunks)
    if name == "C2":
        assert plan["tree"] == [1] * 10, plan
