"""hs_sort on input shapes beyond the BASELINE configs (the distribution sweep of
tools/dist_sweep.py at 2^22 keys), element by element against the oracle.  They
exercise every K5a outcome: equal-width split, per-chunk sampled maps (sorted,
ramp, normal peak), and the in-chunk-merge fallback (heavy duplicates)."""
import numpy as np
import pytest

import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2003_01216_b200 as hs  # noqa: E402

N, D, C = 1 << 22, 9, 8
rng = np.random.default_rng(2024)


def _shape(name):
    if name == "uniform":
        return rng.integers(0, 10**9, N)
    if name == "normal":
        return np.clip(rng.normal(5e8, 2e7, N), 0, 10**9 - 1)
    if name == "sorted":
        return np.arange(N, dtype=np.int64) * 199
    if name == "reversed":
        return (np.arange(N, dtype=np.int64) * 199)[::-1]
    if name == "1000 values":
        return rng.integers(0, 1000, N) * 999_983
    if name == "exponential":
        return np.clip(rng.exponential(5e7, N), 0, 10**9 - 1)
    if name == "all equal":
        return np.full(N, 123_456_789)
    if name == "ramp":
        b = rng.integers(0, 10, N)
        x = (np.sqrt(rng.random(N) * 8 + 1) - 1) / 2
        return b * 10**8 + np.minimum((x * 10**8).astype(np.int64), 10**8 - 1)
    if name == "sorted runs":
        return np.sort(rng.integers(0, 10**9, N).reshape(-1, 1 << 14), axis=1).reshape(-1)
    raise KeyError(name)


@pytest.mark.parametrize("name", ["uniform", "normal", "sorted", "reversed", "1000 values", "exponential",
                                  "all equal", "ramp", "sorted runs"])
def test_shape_parity(name):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    keys = np.ascontiguousarray(_shape(name).astype(np.int32))
    d = torch.from_numpy(keys).to("cuda:0")
    hs.hs_sort(d, D, C)
    torch.cuda.synchronize()
    assert np.array_equal(d.cpu().numpy(), O.sort(keys, D, C)), name


def _shape64(name):
    if name == "uniform":
        return rng.integers(0, 10**18, N)
    if name == "near-duplicate clusters":
        # groups of 4 keys within 1000 of each other: inside a K5 bucket spanning > 2^27 values
        # they share the 32-bit rank's high part, so the rank network leaves them in slot
        # order and the repair pass must order them (k_tilesort.cu, HS_SORT_RANK64)
        c = np.repeat(rng.integers(0, 10**18 - 1000, N // 4), 4)
        return rng.permutation(c + rng.integers(0, 1000, N))
    if name == "dense core + wide tail":
        core = 5 * 10**17 + rng.integers(0, 10**6, N // 2)
        return rng.permutation(np.concatenate([core, rng.integers(0, 10**18, N - N // 2)]))
    raise KeyError(name)


@pytest.mark.parametrize("name", ["uniform", "near-duplicate clusters", "dense core + wide tail"])
def test_shape_parity_int64(name):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    keys = np.ascontiguousarray(_shape64(name).astype(np.int64))
    d = torch.from_numpy(keys).to("cuda:0")
    hs.hs_sort(d, 18, C)
    torch.cuda.synchronize()
    assert np.array_equal(d.cpu().numpy(), O.sort(keys, 18, C)), name
