"""The ABI's largest call: n = 2^31 - 1 int32 keys (include/hs.h: 0 <= n < 2^31) through hs_sort
on the GPU -- every 32-bit position, cursor and leaf index at its limit (split table, padded
regions, merge blocks).  The oracle would take minutes at this size, so the result is checked by
properties that hold at any size: non-decreasing order, and the same multiset as the input
(count, sum, sum of squares and a 65,536-bin histogram of the low 16 bits), computed with
torch in slices on the device; int64 keys (D = 18) as well.  D = 9 runs the K5a split (padded layout) everywhere; D = 10 over
[0, 2^31 - 1) fills only buckets 0-2, whose chunks (~125M keys) need more sub-ranges than the split
takes (4096), so they run the leaf plan: 13 in-chunk merge levels + the 3 tree levels."""
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2003_01216_b200 as hs  # noqa: E402

N = (1 << 31) - 1


def _props(x):
    s = s2 = 0
    h = torch.zeros(1 << 16, dtype=torch.int64, device=x.device)
    for i in range(0, x.numel(), 1 << 27):
        c = x[i:i + (1 << 27)].to(torch.int64)
        s = (s + int(c.sum())) % (1 << 64)  # int64 sums wrap: compare mod 2^64
        s2 = (s2 + int((c * c).sum())) % (1 << 64)
        h += torch.bincount(c & 0xFFFF, minlength=1 << 16)
    return s, s2, h


def _sorted(x):
    ok = True
    for i in range(0, x.numel() - 1, 1 << 27):
        c = x[i:i + (1 << 27) + 1]
        ok &= bool(torch.all(c[1:] >= c[:-1]))
    return ok


@pytest.mark.parametrize("dtype,D,hi", [(torch.int32, 9, 10**9), (torch.int32, 10, 2**31 - 1),
                                        (torch.int64, 18, 10**18)])
def test_max_size_hs_sort(dtype, D, hi):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    free, _ = torch.cuda.mem_get_info()
    need = (40 if dtype == torch.int32 else 80) * (1 << 30)
    if free < need:
        pytest.skip(f"needs ~{need >> 30} GiB of free device memory")
    g = torch.Generator(device="cuda").manual_seed(2024 + D)
    x = torch.randint(0, hi, (N,), dtype=dtype, device="cuda", generator=g)
    before = _props(x)
    hs.hs_sort(x, D, 8)
    torch.cuda.synchronize()
    assert _sorted(x)
    after = _props(x)
    assert before[0] == after[0] and before[1] == after[1]
    assert torch.equal(before[2], after[2])
    del x
    torch.cuda.empty_cache()
