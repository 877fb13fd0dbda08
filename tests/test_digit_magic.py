"""Pin of the device's leading-digit arithmetic (K1/K3, hs_device.cuh msd_digit).

The kernels compute d(k) = clamp(floor(k / 10^(D-1)), 0, 9) (readings
#1, #3) by one multiply-high and a shift: magic = ceil(2^(N+l) / div),
l = ceil(log2 div), N = w - 1, q = mulhi_w(u, magic) >> (l - 1) (div = 1:
q = u).  This mirror of digit_params (hs_api.cu) checks the scheme against
Python's exact floor division at every digit boundary +-2 and on random keys
of the full non-negative range, for every D of both key widths.  The GPU tests
(test_partition_digit_boundaries) then check the kernels themselves.
"""
import random


def params(D, w):
    d = 10 ** (D - 1)
    l = 0
    while (1 << l) < d:
        l += 1
    magic = 0 if d == 1 else -(-(1 << (w - 1 + l)) // d)
    assert magic < (1 << w)
    return d, magic, (-1 if d == 1 else l - 1)


def digit(k, D, w):
    d, magic, post = params(D, w)
    u = max(k, 0)
    q = ((u * magic) >> w) >> post if post >= 0 else u
    return min(q, 9)


def test_magic_digit_exact():
    rng = random.Random(78)
    for w, dmax in ((32, 10), (64, 19)):
        for D in range(1, dmax + 1):
            d = 10 ** (D - 1)
            keys = [0, 1, (1 << (w - 1)) - 1, -1, -(1 << (w - 1))]
            keys += [j * d + e for j in range(11) for e in (-2, -1, 0, 1, 2) if 0 <= j * d + e < (1 << (w - 1))]
            keys += [rng.randrange(0, 1 << (w - 1)) for _ in range(3000)]
            for k in keys:
                assert digit(k, D, w) == min(max(k, 0) // d, 9), (w, D, k)
