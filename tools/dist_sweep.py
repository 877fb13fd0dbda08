"""Distribution sweep (dev aid): hs_sort time and split decisions at 2^28 int32 keys, D = 9, c = 8,
for input shapes beyond the uniform headline config.  Correctness: sorted order and the multiset
(sum and sum of squares) checked with torch on the device."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2003_01216_b200 as hs

if os.environ.get("HS_VARIANT"):  # a variant build from tools/exp.py (var/NAME/libhybridsort.so)
    hs._LIB = hs.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "var",
                                   os.environ["HS_VARIANT"], "libhybridsort.so"))

n = 1 << 28
g = torch.Generator(device="cuda").manual_seed(7)
def uni(lo, hi, size):
    return torch.randint(lo, hi, (size,), device="cuda", generator=g, dtype=torch.int64)

cases = {
    "uniform [0,1e9)": lambda: uni(0, 10**9, n),
    "normal(5e8, 2e7)": lambda: (torch.randn(n, device="cuda", generator=g) * 2e7 + 5e8).clamp(0, 10**9 - 1).long(),
    "sorted": lambda: torch.arange(n, device="cuda") * 3,
    "reversed": lambda: torch.arange(n, device="cuda").flip(0) * 3,
    "1000 distinct values": lambda: uni(0, 1000, n) * 999_983,
    "exponential (scale 5e7)": lambda: (torch.empty(n, device="cuda").exponential_(generator=g) * 5e7).clamp(0, 10**9 - 1).long(),
    "all equal": lambda: torch.full((n,), 123_456_789, device="cuda", dtype=torch.int64),
    "linear ramp 1:3 per bucket": lambda: (torch.div(uni(0, 10**9, n), 10**8, rounding_mode="floor") * 10**8
                                           + (torch.sqrt(torch.rand(n, device="cuda", generator=g) * 8 + 1) - 1)
                                           .mul(10**8 / 2).long().clamp(0, 10**8 - 1)),
    "sorted runs of 2^16": lambda: torch.sort(uni(0, 10**9, n).view(-1, 1 << 16), dim=1).values.reshape(-1),
}
for name, make in cases.items():
    k = make().to(torch.int32)
    s1, s2 = k.long().sum().item(), (k.double() ** 2).sum().item()
    plan = hs.hs_sort_plan(k, 9, 8)
    ts = []
    for _ in range(4):
        b = k.clone()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); hs.hs_sort(b, 9, 8); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ok = bool((b[1:] >= b[:-1]).all()) and b.long().sum().item() == s1 and abs((b.double() ** 2).sum().item() - s2) <= 1e-9 * s2
    ms = sorted(ts)[1]
    print(f"{name:28s} {ms:7.3f} ms {n / ms / 1e6:6.1f} Gkeys/s  ok={ok}  split={plan['split']}  levels={plan['levels']}")
    if "--kernels" in sys.argv:
        b = k.clone()
        hs.profile_enable(True)
        hs.hs_sort(b, 9, 8)
        prof = hs.profile_read()
        hs.profile_enable(False)
        print("      " + "  ".join(f"{kk} {v[0]:.3f}" for kk, v in sorted(prof.items(), key=lambda kv: -kv[1][0]) if v[1]))
    del k, b
    torch.cuda.empty_cache()
