"""Dev probe: hs_sort twice on 2^28 normal(5e8, 2e7) int32 keys (the dist sweep's skewed case), for
ncu captures of the second call's kernels."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2003_01216_b200 as hs

n = 1 << 28
g = torch.Generator(device="cuda").manual_seed(7)
k = (torch.randn(n, device="cuda", generator=g) * 2e7 + 5e8).clamp(0, 10**9 - 1).long().to(torch.int32)
print(hs.hs_sort_plan(k, 9, 8))
for _ in range(2):
    b = k.clone()
    hs.hs_sort(b, 9, 8)
    torch.cuda.synchronize()
print("sorted", bool((b[1:] >= b[:-1]).all()))
