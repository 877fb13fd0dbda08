"""Run one warm-up and one measured call of an API on a config (for ncu launch lists)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2003_01216_b200 as hs
import workload as W

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
what = sys.argv[2] if len(sys.argv) > 2 else "sort"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
cfg = W.CONFIGS[name]
src = torch.from_numpy(W.generate(name)).cuda()
buf = src.clone()
out = torch.empty_like(src)
for _ in range(reps):
    buf.copy_(src)
    if what == "sort":
        hs.hs_sort(buf, cfg.num_digits, cfg.chunks)
    else:
        hs.hs_msd_partition(buf, cfg.num_digits, out=out)
    torch.cuda.synchronize()
print("done", name, what, hs.last_launch_count())
