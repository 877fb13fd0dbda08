"""Quick device timing of hs_sort / hs_msd_partition per config (dev aid, not the bench)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2003_01216_b200 as hs
import workload as W

names = sys.argv[1:] or ["C1", "C2", "C3", "C4", "C5"]
for name in names:
    cfg = W.CONFIGS[name]
    keys = W.generate(name)
    src = torch.from_numpy(keys).cuda()
    buf = src.clone()
    out = torch.empty_like(src)
    off = torch.empty(11, dtype=torch.int64, device="cuda")
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    res = {}
    for what in ("partition", "sort"):
        ts = []
        for it in range(8):
            buf.copy_(src)
            torch.cuda.synchronize()
            s.record()
            if what == "sort":
                hs.hs_sort(buf, cfg.num_digits, cfg.chunks)
            else:
                hs.hs_msd_partition(buf, cfg.num_digits, out=out, bucket_offsets=off)
            e.record()
            torch.cuda.synchronize()
            if it >= 3:
                ts.append(s.elapsed_time(e))
        res[what] = float(np.median(ts))
    ok = bool(torch.all(buf[1:] >= buf[:-1]))
    launches = hs.last_launch_count()
    # the same call replayed from a CUDA graph (SortGraph; the bench's launch configuration): no
    # per-launch host work, the merge levels past the tree rounds behind the device-opened gate
    gbuf = src.clone()
    g = hs.SortGraph(gbuf, cfg.num_digits, cfg.chunks)
    ts = []
    for it in range(8):
        gbuf.copy_(src)
        torch.cuda.synchronize()
        s.record()
        g.replay()
        e.record()
        torch.cuda.synchronize()
        if it >= 3:
            ts.append(s.elapsed_time(e))
    res["graph"] = float(np.median(ts))
    ok = ok and bool(torch.all(gbuf[1:] >= gbuf[:-1]))
    print(f"{name}: n={cfg.n} partition {res['partition']:.3f} ms  sort {res['sort']:.3f} ms "
          f"= {cfg.n / res['sort'] / 1e6:.2f} Gkeys/s  graph {res['graph']:.3f} ms = "
          f"{cfg.n / res['graph'] / 1e6:.2f} Gkeys/s  sorted={ok} launches={launches}", flush=True)
    del g, gbuf
    del src, buf, out
    torch.cuda.empty_cache()
