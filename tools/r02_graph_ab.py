"""Graph-replay timing of hs_sort for library variants (dev aid): one process per variant."""
import os, sys, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

def one(name, cfg_name):
    import torch, numpy as np, ctypes
    import paper_2003_01216_b200 as hs
    import workload as W
    path = hs._build.SO if name == "main" else os.path.join(ROOT, "var", name, "libhybridsort.so")
    hs._LIB = hs.load(path)
    cfg = W.CONFIGS[cfg_name]
    src = torch.from_numpy(W.generate(cfg_name)).cuda()
    buf = src.clone()
    g = hs.SortGraph(buf, cfg.num_digits, cfg.chunks)
    ts = []
    for i in range(15):
        buf.copy_(src)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); b.record(); torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b))
    ok = bool(torch.all(buf[1:] >= buf[:-1]))
    print(f"{name} {cfg_name}: graph replay median {np.median(ts):.3f} ms ({cfg.n / np.median(ts) / 1e6:.2f} Gkeys/s) sorted={ok}", flush=True)

if __name__ == "__main__":
    if sys.argv[1] == "one":
        one(sys.argv[2], sys.argv[3])
    else:
        cfg = os.environ.get("CFG", "C3")
        for name in sys.argv[1:]:
            subprocess.call([sys.executable, __file__, "one", name, cfg])
