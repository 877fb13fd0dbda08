"""Small calls of every entry point, checked against the oracle; run under
compute-sanitizer by tests/sanitize.sh (one tool per run)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle as O
import paper_2003_01216_b200 as hs
import workload as W


def main():
    dev = "cuda:0"
    for n, dt, D in [(1, np.int32, 6), (1000, np.int32, 6), (40_001, np.int32, 9), (30_003, np.int64, 18)]:
        keys = W.uniform(n, 11 + n % 7, 10 ** D, dtype=dt)
        d = torch.from_numpy(keys).to(dev)
        hs.hs_sort(d, D, 8)
        assert np.array_equal(d.cpu().numpy(), O.sort(keys, D, 8)), ("sort", n, dt)
        out, off = hs.hs_msd_partition(torch.from_numpy(keys).to(dev), D)
        ro, roff = O.msd_partition(keys, D)
        assert np.array_equal(out.cpu().numpy(), ro) and np.array_equal(off.cpu().numpy(), roff)
        x = torch.from_numpy(ro).to(dev)
        sc = hs.hs_sort_chunks(x, off, 4)
        assert np.array_equal(sc.cpu().numpy(), O.sort_chunks(ro, roff, 4))
        mg = hs.hs_merge(sc, off, 4)
        assert np.array_equal(mg.cpu().numpy(), O.sort(keys, D, 4))
        s2 = torch.from_numpy(keys).to(dev)
        hs.hs_sort_shared(s2, 8)
        assert np.array_equal(s2.cpu().numpy(), np.sort(keys))
    keys = W.uniform(20_011, 5, 1000, dtype=np.int32)
    tags = np.arange(keys.size, dtype=np.int64)
    dk, dt_ = torch.from_numpy(keys).to(dev), torch.from_numpy(tags).to(dev)
    hs.hs_sort_pairs(dk, dt_, 3, 8)
    rk, rt = O.sort_pairs(keys, tags.astype(np.uint64), 3, 8)
    assert np.array_equal(dk.cpu().numpy(), rk) and np.array_equal(dt_.cpu().numpy().view(np.uint64), rt)
    torch.cuda.synchronize()
    print("sanitize driver: all calls bit-exact")


if __name__ == "__main__":
    main()
