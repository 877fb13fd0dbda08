"""multi-GPU bucket sharding (the paper's cluster model).

CPU (``-m "not gpu"``): hs_assign_buckets against brute force and SPEC's
examples, and dist_sort's host logic (histogram all-gather,
digit-group assignment, one all-to-all-v, local sort) on world sizes 2 and 3
with the gloo backend, the per-rank partition / sort supplied by the CPU
oracle (test infrastructure).  The concatenated rank outputs must equal the
sorted union (np.sort and the oracle), every rank's keys must carry only its
group's digits (range disjointness), and every rank sends exactly one
contiguous segment to each other rank ("one data message").

GPU (``-m gpu``): the product ops (hs_msd_partition + hs_sort) through
dist_sort on a world of one NCCL rank -- only one GPU is available here, so
the N > 1 exchange is covered by the gloo tests.
"""
import itertools
import os
import socket

import numpy as np
import pytest
import torch

import oracle as O
import workload as W


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


# ------------------------------------------------------------ assign_buckets
def brute_assign(sizes, m):
    best = None
    for cuts in itertools.combinations(range(1, 10), m - 1):   # lexicographic order
        b = (0,) + cuts + (10,)
        load = max(sum(sizes[b[g]:b[g + 1]]) for g in range(m))
        if best is None or load < best[1]:
            best = (list(b), load)
    return best


def test_assign_buckets_spec_examples():
    import paper_2003_01216_b200 as hs
    assert hs.assign_buckets([7] * 10, 10) == (list(range(11)), 7)
    assert hs.assign_buckets([3] * 10, 5) == ([0, 2, 4, 6, 8, 10], 6)
    assert hs.assign_buckets([100] + [0] * 8 + [100], 2) == ([0, 1, 10], 100)
    with pytest.raises(hs.HybridSortError):
        hs.assign_buckets([1] * 10, 0)
    with pytest.raises(hs.HybridSortError):
        hs.assign_buckets([1] * 10, 11)


def test_assign_buckets_bruteforce():
    import paper_2003_01216_b200 as hs
    rng = np.random.default_rng(308)
    for _ in range(300):
        m = int(rng.integers(1, 11))
        sizes = rng.integers(0, 50, size=10).tolist()
        if rng.random() < 0.3:
            sizes = rng.choice([0, 1, 1000], size=10).tolist()
        assert hs.assign_buckets(sizes, m) == tuple(brute_assign(sizes, m)), (sizes, m)


# ------------------------------------------------------------ dist_sort, gloo
class OracleOps:
    """CPU stand-ins for the per-rank steps (oracle = test infrastructure)."""

    @staticmethod
    def partition(keys, num_digits):
        out, off = O.msd_partition(keys.numpy(), num_digits)
        return torch.from_numpy(out.astype(keys.numpy().dtype)), torch.from_numpy(off.astype(np.int64))

    @staticmethod
    def sort(keys, num_digits, chunks):
        keys.copy_(torch.from_numpy(O.sort(keys.numpy(), num_digits, chunks)))


def _worker(rank, world, port, cases, q):
    import torch.distributed as dist
    from paper_2003_01216_b200 import dist as hd
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for ci, case in enumerate(cases):
            keys = _case_keys(case, rank, world)
            local, info = hd.dist_sort(torch.from_numpy(keys), case["D"], 8, ops=OracleOps)
            full = hd.gather_to(local, 0)
            q.put((ci, rank, local.numpy(), info.group_start, info.send_counts, info.recv_counts,
                   None if full is None else full.numpy()))
    finally:
        dist.destroy_process_group()


def _case_keys(case, rank, world):
    n = case["n"]
    if case["kind"] == "uniform":
        return W.uniform(n, 1000 * case["seed"] + rank, 10 ** case["D"], dtype=np.int32)
    if case["kind"] == "skewed":   # rank 0 heavy in digit 3, others uniform (unbalanced buckets)
        k = W.uniform(n, 50 + rank, 10 ** case["D"], dtype=np.int32)
        if rank == 0:
            k[: n // 2] = 3 * 10 ** (case["D"] - 1) + k[: n // 2] % 1000
        return k
    if case["kind"] == "p3":       # the paper's 3-digit keys
        return W.generate("P3", rank * n, n)
    raise ValueError(case)


CASES = {
    2: [{"n": 20_000, "D": 9, "kind": "uniform", "seed": 1},
        {"n": 30_000, "D": 3, "kind": "p3", "seed": 3},
        {"n": 0, "D": 9, "kind": "uniform", "seed": 4}],
    3: [{"n": 15_001, "D": 6, "kind": "skewed", "seed": 2},
        {"n": 9_999, "D": 9, "kind": "uniform", "seed": 5}],
}


@pytest.mark.parametrize("world", [2, 3])
def test_dist_sort_gloo(world):
    import multiprocessing as pymp
    ctx = pymp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    cases = CASES[world]
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=180) for _ in range(world * len(cases))]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for ci, case in enumerate(cases):
        res = sorted([g[1:] for g in got if g[0] == ci], key=lambda t: t[0])
        allkeys = np.concatenate([_case_keys(case, r, world) for r in range(world)])
        concat = np.concatenate([r[1] for r in res])
        assert np.array_equal(concat, np.sort(allkeys)), case
        assert np.array_equal(concat, O.sort(allkeys, case["D"], 8)), case
        assert np.array_equal(res[0][5], concat)                     # gather_to(rank 0)
        gs = res[0][2]
        for r, local, g, send, recv, _ in res:
            assert g == gs                                           # same assignment everywhere
            if local.size:                                           # only its group's digits
                d = O.histogram(local, case["D"])
                lo, hi = g[r], g[r + 1]
                assert d[:lo].sum() == 0 and d[hi:].sum() == 0
            assert sum(send) == case["n"]                            # one segment per destination
        sent = np.array([r[3] for r in res])
        recvd = np.array([r[4] for r in res])
        assert np.array_equal(sent, recvd.T)                         # conservation of the exchange


# ------------------------------------------------------------ GPU, one rank
@pytest.mark.gpu
def test_dist_sort_one_rank_nccl():
    import torch.distributed as dist
    from paper_2003_01216_b200 import dist as hd
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        keys = W.generate("C1")
        local, info = hd.dist_sort(torch.from_numpy(keys).cuda(), 6, 8)
        torch.cuda.synchronize()
        assert np.array_equal(local.cpu().numpy(), O.sort(keys, 6, 8))
        assert info.group_start == [0, 10] and info.send_counts == [keys.size]
    finally:
        dist.destroy_process_group()


# ------------------------------------------------------------ fused exchange layout (CPU)
def test_exchange_layout_simulated():
    """The fused exchange's layout: every (rank, digit) segment lands once, owners' buffers are
    partitioned by digit, and chunk sort + tree merge of each buffer gives the sorted union."""
    from paper_2003_01216_b200.dist import exchange_layout
    import paper_2003_01216_b200 as hs
    rng = np.random.default_rng(80)
    for world in (1, 2, 3, 4, 12):
        keys = [W.uniform(int(rng.integers(0, 3000)), 10 + r, 10**6, dtype=np.int32) for r in range(world)]
        if world > 1:
            keys[1][: keys[1].size // 2] = 400_000 + keys[1][: keys[1].size // 2] % 1000  # skew
        parts = [O.msd_partition(k, 6) for k in keys]
        sizes = [np.diff(off).tolist() for _, off in parts]
        gs, _ = hs.assign_buckets([sum(s[d] for s in sizes) for d in range(10)], min(world, 10))
        owner, offset, roff, rtot = exchange_layout(sizes, gs)
        bufs = [np.full(t, -1, dtype=np.int32) for t in rtot]
        for r, (part, off) in enumerate(parts):       # what every rank's fused scatter stores
            for d in range(10):
                seg = part[off[d]:off[d + 1]]
                b = bufs[owner[d]]
                assert (b[offset[r][d]:offset[r][d] + seg.size] == -1).all()   # written once
                b[offset[r][d]:offset[r][d] + seg.size] = seg
        out = []
        for g in range(world):
            assert (bufs[g] >= 0).all()                                         # fully covered
            if bufs[g].size:
                d = O.histogram(bufs[g], 6)
                assert np.array_equal(np.diff(roff[g]), d)                      # partitioned by digit
                x = O.sort_chunks(bufs[g], np.array(roff[g]), 8)
                out.append(O.merge(x, np.array(roff[g]), 8))
        allk = np.concatenate(keys)
        assert np.array_equal(np.concatenate(out) if out else allk[:0], np.sort(allk))


@pytest.mark.gpu
def test_dist_sort_fused_one_rank():
    """The fused path end to end on one rank: K1-K2, symmetric-memory buffer, K3 storing into it
    through peer pointers (self), chunk sort + tree merge in place."""
    import torch.distributed as dist
    from paper_2003_01216_b200 import dist as hd
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        for name, n in (("C1", None), ("C4", 2_000_000), ("P3", 1_000_000)):
            cfg = W.CONFIGS[name]
            keys = W.generate(name, 0, n)
            local, info = hd.dist_sort_fused(torch.from_numpy(keys).cuda(), cfg.num_digits, 8)
            torch.cuda.synchronize()
            assert np.array_equal(local.cpu().numpy(), O.sort(keys, cfg.num_digits, 8)), name
            assert info.send_counts == [keys.size]
    finally:
        dist.destroy_process_group()
