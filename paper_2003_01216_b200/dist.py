"""Multi-GPU bucket sharding: the paper's cluster model on N GPUs.

PAPER.md §3.4 (Fig 4): "The master node divides the data into ten
parts based on the most significant digit ... Then sends each bucket or
buckets to proper node ... the Shared-Parallel Hybrid Quicksort and Merge Sort
is executed by parallel threads in a node, the sorted data is then sent to the
master node to its place in the original array."  Buckets are range-disjoint,
so no node ever merges with another ("eliminate all internal data
transfers between different nodes").

B200 shape (one process per GPU, torch.distributed over NCCL; every rank
already holds its shard of the keys, i.e. weak scaling -- there is no master
scatter):

  1. local one-step MSD partition (hs_msd_partition): keys grouped by leading
     digit, bucket_offsets[11];
  2. all_gather of the ten local bucket sizes (the only metadata exchange);
  3. assign_buckets (hs_assign_buckets): contiguous digit groups,
     group g -> rank g, minimising the largest group;
  4. one all-to-all-v (all_to_all_single with split sizes) moves every
     rank's segment of group g -- a contiguous slice of its partitioned keys --
     to rank g: the paper's "sends each bucket or buckets to proper node",
     done by all ranks at once over NVLink/NVSwitch;
  5. every rank sorts what it received with hs_sort (its keys all carry the
     leading digits of its group, so its result is one contiguous, range-
     disjoint piece of the global order).

The global result is the concatenation of the ranks' outputs in rank order
(``gather_to`` assembles it on one rank, the paper's final gather).  With
more than 10 ranks the extra ranks own no digit (at most ten nodes).

``dist_sort`` runs the exchange through the collectives of the process group
(NCCL on GPUs).  ``dist_sort_fused`` fuses it into the scatter instead: each
rank's K3 stores every digit's keys straight into the owner rank's
symmetric-memory receive buffer over NVLink (hs_partition_scatter with peer
destination pointers), so step 4 costs no collective call and no staging copy,
and the owner's buffer arrives already partitioned by digit (step 5 is then
hs_sort_buckets: chunk sort + tree merge, no second MSD pass).

In ``dist_sort`` the per-rank steps 1 and 5 are injected as ``ops`` so the host logic
can be tested on CPU with the gloo backend (tests/test_dist.py passes
oracle-based ops there); the default ops are the CUDA path and there is no
CPU fallback in it.
"""
from __future__ import annotations

from dataclasses import dataclass

from . import PartitionPlan, assign_buckets, hs_msd_partition, hs_sort, hs_sort_buckets


@dataclass
class DistInfo:
    group_start: list      # digits of rank g: [group_start[g], group_start[g+1])
    global_sizes: list     # ten global bucket sizes
    send_counts: list      # keys this rank sent to each rank
    recv_counts: list      # keys this rank received from each rank
    max_load: int          # largest group total (the load-balance bound)


class CudaOps:
    """The product per-rank steps: hs_msd_partition and hs_sort (CUDA only)."""

    @staticmethod
    def partition(keys, num_digits):
        return hs_msd_partition(keys, num_digits)

    @staticmethod
    def sort(keys, num_digits, chunks):
        return hs_sort(keys, num_digits, chunks)


def dist_sort(keys, num_digits: int, chunks: int = 8, group=None, ops=CudaOps):
    """Sort the union of every rank's ``keys`` across the process group.

    Returns (local_sorted, info): this rank's contiguous piece of the global
    ascending order (possibly empty) and the exchange bookkeeping.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    part, off = ops.partition(keys, num_digits)
    off = off.to(torch.int64)
    local_sizes = (off[1:] - off[:-1]).contiguous()
    gathered = [torch.empty_like(local_sizes) for _ in range(world)]
    dist.all_gather(gathered, local_sizes, group=group)
    sizes = torch.stack(gathered).cpu()                       # [world, 10]
    global_sizes = sizes.sum(0).tolist()
    nodes = min(world, 10)
    group_start, max_load = assign_buckets(global_sizes, nodes)
    group_start = group_start + [10] * (world - nodes)        # ranks >= 10 own nothing

    def seg(src_sizes, g):                                     # keys of group g in a rank's partition
        return int(src_sizes[group_start[g]:group_start[g + 1]].sum())

    send = [seg(sizes[rank], g) for g in range(world)]
    recv = [seg(sizes[r], rank) for r in range(world)]
    out = torch.empty(sum(recv), dtype=keys.dtype, device=keys.device)
    dist.all_to_all_single(out, part, output_split_sizes=recv, input_split_sizes=send, group=group)
    if out.numel():
        ops.sort(out, num_digits, chunks)
    return out, DistInfo(group_start, global_sizes, send, recv, max_load)


def gather_to(local_sorted, dst: int = 0, group=None):
    """The paper's final gather: concatenate every rank's piece on rank ``dst``."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    n = torch.tensor([local_sorted.numel()], dtype=torch.int64, device=local_sorted.device)
    counts = [torch.empty_like(n) for _ in range(world)]
    dist.all_gather(counts, n, group=group)
    counts = [int(c.item()) for c in counts]
    rank = dist.get_rank(group)
    recv = counts if rank == dst else [0] * world
    send = [local_sorted.numel() if r == dst else 0 for r in range(world)]
    out = torch.empty(sum(recv), dtype=local_sorted.dtype, device=local_sorted.device)
    dist.all_to_all_single(out, local_sorted, output_split_sizes=recv, input_split_sizes=send, group=group)
    return out if rank == dst else None


# ----------------------------------------------------------------- fused exchange
def exchange_layout(sizes, group_start):
    """Where every (source rank, digit) segment lands in its owner's receive buffer.

    sizes[r][d]: keys of digit d on rank r.  Owner g's buffer holds its digits
    in ascending order, each digit's segments in source-rank order -- i.e. it
    is already partitioned by digit, ready for the per-bucket chunk sort and
    tree merge.  Returns (owner[d], offset[r][d], recv_offsets[g] (11 entries),
    recv_total[g]).  Pure host logic (tests/test_dist.py checks it on CPU).
    """
    world = len(sizes)
    total = [sum(sizes[r][d] for r in range(world)) for d in range(10)]
    owner = [0] * 10
    for g in range(len(group_start) - 1):
        for d in range(group_start[g], group_start[g + 1]):
            owner[d] = g
    offset = [[0] * 10 for _ in range(world)]
    recv_offsets, recv_total = [], []
    for g in range(world):
        off = [0] * 11
        pos = 0
        for d in range(10):
            if g < len(group_start) - 1 and owner[d] == g:
                for r in range(world):
                    offset[r][d] = pos + sum(sizes[rr][d] for rr in range(r))
                pos += total[d]
            off[d + 1] = pos
        recv_offsets.append(off)
        recv_total.append(pos)
    return owner, offset, recv_offsets, recv_total


class _SymmBuffer:
    """Cached symmetric-memory receive buffers, one per (dtype, device, process
    group); a buffer is re-made only when it must grow.  The buffer is the
    library's: dist_sort_fused hands the caller a copy, never a view of it."""

    def __init__(self):
        self.entries = {}

    def get(self, numel, dtype, device, group):
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem
        pg = group if group is not None else dist.group.WORLD
        key = (dtype, str(device), id(pg))
        ent = self.entries.get(key)
        if ent is None or ent[0].numel() < numel:
            buf = symm_mem.empty(max(numel, 1), dtype=dtype, device=device)
            ent = (buf, symm_mem.rendezvous(buf, pg), pg)  # pg kept alive with its handle
            self.entries[key] = ent
        return ent[0], ent[1]


_SYMM = _SymmBuffer()


def dist_sort_fused(keys, num_digits: int, chunks: int = 8, group=None):
    """dist_sort with the bucket exchange fused into the scatter kernel.

    Every rank's K3 writes each digit's keys straight into the owner rank's
    symmetric-memory receive buffer over NVLink (peer stores from the kernel,
    hs_partition_scatter) -- no all-to-all call and no staging copy; then every
    owner chunk-sorts and tree-merges its received buckets in place.  Returns
    (local_sorted, DistInfo); local_sorted is a tensor the caller owns (a copy
    out of the cached receive buffer, which the next call overwrites).  CUDA +
    NCCL process group only.

    Cross-GPU ordering: (1) handle.barrier() before the scatter
    -- no rank's K3 stores into an owner's buffer until every rank has finished
    with the previous call's contents; (2) K3 ends with a system-scope fence
    (__threadfence_system) after its last peer store, and the host waits for
    the K3 grid to complete (stream synchronize); (3) handle.barrier() after it
    -- a release/acquire signal exchange among all ranks, so when an owner
    passes it every rank's stores into its buffer have completed and are
    visible; only then does the owner's hs_sort_buckets read the buffer.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    plan = PartitionPlan(keys, num_digits)
    off = plan.offsets
    local_sizes = (off[1:] - off[:-1]).contiguous()
    gathered = [torch.empty_like(local_sizes) for _ in range(world)]
    dist.all_gather(gathered, local_sizes, group=group)
    sizes = torch.stack(gathered).cpu().tolist()
    global_sizes = [sum(sizes[r][d] for r in range(world)) for d in range(10)]
    nodes = min(world, 10)
    group_start, max_load = assign_buckets(global_sizes, nodes)
    owner, offset, recv_offsets, recv_total = exchange_layout(sizes, group_start)
    buf, handle = _SYMM.get(max(recv_total), keys.dtype, keys.device, group)
    handle.barrier()  # every owner's buffer is free (previous call finished reading it)
    esz = keys.element_size()
    dst = []
    for d in range(10):
        if sizes[rank][d] == 0:
            dst.append(0)
            continue
        peer = handle.get_buffer(owner[d], (buf.numel(),), keys.dtype)
        dst.append(peer.data_ptr() + offset[rank][d] * esz)
    plan.scatter(dst)
    torch.cuda.current_stream().synchronize()
    plan.close()
    handle.barrier()  # every rank's stores into this rank's buffer have landed
    n_local = recv_total[rank] if rank < len(recv_total) else 0
    local = buf[:n_local]
    if n_local:
        roff = torch.tensor(recv_offsets[rank], dtype=torch.int64, device=keys.device)
        hs_sort_buckets(local, roff, num_digits, chunks)  # chunk sort (+ value split) + tree merge, in place
    local = local.clone()  # owned by the caller: the receive buffer is reused by the next call
    send = [sum(sizes[rank][d] for d in range(10) if owner[d] == g) for g in range(world)]
    recv = [sum(sizes[r][d] for d in range(10) if owner[d] == rank) for r in range(world)]
    return local, DistInfo(group_start, global_sizes, send, recv, max_load)
