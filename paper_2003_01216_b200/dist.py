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

The exchange runs through the collectives of the process group, NCCL on
GPUs.  The per-rank steps 1 and 5 are injected as ``ops`` so the host logic
can be tested on CPU with the gloo backend (tests/test_dist.py passes
oracle-based ops there); the default ops are the CUDA path and there is no
CPU fallback in it.
"""
from __future__ import annotations

from dataclasses import dataclass

from . import assign_buckets, hs_msd_partition, hs_sort


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
