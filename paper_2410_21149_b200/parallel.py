"""Host-side multi-GPU plumbing of the submap builder.

Submaps are independent units, so ranks build whole submaps with no collective on the
data path; the only exchange is the gather of finished, packed ESDF blocks (cvx_pack_esdf payloads) for
downstream registration / queries.  Nothing here computes any step of the method.
"""
from __future__ import annotations

import heapq

import torch
import torch.distributed as dist


def shard_submaps(work, world: int):
    """Longest-processing-time-first assignment of submaps to ranks.

    work: per-submap cost estimates (e.g. rays x mean range).  Returns one list of submap indices per
    rank; ties go to the lower rank, so the assignment is deterministic.
    """
    if world < 1:
        raise ValueError("world must be >= 1")
    heap = [(0.0, r) for r in range(world)]
    out = [[] for _ in range(world)]
    for i in sorted(range(len(work)), key=lambda i: (-float(work[i]), i)):
        load, r = heapq.heappop(heap)
        out[r].append(i)
        heapq.heappush(heap, (load + float(work[i]), r))
    return [sorted(x) for x in out]


def gather_packed(payload: torch.Tensor, group=None):
    """All-gather variable-size uint8 payloads (one per rank); returns the list of payloads.

    Sizes are all-gathered first, then one padded all_gather_into_tensor (NCCL: a single collective over
    NVLink / NVSwitch); with gloo (CPU tests) a list all_gather is used.
    """
    world = dist.get_world_size(group)
    dev = payload.device
    n = torch.tensor([payload.numel()], dtype=torch.int64, device=dev)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    mx = max(sizes)
    buf = torch.zeros(mx, dtype=torch.uint8, device=dev)
    buf[:payload.numel()] = payload
    if dist.get_backend(group) == "nccl":
        out = torch.empty(world * mx, dtype=torch.uint8, device=dev)
        dist.all_gather_into_tensor(out, buf, group=group)
        parts = [out[r * mx:r * mx + sizes[r]] for r in range(world)]
    else:
        outs = [torch.empty(mx, dtype=torch.uint8, device=dev) for _ in range(world)]
        dist.all_gather(outs, buf, group=group)
        parts = [outs[r][:sizes[r]] for r in range(world)]
    return parts
