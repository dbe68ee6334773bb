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


def scan_work(scans: torch.Tensor) -> float:
    """Work estimate of a batch of scans for shard_submaps (rays x mean range): the
    integration cost is the voxel updates, ~ sum over valid rays of the ray length.  scans: [F, N, 3]
    sensor-frame points (NaN = no return).  Input statistics only."""
    r = torch.linalg.vector_norm(scans.double(), dim=-1)
    return float(torch.nan_to_num(r, nan=0.0).sum())


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


def gather_esdfs(payloads, max_per_rank: int, group=None):
    """All-gather the packed ESDFs (cvx_pack_esdf payloads, one uint8 tensor per local submap) of every
    rank into one buffer for cvx_esdf_set_create.  Every rank knows max_per_rank from the
    shard assignment.  One small all_gather of the per-submap sizes (one host read of a (world, 1 + S)
    int64 tensor), then ONE padded all_gather_into_tensor over NCCL (list all_gather on gloo).  Returns
    (buffer, offsets, per_rank_counts): payload j of rank r sits at offsets[sum(counts[:r]) + j]."""
    world = dist.get_world_size(group)
    dev = payloads[0].device if payloads else torch.device("cuda", torch.cuda.current_device())
    S = int(max_per_rank)
    if len(payloads) > S:
        raise ValueError("more local payloads than max_per_rank")
    meta = torch.zeros(1 + S, dtype=torch.int64, device=dev)
    meta[0] = len(payloads)
    if payloads:
        meta[1:1 + len(payloads)] = torch.tensor([p.numel() for p in payloads], dtype=torch.int64)
    metas = [torch.empty_like(meta) for _ in range(world)]
    dist.all_gather(metas, meta, group=group)
    table = torch.stack(metas).cpu().tolist()                  # the one host synchronisation
    totals = [sum(row[1:1 + row[0]]) for row in table]
    mx = max(max(totals), 16)
    blob = torch.zeros(mx, dtype=torch.uint8, device=dev)
    if payloads:
        blob[:totals[dist.get_rank(group)]] = torch.cat(payloads)
    if dist.get_backend(group) == "nccl":
        out = torch.empty(world * mx, dtype=torch.uint8, device=dev)
        dist.all_gather_into_tensor(out, blob, group=group)
    else:
        outs = [torch.empty(mx, dtype=torch.uint8, device=dev) for _ in range(world)]
        dist.all_gather(outs, blob, group=group)
        out = torch.cat(outs)
    offsets, counts = [], []
    for r, row in enumerate(table):
        o = r * mx
        counts.append(row[0])
        for j in range(row[0]):
            offsets.append(o)
            o += row[1 + j]
    return out, offsets, counts
