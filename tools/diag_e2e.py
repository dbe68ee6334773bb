"""Where the end-to-end (host-buffer) bench step loses time against the device-resident one (configs[1])."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2410_21149_b200 as cvx  # noqa: E402

dev = torch.device("cuda", 0)
cfg, data, poses = bench.make_workload(0, dev)
sensor = cfg["sensor"]
N = data.shape[0]
B = int(os.environ.get("BATCH", "200"))
host = data.cpu().pin_memory()
q = torch.rand((1 << 20, 3), device=dev) * 50
hq = q.cpu().pin_memory()
builders = [cvx.Submap(cfg["grid"], cfg["submaps"][0]["T_world_submap"], 0) for _ in range(2)]
streams = [torch.cuda.current_stream(), torch.cuda.Stream(dev)]
outs = [(torch.empty(1 << 20, device=dev), torch.empty(1 << 20, dtype=torch.uint8, device=dev)) for _ in range(2)]
houts = [(torch.empty(1 << 20).pin_memory(), torch.empty(1 << 20, dtype=torch.uint8).pin_memory()) for _ in range(2)]
dq = [torch.empty_like(q) for _ in range(2)]


def step(i, host_frames, queries_host, pipelined=True):
    k = i % 2 if pipelined else 0
    m = builders[k]
    with torch.cuda.stream(streams[k]):
        if queries_host:
            dq[k].copy_(hq, non_blocking=True)
        m.reset()
        for c in range(0, N, B):
            if host_frames:
                m.integrate_batch_host(host[c:c + B], poses[c:c + B], sensor)
            else:
                m.integrate_batch(data[c:c + B], poses[c:c + B], sensor)
        m.finalize_esdf()
        m.query(dq[k] if queries_host else q, *outs[k])
        if queries_host:
            houts[k][0].copy_(outs[k][0], non_blocking=True)
            houts[k][1].copy_(outs[k][1], non_blocking=True)


def timed(fn, n=10):
    for i in range(3):
        fn(i)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(streams[0])
    streams[1].wait_stream(streams[0])
    for i in range(n):
        fn(i)
    streams[0].wait_stream(streams[1])
    b.record(streams[0])
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


print("device pipelined      ", timed(lambda i: step(i, False, False)))
print("host frames+queries   ", timed(lambda i: step(i, True, True)))
print("host frames only      ", timed(lambda i: step(i, True, False)))
print("host queries only     ", timed(lambda i: step(i, False, True)))
print("host frames, 1 in flt ", timed(lambda i: step(i, True, True, pipelined=False)))
print("device, 1 in flight   ", timed(lambda i: step(i, False, False, pipelined=False)))
x = torch.empty_like(data)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5):
    x.copy_(host, non_blocking=True)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / 5
print(f"H2D of the scans alone  {ms:.3f} ms  ({data.numel() * 4 / ms / 1e6:.1f} GB/s)")
