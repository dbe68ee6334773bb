#!/usr/bin/env python
"""bench.py — submap build throughput of the B200-native coVoxSLAM path (BASELINE.json metric).

One step = one whole submap build per rank, all §8(a) rows: reset -> integrate 200 OS1-64-shaped
LiDAR scans (a1-a5) -> finalize_esdf (a6) -> 1 M distance queries (a7) -> (N > 1) all-gather of the
packed ESDF blocks over NCCL (§8e).  Inputs are synthetic (BASELINE.json configs[1]) and resident
in HBM before timing; the scans alone (157 MB) exceed the 126 MB L2.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl cvx|reference]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N

Prints ONE JSON line on rank 0.  `--impl reference` times the CPU oracle (oracle/, the reference of
this tier) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

METRIC = "scans/s TSDF fusion + ESDF Mvoxels/s per submap; HBM GB/s vs peak; 1/2/4/8 GPU"
N_SCANS = 200
FALLBACK_HBM_GBS = 6650.0     # /opt/skills/guides/B200_PROFILING.md fallback (no MEASURED_PEAKS.json)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        try:
            d = json.load(open(p))
            return float(d.get("hbm_gbs", FALLBACK_HBM_GBS)), "measured", d
        except Exception:
            pass
    return FALLBACK_HBM_GBS, "fallback", {}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 20 ms during the timed region.  __enter__ returns
    only once nvidia-smi has printed its first sample (that one, taken before the region, is not counted),
    so a short timed region is still covered; a reader thread collects the samples."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.active", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self.out = ""

    def __enter__(self):
        import threading
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return self
        first = threading.Event()

        def reader():
            for k, line in enumerate(self.proc.stdout):
                if k == 0:
                    first.set()          # taken before the timed region: not counted
                    continue
                self.lines.append(line)
            first.set()

        self.thread = threading.Thread(target=reader, daemon=True)
        self.thread.start()
        first.wait(timeout=10)
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.thread.join(timeout=5)
        self.out = "".join(self.lines)

    def summary(self):
        rows = [r.split(",") for r in (getattr(self, "out", "") or "").strip().splitlines() if r.strip()]
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            r = [x.strip() for x in r]
            try:
                sm.append(float(r[0])); mx.append(float(r[1]))
            except Exception:
                continue
            for nm, v in zip(names, r[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("CVX_BENCH_ONE_GPU") == "1":
        local = 0        # test knob: every rank on cuda:0 (exercises the N > 1 code path on a 1-GPU box)
    return world, rank, local


def init_pg(dev):
    """NCCL process group (one rank per GPU); CVX_BENCH_BACKEND=gloo is the 1-GPU test knob (NCCL refuses
    two ranks on one device)."""
    import torch.distributed as dist
    backend = os.environ.get("CVX_BENCH_BACKEND", "nccl")
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group(backend)


def esdf_alg_bytes(va: int, n: int) -> dict:
    """Algorithmic HBM bytes per launch of the ESDF passes: va allocated voxels, n dense AABB
    voxels.  pass x: the 16-byte sums of every allocated voxel + 2-byte 1-D distances + 3 bit-planes
    (3/8 byte per allocated voxel); pass y: 2-byte in + 4-byte out per dense voxel; pass z: 4-byte in per
    dense voxel + 4-byte E out + 2 bit-planes per allocated voxel."""
    return {"esdf_pass_x": int(16 * va + 2 * n + 3 * va // 8),
            "esdf_pass_y": int(6 * n),
            "esdf_pass_z": int(4 * n + 4 * va + va // 4)}


def make_workload(rank: int, device: torch.device):
    import synth
    # weak scaling: every rank builds the configs[1] submap (same seed, so identical per-rank work and the
    # max over ranks measures scaling, not scene imbalance)
    cfg = synth.make_config("lidar", device=device)
    data = torch.stack([cfg["frames"][k]["data"] for k in range(N_SCANS)]).contiguous()
    poses = np.stack([cfg["frames"][k]["T_world_sensor"] for k in range(N_SCANS)])
    return cfg, data, poses


# ------------------------------------------------------------------------------------ reference arm
def run_reference(args, world, rank):
    if rank != 0:
        return
    import oracle
    import synth
    dev = torch.device("cuda", 0) if torch.cuda.is_available() else torch.device("cpu")
    cfg = synth.make_config("lidar", frames=list(range(0, N_SCANS, 20)), device=dev)
    keys = sorted(cfg["frames"])
    frames = {k: cfg["frames"][k]["data"].cpu().numpy() for k in keys}
    g = cfg["grid"]
    per_step = 2

    def step(i):
        o = oracle.OracleSubmap(g, cfg["submaps"][0]["T_world_submap"])
        t0 = time.perf_counter()
        for j in range(per_step):
            k = keys[(i * per_step + j) % len(keys)]
            o.integrate(frames[k], cfg["frames"][k]["T_world_sensor"], cfg["sensor"])
        t1 = time.perf_counter()
        b, D, W = o.export()
        oracle.esdf(b, D, W, g["voxel_size"], g["site_threshold"])
        t2 = time.perf_counter()
        return t1 - t0, t2 - t1, int((W > 0).sum()), b.shape[0]

    for i in range(args.warmup):
        step(i)
    times = [step(args.warmup + i) for i in range(args.steps)]
    tot = sum(a + b for a, b, _, _ in times)
    ms = 1000 * tot / args.steps
    value = per_step * args.steps / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "scans/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "lidar_submap_os1_64x1024_200scans_0.2m (BJ configs[1])",
                   "sample": f"{per_step} scans + ESDF of their submap per step"},
        "cpu_baseline": {"value": value, "unit": "scans/s", "cores": 1, "kind": "oracle",
                         "sample": f"{per_step} of 200 scans per step (fresh submap) + exact ESDF of that submap",
                         "integrate_scans_per_s": per_step * args.steps / sum(a for a, _, _, _ in times),
                         "esdf_mvox_per_s": sum(n * 512 for _, _, _, n in times) / 1e6 / sum(b for _, b, _, _ in times)},
        "e2e": {"value": value, "unit": "scans/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_sample(cfg, data, poses, n=20):
    """The oracle as it stands, single-threaded, on the first n scans of the same workload."""
    import oracle
    g = cfg["grid"]
    o = oracle.OracleSubmap(g, cfg["submaps"][0]["T_world_submap"])
    t0 = time.perf_counter()
    for k in range(n):
        o.integrate(data[k].cpu().numpy(), poses[k], cfg["sensor"])
    t1 = time.perf_counter()
    b, D, W = o.export()
    oracle.esdf(b, D, W, g["voxel_size"], g["site_threshold"])
    t2 = time.perf_counter()
    return {"value": n / (t2 - t0), "unit": "scans/s", "cores": 1, "kind": "oracle",
            "sample": f"first {n} of 200 scans integrated + exact ESDF of that {b.shape[0]}-block submap",
            "integrate_scans_per_s": n / (t1 - t0), "esdf_mvox_per_s": b.shape[0] * 512 / 1e6 / (t2 - t1),
            "seconds": t2 - t0}


NCU_FILES = {"ray_walk_update": "ncu_walk.txt", "block_walk_allocate": "ncu_block_walk.txt",
             "dense_fold_allocate": "ncu_dense_fold.txt",
             "ray_prepare": "ncu_prepare.txt", "esdf_pass_x": "ncu_esdf_pass_x.txt",
             "esdf_pass_y": "ncu_esdf_pass_y.txt", "esdf_pass_z": "ncu_esdf_pass_z.txt", "fold": "ncu_fold.txt"}


def ncu_metric(kernel, name, workload="lidar"):
    """A '<name>  <unit>  <value>' line (e.g. Issue Slots Busy, %) of the newest committed ncu summary of
    `kernel` under profiles/, as {"value", "unit", "source"} (None if there is none)."""
    prof = os.path.join(ROOT, "profiles")
    if kernel not in NCU_FILES or not os.path.isdir(prof):
        return None
    fname = NCU_FILES[kernel]
    if workload == "esdf_stress":
        fname = fname.replace("ncu_esdf_", "ncu_stress_")
    for tag in sorted(os.listdir(prof), reverse=True):
        f = os.path.join(prof, tag, fname)
        if not os.path.exists(f):
            continue
        for line in open(f):
            if line.startswith(name):
                parts = line[len(name):].split()
                try:
                    return {"value": float(parts[-1]), "unit": parts[0] if len(parts) > 1 else "",
                            "source": f"profiles/{tag}/{fname}"}
                except ValueError:
                    return None
        return None
    return None


def l2_red_view(kernel):
    """The walk's per-voxel reductions against the MEASURED L2 reduction ceiling: RED sectors
    per second of the newest ncu capture (lts__t_sectors_srcunit_tex_op_red.sum / gpu__time_duration.sum)
    vs microbench/l2_atomics.cu's scattered and lane-coherent 64-bit RED rates (profiles/*/l2_atomics.json,
    32 MB footprint, i.e. L2-resident like the accumulators of the hot blocks)."""
    sec = ncu_metric(kernel, "lts__t_sectors_srcunit_tex_op_red.sum")
    dur = ncu_metric(kernel, "gpu__time_duration.sum")
    prof = os.path.join(ROOT, "profiles")
    ceil = None
    for tag in sorted(os.listdir(prof), reverse=True) if os.path.isdir(prof) else []:
        f = os.path.join(prof, tag, "l2_atomics.json")
        if os.path.exists(f):
            d = json.load(open(f)).get("32MB", {})
            ceil = {"scattered_Gops": d.get("red64_Gops"), "coherent_Gops": d.get("red64_coherent_Gops"),
                    "source": f"profiles/{tag}/l2_atomics.json"}
            break
    if not sec or not dur or not dur["value"]:
        return None
    scale = {"ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1.0, "msecond": 1e-3, "usecond": 1e-6}.get(dur["unit"], 1e-3)
    ach = sec["value"] / (dur["value"] * scale) / 1e9
    out = {"achieved_Gsectors_per_s": ach, "source": sec["source"]}
    if ceil and ceil["scattered_Gops"]:
        out.update({"ceiling": ceil, "frac_of_scattered": ach / ceil["scattered_Gops"],
                    "frac_of_coherent": ach / ceil["coherent_Gops"] if ceil["coherent_Gops"] else None})
    return out


def ncu_traffic(kernel, workload="lidar"):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` from the newest committed
    `ncu --set full` capture of that workload under profiles/ (None if there is none)."""
    prof = os.path.join(ROOT, "profiles")
    if kernel not in NCU_FILES or not os.path.isdir(prof):
        return None
    name = NCU_FILES[kernel]
    if workload == "esdf_stress":
        name = name.replace("ncu_esdf_", "ncu_stress_")
    for tag in sorted(os.listdir(prof), reverse=True):
        f = os.path.join(prof, tag, name)
        if not os.path.exists(f):
            continue
        tot = 0.0
        for line in open(f):
            parts = line.split()
            if parts and parts[0] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(parts[1], 1)
                tot += float(parts[2]) * scale
        return {"bytes_per_launch": tot, "source": f"profiles/{tag}/{name}"}
    return None


def run_mav(args, world, rank, local):
    """BASELINE.json configs[3]: a ~400 m MAV flight (2000 OS1-64 scans) cut into 40 submaps of 50
    contiguous scans, sharded over the ranks by longest-processing-time on the rays per submap (strong
    scaling: the whole flight is the fixed job).  Each rank builds its submaps (integrate -> exact ESDF
    -> pack); the packed ESDFs of all ranks are then all-gathered (NCCL when N > 1)."""
    import paper_2410_21149_b200 as cvx
    import synth
    from paper_2410_21149_b200.parallel import gather_esdfs, shard_submaps
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        init_pg(dev)
        pg = dist
    cfg = synth.make_config("mav", frames=[], device=dev)
    subs = cfg["submaps"]
    # work estimate per submap (rays x mean range), identical on every rank: sum of the ray
    # lengths of every 10th scan of the submap, times 10 (input statistics from the seeded generator)
    from paper_2410_21149_b200.parallel import scan_work
    sample = sorted(k for sm_ in subs for k in sm_["frames"][::10])
    cfs = synth.make_config("mav", frames=sample, device=dev)
    work = [10.0 * scan_work(torch.stack([cfs["frames"][k]["data"] for k in sm_["frames"][::10]])) for sm_ in subs]
    del cfs
    assign = shard_submaps(work, world)
    mine = assign[rank]
    frames = sorted(k for i in mine for k in subs[i]["frames"])
    cfgf = synth.make_config("mav", frames=frames, device=dev)
    data = {i: torch.stack([cfgf["frames"][k]["data"] for k in subs[i]["frames"]]).contiguous() for i in mine}
    poses = {i: np.stack([cfgf["frames"][k]["T_world_sensor"] for k in subs[i]["frames"]]) for i in mine}
    grid = cfg["grid"]
    # two builders on two streams: the exact ESDF of submap j overlaps the integration of submap j+1
    # (the packed result of submap j is taken after submap j+1's integration has been enqueued)
    builders = [cvx.Submap(grid, subs[i]["T_world_submap"], local) for i in mine[:2]]
    stream = torch.cuda.current_stream(dev)
    streams = [stream, torch.cuda.Stream(dev)]

    gathered = [0]
    gq = torch.Generator(device=dev).manual_seed(11)
    set_pts = (torch.rand((1 << 16, 3), device=dev, generator=gq) * torch.tensor([200.0, 120.0, 10.0], device=dev)
               - torch.tensor([100.0, 60.0, 0.0], device=dev)).contiguous()
    set_idx = torch.randint(0, len(subs), (1 << 16,), device=dev, generator=gq, dtype=torch.int32)

    def step():
        payloads = []
        pending = None

        def take(k):
            with torch.cuda.stream(streams[k]):
                payloads.append(builders[k].pack().clone())

        for j, i in enumerate(mine):
            k = j % 2
            with torch.cuda.stream(streams[k]):
                builders[k].reset(subs[i]["T_world_submap"])
                builders[k].integrate_batch(data[i], poses[i], cfg["sensor"])
                builders[k].finalize_esdf()
            if pending is not None:
                take(pending)
            pending = k
        if pending is not None:
            take(pending)
        stream.wait_stream(streams[1])
        if pg is not None:   # every rank gets every submap's ESDF and indexes them for registration look-ups
            buf, offsets, _ = gather_esdfs(payloads, max_per_rank=max(len(a) for a in assign))
            gathered[0] = int(buf.numel())
            es = cvx.EsdfSet(buf, offsets)
            es.query(set_idx, set_pts)
            es.close()
        return payloads

    for _ in range(args.warmup):
        step()
    if pg is not None:
        pg.barrier()
    torch.cuda.synchronize()
    mav_prof = os.environ.get("CVX_BENCH_MAV_PROFILE", "0") == "1"   # per-kernel events perturb the pipeline
    for b_ in builders:
        b_.profile(mav_prof)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        streams[1].wait_stream(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    kms = {}
    for b_ in builders:
        if mav_prof:
            for k_, v_ in b_.profile_report().items():
                kms[k_] = kms.get(k_, 0.0) + v_["ms"] / args.steps
        b_.profile(False)
    if pg is not None:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        ms = float(t.item())
    n_scans = sum(len(sm_["frames"]) for sm_ in subs)
    line = {"metric": METRIC, "value": n_scans / (ms / 1e3), "unit": "scans/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32+i64", "data": "synthetic",
            "config": {"workload": "mav_400m_flight_2000scans_40submaps_0.2m (BJ configs[3])",
                       "submaps": len(subs), "submaps_per_rank_max": max(len(x) for x in assign),
                       "lpt_work": "sum of ray lengths of every 10th scan x 10 (rays x mean range, SURVEY §8e)",
                       "work_imbalance": max(sum(work[i] for i in a) for a in assign) / (sum(work) / world),
                       "parallelism": f"submap-sharded x{world} (LPT)",
                       "pipeline": "2 submaps in flight (ESDF of submap j overlaps integration of submap j+1)"},
            "clocks": clk.summary()}
    line["kernel_ms_per_step"] = kms
    if world > 1:
        line["gather_bytes_per_step"] = gathered[0]
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = mav_cpu_baseline(cfgf, subs[mine[0]], n=8)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if pg is not None:
        pg.barrier()
        pg.destroy_process_group()


def mav_cpu_baseline(cfg, sub, n=8):
    """The oracle as it stands, single-threaded, on the first n scans of submap 0 of configs[3] + the
    exact ESDF of that partial submap."""
    import oracle
    g = cfg["grid"]
    o = oracle.OracleSubmap(g, sub["T_world_submap"])
    t0 = time.perf_counter()
    for k in sub["frames"][:n]:
        o.integrate(cfg["frames"][k]["data"].cpu().numpy(), cfg["frames"][k]["T_world_sensor"], cfg["sensor"])
    t1 = time.perf_counter()
    b, D, W = o.export()
    oracle.esdf(b, D, W, g["voxel_size"], g["site_threshold"])
    t2 = time.perf_counter()
    return {"value": n / (t2 - t0), "unit": "scans/s", "cores": 1, "kind": "oracle",
            "sample": f"first {n} of the 50 scans of submap 0 integrated + exact ESDF of that {b.shape[0]}-block "
                      "partial submap", "integrate_scans_per_s": n / (t1 - t0), "seconds": t2 - t0}


def run_color(args, world, rank, local):
    """TSDF + Color: the configs[1] submap build with per-point colour fused in the
    band, timed beside the same build without colour (weak scaling: every rank builds its own submap)."""
    import paper_2410_21149_b200 as cvx
    import synth
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        init_pg(dev)
        pg = dist
    cfg = synth.make_config("lidar", device=dev, seed=1 + 1000 * rank, color=True)
    data = torch.stack([cfg["frames"][k]["data"] for k in range(N_SCANS)]).contiguous()
    rgb = torch.stack([cfg["frames"][k]["rgb"] for k in range(N_SCANS)]).contiguous()
    poses = np.stack([cfg["frames"][k]["T_world_sensor"] for k in range(N_SCANS)])
    T_sub = cfg["submaps"][0]["T_world_submap"]
    stream = torch.cuda.current_stream(dev)
    res = {}
    for mode in ("plain", "color"):
        sm = cvx.Submap(dict(cfg["grid"], color=1 if mode == "color" else 0), T_sub, local)

        def step():
            sm.reset()
            for c in range(0, N_SCANS, args.batch):
                if mode == "color":
                    sm.integrate_color(data[c:c + args.batch], rgb[c:c + args.batch], poses[c:c + args.batch], cfg["sensor"])
                else:
                    sm.integrate_batch(data[c:c + args.batch], poses[c:c + args.batch], cfg["sensor"])
            sm.finalize_esdf()

        for _ in range(args.warmup):
            step()
        if pg is not None:
            pg.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(local) as clk:
            e0.record(stream)
            for _ in range(args.steps):
                step()
            e1.record(stream)
            torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        if pg is not None:
            t = torch.tensor([ms], device=dev, dtype=torch.float64)
            pg.all_reduce(t, op=pg.ReduceOp.MAX)
            ms = float(t.item())
        res[mode] = (ms, clk.summary())
        del sm
    ms, clk = res["color"]
    line = {"metric": METRIC, "value": world * N_SCANS / (ms / 1e3), "unit": "scans/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32+i64", "data": "synthetic",
            "config": {"workload": "lidar_submap_os1_64x1024_200scans_0.2m_color (BJ configs[1] + TSDF+Color)",
                       "scans_per_rank": N_SCANS, "batch_scans": args.batch,
                       "parallelism": f"submap-sharded x{world}"},
            "plain_ms_per_step": res["plain"][0], "color_overhead": ms / res["plain"][0] - 1.0,
            "clocks": clk}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if pg is not None:
        pg.barrier()
        pg.destroy_process_group()


def run_incremental(args, world, rank, local, every=10):
    """configs[1] integrated in batches of `every` scans with an incremental ESDF update
    after each batch (the paper's per-frame ESDF maintenance; the exact EDT clamped at
    esdf_max_distance = 2 m, R11), against one exact finalize_esdf of the same submap per batch."""
    import paper_2410_21149_b200 as cvx
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cfg, data, poses = make_workload(rank, dev)
    sm = cvx.Submap(cfg["grid"], cfg["submaps"][0]["T_world_submap"], local)
    stream = torch.cuda.current_stream(dev)

    def run(mode):
        sm.reset()
        t_upd, queued = 0.0, 0
        for c in range(0, N_SCANS, every):
            sm.integrate_batch(data[c:c + every], poses[c:c + every], cfg["sensor"])
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            if mode == "inc":
                queued += sm.update_esdf()
            else:
                sm.finalize_esdf()
            e1.record(stream)
            torch.cuda.synchronize()
            t_upd += e0.elapsed_time(e1)
            if mode == "full":
                sm.reset()                      # finalize freezes the submap: rebuild up to this batch
                sm.integrate_batch(data[:c + every].contiguous(), poses[:c + every], cfg["sensor"])
        return t_upd, queued

    for _ in range(max(1, args.warmup)):
        run("inc")
    sm.profile(True)
    t_inc, queued = run("inc")
    prof = {k: v for k, v in sm.profile_report().items() if k.startswith("inc_")}
    sm.profile(False)
    sm.reset()                                  # warm the grow-only EDT scratch at the final AABB size
    sm.integrate_batch(data, poses, cfg["sensor"])
    sm.finalize_esdf()
    t_full, _ = run("full")
    n_upd = N_SCANS // every
    line = {"metric": "incremental ESDF update ms (configs[1], update every %d scans)" % every,
            "value": t_inc / n_upd, "unit": "ms/update", "higher_is_better": False, "n_gpus": world,
            "steps": n_upd, "warmup": args.warmup, "data": "synthetic", "dtype": "i64",
            "config": {"workload": "lidar_submap_os1_64x1024_200scans_0.2m (BJ configs[1])", "every_scans": every},
            "esdf_max_distance_m": cfg["grid"].get("esdf_max_distance", 2.0),
            "blocks_recomputed_per_update": queued / n_upd,
            "exact_finalize_ms_per_update": t_full / n_upd,
            "inc_kernel_ms_per_update": {k: v["ms"] / n_upd for k, v in prof.items()},
            "inc_launches_per_update": {k: v["n"] / n_upd for k, v in prof.items()},
            "speedup_vs_exact_recompute": t_full / t_inc}
    if rank == 0:
        print(json.dumps(line), flush=True)


def run_esdf_stress(args, world, rank, local):
    """BASELINE.json configs[4]: 2 cm voxels over 40 x 40 x 10 m (2e9 voxels, ~3.9 M blocks), TSDF imported
    from an analytic SDF (D = clamp(sdf, +-0.06), W = 1), one full exact ESDF recompute per step."""
    import paper_2410_21149_b200 as cvx
    import synth.scenes as S
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    s, tau = 0.02, 0.06
    grid = dict(voxel_size=s, truncation=tau, site_threshold=s, max_blocks=4_000_000)
    sm = cvx.Submap(grid, np.eye(4), local)
    nb = 0
    for b, D, W in S.esdf_stress_blocks(voxel_size=s, truncation=tau, device=dev, seed=4 + rank):
        sm.import_tsdf(b, D, W)
        nb += b.shape[0]
    torch.cuda.synchronize()
    for _ in range(args.warmup):
        sm.finalize_esdf()
    lo, hi = sm.aabb()
    dims = (hi - lo + 1) * 8
    N = int(np.prod(dims.astype(np.int64)))
    va = nb * 512
    sm.profile(True)
    stream = torch.cuda.current_stream(dev)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            sm.finalize_esdf()
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    prof = sm.profile_report()
    per = {k: v["ms"] / args.steps for k, v in prof.items()}
    hbm, hbm_src, _ = peaks()
    alg = esdf_alg_bytes(va, N)
    dom = max(alg, key=lambda k: per.get(k, 0.0))
    ach = alg[dom] / (per[dom] / 1e3) / 1e9
    tot_alg = sum(alg.values()) / (sum(per[k] for k in alg) / 1e3) / 1e9
    line = {"metric": "ESDF Mvoxels/s (configs[4] full exact recompute)", "value": va / 1e6 / (ms / 1e3),
            "unit": "Mvox/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "i64/u32+f32",
            "data": "synthetic", "config": {"workload": "esdf_stress_40x40x10m_2cm (BJ configs[4])",
                                            "blocks": nb, "allocated_voxels": va, "aabb_voxels": dims.tolist()},
            "dense_gvox_per_s": N / 1e9 / (ms / 1e3), "kernel_ms_per_step": per,
            "roofline": {"kernel": dom, "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
                         "frac": ach / hbm, "traffic": (ncu_traffic(dom, "esdf_stress") or {}).get("bytes_per_launch"),
                         "traffic_source": (ncu_traffic(dom, "esdf_stress") or {}).get("source"), "peak_source": hbm_src,
                         "all_passes_gbs": tot_alg},
            "gpu_launches": sum(v["n"] for v in prof.values()), "clocks": clk.summary(),
            "esdf_roofline": {k: {"ms": per[k], "alg_bytes": alg[k], "achieved_gbs": alg[k] / (per[k] / 1e3) / 1e9,
                                  "frac": alg[k] / (per[k] / 1e3) / 1e9 / hbm} for k in alg if per.get(k)}}
    del sm
    torch.cuda.empty_cache()
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = stress_cpu_baseline(s, tau, dev)
    if rank == 0:
        print(json.dumps(line), flush=True)


def stress_cpu_baseline(s, tau, dev, sub=(48, 48, 25)):
    """The oracle's exact ESDF (single-threaded, stage-isolated: the same analytic TSDF) on a sub-volume of
    configs[4]: the blocks with (bx, by, bz - bz0) < sub, i.e. 384 x 384 x 200 voxels (SURVEY §8(d) plans a
    1000 x 1000 x 250 sub-volume; this one keeps the CPU leg to ~10-30 s)."""
    import oracle
    import synth.scenes as S
    keep_b, keep_D, keep_W = [], [], []
    bz0 = None
    for b, D, W in S.esdf_stress_blocks(voxel_size=s, truncation=tau, device=dev):
        if bz0 is None:
            bz0 = int(b[:, 2].min())
        m = (b[:, 0] < sub[0]) & (b[:, 1] < sub[1]) & (b[:, 2] - bz0 < sub[2])
        if m.any():
            keep_b.append(b[m].cpu()); keep_D.append(D[m].cpu()); keep_W.append(W[m].cpu())
    b = torch.cat(keep_b).numpy()
    D = torch.cat(keep_D).double().numpy()
    W = torch.cat(keep_W).double().numpy()
    t0 = time.perf_counter()
    oracle.esdf(b, D, W, s, s)
    dt = time.perf_counter() - t0
    va = b.shape[0] * 512
    return {"value": va / 1e6 / dt, "unit": "Mvox/s", "cores": 1, "kind": "oracle",
            "sample": f"exact ESDF of a {sub[0] * 8} x {sub[1] * 8} x {sub[2] * 8}-voxel sub-volume of configs[4] "
                      f"({b.shape[0]} blocks), same analytic TSDF (stage-isolated)", "seconds": dt}


def rgbd_cpu_baseline(cfg, sub, depth, poses, n=2):
    """The oracle as it stands, single-threaded, on the first n frames of one configs[2] submap with each
    integrator, plus the exact ESDF of the raycast result."""
    import oracle
    g = cfg["grid"]
    frames = [depth[k].cpu().numpy() for k in range(n)]
    out = {}
    for mode in ("raycast", "projective"):
        o = oracle.OracleSubmap(g, sub["T_world_submap"])
        t0 = time.perf_counter()
        for k in range(n):
            (o.integrate if mode == "raycast" else o.integrate_projective)(frames[k], poses[k], cfg["sensor"])
        out[mode] = time.perf_counter() - t0
        if mode == "raycast":
            b, D, W = o.export()
            t1 = time.perf_counter()
            oracle.esdf(b, D, W, g["voxel_size"], g["site_threshold"])
            out["esdf"] = time.perf_counter() - t1
    return {"value": n / (out["raycast"] + out["esdf"]), "unit": "scans/s", "cores": 1, "kind": "oracle",
            "sample": f"first {n} of the 100 frames of submap 0, raycast integration + exact ESDF "
                      f"({b.shape[0]} blocks); projection integration of the same frames timed beside it",
            "raycast_frames_per_s": n / out["raycast"], "projective_frames_per_s": n / out["projective"],
            "seconds": out["raycast"] + out["esdf"] + out["projective"]}


def run_rgbd(args, world, rank, local):
    """BASELINE.json configs[2]: 1000 synthetic 640x480 depth frames of an indoor room, 5 cm voxels, a
    submap every 100 frames (10 submaps, sharded over the ranks: strong scaling).  Each submap is built
    twice per step — by the paper's raycasting integrator (the value) and by the projection-mapping
    integrator (the comparison systems' scheme) — each followed by the exact
    ESDF.  Both times are reported, with their voxel-update counts."""
    import paper_2410_21149_b200 as cvx
    import synth
    from paper_2410_21149_b200.parallel import shard_submaps
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        init_pg(dev)
        pg = dist
    cfg0 = synth.make_config("rgbd", frames=[], device=dev)
    subs = cfg0["submaps"]
    mine = shard_submaps([len(sm["frames"]) for sm in subs], world)[rank]
    frames = sorted(k for i in mine for k in subs[i]["frames"])
    cfg = synth.make_config("rgbd", frames=frames, device=dev)
    data = {i: torch.stack([cfg["frames"][k]["data"] for k in subs[i]["frames"]]).contiguous() for i in mine}
    poses = {i: np.stack([cfg["frames"][k]["T_world_sensor"] for k in subs[i]["frames"]]) for i in mine}
    sm = cvx.Submap(cfg["grid"], subs[mine[0]]["T_world_submap"] if mine else np.eye(4), local)
    stream = torch.cuda.current_stream(dev)
    res = {}
    for mode in ("raycast", "projective"):
        def step():
            for i in mine:
                sm.reset(subs[i]["T_world_submap"])
                if mode == "raycast":
                    sm.integrate_batch(data[i], poses[i], cfg["sensor"])
                else:
                    sm.integrate_projective(data[i], poses[i], cfg["sensor"])
                sm.finalize_esdf()

        for _ in range(args.warmup):
            step()
        upd = 0
        if mine:   # updates per step (from the last warm-up's counters, summed over my submaps)
            for i in mine:
                sm.reset(subs[i]["T_world_submap"])
                st = (sm.integrate_batch(data[i], poses[i], cfg["sensor"], stats=True) if mode == "raycast"
                      else sm.integrate_projective(data[i], poses[i], cfg["sensor"], stats=True))
                upd += st["voxel_updates"]
        if pg is not None:
            pg.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(local) as clk:
            e0.record(stream)
            for _ in range(args.steps):
                step()
            e1.record(stream)
            torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        if pg is not None:
            t = torch.tensor([ms], device=dev, dtype=torch.float64)
            pg.all_reduce(t, op=pg.ReduceOp.MAX)
            ms = float(t.item())
        sm.profile(True, serialize=True)     # one more step, per-kernel solo times (CUDA events)
        step()
        prof = {k: round(v["ms"], 4) for k, v in sm.profile_report().items()}
        sm.profile(False)
        res[mode] = (ms, clk.summary(), upd, prof)
    n_frames = sum(len(x["frames"]) for x in subs)
    ms, clk, upd, prof = res["raycast"]
    line = {"metric": METRIC, "value": n_frames / (ms / 1e3), "unit": "scans/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32+i64", "data": "synthetic",
            "config": {"workload": "rgbd_indoor_640x480_1000frames_0.05m_submap_per_100 (BJ configs[2])",
                       "submaps": len(subs), "parallelism": f"submap-sharded x{world} (LPT)",
                       "inputs_exceed_l2": True, "l2_note": "1.2 GB of depth frames resident in HBM"},
            "raycast": {"ms_per_step": ms, "frames_per_s": n_frames / (ms / 1e3), "voxel_updates_rank0": upd,
                        "kernel_ms_per_step_serial": prof},
            "projective": {"ms_per_step": res["projective"][0], "frames_per_s": n_frames / (res["projective"][0] / 1e3),
                           "voxel_updates_rank0": res["projective"][2], "kernel_ms_per_step_serial": res["projective"][3]},
            "raycast_over_projective_time": ms / res["projective"][0],
            "clocks": clk}
    if rank == 0 and world == 1 and not args.no_cpu_baseline and mine:
        line["cpu_baseline"] = rgbd_cpu_baseline(cfg, subs[mine[0]], data[mine[0]], poses[mine[0]])
    if rank == 0:
        print(json.dumps(line), flush=True)
    if pg is not None:
        pg.barrier()
        pg.destroy_process_group()


def run_voxel_sweep(args, world, rank, local):
    """SURVEY §2.5 E2 (Fig. 4b: "execution time ... increasing the number of voxels from
    one to four million"): the configs[1] submap (200 scans) integrated at voxel sizes swept so the
    allocated voxels go from ~1 M to beyond 4 M (tau = 3 s), TSDF integration timed alone and with the
    exact ESDF.  Reports (voxels, voxel updates, ms) per size; the paper's claim is near-linear scaling."""
    import paper_2410_21149_b200 as cvx
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cfg, data, poses = make_workload(rank, dev)
    rows = []
    for s in (0.8, 0.64, 0.5, 0.4, 0.32, 0.25, 0.2):
        g = dict(cfg["grid"], voxel_size=s, truncation=3 * s, site_threshold=s)
        sm = cvx.Submap(g, cfg["submaps"][0]["T_world_submap"], local)
        stream = torch.cuda.current_stream(dev)

        def integ():
            sm.reset()
            sm.integrate_batch(data, poses, cfg["sensor"])

        for _ in range(args.warmup):
            integ()
            sm.finalize_esdf()
        st = sm.stats()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        t_int = t_all = 0.0
        for _ in range(args.steps):
            torch.cuda.synchronize()
            e[0].record(stream)
            integ()
            e[1].record(stream)
            sm.finalize_esdf()
            e[2].record(stream)
            torch.cuda.synchronize()
            t_int += e[0].elapsed_time(e[1])
            t_all += e[0].elapsed_time(e[2])
        rows.append({"voxel_size": s, "blocks": st["total_blocks"], "voxels": st["total_blocks"] * 512,
                     "voxel_updates": st["voxel_updates"], "integrate_ms": t_int / args.steps,
                     "integrate_esdf_ms": t_all / args.steps})
        del sm
    base = next(r for r in rows if r["voxels"] >= 0.8e6)
    for r in rows:
        r["voxels_rel"] = r["voxels"] / base["voxels"]
        r["time_rel"] = r["integrate_ms"] / base["integrate_ms"]
    line = {"metric": METRIC, "value": N_SCANS / (rows[-1]["integrate_esdf_ms"] / 1e3), "unit": "scans/s",
            "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": rows[-1]["integrate_esdf_ms"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32+i64",
            "data": "synthetic",
            "config": {"workload": "voxel_sweep_lidar_submap_200scans (BJ configs[1], E2 / Fig. 4b shape)",
                       "voxel_sizes": [r["voxel_size"] for r in rows]},
            "sweep": rows}
    if rank == 0:
        print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------ product arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="cvx", choices=["cvx", "reference"])
    ap.add_argument("--batch", type=int, default=200, help="scans per integrate_batch call (the library splits them into equal launches of <= 2^24 - 1 rays and <= 200 frames: one launch for 200 OS1-64 scans)")
    ap.add_argument("--queries", type=int, default=1 << 20)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--workload", default="lidar", choices=["lidar", "esdf_stress", "incremental", "mav", "color", "rgbd", "voxel_sweep"],
                    help="lidar: configs[1] (default bench line); esdf_stress: configs[4] full ESDF recompute")
    args = ap.parse_args()
    world, rank, local = dist_setup()
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    if args.workload == "esdf_stress":
        run_esdf_stress(args, world, rank, local)
        return
    if args.workload == "incremental":
        run_incremental(args, world, rank, local)
        return
    if args.workload == "color":
        return run_color(args, world, rank, local)
    if args.workload == "mav":
        run_mav(args, world, rank, local)
        return
    if args.workload == "rgbd":
        run_rgbd(args, world, rank, local)
        return
    if args.workload == "voxel_sweep":
        run_voxel_sweep(args, world, rank, local)
        return

    import paper_2410_21149_b200 as cvx
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        init_pg(dev)
        pg = dist
    cfg, data, poses = make_workload(rank, dev)
    sensor = cfg["sensor"]
    sm = cvx.Submap(cfg["grid"], cfg["submaps"][0]["T_world_submap"], local)
    s = cfg["grid"]["voxel_size"]
    stream = torch.cuda.current_stream(dev)

    # queries: uniform over the submap's AABB (world frame), fixed per run
    def build_once():
        sm.reset()
        for c in range(0, N_SCANS, args.batch):
            sm.integrate_batch(data[c:c + args.batch], poses[c:c + args.batch], sensor)
        sm.finalize_esdf()

    build_once()
    lo, hi = sm.aabb()
    gq = torch.Generator(device=dev).manual_seed(7 + rank)
    qs = torch.rand((args.queries, 3), device=dev, generator=gq, dtype=torch.float64)
    lo_m = torch.tensor(lo * 8 * s, device=dev, dtype=torch.float64)
    ext = torch.tensor((hi - lo + 1) * 8 * s, device=dev, dtype=torch.float64)
    xs = lo_m + qs * ext
    T = torch.tensor(sm.T_ws, device=dev, dtype=torch.float64)
    queries = (xs @ T[:3, :3].T + T[:3, 3]).to(torch.float32).contiguous()
    qout = torch.empty(args.queries, dtype=torch.float32, device=dev)
    qst = torch.empty(args.queries, dtype=torch.uint8, device=dev)
    gather_bytes = [0]
    gather_ms = []
    set_queries = torch.zeros((1 << 16, 3), dtype=torch.float32, device=dev)
    set_idx = (torch.arange(1 << 16, device=dev, dtype=torch.int32) % world).contiguous()
    set_queries.copy_(queries[:1 << 16])

    def gather(m):
        """N > 1: all-gather every rank's packed ESDF (one size exchange + one NCCL all-gather), index the
        gathered payloads as a cvx_esdf_set and run 64 k cross-submap look-ups on it (the registration
        consumer, SURVEY §8 e / f4)."""
        if pg is None:
            return
        from paper_2410_21149_b200.parallel import gather_esdfs
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cur = torch.cuda.current_stream(dev)
        e0.record(cur)
        buf, offsets, _ = gather_esdfs([m.pack()], max_per_rank=1)
        e1.record(cur)
        gather_ms.append((e0, e1))
        gather_bytes[0] = int(buf.numel())
        es = cvx.EsdfSet(buf, offsets)
        es.query(set_idx, set_queries)
        es.close()

    # Two submaps in flight (the paper's frontend/backend queues): step i builds submap i on builder i % 2
    # and its own stream.  Its front half (reset + integration) is enqueued first, then the back half
    # (finalize_esdf, queries, N > 1 gather) of step i - 1, so the exact ESDF + queries of step i - 1
    # (HBM / latency bound) overlap the integration of step i (ALU bound) and the host syncs of the back
    # half (finalize reads the block count / AABB; the gather exchanges sizes) never stall the next
    # integration.  Every step is still one complete pass of a1-a7 over its own submap; the last back half
    # runs inside the timed region (flush); `one_submap_in_flight` below times the same steps strictly one
    # after another.
    # The integrations themselves stay in order (step i's waits for step i - 1's on the device, not the
    # host): two concurrent walks only compete for the same ALU slots, while a walk beside an ESDF pass
    # fills them.  With host frames the library's copies of step i still start early (copy stream).
    backlog = []
    integrated = [torch.cuda.Event(), torch.cuda.Event()]
    last_integrated = [None]

    def flush():
        while backlog:
            backlog.pop()()

    order = os.environ.get("CVX_BENCH_ORDER", "1") != "0"   # test knob: integrations of consecutive steps ordered

    def after_previous_integration(k):
        if order and last_integrated[0] is not None:
            streams[k].wait_event(last_integrated[0])

    def mark_integrated(k):
        integrated[k].record(streams[k])
        last_integrated[0] = integrated[k]
    sm2 = cvx.Submap(cfg["grid"], cfg["submaps"][0]["T_world_submap"], local)
    builders = [sm, sm2]
    streams = [stream, torch.cuda.Stream(dev)]
    qouts = [(qout, qst), (torch.empty_like(qout), torch.empty_like(qst))]

    def step(i=0, src=None, pipelined=True):
        k = i % 2 if pipelined else 0
        m = builders[k]
        with torch.cuda.stream(streams[k]):
            after_previous_integration(k)
            m.reset()
            d = data if src is None else src
            for c in range(0, N_SCANS, args.batch):
                m.integrate_batch(d[c:c + args.batch], poses[c:c + args.batch], sensor)
            mark_integrated(k)

        def back():
            with torch.cuda.stream(streams[k]):
                m.finalize_esdf()
                m.query(queries, *qouts[k])
                gather(m)
        flush()                          # back half of the previous step
        backlog.append(back)
        if not pipelined:
            flush()

    def timed(fn, n):
        """Device time of n steps: events on the caller's stream, both builder streams joined."""
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(stream)
        streams[1].wait_stream(stream)
        for i in range(n):
            fn(i)
        flush()
        stream.wait_stream(streams[1])
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b)

    for i in range(args.warmup):
        step(i)
    flush()
    torch.cuda.synchronize()
    st = sm.stats()
    nb = sm.block_count()
    lo, hi = sm.aabb()
    dims = (hi - lo + 1) * 8
    nvox_dense = int(np.prod(dims.astype(np.int64)))

    # ---------------------------------------------------------------- timed region (device time)
    for m in builders:
        m.profile(True)
    if pg is not None:
        pg.barrier()
    with ClockSampler(local) as clk:
        ms_total = timed(step, args.steps)
    if pg is not None:
        pg.barrier()
    prof = {}
    for m in builders:
        for k_, v_ in m.profile_report().items():
            e_ = prof.setdefault(k_, {"ms": 0.0, "n": 0})
            e_["ms"] += v_["ms"]
            e_["n"] += v_["n"]
        m.profile(False)
    ms_one = timed(lambda i: step(i, pipelined=False), args.steps)   # one submap in flight, for reference
    if pg is not None:
        t = torch.tensor([ms_total, ms_one], device=dev, dtype=torch.float64)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        ms_total, ms_one = float(t[0].item()), float(t[1].item())
    ms_step = ms_total / args.steps
    value = world * N_SCANS / (ms_step / 1e3)

    # ---------------------------------------------------------------- e2e through host buffers
    e2e = None
    if not args.no_e2e:
        host_frames = data.cpu().pin_memory()
        host_outs = [(torch.empty(args.queries, dtype=torch.float32).pin_memory(),
                      torch.empty(args.queries, dtype=torch.uint8).pin_memory()) for _ in range(2)]
        host_q = queries.cpu().pin_memory()
        dev_qs = [torch.empty_like(queries) for _ in range(2)]

        def e2e_step(i):
            # the library copies each launch's scans from pinned host memory on its side stream, so the
            # transfer of launch k+1 overlaps the walk of launch k (cvx_integrate_batch_host)
            k = i % 2
            m = builders[k]
            with torch.cuda.stream(streams[k]):
                dev_qs[k].copy_(host_q, non_blocking=True)
                after_previous_integration(k)
                m.reset()
                for c in range(0, N_SCANS, args.batch):
                    m.integrate_batch_host(host_frames[c:c + args.batch], poses[c:c + args.batch], sensor)
                mark_integrated(k)

            def back():
                with torch.cuda.stream(streams[k]):
                    m.finalize_esdf()
                    m.query(dev_qs[k], *qouts[k])
                    host_outs[k][0].copy_(qouts[k][0], non_blocking=True)
                    host_outs[k][1].copy_(qouts[k][1], non_blocking=True)
                    gather(m)
            flush()
            backlog.append(back)

        e2e_step(0)
        e2e_step(1)
        flush()
        if pg is not None:
            pg.barrier()
        ems = timed(e2e_step, args.steps)
        if pg is not None:
            t = torch.tensor([ems], device=dev, dtype=torch.float64)
            pg.all_reduce(t, op=pg.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": world * N_SCANS / (ems / args.steps / 1e3), "unit": "scans/s",
               "h2d_bytes_per_step": int(data.numel() * 4 + queries.numel() * 4),
               "d2h_bytes_per_step": int(args.queries * 5), "ms_per_step": ems / args.steps}

    # ---------------------------------------------------------------- serialised pass (solo kernel times)
    # the pipelined timed region overlaps a1-a3 of launch k+1 with the walk of launch k, so side-stream
    # event times include waiting; two more steps with the side work on the caller's stream give every
    # kernel's solo time (untimed for `value`; used for the kernel shares and per-stage throughputs)
    sm.profile(True, serialize=True)
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(stream)
    for _ in range(2):
        step(pipelined=False)
    s1.record(stream)
    torch.cuda.synchronize()
    serial_ms = s0.elapsed_time(s1) / 2
    per_step_serial = {k: v["ms"] / 2 for k, v in sm.profile_report().items()}
    sm.profile(False)

    # ---------------------------------------------------------------- roofline of the dominant kernel
    hbm, hbm_src, mp = peaks()
    K = args.steps
    per_step = {k: v["ms"] / K for k, v in prof.items()}
    launches = sum(v["n"] for v in prof.values())
    va = nb * 512
    # algorithmic bytes per launch
    alg_bytes = esdf_alg_bytes(va, nvox_dense)
    alg_bytes["reset_zero_blocks"] = 16 * va
    n_rays_launch = st["rays_in"] / max(1, prof.get("ray_prepare", {"n": 1})["n"] / K)
    alg_bytes["ray_prepare"] = int(n_rays_launch * (12 + 48))   # 12 B point in, 48 B ray record out
    dom = max(per_step, key=per_step.get)
    esdf_ms = sum(v for k, v in per_step_serial.items() if k.startswith("esdf_"))
    integ_ms = sum(v for k, v in per_step_serial.items()
                   if k in ("compose_poses", "ray_prepare", "block_walk_allocate", "ray_walk_update", "fold",
                            "dense_fold_allocate"))
    walk = prof.get("ray_walk_update", {"ms": 0.0, "n": 1})
    updates_per_step = st["voxel_updates"]
    roofline = {}
    if dom in alg_bytes:
        n_l = prof[dom]["n"] / K
        avg_ms = prof[dom]["ms"] / prof[dom]["n"]
        ach = alg_bytes[dom] / (avg_ms / 1e3) / 1e9
        roofline = {"kernel": dom, "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
                    "frac": ach / hbm, "traffic": None, "peak_source": hbm_src, "launches_per_step": n_l}
    else:
        # ray_walk_update: bound by issue (ALU).  Algorithmic work per voxel update = SURVEY §8(d)'s 25-30
        # int/fp32 lane-ops (DDA step, sdf, weight, address, merge); `achieved` uses the low end (25), the
        # 30-op and this build's own 13-op count are reported beside it.  peak = SMs (from
        # the device properties) x 128 lanes x the SM clock sampled during the timed region.
        clk_mhz = (clk.summary().get("sm_mhz") or 1965.0)
        n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
        peak_tops = n_sm * 128 * clk_mhz * 1e6 / 1e12
        avg_ms = walk["ms"] / walk["n"]
        upd_launch = updates_per_step / (walk["n"] / K)
        ups = upd_launch / (avg_ms / 1e3)
        ach = 25 * ups / 1e12
        roofline = {"kernel": dom, "bound": "alu", "achieved": ach, "peak": peak_tops, "unit": "Tops/s",
                    "frac": ach / peak_tops, "traffic": None,
                    "updates_per_s": ups, "ops_per_update": 25, "ops_per_update_source": "SURVEY §8(d) (25-30)",
                    "frac_at_30_ops": 30 * ups / 1e12 / peak_tops, "frac_at_13_ops": 13 * ups / 1e12 / peak_tops,
                    "peak_source": f"{n_sm} SMs (device properties) x 128 lanes x {clk_mhz:.0f} MHz "
                                   "(SM clock sampled during the timed region)"}
    tr = ncu_traffic(dom)
    roofline["traffic"] = tr["bytes_per_launch"] if tr else None   # DRAM bytes per launch (ncu)
    roofline["traffic_source"] = tr["source"] if tr else None
    if dom == "ray_walk_update":
        # what binds the walk: with the dense window (R19) its instruction stream alone would
        # run in ~3.7 ms (reductions removed, CVX_DW_EXP=1); the L2 reductions are the rest — ncu's issue
        # utilisation and the RED sector rate against the measured L2 reduction ceiling say how close each is
        roofline["ncu_issue_slots_busy"] = ncu_metric(dom, "Issue Slots Busy")
        roofline["l2_red"] = l2_red_view(dom)
    line = {
        "metric": METRIC, "value": value, "unit": "scans/s", "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32+i64", "data": "synthetic",
        "config": {"workload": "lidar_submap_os1_64x1024_200scans_0.2m (BJ configs[1])", "scans_per_rank": N_SCANS,
                   "batch_scans": args.batch, "queries": args.queries, "voxel_size": s,
                   "truncation": cfg["grid"]["truncation"], "inputs_exceed_l2": True,
                   "l2_note": "157 MB of scans resident in HBM > 126 MB L2; no explicit flush",
                   "parallelism": f"submap-sharded x{world}",
                   "pipeline": "2 submaps in flight (ESDF + queries of step i overlap integration of step i+1)"},
        "esdf_mvox_per_s": va / 1e6 / (esdf_ms / 1e3) if esdf_ms else None,
        "esdf_dense_mvox_per_s": nvox_dense / 1e6 / (esdf_ms / 1e3) if esdf_ms else None,
        "tsdf_scans_per_s_kernels": N_SCANS / (integ_ms / 1e3) if integ_ms else None,
        "voxel_updates_per_step": updates_per_step, "blocks": nb, "aabb_voxels": dims.tolist(),
        "kernel_ms_per_step": per_step,
        "kernel_ms_per_step_serial": per_step_serial, "serial_ms_per_step": serial_ms,
        "one_submap_in_flight": {"ms_per_step": ms_one / args.steps,
                                 "value": world * N_SCANS / (ms_one / args.steps / 1e3)},
        "roofline": roofline,
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "e2e": e2e,
    }
    # the ESDF passes against the HBM roofline (solo times of the serialised pass)
    line["esdf_roofline"] = {
        k: {"ms": per_step_serial[k], "alg_bytes": alg_bytes[k],
            "achieved_gbs": alg_bytes[k] / (per_step_serial[k] / 1e3) / 1e9,
            "frac": alg_bytes[k] / (per_step_serial[k] / 1e3) / 1e9 / hbm}
        for k in ("esdf_pass_x", "esdf_pass_y", "esdf_pass_z") if per_step_serial.get(k)}
    line["esdf_roofline"]["peak_gbs"] = hbm
    line["esdf_roofline"]["peak_source"] = hbm_src
    if world > 1:
        torch.cuda.synchronize()
        g_ms = [a.elapsed_time(b) for a, b in gather_ms[-args.steps:]] or [0.0]
        g_avg = sum(g_ms) / len(g_ms)
        line["gather"] = {"bytes_per_step": gather_bytes[0], "ms": g_avg,
                          "algbw_gbs": gather_bytes[0] / (g_avg / 1e3) / 1e9 if g_avg else None,
                          "busbw_gbs": gather_bytes[0] * (world - 1) / world / (g_avg / 1e3) / 1e9 if g_avg else None,
                          "note": "all-gather of every rank's packed ESDF + cvx_esdf_set over it + 64 k look-ups; "
                                  "time = size exchange + all_gather_into_tensor on the rank's stream"}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_sample(cfg, data, poses)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if pg is not None:
        pg.barrier()
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
