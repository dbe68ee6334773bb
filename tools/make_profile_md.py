"""Write profiles/<tag>/ from a gpurun_out/<tag>/ capture (tools/capture_round.sh): the bench line, the
ncu launch list, per-kernel ncu summaries and a markdown digest.  usage: python tools/make_profile_md.py r1"""
import json
import os
import shutil
import subprocess
import sys

tag = sys.argv[1]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = os.path.join(ROOT, "gpurun_out", tag)
dst = os.path.join(ROOT, "profiles", tag)
os.makedirs(dst, exist_ok=True)
bench = json.loads(open(os.path.join(src, "bench.json")).read().strip().splitlines()[-1])
json.dump(bench, open(os.path.join(dst, "bench.json"), "w"), indent=1)
shutil.copy(os.path.join(src, "launches.csv"), os.path.join(dst, "launches.csv"))
shares = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "launch_shares.py"), os.path.join(src, "launches.csv"),
                         os.path.join(src, "bench.json")], capture_output=True, text=True).stdout
kern = ["walk", "walk_cw", "dense_fold", "block_walk", "prepare", "fold", "esdf_pass_x", "esdf_pass_y", "esdf_pass_z", "query", "project",
        "stress_pass_x", "stress_pass_y", "stress_pass_z", "inc_window"]
summ = {}
for k in kern:
    rep = os.path.join(src, k + ".ncu-rep")
    if os.path.exists(rep):
        out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep, "12"],
                             capture_output=True, text=True).stdout
        open(os.path.join(dst, f"ncu_{k}.txt"), "w").write(out)
        summ[k] = out
if os.path.exists(os.path.join(src, "walk.ncu-rep")):
    shutil.copy(os.path.join(src, "walk.ncu-rep"), os.path.join(dst, "walk.ncu-rep"))


def metric(txt, name):
    for line in txt.splitlines():
        if line.startswith(name):
            return line[40:].split()[-1]
    return "-"


def unit(txt, name):
    for line in txt.splitlines():
        if line.startswith(name):
            return line.split()[1]
    return ""


rows = []
for k, t in summ.items():
    rows.append(f"| {k} | {metric(t, 'Duration')} {'ms' if 'Duration                                 ms' in t else 'us'} | "
                f"{metric(t, 'DRAM Throughput')} % | {metric(t, 'Issue Slots Busy')} % | {metric(t, 'Avg. Active Threads Per Warp')} | "
                f"{metric(t, 'Achieved Occupancy')} % | {metric(t, 'dram__bytes_read.sum')} / {metric(t, 'dram__bytes_write.sum')} {unit(t, 'dram__bytes_read.sum')} |")
b = bench
md = f"""# Profile {tag} — bench line, launch list and ncu captures

Produced by `tools/capture_round.sh {tag}` on one B200 (gpurun) and `tools/make_profile_md.py {tag}`.
ncu numbers come from separate profiled runs (`--clock-control none`, serialised, cold caches);
the bench numbers come from an unprofiled run with CUDA events.

## Bench (`bench.py`, N = 1, configs[1]: 200 OS1-64 scans, 0.2 m voxels)

* value **{b['value']:.0f} scans/s** ({b['ms_per_step']:.2f} ms per submap step); e2e (host buffers) {b['e2e']['value']:.0f} scans/s
* ESDF {b['esdf_mvox_per_s']:.0f} Mvox/s allocated ({b['esdf_dense_mvox_per_s']:.0f} Mvox/s over the dense AABB {b['aabb_voxels']})
* voxel updates per step {b['voxel_updates_per_step']:.3e}, blocks {b['blocks']}
* roofline (dominant kernel `{b['roofline']['kernel']}`): bound {b['roofline']['bound']}, achieved {b['roofline']['achieved']:.2f} of {b['roofline']['peak']:.1f} {b['roofline']['unit']} (frac {b['roofline']['frac']:.3f}); {b['roofline'].get('updates_per_s', 0):.3e} voxel updates/s
* clocks {b['clocks']}
* cpu_baseline (oracle, {b['cpu_baseline']['cores']} core): {b['cpu_baseline']['value']:.2f} scans/s — {b['cpu_baseline']['sample']}

## Kernel shares: ncu launch list vs bench CUDA events (serialised pass, solo kernel times)

```
{shares}```

## ncu (`--set full`) per kernel, one launch each

| kernel | duration | DRAM thr | issue busy | active thr/warp | achieved occ | DRAM read / write |
|---|---|---|---|---|---|---|
""" + "\n".join(rows) + """

Per-kernel stall breakdowns and the hottest SASS lines: `ncu_<kernel>.txt`. The dominant kernel's
full report is `walk.ncu-rep` (open with `ncu -i`).
"""
for extra in ("bench_rgbd.json", "bench_esdf_stress.json", "bench_mav.json", "bench_incremental.json", "bench_color.json",
              "bench_voxel_sweep.json", "bench_reference.json", "bench_n2_onegpu_gloo.json"):
    f = os.path.join(src, extra)
    if os.path.exists(f) and os.path.getsize(f):
        d = json.loads(open(f).read().strip().splitlines()[-1])
        json.dump(d, open(os.path.join(dst, extra), "w"), indent=1)
        md += f"\n## `{extra}`\n\n* value {d['value']:.4g} {d['unit']}, {d.get('ms_per_step') or 0:.2f} ms per step; " \
              f"workload {d['config']['workload']}\n"
        if "roofline" in d:
            r = d["roofline"]
            md += f"* roofline `{r['kernel']}`: {r['achieved']:.0f} of {r['peak']:.0f} {r['unit']} (frac {r['frac']:.3f})\n"
        if "projective" in d:
            md += f"* raycast {d['raycast']['ms_per_step']:.1f} ms vs projection {d['projective']['ms_per_step']:.1f} ms " \
                  f"per 1000 frames\n"
md += "\n`stress_pass_*`: ncu of the ESDF passes on configs[4] (2e9 voxels); `project`: the projection-mapping kernel on configs[2].\n"
open(os.path.join(dst, "summary.md"), "w").write(md)
print(md)
