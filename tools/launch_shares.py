"""Per-kernel share of a bench step from an ncu launch list (gpu__time_duration.sum per launch).

ncu serialises launches and runs them cold-cache, so only SHARES are comparable with bench.py's
CUDA-event kernel_ms_per_step, not absolute times.
usage: python tools/launch_shares.py launches.csv [bench.json-line-file]
"""
import csv
import json
import re
import sys
from collections import defaultdict

NAMES = [("prepare_kernel", "ray_prepare"), ("box_reduce_kernel", "ray_prepare"), ("walk_dw_kernel", "ray_walk_update"),
         ("dense_fold_kernel", "dense_fold_allocate"), ("ring_line_kernel<0", "esdf_pass_y"), ("ring_line_kernel<1", "esdf_pass_z"),
         ("ring_line_kernel<false", "esdf_pass_y"), ("ring_line_kernel<true", "esdf_pass_z"), ("block_walk_kernel", "block_walk_allocate"),
         ("block_walk2_kernel", "block_walk_allocate"), ("block_walk3_kernel", "block_walk_allocate"),
         ("walk_cw_kernel", "ray_walk_update"), ("link_line_kernel<0", "esdf_pass_y"), ("link_line_kernel<1", "esdf_pass_z"),
         ("link_line_kernel<false", "esdf_pass_y"), ("link_line_kernel<true", "esdf_pass_z"),
         ("pba_line_kernel<0", "esdf_pass_y"), ("pba_line_kernel<1", "esdf_pass_z"), ("clear_grid", "reset_grid"),
         ("fold_color_kernel", "fold_color"), ("pass_line_kernelILb0", "esdf_pass_y"), ("pass_line_kernelILb1", "esdf_pass_z"), ("pass_line_kernel<0", "esdf_pass_y"), ("pass_line_kernel<1", "esdf_pass_z"),
         ("walk_kernel", "ray_walk_update"), ("fold_kernel", "fold"), ("zero_blocks", "reset_zero_blocks"),
         ("reset_counters", "reset_counters"), ("compose_kernel", "compose_poses"),
         ("block_grid", "esdf_block_grid"), ("pass_x", "esdf_pass_x"), ("pass_line_kernel<0>", "esdf_pass_y"), ("pass_line_kernel<false>", "esdf_pass_y"),
         ("pass_line_kernel<1>", "esdf_pass_z"), ("pass_line_kernel<true>", "esdf_pass_z"), ("query_kernel", "query"), ("pack_kernel", "pack"),
         ("export_kernel", "export")]


def short(name):
    for pat, nm in NAMES:
        if pat in name.replace("(bool)0", "false").replace("(bool)1", "true"):
            return nm
    return re.sub(r"\(.*", "", name)


rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
h = rows[0]
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[1:]:
    d = dict(zip(h, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    k = short(d["Kernel Name"])
    tot[k] += float(d["Metric Value"]) / (1e3 if d["Metric Unit"] == "ns" else 1.0)
    cnt[k] += 1
T = sum(tot.values())
bench = None
if len(sys.argv) > 2:
    bl = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    # solo (serialised) event times when present: comparable with ncu's serialised launches
    bench = bl.get("kernel_ms_per_step_serial") or bl["kernel_ms_per_step"]
    BT = sum(bench.values())
print(f"{'kernel':<26}{'launches':>9}{'ncu us':>12}{'ncu share':>11}" + (f"{'bench share':>13}" if bench else ""))
for k in sorted(tot, key=lambda k: -tot[k]):
    line = f"{k:<26}{cnt[k]:>9}{tot[k]:>12.1f}{100 * tot[k] / T:>10.1f}%"
    if bench:
        line += f"{100 * bench.get(k, 0.0) / BT:>12.1f}%"
    print(line)
