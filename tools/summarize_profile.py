"""Summarise an ncu capture of the colored kernel into profiles/.

python tools/summarize_profile.py TAG CONFIG
reads gpurun_out/launches_TAG.csv and gpurun_out/prof_TAG.ncu-rep, writes
profiles/TAG_launches.csv (kernel share of the launch list),
profiles/TAG_summary.md and profiles/traffic_CONFIG.json (DRAM bytes per
captured launch vs the algorithmic bytes bench.py uses for `achieved`).
The captured launches are stage 2 (a = 0.75) colors 1..n of one SSP-RK3 step.
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

tag, cfg = sys.argv[1], sys.argv[2]
out = ROOT / "profiles"
out.mkdir(exist_ok=True)

# ---- launch list shares
rows = list(csv.reader(open(ROOT / "gpurun_out" / f"launches_{tag}.csv")))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = defaultdict(list)
for r in rows[hi + 1:]:
    agg[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")))
tot = sum(sum(v) for v in agg.values())
with open(out / f"{tag}_launches.csv", "w") as f:
    f.write("kernel,launches,total_ns,avg_ns,share_pct\n")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        f.write(f"\"{k}\",{len(v)},{sum(v):.0f},{sum(v)/len(v):.0f},{100*sum(v)/tot:.2f}\n")

# ---- full capture
raw = subprocess.run(["ncu", "-i", str(ROOT / "gpurun_out" / f"prof_{tag}.ncu-rep"), "--page", "raw",
                      "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
H = rr[0]
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_issued.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "launch__grid_size", "launch__block_size"]
units = rr[1]
launches = []
for r in rr[2:]:
    d = {k: r[H.index(k)] for k in keys if k in H}
    stall_cols = [i for i, n in enumerate(H) if n.startswith("smsp__pcsamp_warps_issue_stalled_")
                  and not n.endswith("not_issued")]
    st = sorted(((float(r[i].replace(",", "") or 0), H[i][len("smsp__pcsamp_warps_issue_stalled_"):])
                 for i in stall_cols if r[i] not in ("", "n/a")), reverse=True)[:5]
    d["stalls"] = st
    launches.append(d)


def mb(x, unit):
    v = float(x.replace(",", ""))
    return v * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(unit, 1.0)


ui = {k: units[H.index(k)] for k in keys if k in H}

# ---- algorithmic bytes of the same launches (CPU-side layout, no device)
import bench  # noqa: E402
import paper_1601_07613_b200 as P  # noqa: E402
from paper_1601_07613_b200.dg.layout import build_surface_list  # noqa: E402
from paper_1601_07613_b200.dg.basis import reference_tables  # noqa: E402
spec = bench.config_spec(cfg, device=None)
obj = spec["build"]()
if isinstance(obj, tuple):
    mesh, col = obj[0].mesh, obj[1]
    mort = obj[0].hanging_array()
else:
    mesh = obj
    col, _ = P.color(mesh)
    mort = None
plan = P.build_plan(mesh, col)
lm, lc = P.apply_plan(mesh, col, plan)
sl = build_surface_list(lm, lc.colors, lc.n_colors,
                        mortars=None if mort is None else plan.surface_perm[mort])


class _Op:
    pass


op = _Op()
op.surfaces = sl
op.dim = mesh.dim
op.n_equations = 1 if spec["physics"] == "advection" else mesh.dim + 2
op.n_basis = reference_tables(sl.kind, spec["p"]).n_basis
algo = [bench.launch_bytes(op, c, 1, 0.75) for c in range(1, sl.n_colors + 1)]

lines = [f"# ncu summary `{tag}` (config {cfg})", "",
         "Captured: stage 2 (a=0.75) color launches of one SSP-RK3 step, "
         "`ncu --set full --clock-control none` (cold-cache, serialised; shares and "
         "traffic are meaningful, absolute times are not bench numbers).", "",
         "| launch | kernel | ncu us | DRAM rd MB | DRAM wr MB | algorithmic MB | traffic/algo | "
         "DRAM % | warps active % | L1 % | fp64 % | issue % | regs | top stalls |",
         "|---|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
traffic = []
for i, d in enumerate(launches):
    rd = mb(d["dram__bytes_read.sum"], ui["dram__bytes_read.sum"])
    wr = mb(d["dram__bytes_write.sum"], ui["dram__bytes_write.sum"])
    al = algo[i % len(algo)] / 1e6
    traffic.append((rd + wr) * 1e6)
    lines.append(f"| color {i % len(algo) + 1} | {d['Kernel Name'].split('<')[0]} | "
                 f"{float(d['gpu__time_duration.sum'].replace(',', '')) * {'nsecond': 1e-3, 'ns': 1e-3, 'usecond': 1.0, 'us': 1.0, 'msecond': 1e3, 'ms': 1e3}.get(ui['gpu__time_duration.sum'], 1.0):.1f} | "
                 f"{rd:.0f} | {wr:.0f} | {al:.0f} | {(rd + wr) / al:.2f} | "
                 f"{d.get('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', '')} | "
                 f"{d['sm__warps_active.avg.pct_of_peak_sustained_active']} | "
                 f"{d['l1tex__throughput.avg.pct_of_peak_sustained_active']} | "
                 f"{d['sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active']} | "
                 f"{d['sm__inst_issued.avg.pct_of_peak_sustained_active']} | "
                 f"{d['launch__registers_per_thread']} | "
                 + ", ".join(f"{n} {int(v)}" for v, n in d["stalls"][:3]) + " |")
lines += ["", "Launch list shares (`launches` csv, all kernels of a 2+1-step bench run):", ""]
for line in open(out / f"{tag}_launches.csv").read().splitlines()[1:6]:
    lines.append("    " + line)
(out / f"{tag}_summary.md").write_text("\n".join(lines) + "\n")
json.dump({"tag": tag, "config": cfg, "bytes_per_launch_avg": float(np.mean(traffic)),
           "algorithmic_bytes_per_launch_avg": float(np.mean(algo)),
           "per_launch_dram_bytes": traffic, "per_launch_algorithmic_bytes": algo,
           "note": "DRAM read+write per captured colored launch (stage 2, colors 1..n)"},
          open(out / f"traffic_{cfg}.json", "w"), indent=1)
print("\n".join(lines))
