"""DESIGN.md §8 tables from committed bench lines:
python tools/results_table.py profiles/r2_{c1,c2,c3,c4,c5}_bench.json"""
import json
import sys

rows = []
print("| cfg | G edges/s | G DOF-updates/s | ms/step | HBM frac (of 6,451.5 GB/s) | per-color GB/s | "
      "e2e G edges/s (public API, host arrays) | CPU oracle M edges/s (cores) | colored / buffered / "
      "atomic RHS ms | buffer avoided |")
print("|---|---|---|---|---|---|---|---|---|---|")
for f in sys.argv[1:]:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    r = d["roofline"]
    cfg = f.split("_")[1]
    cpu = d.get("cpu_baseline")
    cm = d.get("comparisons") or {}
    print(f"| {cfg} | {d['value'] / 1e9:.3f} | {d['dof_updates_per_s'] / 1e9:.1f} | "
          f"{d['ms_per_step']:.3f} | {r['frac']:.3f} | "
          + " / ".join(f"{v:.0f}" for v in r["per_color_gbs"].values()) + " | "
          f"{d['e2e']['value'] / 1e9:.3f} | "
          + (f"{cpu['value'] / 1e6:.2f} ({cpu['cores']})" if cpu else "—") + " | "
          + (f"{cm['rhs_colored_ms']:.3f} / {cm['rhs_buffered_ms']:.3f} / {cm['rhs_atomic_ms']:.3f}"
             if cm else "—") + " | "
          + (f"{cm['buffer_gb_truncated']} GB" if cm else "—") + " |")
