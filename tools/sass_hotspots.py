"""Per-instruction stall samples of one launch in an ncu report (needs
-lineinfo): totals by stall reason and by opcode, and the hottest
instructions.  python tools/sass_hotspots.py REPORT LAUNCH_INDEX [TOP]"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep, idx = sys.argv[1], int(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-skip", str(idx),
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
print(rows[0][1][:120])
h = rows[1]
ci = {n: i for i, n in enumerate(h)}
reasons = [n for n in h if n.startswith("stall_") and "Not Issued" not in n]
body = [r for r in rows[2:] if len(r) == len(h) and r[0].startswith("0x")]
tot = Counter()
op = Counter()
for r in body:
    s = int(r[ci["Warp Stall Sampling (All Samples)"]] or 0)
    code = r[ci["Source"]].strip().split()
    opc = (code[1] if code and code[0].startswith("@") and len(code) > 1 else (code[0] if code else "?")).split(".")[0]
    op[opc] += s
    for n in reasons:
        tot[n] += int(r[ci[n]] or 0)
allS = sum(tot.values())
print("samples", allS)
print("by reason:", ", ".join(f"{k[6:]} {100 * v / allS:.1f}%" for k, v in tot.most_common(8)))
print("by opcode:", ", ".join(f"{k} {100 * v / allS:.1f}%" for k, v in op.most_common(12)))
hot = sorted(body, key=lambda r: -int(r[ci["Warp Stall Sampling (All Samples)"]] or 0))[:top]
for r in hot:
    s = int(r[ci["Warp Stall Sampling (All Samples)"]] or 0)
    why = sorted(((int(r[ci[n]] or 0), n[6:]) for n in reasons), reverse=True)[:2]
    print(f"{100 * s / allS:5.2f}% {r[ci['Address']][-5:]} {r[ci['Source']].strip()[:60]:60s} {why}")
