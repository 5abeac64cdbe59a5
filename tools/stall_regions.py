"""Stall samples of one launch of an ncu report aggregated over SASS
address ranges (e.g. the volume point-pair loop vs the surface part):
    python tools/stall_regions.py REPORT LAUNCH_INDEX NAME=LO:HI [NAME=LO:HI ...]
LO/HI are hex SASS offsets (from cuobjdump -sass of the same build); the
rest of the kernel is reported as "other".  Per region: share of the stall
samples, share of the executed warp instructions, top stall reasons and
the executed-opcode mix."""
import csv
import io
import subprocess
import sys
from collections import Counter, defaultdict

rep, idx = sys.argv[1], int(sys.argv[2])
regions = []
for a in sys.argv[3:]:
    name, rng = a.split("=")
    lo, hi = rng.split(":")
    regions.append((name, int(lo, 16), int(hi, 16)))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-skip", str(idx),
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ci = {n: i for i, n in enumerate(h)}
reasons = [n for n in h if n.startswith("stall_") and "Not Issued" not in n]
body = [r for r in rows[2:] if len(r) == len(h) and r[0].startswith("0x")]
samples = Counter()
execd = Counter()
why = defaultdict(Counter)
ops = defaultdict(Counter)
base = int(body[0][ci["Address"]], 16)
for r in body:
    addr = int(r[ci["Address"]], 16) - base
    s = int(r[ci["Warp Stall Sampling (All Samples)"]] or 0)
    reg = "other"
    for name, lo, hi in regions:
        if lo <= addr <= hi:
            reg = name
            break
    samples[reg] += s
    n_ex = int(r[ci["Instructions Executed"]] or 0)
    execd[reg] += n_ex
    for n in reasons:
        why[reg][n[6:]] += int(r[ci[n]] or 0)
    code = r[ci["Source"]].strip().split()
    opc = (code[1] if code and code[0].startswith("@") and len(code) > 1 else (code[0] if code else "?"))
    ops[reg][opc.split(".")[0]] += n_ex
tot = sum(samples.values())
tex = sum(execd.values())
print(rows[0][1][:100], "samples", tot)
for reg, s in samples.most_common():
    w = why[reg]
    ws = sum(w.values()) or 1
    print(f"{reg:8s} stalls {100 * s / tot:5.1f}% instrs {100 * execd[reg] / tex:5.1f}%  " +
          ", ".join(f"{k} {100 * v / ws:.0f}%" for k, v in w.most_common(5)) +
          "  | executed: " + ", ".join(f"{k} {100 * v / (execd[reg] or 1):.0f}%"
                                   for k, v in ops[reg].most_common(5)))
