"""Per-phase instruction / stall split of an ncu report (development aid):
    python tools/sass_phases.py report.ncu-rep [topN] [kernel-filter, e.g. regex:canon]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
kflt = ["-k", sys.argv[3]] if len(sys.argv) > 3 else []
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"] + kflt,
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
hdr, data = rows[1], rows[2:]
i_src, i_s, i_ex = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
data = [r for r in data if len(r) > max(i_ex, i_s) and r[i_ex].isdigit()]
ex = [int(r[i_ex] or 0) for r in data]
st = [int(r[i_s] or 0) for r in data]
bars = [k for k, r in enumerate(data) if "BAR.SYNC" in r[i_src]]
print("barriers at", bars, "total warp instr", sum(ex))
b = [0] + bars + [len(data)]
for a, c in zip(b[:-1], b[1:]):
    print(f"  [{a:5d},{c:5d}) instr {sum(ex[a:c]):>12d}  stall {100 * sum(st[a:c]) / max(sum(st), 1):5.1f}%")
tot = max(sum(st), 1)
for s_, k in sorted(((st[k], k) for k in range(len(data))), reverse=True)[:top]:
    print(f"{100 * s_ / tot:5.1f}% #{k:4d} ex={ex[k]:>10} {data[k][i_src].strip()[:70]}")
