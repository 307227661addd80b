"""Digest of an ncu launch list (--metrics gpu__time_duration.sum --csv):
per step kernel, launches, mean duration and share of the step.

    python tools/launch_summary.py launches.csv [kernel-regex]
"""
import csv
import re
import sys
from collections import defaultdict


def main(path, pat=r"k_kuhn|k_rows_pairs|k_blk_rhs|k_blk_gather"):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ik, iv = h.index("Kernel Name"), h.index("Metric Value")
    tot, cnt, n = defaultdict(float), defaultdict(int), 0
    for r in rows[hdr + 1:]:
        if len(r) <= iv:
            continue
        n += 1
        name = re.sub(r"\(.*", "", r[ik])
        if re.search(pat, name):
            tot[name] += float(r[iv].replace(",", "")) / 1e6
            cnt[name] += 1
    step = sum(tot[k] / cnt[k] for k in tot)
    print(f"{n} launches captured (setup + warm-up + timed); the step kernels:")
    for k in sorted(tot, key=lambda k: -tot[k]):
        m = tot[k] / cnt[k]
        print(f"  {k[:44]:44s} n={cnt[k]:3d} mean={m:8.3f} ms  share={100 * m / step:5.1f} %")
    print(f"{len(tot)} launches per step, {step:.3f} ms summed; per-launch times are cold-cache and serialised "
          "(ncu): compare shares with bench.json kernels_ms")


if __name__ == "__main__":
    main(*sys.argv[1:])
