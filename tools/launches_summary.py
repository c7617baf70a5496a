"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) of bench.py.

Splits prefill (everything up to the last prefill_attn launch) from decode and
prints per-kernel totals and shares of the decode region.

    python tools/launches_summary.py gpurun_out/r01_launches.csv > profiles/r01_launches_summary.txt
"""

import csv
import sys
from collections import defaultdict


def load(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[start]
    ki, vi, ui, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit"), hdr.index(
        "Metric Name")
    out = []
    for r in rows[start + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}[r[ui]]
        out.append((r[ki], v))
    return out


def short(name):
    n = name.split("(")[0]
    return n.replace("void ", "").replace("kvpr::<unnamed>::", "kvpr::")[:70]


def main(path):
    seq = load(path)
    last_prefill = max((i for i, (n, _) in enumerate(seq) if "prefill_attn" in n or "prefill_fa" in n or "prefill_tc" in n), default=-1)
    regions = {"prefill+setup": seq[: last_prefill + 1], "decode": seq[last_prefill + 1:]}
    for name, part in regions.items():
        tot = defaultdict(float)
        cnt = defaultdict(int)
        for n, v in part:
            tot[short(n)] += v
            cnt[short(n)] += 1
        all_us = sum(tot.values())
        print(f"== {name}: {len(part)} launches, {all_us / 1e3:.3f} ms of kernel time (serialised, cold-cache) ==")
        for k in sorted(tot, key=lambda k: -tot[k]):
            print(f"  {tot[k] / 1e3:10.3f} ms  {100 * tot[k] / all_us:5.1f}%  n={cnt[k]:5d}  avg {tot[k] / cnt[k]:9.2f} us  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
