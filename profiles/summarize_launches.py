"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel shares: python profiles/summarize_launches.py launches.csv "title" > summary.txt"""

import collections
import csv
import re
import sys


def main(path, title):
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    h = rows[0]
    ik, ig, iv, iu = h.index("Kernel Name"), h.index("Grid Size"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    total = 0.0
    for r in rows[1:]:
        name = re.sub(r"^void ", "", r[ik])
        name = re.sub(r"\(.*$", "", name).replace("amrb::<unnamed>::", "").replace("amrb::", "")
        us = float(r[iv]) * {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3}.get(r[iu], 1e-3)
        key = (name[:60], r[ig])
        agg[key][0] += 1
        agg[key][1] += us
        total += us
    print(title)
    print("gpu__time_duration.sum, --clock-control none; serialised + cold-cache: compare SHARES, not absolutes")
    print(f"total launches {sum(v[0] for v in agg.values())}, total kernel time {total / 1e3:.2f} ms")
    print("  share  count    avg_us  kernel (grid)")
    for (name, grid), (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:30]:
        print(f"{100 * us / total:6.2f}% {n:6d} {us / n:9.2f}  {name} {grid}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else path)
