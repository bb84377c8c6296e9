"""Per-kernel mean duration over the last N launches of an ncu launch-list CSV
(--metrics gpu__time_duration.sum[,launch__grid_size]).

  python tools/launch_breakdown.py gpurun_out/launches.csv [last_n]
"""
import csv
import sys
from collections import defaultdict


def main():
    path = sys.argv[1]
    last_n = int(sys.argv[2]) if len(sys.argv) > 2 else 280
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[start]
    ik, iv, im, iid = (h.index(x) for x in ("Kernel Name", "Metric Value", "Metric Name", "ID"))
    per = defaultdict(dict)
    for r in rows[start + 1:]:
        if len(r) > iv:
            per[int(r[iid])][r[im]] = r[iv]
            per[int(r[iid])]["k"] = r[ik].split("(")[0][:48]
    agg = defaultdict(list)
    for i in sorted(per)[-last_n:]:
        d = per[i]
        agg[d["k"]].append((float(d["gpu__time_duration.sum"].replace(",", "")),
                            d.get("launch__grid_size", "")))
    for k, v in agg.items():
        print(f"{k:50s} n={len(v):4d} mean {sum(x for x, _ in v) / len(v) / 1000:8.2f} us"
              f"  grid {v[0][1]}")


if __name__ == "__main__":
    main()
