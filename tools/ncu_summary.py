"""Summarise an ncu report (or a launch-list CSV) into a committed text file.

  python tools/ncu_summary.py rep gpurun_out/prof.ncu-rep > profiles/rN_x.txt
  python tools/ncu_summary.py launches gpurun_out/launches.csv > profiles/rN_launches.txt
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

DETAILS = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
           "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread",
           "Dynamic Shared Memory Per Block", "Waves Per SM", "L2 Hit Rate", "Executed Ipc Active"]
RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "pcie__read_bytes.sum.per_second", "pcie__write_bytes.sum.per_second",
       "syslts__t_sectors_srcunit_tex_aperture_sysmem_op_read_lookup_miss.sum",
       "syslts__t_sectors_aperture_sysmem_lookup_miss.sum",
       "sm__throughput.avg.pct_of_peak_sustained_elapsed",
       "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
       "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]


def ncu_csv(rep, page):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True,
                         text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def summarize_rep(rep):
    rows = ncu_csv(rep, "details")
    h = rows[0]
    per = defaultdict(list)
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") in DETAILS:
            per[(d["ID"], d["Kernel Name"])].append(
                f"  {d['Metric Name']:32s} {d['Metric Value']:>14s} {d['Metric Unit']}")
    raw = ncu_csv(rep, "raw")
    rh, ru = raw[0], raw[1]
    rawper = {}
    for i, r in enumerate(raw[2:]):
        lines = []
        for k, v, u in zip(rh, r, ru):
            if k in RAW:
                lines.append(f"  {k:70s} {v:>16s} {u}")
        rawper[i] = lines
    for i, ((kid, name), lines) in enumerate(sorted(per.items(), key=lambda x: int(x[0][0]))):
        print(f"[{kid}] {name}")
        print("\n".join(lines))
        print("\n".join(rawper.get(i, [])))
        print()


def summarize_launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = defaultdict(list)
    unit = None
    for r in rows[hi + 1:]:
        if len(r) > vi:
            agg[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")))
            unit = r[ui]
    tot = sum(sum(v) for v in agg.values())
    print(f"launches: {sum(len(v) for v in agg.values())}, total {tot:.0f} {unit} "
          "(ncu --clock-control none, serialised, cold-cache: compare shares)")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f"  {k:40s} n={len(v):4d} mean={sum(v) / len(v):14.0f} {unit} "
              f"share={100 * sum(v) / tot:6.2f}%")


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    summarize_rep(path) if kind == "rep" else summarize_launches(path)
