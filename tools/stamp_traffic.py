"""Write profiles/traffic.json from `ncu --set full` captures of the dominant
kernels, stamped with each kernel's SASS signature (tools/kernel_sig.py) and
the git head, so bench.py reports `roofline.traffic` only while the loaded
kernel is the one that was measured.

  python tools/stamp_traffic.py KERNEL@WORKLOAD=REPORT.ncu-rep[:algorithmic_bytes] ...

KERNEL is the kernel name (slow_attn_kernel, slow_attn_tc_kernel, ...),
WORKLOAD the bench workload (cfg2, ...); the report holds one launch of it.
Per launch: dram__bytes_read.sum + dram__bytes_write.sum, and the sysmem
(PCIe) read sectors x 32 B.
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import kernel_sig  # noqa: E402

OUT = os.path.join(ROOT, "profiles", "traffic.json")


def raw_metrics(rep, kernel):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(h, r))
        if kernel in d.get("Kernel Name", ""):
            u = dict(zip(h, units))
            return d, u
    raise SystemExit(f"{kernel} not in {rep}")


def to_bytes(v, unit):
    x = float(v.replace(",", ""))
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6,
                "GB": 1e9}.get(unit, 1)


def main():
    try:
        with open(OUT) as f:
            doc = {k: v for k, v in json.load(f).items() if "@" in k}
    except (OSError, ValueError):
        doc = {}
    git = subprocess.run(["git", "-C", ROOT, "rev-parse", "--short=12", "HEAD"],
                         capture_output=True, text=True).stdout.strip()
    for arg in sys.argv[1:]:
        key, rest = arg.split("=", 1)
        kernel = key.split("@")[0]
        rep, _, alg = rest.partition(":")
        d, u = raw_metrics(rep, kernel)
        dram = (to_bytes(d["dram__bytes_read.sum"], u["dram__bytes_read.sum"]) +
                to_bytes(d["dram__bytes_write.sum"], u["dram__bytes_write.sum"]))
        summary = os.path.join("profiles", os.path.basename(rep).replace(".ncu-rep", "_ncu.txt"))
        ent = {"source": summary + " (ncu --set full, one launch; report " +
                         os.path.basename(rep) + ")", "git": git,
               "sig": kernel_sig.kernel_sig(kernel),
               "dram_bytes_per_launch": dram,
               "duration_ns": float(d.get("gpu__time_duration.sum", "0").replace(",", "")) *
               {"nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6,
                "second": 1e9, "s": 1e9}.get(
                   u.get("gpu__time_duration.sum", "nsecond"), 1)}
        sec = "lts__t_sectors_srcunit_tex_aperture_sysmem_op_read.sum"
        for mk in (sec, "syslts__t_sectors_srcunit_tex_aperture_sysmem_op_read_lookup_miss.sum",
                   "syslts__t_sectors_aperture_sysmem_lookup_miss.sum"):
            if mk in d and d[mk].strip():
                ent["sysmem_read_bytes_per_launch"] = float(d[mk].replace(",", "")) * 32
                ent["sysmem_metric"] = mk
                break
        if alg:
            ent["algorithmic_bytes_per_launch"] = float(alg)
        doc[key] = ent
    with open(OUT, "w") as f:
        json.dump(doc, f, indent=1)
        f.write("\n")
    print(json.dumps(doc, indent=1))


if __name__ == "__main__":
    main()
