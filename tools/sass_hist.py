"""Opcode / stall histogram of one kernel from an ncu report's SASS source page.
  python tools/sass_hist.py gpurun_out/x.ncu-rep"""
import csv
import io
import subprocess
import sys
from collections import Counter

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source",
                      "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = rows[2:]
ix, sx, src = (h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)"),
               h.index("Source"))
stall_cols = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
tot_i = sum(int(r[ix] or 0) for r in data)
tot_s = sum(int(r[sx] or 0) for r in data)
print(f"instructions {tot_i}  stall samples {tot_s}")
ci, cs = Counter(), Counter()
for r in data:
    t = r[src].strip().split()
    if not t:
        continue
    op = t[1] if t[0].startswith("@") else t[0]
    op = op.split(".")[0]
    ci[op] += int(r[ix] or 0)
    cs[op] += int(r[sx] or 0)
for op, n in ci.most_common(24):
    print(f"  {op:12s} inst {100 * n / tot_i:5.1f}%  stall-samples {100 * cs[op] / tot_s:5.1f}%")
st = Counter()
for r in data:
    for i in stall_cols:
        try:
            st[h[i]] += int(r[i] or 0)
        except ValueError:
            pass
print("stalls:", ", ".join(f"{k[6:]} {100 * v / tot_s:.1f}%" for k, v in st.most_common(10)))

# per CUDA source line (needs -lineinfo): top lines by stall samples
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
lines, fname = [], ""
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
    elif r and r[0] and r[0] not in ("Line No", "Function Name", "File Path") and len(r) > 7:
        try:
            lines.append((int(r[4] or 0), int(r[7] or 0), fname, r[0], r[1].strip()[:70]))
        except ValueError:
            pass
tot_l = sum(x[0] for x in lines) or 1
tot_li = sum(x[1] for x in lines) or 1
print("top source lines (stall-sample %, instruction %):")
for smp, ins, f, ln, text in sorted(lines, reverse=True)[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"  {100 * smp / tot_l:5.1f}% {100 * ins / tot_li:5.1f}%  {f}:{ln}  {text}")
