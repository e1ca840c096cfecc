"""Top CUDA source lines by warp-stall samples / instructions for one kernel of an ncu
report (needs -lineinfo).  Usage: python tools/ncu_source.py report.ncu-rep kernel_regex [n]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
lines = []
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0] not in ("", "-"):
        lines.append(r)
if not lines:
    print(out[:1500])
    sys.exit()
i_st = hdr.index("Warp Stall Sampling (All Samples)")
i_ie = hdr.index("Instructions Executed")
tot = sum(float(r[i_st] or 0) for r in lines) or 1
lines.sort(key=lambda r: -float(r[i_st] or 0))
for r in lines[:n]:
    print(f"{100 * float(r[i_st] or 0) / tot:5.1f}%  L{r[0]:>5} inst={r[i_ie]:>10}  {r[1][:100]}")
