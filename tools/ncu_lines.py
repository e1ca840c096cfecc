"""Per-source-line totals (instructions executed, shared wavefronts, stall samples) of
one kernel in an ncu report, grouped by file.  usage: ncu_lines.py report kernel [n]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
f, hdr, lines = "?", None, []
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "File Path":
        f = r[1].rsplit("/", 1)[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0].isdigit():
        lines.append((f, r))
ie = hdr.index("Instructions Executed")
wf = hdr.index("L1 Wavefronts Shared") if "L1 Wavefronts Shared" in hdr else hdr.index("Instructions Executed")
st = hdr.index("Warp Stall Sampling (All Samples)")
g = lambda r, i: float(r[i] or 0)  # noqa: E731
tot = sum(g(r, ie) for _, r in lines) or 1
print(f"total instructions {tot:.0f}")
for fn, r in sorted(lines, key=lambda x: -g(x[1], ie))[:n]:
    print(f"{g(r, ie):8.0f} {100 * g(r, ie) / tot:5.1f}% wf={g(r, wf):7.0f} st={g(r, st):4.0f} "
          f"{fn}:{r[0]:>4} {r[1].strip()[:80]}")
