"""Copy the summaries of one tools/gpu_check.sh run into profiles/ (tracked).
Usage: python tools/save_profiles.py gpurun_out/TAG [prefix=r1]"""
import csv
import json
import os
import shutil
import sys

S = sys.argv[1]
pre = sys.argv[2] if len(sys.argv) > 2 else "r1"
P = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles")
for src, dst in (("bench.json", "bench_c2"), ("bench_c3.json", "bench_c3"), ("bench_c4.json", "bench_c4"),
                 ("bench_c1.json", "bench_c1"),
                 ("bench_dispatch.json", "bench_c2_dispatch"), ("bench_ref.json", "bench_reference_arm")):
    if os.path.exists(os.path.join(S, src)):
        shutil.copy(os.path.join(S, src), os.path.join(P, f"{pre}_{dst}.json"))
shutil.copy(os.path.join(S, "full_summary.json"), os.path.join(P, f"{pre}_ncu_c2_kernels.json"))
for extra in ("timeline_c2.txt", "pytest_gpu.log", "smoke.log", "reference_python_host.jsonl"):
    if os.path.exists(os.path.join(S, extra)):
        shutil.copy(os.path.join(S, extra), os.path.join(P, f"{pre}_{extra}"))
for k in ("k_pack_bulk", "k_pack_stream", "k_histogram", "k_sort_pass", "k_dispatch", "k_size_next", "k_chain_walk"):
    f = os.path.join(S, f"src_{k}.txt")
    if os.path.exists(f):
        shutil.copy(f, os.path.join(P, f"{pre}_ncu_src_{k}.txt"))
rows = list(csv.reader(open(os.path.join(S, "launches.csv"))))
out, hdr = [], None
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        out.append([d["ID"], d["Kernel Name"].split("(")[0], d["Grid Size"], d["Block Size"], d["Metric Value"]])
with open(os.path.join(P, f"{pre}_launches_c2.csv"), "w", newline="") as f:
    w = csv.writer(f)
    w.writerow(["id", "kernel", "grid", "block", "gpu__time_duration.sum_ns"])
    w.writerows(out)
full = json.load(open(os.path.join(S, "full_summary.json")))
summ = {"note": "per-launch DRAM bytes and duration from `ncu --set full --clock-control none` "
                "(tools/gpu_check.sh: stage_profile.py --config c2 --steps 1); all kernels in "
                f"{pre}_ncu_c2_kernels.json"}
for e in full:
    k = e["kernel"].replace("void ", "").split("<")[0]
    ent = {"dram_bytes": e.get("dram_bytes"), "dram_read": e.get("dram_read"),
           "dram_write": e.get("dram_write"), "duration_us": e.get("duration_us")}
    if k == "k_histogram":
        ent.update(smem_atom_inst=e.get("smem_atom_inst"), gmem_atom_accesses=e.get("gmem_atom_accesses"))
    summ.setdefault(k, {}).setdefault("c2", ent)
for c in ("c1", "c3", "c4"):  # pack launches of the other configs (gpu_check.sh)
    f = os.path.join(S, f"pack_traffic_{c}.csv")
    if not os.path.exists(f):
        continue
    rows = [r for r in csv.reader(open(f)) if len(r) > 10 and r[0] != "" and not r[0].startswith("{")]
    if not rows or rows[0][0] != "ID":
        continue
    hdr, m = rows[0], {}
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        k = d["Kernel Name"].replace("void ", "").split("(")[0].split("<")[0].replace("bsk::", "")
        m.setdefault(k, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    for k, v in m.items():
        rd, wr = v.get("dram__bytes_read.sum", 0.0), v.get("dram__bytes_write.sum", 0.0)
        summ.setdefault(k, {})[c] = {"dram_bytes": rd + wr, "dram_read": rd, "dram_write": wr,
                                     "duration_us": v.get("gpu__time_duration.sum", 0.0) / 1e3}
json.dump(summ, open(os.path.join(P, "ncu_summary.json"), "w"), indent=1)
print(f"{len(out)} launches; kernels: {sorted(summ)}")
