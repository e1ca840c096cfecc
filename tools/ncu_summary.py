"""Summarise an ncu --set full report: per kernel duration, DRAM bytes/throughput,
occupancy, top stall reasons.  Usage: python tools/ncu_summary.py report.ncu-rep [--json out]"""
import csv
import io
import json
import subprocess
import sys

METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum": "smem_atom_wavefronts",
    "l1tex__t_set_accesses_pipe_lsu_mem_global_op_atom.sum": "gmem_atom_accesses",
    "smsp__inst_executed_op_shared_atom.sum": "smem_atom_inst",
    "sm__sass_inst_executed_op_shared_atom.sum": "smem_atom_sass",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
}


def to_bytes(v, u):
    f = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "B": 1,
             "KB": 1e3, "MB": 1e6, "GB": 1e9}
    return f * scale.get(u, 1)


def to_ns(v, u):
    f = float(v.replace(",", ""))
    return f * {"nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6,
                "ms": 1e6}.get(u, 1)


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        e = {"kernel": d["Kernel Name"].split("(")[0]}
        for m, k in METRICS.items():
            if m in d and d[m] not in ("", "n/a"):
                if k.startswith("dram_r") or k.startswith("dram_w"):
                    e[k] = to_bytes(d[m], u[m])
                elif k == "duration":
                    e[k + "_us"] = to_ns(d[m], u[m]) / 1e3
                else:
                    try:
                        e[k] = float(d[m].replace(",", ""))
                    except ValueError:
                        e[k] = d[m]
        stalls = []
        for h in hdr:
            if h.startswith("smsp__average_warp_latency_issue_stalled_") and h.endswith("_per_warp_active.ratio"):
                pass
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    stalls.append((float(d[h].replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        tot = sum(s for s, _ in stalls) or 1
        e["top_stalls"] = [(n, round(100 * s / tot, 1)) for s, n in stalls[:5]]
        if "dram_read" in e:
            e["dram_bytes"] = e["dram_read"] + e.get("dram_write", 0)
            e["dram_gbs"] = e["dram_bytes"] / (e["duration_us"] * 1e3)
        res.append(e)
    for e in res:
        print(json.dumps(e))
    if len(sys.argv) > 3 and sys.argv[2] == "--json":
        with open(sys.argv[3], "w") as fh:
            json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
