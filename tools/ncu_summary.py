"""Summarise an ncu report (read here, no GPU) into profiles/:

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r01/<name>.json [graph=kernel|graph=#idx ...]

Writes the per-kernel metrics we cite (duration, DRAM bytes, DRAM throughput,
registers, occupancy, issue activity, top stall reasons) and updates
profiles/ncu_summary.json {graph: {kernel, dram_bytes, ...}} which bench.py
reads for roofline.traffic.
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {
    "gpu__time_duration.sum": "duration_us",
    "dram__bytes_read.sum": "dram_read_MB",
    "dram__bytes_write.sum": "dram_write_MB",
    "l1tex__m_l1tex2xbar_write_bytes.sum": "sm_to_l2_write_MB",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__cycles_active.max": "sm_active_cycles_max",
    "sm__cycles_elapsed.max": "sm_elapsed_cycles",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "smsp__inst_executed.sum": "warp_instructions",
    "launch__shared_mem_per_block_dynamic": "dyn_smem_B",
}


def rows(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return r[0], r[1], r[2:]


def main():
    report, dest = sys.argv[1], sys.argv[2]
    graph_of = dict(a.split("=") for a in sys.argv[3:])
    h, units, data = rows(report)
    res = []
    scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3,  # -> MB
             "ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}  # -> us
    for r in data:
        rec = {"kernel": r[h.index("Kernel Name")]}
        for k, name in KEYS.items():
            if k in h:
                v = r[h.index(k)].replace(",", "")
                u = units[h.index(k)]
                try:
                    rec[name] = float(v) * (scale.get(u, 1.0) if (name.endswith("_MB") or name.endswith("_us")) else 1.0)
                except ValueError:
                    rec[name] = v
        stalls = []
        for i, name in enumerate(h):
            if "smsp__average_warps_issue_stalled" in name and name.endswith("per_issue_active.ratio"):
                try:
                    stalls.append((float(r[i]), name.split("stalled_")[1].replace("_per_issue_active.ratio", "")))
                except ValueError:
                    pass
        rec["top_stalls"] = [[n, round(v, 2)] for v, n in sorted(stalls, reverse=True)[:4]]
        res.append(rec)
    os.makedirs(os.path.dirname(dest), exist_ok=True)
    with open(dest, "w") as f:
        json.dump(res, f, indent=1)
    summ_path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    summ = json.load(open(summ_path)) if os.path.exists(summ_path) else {}
    for g, kname in graph_of.items():
        # "graph=<kernel name>" (first launch of that name) or "graph=#<launch index>"
        cands = [res[int(kname[1:])]] if kname.startswith("#") else res
        for rec in cands:
            if rec["kernel"] == kname or kname.startswith("#"):
                kname = rec["kernel"]
                summ[g] = {"kernel": kname, "report": os.path.relpath(dest, ROOT),
                           "dram_bytes": int((rec.get("dram_read_MB", 0) + rec.get("dram_write_MB", 0)) * 1e6),
                           "dram_read_bytes": int(rec.get("dram_read_MB", 0) * 1e6),
                           "dram_write_bytes": int(rec.get("dram_write_MB", 0) * 1e6),
                           "sm_to_l2_write_bytes": int(rec.get("sm_to_l2_write_MB", 0) * 1e6),
                           "duration_us_cold": rec.get("duration_us")}
                break
    with open(summ_path, "w") as f:
        json.dump(summ, f, indent=1, sort_keys=True)
    print(json.dumps(res, indent=1)[:3000])


if __name__ == "__main__":
    main()
