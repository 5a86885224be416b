"""Summarise ncu reports / launch lists into profiles/ (run in the build container).

python tools/ncu_summary.py gpurun_out/prof_batch_r01.ncu-rep --tag batch_r01 --algo-bytes 33924775936 --images 1024
python tools/ncu_summary.py --launches gpurun_out/launches_r01.csv --tag r01
"""
import argparse
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_sector_hit_rate.pct",
    "sm__cycles_elapsed.avg.per_second", "dram__cycles_elapsed.avg.per_second",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_sleeping_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_misc_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")]}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                v = vals[i].replace(",", "")
                try:
                    v = float(v)
                except ValueError:
                    pass
                d[m] = {"value": v, "unit": units[i]}
        res.append(d)
    return res


def to_bytes(v):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return v["value"] * scale.get(v["unit"], 1)


def to_seconds(v):
    scale = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1, "second": 1}
    return v["value"] * scale.get(v["unit"], 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep", nargs="?")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--algo-bytes", type=float, default=None)
    ap.add_argument("--images", type=int, default=1)
    ap.add_argument("--workload", default=None)
    ap.add_argument("--launches", default=None)
    a = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    if a.launches:
        rows = [r for r in csv.reader(open(a.launches)) if len(r) > 10]
        hdr = rows[0]
        ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
        ls = [(r[ki], float(r[vi].replace(",", ""))) for r in rows[1:]]
        tot = {}
        for k, v in ls:
            tot[k] = tot.get(k, 0.0) + v
        s = sum(tot.values())
        summary = {"source": os.path.basename(a.launches), "launches": [{"kernel": k, "ns": v} for k, v in ls],
                   "share": {k: v / s for k, v in tot.items()}}
        json.dump(summary, open(os.path.join(PROF, f"launches_{a.tag}.json"), "w"), indent=1)
        print(json.dumps(summary["share"], indent=1))
    if a.rep:
        res = raw(a.rep)
        for d in res:
            t = to_seconds(d["gpu__time_duration.sum"])
            rd = to_bytes(d["dram__bytes_read.sum"])
            wr = to_bytes(d["dram__bytes_write.sum"])
            d["derived"] = {"duration_s": t, "dram_bytes": rd + wr, "dram_gbs": (rd + wr) / t / 1e9}
            if a.algo_bytes:
                d["derived"]["algorithmic_bytes"] = a.algo_bytes
                d["derived"]["traffic_over_algorithmic"] = (rd + wr) / a.algo_bytes
                d["derived"]["algorithmic_gbs_under_ncu"] = a.algo_bytes / t / 1e9
            d["derived"]["dram_bytes_per_image"] = (rd + wr) / a.images
        json.dump({"source": os.path.basename(a.rep), "kernels": res},
                  open(os.path.join(PROF, f"ncu_{a.tag}.json"), "w"), indent=1)
        for d in res:
            print(d["kernel"], json.dumps(d["derived"]))
        if a.workload:
            p = os.path.join(PROF, "ncu_traffic.json")
            cur = json.load(open(p)) if os.path.exists(p) else {}
            d = res[-1]["derived"]
            cur[a.workload] = {"dram_bytes_per_image": d["dram_bytes_per_image"] if a.images > 1 else None,
                               "dram_bytes_per_launch": d["dram_bytes"],
                               "images_per_launch": a.images,
                               "source": f"profiles/ncu_{a.tag}.json"}
            json.dump(cur, open(p, "w"), indent=1)


if __name__ == "__main__":
    main()
