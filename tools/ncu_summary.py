"""Summarise an `ncu --set full` report into profiles/: per launch the
duration, DRAM traffic, FP64-pipe / L1 / issue utilisation and the top stall
reasons, plus a JSON with the DRAM bytes per launch of each kernel (bench.py
reads it for roofline.traffic).

usage: python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/rNN/ncu_<tag>
"""
import csv
import io
import json
import re
import subprocess
import sys

METRICS = {
    "duration_us": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "fp64_pipe_active_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "tensor_pipe_active_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "l2_throughput_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "l2_to_l1_read_bytes": "l1tex__m_xbar2l1tex_read_bytes.sum",
    "l1_lsu_wavefronts_pct": "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1_hit_pct": "l1tex__t_sector_pipe_lsu_mem_global_op_ld_hit_rate.pct",
    "issue_active_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
    "achieved_occupancy_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "registers": "launch__registers_per_thread",
    "xu_pipe_pct": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "lsu_pipe_pct": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
}
STALLS = ["long_scoreboard", "wait", "short_scoreboard", "math_pipe_throttle", "barrier",
          "not_selected", "mio_throttle", "lg_throttle", "branch_resolving", "dispatch_stall"]


def to_num(v):
    try:
        return float(v.replace(",", ""))
    except Exception:
        return None


def main(rep, out_prefix):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    recs = []
    for r in rows[2:]:
        name = re.sub(r"\(.*", "", r[col["Kernel Name"]])
        name = re.sub(r"void |ifgf_b200::|<unnamed>::|unnamed>::", "", name)
        rec = {"id": r[col["ID"]], "kernel": name}
        for k, m in METRICS.items():
            if m in col:
                v = to_num(r[col[m]])
                u = units[col[m]]
                if k == "duration_us" and v is not None:
                    v = v * {"ns": 1e-3, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3,
                             "s": 1e6, "second": 1e6}.get(u, 1.0)
                if (k.startswith("dram_") or k.endswith("_bytes")) and v is not None:
                    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
                             "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u, 1)
                    v = v * scale
                rec[k] = v
        for s in STALLS:
            m = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
            if m in col:
                rec[f"stall_{s}"] = to_num(r[col[m]])
        recs.append(rec)
    keys = list(recs[0].keys()) if recs else []
    with open(out_prefix + ".csv", "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=keys)
        w.writeheader()
        w.writerows(recs)
    traffic = {}
    for rec in recs:
        t = (rec.get("dram_read_bytes") or 0) + (rec.get("dram_write_bytes") or 0)
        traffic.setdefault(rec["kernel"], []).append(t)
    summary = {"report": rep, "launches": recs,
               "traffic_bytes_per_launch": {k: sum(v) / len(v) for k, v in traffic.items()}}
    with open(out_prefix + ".json", "w") as f:
        json.dump(summary, f, indent=1)
    for rec in recs:
        print({k: (round(v, 2) if isinstance(v, float) else v) for k, v in rec.items()})


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
