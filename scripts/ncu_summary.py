"""Summarise ncu captures of the K1 kernel into profiles/ (run in the build container).

    python scripts/ncu_summary.py --round r01 gpurun_out/prof_r01_c4.ncu-rep:c4:1024 ...

Each argument is REPORT:CONFIG:ROWS[:PREC] (ROWS = window rows the capture launched,
0 = all; PREC = fp32 / fp64, default the config's precision).  Writes
profiles/ncu_<round>.md (human table) and merges the numbers into
profiles/ncu_summary.json under "<config>/<prec>" (read by bench.py for
roofline.traffic when a full-launch capture of that config AND precision exists).
"""
import argparse
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1707_08213_b200.workloads import CONFIGS  # noqa: E402

METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "dram__bytes_write.sum.per_second": "dram_write_rate",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "launch__registers_per_thread": "regs",
    "launch__block_size": "block",
    "launch__grid_size": "grid",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio": "stall_long_sb",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio": "stall_barrier",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio": "stall_short_sb",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio": "stall_lg_throttle",
}
SCALE = {"nsecond": 1e-9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9,
         "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "byte/second": 1, "Gbyte/second": 1e9, "Tbyte/second": 1e12, "Mbyte/second": 1e6,
         "byte/s": 1, "Mbyte/s": 1e6, "Gbyte/s": 1e9, "Tbyte/s": 1e12,
         "hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9}


def read_raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {}
        for i, h in enumerate(hdr):
            if h in METRICS and vals[i] != "":
                v = float(vals[i].replace(",", ""))
                d[METRICS[h]] = v * SCALE.get(units[i], 1.0)
        d["kernel"] = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else ""
        res.append(d)
    return res


def traffic_table(paths):
    """Single-pass `ncu --metrics dram__bytes_*` CSVs (TRAFFIC_CSV:CONFIG) of full launches."""
    rows = ["", "## Full-launch DRAM traffic (single-pass `ncu --metrics "
            "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum`)", "",
            "| config | launch | duration ms | alg GB | dram read GB | dram write GB | traffic/alg | "
            "write TB/s |", "|---|---|---|---|---|---|---|---|"]
    per_cfg = {}
    for spec in paths:
        path, name, *pp = spec.split(":")
        cfg = CONFIGS[name]
        prec = pp[0] if pp else cfg.precision
        lines = [l for l in open(path) if not l.startswith("==")]
        per = {}
        for row in csv.DictReader(lines):
            v = float(row["Metric Value"].replace(",", "")) * SCALE.get(row["Metric Unit"], 1.0)
            per.setdefault(int(row["ID"]), {})[row["Metric Name"]] = v
        alg = cfg.algorithmic_bytes(precision=prec)
        for i, (_, m) in enumerate(sorted(per.items())):
            rd, wr = m["dram__bytes_read.sum"], m["dram__bytes_write.sum"]
            du = m["gpu__time_duration.sum"]
            rows.append(f"| {name} {prec} | {i} | {du * 1e3:.3f} | {alg / 1e9:.3f} | {rd / 1e9:.4f} | "
                        f"{wr / 1e9:.3f} | {(rd + wr) / alg:.4f} | "
                        f"{m.get('dram__bytes_write.sum.per_second', wr / du) / 1e12:.2f} |")
            per_cfg[f"{name}/{prec}"] = {"dram_bytes_per_launch": rd + wr,
                                         "full_launch_duration_s": du}
    return rows, per_cfg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", required=True)
    ap.add_argument("--traffic", nargs="*", default=[], help="TRAFFIC_CSV:CONFIG")
    ap.add_argument("captures", nargs="+")
    a = ap.parse_args()
    summ_path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    summ = json.load(open(summ_path)) if os.path.exists(summ_path) else {}
    lines = [f"# ncu captures, round {a.round[1:]}", "",
             "K1 (`k1_stream_kernel`), `ncu --set full --clock-control none`, one launch per row. "
             "`alg` = algorithmic bytes of that launch (coefficients written + input rows read); "
             "`traffic` = dram__bytes_read.sum + dram__bytes_write.sum.", "",
             "| config | rows | duration ms | alg GB | traffic GB | traffic/alg | DRAM write TB/s | "
             "DRAM % peak | SM % | issue % | FMA pipe % | regs | block x grid | warps active % | "
             "stall long-sb / barrier / short-sb (per issue) |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for spec in a.captures:
        rep, name, rows, *pp = spec.split(":")
        cfg = CONFIGS[name]
        prec = pp[0] if pp else cfg.precision
        rows = int(rows) or cfg.P0
        for d in read_raw(rep):
            alg = cfg.algorithmic_bytes(rows=rows, precision=prec)
            traffic = d.get("dram_read", 0) + d.get("dram_write", 0)
            lines.append(
                f"| {name} {prec} | {rows} | {d['duration']*1e3:.3f} | {alg/1e9:.3f} | {traffic/1e9:.3f} | "
                f"{traffic/alg:.4f} | {d.get('dram_write_rate', 0)/1e12:.2f} | "
                f"{d.get('dram_pct_of_peak', 0):.1f} | {d.get('sm_pct', 0):.1f} | "
                f"{d.get('issue_pct', 0):.1f} | {d.get('fma_pipe_pct', 0):.1f} | {d.get('regs', 0):.0f} | "
                f"{d.get('block', 0):.0f} x {d.get('grid', 0):.0f} | {d.get('occupancy_pct', 0):.1f} | "
                f"{d.get('stall_long_sb', 0):.2f} / {d.get('stall_barrier', 0):.2f} / "
                f"{d.get('stall_short_sb', 0):.2f} |")
            e = summ.setdefault(f"{name}/{prec}", {})
            e.update({"round": a.round, "capture_rows": rows, "duration_s": d["duration"],
                      "alg_bytes": alg, "traffic_bytes": traffic, "traffic_over_alg": traffic / alg})
            if rows == cfg.P0:
                e["dram_bytes_per_launch"] = traffic
    if a.traffic:
        trows, per_cfg = traffic_table(a.traffic)
        lines += trows
        for name, d in per_cfg.items():
            summ.setdefault(name, {}).update(d)
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    lines += ["", f"Notes on these captures: `ncu_{a.round}_notes.md` (when present)."]
    with open(os.path.join(ROOT, "profiles", f"ncu_{a.round}.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(summ_path, "w") as f:
        json.dump(summ, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
