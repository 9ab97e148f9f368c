"""Reduce tools/ncu_kernels.sh captures to one table (dev tool).

    python tools/ncu_table.py <dir with ncu_<w>.csv and prof_<w>.json> [--json out.json]

Per (workload, kernel): launches, mean duration, DRAM read/write per launch,
DRAM GB/s, L2 hit rate, warp instructions (and per nonzero for the variant
kernels), issue-active and warps-active percentages, registers, thread
efficiency, SHFL share of the executed warp instructions.  For the dominant
launch of each workload (the variant kernel) also the algorithmic bytes
(rowPtr + colIdx/val + X once + Y), its achieved GB/s and fraction of the
measured HBM peak, and the X L2 hit rate of SURVEY §5:
    1 - (DRAM read - A bytes) / (gathered X bytes = nnz * 4N).
"""
import csv
import glob
import json
import os
import re
import sys
from collections import defaultdict


def num(v):
    try:
        return float(str(v).split(" ")[0].replace(",", ""))
    except ValueError:
        return None


def opcode_counts(v):
    out = {}
    for op, c in re.findall(r"([A-Z][A-Z0-9_.]*)\s*[:=]\s*([\d,.]+)", str(v)):
        out[op] = out.get(op, 0.0) + float(c.replace(",", ""))
    return out


def load(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        rows.append(r)
    launches = defaultdict(dict)
    for r in rows:
        lid = r["ID"]
        launches[lid]["kernel"] = r["Kernel Name"]
        launches[lid][r["Metric Name"]] = (r["Metric Value"], r.get("Metric Unit", ""))
    return launches


def short(name):
    name = re.sub(r"\(.*$", "", name)
    name = name.replace("spmk_dev::", "")
    return name[:60]


def main():
    d = sys.argv[1]
    peak = 6547.5
    try:
        peak = float(json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..",
                                                 "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        pass
    table = []
    for path in sorted(glob.glob(os.path.join(d, "ncu_*.csv"))):
        w = os.path.basename(path)[4:-4]
        meta = {}
        mp = os.path.join(d, f"prof_{w}.json")
        if os.path.exists(mp):
            meta = json.load(open(mp))
        L = load(path)
        per = defaultdict(list)
        for lid, m in L.items():
            per[m["kernel"]].append(m)
        if not per:
            continue
        agg = []
        for k, ms in per.items():
            def mean(key, scale=1.0):
                vals = [num(m[key][0]) for m in ms if key in m and num(m[key][0]) is not None]
                return sum(vals) / len(vals) * scale if vals else None
            dur_ns = mean("gpu__time_duration.sum")
            unit = next((m["gpu__time_duration.sum"][1] for m in ms if "gpu__time_duration.sum" in m), "ns")
            dur_us = dur_ns / 1000.0 if unit in ("ns", "nsecond") else (dur_ns if unit in ("us", "usecond") else dur_ns * 1e3)
            def bytes_of(key):
                v = mean(key)
                u = next((m[key][1] for m in ms if key in m), "byte")
                f = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u, 1)
                return v * f if v is not None else None
            rd, wr = bytes_of("dram__bytes_read.sum"), bytes_of("dram__bytes_write.sum")
            ops = defaultdict(float)
            for m in ms:
                if "sass__inst_executed_per_opcode" in m:
                    for op, c in opcode_counts(m["sass__inst_executed_per_opcode"][0]).items():
                        ops[op] += c / len(ms)
            inst = mean("smsp__inst_executed.sum")
            shfl = sum(c for op, c in ops.items() if op.startswith("SHFL"))
            agg.append({
                "workload": w, "kernel": short(k), "launches": len(ms), "us": round(dur_us, 2),
                "dram_read_MB": round(rd / 1e6, 2) if rd is not None else None,
                "dram_write_MB": round(wr / 1e6, 2) if wr is not None else None,
                "dram_GBps": round((rd + wr) / (dur_us * 1e-6) / 1e9, 1) if rd is not None and dur_us else None,
                "l2_hit_pct": round(mean("lts__t_sector_hit_rate.pct"), 1) if mean("lts__t_sector_hit_rate.pct") is not None else None,
                "warp_inst": inst, "issue_active_pct": mean("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                "warps_active_pct": mean("sm__warps_active.avg.pct_of_peak_sustained_active"),
                "regs": mean("launch__registers_per_thread"),
                "thread_eff": (mean("smsp__thread_inst_executed_per_inst_executed.ratio") or 0) / 32.0,
                "shfl_share": round(shfl / inst, 4) if inst and ops else None,
                "fp32x2": {op: round(c) for op, c in ops.items() if op in ("FMUL2", "FFMA2", "FADD2")},
            })
        agg.sort(key=lambda r: -r["us"])
        dom = agg[0]
        if meta:
            alg = meta["a_bytes"] + meta["x_bytes"] + meta["y_bytes"]
            dom["dominant"] = True
            dom["alg_bytes"] = alg
            dom["alg_GBps"] = round(alg / (dom["us"] * 1e-6) / 1e9, 1)
            dom["hbm_frac"] = round(dom["alg_GBps"] / peak, 4)
            if dom["dram_read_MB"] is not None:
                dom["x_l2_hit"] = round(1.0 - (dom["dram_read_MB"] * 1e6 - meta["a_bytes"]) / meta["x_gather_bytes"], 4)
            if dom["warp_inst"]:
                dom["inst_per_nnz"] = round(dom["warp_inst"] / meta["nnz"], 2)
            dom["matrix"] = meta.get("matrix")
            dom["n"] = meta.get("n")
        table += agg
    if "--json" in sys.argv:
        json.dump(table, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
    cols = ["workload", "kernel", "launches", "us", "dram_read_MB", "dram_write_MB", "dram_GBps", "l2_hit_pct",
            "alg_GBps", "hbm_frac", "x_l2_hit", "inst_per_nnz", "issue_active_pct", "warps_active_pct", "regs",
            "thread_eff", "shfl_share"]
    print("| " + " | ".join(cols) + " |")
    print("|" + "---|" * len(cols))
    for r in table:
        def f(v):
            if v is None:
                return ""
            if isinstance(v, float):
                return f"{v:.3g}" if abs(v) < 1000 else f"{v:.0f}"
            return str(v)
        print("| " + " | ".join(f(r.get(c)) for c in cols) + " |")


if __name__ == "__main__":
    main()
