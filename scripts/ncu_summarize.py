"""Summarise an `ncu --set full` capture of the step kernels into profiles/<tag>/.

Usage: python scripts/ncu_summarize.py <tag>   (reads gpurun_out/<tag>_prof.ncu-rep)
Writes profiles/<tag>/ncu_full_raw.csv, ncu_summary.txt and refreshes
profiles/ncu_kernels.json (per kernel: DRAM bytes and FP64 issue of one
launch — bench.py's roofline.traffic and fp64 fractions).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

ROWS = [
    ("Duration", "gpu__time_duration.sum", "us"),
    ("DRAM Throughput", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "%"),
    ("Issue Slots Busy", "sm__inst_issued.avg.pct_of_peak_sustained_active", "%"),
    ("Achieved Occupancy", "sm__warps_active.avg.pct_of_peak_sustained_active", "%"),
    ("Registers Per Thread", "launch__registers_per_thread", ""),
    ("L1/TEX Hit Rate", "l1tex__t_sector_hit_rate.pct", "%"),
    ("L2 Hit Rate", "lts__t_sector_hit_rate.pct", "%"),
    ("Warp Cycles Per Issued Instruction", "smsp__average_warp_latency_per_inst_issued.ratio", "cycle"),
    ("FP64 pipe (avg / max SM)", ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
                                  "sm__inst_executed_pipe_fp64.max.pct_of_peak_sustained_active"), "%"),
    ("SM active cycles (avg / max / min)", ("sm__cycles_active.avg", "sm__cycles_active.max",
                                            "sm__cycles_active.min"), ""),
    ("Grid Size", "launch__grid_size", ""),
]


def main(tag):
    rep = os.path.join(ROOT, "gpurun_out", f"{tag}_prof.ncu-rep")
    out = os.path.join(ROOT, "profiles", tag)
    os.makedirs(out, exist_ok=True)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    with open(os.path.join(out, "ncu_full_raw.csv"), "w") as f:
        f.write(raw)
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, data = rows[0], rows[2:]
    lines = [f"ncu --set full (cold, serialised, one launch each) of the steady-state step kernels, "
             f"L = 11 river flood ({tag})", ""]
    dram = {}
    for r in data:
        d = dict(zip(hdr, r))
        name = d.get("Kernel Name", "?")
        short = name.split("(")[0].replace("void ", "").replace("hwfv1::", "")
        lines.append(f"[{d.get('ID', '?')}] {short}")
        for label, key, unit in ROWS:
            if isinstance(key, tuple):
                val = " / ".join(d.get(k, "n/a") for k in key)
            else:
                val = d.get(key, "n/a")
            lines.append(f"  {label:<40} {val} {unit}".rstrip())
        try:
            rd = float(d["dram__bytes_read.sum"].replace(",", ""))
            wr = float(d["dram__bytes_write.sum"].replace(",", ""))
            sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            ur = sc.get(rows[1][hdr.index("dram__bytes_read.sum")], 1)
            uw = sc.get(rows[1][hdr.index("dram__bytes_write.sum")], 1)  # (ncu picks each column's unit)
            dram[short] = (rd * ur, wr * uw)
            lines.append(f"  {'DRAM bytes read / written':<40} {rd * ur / 1e6:.3f} / {wr * uw / 1e6:.3f} Mbyte")
        except (KeyError, ValueError):
            pass
        lines.append("")
    with open(os.path.join(out, "ncu_summary.txt"), "w") as f:
        f.write("\n".join(lines) + "\n")
    # per-kernel DRAM bytes and FP64 issue of one launch each (bench.py's
    # roofline.traffic / kernels[*].dram_*, fp64 fraction)
    per = {}
    for r in data:
        d = dict(zip(hdr, r))
        short = d.get("Kernel Name", "?").split("(")[0].replace("void ", "").replace("hwfv1::", "")
        base = short.split("<")[0]
        if base in per:
            continue
        try:
            def num(k):
                v = d[k].replace(",", "")
                u = rows[1][hdr.index(k)]
                return float(v) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6,
                                   "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9}.get(u, 1)
            dur = num("gpu__time_duration.sum")
            ent = {"kernel": short, "duration_s": dur,
                   "dram_bytes": num("dram__bytes_read.sum") + num("dram__bytes_write.sum")}
            f64 = 0.0
            for op in ("dadd", "dmul", "dfma"):
                k = f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum.per_cycle_elapsed"
                if k in d and d[k] not in ("", "n/a"):
                    f64 += float(d[k].replace(",", ""))
            ent["fp64_thread_inst_per_smsp_cycle"] = f64
            ent["fp64_pipe_pct_active"] = float(d.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "nan"))
            ent["issue_pct"] = float(d.get("sm__inst_issued.avg.pct_of_peak_sustained_active", "nan"))
            per[base] = ent
        except (KeyError, ValueError):
            continue
    with open(os.path.join(ROOT, "profiles", "ncu_kernels.json"), "w") as f:
        json.dump({"source": f"profiles/{tag}/ncu_full_raw.csv (one ncu --set full launch each, cold, serialised)",
                   "kernels": per}, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r1")
