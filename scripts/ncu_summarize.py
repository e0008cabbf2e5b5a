"""Summarise an `ncu --set full` capture of the step kernels into profiles/<tag>/.

Usage: python scripts/ncu_summarize.py <tag>   (reads gpurun_out/<tag>_prof.ncu-rep)
Writes profiles/<tag>/ncu_full_raw.csv, ncu_summary.txt and refreshes
profiles/fv1_dram_bytes.json (bench.py's roofline.traffic per leaf).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LEAVES = 1.72e6  # config 5 leaves per step (bench.py config.leaves_mean)

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
            unit = rows[1][hdr.index("dram__bytes_read.sum")]
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            dram[short] = (rd * scale, wr * scale)
            lines.append(f"  {'DRAM bytes read / written':<40} {rd} / {wr} {unit}")
        except (KeyError, ValueError):
            pass
        lines.append("")
    with open(os.path.join(out, "ncu_summary.txt"), "w") as f:
        f.write("\n".join(lines) + "\n")
    fv1 = [v for k, v in dram.items() if k.startswith("k_fv1")]
    if fv1:
        rd, wr = fv1[0]
        with open(os.path.join(ROOT, "profiles", "fv1_dram_bytes.json"), "w") as f:
            json.dump({"kernel": "k_fv1", "dram_bytes_per_leaf": (rd + wr) / LEAVES,
                       "source": f"profiles/{tag}/ncu_full_raw.csv (dram__bytes_read.sum + dram__bytes_write.sum of "
                                 f"one ncu --set full k_fv1 launch, N = 1.72 M leaves)"}, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r1")
