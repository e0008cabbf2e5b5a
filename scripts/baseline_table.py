"""BASELINE.md §5 table from a round's bench.json + cpu_baselines.json:
python scripts/baseline_table.py profiles/<tag>/<tag>_bench.json profiles/<tag>/<tag>_cpu_baselines.json"""
import json, sys

b = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
c = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
sims = b["sim_runtimes_s"]
rows = [("1 pseudo-2D L8, 2.5 s", "pseudo2d_L8_2.5s", "1_pseudo2d_L8"),
        ("2 humps L9, 100 s", "quiescent_humps_L9_100s", "2_humps_L9"),
        ("3 circular L10 ε=1e-3, 3.5 s", "circular_L10_eps1e-3_3.5s", "3_circular_L10_eps1e-3"),
        ("3 circular L10 ε=1e-2, 3.5 s", "circular_L10_eps1e-2_3.5s", None),
        ("3 circular L10 ε=1e-4, 3.5 s", "circular_L10_eps1e-4_3.5s", None),
        ("4 Monai L10, 22.5 s", "monai_L10_22.5s", "4_monai_L10")]
n = c["nproc"]
print(f"| config | GPU runtime (s) | GPU µs/step | steps | CPU ×1 ms/step (est. runtime s) | CPU ×{n} ms/step (est. runtime s) | GPU / CPU×{n} |")
print("|---|---|---|---|---|---|---|")
for label, sk, ck in rows:
    s = sims[sk]
    us = 1e6 * s["seconds"] / s["steps"]
    if ck:
        c1, cn = c[ck]["threads_1"]["ms_per_step"], c[ck][f"threads_{n}"]["ms_per_step"]
        print(f"| {label} | {s['seconds']:.4f} | {us:.1f} | {s['steps']} | {c1:.2f} ({c1 * s['steps'] / 1e3:.1f}) | "
              f"{cn:.2f} ({cn * s['steps'] / 1e3:.1f}) | {cn * 1e3 / us:.0f}× |")
    else:
        print(f"| {label} | {s['seconds']:.4f} | {us:.1f} | {s['steps']} | — | — | — |")
c5 = c["5_river_L11"]
print(f"| 5 river L11 (fixed step count) | — | {1e3 * b['ms_per_step']:.1f} | — | {c5['threads_1']['ms_per_step']:.1f} | "
      f"{c5[f'threads_{n}']['ms_per_step']:.1f} | {c5[f'threads_{n}']['ms_per_step'] / b['ms_per_step']:.0f}× |")
print()
print(f"Config 5 at N = 1: {b['value']:.3e} adapted-cell updates/s ({1e3 * b['ms_per_step']:.1f} µs/step), "
      f"MRA {1e3 * b['mra_ms_per_step']:.1f} µs/step, FV1 roofline fraction {b['roofline']['frac']:.2f} "
      f"(algorithmic bytes), e2e {b['e2e']['value']:.3e}; wet point {1e3 * b['wet_point']['ms_per_step']:.1f} µs/step.")
