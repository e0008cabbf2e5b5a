"""Sim runtime (initialise + run() to t_end, warm block cache) of a config
under env variants, each in a fresh process: python scripts/sim_variants.py
<case> <L> [eps]  with VARIANTS="A=1,B=0;C=1" (';' separates variants)."""
import os, subprocess, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if len(sys.argv) > 1 and sys.argv[1] == "--child":
    import time
    from paper_2206_05761_b200 import cases, gpu
    case, L, eps = sys.argv[2], int(sys.argv[3]), float(sys.argv[4])
    fn = getattr(cases, case)
    kw = dict(L=L) if eps <= 0 else dict(L=L, epsilon=eps)
    cfg, h, qx, qy, z = fn(**kw)
    gpu.initialise(cfg, h, qx, qy, z).close()
    best = None
    for _ in range(3):
        t0 = time.perf_counter()
        e = gpu.initialise(cfg, h, qx, qy, z)
        r = e.run()
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
        e.close()
    print(json.dumps({"s": round(best, 4), "steps": r["step"], "us_per_step": round(1e6 * best / r["step"], 1)}))
    sys.exit(0)

case, L = sys.argv[1], sys.argv[2]
eps = sys.argv[3] if len(sys.argv) > 3 else "0"
for v in os.environ.get("VARIANTS", "").split(";"):
    env = dict(os.environ)
    for kv in filter(None, v.split(",")):
        k, val = kv.split("=")
        env[k] = val
    r = subprocess.run([sys.executable, __file__, "--child", case, L, eps], env=env, capture_output=True, text=True)
    print((v or "default").ljust(30), case, L, eps, r.stdout.strip() or r.stderr[-300:])
