import time, sys, json
import numpy as np
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import paper_1506_05393_b200 as P
from paper_1506_05393_b200 import workloads

def gpu_sim(s, params):
    with P.Context(s) as c:
        return c.simulate(params, precision=64)

wl = workloads.make(2, gpu_sim, nvox=int(sys.argv[1]) if len(sys.argv) > 1 else 4096)
res = {}
with P.Context(wl.schedule) as c:
    for coarse in (1.0, 5.0):
        cfg = P.zoom_config(df_coarse_hz=coarse, omega_hz=82.0)
        c.quantify(wl.fps[:64], wl.grid, cfg)
        t = time.perf_counter(); q = c.quantify(wl.fps, wl.grid, cfg); dt = time.perf_counter() - t
        ok = np.mean((q["i1"] == wl.truth[:, 0]) & (q["i2"] == wl.truth[:, 1]) & (q["idf"] == wl.truth[:, 2]))
        res[coarse] = dict(s=dt, vox_per_s=len(wl.fps) / dt, evals=float(np.mean(q["evaluations"])), truth_frac=float(ok))
print(json.dumps(res))
