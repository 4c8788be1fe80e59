import sys, time, json
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import numpy as np
import paper_1506_05393_b200 as P
from paper_1506_05393_b200 import workloads
res = {}
for n in (1000, 250, 100):
    def gpu_sim(s, params):
        with P.Context(s) as c:
            return c.simulate(params, precision=64)
    wl = workloads.make(2, gpu_sim, nvox=4096, n=n)
    with P.Context(wl.schedule) as c:
        cfg = P.zoom_config(df_coarse_hz=5.0, omega_hz=82.0)
        c.quantify(wl.fps[:64], wl.grid, cfg)
        t = time.perf_counter(); q = c.quantify(wl.fps, wl.grid, cfg); dt = time.perf_counter() - t
        res[n] = dict(s=round(dt, 4), evals=float(q["evaluations"].mean()))
print(json.dumps(res))
