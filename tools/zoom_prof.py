import sys
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import numpy as np
import paper_1506_05393_b200 as P
from paper_1506_05393_b200 import workloads
def gpu_sim(s, params):
    with P.Context(s) as c:
        return c.simulate(params, precision=64)
wl = workloads.make(2, gpu_sim, nvox=int(sys.argv[1]))
with P.Context(wl.schedule) as c:
    cfg = P.zoom_config(df_coarse_hz=5.0, omega_hz=82.0)
    q = c.quantify(wl.fps, wl.grid, cfg)
    print("evals", q["evaluations"].mean())
