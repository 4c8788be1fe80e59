"""Config-4 neighbour-seeded slices (K5 row kernel): quantify_slice with the
reference's strict raster prior (use_prior 1) and the row relaxation (2);
wall time of the host API, evaluations, and identity of the maps against a
second run with MRFG_ZOOM_PIT toggled when --compare is given.
Usage: python tools/zoom4_prior.py [modes...]   (default: 2 1)"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1506_05393_b200 as P  # noqa: E402
from paper_1506_05393_b200 import workloads as W  # noqa: E402


def main():
    modes = [int(a) for a in sys.argv[1:]] or [2, 1]

    def gpu_sim(s, params):
        with P.Context(s) as c:
            return c.simulate(params, precision=64)

    wl = W.make(4, gpu_sim)
    cfg = P.zoom_config(**W.CONFIG4_ZOOM)
    mask = np.ones(wl.nvox, np.uint8)
    out = {"pit": os.environ.get("MRFG_ZOOM_PIT", "1")}
    with P.Context(wl.schedule) as c:
        c.quantify_slice(wl.fps[:64], mask[:64], 64, 1, wl.grid, cfg, use_prior=2)  # tables, scratch
        for m in modes:
            t0 = time.perf_counter()
            q, _ = c.quantify_slice(wl.fps, mask, wl.nx, wl.ny, wl.grid, cfg, use_prior=m)
            s = time.perf_counter() - t0
            np.save(os.path.join(ROOT, "gpurun_out", f"prior{m}_pit{out['pit']}.npy"), q)
            out[f"use_prior_{m}"] = {"seconds": s, "evals_per_voxel": float(q["evaluations"].mean())}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
