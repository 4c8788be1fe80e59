"""Per-off-resonance subspace screening (MRFG_SUBSPACE=r) against the
full-length screening (MRFG_SUBSPACE=0) on the same queries: best atoms and exact scores must be
identical; prints both scans' statistics (times, candidates, audit errors).
Usage: python tools/subspace_check.py [config] [rank ...]
"""
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
    config = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    ranks = [int(a) for a in sys.argv[2:]] or [32]

    def gpu_sim(s, params):
        with P.Context(s) as c:
            return c.simulate(params, precision=64)

    wl = W.make(config, gpu_sim)
    out = {"config": config, "voxels": int(wl.nvox), "atoms": int(P.grid_total(wl.grid))}
    keys = ("total_ms", "bloch_ms", "project_ms", "gemm_ms", "rerank_ms", "candidates", "reranked",
            "screen_err_audit_max", "screen_err_max", "delta_used", "rescans", "subspace_rank",
            "subspace_residual_max", "subspace_residual_device", "chunks")
    with P.Context(wl.schedule) as c:
        os.environ["MRFG_SUBSPACE"] = "0"  # full-length screening
        c.scan_grid(wl.grid, wl.fps[:64])  # tables, warm
        f0, s0, st0 = c.scan_grid(wl.grid, wl.fps)
        out["default"] = {k: getattr(st0, k) for k in keys}
        for r in ranks:
            os.environ["MRFG_SUBSPACE"] = str(r)
            t0 = time.perf_counter()
            c.scan_grid(wl.grid, wl.fps[:64])  # bases, warm
            t_first = time.perf_counter() - t0
            f1, s1, st1 = c.scan_grid(wl.grid, wl.fps)
            d = {k: getattr(st1, k) for k in keys}
            d["first_call_s_incl_bases"] = t_first
            d["same_flat"] = int((f0 == f1).sum())
            d["same_score"] = int((s0 == s1).sum())
            out[f"rank{r}"] = d
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
