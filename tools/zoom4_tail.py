"""Config-4 K5 tail analysis: per-voxel cycle counters of the whole slice
(MRFG_ZOOM_STATS_FILE), and the slowest voxels timed ALONE (one voxel per
launch), so the kernel's makespan can be split into single-voxel latency and
co-residency contention.
Usage: python tools/zoom4_tail.py [top_k]
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1506_05393_b200 as P  # noqa: E402
from paper_1506_05393_b200 import workloads as W  # noqa: E402


def main():
    import torch
    top = int(sys.argv[1]) if len(sys.argv) > 1 else 8

    def gpu_sim(s, params):
        with P.Context(s) as c:
            return c.simulate(params, precision=64)

    wl = W.make(4, gpu_sim)
    cfg = P.zoom_config(**W.CONFIG4_ZOOM)
    n, nq = wl.schedule.n, wl.nvox
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    sf = os.path.join(ROOT, "gpurun_out", "zoom4_vstats.bin")
    out = {}

    def timed(c, d_q, k, d_o):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        c.quantify_device(d_q.data_ptr(), k, wl.grid, cfg, d_o.data_ptr())
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    with P.Context(wl.schedule) as c:
        c.set_stream(stream.cuda_stream)
        d_q = torch.from_numpy(wl.fps.view(np.float64).reshape(nq, 2 * n)).to(dev)
        d_o = torch.empty(nq * P.dgs.QUANT_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        timed(c, d_q, nq, d_o)
        out["slice_ms"] = min(timed(c, d_q, nq, d_o) for _ in range(3))
        os.environ["MRFG_ZOOM_STATS"] = "1"
        os.environ["MRFG_ZOOM_STATS_FILE"] = sf
        out["slice_ms_stats"] = timed(c, d_q, nq, d_o)
        rec = d_o.cpu().numpy().view(P.dgs.QUANT_DTYPE).copy()
        vs = np.fromfile(sf, dtype=np.int64).reshape(nq, 4)
        del os.environ["MRFG_ZOOM_STATS"], os.environ["MRFG_ZOOM_STATS_FILE"]
        cyc = vs[:, 0].astype(np.float64)
        ev = rec["evaluations"].astype(np.float64)
        out["cycles_pct"] = {p: float(np.percentile(cyc, p)) for p in (50, 90, 99, 100)}
        out["corr_cycles_evals"] = float(np.corrcoef(cyc, ev)[0, 1])
        out["corr_cycles_exact_rounds"] = float(np.corrcoef(cyc, vs[:, 2])[0, 1])
        out["mean"] = {"cycles": cyc.mean(), "screen_cycles": float(vs[:, 1].mean()),
                       "exact_rounds": float(vs[:, 2].mean()), "exact_cycles": float(vs[:, 3].mean()),
                       "evals": ev.mean()}
        order = np.argsort(-cyc)[:top]
        slow = []
        for v in order:
            d1 = d_q[v:v + 1].contiguous()
            timed(c, d1, 1, d_o)
            ms = min(timed(c, d1, 1, d_o) for _ in range(2))
            slow.append({"voxel": int(v), "cycles": int(cyc[v]), "screen_cycles": int(vs[v, 1]),
                         "exact_rounds": int(vs[v, 2]), "exact_cycles": int(vs[v, 3]), "evals": int(ev[v]),
                         "alone_ms": ms})
        out["slowest"] = slow
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
