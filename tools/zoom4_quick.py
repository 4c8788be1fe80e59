"""Config-4 K5 timing (device-resident queries, CUDA events) for the certified
FP32-screening path and the all-FP64 path (MRFG_ZOOM_EPS=-1), plus a
whole-slice comparison of the two maps (answers, scores, evaluation counts).
Set MRFG_ZOOM_STATS=1 for the kernel's per-phase counters on stderr.
Usage: python tools/zoom4_quick.py [nvox] [eps ...]
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
    nq = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    epss = sys.argv[2:] or ["1e-5", "-1"]

    def gpu_sim(s, params):
        with P.Context(s) as c:
            return c.simulate(params, precision=64)

    wl = W.make(4, gpu_sim)
    cfg = P.zoom_config(**W.CONFIG4_ZOOM)
    n = wl.schedule.n
    nq = min(nq, wl.nvox)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    out = {"voxels": nq}
    recs = {}
    with P.Context(wl.schedule) as c:
        c.set_stream(stream.cuda_stream)
        d_q = torch.from_numpy(wl.fps[:nq].view(np.float64).reshape(nq, 2 * n)).to(dev)
        d_o = torch.empty(nq * P.dgs.QUANT_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        for eps in epss:
            os.environ["MRFG_ZOOM_EPS"] = eps
            c.quantify_device(d_q.data_ptr(), nq, wl.grid, cfg, d_o.data_ptr())  # warm (tables)
            torch.cuda.synchronize()
            reps = int(os.environ.get("ZOOM_REPS", "5"))
            times = []
            for _ in range(reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                c.quantify_device(d_q.data_ptr(), nq, wl.grid, cfg, d_o.data_ptr())
                e1.record(stream)
                torch.cuda.synchronize()
                times.append(e0.elapsed_time(e1))
            ms = float(np.median(times))
            rec = d_o.cpu().numpy().view(P.dgs.QUANT_DTYPE).copy()
            recs[eps] = rec
            np.save(os.path.join(ROOT, "gpurun_out", f"zoom4_rec_{eps}.npy"), rec)
            out[eps] = {"ms": ms, "ms_all": [round(t, 1) for t in times], "voxels_per_s": nq / (ms * 1e-3),
                        "evals_per_voxel": float(rec["evaluations"].mean())}
    if len(recs) > 1:
        b = recs[epss[-1]]
        for e in epss[:-1]:
            a = recs[e]
            out[e]["identical_to_" + epss[-1]] = {
                k: int((a[k] == b[k]).sum()) for k in ("i1", "i2", "idf", "evaluations", "score", "pd")}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
