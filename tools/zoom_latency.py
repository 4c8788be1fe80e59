"""Single-voxel K5 latency (the prior / wavefront mode is a chain of such
latencies): config-4 lattice and steps, k voxels per launch, device-resident
queries, CUDA events; MRFG_ZOOM_STATS=1 adds the kernel's cycle counters.
Usage: python tools/zoom_latency.py [k ...]
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
    ks = [int(a) for a in sys.argv[1:]] or [1, 8, 64]

    def gpu_sim(s, params):
        with P.Context(s) as c:
            return c.simulate(params, precision=64)

    wl = W.make(4, gpu_sim)
    cfg = P.zoom_config(**W.CONFIG4_ZOOM)
    n = wl.schedule.n
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    out = {}
    with P.Context(wl.schedule) as c:
        c.set_stream(stream.cuda_stream)
        d_q = torch.from_numpy(wl.fps[:max(ks)].view(np.float64).reshape(-1, 2 * n)).to(dev)
        d_o = torch.empty(max(ks) * P.dgs.QUANT_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        c.quantify_device(d_q.data_ptr(), max(ks), wl.grid, cfg, d_o.data_ptr())
        for k in ks:
            times = []
            for _ in range(3):
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                c.quantify_device(d_q.data_ptr(), k, wl.grid, cfg, d_o.data_ptr())
                e1.record(stream)
                torch.cuda.synchronize()
                times.append(e0.elapsed_time(e1))
            out[k] = {"ms": float(np.median(times)), "ms_all": [round(t, 2) for t in times]}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
