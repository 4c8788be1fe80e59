"""One config-4 K5 launch after a warm-up (for ncu captures: -k regex:k_zoom -s 1 -c 1)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1506_05393_b200 as P  # noqa: E402
from paper_1506_05393_b200 import workloads as W  # noqa: E402


def main():
    import torch

    def gpu_sim(s, params):
        with P.Context(s) as c:
            return c.simulate(params, precision=64)

    wl = W.make(4, gpu_sim)
    cfg = P.zoom_config(**W.CONFIG4_ZOOM)
    n, nq = wl.schedule.n, wl.nvox
    dev = torch.device("cuda", 0)
    with P.Context(wl.schedule) as c:
        c.set_stream(torch.cuda.current_stream(dev).cuda_stream)
        d_q = torch.from_numpy(wl.fps.view(np.float64).reshape(nq, 2 * n)).to(dev)
        d_o = torch.empty(nq * P.dgs.QUANT_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        for _ in range(2):
            c.quantify_device(d_q.data_ptr(), nq, wl.grid, cfg, d_o.data_ptr())
        torch.cuda.synchronize()


if __name__ == "__main__":
    main()
