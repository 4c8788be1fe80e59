import sys, os, json
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_1506_05393_b200 as P
from paper_1506_05393_b200 import workloads
from paper_1506_05393_b200._native import ScanOpts
dev = torch.device("cuda", 0); stream = torch.cuda.current_stream(dev)
def gpu_sim(sched, params):
    with P.Context(sched, 0) as c:
        return c.simulate(params, precision=64)
wl = workloads.make(2, gpu_sim)
g, nq, n = wl.grid, wl.nvox, wl.schedule.n
ctx = P.Context(wl.schedule, 0); ctx.set_stream(stream.cuda_stream)
d_q = torch.from_numpy(wl.fps.view(np.float64).reshape(nq, 2 * n)).to(dev)
d_out = torch.empty(nq * 16, dtype=torch.uint8, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 8):
    flush.fill_(1)
    st = ctx.scan_grid_device(g, d_q.data_ptr(), nq, d_out.data_ptr(), opts=ScanOpts(1e-3, 524288, 0, 0))
    torch.cuda.synchronize()
    print(i, round(st.bloch_ms, 1), round(st.gemm_ms, 1), round(st.rerank_ms, 1), st.reranked, st.candidates, flush=True)
