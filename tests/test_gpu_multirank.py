"""The N>1 protocol with the REAL kernels: two processes, each with its own
context on the box's one GPU, a gloo process group (NCCL needs one GPU per
rank), run distributed.scan_grid_distributed (seed pass + all_reduce(MAX) of
the screening floors, floored T1-slab scans K1 -> K2 -> K3, one all_gather,
k_merge) and distributed.quantify_distributed (voxel blocks + one
all_gather).  The ranks' kernels never wait on each other -- only the
host-side collectives synchronise them -- so sharing a GPU changes timing,
not results: the merged answers must equal a single-process scan and
quantify bit for bit (identical for any world size)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    import paper_1506_05393_b200 as P
    from paper_1506_05393_b200 import workloads

    def gpu_sim(s, params):
        with P.Context(s) as c:
            return c.simulate(params, precision=64)
    wl = workloads.make(1, gpu_sim, nvox=96)
    return wl


def _worker(rank, world, port, out):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    import paper_1506_05393_b200 as P
    from paper_1506_05393_b200 import distributed as D
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    wl = _problem()
    nq, n = wl.fps.shape
    dev = torch.device("cuda", 0)
    with P.Context(wl.schedule, 0) as ctx:
        d_q = torch.from_numpy(wl.fps.view(np.float64).reshape(nq, 2 * n)).to(dev)
        merged, _ = D.scan_grid_distributed(ctx, wl.grid, d_q, nq)
        m = merged.cpu().numpy().view([("flat", np.int64), ("score", np.float64)]).copy()
        cfg = P.zoom_config(df_coarse_hz=5.0, omega_hz=82.0)
        z = D.quantify_distributed(ctx, wl.grid, cfg, d_q, nq).cpu().numpy().view(P.dgs.QUANT_DTYPE).copy()
        torch.cuda.synchronize()
    if rank == 0:
        np.savez(out, flat=m["flat"], score=m["score"], zi1=z["i1"], zi2=z["i2"], zidf=z["idf"], zs=z["score"],
                 ze=z["evaluations"])
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_multirank_scan_and_zoom_equal_single_process(tmp_path, world):
    import torch.multiprocessing as mp
    import paper_1506_05393_b200 as P
    out = str(tmp_path / "r.npz")
    mp.spawn(_worker, args=(world, _port(), out), nprocs=world, join=True)
    r = np.load(out)
    wl = _problem()
    with P.Context(wl.schedule) as c:
        f, s, _ = c.scan_grid(wl.grid, wl.fps)
        q = c.quantify(wl.fps, wl.grid, P.zoom_config(df_coarse_hz=5.0, omega_hz=82.0))
    np.testing.assert_array_equal(r["flat"], f)
    np.testing.assert_array_equal(r["score"], s)
    for a, b in (("zi1", "i1"), ("zi2", "i2"), ("zidf", "idf"), ("zs", "score"), ("ze", "evaluations")):
        np.testing.assert_array_equal(r[a], q[b])
