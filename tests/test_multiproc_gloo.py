"""N>1 path on CPU: world_size-2 gloo process group.

Each rank owns one contiguous T1 slab (distributed.grid_shard) / voxel block
(distributed.voxel_shard).  The brute-force test runs the production driver
distributed.scan_grid_distributed itself (seed all_reduce, floored slab
scans, ONE all_gather, merge) over a CPU stub context whose per-rank compute
is the CPU oracle, since the CUDA kernels need a B200.  The merged result must equal the single-process reference scan
bit-for-bit, for any world size.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1506_05393_b200 import distributed as D

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def problem():
    import oracle
    orc = oracle.Oracle("restatement")
    s = orc.build_schedule(48, 7)
    grid = (600, 50, 9), (80, 20, 5), (-20, 10, 5)
    rng = np.random.default_rng(0)
    q = np.stack([orc.add_noise(orc.simulate(s, 0.55 + 0.4 * rng.random(), 0.07 + 0.12 * rng.random(),
                                             40 * rng.random() - 20), 0.002, 80 + k) for k in range(7)])
    return orc, s, grid, q


class StubCtx:
    """CPU stand-in for dgs.Context exposing the device entry points that
    distributed.scan_grid_distributed drives (the CUDA kernels need a B200):
    raw pointers of CPU tensors in, the restatement oracle as the per-rank
    compute.  Seed: exact best over the shard's first T1 row (a valid
    screening seed: a real atom's score); floor: a voxel whose slab best is
    below floor - delta reports flat -1, as the GPU scan does."""

    def __init__(self, orc, sched, n):
        self.orc, self.sched, self.n = orc, sched, n

    @staticmethod
    def _view(ptr, ctype, count):
        import ctypes as C
        return np.ctypeslib.as_array((ctype * count).from_address(ptr))

    def _q(self, ptr, nq):
        import ctypes as C
        return self._view(ptr, C.c_double, nq * 2 * self.n).view(np.complex128).reshape(nq, self.n).copy()

    def _sub(self, grid, fb, fe):
        import oracle
        slab = grid.t2_ms.count * grid.df_hz.count
        a, b = fb // slab, fe // slab
        return oracle.make_grid((grid.t1_ms.min + a * grid.t1_ms.step, grid.t1_ms.step, b - a),
                                (grid.t2_ms.min, grid.t2_ms.step, grid.t2_ms.count),
                                (grid.df_hz.min, grid.df_hz.step, grid.df_hz.count))

    def scan_seed_device(self, grid, q_ptr, nq, seed_ptr, metric="cc", flat_range=(0, 0), opts=None):
        import ctypes as C
        fb, _ = flat_range
        slab = grid.t2_ms.count * grid.df_hz.count
        _, sc, _ = self.orc.scan_grid(self.sched, self._sub(grid, fb, fb + slab), self._q(q_ptr, nq), threads=1)
        self._view(seed_ptr, C.c_float, nq)[:] = sc.astype(np.float32)

    def scan_grid_device(self, grid, q_ptr, nq, out_ptr, metric="cc", flat_range=(0, 0), opts=None):
        import ctypes as C
        fb, fe = flat_range
        f, sc, _ = self.orc.scan_grid(self.sched, self._sub(grid, fb, fe), self._q(q_ptr, nq), threads=1)
        f = f + fb
        if opts is not None and opts.floor_matches:
            floor = self._view(opts.floor_matches, C.c_double, 2 * nq).reshape(nq, 2)[:, 1]
            f = np.where(sc >= np.float32(floor) - 2.5e-3, f, -1)
        out = self._view(out_ptr, C.c_uint8, 16 * nq).view([("flat", np.int64), ("score", np.float64)])
        out["flat"], out["score"] = f, sc
        self.last = (f.copy(), sc.copy())
        return None

    def merge_matches_device(self, in_ptr, nranks, nq, out_ptr):
        import ctypes as C
        rec = self._view(in_ptr, C.c_uint8, 16 * nq * nranks).view([("flat", np.int64), ("score", np.float64)])
        rec = rec.reshape(nranks, nq)
        mf, ms = D.merge_matches(rec["flat"], rec["score"])
        out = self._view(out_ptr, C.c_uint8, 16 * nq).view([("flat", np.int64), ("score", np.float64)])
        out["flat"], out["score"] = mf, ms


def worker(rank, world, port, out_path):
    import sys
    sys.path.insert(0, ROOT)
    import oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc, s, (t1, t2, df), q = problem()
    g = oracle.make_grid(t1, t2, df)
    nq, n = q.shape
    ctx = StubCtx(orc, s, n)
    d_q = torch.from_numpy(np.ascontiguousarray(q).view(np.float64).reshape(nq, 2 * n))
    # the production protocol: seed all_reduce, floored slab scans, ONE all_gather, merge
    merged, _ = D.scan_grid_distributed(ctx, g, d_q, nq)
    m = merged.numpy().view([("flat", np.int64), ("score", np.float64)])
    # some rank's slab had nothing above the global seed for some voxel (the
    # floor did work), unless every voxel's best is on every slab
    lf = torch.from_numpy(ctx.last[0])
    alls = [torch.empty_like(lf) for _ in range(world)]
    dist.all_gather(alls, lf)
    # voxel-sharded "ZOOM-like" gather: each rank labels its voxel block
    vb, ve = D.voxel_shard(nq, world, rank)
    part = torch.zeros(nq, dtype=torch.int64)
    part[vb:ve] = torch.from_numpy(m["flat"][vb:ve].copy())
    dist.all_reduce(part)
    if rank == 0:
        np.savez(out_path, flat=m["flat"], score=m["score"], vox=part.numpy(),
                 floored=int((torch.stack(alls) < 0).sum()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_scan_equals_single_process(tmp_path, world):
    out = str(tmp_path / "res.npz")
    mp.spawn(worker, args=(world, free_port(), out), nprocs=world, join=True)
    r = np.load(out)
    import oracle
    orc, s, (t1, t2, df), q = problem()
    f, sc, _ = orc.scan_grid(s, oracle.make_grid(t1, t2, df), q, threads=1)
    assert np.array_equal(r["flat"], f)
    assert np.array_equal(r["score"], sc)
    assert np.array_equal(r["vox"], f)
    assert r["floored"] > 0  # the global seed pruned some slab's voxels


def test_merge_rule_ties_and_empty_ranks():
    flats = np.array([[5, -1, 9], [3, 4, 9], [7, 2, -1]])
    scores = np.array([[0.9, -1e300, 0.5], [0.9, 0.7, 0.5], [0.8, 0.7, -1e300]])
    f, s = D.merge_matches(flats, scores)
    assert f.tolist() == [3, 2, 9] and s.tolist() == [0.9, 0.7, 0.5]


def test_shards_partition_the_grid():
    for n1, world in ((96, 8), (491, 8), (5, 8), (3, 2)):
        cuts = [D.shard_range(n1, 100, world, r) for r in range(world)]
        assert cuts[0][0] == 0 and cuts[-1][1] == n1 * 100
        assert all(cuts[r][1] == cuts[r + 1][0] for r in range(world - 1))


def zoom_worker(rank, world, port, out_path):
    import sys
    sys.path.insert(0, ROOT)
    import oracle
    from paper_1506_05393_b200 import dgs
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc, s, (t1, t2, df), q = problem()
    g = oracle.make_grid(t1, t2, df)
    cfg = oracle.zoom_cfg(df_coarse_hz=10.0)
    nq = len(q)
    vb, ve = D.voxel_shard(nq, world, rank)
    rec = np.zeros(ve - vb, dtype=dgs.QUANT_DTYPE)
    for k, v in enumerate(range(vb, ve)):  # per-rank compute: the CPU oracle (K5 needs a B200)
        r = orc.quantify(s, g, cfg, q[v])
        rec[k] = (r.i1, r.i2, r.idf, r.t1_ms, r.t2_ms, r.df_hz, r.pd, r.score, r.evaluations)
    local = torch.from_numpy(rec.view(np.uint8).copy())
    full = D.gather_voxel_shards(local, nq, dgs.QUANT_DTYPE.itemsize)
    if rank == 0:
        np.save(out_path, full.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_zoom_voxel_shards_gather(tmp_path, world):
    """ZOOM's N>1 exchange: voxel blocks quantified per rank,
    ONE all_gather of the 72-byte result structs; rank 0 holds every voxel's
    record, identical to the single-process results."""
    import oracle
    from paper_1506_05393_b200 import dgs
    out = str(tmp_path / "zoom.npy")
    mp.spawn(zoom_worker, args=(world, free_port(), out), nprocs=world, join=True)
    got = np.load(out).view(dgs.QUANT_DTYPE)
    orc, s, (t1, t2, df), q = problem()
    g = oracle.make_grid(t1, t2, df)
    cfg = oracle.zoom_cfg(df_coarse_hz=10.0)
    for v in range(len(q)):
        r = orc.quantify(s, g, cfg, q[v])
        assert (got["i1"][v], got["i2"][v], got["idf"][v], got["score"][v], got["evaluations"][v]) == \
               (r.i1, r.i2, r.idf, r.score, r.evaluations)
