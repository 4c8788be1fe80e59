"""N>1 path on CPU: world_size-2 gloo process group.

Each rank owns one contiguous T1 slab (distributed.grid_shard) / voxel block
(distributed.voxel_shard), computes its part (here with the CPU oracle as the
per-rank compute, since the CUDA kernels need a B200), exchanges through ONE
all_gather, and reduces with distributed.merge_matches -- the host form of the
device merge.  The merged result must equal the single-process reference scan
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


def worker(rank, world, port, out_path):
    import sys
    sys.path.insert(0, ROOT)
    import oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc, s, (t1, t2, df), q = problem()
    slab = t2[2] * df[2]
    fb, fe = D.shard_range(t1[2], slab, world, rank)
    i1b, i1e = fb // slab, fe // slab
    nq = len(q)
    if fe > fb:
        sub = oracle.make_grid((t1[0] + i1b * t1[1], t1[1], i1e - i1b), t2, df)
        f, sc, _ = orc.scan_grid(s, sub, q, threads=1)
        f = f + fb  # local -> global flat
    else:
        f, sc = np.full(nq, -1, np.int64), np.full(nq, -1e300)
    ft = torch.from_numpy(f)
    st = torch.from_numpy(sc)
    fall = [torch.empty_like(ft) for _ in range(world)]
    sall = [torch.empty_like(st) for _ in range(world)]
    dist.all_gather(fall, ft)
    dist.all_gather(sall, st)
    mf, ms = D.merge_matches(torch.stack(fall).numpy(), torch.stack(sall).numpy())
    # voxel-sharded "ZOOM-like" gather: each rank labels its voxel block
    vb, ve = D.voxel_shard(nq, world, rank)
    part = torch.zeros(nq, dtype=torch.int64)
    part[vb:ve] = torch.from_numpy(mf[vb:ve])
    dist.all_reduce(part)
    if rank == 0:
        np.savez(out_path, flat=mf, score=ms, vox=part.numpy())
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
