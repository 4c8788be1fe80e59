"""Multi-GPU data parallelism for the DGS path.

One process per GPU.  Brute force shards the ATOMS: contiguous T1-major slabs
of the flat lattice, so every rank simulates and matches only its own atoms
and the reduction order of every score stays intact (K is never split).  The
per-voxel (flat, score) pairs of all ranks meet in ONE all_gather (NCCL over
NVLink on GPUs, gloo in the CPU tests) and are reduced with the reference's
rule: highest score, lowest flat on ties (dictionary.cpp:291-294).  ZOOM
shards the VOXELS (independent without priors) and gathers the result rows.
Results are identical for any number of ranks.
"""
from __future__ import annotations

import numpy as np

MATCH_DTYPE = np.dtype([("flat", np.int64), ("score", np.float64)])


def shard_range(n1: int, slab_atoms: int, world: int, rank: int) -> tuple[int, int]:
    """Flat range [begin, end) of rank's T1 slab: rows i1 in [n1*r/W, n1*(r+1)/W)."""
    a = n1 * rank // world
    b = n1 * (rank + 1) // world
    return a * slab_atoms, b * slab_atoms


def grid_shard(grid, world: int, rank: int) -> tuple[int, int]:
    return shard_range(grid.t1_ms.count, grid.t2_ms.count * grid.df_hz.count, world, rank)


def voxel_shard(nvox: int, world: int, rank: int) -> tuple[int, int]:
    return nvox * rank // world, nvox * (rank + 1) // world


def merge_matches(flats: np.ndarray, scores: np.ndarray):
    """Host form of the C1 reduction (k_merge in rerank.cu): (ranks, nq) -> (nq,).

    Ranks without atoms report flat -1 and are skipped."""
    flats = np.asarray(flats)
    scores = np.asarray(scores)
    best_f = flats[0].copy()
    best_s = scores[0].copy()
    for r in range(1, flats.shape[0]):
        f, s = flats[r], scores[r]
        take = (f >= 0) & ((best_f < 0) | (s > best_s) | ((s == best_s) & (f < best_f)))
        best_f = np.where(take, f, best_f)
        best_s = np.where(take, s, best_s)
    return best_f, best_s


def _gloo(group) -> bool:
    import torch.distributed as dist
    return dist.get_backend(group) == "gloo"


def _all_gather(out, inp, group):
    """all_gather_into_tensor (NCCL, device tensors) or, under gloo, its list
    form on host copies (CPU tests; ranks sharing one GPU)."""
    import torch.distributed as dist
    if inp.device.type == "cuda" and not _gloo(group):
        dist.all_gather_into_tensor(out, inp, group=group)
        return
    world = out.numel() // inp.numel()
    o = out.cpu() if out.device.type == "cuda" else out
    dist.all_gather(list(o.view(world, -1).unbind(0)), inp.cpu().view(-1), group=group)
    if o is not out:
        out.copy_(o)


def _all_reduce_max(t, group):
    """all_reduce(MAX) (NCCL), or on a host copy under gloo."""
    import torch.distributed as dist
    if t.device.type == "cuda" and _gloo(group):
        h = t.cpu()
        dist.all_reduce(h, op=dist.ReduceOp.MAX, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)


def scan_grid_distributed(ctx, grid, d_queries, nq: int, group=None, opts=None, metric="cc",
                          global_seed: bool = True):
    """Brute-force scan of the whole grid across the process group.

    d_queries: float64 tensor (nq, 2N) on this rank's device (CUDA; CPU with
    the test stub context).  Protocol:
      1. (cc, global_seed) each rank's seed pass over its slab -> screening
         maxima; one all_reduce(MAX) makes them global; they seed every rank's
         screening (floor_matches), so per-rank candidates and re-rank work
         do not grow with the world size;
      2. each rank scans its contiguous T1 slab (K1 -> K2 -> K3), exact
         (flat, score) per voxel, flat -1 where nothing on the slab reaches
         the global seed;
      3. ONE all_gather of the nq x 16 B match records and the merge (highest
         score, lowest flat on ties; dictionary.cpp:291-294).
    Returns (uint8 tensor of nq mrfg_match records (flat i64, score f64),
    identical on every rank; this rank's ScanStats or None)."""
    import ctypes as C

    import torch
    import torch.distributed as dist
    from ._native import ScanOpts

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    fb, fe = grid_shard(grid, world, rank)
    dev = d_queries.device
    d_out = torch.empty(nq * 16, dtype=torch.uint8, device=dev)
    stats = None
    o = opts
    if dev.type == "cuda":  # the queries may still be in flight on torch's stream
        torch.cuda.current_stream(dev).synchronize()
    if world > 1 and global_seed and metric == "cc":
        seed = torch.full((nq,), -3.0, dtype=torch.float32, device=dev)
        if fe > fb:
            ctx.scan_seed_device(grid, d_queries.data_ptr(), nq, seed.data_ptr(), metric=metric,
                                 flat_range=(fb, fe), opts=opts)
        # the context may run on its own stream: its seed copy must have landed
        # before torch's stream reads `seed`, and the floors torch builds below
        # must exist before the context's stream reads them (a cold start
        # stretches these windows: without the two syncs the scan could see
        # uninitialised floors and return "no atom above the floor")
        if dev.type == "cuda":
            torch.cuda.synchronize(dev)
        _all_reduce_max(seed, group)
        floor = torch.zeros((nq, 2), dtype=torch.float64, device=dev)
        floor[:, 1] = seed.double()
        floor_rec = floor.view(torch.int64)
        floor_rec[:, 0] = 0  # flat 0: "a floor is present"
        o = ScanOpts() if opts is None else ScanOpts.from_buffer_copy(opts)
        o.floor_matches = C.c_void_p(floor_rec.data_ptr())
        if dev.type == "cuda":
            torch.cuda.current_stream(dev).synchronize()
    if fe > fb:
        stats = ctx.scan_grid_device(grid, d_queries.data_ptr(), nq, d_out.data_ptr(), metric=metric,
                                     flat_range=(fb, fe), opts=o)
    else:  # more ranks than T1 slabs: contribute "no atoms"
        d_out.view(torch.int64).view(nq, 2)[:, 0] = -1
    if world == 1:
        return d_out, stats
    d_all = torch.empty(world * nq * 16, dtype=torch.uint8, device=dev)
    _all_gather(d_all, d_out, group)
    d_merged = torch.empty(nq * 16, dtype=torch.uint8, device=dev)
    ctx.merge_matches_device(d_all.data_ptr(), world, nq, d_merged.data_ptr())
    return d_merged, stats


def gather_voxel_shards(local, nvox: int, rec_bytes: int, group=None):
    """All-gather per-rank voxel blocks (voxel_shard order) of fixed-size
    records into the full array on every rank (ZOOM shards voxels
    and all-gathers the per-voxel result structs).  `local` is a uint8 tensor of
    (ve - vb) * rec_bytes bytes on the process group's device; blocks are padded
    to the largest shard for one all_gather_into_tensor.  Works with NCCL (CUDA
    tensors) and gloo (CPU tensors)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return local
    cap = max(ve - vb for vb, ve in (voxel_shard(nvox, world, r) for r in range(world)))
    pad = torch.zeros(cap * rec_bytes, dtype=torch.uint8, device=local.device)
    pad[: local.numel()] = local
    allb = torch.empty(world * cap * rec_bytes, dtype=torch.uint8, device=local.device)
    _all_gather(allb, pad, group)
    parts = []
    for r in range(world):
        vb, ve = voxel_shard(nvox, world, r)
        parts.append(allb[r * cap * rec_bytes: (r * cap + (ve - vb)) * rec_bytes])
    return torch.cat(parts)


def quantify_distributed(ctx, lattice, cfg, d_fps, nvox: int, group=None):
    """MRF-ZOOM over the process group (GPU): each rank quantifies its voxel
    block (voxel_shard) with K5, then one all_gather gives every rank all
    nvox mrfg_quant records (uint8 CUDA tensor, dgs.QUANT_DTYPE layout).
    d_fps: CUDA float64 tensor (nvox, 2N) of raw fingerprints on this rank."""
    import torch
    import torch.distributed as dist
    from . import dgs

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    vb, ve = voxel_shard(nvox, world, rank)
    rb = dgs.QUANT_DTYPE.itemsize
    local = torch.empty(max(ve - vb, 0) * rb, dtype=torch.uint8, device=d_fps.device)
    if ve > vb:
        ctx.quantify_device(d_fps[vb:ve].data_ptr(), ve - vb, lattice, cfg, local.data_ptr())
    return gather_voxel_shards(local, nvox, rb, group)
