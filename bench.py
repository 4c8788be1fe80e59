#!/usr/bin/env python
"""DGS benchmark (BASELINE.json configs[1]: 64x64 slice, N=1000, 97.7M-atom grid).

One step = one full brute-force dictionary generating-and-searching pass of
the 4,096-voxel slice over the whole T1 x T2 x df grid: FP32 Bloch producer
(K1) -> [projection of each off-resonance slab onto its subspace basis] ->
fp16 tcgen05 screening GEMM with fused candidate epilogue (K2) -> exact FP64
re-rank (K3), streamed in chunks so the dictionary never exists.  The
library screens this lattice in per-off-resonance subspaces by default
(csrc/subspace.cu); `full_length_screening` in the JSON line is one scan of the
same step with the 2N-dimensional screening (MRFG_SUBSPACE=0).
With N GPUs the atom range is sharded (contiguous T1-major slabs) and the
per-voxel (flat, score) pairs are merged after one NCCL all_gather (C1):
total work is fixed, so scaling is "strong".

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Prints ONE JSON line on rank 0.  `value` is device-timed (CUDA events on the
launching stream, max over ranks) with queries resident in HBM; `e2e` is the
same metric through the host-buffer public API (pinned H2D of the queries and
D2H of the matches inside the timed region).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "64x64-slice DGS wall time; Bloch atom-steps/s; voxel-atom CC evals/s"
UNIT = "voxel-atom CC evals/s"
FP32_PEAK_TFLOPS_NOMINAL = 148 * 128 * 2 * 1.965e9 / 1e12  # 74.4 at max SM clock
BLOCH_FLOP_PER_STEP = 37


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def k2_traffic(chunk_atoms, n, nq):
    """DRAM bytes (read + write) of one K2 launch from the committed ncu --set
    full capture (profiles/r02_k2_traffic.json), when it was taken on this
    workload shape; else None."""
    p = os.path.join(ROOT, "profiles", "r02_k2_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
    except (OSError, ValueError):
        return None
    if (d.get("chunk_atoms"), d.get("voxels"), d.get("timepoints")) != (chunk_atoms, nq, n):
        return None
    return d.get("dram_bytes_per_launch")


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.rows = []
        if self.proc is None:
            return
        time.sleep(0.25)
        self.proc.terminate()
        out = self.proc.communicate(timeout=10)[0]
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def summary(self):
        if not getattr(self, "rows", None):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i] == "Active"})
        loaded = [s for s in sm if s > 0.5 * (max(sm) if sm else 1)]
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def spawn_ranks(args) -> int:
    """`bench.py --gpus N` outside torchrun: launch N NCCL ranks (one process
    per GPU) through torch.distributed.run on 127.0.0.1 and relay rank 0's
    line.  Fails when fewer than N GPUs are visible."""
    import socket
    try:
        import torch
        ngpu = torch.cuda.device_count()
    except Exception:  # noqa: BLE001
        ngpu = 0
    if ngpu < args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} needs {args.gpus} visible GPUs, found {ngpu}"}),
              flush=True)
        return 1
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def allmax(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def shard(total: int, world: int, rank: int):
    cuts = [total * r // world for r in range(world + 1)]
    return cuts[rank], cuts[rank + 1]


# ------------------------------------------------------------- CPU baseline
def cpu_sample(config: int, nvox_sample: int, which: str | None = None):
    """Reference CPU path on a bounded sample: nvox_sample voxels x one T1 slab
    (all T2 x df atoms at one T1 value), on ALL host cores: the reference's own
    mrf::generate for the slab's rows (row-parallel) and mrf::brute_force_search
    per voxel (voxel-parallel) -- SURVEY 8(d)'s plan, since scan_grid's own
    scan loop is serial over queries (dictionary.cpp:283-299).  The C
    restatement stands in where the reference library was not built."""
    import oracle
    from paper_1506_05393_b200 import workloads
    kind = which or ("reference" if oracle.available("reference") else "restatement")
    orc = oracle.Oracle(kind)
    c = workloads.CONFIGS[config]
    s = orc.baseline_schedule(c["n"], 1)
    n1 = int(round((c["t1"][1] - c["t1"][0]) / c["t1"][2])) + 1
    n2 = int(round((c["t2"][1] - c["t2"][0]) / c["t2"][2])) + 1
    nd = int(round((c["df"][1] - c["df"][0]) / c["df"][2])) + 1
    i1 = n1 // 2
    t1v = c["t1"][0] + i1 * c["t1"][2]
    # queries: noisy on-grid fingerprints (uniform over the grid, SNR as configured)
    rng_idx = [(k * 7919) % (n1 * n2 * nd) for k in range(nvox_sample)]
    fps = []
    for k, f in enumerate(rng_idx):
        idf, rest = f % nd, f // nd
        a, b = rest // n2, rest % n2
        fp = orc.simulate(s, (c["t1"][0] + a * c["t1"][2]) * 1e-3, (c["t2"][0] + b * c["t2"][2]) * 1e-3,
                          c["df"][0] + idf * c["df"][2])
        sigma = float(np.linalg.norm(fp)) / math.sqrt(c["n"]) / c["snr"]
        fps.append(orc.add_noise(fp, sigma, 1_000_000 + k))
    fps = np.stack(fps)
    threads = os.cpu_count() or 1
    t2v = c["t2"][0] + np.arange(n2, dtype=np.float64) * c["t2"][2]
    t0 = time.perf_counter()
    if kind == "reference":
        orc.scan_rows(s, np.array([t1v]), t2v, (c["df"][0], c["df"][2], nd), fps, threads=threads)
        how = "mrf::generate rows + mrf::brute_force_search, voxel-parallel"
    else:
        import concurrent.futures as cf
        slab = oracle.make_grid((t1v, c["t1"][2], 1), (c["t2"][0], c["t2"][2], n2), (c["df"][0], c["df"][2], nd))
        with cf.ThreadPoolExecutor(threads) as ex:
            list(ex.map(lambda b: orc.scan_grid(s, slab, fps[b], threads=1),
                        np.array_split(np.arange(nvox_sample), threads)))
        how = "C restatement scan_grid, voxel blocks in parallel"
    dt = time.perf_counter() - t0
    evals = nvox_sample * n2 * nd
    return {"value": evals / dt, "unit": UNIT, "cores": threads,
            "kind": "reference" if kind == "reference" else "port",
            "sample": f"{nvox_sample} noisy config-{config} voxels x one T1 slab ({n2 * nd} atoms, "
                      f"N={c['n']}), simulate+match ({how}, {threads} threads), {dt:.2f} s"}


def arm_config(args, world, nx, ny, n, nq, total):
    """The workload description both arms print (config of the JSON line)."""
    return {"workload": f"BASELINE configs[{args.config - 1}]: {nx}x{ny} slice, N={n}, "
                        f"{total} atoms, brute-force streamed DGS",
            "voxels": nq, "atoms": total, "timepoints": n,
            "chunk_atoms": args.chunk or "library default (one K1 wave of whole lattice rows)",
            "delta": args.delta or "library default (2.5e-3; + twice the held-out residual with subspace screening)", "parallelism": f"atom-shard x{world}",
            "l2": "256 MB flush per step; each step streams >100 GB of fp16 atoms"}


def ref_config(args, world):
    """Our arm's config for the same workload (the reference arm times a
    bounded sample of it: cpu_baseline.sample says which)."""
    from paper_1506_05393_b200 import workloads
    c = workloads.CONFIGS[args.config]
    axes = [int(round((c[k][1] - c[k][0]) / c[k][2])) + 1 for k in ("t1", "t2", "df")]
    total = axes[0] * axes[1] * axes[2]
    if args.atoms:
        total = min(total, args.atoms)
    nx, ny = c.get("nx", 0), c.get("ny", 0)
    nq = args.nvox or (nx * ny)
    return arm_config(args, world, nx, ny, c["n"], nq, total)


def run_reference(args, world, rank):
    if rank != 0:
        return
    vals = []
    for k in range(args.warmup + args.steps):
        r = cpu_sample(args.config, args.ref_voxels)
        if k >= args.warmup:
            vals.append(r["value"])
    v = statistics.mean(vals)
    r["value"] = v
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": ref_config(args, world),
            "cpu_baseline": r,
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm
def run_ours(args, world, rank, local):
    import torch
    import paper_1506_05393_b200 as P
    from paper_1506_05393_b200 import workloads
    from paper_1506_05393_b200._native import ScanOpts

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)

    def gpu_sim(sched, params):
        with P.Context(sched, local) as c:
            return c.simulate(params, precision=64)

    wl = workloads.make(args.config, gpu_sim, nvox=args.nvox)
    g, nq, n = wl.grid, wl.nvox, wl.schedule.n
    total = P.grid_total(g)
    if args.atoms:
        total = min(total, args.atoms)
    from paper_1506_05393_b200 import distributed as D
    fb, fe = shard(total, world, rank) if args.atoms else D.grid_shard(g, world, rank)
    ctx = P.Context(wl.schedule, local)
    ctx.set_stream(stream.cuda_stream)
    opts = ScanOpts(args.delta, args.chunk, 0, 0)

    d_q = torch.from_numpy(wl.fps.view(np.float64).reshape(nq, 2 * n)).to(dev)
    d_out = torch.empty(nq * 16, dtype=torch.uint8, device=dev)
    d_all = torch.empty(world * nq * 16, dtype=torch.uint8, device=dev)
    d_merged = torch.empty(nq * 16, dtype=torch.uint8, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > L2 (126 MB)

    def step(collect=None):
        flush.fill_(1)
        if args.atoms:  # debug: truncated range, plain contiguous shards
            st = ctx.scan_grid_device(g, d_q.data_ptr(), nq, d_out.data_ptr(), flat_range=(fb, fe),
                                      opts=opts)
            if world > 1:
                import torch.distributed as dist
                dist.all_gather_into_tensor(d_all, d_out)
                ctx.merge_matches_device(d_all.data_ptr(), world, nq, d_merged.data_ptr())
        else:  # shard scan + one all_gather + merge (C1)
            _, st = D.scan_grid_distributed(ctx, g, d_q, nq, opts=opts)
        if collect is not None and st is not None:
            collect.append(st)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    stats = []
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            step(stats)
        ev1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    ms = allmax(ev0.elapsed_time(ev1), world) / args.steps
    evals_step = nq * total  # whole job: every voxel against every atom
    value = evals_step / (ms * 1e-3)

    # ---- e2e through the host-buffer public API (pinned H2D + D2H inside)
    h_q = torch.from_numpy(wl.fps.view(np.float64).reshape(nq, 2 * n)).pin_memory()
    h_res = torch.empty(nq * 16, dtype=torch.uint8).pin_memory()

    def e2e_step():
        if world == 1:
            q = h_q.numpy().view(np.complex128)
            f, s, _ = ctx.scan_grid(g, q, opts=opts, flat_range=(fb, fe))
            return f
        dq = h_q.to(dev, non_blocking=True)
        merged, _ = D.scan_grid_distributed(ctx, g, dq, nq, opts=opts)
        h_res.copy_(merged, non_blocking=True)
        torch.cuda.synchronize()
        return h_res

    e2e_step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    e2e_steps = max(1, args.steps)
    for _ in range(e2e_steps):
        e2e_step()
    torch.cuda.synchronize()
    e2e_s = allmax((time.perf_counter() - t0) / e2e_steps, world)

    # ---- the same step with full-length (2N-dimensional) screening, one scan:
    # the regime the K2 tensor roofline describes
    full = None
    if world == 1 and not args.no_full and os.environ.get("MRFG_SUBSPACE") is None:
        os.environ["MRFG_SUBSPACE"] = "0"
        try:
            ctx.scan_grid_device(g, d_q.data_ptr(), nq, d_out.data_ptr(), opts=opts, flat_range=(fb, fe))  # warm
            sf = ctx.scan_grid_device(g, d_q.data_ptr(), nq, d_out.data_ptr(), opts=opts, flat_range=(fb, fe))
            torch.cuda.synchronize()
        finally:
            del os.environ["MRFG_SUBSPACE"]
        ftf = 8.0 * n * nq * (fe - fb) / (sf.gemm_ms * 1e-3) / 1e12
        pkf, _ = peaks()
        full = {"ms_per_step": sf.total_ms, "value": nq * (fe - fb) / (sf.total_ms * 1e-3), "unit": UNIT,
                "breakdown_ms": {"bloch": sf.bloch_ms, "gemm": sf.gemm_ms, "rerank": sf.rerank_ms},
                "k2_tflops": ftf, "k2_frac_of_tensor_peak": ftf / pkf.get("bf16_tflops_sustained", pkf["bf16_tflops"]),
                "screen_err_audit_max": sf.screen_err_audit_max, "delta": sf.delta_used,
                "candidates": sf.candidates, "atoms_per_launch": int(sf.chunk_atoms),
                "how": "MRFG_SUBSPACE=0, one scan after a warm-up scan, device-resident queries, the ABI's CUDA events"}

    # ---- MRF-ZOOM on the same slice (K5), voxel-sharded, device-resident
    zoom = None
    if not args.no_zoom:
        from paper_1506_05393_b200 import distributed as Dz
        zcfg = P.zoom_config(df_coarse_hz=5.0, omega_hz=82.0)
        # voxel blocks per rank + one all_gather of the result structs
        Dz.quantify_distributed(ctx, g, zcfg, d_q, nq)  # warm-up
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        z0, z1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        z0.record(stream)
        d_zq = Dz.quantify_distributed(ctx, g, zcfg, d_q, nq)
        z1.record(stream)
        torch.cuda.synchronize()
        zms = allmax(z0.elapsed_time(z1), world)
        recs = d_zq.cpu().numpy().view(P.dgs.QUANT_DTYPE)
        zoom = {"voxels_per_s": nq / (zms * 1e-3), "slice_ms": zms,
                "evals_per_voxel_mean": float(recs["evaluations"].mean()),
                "config": "df_coarse 5 Hz, omega 82 Hz, reference defaults otherwise; voxel blocks per rank + "
                          "one all_gather of the result structs"}
        # BASELINE configs[3]: ZOOM only on the 1 ms / 0.5 ms / 0.1 Hz lattice
        # (9.7e10 points; brute force infeasible), same voxel sharding, median of 3
        wl4 = workloads.make(4, gpu_sim)
        g4, nq4 = wl4.grid, wl4.nvox
        z4cfg = P.zoom_config(**workloads.CONFIG4_ZOOM)
        with P.Context(wl4.schedule, local) as ctx4:
            ctx4.set_stream(stream.cuda_stream)
            d_q4 = torch.from_numpy(wl4.fps.view(np.float64).reshape(nq4, 2 * n)).to(dev)
            Dz.quantify_distributed(ctx4, g4, z4cfg, d_q4, nq4)  # tables + warm-up
            times = []
            for _ in range(3):
                torch.cuda.synchronize()
                if world > 1:
                    torch.distributed.barrier()
                z0, z1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                z0.record(stream)
                d_z4 = Dz.quantify_distributed(ctx4, g4, z4cfg, d_q4, nq4)
                z1.record(stream)
                torch.cuda.synchronize()
                times.append(allmax(z0.elapsed_time(z1), world))
            z4ms = float(np.median(times))
            r4 = d_z4.cpu().numpy().view(P.dgs.QUANT_DTYPE)
        def zoom_roofline(vps, evals):
            # reference-equivalent unique evaluations x N x (37 Bloch + 8 CC)
            # flop against the FP32 CUDA-core peak (148 SMs x 128 lanes x 2 x max clock)
            ach = vps * evals * n * 45.0 / 1e12
            pk32 = 148 * 128 * 2 * pk_all.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
            return {"bound": "fp32", "achieved": ach, "peak": pk32, "unit": "TFLOP/s", "frac": ach / pk32,
                    "peak_kind": "nominal FP32 at sm_max_mhz",
                    "work": "unique evaluations x N x 45 flop (speculative screening not counted)"}
        pk_all, _ = peaks()
        zoom["roofline"] = zoom_roofline(zoom["voxels_per_s"], zoom["evals_per_voxel_mean"])
        zoom["config4"] = {"voxels_per_s": nq4 / (z4ms * 1e-3), "slice_ms": z4ms,
                           "evals_per_voxel_mean": float(r4["evaluations"].mean()),
                           "config": "BASELINE configs[3] 64x64 smooth phantom, lattice 1 ms/0.5 ms/0.1 Hz, "
                                     "zoom steps " + str(workloads.CONFIG4_ZOOM)}
        zoom["config4"]["roofline"] = zoom_roofline(zoom["config4"]["voxels_per_s"],
                                                    zoom["config4"]["evals_per_voxel_mean"])
        if world == 1:
            # the reference's strict raster prior (zoom.cpp:589-615) on the same
            # slice: one launch, the voxel chain on one SM (host API, wall time)
            with P.Context(wl4.schedule, local) as ctx4:
                mask = np.ones(nq4, np.uint8)
                ctx4.quantify_slice(wl4.fps[:64], mask[:64], 64, 1, g4, z4cfg, use_prior=1)  # tables, warm
                rp, secs = ctx4.quantify_slice(wl4.fps, mask, wl4.nx, wl4.ny, g4, z4cfg, use_prior=1)
            zoom["config4"]["raster_prior"] = {"seconds": secs, "voxels_per_s": nq4 / secs,
                                               "evals_per_voxel_mean": float(rp["evaluations"].mean())}
            # BASELINE configs[4]: four-parameter ZOOM (outer B1 zoom_1d of K5,
            # mrfg_quantify_b1) on the whole 128x128 slice, N = 3000 (host API, wall time)
            sc5, g5, _, fps5 = workloads.config5_voxels(gpu_sim, np.arange(workloads.CONFIG5["nvox"]))
            c5cfg = P.zoom_config(**workloads.CONFIG5_ZOOM)
            ctx5 = [P.Context(s5, local) for s5 in sc5]
            try:
                P.quantify_b1(ctx5, fps5[:256], g5, c5cfg, workloads.CONFIG5_B1_STEPS, workloads.CONFIG5_B1_INIT)
                t5 = time.perf_counter()
                q5, _ = P.quantify_b1(ctx5, fps5, g5, c5cfg, workloads.CONFIG5_B1_STEPS, workloads.CONFIG5_B1_INIT)
                s5 = time.perf_counter() - t5
            finally:
                for c5 in ctx5:
                    c5.close()
            zoom["config5_b1"] = {"voxels_per_s": len(fps5) / s5, "seconds": s5,
                                  "evals_per_voxel_mean": float(q5["evaluations"].mean()),
                                  "config": "BASELINE configs[4] 128x128, B1 x T1 x T2 x df = 13 x 117 x 49 x 21, "
                                            "N=3000; outer B1 zoom_1d (steps 4, 1) of three-parameter ZOOM "
                                            + str(workloads.CONFIG5_ZOOM)}

    # ---- roofline of the dominant kernel (K2) from the in-ABI CUDA events
    pk, pk_kind = peaks()
    gemm_ms = sum(s.gemm_ms for s in stats)
    launches = sum(s.gemm_launches for s in stats)
    # K2 flops: 8 flop per voxel-atom pair and complex dimension it multiplies
    # over -- N timepoints with full-length screening, r with per-off-resonance
    # subspace screening (the library's default on this lattice)
    sub_r = int(stats[-1].subspace_rank)
    kdim = sub_r if sub_r else n
    flops_alg = 8.0 * kdim * nq * (fe - fb) * len(stats)
    gemm_tflops = flops_alg / (gemm_ms * 1e-3) / 1e12
    project_ms = sum(s.project_ms for s in stats)
    chunk_atoms = int(stats[-1].chunk_atoms)  # atoms per K2 launch (the library's choice when --chunk 0)
    peak_t = pk.get("bf16_tflops_sustained", pk["bf16_tflops"])
    bloch_ms = sum(s.bloch_ms for s in stats)
    bloch_rate = (fe - fb) * n * len(stats) / (bloch_ms * 1e-3)
    cand = stats[-1].candidates
    rer = stats[-1].reranked

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "fp16 screen / fp32 accum / f64 rerank",
        "data": "synthetic (seeded BASELINE configs[1] phantom, SNR 30)",
        "config": arm_config(args, world, wl.nx, wl.ny, n, nq, total),
        "slice_dgs_wall_s": ms * 1e-3,
        "bloch_atom_steps_per_s": bloch_rate * world,
        "bloch_fp32_tflops": bloch_rate * BLOCH_FLOP_PER_STEP / 1e12,
        "bloch_frac_of_fp32_peak_nominal": bloch_rate * BLOCH_FLOP_PER_STEP / 1e12 / FP32_PEAK_TFLOPS_NOMINAL,
        "candidates_per_step": cand, "reranked_per_step": rer,
        "breakdown_ms_per_step": {"bloch": bloch_ms / len(stats), "project": project_ms / len(stats),
                                  "gemm": gemm_ms / len(stats),
                                  "rerank": sum(s.rerank_ms for s in stats) / len(stats),
                                  "scan_total": sum(s.total_ms for s in stats) / len(stats)},
        "screen_err_max": max(s.screen_err_max for s in stats),
        "screen_audit": {"err_max": max(s.screen_err_audit_max for s in stats),
                         "rescreen32_err_max": max(s.rescreen_err_audit_max for s in stats),
                         "samples_per_step": stats[-1].audit_samples,
                         "delta": stats[-1].delta_used, "rescans": sum(s.rescans for s in stats),
                         "rule": "hash sample of ALL screened (voxel, atom) pairs, scored exactly; "
                                 "certificate needs err_max <= delta/2"},
        "roofline": {"bound": "tensor", "achieved": gemm_tflops, "peak": peak_t, "unit": "TFLOP/s",
                     "frac": gemm_tflops / peak_t, "traffic": k2_traffic(chunk_atoms, n, nq),
                     "kernel": "k_match_sm100_2cta (K2)" + (f" on {2 * sub_r} subspace dimensions" if sub_r else ""),
                     "peak_kind": f"{pk_kind} bf16 dense sustained",
                     "avg_launch_ms": gemm_ms / max(launches, 1),
                     "flop_per_launch": 8.0 * kdim * nq * chunk_atoms, "atoms_per_launch": chunk_atoms,
                     "k_dims": 2 * kdim,
                     "pairs_per_s": nq * (fe - fb) * len(stats) / (gemm_ms * 1e-3),
                     "note": ("executed tensor flops (8 r per voxel-atom pair); with 2r-dimensional operands K2 "
                              "is bound by its epilogue (TMEM loads, score, threshold per pair), see "
                              "full_length_screening for the 2N-dimensional regime") if sub_r else
                             "algorithmic flops 8 N per voxel-atom pair"},
        # the projection kernel of subspace screening: HBM-bound (reads the fp16
        # atom operand once, writes 2r coefficients per atom)
        "roofline_project": None if not sub_r else {
            "bound": "hbm", "unit": "GB/s", "peak": pk["hbm_gbs"], "kernel": "k_project (mma.sync m16n8k16)",
            "achieved": (fe - fb) * len(stats) * 2.0 * (2 * n + 2 * sub_r) / (project_ms * 1e-3) / 1e9,
            "frac": (fe - fb) * len(stats) * 2.0 * (2 * n + 2 * sub_r) / (project_ms * 1e-3) / 1e9 / pk["hbm_gbs"],
            "bytes_per_atom": 2.0 * (2 * n + 2 * sub_r), "traffic": None},
        "screening": {"subspace_rank": sub_r, "residual_held_out_max": stats[-1].subspace_residual_max,
                      "residual_device_estimate_max": stats[-1].subspace_residual_device,
                      "note": "per-off-resonance subspace screening (csrc/subspace.cu); MRFG_SUBSPACE=0 = full length"},
        "full_length_screening": full,
        "e2e": {"value": nq * total / e2e_s, "unit": UNIT, "h2d_bytes_per_step": nq * n * 16,
                "d2h_bytes_per_step": nq * 16, "seconds_per_step": e2e_s},
        # our kernels per scan: per chunk K1 + K2 (+ k_zero_rows for the chunk's
        # edge rows); seed pass (table producer + K2), k_fill, query prep;
        # re-rank: filter, keys, FP32 re-screen, flag, FP64 re-rank, select,
        # FP32 error check, write (CUB sort/select kernels not counted); the
        # screening audit; + seed pass and k_merge when N > 1
        # subspace screening: per scan one K1 launch per off-resonance quad (chunks),
        # per off-resonance value a slab projection and a K2 launch, one query projection
        "gpu_launches": int(sum((s.chunks + 2 * g.df_hz.count + 14) if s.subspace_rank else (3 * s.chunks + 13)
                                for s in stats) + (3 * args.steps if world > 1 else 0)),
        "clocks": clk.summary(),
        "zoom": zoom,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_sample(args.config, args.ref_voxels)
        except Exception as e:  # the oracle is test infrastructure; never fatal here
            line["cpu_baseline"] = {"value": None, "error": str(e)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--nvox", type=int, default=None)
    ap.add_argument("--atoms", type=int, default=0, help="limit atoms (debug only)")
    ap.add_argument("--no-full", action="store_true", help="skip the full-length-screening comparison scan")
    ap.add_argument("--chunk", type=int, default=0, help="atoms per streamed chunk (0: the library default)")
    ap.add_argument("--delta", type=float, default=0.0, help="screening margin (0: library default 2.5e-3)")
    ap.add_argument("--ref-voxels", type=int, default=64)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-zoom", action="store_true")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    world, rank, local = dist_setup(args)
    if world != args.gpus and rank == 0:
        print(f"[bench] note: --gpus {args.gpus} but WORLD_SIZE {world}; using {world}", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_ours(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
