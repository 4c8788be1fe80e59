"""BASELINE configs[4]: four-parameter brute force with a B1 flip scale.

N = 3000, B1 0.7-1.3 step 0.05 (13) x T1 100-3000 step 25 (117) x T2 20-500
step 10 (49) x df -100..100 step 10 (21) = 1,565,109 atoms (endpoint-inclusive
axes), 128x128 = 16,384 voxels with parameters uniform on the grid
(rng_at(11, axis, voxel)), SNR 25.

The reference has no B1 axis: B1 scales every excitation flip (the ideal
inversion stays), so SURVEY 8(d)'s oracle uses 13 schedules with flip_deg*B1.
The GPU path does the same: one K1->K2->K3 streamed scan_grid per B1 schedule
(bit-exact per slab), then the per-voxel merge over B1 (max score, lowest 4-D
flat b1*A3 + flat) with the C1 merge kernel (mrfg_merge_matches_dev).  Check:
the reference library's scan_grid on the 13 schedules for a voxel sample,
merged the same way on the host -- flats and scores must be identical.
ZOOM with B1 has no oracle and is not run.  Prints one JSON line.
Usage: python tools/bench_config5.py [nvox] [sample]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1506_05393_b200 as P  # noqa: E402
from paper_1506_05393_b200._native import ScanOpts  # noqa: E402


def main():
    import torch
    nvox = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    sample = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    use_floor = os.environ.get("CONFIG5_FLOOR", "1") != "0"
    n = 3000
    base = P.baseline_schedule(n, 1)
    b1 = [round(0.7 + 0.05 * k, 10) for k in range(13)]
    g = P.grid_inclusive((100.0, 3000.0, 25.0), (20.0, 500.0, 10.0), (-100.0, 100.0, 10.0))
    A3 = P.grid_total(g)
    A = A3 * len(b1)
    scheds = [P.Schedule(base.flip_deg * s, base.phase_deg, base.tr_ms, base.te_ms) for s in b1]
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    out = {"workload": "BASELINE configs[4]: 16,384 voxels, B1 x T1 x T2 x df = 1,565,109 atoms, N=3000, SNR 25",
           "voxels": nvox, "atoms": A, "b1_values": len(b1)}
    # ---- voxels: truth on the 4-D grid, noisy fingerprints from the scaled schedule
    t0 = time.perf_counter()
    counts = (len(b1), g.t1_ms.count, g.t2_ms.count, g.df_hz.count)
    idx = np.array([[P.dgs.rng_at(11, ax, v) % cnt for ax, cnt in enumerate(counts)] for v in range(nvox)],
                   dtype=np.int64)
    fps = np.empty((nvox, n), dtype=np.complex128)
    for k, s in enumerate(scheds):
        sel = np.nonzero(idx[:, 0] == k)[0]
        if sel.size == 0:
            continue
        prm = np.stack([P.params_at(g, *idx[v, 1:]) for v in sel])
        with P.Context(s) as c:
            fps[sel] = c.simulate(prm, precision=64)
    for v in range(nvox):
        fps[v] = P.dgs.add_noise(fps[v], float(np.linalg.norm(fps[v])) / np.sqrt(n) / 25.0, 9_000_000 + v)
    out["voxel_setup_s"] = time.perf_counter() - t0
    # ---- 13 streamed scans + merge over B1, device-resident queries
    d_q = torch.from_numpy(fps.view(np.float64).reshape(nvox, 2 * n)).to(dev)
    d_all = torch.empty((len(b1), nvox, 2), dtype=torch.int64, device=dev)  # Match {flat, score}
    d_merged = torch.empty((nvox, 2), dtype=torch.int64, device=dev)
    ctxs = [P.Context(s) for s in scheds]
    for c in ctxs:
        c.set_stream(stream.cuda_stream)
    # warm-up (like bench.py's W steps): one scan per B1 context builds its
    # schedule tables, sizes its scratch and loads every kernel before the timed region
    for k, c in enumerate(ctxs):
        c.scan_grid_device(g, d_q.data_ptr(), nvox, d_all[k].data_ptr())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    # slabs in B1 order; each later slab is screened against the running merged
    # best (floor_matches), so only atoms that can still win are re-ranked
    stats = []
    for k, c in enumerate(ctxs):
        opts = ScanOpts(0.0, 0, 0, 0, d_merged.data_ptr() if (k > 0 and use_floor) else None)
        stats.append(c.scan_grid_device(g, d_q.data_ptr(), nvox, d_all[k].data_ptr(), opts=opts))
        f = d_all[k, :, 0]
        f.copy_(torch.where(f >= 0, f + k * A3, f))  # 4-D flat (flat -1: nothing above the floor)
        ctxs[0].merge_matches_device(d_all.data_ptr(), k + 1, nvox, d_merged.data_ptr())
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    for c in ctxs:
        c.close()
    merged = d_merged.cpu().numpy()
    flat = merged[:, 0]
    score = merged[:, 1].view(np.float64)
    out["scan_s"] = ms / 1e3
    out["voxel_atom_cc_evals_per_s"] = nvox * A / (ms * 1e-3)
    out["bloch_atom_steps_per_s"] = A * n / (ms * 1e-3)
    out["breakdown_ms"] = {k: sum(getattr(s, k) for s in stats) for k in ("bloch_ms", "gemm_ms", "rerank_ms")}
    out["gemm_tflops"] = 8.0 * n * nvox * A / (out["breakdown_ms"]["gemm_ms"] * 1e-3) / 1e12
    out["screen_err_max"] = max(s.screen_err_max for s in stats)
    out["reranked"] = sum(s.reranked for s in stats)
    out["floor_between_slabs"] = use_floor
    truth = idx[:, 0] * A3 + (idx[:, 1] * g.t2_ms.count + idx[:, 2]) * g.df_hz.count + idx[:, 3]
    out["truth_recovered_fraction"] = float((flat == truth).mean())
    # ---- reference library (CPU) on a voxel sample, 13 schedules, host merge
    import oracle
    kind = "reference" if oracle.available("reference") else "restatement"
    orc = oracle.Oracle(kind)
    og = oracle.make_grid((g.t1_ms.min, g.t1_ms.step, g.t1_ms.count), (g.t2_ms.min, g.t2_ms.step, g.t2_ms.count),
                          (g.df_hz.min, g.df_hz.step, g.df_hz.count))
    pick = np.linspace(0, nvox - 1, sample).astype(np.int64)
    best_f = np.full(sample, -1, dtype=np.int64)
    best_s = np.full(sample, -np.inf)
    t0 = time.perf_counter()
    for k, s in enumerate(scheds):
        os_ = oracle.Schedule(s.flip_deg, s.phase_deg, s.tr_ms, s.te_ms)
        f, sc, _ = orc.scan_grid(os_, og, fps[pick], threads=os.cpu_count() or 1)
        better = sc > best_s  # strict: ties keep the lower B1 (lower 4-D flat)
        best_f = np.where(better, k * A3 + f, best_f)
        best_s = np.where(better, sc, best_s)
    dt = time.perf_counter() - t0
    same = int(((best_f == flat[pick]) & (best_s == score[pick])).sum())
    out["check_sample"] = {"voxels": int(sample), "identical_flat_and_score": same, "kind": kind}
    out["cpu_baseline"] = {"value": sample * A / dt, "unit": "voxel-atom CC evals/s",
                           "cores": os.cpu_count() or 1, "kind": "reference" if kind == "reference" else "port",
                           "sample": f"scan_grid of {sample} voxels over 13 B1 schedules, {dt:.1f} s"}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
