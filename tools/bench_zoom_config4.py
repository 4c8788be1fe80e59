"""BASELINE configs[3] (ZOOM only): 64x64 smooth phantom, N=1000, 1 ms / 0.5 ms /
0.1 Hz lattice (4901 x 3961 x 5001 = 9.7e10 points, brute force infeasible).

Times the K5 kernel (device-resident fingerprints, CUDA events) without and
with neighbour priors, checks a voxel sample against the reference CPU
implementation (oracle/_ref when built, else the C restatement), and times that
reference on the same sample with all host cores.  Prints one JSON line.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1506_05393_b200 as P  # noqa: E402
from paper_1506_05393_b200 import workloads as W  # noqa: E402


def main():
    import torch
    sample = int(sys.argv[1]) if len(sys.argv) > 1 else 32

    def gpu_sim(s, params):
        with P.Context(s) as c:
            return c.simulate(params, precision=64)

    wl = W.make(4, gpu_sim)
    cfg = P.zoom_config(**W.CONFIG4_ZOOM)
    nq, n = wl.nvox, wl.schedule.n
    out = {"workload": "BASELINE configs[3]: 64x64 smooth phantom, N=1000, lattice 1 ms/0.5 ms/0.1 Hz",
           "lattice_points": P.grid_total(wl.grid), "zoom_config": W.CONFIG4_ZOOM}
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    with P.Context(wl.schedule) as c:
        c.set_stream(stream.cuda_stream)
        t0 = time.perf_counter()
        c.quantify(wl.fps[:8], wl.grid, cfg)  # builds the lattice tables (host libm)
        out["table_setup_s"] = time.perf_counter() - t0
        d_q = torch.from_numpy(wl.fps.view(np.float64).reshape(nq, 2 * n)).to(dev)
        d_o = torch.empty(nq * P.dgs.QUANT_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        c.quantify_device(d_q.data_ptr(), nq, wl.grid, cfg, d_o.data_ptr())
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        c.quantify_device(d_q.data_ptr(), nq, wl.grid, cfg, d_o.data_ptr())
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        rec = d_o.cpu().numpy().view(P.dgs.QUANT_DTYPE)
        out["noprior"] = {"slice_ms": ms, "voxels_per_s": nq / (ms * 1e-3),
                          "evals_per_voxel_mean": float(rec["evaluations"].mean())}
        mask = np.ones(nq, dtype=np.uint8)
        res, secs = c.quantify_slice(wl.fps, mask, 64, 64, wl.grid, cfg, use_prior=2)
        same = (res["i1"] == rec["i1"]) & (res["i2"] == rec["i2"]) & (res["idf"] == rec["idf"])
        out["prior_wavefront"] = {"slice_s": secs, "evals_per_voxel_mean": float(res["evaluations"].mean()),
                                  "maps_equal_noprior": bool(same.all()),
                                  "voxels_equal_noprior": int(same.sum()),
                                  "score_prior_minus_noprior_mean": float((res["score"] - rec["score"]).mean()),
                                  "prior_score_higher": int((res["score"] > rec["score"]).sum()),
                                  "prior_score_lower": int((res["score"] < rec["score"]).sum())}
        truth_hit = (rec["i1"] == wl.truth[:, 0]) & (rec["i2"] == wl.truth[:, 1]) & (rec["idf"] == wl.truth[:, 2])
        out["exact_truth_fraction"] = float(truth_hit.mean())
        out["df_truth_fraction"] = float((rec["idf"] == wl.truth[:, 2]).mean())
    # reference on a voxel sample (parity + CPU baseline)
    import oracle
    kind = "reference" if oracle.available("reference") else "restatement"
    orc = oracle.Oracle(kind)
    os_ = oracle.Schedule(wl.schedule.flip_deg, wl.schedule.phase_deg, wl.schedule.tr_ms, wl.schedule.te_ms)
    g = wl.grid
    og = oracle.make_grid((g.t1_ms.min, g.t1_ms.step, g.t1_ms.count), (g.t2_ms.min, g.t2_ms.step, g.t2_ms.count),
                          (g.df_hz.min, g.df_hz.step, g.df_hz.count))
    oc = oracle.ZoomCfg()
    for name, _ in oracle.ZoomCfg._fields_:
        v = getattr(cfg, name)
        if name.startswith("t1t2"):
            for i in range(8):
                getattr(oc, name)[i] = v[i]
        else:
            setattr(oc, name, v)
    idx = np.linspace(0, nq - 1, sample).astype(int)
    smask = np.zeros(nq, dtype=np.uint8)
    smask[idx] = 1
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    ref = orc.quantify_slice(os_, og, oc, wl.fps, smask, 64, 64, False, threads)
    dt = time.perf_counter() - t0
    same = sum(int((ref[v].i1, ref[v].i2, ref[v].idf, ref[v].evaluations) ==
                   (rec["i1"][v], rec["i2"][v], rec["idf"][v], rec["evaluations"][v])) for v in idx)
    out["parity_sample"] = {"voxels": int(sample), "identical_answer_and_evals": same}
    out["cpu_baseline"] = {"value": sample / dt, "unit": "voxels/s", "cores": threads, "kind": kind,
                           "sample": f"quantify_slice (no prior) of {sample} voxels, {dt:.1f} s"}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
