"""Reference answers at BASELINE scale -> tests/golden/scale_c{2,3,4,5}.npz.

Run HERE, where /root/reference exists and oracle/_ref/libmrf_ref.so (the
reference library compiled from its own sources by oracle/Makefile) is built;
the fixtures are committed and tests/test_gpu_scale.py checks the GPU path
against them on the GPU box (which has no /root/reference).

Inputs are regenerated bit-identically at test time: schedules, phantoms and
noise come from paper_1506_05393_b200/workloads.py (host code, the reference's
counter RNG), truth fingerprints from the C restatement oracle (pinned
bit-exact to the reference by tests/test_oracle.py).  Every answer below is the
REFERENCE LIBRARY's own:

* c2: BASELINE configs[1], full 491 x 397 x 501 = 97,658,427-atom lattice,
  N = 1000; 256 of the 4,096 voxels, stratified over the 6 tissue classes;
  mrf::generate rows + mrf::brute_force_search (oracle.scan_rows, lowest flat
  on ties) -- about 2 h on 8 cores.
* c3: BASELINE configs[2], log-spaced T1/T2 (300 x 200) x 41 df = 2,460,000
  atoms, N = 1000; 256 of the 262,144 voxels.
* c4: BASELINE configs[3], the whole 64 x 64 slice, mrf::quantify_slice with
  the CONFIG4_ZOOM settings, without and with priors (strict raster).
* c5: BASELINE configs[4], 13 B1 schedules x 117 x 49 x 21, N = 3000; 128 of
  the 16,384 voxels; per-B1 argmax then max over B1 (ties: lower B1).
* c5z: the same 128 voxels through four-parameter ZOOM (CONFIG5_ZOOM; the
  reference's zoom_1d over B1 of the reference's quantify).

Usage: python tests/golden/make_scale_fixtures.py {c2,c3,c4,c5,c5z} [threads]
"""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1506_05393_b200 import workloads  # noqa: E402

REST = oracle.Oracle("restatement")


def osched(s):
    return oracle.Schedule(s.flip_deg, s.phase_deg, s.tr_ms, s.te_ms)


def sim(s, params):
    """Truth fingerprints from the restatement oracle (bit-exact to the reference)."""
    os_ = osched(s)
    return np.stack([REST.simulate(os_, *p) for p in params])


def c2_voxels(nvox=256):
    """256 voxels over the 6 classes: an equal share per class, evenly spaced in raster order."""
    cls = workloads.ellipse_classes(64, 64)
    per = nvox // 6
    pick = []
    for c in range(6):
        ids = np.nonzero(cls == c)[0]
        k = per + (1 if c < nvox - 6 * per else 0)
        pick += list(ids[np.linspace(0, ids.size - 1, min(k, ids.size)).astype(np.int64)])
    return np.array(sorted(set(int(v) for v in pick)), dtype=np.int64)


def axis_values(ax):
    return ax.min + np.arange(ax.count, dtype=np.float64) * ax.step  # AxisSpec::value


def run_c2(ref, threads, t1_chunk=8):
    """Resumable: the T1 axis is scanned in chunks of t1_chunk rows; after each
    chunk the running (flat, score) is saved to scale_c2.partial.npz, so an
    interrupted run continues where it stopped.  Chunks are merged in T1 order
    with a strict '>' -- exactly the reference's own running argmax over slabs
    (oracle/ref_capi.cpp orc_ref_scan_rows), so the result equals one call."""
    wl = workloads.make(2, sim)
    g = wl.grid
    vox = c2_voxels()
    t1 = axis_values(g.t1_ms)
    t2 = axis_values(g.t2_ms)
    a_row = g.t2_ms.count * g.df_hz.count
    part = os.path.join(HERE, "scale_c2.partial.npz")
    best_f = np.zeros(len(vox), dtype=np.int64)
    best_s = np.full(len(vox), -1e300)
    done, secs = 0, 0.0
    if os.path.exists(part):
        p = np.load(part)
        assert np.array_equal(p["voxels"], vox)
        best_f, best_s, done, secs = p["flat"], p["score"], int(p["done"]), float(p["seconds"])
    q = wl.fps[vox]
    while done < len(t1):
        hi = min(len(t1), done + t1_chunk)
        t0 = time.time()
        f, sc = ref.scan_rows(osched(wl.schedule), t1[done:hi], t2,
                              (g.df_hz.min, g.df_hz.step, g.df_hz.count), q, threads=threads)
        better = sc > best_s
        best_f = np.where(better, f + done * a_row, best_f)
        best_s = np.where(better, sc, best_s)
        done, secs = hi, secs + time.time() - t0
        np.savez(part, voxels=vox, flat=best_f, score=best_s, done=done, seconds=secs)
        print(f"c2: T1 rows {done}/{len(t1)}, {secs:.0f} s", flush=True)
    return dict(voxels=vox, flat=best_f, score=best_s, seconds=secs,
                classes=workloads.ellipse_classes(64, 64)[vox])


def run_c3(ref, threads):
    vox = np.linspace(0, workloads.CONFIG3["nvox"] - 1, 256).astype(np.int64)
    sched, idx, fps = workloads.config3_voxels(sim, vox)
    t1, t2, df = workloads.config3_axes()
    t0 = time.time()
    flat, score = ref.scan_rows(osched(sched), t1, t2, df, fps, threads=threads)
    return dict(voxels=vox, flat=flat, score=score, seconds=time.time() - t0, t1_ms=t1, t2_ms=t2)


def run_c4(ref, threads):
    wl = workloads.make(4, sim)
    g = wl.grid
    og = oracle.make_grid((g.t1_ms.min, g.t1_ms.step, g.t1_ms.count), (g.t2_ms.min, g.t2_ms.step, g.t2_ms.count),
                          (g.df_hz.min, g.df_hz.step, g.df_hz.count))
    cfg = oracle.zoom_cfg(**workloads.CONFIG4_ZOOM)
    mask = np.ones(wl.nvox, np.uint8)
    out = {}
    for prior in (0, 1):
        t0 = time.time()
        r = ref.quantify_slice(osched(wl.schedule), og, cfg, wl.fps, mask, wl.nx, wl.ny, bool(prior),
                               threads=threads)
        sfx = "_prior" if prior else ""
        out["seconds" + sfx] = time.time() - t0
        out["ijk" + sfx] = np.array([[q.i1, q.i2, q.idf] for q in r], dtype=np.int64)
        out["score" + sfx] = np.array([q.score for q in r])
        out["pd" + sfx] = np.array([q.pd for q in r])
        out["evals" + sfx] = np.array([q.evaluations for q in r], dtype=np.int64)
    return out


def run_c5(ref, threads):
    vox = np.linspace(0, workloads.CONFIG5["nvox"] - 1, 128).astype(np.int64)
    scheds, g, idx, fps = workloads.config5_voxels(sim, vox)
    a3 = g.t1_ms.count * g.t2_ms.count * g.df_hz.count
    best_f = np.full(len(vox), -1, dtype=np.int64)
    best_s = np.full(len(vox), -np.inf)
    t0 = time.time()
    for k, s in enumerate(scheds):
        f, sc = ref.scan_rows(osched(s), axis_values(g.t1_ms), axis_values(g.t2_ms),
                              (g.df_hz.min, g.df_hz.step, g.df_hz.count), fps, threads=threads)
        better = sc > best_s  # strict: ties keep the lower B1 (lower 4-D flat)
        best_f = np.where(better, k * a3 + f, best_f)
        best_s = np.where(better, sc, best_s)
    return dict(voxels=vox, flat=best_f, score=best_s, seconds=time.time() - t0)


def run_c5z(ref, threads):
    """Four-parameter ZOOM on the config-5 lattice: the reference's own zoom_1d
    over the B1 index of its own quantify (oracle/ref_capi.cpp
    orc_quantify_b1), 128 voxels, voxel-parallel."""
    import concurrent.futures as cf
    vox = np.linspace(0, workloads.CONFIG5["nvox"] - 1, 128).astype(np.int64)
    scheds, g, idx, fps = workloads.config5_voxels(sim, vox)
    og = oracle.make_grid((g.t1_ms.min, g.t1_ms.step, g.t1_ms.count), (g.t2_ms.min, g.t2_ms.step, g.t2_ms.count),
                          (g.df_hz.min, g.df_hz.step, g.df_hz.count))
    cfg = oracle.zoom_cfg(**workloads.CONFIG5_ZOOM)
    os_ = [osched(x) for x in scheds]
    t0 = time.time()

    def one(k):
        return ref.quantify_b1(os_, og, cfg, fps[k], list(workloads.CONFIG5_B1_STEPS), workloads.CONFIG5_B1_INIT)
    with cf.ThreadPoolExecutor(threads) as ex:
        r = list(ex.map(one, range(len(vox))))
    return dict(voxels=vox, ib=np.array([b for _, b in r], dtype=np.int64),
                ijk=np.array([[q.i1, q.i2, q.idf] for q, _ in r], dtype=np.int64),
                score=np.array([q.score for q, _ in r]), pd=np.array([q.pd for q, _ in r]),
                evals=np.array([q.evaluations for q, _ in r], dtype=np.int64), truth=idx,
                seconds=time.time() - t0)


def main():
    which = sys.argv[1]
    threads = int(sys.argv[2]) if len(sys.argv) > 2 else (os.cpu_count() or 1)
    ref = oracle.Oracle("reference")
    out = {"c2": run_c2, "c3": run_c3, "c4": run_c4, "c5": run_c5, "c5z": run_c5z}[which](ref, threads)
    out["threads"] = threads
    np.savez_compressed(os.path.join(HERE, f"scale_{which}.npz"), **out)
    print(json.dumps({k: (v if np.isscalar(v) else f"array{np.shape(v)}") for k, v in out.items()}))


if __name__ == "__main__":
    main()
