"""Seeded synthetic inputs for the BASELINE.json configurations.

No public dataset is involved: every schedule, phantom and noise sample is a
pure function of fixed seeds through the reference's counter RNG (rng.hpp).
Conventions that the reference does not define are stated here once:

* schedule: ``baseline_schedule(N, seed=1)``;
* grids are endpoint-inclusive (BASELINE.json counts), e.g. config 1 is
  96 x 29 x 21 = 58,464 atoms;
* voxel parameters "uniform on the grid": index ``rng_at(7, 20/21/22, v) % count``
  (the pattern of cli.cpp:335-337);
* config 2 phantom: 6 tissue classes (class params uniform on the grid from
  ``rng_at(11, 30/31/32, c)``), classes 1..5 are rotated ellipses drawn from
  ``uniform01(11, 33..37, c)`` painted over class 0 (all voxels in the mask),
  proton density 0.6 + 0.8 * uniform01(11, 38, c);
* config 4 phantom: three white fields ``rng::gaussian(13, 40+k, y*64+x)``,
  periodic Gaussian filter sigma = 3 voxels, each rescaled to [0, 1] and mapped
  affinely into T1 400-3000 ms, T2 40-300 ms, df -150..150 Hz, snapped to the
  1 ms / 0.5 ms / 0.1 Hz lattice; ZOOM settings ``CONFIG4_ZOOM``;
* noise: ``add_noise(pd*s, sigma, seed=1_000_000 + v)`` with
  sigma = ||pd*s||_2 / sqrt(N) / SNR per real channel.

* config 3 (materialized log-axis dictionary): T1 = geomspace(100, 4000, 300) ms,
  T2 = geomspace(10, 2000, 200) ms, df -100..100 step 5 Hz (41); voxel indices
  ``rng_at(7, axis, v) % count``; noise seed 5_000_000 + v, SNR 20;
* config 5 (B1): 13 schedules with flip_deg * B1, B1 = 0.70..1.30 step 0.05;
  voxel indices ``rng_at(11, axis, v) % count`` over (B1, T1, T2, df); noise
  seed 9_000_000 + v, SNR 25; the 4-D flat is b1 * A3 + flat3.

``simulate`` is injected ((schedule, params (k,3)) -> (k,N) complex128) so tests can make
the truth fingerprints with the CPU oracle and the benchmark with the GPU.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import dgs

CONFIGS = {
    1: dict(n=500, t1=(100, 2000, 20), t2=(20, 300, 10), df=(-50, 50, 5), nx=32, ny=32, snr=30.0,
            phantom="uniform"),
    2: dict(n=1000, t1=(100, 5000, 10), t2=(20, 2000, 5), df=(-250, 250, 1), nx=64, ny=64,
            snr=30.0, phantom="ellipses"),
    # config 4 is a ZOOM-only lattice (1 ms / 0.5 ms / 0.1 Hz)
    4: dict(n=1000, t1=(100, 5000, 1), t2=(20, 2000, 0.5), df=(-250, 250, 0.1), nx=64, ny=64,
            snr=30.0, phantom="smooth"),
}


@dataclass
class Workload:
    config: int
    schedule: dgs.Schedule
    grid: dgs.Grid
    nx: int
    ny: int
    truth: np.ndarray        # (V, 3) lattice indices
    pd: np.ndarray           # (V,)
    fps: np.ndarray          # (V, N) noisy complex128 queries
    snr: float
    meta: dict = field(default_factory=dict)

    @property
    def nvox(self) -> int:
        return self.fps.shape[0]


def uniform_truth(g: dgs.Grid, nvox: int, seed: int = 7) -> np.ndarray:
    out = np.empty((nvox, 3), dtype=np.int64)
    for v in range(nvox):
        out[v] = (dgs.rng_at(seed, 20, v) % g.t1_ms.count, dgs.rng_at(seed, 21, v) % g.t2_ms.count,
                  dgs.rng_at(seed, 22, v) % g.df_hz.count)
    return out


def ellipse_classes(nx: int, ny: int, nclass: int = 6, seed: int = 11) -> np.ndarray:
    cls = np.zeros((ny, nx), dtype=np.int64)
    yy, xx = np.mgrid[0:ny, 0:nx].astype(np.float64)
    for c in range(1, nclass):
        cx = 0.125 * nx + 0.75 * nx * dgs.uniform01(seed, 33, c)
        cy = 0.125 * ny + 0.75 * ny * dgs.uniform01(seed, 34, c)
        rx = 0.0625 * nx + 0.22 * nx * dgs.uniform01(seed, 35, c)
        ry = 0.0625 * ny + 0.22 * ny * dgs.uniform01(seed, 36, c)
        th = math.pi * dgs.uniform01(seed, 37, c)
        u = (xx - cx) * math.cos(th) + (yy - cy) * math.sin(th)
        w = -(xx - cx) * math.sin(th) + (yy - cy) * math.cos(th)
        cls[(u / rx) ** 2 + (w / ry) ** 2 <= 1.0] = c
    return cls.reshape(-1)


def smooth_fields(nx: int, ny: int, sigma: float = 3.0, seed: int = 13, nfields: int = 3) -> np.ndarray:
    """Config 4 phantom: Gaussian-filtered (sigma voxels, periodic) white fields
    from rng::gaussian(seed, 40+k, y*nx+x), each rescaled to [0, 1]."""
    r = int(np.ceil(3 * sigma))
    x = np.arange(-r, r + 1, dtype=np.float64)
    w = np.exp(-0.5 * (x / sigma) ** 2)
    w /= w.sum()
    out = np.empty((nfields, ny * nx))
    for k in range(nfields):
        g = np.array([dgs.gaussian(seed, 40 + k, i) for i in range(nx * ny)]).reshape(ny, nx)
        for axis in (0, 1):
            g = sum(wi * np.roll(g, s, axis=axis) for wi, s in zip(w, range(-r, r + 1)))
        g = g.reshape(-1)
        out[k] = (g - g.min()) / (g.max() - g.min())
    return out


# config 4 tissue ranges the smooth fields are mapped into [ms, ms, Hz]
CONFIG4_RANGES = ((400.0, 3000.0), (40.0, 300.0), (-150.0, 150.0))

# config 4 ZOOM settings (coarse 100 ms / 50 ms / 10 Hz, x10
# refinement per level, 3 levels), the same on the GPU and the reference.
CONFIG4_ZOOM = dict(df_coarse_hz=10.0, df_refine_hz=1.0, df_window_hz=20.0, omega_hz=82.0,
                    t1t2_2d_steps_ms=[100.0, 10.0], t1t2_1d_steps_ms=[50.0, 5.0, 1.0],
                    final_2d_step_ms=0.5)


def noisy(fps_clean: np.ndarray, snr: float, seed0: int = 1_000_000) -> np.ndarray:
    out = np.empty_like(fps_clean)
    n = fps_clean.shape[1]
    for v in range(fps_clean.shape[0]):
        sigma = float(np.sqrt(np.sum(np.abs(fps_clean[v]) ** 2))) / math.sqrt(n) / snr
        out[v] = dgs.add_noise(fps_clean[v], sigma, seed0 + v)
    return out


def make(config: int, simulate, nvox: int | None = None, n: int | None = None,
         grid_override: dgs.Grid | None = None) -> Workload:
    """Build config `config`'s inputs.  `nvox`/`n`/`grid_override` shrink it for tests."""
    c = CONFIGS[config]
    n = n or c["n"]
    sched = dgs.baseline_schedule(n, 1)
    g = grid_override or dgs.grid_inclusive(c["t1"], c["t2"], c["df"])
    nx, ny = c["nx"], c["ny"]
    V = nvox or nx * ny
    if c["phantom"] == "ellipses":
        cls = ellipse_classes(nx, ny)[:V]
        nclass = int(cls.max()) + 1 if V else 0
        ctruth = np.array([[dgs.rng_at(11, 30, k) % g.t1_ms.count, dgs.rng_at(11, 31, k) % g.t2_ms.count,
                            dgs.rng_at(11, 32, k) % g.df_hz.count] for k in range(max(nclass, 6))],
                          dtype=np.int64)
        cpd = np.array([0.6 + 0.8 * dgs.uniform01(11, 38, k) for k in range(max(nclass, 6))])
        truth = ctruth[cls]
        pd = cpd[cls]
        uniq, inv = np.unique(truth, axis=0, return_inverse=True)
        base = simulate(sched, np.stack(dgs.params_at(g, uniq[:, 0], uniq[:, 1], uniq[:, 2]), axis=1))
        clean = base[inv.reshape(-1)] * pd[:, None]
    elif c["phantom"] == "smooth":
        f = smooth_fields(nx, ny)[:, :V]
        truth = np.empty((V, 3), dtype=np.int64)
        for k, (ax, (lo, hi)) in enumerate(zip((g.t1_ms, g.t2_ms, g.df_hz), CONFIG4_RANGES)):
            truth[:, k] = np.clip(np.rint((lo + (hi - lo) * f[k] - ax.min) / ax.step), 0, ax.count - 1)
        pd = np.ones(V)
        clean = simulate(sched, np.stack(dgs.params_at(g, truth[:, 0], truth[:, 1], truth[:, 2]), axis=1))
    else:
        truth = uniform_truth(g, V)
        pd = np.ones(V)
        clean = simulate(sched, np.stack(dgs.params_at(g, truth[:, 0], truth[:, 1], truth[:, 2]), axis=1))
    fps = noisy(clean, c["snr"])
    return Workload(config, sched, g, nx, ny, truth, pd, fps, c["snr"],
                    meta=dict(atoms=dgs.grid_total(g)))


# --------------------------------------------------------------- config 3
CONFIG3 = dict(n=1000, nvox=16 * 128 * 128, snr=20.0, df=(-100.0, 5.0, 41))


def config3_axes():
    """(t1_ms, t2_ms, df (min, step, count)): log-spaced T1/T2, linear df."""
    return (np.geomspace(100.0, 4000.0, 300), np.geomspace(10.0, 2000.0, 200), CONFIG3["df"])


def config3_voxels(simulate, voxels) -> tuple:
    """Config 3 inputs for the given voxel ids -> (schedule, truth (V,3), fps (V,N))."""
    n = CONFIG3["n"]
    sched = dgs.baseline_schedule(n, 1)
    t1, t2, (dmin, dstep, dcnt) = config3_axes()
    voxels = np.asarray(voxels, dtype=np.int64)
    idx = np.array([[dgs.rng_at(7, ax, int(v)) % c for ax, c in enumerate((t1.size, t2.size, dcnt))]
                    for v in voxels], dtype=np.int64).reshape(-1, 3)
    prm = np.stack([t1[idx[:, 0]] * 1e-3, t2[idx[:, 1]] * 1e-3, dmin + idx[:, 2] * dstep], 1)
    fps = simulate(sched, prm) if len(voxels) else np.zeros((0, n), np.complex128)
    for k, v in enumerate(voxels):
        sig = float(np.sqrt(np.sum(np.abs(fps[k]) ** 2))) / math.sqrt(n) / CONFIG3["snr"]
        fps[k] = dgs.add_noise(fps[k], sig, 5_000_000 + int(v))
    return sched, idx, fps


# --------------------------------------------------------------- config 5
CONFIG5 = dict(n=3000, nvox=128 * 128, snr=25.0, b1=[round(0.7 + 0.05 * k, 10) for k in range(13)],
               t1=(100.0, 3000.0, 25.0), t2=(20.0, 500.0, 10.0), df=(-100.0, 100.0, 10.0))


# Four-parameter ZOOM on the config-5 lattice (T1 25 ms, T2 10 ms, df 10 Hz,
# B1 0.05): the three-parameter stages in lattice units (df coarse 1, omega
# 8; 2-D steps 8/4 x 20/10; 1-D 2/1 x 5/3; final 1 x 1), T2 started at
# 100 ms (the axis ends at 500 ms), and the outer B1 walk from B1 = 1.0
# (index 6) in steps of 0.2 then 0.05 (4, 1 index units).
CONFIG5_ZOOM = dict(df_coarse_hz=10.0, df_refine_hz=10.0, df_window_hz=20.0, omega_hz=82.0,
                    t1t2_2d_steps_ms=[200.0, 100.0], t1t2_1d_steps_ms=[50.0, 25.0], final_2d_step_ms=10.0,
                    init_t2_ms=100.0)
CONFIG5_B1_STEPS = (4, 1)
CONFIG5_B1_INIT = 6


def config5_schedules():
    base = dgs.baseline_schedule(CONFIG5["n"], 1)
    return [dgs.Schedule(base.flip_deg * b, base.phase_deg, base.tr_ms, base.te_ms) for b in CONFIG5["b1"]]


def config5_grid() -> dgs.Grid:
    return dgs.grid_inclusive(CONFIG5["t1"], CONFIG5["t2"], CONFIG5["df"])


def config5_voxels(simulate, voxels) -> tuple:
    """Config 5 inputs -> (schedules, grid, truth (V,4) = (b1, i1, i2, idf), fps (V,N)).
    ``simulate(schedule, params)`` is called once per B1 schedule present."""
    n = CONFIG5["n"]
    scheds = config5_schedules()
    g = config5_grid()
    counts = (len(scheds), g.t1_ms.count, g.t2_ms.count, g.df_hz.count)
    voxels = np.asarray(voxels, dtype=np.int64)
    idx = np.array([[dgs.rng_at(11, ax, int(v)) % c for ax, c in enumerate(counts)] for v in voxels],
                   dtype=np.int64).reshape(-1, 4)
    fps = np.zeros((len(voxels), n), dtype=np.complex128)
    for k, s in enumerate(scheds):
        sel = np.nonzero(idx[:, 0] == k)[0]
        if sel.size:
            prm = np.stack(dgs.params_at(g, idx[sel, 1], idx[sel, 2], idx[sel, 3]), axis=1)
            fps[sel] = simulate(s, prm)
    for k, v in enumerate(voxels):
        sig = float(np.sqrt(np.sum(np.abs(fps[k]) ** 2))) / math.sqrt(n) / CONFIG5["snr"]
        fps[k] = dgs.add_noise(fps[k], sig, 9_000_000 + int(v))
    return scheds, g, idx, fps
