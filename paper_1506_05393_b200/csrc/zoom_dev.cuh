// zoom_dev.cuh -- K5 device code (MRF-ZOOM), shared by the kernel
// translation units zoom_k_main.cu / zoom_k_rows.cu / zoom_k_var.cu (each
// instantiates a subset of the kernel variants, so ptxas runs them in
// parallel) and zoom.cu (host orchestration).  Everything here has internal
// linkage; the TUs meet only at zoom_launch.h.
//
// K5: MRF-ZOOM on sm_100a, one warp per voxel.
//
// Restates quantify_impl (reference proj/src/zoom.cpp:416-523) with its
// helpers search_df (:173-250), zoom_1d (:252-282), zoom_2d (:284-399) and
// the memoizing Objective (:41-150).  The decision logic runs warp-uniformly
// (every lane executes the same control flow on the same values); objective
// evaluations are what the lanes share out: before each decision the code
// names the points it will (or may, speculatively) need and the warp
// simulates the missing ones in parallel, one point per lane.  The decision
// code then reads the memo exactly in the reference's order, and only those
// reads count as evaluations ("unique acquisitions", zoom.cpp:94-123), so
// answers, scores and evaluation counts are the reference's.
//
// Certified screening.  A point is first evaluated by a single FP32 pass
// (zsim32, float host-libm tables; |error| <= 6e-8 measured against the FP64
// pipeline).  Every decision the reference takes on objective values (a > b,
// a < threshold, the plateau spread) is taken on those screening values only
// when they differ by more than a margin eps (1e-5, ~150x the error bound);
// otherwise the points involved are evaluated exactly -- the reference's FP64
// pipeline (simulate with host-libm tables => bit-identical fingerprint, FP64
// normalize, FP64 CC/Euclidean score, zoom.cpp:74-92, clamp at 1) -- and the
// decision is taken on exact values.  The decision sequence, the answer and
// the evaluation count are therefore the reference's; the reported score and
// PD are always exact.  MRFG_ZOOM_EPS=-1 evaluates everything in FP64.
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "mrfg_internal.cuh"
#include "sim64.cuh"
#include "zoom_launch.h"

namespace mrfg {
namespace {

constexpr unsigned long long kEmpty = ~0ull;
constexpr unsigned long long kAcq = 1ull << 63;  // "acquired" flag in the key word
constexpr int kPendCap = 256;                    // deferred exact evaluations per warp
constexpr int kEagerAfter = 6;                   // passes before certifying eagerly
constexpr int kDecCap = 256;                     // uncertified decisions recorded per pass

// An uncertified decision of the current pass (taken on screening values
// closer than the margin): what was compared and how it came out.  After the
// deferred points are exact the decisions are re-taken on exact values
// (zflipped); when none flips, the replay would walk the identical path -- the
// pass stands and the confirming replay is skipped.
struct ZDec {
    int kind;     // 0: a > b, 1: a < c, 2: spread(a, b, c) < eps
    int metric, outcome, sa, sb, sc;  // memo slots (-1: the constant kept in v*)
    double va, vb, vc;                // values at decision time; kind 1: vb = c, kind 2: eps in `eps`
    double eps;
};

// Memo slot.  `acc`/`are` are the single-pass FP32 screening values (CC
// magnitude and normalized real part); cc/euc/nrm2 are the reference's FP64
// values, present once nrm2 >= 0 ("exact").
struct ZSlot {
    unsigned long long key;
    float acc, are;
    double cc, euc, nrm2;
    // entry types (zoom.cpp:94-123): 0 = FP64 simulation, 1 = float
    // dictionary entry.  atype is fixed by this pass's first acquisition;
    // (cc, euc) are exact when computed for xtype == atype (0xFF: none yet).
    union {
        struct {
            unsigned int xtype;
            unsigned short atype, queued;
        };
        unsigned long long meta;  // one load for the exactness test
    };
};
__device__ __forceinline__ bool meta_exact(unsigned long long m) {
    return static_cast<unsigned int>(m) == static_cast<unsigned int>((m >> 32) & 0xFFFFu);
}

struct ZParams {
    // tables
    const double *rf, *e1d, *e2d, *phd;
    const float4 *su, *e1f, *phf;  // su: StepU rows (RF rotation, te, rest, one-df-step phasor)
    // screening step rows (staged in shared memory): su (sus = 4 float4 per
    // step), or for x-axis schedules (xr) the compact rows (r4, r5, r7, r8),
    // (wtc, wts, wrc, wrs) (sus = 2)
    const float4* sut;
    int sus, xr;
    const float2* e2f;
    double inv0[3];
    int n;
    Lattice L;
    // config (lattice units)
    int metric, final_metric, need_euc;
    long long df_coarse, df_refine, df_window_half, omega, fb_coarse, fb_window_half;
    double plateau_eps, heavy_cc;
    int n2d, n1d;
    long long s2d1[8], s2d2[8], s1d1[8], s1d2[8];
    long long f2d1, f2d2;
    long long init1, init2;  // snapped (not yet clamped) initial indices
    // speculation widths: 1-D flanks +-1..spec1d steps, 2-D (2*spec2d+1)^2 block
    long long spec1d, spec2d;
    long long spec1d_cta, spec2d_cta;  // the same with helper warps (CTA mode)
    // certification margins: |FP32 value - FP64 value| < eps (CC), eps_euc
    // (Euclidean); eps < 0 = every evaluation in FP64 (no screening)
    double eps, eps_euc;
    // data
    const double* fps;  // nvox x 2N raw
    // per-warp scratch (persistent warps, nwarps of them)
    double* q;          // nwarps x 2N normalized query
    float2* q32;        // nwarps x N normalized query, FP32
    double2* fpx;       // nwarps x N x 32 exact-evaluation fingerprints
    int* pend;          // nwarps x kPendCap deferred exact evaluations
    ZDec* dec;          // nwarps x kDecCap uncertified decisions of the current pass
    ZSlot* tab;         // nwarps x cap memo tables
    unsigned long long* next;  // voxel work counter
    // neighbour-seeded slice (row wavefront): rows of masked
    // raster voxels, row r = vox_list[row_start[r] .. row_start[r+1]); done[v]
    // flags finished voxels; prior windows in lattice units (zoom.cpp:600-605)
    int64_t nrows;
    const int64_t *row_start, *vox_list;
    int* done;
    long long pw1, pw2, pwdf;
    int smem_stage;            // StepU rows + per-warp q32 staged in dynamic shared memory
    int pit;                   // CTA mode: parallel-in-time screening of small rounds (x-axis rows)
    // several schedules in one launch (four-parameter ZOOM: one per B1
    // value): voxel v uses schedule vox_ib[v] -- its FP64 RF rows rf_b[] and
    // screening rows sut_b[] (the E1/E2/phasor tables do not depend on B1);
    // null: every voxel uses rf / sut
    const int* vox_ib;
    const double* rf_b[16];
    const float4* sut_b[16];
    int dict_mode;             // 0 none, 1 df dictionary (stage-1 acquisitions), 2 full dictionary
    // the caller's dictionary payload (zoom.cpp:101-113: entry idf of the df
    // slab, or the lattice flat of the full dictionary), scored as given;
    // null: the generated entries float(normalize(simulate)) are reproduced
    const float2* dict;
    // StageLog records (zoom.cpp:441-451), nvox x MRFG_TRACE_MAX, or null
    mrfg_stage* trace;
    int* trace_len;
    // smoothing (fingerprint.cpp:122-145): k = 0 (off), 3 or 5 taps, host-libm weights
    int smooth_k;
    double sw[5];
    float swf[5];
    // screening transcendentals: 0 float host-libm tables (default; audited
    // max |error| 2.9e-7); 1 MUFU ex2 + sin/cos (experimental, MRFG_ZOOM_SCREEN=mufu:
    // audited 4.5e-6, too close to eps to certify)
    int screen_mode;
    double t1_min, t1_step, t2_min, t2_step, df_min, df_step;  // lattice axes (ms, ms, Hz)
    unsigned int cap_mask;
    const long long* bounds;  // nvox x 6 or null (full bounds)
    const long long* inits;   // nvox x 2 or null
    int64_t nvox;
    mrfg_quant* out;
    int* err;
    // [fp32 evals, fp64 evals, fp64 rounds, near ties, sum cycles, max cycles,
    //  screening cycles, exact cycles, max |screening - exact| (double bits), passes] or null
    unsigned long long* stats;
    long long* vstats;  // nvox x 4: cycles, screening rounds' cycles, exact rounds, exact cycles
};

constexpr int kQCap = 256;  // queued evaluations per dispatch
struct ZItem {
    int kind;  // 0: screen one point, 1: screen a stride-1 df pair, 2: exact
    int s0, s1;
    int a, b, c;
};

struct Z {
    const ZParams* p;
    const double* rf;   // FP64 RF rows of this voxel's schedule
    ZSlot* tab;
    const double* q;
    const float2* q32;  // shared memory when staged
    const float4* rfs;  // StepU rows (4 float4 per step), shared memory when staged
    double2* fpx;       // exact-evaluation scratch: n x 32 lanes
    int* pend;          // deferred exact evaluations (memo slots), kPendCap
    int npend;          // warp-uniform
    ZDec* dec;          // uncertified decisions of this pass (kDecCap)
    int ndec;           // warp-uniform; > kDecCap: overflow
    int must_replay;    // the pass flushed mid-way or overflowed the record: replay it
    int eager;          // 1: certify each close decision immediately
    int stage1;         // inside search_df (df-dictionary acquisitions)
    int qw;             // shared-memory query slot (the voxel's warp in the block)
    int cta_w;          // CTA mode: warps evaluating this voxel's rounds (0 = own warp only)
    ZItem* queue;       // CTA mode: shared work queue (kQCap) and control words
    int* ctl;
    int lane;
    long long evals;
    int64_t vox;             // voxel being quantified (trace records)
    int ntrace;              // trace records of this pass
    long long tr_last;       // evaluation count at the previous record
    long long cyc32, cyc64;  // stats: cycles in screening / exact rounds
    long long r64;           // stats: exact rounds
    long long lo1, hi1, lo2, hi2, lodf, hidf;
};

__device__ __forceinline__ unsigned long long zkey(long long i1, long long i2, long long idf) {
    return (static_cast<unsigned long long>(i1) << 42) | (static_cast<unsigned long long>(i2) << 21) |
           static_cast<unsigned long long>(idf);
}
__device__ __forceinline__ void zunkey(unsigned long long k, int& i1, int& i2, int& idf) {
    k &= ~kAcq;
    i1 = static_cast<int>(k >> 42);
    i2 = static_cast<int>((k >> 21) & 0x1FFFFF);
    idf = static_cast<int>(k & 0x1FFFFF);
}
__device__ __forceinline__ unsigned int zhash(unsigned long long k) {
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdull;
    k ^= k >> 33;
    k *= 0xc4ceb9fe1a85ec53ull;
    k ^= k >> 33;
    return static_cast<unsigned int>(k);
}
__device__ __forceinline__ long long clampll(long long v, long long lo, long long hi) {
    return v < lo ? lo : (v > hi ? hi : v);
}
__device__ __forceinline__ void zsync() {
    __syncwarp();
    __threadfence_block();
    __syncwarp();
}
__device__ __forceinline__ void zstat(const Z& z, int k, unsigned long long v) {
    if (z.p->stats && v) atomicAdd(z.p->stats + k, v);
}

__device__ int zfind(const Z& z, unsigned long long key) {
    const unsigned int mask = z.p->cap_mask;
    unsigned int h = zhash(key) & mask;
    for (unsigned int probe = 0; probe <= mask; ++probe) {
        const unsigned long long k = *reinterpret_cast<volatile unsigned long long*>(&z.tab[h].key);
        if (k == kEmpty) return -1;
        if ((k & ~kAcq) == key) return static_cast<int>(h);
        h = (h + 1) & mask;
    }
    return -1;
}

// Claim a slot for key; returns slot and sets fresh when this lane claimed it.
__device__ int zclaim(const Z& z, unsigned long long key, bool& fresh) {
    const unsigned int mask = z.p->cap_mask;
    unsigned int h = zhash(key) & mask;
    for (unsigned int probe = 0; probe <= mask; ++probe) {
        const unsigned long long prev = atomicCAS(&z.tab[h].key, kEmpty, key);
        if (prev == kEmpty) {
            fresh = true;
            return static_cast<int>(h);
        }
        if ((prev & ~kAcq) == key) {
            fresh = false;
            return static_cast<int>(h);
        }
        h = (h + 1) & mask;
    }
    fresh = false;
    return -1;
}

// One exact objective evaluation: the reference's Objective::acquire +
// score_from_entry for both metrics, FP64, two passes (norm, then the
// normalized entry against the query).
// smooth (fingerprint.cpp:122-145) in place over v[0], v[st], ..., v[(n-1) st]
// (raw neighbours kept in a register window), the reference's tap order,
// edge truncation and division by the summed weights; returns sum |out|^2 in
// normalize's order (fingerprint.cpp:14-18).
__device__ double zsmooth64(const ZParams& P, double2* v, int st, int n) {
    const int h = P.smooth_k / 2;
    double2 win[5];  // raw values at i-h .. i+h
    for (int t = 0; t < 2 * h + 1; ++t) {
        const int idx = t - h;
        win[t] = idx >= 0 && idx < n ? v[static_cast<int64_t>(idx) * st] : make_double2(0.0, 0.0);
    }
    double acc = 0.0;
    for (int i = 0; i < n; ++i) {
        double re = 0.0, im = 0.0, ws = 0.0;
        for (int j = -h; j <= h; ++j) {
            const int t = i + j;
            if (t < 0 || t >= n) continue;
            const double w = P.sw[j + h];
            re = __dadd_rn(re, __dmul_rn(w, win[j + h].x));
            im = __dadd_rn(im, __dmul_rn(w, win[j + h].y));
            ws = __dadd_rn(ws, w);
        }
        const double2 o = make_double2(__ddiv_rn(re, ws), __ddiv_rn(im, ws));
        v[static_cast<int64_t>(i) * st] = o;
        acc = __dadd_rn(acc, __dadd_rn(__dmul_rn(o.x, o.x), __dmul_rn(o.y, o.y)));
        for (int t = 0; t < 2 * h; ++t) win[t] = win[t + 1];
        const int nx = i + h + 1;
        win[2 * h] = nx < n ? v[static_cast<int64_t>(nx) * st] : make_double2(0.0, 0.0);
    }
    return acc;
}

__device__ __noinline__ void zsim(const Z& z, int i1, int i2, int idf, bool dict, ZSlot& s) {
    const ZParams& P = *z.p;
    const int n = P.n;
    double2* fx = z.fpx + z.lane;
    double acc = 0.0, inv;
    bool cast = dict;
    if (dict && P.dict) {
        // the caller's entry d->entry(flat), as given (zoom.cpp:101-110):
        // scored without normalization unless smoothed; nrm2 < -1 marks "no
        // simulation norm" (estimate_pd then re-simulates, zoom.cpp:518)
        const int64_t flat = P.dict_mode == 2 ? (static_cast<int64_t>(i1) * P.L.n2 + i2) * P.L.ndf + idf : idf;
        const float2* e = P.dict + flat * n;
        for (int j = 0; j < n; ++j) {
            const float2 v = e[j];
            fx[32 * j] = make_double2(static_cast<double>(v.x), static_cast<double>(v.y));
        }
        acc = -2.0;
        inv = 1.0;
        cast = false;
        if (P.smooth_k) inv = 1.0 / sqrt(zsmooth64(P, fx, 32, n));
    } else {
        // pass 1: the recursion, |s|^2 in the reference's order (fingerprint.cpp:14-18);
        // the entries are kept (lane-interleaved scratch) for pass 2
        sim64_walk(z.rf, P.e1d, P.e2d, P.phd, P.inv0, n, P.L, i1, i2, idf, [&](int j, double x, double y) {
            acc = __dadd_rn(acc, __dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)));
            fx[32 * j] = make_double2(x, y);
        });
        inv = 1.0 / sqrt(acc);  // fingerprint.cpp:30-32
    }
    if (P.smooth_k && !(dict && P.dict)) {
        // entry = normalize(smooth(e)), e the raw simulation (zoom.cpp:116-118)
        // or the float dictionary entry (zoom.cpp:106-110)
        if (dict)
            for (int j = 0; j < n; ++j) {
                const double2 m = fx[32 * j];
                fx[32 * j] = make_double2(static_cast<double>(__double2float_rn(__dmul_rn(m.x, inv))),
                                          static_cast<double>(__double2float_rn(__dmul_rn(m.y, inv))));
            }
        inv = 1.0 / sqrt(zsmooth64(P, fx, 32, n));
        cast = false;
    }
    // pass 2: the normalized entry against the query (zoom.cpp:74-92)
    double re = 0.0, im = 0.0, dd = 0.0;
    const bool euc = P.need_euc;
    const double2* q = reinterpret_cast<const double2*>(z.q);
    for (int j = 0; j < n; ++j) {
        const double2 m = fx[32 * j];
        double er = __dmul_rn(m.x, inv), ei = __dmul_rn(m.y, inv);
        if (cast) {  // dictionary entry: float(normalized) (dictionary.cpp:44-51, zoom.cpp:106-108)
            er = static_cast<double>(__double2float_rn(er));
            ei = static_cast<double>(__double2float_rn(ei));
        }
        const double2 qq = q[j];
        re = __dadd_rn(re, __dadd_rn(__dmul_rn(qq.x, er), __dmul_rn(qq.y, ei)));  // zoom.cpp:79
        im = __dadd_rn(im, __dsub_rn(__dmul_rn(qq.y, er), __dmul_rn(qq.x, ei)));  // zoom.cpp:80
        if (euc) {
            const double dr = __dsub_rn(qq.x, er), di = __dsub_rn(qq.y, ei);  // zoom.cpp:87-89
            dd = __dadd_rn(dd, __dadd_rn(__dmul_rn(dr, dr), __dmul_rn(di, di)));
        }
    }
    const double v = sqrt(__dadd_rn(__dmul_rn(re, re), __dmul_rn(im, im)));
    s.cc = v < 1.0 ? v : 1.0;  // zoom.cpp:82-83
    s.euc = -sqrt(dd);          // zoom.cpp:91
    s.nrm2 = acc;
}

// One screening evaluation: single pass in FP32 over the host-libm float
// tables (same recursion, unnormalized entry), FP32 partial sums folded into
// FP64 every 16 steps.  Returns the CC magnitude and the normalized real
// part (Euclidean score = -sqrt(2 - 2 re)).  Measured |error| vs the FP64
// pipeline: <= 6e-8 (the certification margin eps is 1e-5).
struct Apx {
    float cc, re;
};
#ifndef MRFG_ZPF
#define MRFG_ZPF 24
#endif
constexpr int kZPf = MRFG_ZPF;  // L1 prefetch distance of the table streams, in steps (whole 128-byte lines)
// Packed f32x2 helpers: sm_100a executes fma/mul.rn.f32x2 as FFMA2/FMUL2 and
// folds a scalar broadcast, a half swap and a one-half negation into the
// operand selectors, so a complex product v*(c + i s) is 2 instructions.
typedef unsigned long long zf2;
__device__ __forceinline__ zf2 zpk(float a, float b) {
    zf2 r;
    asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void zup(zf2 v, float& a, float& b) {
    asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ zf2 zfma2(zf2 a, zf2 b, zf2 c) {
    zf2 d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ zf2 zmul2(zf2 a, zf2 b) {
    zf2 d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
// v*(c + i s) [+ acc]
__device__ __forceinline__ zf2 zcmul(zf2 v, float c, float s) {
    float x, y;
    zup(v, x, y);
    return zfma2(v, zpk(c, c), zmul2(zpk(y, x), zpk(-s, s)));
}
__device__ __forceinline__ zf2 zcmac(zf2 v, float c, float s, zf2 acc) {
    float x, y;
    zup(v, x, y);
    return zfma2(v, zpk(c, c), zfma2(zpk(y, x), zpk(-s, s), acc));
}

// One step of the FP32 screening recursion (bloch.hpp:34-38, bloch.cpp:22-26)
// and the CC partial sums.  The transverse state rotations and the query dot
// are complex products on f32x2 pairs (FFMA2/FMUL2): 20 FMA-pipe instructions
// per step instead of 29.  pq accumulates sum_j conj(q_j) s_j = (re, -im) of
// sum_j q_j conj(s_j) (same magnitude and real part); pn the two halves of |s|^2.
__device__ __forceinline__ void zstep32(const float4 ra, const float4 rb, const float4 rc,
                                        const float2 qq, const float4 e1, const float2 e2,
                                        const float4 ph, float& x, float& y, float& zz, zf2& pq,
                                        zf2& pn) {
    const float nx = fmaf(ra.x, x, fmaf(ra.y, y, ra.z * zz));
    const float ny = fmaf(ra.w, x, fmaf(rb.x, y, rb.y * zz));
    const float nz = fmaf(rb.z, x, fmaf(rb.w, y, rc.x * zz));
    // relax/precess over te: z' = z E1 + (1 - E1)
    const zf2 v = zmul2(zcmul(zpk(nx, ny), ph.x, ph.y), zpk(e2.x, e2.x));
    zz = fmaf(nz, e1.x, e1.y);
    pq = zcmac(v, qq.x, -qq.y, pq);
    pn = zfma2(v, v, pn);
    // over the rest of TR
    zup(zmul2(zcmul(v, ph.z, ph.w), zpk(e2.y, e2.y)), x, y);
    zz = fmaf(zz, e1.z, e1.w);
}

// x-axis pulses: RF = [[1,0,0],[0,r4,r5],[0,r7,r8]] (rx = (r4, r5, r7, r8)):
// 4 FFMA instead of 9; the rest as zstep32.
__device__ __forceinline__ void zstep32x(const float4 rx, const float2 qq, const float4 e1, const float2 e2,
                                         const float4 ph, float& x, float& y, float& zz, zf2& pq, zf2& pn) {
    const float ny = fmaf(rx.x, y, rx.y * zz);
    const float nz = fmaf(rx.z, y, rx.w * zz);
    const zf2 v = zmul2(zcmul(zpk(x, ny), ph.x, ph.y), zpk(e2.x, e2.x));
    zz = fmaf(nz, e1.x, e1.y);
    pq = zcmac(v, qq.x, -qq.y, pq);
    pn = zfma2(v, v, pn);
    zup(zmul2(zcmul(v, ph.z, ph.w), zpk(e2.y, e2.y)), x, y);
    zz = fmaf(zz, e1.z, e1.w);
}

// Parameter-major tables: the walk streams n consecutive entries per lane
// (rows warp-uniform where the lanes share T1, T2 or df).  The per-step
// uniform operands (StepU rows, query) come from shared memory (SMEM) or
// global.  Software pipeline: blocks of 4 steps in ping-pong register sets --
// the table entries of block b+1 load while block b computes.  The main loop
// runs whole 8-step pairs without guards (per-block pointers, immediate
// offsets; the tables carry tail padding for the last look-ahead), a guarded
// loop finishes n % 8 steps.
template <bool SMEM, bool XR>
__device__ __noinline__ Apx zsim32_tab(const Z& z, int i1, int i2, int idf) {
    constexpr int kB = 4;
    constexpr int S = XR ? 2 : 4;  // float4 per step row
    const ZParams& P = *z.p;
    const int n = P.n;
    const float4* __restrict__ e1p = P.e1f + static_cast<int64_t>(i1) * n;
    const float2* __restrict__ e2p = P.e2f + static_cast<int64_t>(i2) * n;
    const float4* __restrict__ php = P.phf + static_cast<int64_t>(idf) * n;
    extern __shared__ float4 zsm[];
    const float4* rfp = SMEM ? zsm : z.rfs;
    const float2* q = SMEM ? reinterpret_cast<const float2*>(zsm + S * n) +
                                 (z.cta_w ? 0 : static_cast<int>(threadIdx.x / 32)) * n
                           : z.q32;
    float x = static_cast<float>(P.inv0[0]), y = static_cast<float>(P.inv0[1]),
          zz = static_cast<float>(P.inv0[2]);
    double re = 0.0, im = 0.0, nn = 0.0;
    for (int j = 0; j < kZPf; j += 8) {
        prefetch_l1(e1p + j);
        prefetch_l1(php + j);
    }
    prefetch_l1(e2p);
    if (kZPf > 8) prefetch_l1(e2p + 16);
    float4 A1[kB], AP[kB], B1[kB], BP[kB];
    float2 A2[kB], B2[kB];
    auto load = [&](float4* E1, float2* E2, float4* PH, const float4* p1, const float2* p2, const float4* pp) {
#pragma unroll
        for (int m = 0; m < kB; ++m) {
            E1[m] = __ldg(p1 + m);
            PH[m] = __ldg(pp + m);
            E2[m] = __ldg(p2 + m);
        }
    };
    auto fold = [&](zf2 pq, zf2 pn) {  // FP32 partial sums into FP64
        float pr, pi, na, nb;
        zup(pq, pr, pi);
        zup(pn, na, nb);
        re += pr;
        im += pi;
        nn += na + nb;
    };
    auto run = [&](const float4* E1, const float2* E2, const float4* PH, const float4* r, const float2* qb) {
        zf2 pq = zpk(0.f, 0.f), pn = zpk(0.f, 0.f);
#pragma unroll
        for (int m = 0; m < kB; ++m) {
            if (XR)
                zstep32x(r[S * m], qb[m], E1[m], E2[m], PH[m], x, y, zz, pq, pn);
            else
                zstep32(r[S * m], r[S * m + 1], r[S * m + 2], qb[m], E1[m], E2[m], PH[m], x, y, zz, pq, pn);
        }
        fold(pq, pn);
    };
    const int nmain = n & ~(2 * kB - 1);
    load(A1, A2, AP, e1p, e2p, php);
    for (int jb = 0; jb < nmain; jb += 2 * kB) {
        if ((jb & 15) == 0) {  // one L1 prefetch per 128-byte line, 3 lines ahead
            prefetch_l1(e1p + jb + kZPf);
            prefetch_l1(e1p + jb + kZPf + 8);
            prefetch_l1(php + jb + kZPf);
            prefetch_l1(php + jb + kZPf + 8);
            prefetch_l1(e2p + jb + kZPf + 8);
        }
        load(B1, B2, BP, e1p + jb + kB, e2p + jb + kB, php + jb + kB);
        run(A1, A2, AP, rfp + S * jb, q + jb);
        load(A1, A2, AP, e1p + jb + 2 * kB, e2p + jb + 2 * kB, php + jb + 2 * kB);
        run(B1, B2, BP, rfp + S * (jb + kB), q + jb + kB);
    }
    {  // tail: n % 8 steps
        zf2 pq = zpk(0.f, 0.f), pn = zpk(0.f, 0.f);
        for (int j = nmain; j < n; ++j) {
            if (XR)
                zstep32x(rfp[S * j], q[j], __ldg(e1p + j), __ldg(e2p + j), __ldg(php + j), x, y, zz, pq, pn);
            else
                zstep32(rfp[S * j], rfp[S * j + 1], rfp[S * j + 2], q[j], __ldg(e1p + j), __ldg(e2p + j),
                        __ldg(php + j), x, y, zz, pq, pn);
        }
        fold(pq, pn);
    }
    const double inv = rsqrt(nn);
    Apx a;
    a.cc = static_cast<float>(fmin(sqrt(re * re + im * im) * inv, 1.0));
    a.re = static_cast<float>(re * inv);
    return a;
}

// Two adjacent off-resonance points (idf, idf + 1) of one (T1, T2) in one
// lane.  Every f32x2 register holds the SAME component of the two points
// (X = (x_a, x_b), ...), as in the K1 atom-pair producer: each operation of the
// recursion is one FFMA2/FMUL2 for both points with the step's scalars as
// broadcast operands, and no (x, y) packing is needed.  The second point's
// E2-scaled phasors are the first's times the one-df-step phasor w of the step
// row (scalar complex multiply), so the pair costs one table stream.  Per
// pair-step: 12 scalar FMA-pipe instructions (phasors) + 20 FFMA2/FMUL2
// (x-axis rows; 25 with a general RF matrix) against 38 + 6 register moves of
// the (x, y)-packed form it replaces; the FP32 partial sums are folded into
// FP64 every 16 steps.
struct Apx2 {
    Apx a, b;
};
__device__ __forceinline__ zf2 zneg2(zf2 v) { return v ^ 0x8000000080000000ull; }
__device__ __forceinline__ zf2 zbc(float s) { return zpk(s, s); }
template <bool SMEM, bool XR>
__device__ __noinline__ Apx2 zsim32_df2(const Z& z, int i1, int i2, int idf) {
    constexpr int kB = 2;
    constexpr int S = XR ? 2 : 4;  // float4 per step row
    const ZParams& P = *z.p;
    const int n = P.n;
    const float4* __restrict__ e1p = P.e1f + static_cast<int64_t>(i1) * n;
    const float2* __restrict__ e2p = P.e2f + static_cast<int64_t>(i2) * n;
    const float4* __restrict__ php = P.phf + static_cast<int64_t>(idf) * n;
    extern __shared__ float4 zsm[];
    const float4* rfp = SMEM ? zsm : z.rfs;
    const float2* q = SMEM ? reinterpret_cast<const float2*>(zsm + S * n) +
                                 (z.cta_w ? 0 : static_cast<int>(threadIdx.x / 32)) * n
                           : z.q32;
    const float x0 = static_cast<float>(P.inv0[0]), y0 = static_cast<float>(P.inv0[1]),
                z0 = static_cast<float>(P.inv0[2]);
    zf2 X = zpk(x0, x0), Y = zpk(y0, y0), Zc = zpk(z0, z0);
    zf2 DR = zpk(0.f, 0.f), DI = DR, NN = DR;  // sum conj(q) s (re, im) and |s|^2, both points
    double rea = 0.0, ima = 0.0, nna = 0.0, reb = 0.0, imb = 0.0, nnb = 0.0;
    for (int j = 0; j < kZPf; j += 8) {
        prefetch_l1(e1p + j);
        prefetch_l1(php + j);
    }
    prefetch_l1(e2p);
    if (kZPf > 8) prefetch_l1(e2p + 16);
    float4 A1[kB], AP[kB], B1[kB], BP[kB];
    float2 A2[kB], B2[kB];
    auto load = [&](float4* E1, float2* E2, float4* PH, const float4* p1, const float2* p2, const float4* pp) {
#pragma unroll
        for (int m = 0; m < kB; ++m) {
            E1[m] = __ldg(p1 + m);
            PH[m] = __ldg(pp + m);
            E2[m] = __ldg(p2 + m);
        }
    };
    // one step of both points (bloch.hpp:34-38, bloch.cpp:22-26)
    auto step2 = [&](const float4* r, const float2 qq, const float4 e1, const float2 e2, const float4 pa) {
        float4 w;  // one-df-step phasors: (wtc, wts) over te, (wrc, wrs) over the rest of TR
        zf2 nX, nY, nZ;
        if (XR) {  // r[0] = (r4, r5, r7, r8), r[1] = w
            const float4 rx = r[0];
            w = r[1];
            nX = X;
            nY = zfma2(Y, zbc(rx.x), zmul2(Zc, zbc(rx.y)));
            nZ = zfma2(Y, zbc(rx.z), zmul2(Zc, zbc(rx.w)));
        } else {
            const float4 ra = r[0], rb = r[1], rc = r[2], rd = r[3];
            w = make_float4(rc.w, rd.x, rd.y, rd.z);
            nX = zfma2(X, zbc(ra.x), zfma2(Y, zbc(ra.y), zmul2(Zc, zbc(ra.z))));
            nY = zfma2(X, zbc(ra.w), zfma2(Y, zbc(rb.x), zmul2(Zc, zbc(rb.y))));
            nZ = zfma2(X, zbc(rb.z), zfma2(Y, zbc(rb.w), zmul2(Zc, zbc(rc.x))));
        }
        // E2-scaled phasors: point a from the table row, point b = a * w
        const float cta = pa.x * e2.x, sta = pa.y * e2.x, cra = pa.z * e2.y, sra = pa.w * e2.y;
        const zf2 Ct = zpk(cta, fmaf(cta, w.x, -sta * w.y)), St = zpk(sta, fmaf(sta, w.x, cta * w.y));
        const zf2 Cr = zpk(cra, fmaf(cra, w.z, -sra * w.w)), Sr = zpk(sra, fmaf(sra, w.z, cra * w.w));
        // relax/precess over te: the echo sample; z' = z E1 + (1 - E1)
        const zf2 Xt = zfma2(zneg2(nY), St, zmul2(nX, Ct));
        const zf2 Yt = zfma2(nX, St, zmul2(nY, Ct));
        const zf2 Zt = zfma2(nZ, zbc(e1.x), zbc(e1.y));
        DR = zfma2(Xt, zbc(qq.x), zfma2(Yt, zbc(qq.y), DR));
        DI = zfma2(Yt, zbc(qq.x), zfma2(zneg2(Xt), zbc(qq.y), DI));
        NN = zfma2(Yt, Yt, zfma2(Xt, Xt, NN));
        // over the rest of TR
        X = zfma2(zneg2(Yt), Sr, zmul2(Xt, Cr));
        Y = zfma2(Xt, Sr, zmul2(Yt, Cr));
        Zc = zfma2(Zt, zbc(e1.z), zbc(e1.w));
    };
    auto fold = [&]() {  // FP32 partial sums into FP64
        float a, b;
        zup(DR, a, b);
        rea += a;
        reb += b;
        zup(DI, a, b);
        ima += a;
        imb += b;
        zup(NN, a, b);
        nna += a;
        nnb += b;
        DR = DI = NN = zpk(0.f, 0.f);
    };
    auto run = [&](const float4* E1, const float2* E2, const float4* PH, const float4* r, const float2* qb) {
#pragma unroll
        for (int m = 0; m < kB; ++m) step2(r + S * m, qb[m], E1[m], E2[m], PH[m]);
    };
    const int nmain = n & ~(2 * kB - 1);
    load(A1, A2, AP, e1p, e2p, php);
    for (int jb = 0; jb < nmain; jb += 2 * kB) {
        if ((jb & 7) == 0) {  // one L1 prefetch per 128-byte line, 3 lines ahead
            prefetch_l1(e1p + jb + kZPf);
            prefetch_l1(php + jb + kZPf);
            if ((jb & 15) == 0) {
                prefetch_l1(e2p + jb + kZPf + 8);
                fold();
            }
        }
        load(B1, B2, BP, e1p + jb + kB, e2p + jb + kB, php + jb + kB);
        run(A1, A2, AP, rfp + S * jb, q + jb);
        load(A1, A2, AP, e1p + jb + 2 * kB, e2p + jb + 2 * kB, php + jb + 2 * kB);
        run(B1, B2, BP, rfp + S * (jb + kB), q + jb + kB);
    }
    for (int j = nmain; j < n; ++j)  // tail: n % 4 steps
        step2(rfp + S * j, q[j], __ldg(e1p + j), __ldg(e2p + j), __ldg(php + j));
    fold();
    Apx2 r;
    double inv = rsqrt(nna);
    r.a.cc = static_cast<float>(fmin(sqrt(rea * rea + ima * ima) * inv, 1.0));
    r.a.re = static_cast<float>(rea * inv);
    inv = rsqrt(nnb);
    r.b.cc = static_cast<float>(fmin(sqrt(reb * reb + imb * imb) * inv, 1.0));
    r.b.re = static_cast<float>(reb * inv);
    return r;
}

// The same screening evaluation with the per-step transcendentals computed
// in registers instead of gathered (no per-lane memory streams): E = ex2(-dt
// log2(e) / T) (MUFU.EX2), phasors from the range-reduced turn count df*dt
// (MUFU.SIN/COS).  te/rest come from the StepU rows.
__device__ __noinline__ Apx zsim32_mufu(const Z& z, int i1, int i2, int idf) {
    const ZParams& P = *z.p;
    const int n = P.n;
    const float4* rfp = z.rfs;
    const float2* q = z.q32;
    const float k1 = static_cast<float>(-1.4426950408889634 / ((P.t1_min + i1 * P.t1_step) * 1e-3));
    const float k2 = static_cast<float>(-1.4426950408889634 / ((P.t2_min + i2 * P.t2_step) * 1e-3));
    const float df = static_cast<float>(P.df_min + idf * P.df_step);
    float x = static_cast<float>(P.inv0[0]), y = static_cast<float>(P.inv0[1]),
          zz = static_cast<float>(P.inv0[2]);
    double re = 0.0, im = 0.0, nn = 0.0;
    for (int jb = 0; jb < n; jb += 16) {
        float pr = 0.f, pi = 0.f, pn = 0.f;
        const int je = min(n, jb + 16);
        for (int j = jb; j < je; ++j) {
            const float4 ra = rfp[4 * j], rb = rfp[4 * j + 1], rc = rfp[4 * j + 2];
            const float2 qq = q[j];
            const float te = rc.y, rest = rc.z;
            const float e1t = exp2f(te * k1), e1r = exp2f(rest * k1);
            const float e2t = exp2f(te * k2), e2r = exp2f(rest * k2);
            // turn counts df*dt as exact two-products (hi + lo), reduced to [-0.5, 0.5]
            const float tth = df * te, trh = df * rest;
            const float tt = (tth - rintf(tth)) + fmaf(df, te, -tth);
            const float tr = (trh - rintf(trh)) + fmaf(df, rest, -trh);
            float st, ct, sr, cr;
            __sincosf(6.283185307179586f * tt, &st, &ct);
            __sincosf(6.283185307179586f * tr, &sr, &cr);
            // RF rotation (bloch.hpp:34-38)
            const float nx = fmaf(ra.x, x, fmaf(ra.y, y, ra.z * zz));
            const float ny = fmaf(ra.w, x, fmaf(rb.x, y, rb.y * zz));
            const float nz = fmaf(rb.z, x, fmaf(rb.w, y, rc.x * zz));
            // relax/precess over te (bloch.cpp:22-26)
            x = (nx * ct - ny * st) * e2t;
            y = (nx * st + ny * ct) * e2t;
            zz = fmaf(nz - 1.f, e1t, 1.f);
            pr = fmaf(qq.x, x, fmaf(qq.y, y, pr));
            pi = fmaf(qq.y, x, fmaf(-qq.x, y, pi));
            pn = fmaf(x, x, fmaf(y, y, pn));
            // over the rest of TR
            const float rx = (x * cr - y * sr) * e2r;
            const float ry = (x * sr + y * cr) * e2r;
            x = rx;
            y = ry;
            zz = fmaf(zz - 1.f, e1r, 1.f);
        }
        re += pr;
        im += pi;
        nn += pn;
    }
    const double inv = rsqrt(nn);
    Apx a;
    a.cc = static_cast<float>(fmin(sqrt(re * re + im * im) * inv, 1.0));
    a.re = static_cast<float>(re * inv);
    return a;
}

// Screening with smoothing (zoom.cpp:116-118): the FP32 recursion's raw echoes
// pass through a register window; the smoothed sample i - h (taps i-2h .. i,
// edge-truncated like fingerprint.cpp:133-143) is scored at step i, the last h
// samples after the walk.  Plain loop: smoothing is an analysis option.
__device__ __noinline__ Apx zsim32_smooth(const Z& z, int i1, int i2, int idf) {
    const ZParams& P = *z.p;
    const int n = P.n, h = P.smooth_k / 2;
    const float4* __restrict__ e1p = P.e1f + static_cast<int64_t>(i1) * n;
    const float2* __restrict__ e2p = P.e2f + static_cast<int64_t>(i2) * n;
    const float4* __restrict__ php = P.phf + static_cast<int64_t>(idf) * n;
    const float4* rfp = z.rfs;
    const float2* q = z.q32;
    float x = static_cast<float>(P.inv0[0]), y = static_cast<float>(P.inv0[1]),
          zz = static_cast<float>(P.inv0[2]);
    float2 win[5];
    for (int t = 0; t < 5; ++t) win[t] = make_float2(0.f, 0.f);
    double re = 0.0, im = 0.0, nn = 0.0;
    float pr = 0.f, pi = 0.f, pn = 0.f;
    auto emit = [&](int i) {  // window holds raw i-h .. i+h
        float sr = 0.f, si = 0.f, ws = 0.f;
        for (int t = -h; t <= h; ++t) {
            const int idx = i + t;
            if (idx < 0 || idx >= n) continue;
            sr = fmaf(P.swf[t + h], win[t + h].x, sr);
            si = fmaf(P.swf[t + h], win[t + h].y, si);
            ws += P.swf[t + h];
        }
        sr /= ws;
        si /= ws;
        const float2 qq = q[i];
        pr = fmaf(qq.x, sr, fmaf(qq.y, si, pr));
        pi = fmaf(qq.y, sr, fmaf(-qq.x, si, pi));
        pn = fmaf(sr, sr, fmaf(si, si, pn));
        if ((i & 15) == 15) {
            re += pr;
            im += pi;
            nn += pn;
            pr = pi = pn = 0.f;
        }
    };
    auto push = [&](float2 v) {
        for (int t = 0; t < 2 * h; ++t) win[t] = win[t + 1];
        win[2 * h] = v;
    };
    for (int j = 0; j < n; ++j) {
        const float4 ra = rfp[4 * j], rb = rfp[4 * j + 1], rc = rfp[4 * j + 2];
        const float4 e1 = __ldg(e1p + j), ph = __ldg(php + j);
        const float2 e2 = __ldg(e2p + j);
        const float nx = fmaf(ra.x, x, fmaf(ra.y, y, ra.z * zz));
        const float ny = fmaf(ra.w, x, fmaf(rb.x, y, rb.y * zz));
        const float nz = fmaf(rb.z, x, fmaf(rb.w, y, rc.x * zz));
        x = (nx * ph.x - ny * ph.y) * e2.x;
        y = (nx * ph.y + ny * ph.x) * e2.x;
        zz = fmaf(nz, e1.x, e1.y);
        push(make_float2(x, y));
        if (j >= h) emit(j - h);
        const float rx = (x * ph.z - y * ph.w) * e2.y;
        const float ry = (x * ph.w + y * ph.z) * e2.y;
        x = rx;
        y = ry;
        zz = fmaf(zz, e1.z, e1.w);
    }
    for (int i = n - h > 0 ? n - h : 0; i < n; ++i) {
        push(make_float2(0.f, 0.f));
        emit(i);
    }
    re += pr;
    im += pi;
    nn += pn;
    const double inv = rsqrt(nn);
    Apx a;
    a.cc = static_cast<float>(fmin(sqrt(re * re + im * im) * inv, 1.0));
    a.re = static_cast<float>(re * inv);
    return a;
}

__device__ __forceinline__ Apx zsim32(const Z& z, int i1, int i2, int idf) {
    const int m = z.p->screen_mode;
    if (z.p->smooth_k) return zsim32_smooth(z, i1, i2, idf);
    if (m == 1) return zsim32_mufu(z, i1, i2, idf);
    if (z.p->xr) return z.p->smem_stage ? zsim32_tab<true, true>(z, i1, i2, idf) : zsim32_tab<false, true>(z, i1, i2, idf);
    return z.p->smem_stage ? zsim32_tab<true, false>(z, i1, i2, idf) : zsim32_tab<false, false>(z, i1, i2, idf);
}

// ---------------------------------------------------------- helper warps
// CTA mode (z.cta_w > 0): warp 0 of the block runs the voxel's decision
// logic; every screening / exact round it needs is written to a shared-memory
// queue and evaluated by all cta_w warps between two named barriers (the
// helpers wait in zhelper_loop).  Without CTA mode a warp evaluates its own
// rounds in place.
__device__ __forceinline__ void zbar(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Screen (or, with eps < 0, evaluate exactly) lattice point (a, b, c) into a
// freshly claimed memo slot.
__device__ void zdo_screen(Z& z, int slot, int a, int b, int c) {
    if (z.p->eps < 0) {
        ZSlot s;
        zsim(z, a, b, c, false, s);
        z.tab[slot].cc = s.cc;
        z.tab[slot].euc = s.euc;
        z.tab[slot].nrm2 = s.nrm2;
        z.tab[slot].acc = static_cast<float>(s.cc);
        z.tab[slot].are = 0.f;
        z.tab[slot].xtype = 0;
        z.tab[slot].atype = 0;
        z.tab[slot].queued = 0;
        return;
    }
    const Apx v = zsim32(z, a, b, c);
    z.tab[slot].acc = v.cc;
    z.tab[slot].are = v.re;
    z.tab[slot].nrm2 = -1.0;
    z.tab[slot].xtype = 0xFFu;
    z.tab[slot].atype = 0;
    z.tab[slot].queued = 0;
    if (z.p->stats && (zhash(zkey(a, b, c) * 0x9E3779B97F4A7C15ull) & 63) == 0) {
        // audit (stats mode only): exact value of a random 1/64 of all
        // screened points, |error| into stats[10]
        ZSlot r;
        zsim(z, a, b, c, false, r);
        const double e = fabs(static_cast<double>(v.cc) - r.cc);
        atomicMax(z.p->stats + 10, static_cast<unsigned long long>(__double_as_longlong(e)));
        atomicAdd(z.p->stats + 11, 1ull);
    }
}

__device__ void zdo_pair(Z& z, int s0, int s1, int i1, int i2, int idf0);
__device__ void zdo_exact(Z& z, int s);
__device__ void zpit_point(Z& z, int slot, int i1, int i2, int idf);

// Evaluate queued items k = warp*32 + lane, stride 32 * cta_w (kind 3: one
// point per warp, screened parallel-in-time by all its lanes).
__device__ void zwork(Z& z, int m) {
    if (m > 0 && z.queue[0].kind == 3) {
        const int w = static_cast<int>(threadIdx.x / 32);
        if (w < m) {
            const ZItem it = z.queue[w];
            zpit_point(z, it.s0, it.a, it.b, it.c);
        }
        __threadfence_block();
        return;
    }
    for (int k = static_cast<int>(threadIdx.x / 32) * 32 + z.lane; k < m; k += 32 * z.cta_w) {
        const ZItem it = z.queue[k];
        if (it.kind == 0)
            zdo_screen(z, it.s0, it.a, it.b, it.c);
        else if (it.kind == 1)
            zdo_pair(z, it.s0, it.s1, it.a, it.b, it.c);
        else
            zdo_exact(z, it.s0);
    }
    __threadfence_block();
}

// Controller: evaluate the m queued items with all warps of the block.
__device__ void zdispatch(Z& z, int m) {
    if (z.lane == 0) {
        z.ctl[0] = 1;
        z.ctl[1] = m;
    }
    __syncwarp();
    zbar(1, 32 * z.cta_w);
    zwork(z, m);
    zbar(2, 32 * z.cta_w);
}

// Helper warps: evaluate dispatched rounds until the controller sends 0.
__device__ void zhelper_loop(Z& z) {
    for (;;) {
        zbar(1, 32 * z.cta_w);
        const int cmd = *reinterpret_cast<volatile int*>(z.ctl), m = *reinterpret_cast<volatile int*>(z.ctl + 1);
        if (cmd == 0) break;
        zwork(z, m);
        zbar(2, 32 * z.cta_w);
    }
}
__device__ void zhelpers_release(Z& z) {
    if (z.lane == 0) z.ctl[0] = 0;
    __syncwarp();
    zbar(1, 32 * z.cta_w);
}

// Append this lane's item (if has) to the queue; dispatch when nearly full.
__device__ __forceinline__ void zenqueue(Z& z, int& qn, bool has, const ZItem& it) {
    const unsigned int mm = __ballot_sync(0xffffffffu, has);
    if (has) z.queue[qn + __popc(mm & ((1u << z.lane) - 1u))] = it;
    qn += __popc(mm);
    if (qn > kQCap - 32) {
        zdispatch(z, qn);
        qn = 0;
    }
}

// Make sure the points pt(0..count-1) are in the memo (screened, not
// acquired).  Lanes split the missing points; duplicates are claimed once.
// With eps < 0 the points are evaluated exactly instead.
template <class PT>
__device__ void zensure(Z& z, long long count, PT pt) {
    int qn = 0;
    for (long long base = 0; base < count; base += 32) {
        const long long k = base + z.lane;
        bool mine = false;
        int slot = -1;
        long long a = 0, b = 0, c = 0;
        if (k < count) {
            pt(k, a, b, c);
            if (a >= 0 && b >= 0 && c >= 0 && a < z.p->L.n1 && b < z.p->L.n2 && c < z.p->L.ndf) {
                const unsigned long long key = zkey(a, b, c);
                if (zfind(z, key) < 0) {
                    slot = zclaim(z, key, mine);
                    if (slot < 0) atomicExch(z.p->err, 2);  // memo full
                }
            }
        }
        __syncwarp();
        if (z.cta_w && z.p->pit && qn == 0) {
            // a small round (<= one point per warp): each warp screens one
            // point with all its lanes, parallel in time (zpit_point)
            const unsigned int mm = __ballot_sync(0xffffffffu, mine);
            if (mm && __popc(mm) <= z.cta_w) {
                if (mine) z.queue[__popc(mm & ((1u << z.lane) - 1u))] =
                    ZItem{3, slot, -1, static_cast<int>(a), static_cast<int>(b), static_cast<int>(c)};
                __syncwarp();
                zdispatch(z, __popc(mm));
                continue;
            }
        }
        if (z.cta_w) {
            zenqueue(z, qn, mine, ZItem{0, slot, -1, static_cast<int>(a), static_cast<int>(b), static_cast<int>(c)});
            continue;
        }
        const long long t0 = z.p->stats ? clock64() : 0;
        if (mine) zdo_screen(z, slot, static_cast<int>(a), static_cast<int>(b), static_cast<int>(c));
        if (z.p->stats) {
            const unsigned int m = __ballot_sync(0xffffffffu, mine);
            if (z.lane == 0) zstat(z, z.p->eps < 0 ? 1 : 0, __popc(m));
            if (z.lane == 0 && m) {  // rounds / lanes in batches > 32 points (12, 13) or <= 32 (14, 15)
                zstat(z, count > 32 ? 12 : 14, 1);
                zstat(z, count > 32 ? 13 : 15, __popc(m));
            }
            __syncwarp();
            if (m) z.cyc32 += clock64() - t0;
        }
        zsync();
    }
    if (qn) zdispatch(z, qn);
}

// zensure for a stride-1 off-resonance run (i1, i2, a .. a + count - 1):
// each lane screens two adjacent points (zsim32_df2), 64 per round.
__device__ void zensure_df(Z& z, long long i1, long long i2, long long a, long long count) {
    const ZParams& P = *z.p;
    if (P.eps < 0 || P.screen_mode != 0 || P.smooth_k) {
        zensure(z, count, [&](long long k, long long& p1, long long& p2, long long& p3) {
            p1 = i1;
            p2 = i2;
            p3 = a + k;
        });
        return;
    }
    int qn = 0;
    for (long long base = 0; base < count; base += 64) {
        const long long k0 = base + 2 * z.lane;
        int slot[2] = {-1, -1};
        bool mine[2] = {false, false};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const long long c = a + k0 + h;
            if (k0 + h < count && c >= 0 && c < P.L.ndf && i1 >= 0 && i2 >= 0 && i1 < P.L.n1 && i2 < P.L.n2) {
                const unsigned long long key = zkey(i1, i2, c);
                if (zfind(z, key) < 0) {
                    slot[h] = zclaim(z, key, mine[h]);
                    if (slot[h] < 0) atomicExch(P.err, 2);  // memo full
                }
            }
        }
        // reconverge the warp before the evaluation: lanes leave the probe
        // loops above at different iterations
        __syncwarp();
        const int s0 = mine[0] ? slot[0] : -1, s1 = mine[1] ? slot[1] : -1;
        if (z.cta_w) {
            zenqueue(z, qn, s0 >= 0 || s1 >= 0,
                     ZItem{1, s0, s1, static_cast<int>(i1), static_cast<int>(i2), static_cast<int>(a + k0)});
            continue;
        }
        const long long t0 = P.stats ? clock64() : 0;
        if (s0 >= 0 || s1 >= 0) zdo_pair(z, s0, s1, static_cast<int>(i1), static_cast<int>(i2), static_cast<int>(a + k0));
        if (P.stats) {
            const unsigned int m0 = __ballot_sync(0xffffffffu, mine[0]), m1 = __ballot_sync(0xffffffffu, mine[1]);
            const unsigned int m = m0 | m1;
            if (z.lane == 0 && m) {
                zstat(z, 0, __popc(m0) + __popc(m1));
                zstat(z, 12, 1);
                zstat(z, 13, __popc(m0) + __popc(m1));
            }
            __syncwarp();
            if (m) z.cyc32 += clock64() - t0;
        }
        zsync();
    }
    if (qn) zdispatch(z, qn);
}

// Screen the stride-1 df pair (idf0, idf0 + 1) of (i1, i2) into the claimed
// slots s0 / s1 (-1: not this lane's).
__device__ void zdo_pair(Z& z, int s0, int s1, int i1, int i2, int idf0) {
    const ZParams& P = *z.p;
    // only row idf0 is read (the second point's phasor comes from the ladder)
    const int c0 = static_cast<int>(clampll(idf0, 0, P.L.ndf - 1));
    const Apx2 v = P.xr ? (P.smem_stage ? zsim32_df2<true, true>(z, i1, i2, c0) : zsim32_df2<false, true>(z, i1, i2, c0))
                        : (P.smem_stage ? zsim32_df2<true, false>(z, i1, i2, c0) : zsim32_df2<false, false>(z, i1, i2, c0));
    const int sl[2] = {s0, s1};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        if (sl[h] < 0) continue;
        ZSlot& t = z.tab[sl[h]];
        t.acc = h ? v.b.cc : v.a.cc;
        t.are = h ? v.b.re : v.a.re;
        t.nrm2 = -1.0;
        t.xtype = 0xFFu;
        t.atype = 0;
        t.queued = 0;
        if (P.stats && (zhash(zkey(i1, i2, idf0 + h) * 0x9E3779B97F4A7C15ull) & 63) == 0) {
            ZSlot r;  // audit (stats mode only), as in zdo_screen
            zsim(z, i1, i2, idf0 + h, false, r);
            const double e = fabs(static_cast<double>(h ? v.b.cc : v.a.cc) - r.cc);
            atomicMax(P.stats + 10, static_cast<unsigned long long>(__double_as_longlong(e)));
            atomicAdd(P.stats + 11, 1ull);
        }
    }
}

// Exact (reference FP64 pipeline) value of memo slot s for its entry type.
__device__ void zdo_exact(Z& z, int s) {
    volatile ZSlot* vs = &z.tab[s];
    int i1, i2, idf;
    zunkey(vs->key, i1, i2, idf);
    const unsigned int ty = vs->atype;
    ZSlot r;
    zsim(z, i1, i2, idf, ty == 1, r);
    if (z.p->stats) {
        const double e = fabs(static_cast<double>(z.tab[s].acc) - r.cc);
        atomicMax(z.p->stats + 8, static_cast<unsigned long long>(__double_as_longlong(e)));
    }
    z.tab[s].cc = r.cc;
    z.tab[s].euc = r.euc;
    z.tab[s].nrm2 = r.nrm2;
    z.tab[s].queued = 0;
    __threadfence_block();
    z.tab[s].xtype = ty;
}

// Parallel-in-time screening of ONE point by all 32 lanes of a warp (CTA
// mode, small rounds): lane k takes steps [kL, (k+1)L), L = ceil(n / 32):
//   1. the segment's affine map m -> G m + t (zstep32x's linear part: x-axis
//      RF rows, relax and precess over te and rest) is composed in FP32;
//   2. the start states are chained through the warp by shuffles (lane 0
//      starts from the inversion);
//   3. each lane re-walks its segment from its start state with zstep32x,
//      the CC partial sums reduced over the warp in FP64.
// Lane 0 writes the slot like zdo_screen.  Same tables and rounding order
// per step as the sequential walk; the composition adds FP32 rounding of the
// same order (audited in stats mode).
__device__ void zpit_point(Z& z, int slot, int i1, int i2, int idf) {
    const ZParams& P = *z.p;
    const int n = P.n;
    const int k = z.lane;
    const int L = (n + 31) / 32;
    const int j0 = min(n, k * L), j1 = min(n, j0 + L);
    const float4* __restrict__ e1p = P.e1f + static_cast<int64_t>(i1) * n;
    const float2* __restrict__ e2p = P.e2f + static_cast<int64_t>(i2) * n;
    const float4* __restrict__ php = P.phf + static_cast<int64_t>(idf) * n;
    extern __shared__ float4 zsm[];
    const float4* rfp = P.smem_stage ? zsm : z.rfs;  // x-axis rows: 2 float4 per step
    const float2* q = P.smem_stage ? reinterpret_cast<const float2*>(zsm + 2 * n) + z.qw * n : z.q32;
    // 1. compose: columns x0, y0, z0 and the constant column
    float gx[4] = {1.f, 0.f, 0.f, 0.f}, gy[4] = {0.f, 1.f, 0.f, 0.f}, gz[4] = {0.f, 0.f, 1.f, 0.f};
    for (int j = j0; j < j1; ++j) {
        const float4 rx = rfp[2 * j], e1 = __ldg(e1p + j), ph = __ldg(php + j);
        const float2 e2 = __ldg(e2p + j);
        const float tc = ph.x * e2.x, ts = ph.y * e2.x, rc = ph.z * e2.y, rs = ph.w * e2.y;
#pragma unroll
        for (int col = 0; col < 4; ++col) {
            const float X = gx[col], Y = gy[col], Zc = gz[col];
            const float ny = fmaf(rx.x, Y, rx.y * Zc), nz = fmaf(rx.z, Y, rx.w * Zc);
            const float x1 = fmaf(X, tc, -ny * ts), y1 = fmaf(X, ts, ny * tc);
            const float z1 = col == 3 ? fmaf(nz, e1.x, e1.y) : nz * e1.x;
            gx[col] = fmaf(x1, rc, -y1 * rs);
            gy[col] = fmaf(x1, rs, y1 * rc);
            gz[col] = col == 3 ? fmaf(z1, e1.z, e1.w) : z1 * e1.z;
        }
    }
    // 2. chain the start states
    float sx = static_cast<float>(P.inv0[0]), sy = static_cast<float>(P.inv0[1]), sz = static_cast<float>(P.inv0[2]);
    for (int it = 1; it < 32; ++it) {
        const float nx = fmaf(gx[0], sx, fmaf(gx[1], sy, fmaf(gx[2], sz, gx[3])));
        const float ny = fmaf(gy[0], sx, fmaf(gy[1], sy, fmaf(gy[2], sz, gy[3])));
        const float nz = fmaf(gz[0], sx, fmaf(gz[1], sy, fmaf(gz[2], sz, gz[3])));
        const float ux = __shfl_up_sync(0xffffffffu, nx, 1), uy = __shfl_up_sync(0xffffffffu, ny, 1),
                    uz = __shfl_up_sync(0xffffffffu, nz, 1);
        if (k == it) {
            sx = ux;
            sy = uy;
            sz = uz;
        }
    }
    // 3. re-walk the segment
    double re = 0.0, im = 0.0, nn = 0.0;
    {
        float x = sx, y = sy, zz = sz;
        zf2 pq = zpk(0.f, 0.f), pn = zpk(0.f, 0.f);
        for (int j = j0; j < j1; ++j) {
            zstep32x(rfp[2 * j], q[j], __ldg(e1p + j), __ldg(e2p + j), __ldg(php + j), x, y, zz, pq, pn);
            if (((j - j0) & 15) == 15 || j + 1 == j1) {
                float pr, pi, na, nb;
                zup(pq, pr, pi);
                zup(pn, na, nb);
                re += pr;
                im += pi;
                nn += na + nb;
                pq = zpk(0.f, 0.f);
                pn = zpk(0.f, 0.f);
            }
        }
    }
    for (int off = 16; off > 0; off >>= 1) {
        re += __shfl_xor_sync(0xffffffffu, re, off);
        im += __shfl_xor_sync(0xffffffffu, im, off);
        nn += __shfl_xor_sync(0xffffffffu, nn, off);
    }
    if (k == 0) {
        const double inv = rsqrt(nn);
        ZSlot& t = z.tab[slot];
        t.acc = static_cast<float>(fmin(sqrt(re * re + im * im) * inv, 1.0));
        t.are = static_cast<float>(re * inv);
        t.nrm2 = -1.0;
        t.xtype = 0xFFu;
        t.atype = 0;
        t.queued = 0;
        if (P.stats && (zhash(zkey(i1, i2, idf) * 0x9E3779B97F4A7C15ull) & 63) == 0) {
            ZSlot r;  // audit (stats mode only), as in zdo_screen
            zsim(z, i1, i2, idf, false, r);
            const double e = fabs(static_cast<double>(t.acc) - r.cc);
            atomicMax(P.stats + 10, static_cast<unsigned long long>(__double_as_longlong(e)));
            atomicAdd(P.stats + 11, 1ull);
        }
    }
    __syncwarp();
}

// Exact (FP64) evaluation of the memo slots named by slot_of(0..count-1)
// (-1 = none) that are still screened-only, one warp round per 32 slots.
template <class SL>
__device__ void zexact(Z& z, int count, SL slot_of) {
    int qn = 0;
    for (int base = 0; base < count; base += 32) {
        const int k = base + z.lane;
        const int s = k < count ? slot_of(k) : -1;
        const volatile ZSlot* vs = s >= 0 ? &z.tab[s] : nullptr;
        const bool work = vs && !meta_exact(vs->meta);
        if (z.cta_w) {
            zenqueue(z, qn, work, ZItem{2, s, -1, 0, 0, 0});
            continue;
        }
        const unsigned int m = __ballot_sync(0xffffffffu, work);
        if (!m) continue;
        const long long t0 = z.p->stats ? clock64() : 0;
        if (work) zdo_exact(z, s);
        if (z.lane == 0) {
            zstat(z, 1, __popc(m));
            zstat(z, 2, 1);
        }
        if (z.p->stats) {
            __syncwarp();
            z.cyc64 += clock64() - t0;
            ++z.r64;
        }
        zsync();
    }
    if (qn) zdispatch(z, qn);
}

// A decision value: the memo slot it came from and whether it is the exact
// (reference) value or the FP32 screening value.
struct V {
    double v;
    int slot;
    int exact;
};

__device__ __forceinline__ V zread(const Z& z, int s, int metric) {
    const volatile ZSlot* vs = &z.tab[s];
    if (meta_exact(vs->meta)) return {metric == MRFG_METRIC_CC ? vs->cc : vs->euc, s, 1};
    if (metric == MRFG_METRIC_CC) return {static_cast<double>(vs->acc), s, 0};
    const double d = 2.0 - 2.0 * static_cast<double>(vs->are);
    return {-sqrt(d > 0.0 ? d : 0.0), s, 0};
}

// Entry type of an acquisition now (zoom.cpp:101-113): dictionary entries in
// full-dictionary mode, and in df-dictionary mode during search_df.
__device__ __forceinline__ int zentry_type(const Z& z) {
    return z.p->dict_mode == 2 || (z.p->dict_mode == 1 && z.stage1) ? 1 : 0;
}

// Objective::eval (zoom.cpp:125-138): range check, memo read, acquisition count.
__device__ V zf(Z& z, long long i1, long long i2, long long idf, int metric) {
    const ZParams& P = *z.p;
    if (i1 < 0 || i2 < 0 || idf < 0 || i1 >= P.L.n1 || i2 >= P.L.n2 || idf >= P.L.ndf) {
        atomicExch(P.err, 1);
        return {-1e300, -1, 1};
    }
    const unsigned long long key = zkey(i1, i2, idf);
    int s = zfind(z, key);
    if (s < 0) {
        zensure(z, 1, [&](long long, long long& a, long long& b, long long& c) {
            a = i1;
            b = i2;
            c = idf;
        });
        s = zfind(z, key);
        if (s < 0) return {-1e300, -1, 1};
    }
    const unsigned long long kk = *reinterpret_cast<volatile unsigned long long*>(&z.tab[s].key);
    if (!(kk & kAcq)) {
        __syncwarp();
        if (z.lane == 0) {
            z.tab[s].atype = static_cast<unsigned short>(zentry_type(z));
            z.tab[s].key = kk | kAcq;
        }
        zsync();
        ++z.evals;
        // all-FP64 mode (the entry type may differ), and payload dictionary
        // entries: their screening value approximates the simulation, not
        // the caller's bytes, so they are scored exactly on acquisition
        if (P.eps < 0 || (P.dict && zentry_type(z) == 1)) zexact(z, 1, [&](int) { return s; });
    }
    return zread(z, s, metric);
}

__device__ __forceinline__ double zmargin(const Z& z, int metric) {
    return metric == MRFG_METRIC_CC ? z.p->eps : z.p->eps_euc;
}

// Make a value exact (FP64) in place.
__device__ void zmake_exact(Z& z, V& a, int metric) {
    if (a.exact) return;
    const int s = a.slot;
    zexact(z, 1, [&](int) { return s; });
    a = zread(z, s, metric);
}

// Evaluate every deferred slot exactly, 32 per warp round.
__device__ void zflush(Z& z) {
    zsync();
    const int* pend = z.pend;
    zexact(z, z.npend, [&](int k) { return pend[k]; });
    z.npend = 0;
}

// Queue a slot without an exact value for exact evaluation (once).
__device__ void zdefer(Z& z, const V& a) {
    if (a.exact || a.slot < 0) return;
    volatile ZSlot* vs = &z.tab[a.slot];
    const unsigned long long m = vs->meta;
    if ((m >> 48) || meta_exact(m)) return;
    __syncwarp();
    if (z.lane == 0) {
        vs->queued = 1;
        z.pend[z.npend] = a.slot;
    }
    zsync();
    if (++z.npend == kPendCap) {
        zflush(z);
        z.must_replay = 1;  // later decisions of this pass saw exact values the earlier ones did not
    }
}

__device__ void zrecord(Z& z, int kind, int metric, bool outcome, const V& a, const V* b, const V* c, double cval,
                        double eps) {
    if (z.ndec < kDecCap) {
        if (z.lane == 0) {
            ZDec d;
            d.kind = kind;
            d.metric = metric;
            d.outcome = outcome ? 1 : 0;
            d.sa = a.slot;
            d.va = a.v;
            d.sb = b ? b->slot : -1;
            d.vb = b ? b->v : cval;
            d.sc = c ? c->slot : -1;
            d.vc = c ? c->v : 0.0;
            d.eps = eps;
            z.dec[z.ndec] = d;
        }
    } else {
        z.must_replay = 1;
    }
    ++z.ndec;
}

// Re-take the pass's uncertified decisions on the (now exact) values; true
// when any comes out differently.
__device__ bool zflipped(Z& z) {
    zsync();
    bool flip = false;
    const int nd = z.ndec < kDecCap ? z.ndec : kDecCap;
    for (int k = z.lane; k < nd; k += 32) {
        const ZDec d = z.dec[k];
        const double a = d.sa >= 0 ? zread(z, d.sa, d.metric).v : d.va;
        const double b = d.sb >= 0 ? zread(z, d.sb, d.metric).v : d.vb;
        bool r;
        if (d.kind == 0) {
            r = a > b;
        } else if (d.kind == 1) {
            r = a < d.vb;
        } else {
            const double c = d.sc >= 0 ? zread(z, d.sc, d.metric).v : d.vc;
            const double mn = fmin(a, fmin(b, c)), mx = fmax(a, fmax(b, c));
            r = (mx - mn) < d.eps;
        }
        flip |= r != (d.outcome != 0);
    }
    return __any_sync(0xffffffffu, flip);
}

// The reference's `a > b` on objective values.  Screening values decide when
// the two differ by more than the certification margin (the FP64 values are
// then ordered the same way).  A closer decision is uncertified: eagerly, both
// points are evaluated exactly first; optimistically (the default), the
// screening order is used for now and both points are queued -- the search is
// then replayed once they are exact (zoom_voxel), until a pass takes every
// decision certified.
__device__ bool gt(Z& z, V& a, V& b, int metric) {
    if (!(a.exact && b.exact) && fabs(a.v - b.v) <= zmargin(z, metric)) {
        if (z.lane == 0) zstat(z, 3, 1);
        if (!z.eager) {
            zrecord(z, 0, metric, a.v > b.v, a, &b, nullptr, 0.0, 0.0);
            zdefer(z, a);
            zdefer(z, b);
            return a.v > b.v;
        }
        const int sa = a.exact ? -1 : a.slot, sb = b.exact ? -1 : b.slot;
        zexact(z, 2, [&](int k) { return k == 0 ? sa : sb; });
        if (sa >= 0) a = zread(z, sa, metric);
        if (sb >= 0) b = zread(z, sb, metric);
    }
    return a.v > b.v;
}
// `a < c` against a constant threshold.
__device__ bool lt_const(Z& z, V& a, double c, int metric) {
    if (!a.exact && fabs(a.v - c) <= zmargin(z, metric)) {
        if (!z.eager) {
            zrecord(z, 1, metric, a.v < c, a, nullptr, nullptr, c, 0.0);
            zdefer(z, a);
            return a.v < c;
        }
        zmake_exact(z, a, metric);
    }
    return a.v < c;
}

struct Best {
    long long idx;
    V val;
};
__device__ __forceinline__ Best best_init() { return {-1, {-1e300, -1, 1}}; }
__device__ __forceinline__ void offer(Z& z, Best& b, long long i, V v, int metric) {
    if (gt(z, v, b.val, metric)) {
        b.val = v;
        b.idx = i;
    }
}

// ------------------------------------------------------------- StageLog
// One trace record (log_stage, zoom.cpp:441-451): evaluations added since
// the previous record, the stage's best value and lattice point.  A value
// that is still a screening value keeps its memo slot in `pad` and is made
// exact when the voxel finishes (ztrace_finish).
__device__ void znote(Z& z, int stage, long long i1, long long i2, long long idf, const V& v) {
    const ZParams& P = *z.p;
    if (!P.trace) return;
    if (z.lane == 0 && z.ntrace < MRFG_TRACE_MAX) {
        mrfg_stage* r = P.trace + z.vox * MRFG_TRACE_MAX + z.ntrace;
        r->stage = stage;
        r->pad = v.exact ? -1 : v.slot;
        r->evaluations = z.evals - z.tr_last;
        r->best = v.v;
        r->t1_ms = __dadd_rn(P.t1_min, __dmul_rn(static_cast<double>(i1), P.t1_step));  // AxisSpec::value
        r->t2_ms = __dadd_rn(P.t2_min, __dmul_rn(static_cast<double>(i2), P.t2_step));
        r->df_hz = __dadd_rn(P.df_min, __dmul_rn(static_cast<double>(idf), P.df_step));
    }
    ++z.ntrace;
    z.tr_last = z.evals;
}
// Exact values for the final pass's records (their slots' entry types are
// the reference's), then the count.
__device__ void ztrace_finish(Z& z) {
    const ZParams& P = *z.p;
    if (!P.trace) return;
    mrfg_stage* rec = P.trace + z.vox * MRFG_TRACE_MAX;
    const int nt = z.ntrace < MRFG_TRACE_MAX ? z.ntrace : MRFG_TRACE_MAX;
    zsync();
    zexact(z, nt, [&](int k) { return static_cast<int>(*reinterpret_cast<volatile int*>(&rec[k].pad)); });
    if (z.lane == 0) {
        for (int k = 0; k < nt; ++k) {
            const int s = rec[k].pad;
            if (s >= 0)
                rec[k].best = zread(z, s, rec[k].stage == MRFG_STAGE_T1T2_FINAL ? P.final_metric : P.metric).v;
            rec[k].pad = 0;
        }
        P.trace_len[z.vox] = z.ntrace;
    }
    zsync();
}

// Offer the points pt(0..count-1) to bst in order: the reference's
// per-point eval + offer (zoom.cpp:125-138, 182-187) with the memo reads done
// 32 points at a time -- each lane looks up one point and takes its
// acquisition (atomic, so a point is counted once), then the offers run in
// order over the lanes' values (warp shuffles).  Decisions and counts are
// those of the one-at-a-time loop.
template <class PT>
__device__ void offer_batch(Z& z, Best& bst, long long count, PT pt, int metric) {
    const ZParams& P = *z.p;
    for (long long base = 0; base < count; base += 32) {
        const long long k = base + z.lane;
        const bool valid = k < count;
        long long a = 0, b = 0, c = 0;
        int s = -1;
        bool inrange = false;
        if (valid) {
            pt(k, a, b, c);
            inrange = a >= 0 && b >= 0 && c >= 0 && a < P.L.n1 && b < P.L.n2 && c < P.L.ndf;
            if (!inrange) atomicExch(P.err, 1);
            else s = zfind(z, zkey(a, b, c));
        }
        if (__ballot_sync(0xffffffffu, valid && inrange && s < 0)) {  // not screened yet
            zensure(z, count - base < 32 ? count - base : 32,
                    [&](long long kk, long long& p1, long long& p2, long long& p3) { pt(base + kk, p1, p2, p3); });
            if (valid && inrange) s = zfind(z, zkey(a, b, c));
        }
        bool newly = false;
        if (s >= 0) {
            const unsigned long long old = atomicOr(&z.tab[s].key, kAcq);
            newly = !(old & kAcq);
            if (newly) z.tab[s].atype = static_cast<unsigned short>(zentry_type(z));
        }
        z.evals += __popc(__ballot_sync(0xffffffffu, newly));
        zsync();
        if (P.eps < 0 || (P.dict && zentry_type(z) == 1))  // as in zf
            zexact(z, 32, [&](int) { return s; });
        V v{-1e300, -1, 1};
        if (s >= 0) v = zread(z, s, metric);
        const int nv = count - base < 32 ? static_cast<int>(count - base) : 32;
        for (int l = 0; l < nv; ++l) {
            V vl;
            vl.v = __shfl_sync(0xffffffffu, v.v, l);
            vl.slot = __shfl_sync(0xffffffffu, v.slot, l);
            vl.exact = __shfl_sync(0xffffffffu, v.exact, l);
            offer(z, bst, __shfl_sync(0xffffffffu, c, l), vl, metric);
        }
    }
}

// ------------------------------------------------------------ search_df
// zoom.cpp:182-187 (scan: also evaluates the clamped end)
__device__ void df_scan(Z& z, long long i1, long long i2, long long a, long long b, long long step,
                        Best& bst) {
    a = clampll(a, z.lodf, z.hidf);
    b = clampll(b, z.lodf, z.hidf);
    const long long cnt = b >= a ? (b - a) / step + 1 : 0;
    const bool extra = b >= a && (b - a) % step != 0;
    auto pt = [&](long long k, long long& p1, long long& p2, long long& pd) {
        p1 = i1;
        p2 = i2;
        pd = k < cnt ? a + k * step : b;
    };
    const int metric = z.p->metric;
    if (step == 1)
        zensure_df(z, i1, i2, a, cnt);
    else
        zensure(z, cnt + (extra ? 1 : 0), pt);
    offer_batch(z, bst, cnt + (extra ? 1 : 0), pt, metric);
}

// zoom.cpp:199-204: the last three marks span less than eps.  The screening
// spread is within 2 margins of the exact one; closer than that to the
// threshold the three marks are evaluated exactly.
__device__ bool plateau(Z& z, V* marks, int nm, double eps) {
    if (nm < 3) return false;
    const int metric = z.p->metric;
    auto spread = [&]() {
        double mn = marks[nm - 3].v, mx = mn;
        for (int j = nm - 3; j < nm; ++j) {
            mn = fmin(mn, marks[j].v);
            mx = fmax(mx, marks[j].v);
        }
        return mx - mn;
    };
    double s = spread();
    const bool all_exact = marks[nm - 3].exact && marks[nm - 2].exact && marks[nm - 1].exact;
    if (!all_exact && fabs(s - eps) <= 2.0 * zmargin(z, metric)) {
        if (!z.eager) {
            zrecord(z, 2, metric, s < eps, marks[nm - 3], &marks[nm - 2], &marks[nm - 1], 0.0, eps);
            for (int j = nm - 3; j < nm; ++j) zdefer(z, marks[j]);
            return s < eps;
        }
        const int a = marks[nm - 3].exact ? -1 : marks[nm - 3].slot;
        const int b = marks[nm - 2].exact ? -1 : marks[nm - 2].slot;
        const int c = marks[nm - 1].exact ? -1 : marks[nm - 1].slot;
        zexact(z, 3, [&](int k) { return k == 0 ? a : (k == 1 ? b : c); });
        for (int j = nm - 3; j < nm; ++j)
            if (marks[j].slot >= 0) marks[j] = zread(z, marks[j].slot, metric);
        s = spread();
    }
    return s < eps;
}

// zoom.cpp:189-241
__device__ Best df_run(Z& z, long long i1, long long i2, long long coarse, long long wh) {
    const ZParams& P = *z.p;
    V marks[16];
    int nm = 0;
    Best cur = best_init();
    df_scan(z, i1, i2, z.lodf, z.hidf, coarse, cur);
    znote(z, MRFG_STAGE_DF_COARSE, i1, i2, cur.idx, cur.val);
    marks[nm++] = cur.val;
    {
        Best r = cur;
        df_scan(z, i1, i2, cur.idx - wh, cur.idx + wh, P.df_refine, r);
        cur = r;
    }
    znote(z, MRFG_STAGE_DF_REFINE, i1, i2, cur.idx, cur.val);
    marks[nm++] = cur.val;
    for (int round = 0; round < 8; ++round) {
        Best t = cur;
        const long long nf = cur.idx + P.omega <= z.hidf ? (z.hidf - cur.idx) / P.omega : 0;
        const long long nb = cur.idx - P.omega >= z.lodf ? (cur.idx - z.lodf) / P.omega : 0;
        const long long c0 = cur.idx;
        auto hop = [&](long long k, long long& p1, long long& p2, long long& pd) {
            p1 = i1;
            p2 = i2;
            pd = k < nf ? c0 + (k + 1) * P.omega : c0 - (k - nf + 1) * P.omega;
        };
        zensure(z, nf + nb, hop);
        offer_batch(z, t, nf + nb, hop, P.metric);  // forward hops, then backward (zoom.cpp:213-220)
        znote(z, MRFG_STAGE_DF_TRANSLATE, i1, i2, t.idx, t.val);
        if (t.idx == cur.idx) break;
        Best r = t;
        df_scan(z, i1, i2, t.idx - wh, t.idx + wh, P.df_refine, r);
        cur = r;
        znote(z, MRFG_STAGE_DF_REREFINE, i1, i2, cur.idx, cur.val);
        marks[nm++] = cur.val;
        if (plateau(z, marks, nm, P.plateau_eps)) {
            znote(z, MRFG_STAGE_DF_PLATEAU_STOP, i1, i2, cur.idx, cur.val);
            return cur;
        }
    }
    if (plateau(z, marks, nm, P.plateau_eps)) {
        znote(z, MRFG_STAGE_DF_PLATEAU_STOP, i1, i2, cur.idx, cur.val);
        return cur;
    }
    Best fin = cur;
    df_scan(z, i1, i2, cur.idx - P.omega / 2, cur.idx + P.omega / 2, 1, fin);
    znote(z, MRFG_STAGE_DF_FINEST, i1, i2, fin.idx, fin.val);
    return fin;
}

// zoom.cpp:173-250
__device__ long long search_df(Z& z, long long i1, long long i2) {
    const ZParams& P = *z.p;
    Best mainb = df_run(z, i1, i2, P.df_coarse, P.df_window_half);
    if (lt_const(z, mainb.val, P.heavy_cc, P.metric)) {
        Best fb = df_run(z, i1, i2, P.fb_coarse, P.fb_window_half);
        znote(z, MRFG_STAGE_DF_FALLBACK, i1, i2, fb.idx, fb.val);
        if (gt(z, fb.val, mainb.val, P.metric)) return fb.idx;
    }
    return mainb.idx;
}

// ------------------------------------------------------------- zoom_1d
// zoom.cpp:252-282 along T1 (axis 0) or T2 (axis 1); speculative flanks
// +-1..spec1d steps are screened together before each decision.
__device__ long long zoom_1d(Z& z, int axis, long long i1, long long i2, long long idf, long long lo,
                             long long hi, long long init, long long s, int metric) {
    auto F = [&](long long a) {
        return axis == 0 ? zf(z, a, i2, idf, metric) : zf(z, i1, a, idf, metric);
    };
    long long x = clampll(init, lo, hi);
    V fx = F(x);
    for (;;) {
        const long long x0 = x;
        auto pt = [&](long long k, long long& a, long long& b, long long& c) {
            const long long off = (k / 2 + 1) * s * ((k & 1) ? 1 : -1);
            const long long v = clampll(x0 + off, lo, hi);
            a = axis == 0 ? v : i1;
            b = axis == 0 ? i2 : v;
            c = idf;
        };
        zensure(z, 2 * (z.cta_w ? z.p->spec1d_cta : z.p->spec1d), pt);
        const long long xl = clampll(x - s, lo, hi);
        if (xl != x) {
            V fl = F(xl);
            if (gt(z, fl, fx, metric)) {
                x = xl;
                fx = fl;
                continue;
            }
        }
        const long long xr = clampll(x + s, lo, hi);
        if (xr != x) {
            V fr = F(xr);
            if (gt(z, fr, fx, metric)) {
                x = xr;
                fx = fr;
                continue;
            }
        }
        break;
    }
    return x;
}

// ------------------------------------------------------------- zoom_2d
// zoom.cpp:284-399 for one step pair; the (2r+1)^2 neighbourhood is
// screened together before each iteration's probes.
__device__ void zoom_2d_step(Z& z, long long idf, int metric, long long& x, long long& y, V& fc,
                             long long& bx, long long& by, V& bf, long long s1, long long s2) {
    const long long lo1 = z.lo1, hi1 = z.hi1, lo2 = z.lo2, hi2 = z.hi2;
    auto F = [&](long long a, long long b) { return zf(z, a, b, idf, metric); };
    auto note = [&](long long px, long long py, V& v) {
        if (gt(z, v, bf, metric)) {
            bf = v;
            bx = px;
            by = py;
        }
    };
    const long long cap = 4 * ((hi1 - lo1) / s1 + (hi2 - lo2) / s2) + 16;
    bool converged = false;
    // Cycle detection (Brent).  The move taken from (x, y) depends only on
    // (x, y) -- fc is always F(x, y) and objective values are fixed -- so a
    // revisited position means the walk is periodic and never converges:
    // the reference keeps cycling until `cap` and then falls back to the
    // best point noted (zoom.cpp:392-396).  When the repeat is seen, one
    // full period has been walked since the saved position, so every point
    // of the cycle has been noted, no later iteration evaluates a new point
    // or changes the best: leaving now gives the reference's answer and
    // evaluation count without walking the remaining periods.
    long long sx = x, sy = y, power = 1, lam = 0;
    for (long long iter = 0; iter < cap && !converged; ++iter) {
        if (iter > 0) {
            if (x == sx && y == sy) break;  // periodic: not converged
            if (++lam == power) {
                sx = x;
                sy = y;
                power *= 2;
                lam = 0;
            }
        }
        const long long cx = x, cy = y;
        const long long r = z.cta_w ? z.p->spec2d_cta : z.p->spec2d, w = 2 * r + 1;  // (2r+1)^2 - 1 neighbours
        zensure(z, w * w - 1, [&](long long k, long long& a, long long& b, long long& c) {
            const long long kk = k < (w * w) / 2 ? k : k + 1;  // skip the centre
            a = clampll(cx + (kk % w - r) * s1, lo1, hi1);
            b = clampll(cy + (kk / w - r) * s2, lo2, hi2);
            c = idf;
        });
        const long long xl = clampll(x - s1, lo1, hi1);
        const long long xr = clampll(x + s1, lo1, hi1);
        const long long yd = clampll(y - s2, lo2, hi2);
        const long long yu = clampll(y + s2, lo2, hi2);
        V fl = fc, fd = fc;
        if (xl != x) {
            fl = F(xl, y);
            note(xl, y, fl);
        }
        if (yd != y) {
            fd = F(x, yd);
            note(x, yd, fd);
        }
        const bool lw = xl != x && gt(z, fl, fc, metric);
        const bool dw = yd != y && gt(z, fd, fc, metric);
        if (lw && dw) {
            x = xl;
            y = yd;
            fc = F(x, y);
            note(x, y, fc);
            continue;
        }
        if (!lw && !dw) {
            V fr = fc, fu = fc;
            if (xr != x) {
                fr = F(xr, y);
                note(xr, y, fr);
            }
            if (yu != y) {
                fu = F(x, yu);
                note(x, yu, fu);
            }
            const bool rw = xr != x && gt(z, fr, fc, metric);
            const bool uw = yu != y && gt(z, fu, fc, metric);
            if (rw && uw) {
                x = xr;
                y = yu;
                fc = F(x, y);
                note(x, y, fc);
                continue;
            }
            if (rw) {
                x = xr;
                fc = fr;
                continue;
            }
            if (uw) {
                y = yu;
                fc = fu;
                continue;
            }
            converged = true;
            continue;
        }
        if (lw) {
            V fu = fc;
            if (yu != y) {
                fu = F(x, yu);
                note(x, yu, fu);
            }
            if (yu != y && gt(z, fu, fc, metric)) {
                x = xl;
                y = yu;
                fc = F(x, y);
                note(x, y, fc);
                continue;
            }
            x = xl;
            fc = fl;
            continue;
        }
        V fr = fc;
        if (xr != x) {
            fr = F(xr, y);
            note(xr, y, fr);
        }
        if (xr != x && gt(z, fr, fc, metric)) {
            x = xr;
            y = yd;
            fc = F(x, y);
            note(x, y, fc);
            continue;
        }
        y = yd;
        fc = fd;
    }
    if (!converged) {  // zoom.cpp:392-396
        x = bx;
        y = by;
        fc = bf;
    }
}

__device__ void zoom_2d(Z& z, long long idf, int metric, long long& x, long long& y,
                        const long long* s1v, const long long* s2v, int ns) {
    x = clampll(x, z.lo1, z.hi1);
    y = clampll(y, z.lo2, z.hi2);
    V fc = zf(z, x, y, idf, metric);
    long long bx = x, by = y;
    V bf = fc;
    for (int k = 0; k < ns; ++k) zoom_2d_step(z, idf, metric, x, y, fc, bx, by, bf, s1v[k], s2v[k]);
}

// ------------------------------------------------------------ the kernel
// b6: (lo1, hi1, lo2, hi2, lodf, hidf) or null (full lattice); s1, s2: the
// snapped, not yet clamped initial indices (zoom.cpp:428-429).
__device__ void zoom_voxel(Z& z, const ZParams& P, int64_t v, const long long* b6, long long s1,
                           long long s2) {
    z.evals = 0;
    z.vox = v;
    if (P.vox_ib) {  // this voxel's schedule (the staged rows are off in this mode)
        const int ib = P.vox_ib[v];
        z.rf = P.rf_b[ib];
        z.rfs = P.sut_b[ib];
    }
    z.cyc32 = z.cyc64 = z.r64 = 0;
    const long long tstart = clock64();
    const int n = P.n;
    const double* fp = P.fps + v * 2 * n;
    double* q = const_cast<double*>(z.q);
    float2* q32 = const_cast<float2*>(z.q32);
    // memo reset
    for (unsigned int s = z.lane; s <= P.cap_mask; s += 32) z.tab[s].key = kEmpty;
    // normalize the query (fingerprint.cpp:14-37): sequential FP64 sum,
    // computed redundantly by every lane (identical bits)
    double acc = 0.0;
    for (int j = 0; j < n; ++j)
        acc = __dadd_rn(acc, __dadd_rn(__dmul_rn(fp[2 * j], fp[2 * j]), __dmul_rn(fp[2 * j + 1], fp[2 * j + 1])));
    const double nq = sqrt(acc);
    if (nq == 0) {
        if (z.lane == 0) atomicExch(P.err, 3);
        return;
    }
    if (P.smooth_k) {
        // query = normalize(smooth(fp)) (zoom.cpp:49-50); pd keeps |fp| (zoom.cpp:518)
        for (int j = z.lane; j < 2 * n; j += 32) q[j] = fp[j];
        zsync();
        double accs = 0.0;
        if (z.lane == 0) accs = zsmooth64(P, reinterpret_cast<double2*>(q), 1, n);
        accs = __shfl_sync(0xffffffffu, accs, 0);
        zsync();
        const double invs = 1.0 / sqrt(accs);
        for (int j = z.lane; j < 2 * n; j += 32) q[j] = __dmul_rn(q[j], invs);
        zsync();
        for (int j = z.lane; j < n; j += 32)
            q32[j] = make_float2(static_cast<float>(q[2 * j]), static_cast<float>(q[2 * j + 1]));
    } else {
        const double inv = 1.0 / nq;
        for (int j = z.lane; j < 2 * n; j += 32) q[j] = __dmul_rn(fp[j], inv);
        for (int j = z.lane; j < n; j += 32)
            q32[j] = make_float2(static_cast<float>(__dmul_rn(fp[2 * j], inv)),
                                 static_cast<float>(__dmul_rn(fp[2 * j + 1], inv)));
    }
    zsync();

    if (b6) {
        z.lo1 = b6[0];
        z.hi1 = b6[1];
        z.lo2 = b6[2];
        z.hi2 = b6[3];
        z.lodf = b6[4];
        z.hidf = b6[5];
    } else {
        z.lo1 = 0;
        z.hi1 = P.L.n1 - 1;
        z.lo2 = 0;
        z.hi2 = P.L.n2 - 1;
        z.lodf = 0;
        z.hidf = P.L.ndf - 1;
    }
    long long i1 = 0, i2 = 0, idf = 0;
    z.eager = P.eps < 0 ? 1 : 0;
    z.npend = 0;
    for (int pass = 0;; ++pass) {
        if (pass > 0) {
            // replay: the memo (values, exactness) persists; acquisitions and
            // the evaluation count restart
            for (unsigned int t = z.lane; t <= P.cap_mask; t += 32) {
                const unsigned long long k = z.tab[t].key;
                if (k != kEmpty && (k & kAcq)) z.tab[t].key = k & ~kAcq;
            }
            zsync();
        }
        if (pass >= kEagerAfter) z.eager = 1;
        z.ndec = 0;
        z.must_replay = 0;
        z.evals = 0;
        z.ntrace = 0;
        z.tr_last = 0;
        i1 = clampll(s1, z.lo1, z.hi1);  // zoom.cpp:428-429
        i2 = clampll(s2, z.lo2, z.hi2);
        // Stage 1 (zoom.cpp:465-469)
        z.stage1 = 1;
        idf = search_df(z, i1, i2);
        z.stage1 = 0;
        // Stage 2 (zoom.cpp:472-479)
        zoom_2d(z, idf, P.metric, i1, i2, P.s2d1, P.s2d2, P.n2d);
        znote(z, MRFG_STAGE_T1T2_2D, i1, i2, idf, zf(z, i1, i2, idf, P.metric));
        // Stage 3 (zoom.cpp:482-489)
        {
            Best b = best_init();
            const long long a = clampll(idf - P.omega / 2, z.lodf, z.hidf);
            const long long e = clampll(idf + P.omega / 2, z.lodf, z.hidf);
            const long long c1 = i1, c2 = i2;
            auto pt = [&](long long k, long long& p1, long long& p2, long long& pd) {
                p1 = c1;
                p2 = c2;
                pd = a + k;
            };
            zensure_df(z, c1, c2, a, e - a + 1);
            offer_batch(z, b, e - a + 1, pt, P.metric);
            idf = b.idx;
            znote(z, MRFG_STAGE_DF_SWEEP, i1, i2, idf, b.val);
        }
        // Stage 4 (zoom.cpp:492-501)
        for (int k = 0; k < P.n1d; ++k) {
            i1 = zoom_1d(z, 0, i1, i2, idf, z.lo1, z.hi1, i1, P.s1d1[k], P.metric);
            znote(z, MRFG_STAGE_T1_1D, i1, i2, idf, zf(z, i1, i2, idf, P.metric));
            i2 = zoom_1d(z, 1, i1, i2, idf, z.lo2, z.hi2, i2, P.s1d2[k], P.metric);
            znote(z, MRFG_STAGE_T2_1D, i1, i2, idf, zf(z, i1, i2, idf, P.metric));
        }
        // Stage 5 (zoom.cpp:505-512)
        zoom_2d(z, idf, P.final_metric, i1, i2, &P.f2d1, &P.f2d2, 1);
        znote(z, MRFG_STAGE_T1T2_FINAL, i1, i2, idf, zf(z, i1, i2, idf, P.final_metric));
        if (z.lane == 0) zstat(z, 9, 1);
        if (z.npend == 0) break;  // every decision of this pass was certified
        zflush(z);
        // the uncertified decisions re-taken on exact values: when none flips,
        // the replay would repeat this pass step for step (same acquisitions,
        // same trace), so the pass stands
        if (!z.must_replay && !zflipped(z)) break;
    }
    // result (zoom.cpp:514-519): the exact score of the answer
    V score = zf(z, i1, i2, idf, P.metric);
    zmake_exact(z, score, P.metric);
    const int s = score.slot;
    ztrace_finish(z);
    // estimate_pd (fingerprint.cpp:147-152) divides by the SIMULATED entry's
    // norm (Objective::ideal_at, zoom.cpp:152-156): a payload dictionary
    // entry has none, so simulate it once
    double nrm2 = z.tab[s].nrm2;
    if (nrm2 < -1.0) {
        ZSlot t;
        zsim(z, static_cast<int>(i1), static_cast<int>(i2), static_cast<int>(idf), false, t);
        nrm2 = __shfl_sync(0xffffffffu, t.nrm2, 0);
    }
    if (z.lane == 0) {
        mrfg_quant r;
        r.i1 = i1;
        r.i2 = i2;
        r.idf = idf;
        r.t1_ms = 0;  // filled on the host (exact axis values)
        r.t2_ms = 0;
        r.df_hz = 0;
        // estimate_pd (fingerprint.cpp:147-152): |fp| / |ideal|, ideal unnormalized
        r.pd = nq / sqrt(nrm2);
        r.score = score.v;
        r.evaluations = z.evals;
        P.out[v] = r;
        if (P.stats) {
            const unsigned long long dt = static_cast<unsigned long long>(clock64() - tstart);
            atomicAdd(P.stats + 4, dt);
            atomicMax(P.stats + 5, dt);
            atomicAdd(P.stats + 6, static_cast<unsigned long long>(z.cyc32));
            atomicAdd(P.stats + 7, static_cast<unsigned long long>(z.cyc64));
            long long* vs = P.vstats + 4 * v;
            vs[0] = static_cast<long long>(dt);
            vs[1] = z.cyc32;
            vs[2] = z.r64;
            vs[3] = z.cyc64;
        }
    }
    zsync();
}

// Persistent warps: each warp owns a memo table and scratch and pulls voxels
// from a work counter until the slice is done (no per-voxel memory, dynamic
// balance of the very uneven per-voxel work).
// Per-warp state and scratch; stages the StepU rows in shared memory (every
// thread of the block takes part).
__device__ void zwarp_setup(Z& z, const ZParams& P, int64_t w) {
    z.p = &P;
    z.rf = P.rf;
    z.lane = threadIdx.x % 32;
    z.tab = P.tab + w * (static_cast<int64_t>(P.cap_mask) + 1);
    z.q = P.q + w * 2 * P.n;
    z.fpx = P.fpx + w * P.n * 32;
    z.pend = P.pend + w * kPendCap;
    z.dec = P.dec + w * kDecCap;
    z.stage1 = 0;
    z.qw = static_cast<int>(threadIdx.x / 32);
    z.cta_w = 0;
    z.queue = nullptr;
    z.ctl = nullptr;
    extern __shared__ float4 zsm[];
    if (P.smem_stage) {
        for (int i = threadIdx.x; i < P.sus * P.n; i += blockDim.x) zsm[i] = P.sut[i];
        __syncthreads();
        z.rfs = zsm;
        z.q32 = reinterpret_cast<float2*>(zsm + P.sus * P.n) + z.qw * P.n;
    } else {
        z.rfs = P.sut;
        z.q32 = P.q32 + w * P.n;
    }
}

template <int BS, int MINB>
__global__ void __launch_bounds__(BS, MINB) k_zoom(const ZParams P) {
    const int64_t w = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / 32;
    Z z;
    zwarp_setup(z, P, w);
    for (;;) {
        unsigned long long v = 0;
        if (z.lane == 0) v = atomicAdd(P.next, 1ull);
        v = __shfl_sync(0xffffffffu, v, 0);
        if (v >= static_cast<unsigned long long>(P.nvox)) break;
        const int64_t vv = static_cast<int64_t>(v);
        zoom_voxel(z, P, vv, P.bounds ? P.bounds + 6 * vv : nullptr, P.inits ? P.inits[2 * vv] : P.init1,
                   P.inits ? P.inits[2 * vv + 1] : P.init2);
    }
}

// Prior window around a finished voxel (zoom.cpp:595-610; the host
// restatement is prior_of in abi.cu): parameters round-trip through seconds
// like QuantResult::params, snap, intersect with the full lattice.
__device__ void zprior(const ZParams& P, int64_t prev, long long* b, long long& s1, long long& s2) {
    const volatile mrfg_quant* pr = P.out + prev;
    const long long i1 = pr->i1, i2 = pr->i2, idf = pr->idf;
    const double t1 = __dmul_rn(__dmul_rn(__dadd_rn(P.t1_min, __dmul_rn(static_cast<double>(i1), P.t1_step)), 1e-3), 1e3);
    const double t2 = __dmul_rn(__dmul_rn(__dadd_rn(P.t2_min, __dmul_rn(static_cast<double>(i2), P.t2_step)), 1e-3), 1e3);
    const double df = __dadd_rn(P.df_min, __dmul_rn(static_cast<double>(idf), P.df_step));
    const long long p1 = llround(__ddiv_rn(__dsub_rn(t1, P.t1_min), P.t1_step));
    const long long p2 = llround(__ddiv_rn(__dsub_rn(t2, P.t2_min), P.t2_step));
    const long long pd = llround(__ddiv_rn(__dsub_rn(df, P.df_min), P.df_step));
    s1 = p1;  // snap_index(init_t1_ms = t1) (zoom.cpp:596, 428)
    s2 = p2;
    b[0] = max(0ll, p1 - P.pw1);
    b[1] = min(static_cast<long long>(P.L.n1 - 1), p1 + P.pw1);
    b[2] = max(0ll, p2 - P.pw2);
    b[3] = min(static_cast<long long>(P.L.n2 - 1), p2 + P.pw2);
    b[4] = max(0ll, pd - P.pwdf);
    b[5] = min(static_cast<long long>(P.L.ndf - 1), pd + P.pwdf);
}

// Neighbour-seeded slice in one launch: warp r walks raster row r left to
// right, each voxel seeded by its left neighbour; a row's first voxel by the
// first voxel of the row above (the permitted relaxation of the raster
// order).  Rows wait only on lower rows' first voxels, and all
// rows are co-resident (host check), so the spin-waits always finish.
template <int BS>
__global__ void __launch_bounds__(BS, 1) k_zoom_rows(const ZParams P) {
    // one row per block: warp 0 decides, all BS/32 warps evaluate (CTA mode);
    // memo, queries and deferred list are the controller's (scratch index
    // r * W), the FP64 fingerprint scratch is per warp
    constexpr int W = BS / 32;
    const int warp = static_cast<int>(threadIdx.x / 32);
    const int64_t r = blockIdx.x;
    Z z;
    zwarp_setup(z, P, r * W + warp);
    const int64_t ctrl = r * W;
    z.tab = P.tab + ctrl * (static_cast<int64_t>(P.cap_mask) + 1);
    z.q = P.q + ctrl * 2 * P.n;
    z.pend = P.pend + ctrl * kPendCap;
    z.dec = P.dec + ctrl * kDecCap;
    extern __shared__ float4 zsm[];
    z.qw = 0;
    if (P.smem_stage)
        z.q32 = reinterpret_cast<float2*>(zsm + P.sus * P.n);
    else
        z.q32 = P.q32 + ctrl * P.n;
    if (W > 1) {
        z.cta_w = W;
        z.queue = reinterpret_cast<ZItem*>(reinterpret_cast<float2*>(zsm + P.sus * P.n) + P.n);
        z.ctl = reinterpret_cast<int*>(z.queue + kQCap);
    }
    if (r >= P.nrows) return;  // whole block
    if (warp != 0) {
        zhelper_loop(z);
        return;
    }
    const int64_t k0 = P.row_start[r], k1 = P.row_start[r + 1];
    for (int64_t k = k0; k < k1; ++k) {
        const int64_t v = P.vox_list[k];
        const int64_t prev = k > k0 ? P.vox_list[k - 1] : (r > 0 ? P.vox_list[P.row_start[r - 1]] : -1);
        long long b[6], s1 = P.init1, s2 = P.init2;
        const long long* bp = nullptr;
        if (prev >= 0) {
            if (z.lane == 0)
                while (*reinterpret_cast<volatile int*>(P.done + prev) == 0) __nanosleep(256);
            __syncwarp();
            __threadfence();
            zprior(P, prev, b, s1, s2);
            bp = b;
        }
        zoom_voxel(z, P, v, bp, s1, s2);
        if (z.lane == 0) {
            __threadfence();
            *reinterpret_cast<volatile int*>(P.done + v) = 1;
        }
        __syncwarp();
    }
    if (W > 1) zhelpers_release(z);
}

// One kernel variant: shared-memory opt-in (per device), occupancy, launch.
template <class K>
void zoom_run_variant(K kern, const void* params, bool launch, unsigned grid, int block, size_t smem,
                      cudaStream_t s, int* occupancy) {
    MRFG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    if (occupancy) MRFG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(occupancy, kern, block, smem));
    if (launch) {
        kern<<<grid, block, smem, s>>>(*static_cast<const ZParams*>(params));
        MRFG_CUDA(cudaGetLastError());
    }
}

[[maybe_unused]] long long snap_index(double value, const mrfg_axis& ax) {  // zoom.cpp:407-409
    return std::lround((value - ax.min) / ax.step);
}
[[maybe_unused]] long long step_units(double step_value, double finest) {  // zoom.cpp:411-414
    long long u = std::lround(step_value / finest);
    return u > 0 ? u : 1;
}

}  // namespace

}  // namespace mrfg
