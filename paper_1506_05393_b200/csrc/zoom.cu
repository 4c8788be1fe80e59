// zoom.cu -- K5: MRF-ZOOM on sm_100a, one warp per voxel.
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
// Each evaluation is the reference's FP64 pipeline: simulate (sim64.cuh,
// host-libm tables => bit-identical fingerprint), FP64 normalize, FP64 CC and
// Euclidean score (zoom.cpp:74-92), clamp at 1.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "mrfg_internal.cuh"
#include "sim64.cuh"

namespace mrfg {
namespace {

constexpr unsigned long long kEmpty = ~0ull;
constexpr unsigned long long kAcq = 1ull << 63;  // "acquired" flag in the key word

struct ZSlot {
    unsigned long long key;
    double cc, euc, nrm2;
};

struct ZParams {
    // tables
    const double *rf, *e1d, *e2d, *phd;
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
    // data
    const double* fps;  // nvox x 2N raw
    double* q;          // nvox x 2N normalized scratch
    ZSlot* tab;         // nvox x cap
    unsigned int cap_mask;
    const long long* bounds;  // nvox x 6 or null (full bounds)
    const long long* inits;   // nvox x 2 or null
    int64_t nvox;
    mrfg_quant* out;
    int* err;
};

struct Z {
    const ZParams* p;
    ZSlot* tab;
    const double* q;
    int lane;
    long long evals;
    long long lo1, hi1, lo2, hi2, lodf, hidf;
};

__device__ __forceinline__ unsigned long long zkey(long long i1, long long i2, long long idf) {
    return (static_cast<unsigned long long>(i1) << 42) | (static_cast<unsigned long long>(i2) << 21) |
           static_cast<unsigned long long>(idf);
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

// One objective evaluation: the reference's Objective::acquire +
// score_from_entry for both metrics, FP64, two passes (norm, then the
// normalized entry against the query).
__device__ void zsim(const Z& z, int i1, int i2, int idf, ZSlot& s) {
    const ZParams& P = *z.p;
    const int n = P.n;
    double acc = sim64_lattice<0>(P.rf, P.e1d, P.e2d, P.phd, P.inv0, n, P.L, i1, i2, idf, 0.0, nullptr);
    const double inv = 1.0 / sqrt(acc);  // fingerprint.cpp:30-32
    double re = 0.0, im = 0.0, dd = 0.0;
    const bool euc = P.need_euc;
    const double* q = z.q;
    sim64_walk_pf(P.rf, P.e1d, P.e2d, P.phd, P.inv0, n, P.L, i1, i2, idf, [&](int j, double x, double y) {
        const double er = __dmul_rn(x, inv), ei = __dmul_rn(y, inv);
        const double qr = q[2 * j], qi = q[2 * j + 1];
        re = __dadd_rn(re, __dadd_rn(__dmul_rn(qr, er), __dmul_rn(qi, ei)));  // zoom.cpp:79
        im = __dadd_rn(im, __dsub_rn(__dmul_rn(qi, er), __dmul_rn(qr, ei)));  // zoom.cpp:80
        if (euc) {
            const double dr = __dsub_rn(qr, er), di = __dsub_rn(qi, ei);  // zoom.cpp:87-89
            dd = __dadd_rn(dd, __dadd_rn(__dmul_rn(dr, dr), __dmul_rn(di, di)));
        }
    }, [&](int jj) -> const void* { return q + 2 * jj; });
    const double v = sqrt(__dadd_rn(__dmul_rn(re, re), __dmul_rn(im, im)));
    s.cc = v < 1.0 ? v : 1.0;  // zoom.cpp:82-83
    s.euc = -sqrt(dd);          // zoom.cpp:91
    s.nrm2 = acc;
}

// Make sure the points pt(0..count-1) are in the memo (computed, not
// acquired).  Lanes split the missing points; duplicates are claimed once.
template <class PT>
__device__ void zensure(Z& z, long long count, PT pt) {
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
        if (mine) {
            ZSlot s;
            zsim(z, static_cast<int>(a), static_cast<int>(b), static_cast<int>(c), s);
            z.tab[slot].cc = s.cc;
            z.tab[slot].euc = s.euc;
            z.tab[slot].nrm2 = s.nrm2;
        }
        __syncwarp();
        __threadfence_block();
        __syncwarp();
    }
}

// Objective::eval (zoom.cpp:125-138): range check, memo read, acquisition count.
__device__ double zf(Z& z, long long i1, long long i2, long long idf, int metric) {
    const ZParams& P = *z.p;
    if (i1 < 0 || i2 < 0 || idf < 0 || i1 >= P.L.n1 || i2 >= P.L.n2 || idf >= P.L.ndf) {
        atomicExch(P.err, 1);
        return -1e300;
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
        if (s < 0) return -1e300;
    }
    const unsigned long long kk = *reinterpret_cast<volatile unsigned long long*>(&z.tab[s].key);
    if (!(kk & kAcq)) {
        __syncwarp();
        if (z.lane == 0) z.tab[s].key = kk | kAcq;
        __syncwarp();
        __threadfence_block();
        __syncwarp();
        ++z.evals;
    }
    const volatile ZSlot* vs = &z.tab[s];
    return metric == MRFG_METRIC_CC ? vs->cc : vs->euc;
}

struct Best {
    long long idx;
    double val;
};
__device__ __forceinline__ void offer(Best& b, long long i, double v) {
    if (v > b.val) {
        b.val = v;
        b.idx = i;
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
    zensure(z, cnt + (extra ? 1 : 0), [&](long long k, long long& p1, long long& p2, long long& pd) {
        p1 = i1;
        p2 = i2;
        pd = k < cnt ? a + k * step : b;
    });
    for (long long x = a; x <= b; x += step) offer(bst, x, zf(z, i1, i2, x, z.p->metric));
    if (extra) offer(bst, b, zf(z, i1, i2, b, z.p->metric));
}

__device__ bool plateau(const double* marks, int nm, double eps) {
    if (nm < 3) return false;
    double mn = marks[nm - 3], mx = mn;
    for (int j = nm - 3; j < nm; ++j) {
        mn = fmin(mn, marks[j]);
        mx = fmax(mx, marks[j]);
    }
    return mx - mn < eps;
}

// zoom.cpp:189-241
__device__ Best df_run(Z& z, long long i1, long long i2, long long coarse, long long wh) {
    const ZParams& P = *z.p;
    double marks[16];
    int nm = 0;
    Best cur{-1, -1e300};
    df_scan(z, i1, i2, z.lodf, z.hidf, coarse, cur);
    marks[nm++] = cur.val;
    {
        Best r = cur;
        df_scan(z, i1, i2, cur.idx - wh, cur.idx + wh, P.df_refine, r);
        cur = r;
    }
    marks[nm++] = cur.val;
    for (int round = 0; round < 8; ++round) {
        Best t = cur;
        const long long nf = cur.idx + P.omega <= z.hidf ? (z.hidf - cur.idx) / P.omega : 0;
        const long long nb = cur.idx - P.omega >= z.lodf ? (cur.idx - z.lodf) / P.omega : 0;
        const long long c0 = cur.idx;
        zensure(z, nf + nb, [&](long long k, long long& p1, long long& p2, long long& pd) {
            p1 = i1;
            p2 = i2;
            pd = k < nf ? c0 + (k + 1) * P.omega : c0 - (k - nf + 1) * P.omega;
        });
        for (long long k = 1; cur.idx + k * P.omega <= z.hidf; ++k) {
            const long long q = cur.idx + k * P.omega;
            offer(t, q, zf(z, i1, i2, q, P.metric));
        }
        for (long long k = 1; cur.idx - k * P.omega >= z.lodf; ++k) {
            const long long q = cur.idx - k * P.omega;
            offer(t, q, zf(z, i1, i2, q, P.metric));
        }
        if (t.idx == cur.idx) break;
        Best r = t;
        df_scan(z, i1, i2, t.idx - wh, t.idx + wh, P.df_refine, r);
        cur = r;
        marks[nm++] = cur.val;
        if (plateau(marks, nm, P.plateau_eps)) return cur;
    }
    if (plateau(marks, nm, P.plateau_eps)) return cur;
    Best fin = cur;
    df_scan(z, i1, i2, cur.idx - P.omega / 2, cur.idx + P.omega / 2, 1, fin);
    return fin;
}

// zoom.cpp:173-250
__device__ long long search_df(Z& z, long long i1, long long i2) {
    const ZParams& P = *z.p;
    Best mainb = df_run(z, i1, i2, P.df_coarse, P.df_window_half);
    if (mainb.val < P.heavy_cc) {
        Best fb = df_run(z, i1, i2, P.fb_coarse, P.fb_window_half);
        if (fb.val > mainb.val) return fb.idx;
    }
    return mainb.idx;
}

// ------------------------------------------------------------- zoom_1d
// zoom.cpp:252-282 along T1 (axis 0) or T2 (axis 1); speculative flanks
// +-1..4 steps are simulated together before each decision.
__device__ long long zoom_1d(Z& z, int axis, long long i1, long long i2, long long idf, long long lo,
                             long long hi, long long init, long long s, int metric) {
    auto F = [&](long long a) {
        return axis == 0 ? zf(z, a, i2, idf, metric) : zf(z, i1, a, idf, metric);
    };
    long long x = clampll(init, lo, hi);
    double fx = F(x);
    for (;;) {
        const long long x0 = x;
        zensure(z, 2 * z.p->spec1d, [&](long long k, long long& a, long long& b, long long& c) {
            const long long off = (k / 2 + 1) * s * ((k & 1) ? 1 : -1);
            const long long v = clampll(x0 + off, lo, hi);
            a = axis == 0 ? v : i1;
            b = axis == 0 ? i2 : v;
            c = idf;
        });
        const long long xl = clampll(x - s, lo, hi);
        if (xl != x) {
            const double fl = F(xl);
            if (fl > fx) {
                x = xl;
                fx = fl;
                continue;
            }
        }
        const long long xr = clampll(x + s, lo, hi);
        if (xr != x) {
            const double fr = F(xr);
            if (fr > fx) {
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
// zoom.cpp:284-399 for one step pair; the 3x3 neighbourhood is simulated
// together before each iteration's probes.
__device__ void zoom_2d_step(Z& z, long long idf, int metric, long long& x, long long& y, double& fc,
                             long long& bx, long long& by, double& bf, long long s1, long long s2) {
    const long long lo1 = z.lo1, hi1 = z.hi1, lo2 = z.lo2, hi2 = z.hi2;
    auto F = [&](long long a, long long b) { return zf(z, a, b, idf, metric); };
    auto note = [&](long long px, long long py, double v) {
        if (v > bf) {
            bf = v;
            bx = px;
            by = py;
        }
    };
    const long long cap = 4 * ((hi1 - lo1) / s1 + (hi2 - lo2) / s2) + 16;
    bool converged = false;
    for (long long iter = 0; iter < cap && !converged; ++iter) {
        const long long cx = x, cy = y;
        const long long r = z.p->spec2d, w = 2 * r + 1;  // (2r+1)^2 - 1 neighbours
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
        double fl = fc, fd = fc;
        if (xl != x) {
            fl = F(xl, y);
            note(xl, y, fl);
        }
        if (yd != y) {
            fd = F(x, yd);
            note(x, yd, fd);
        }
        const bool lw = xl != x && fl > fc;
        const bool dw = yd != y && fd > fc;
        if (lw && dw) {
            x = xl;
            y = yd;
            fc = F(x, y);
            note(x, y, fc);
            continue;
        }
        if (!lw && !dw) {
            double fr = fc, fu = fc;
            if (xr != x) {
                fr = F(xr, y);
                note(xr, y, fr);
            }
            if (yu != y) {
                fu = F(x, yu);
                note(x, yu, fu);
            }
            const bool rw = xr != x && fr > fc;
            const bool uw = yu != y && fu > fc;
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
            double fu = fc;
            if (yu != y) {
                fu = F(x, yu);
                note(x, yu, fu);
            }
            if (yu != y && fu > fc) {
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
        double fr = fc;
        if (xr != x) {
            fr = F(xr, y);
            note(xr, y, fr);
        }
        if (xr != x && fr > fc) {
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
    double fc = zf(z, x, y, idf, metric);
    long long bx = x, by = y;
    double bf = fc;
    for (int k = 0; k < ns; ++k) zoom_2d_step(z, idf, metric, x, y, fc, bx, by, bf, s1v[k], s2v[k]);
}

// ------------------------------------------------------------ the kernel
__global__ void __launch_bounds__(128) k_zoom(const ZParams P) {
    const int64_t v = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / 32;
    if (v >= P.nvox) return;
    Z z;
    z.p = &P;
    z.lane = threadIdx.x % 32;
    z.tab = P.tab + v * (static_cast<int64_t>(P.cap_mask) + 1);
    z.evals = 0;
    const int n = P.n;
    const double* fp = P.fps + v * 2 * n;
    double* q = P.q + v * 2 * n;
    z.q = q;
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
    const double inv = 1.0 / nq;
    for (int j = z.lane; j < 2 * n; j += 32) q[j] = __dmul_rn(fp[j], inv);
    __syncwarp();
    __threadfence_block();
    __syncwarp();

    if (P.bounds) {
        const long long* b = P.bounds + 6 * v;
        z.lo1 = b[0];
        z.hi1 = b[1];
        z.lo2 = b[2];
        z.hi2 = b[3];
        z.lodf = b[4];
        z.hidf = b[5];
    } else {
        z.lo1 = 0;
        z.hi1 = P.L.n1 - 1;
        z.lo2 = 0;
        z.hi2 = P.L.n2 - 1;
        z.lodf = 0;
        z.hidf = P.L.ndf - 1;
    }
    const long long s1 = P.inits ? P.inits[2 * v] : P.init1;
    const long long s2 = P.inits ? P.inits[2 * v + 1] : P.init2;
    long long i1 = clampll(s1, z.lo1, z.hi1);  // zoom.cpp:428-429
    long long i2 = clampll(s2, z.lo2, z.hi2);

    // Stage 1 (zoom.cpp:465-469)
    long long idf = search_df(z, i1, i2);
    // Stage 2 (zoom.cpp:472-479)
    zoom_2d(z, idf, P.metric, i1, i2, P.s2d1, P.s2d2, P.n2d);
    zf(z, i1, i2, idf, P.metric);
    // Stage 3 (zoom.cpp:482-489)
    {
        Best b{-1, -1e300};
        const long long a = clampll(idf - P.omega / 2, z.lodf, z.hidf);
        const long long e = clampll(idf + P.omega / 2, z.lodf, z.hidf);
        const long long c1 = i1, c2 = i2;
        zensure(z, e - a + 1, [&](long long k, long long& p1, long long& p2, long long& pd) {
            p1 = c1;
            p2 = c2;
            pd = a + k;
        });
        for (long long k = a; k <= e; ++k) offer(b, k, zf(z, i1, i2, k, P.metric));
        idf = b.idx;
    }
    // Stage 4 (zoom.cpp:492-501)
    for (int k = 0; k < P.n1d; ++k) {
        i1 = zoom_1d(z, 0, i1, i2, idf, z.lo1, z.hi1, i1, P.s1d1[k], P.metric);
        zf(z, i1, i2, idf, P.metric);
        i2 = zoom_1d(z, 1, i1, i2, idf, z.lo2, z.hi2, i2, P.s1d2[k], P.metric);
        zf(z, i1, i2, idf, P.metric);
    }
    // Stage 5 (zoom.cpp:505-512)
    zoom_2d(z, idf, P.final_metric, i1, i2, &P.f2d1, &P.f2d2, 1);
    zf(z, i1, i2, idf, P.final_metric);
    // result (zoom.cpp:514-519)
    const double score = zf(z, i1, i2, idf, P.metric);
    const int s = zfind(z, zkey(i1, i2, idf));
    if (z.lane == 0) {
        mrfg_quant r;
        r.i1 = i1;
        r.i2 = i2;
        r.idf = idf;
        r.t1_ms = 0;  // filled on the host (exact axis values)
        r.t2_ms = 0;
        r.df_hz = 0;
        // estimate_pd (fingerprint.cpp:147-152): |fp| / |ideal|, ideal unnormalized
        r.pd = nq / sqrt(z.tab[s].nrm2);
        r.score = score;
        r.evaluations = z.evals;
        P.out[v] = r;
    }
}

long long snap_index(double value, const mrfg_axis& ax) {  // zoom.cpp:407-409
    return std::lround((value - ax.min) / ax.step);
}
long long step_units(double step_value, double finest) {  // zoom.cpp:411-414
    long long u = std::lround(step_value / finest);
    return u > 0 ? u : 1;
}

}  // namespace

void run_quantify(Ctx& c, const mrfg_grid& lat, const mrfg_zoom_config& cfg, const double* d_fps,
                  int64_t nvox, const int64_t* h_bounds, const double* h_init, mrfg_quant* d_out) {
    for (const mrfg_axis* ax : {&lat.t1_ms, &lat.t2_ms, &lat.df_hz})
        MRFG_REQUIRE(ax->count > 0 && ax->count < (int64_t(1) << 21), MRFG_E_INVALID,
                     "objective: lattice axis empty or too fine");  // zoom.cpp:46-48
    MRFG_REQUIRE(cfg.smooth_k == 0, MRFG_E_INVALID,
                 "quantify: smooth_k is not supported by the GPU MRF-ZOOM kernel");
    MRFG_REQUIRE(cfg.n2d >= 0 && cfg.n2d <= 8 && cfg.n1d >= 0 && cfg.n1d <= 8, MRFG_E_INVALID,
                 "quantify: at most 8 zoom steps per stage");
    const GridTables& t = ensure_tables(c, lat, true);
    ZParams P{};
    P.rf = c.rf64_d.as<double>();
    P.e1d = t.e1d.as<double>();
    P.e2d = t.e2d.as<double>();
    P.phd = t.phd.as<double>();
    P.inv0[0] = c.inv64[2];
    P.inv0[1] = c.inv64[5];
    P.inv0[2] = c.inv64[8];
    P.n = static_cast<int>(c.n);
    P.L = {lat.t1_ms.count, lat.t2_ms.count, lat.df_hz.count};
    P.metric = cfg.metric;
    P.final_metric = cfg.final_metric;
    P.need_euc = cfg.metric == MRFG_METRIC_EUCLIDEAN || cfg.final_metric == MRFG_METRIC_EUCLIDEAN;
    // zoom.cpp:454-463
    const double dfs = lat.df_hz.step;
    P.df_coarse = step_units(cfg.df_coarse_hz, dfs);
    P.df_refine = step_units(cfg.df_refine_hz, dfs);
    P.df_window_half = step_units(cfg.df_window_hz / 2, dfs);
    P.omega = step_units(cfg.omega_hz, dfs);
    P.plateau_eps = cfg.plateau_eps;
    P.heavy_cc = cfg.metric == MRFG_METRIC_CC ? cfg.heavy_noise_cc : -1e300;
    P.fb_coarse = step_units(cfg.fallback_coarse_hz, dfs);
    P.fb_window_half = step_units(cfg.fallback_window_hz / 2, dfs);
    P.n2d = cfg.n2d;
    P.n1d = cfg.n1d;
    for (int k = 0; k < cfg.n2d; ++k) {
        P.s2d1[k] = step_units(cfg.t1t2_2d_steps_ms[k], lat.t1_ms.step);
        P.s2d2[k] = step_units(cfg.t1t2_2d_steps_ms[k], lat.t2_ms.step);
    }
    for (int k = 0; k < cfg.n1d; ++k) {
        P.s1d1[k] = step_units(cfg.t1t2_1d_steps_ms[k], lat.t1_ms.step);
        P.s1d2[k] = step_units(cfg.t1t2_1d_steps_ms[k], lat.t2_ms.step);
    }
    P.f2d1 = step_units(cfg.final_2d_step_ms, lat.t1_ms.step);
    P.f2d2 = step_units(cfg.final_2d_step_ms, lat.t2_ms.step);
    {
        const char* e1 = std::getenv("MRFG_ZOOM_SPEC1D");
        const char* e2 = std::getenv("MRFG_ZOOM_SPEC2D");
        P.spec1d = e1 ? std::max(1, std::atoi(e1)) : 16;
        P.spec2d = e2 ? std::max(1, std::atoi(e2)) : 2;
    }
    P.init1 = snap_index(cfg.init_t1_ms, lat.t1_ms);
    P.init2 = snap_index(cfg.init_t2_ms, lat.t2_ms);
    P.fps = d_fps;
    const unsigned int cap = 8192;
    P.cap_mask = cap - 1;
    P.nvox = nvox;
    // scratch: normalized queries, memo tables, bounds/inits, error flag
    const size_t qbytes = sizeof(double) * 2 * c.n * nvox;
    const size_t tbytes = sizeof(ZSlot) * cap * nvox;
    const size_t bbytes = h_bounds ? sizeof(long long) * 6 * nvox : 0;
    const size_t ibytes = h_init ? sizeof(long long) * 2 * nvox : 0;
    DevBuf scratch;
    scratch.ensure(qbytes + tbytes + bbytes + ibytes + 64);
    char* base = scratch.as<char>();
    P.q = reinterpret_cast<double*>(base);
    P.tab = reinterpret_cast<ZSlot*>(base + qbytes);
    P.bounds = h_bounds ? reinterpret_cast<long long*>(base + qbytes + tbytes) : nullptr;
    P.inits = h_init ? reinterpret_cast<long long*>(base + qbytes + tbytes + bbytes) : nullptr;
    P.err = reinterpret_cast<int*>(base + qbytes + tbytes + bbytes + ibytes);
    MRFG_CUDA(cudaMemsetAsync(P.err, 0, sizeof(int), c.stream));
    if (h_bounds)
        MRFG_CUDA(cudaMemcpyAsync(const_cast<long long*>(P.bounds), h_bounds, bbytes,
                                  cudaMemcpyHostToDevice, c.stream));
    std::vector<long long> inits;
    if (h_init) {
        inits.resize(2 * nvox);
        for (int64_t k = 0; k < nvox; ++k) {
            inits[2 * k] = snap_index(h_init[2 * k], lat.t1_ms);
            inits[2 * k + 1] = snap_index(h_init[2 * k + 1], lat.t2_ms);
        }
        MRFG_CUDA(cudaMemcpyAsync(const_cast<long long*>(P.inits), inits.data(), ibytes,
                                  cudaMemcpyHostToDevice, c.stream));
    }
    P.out = d_out;
    const int bs = 128;
    const int64_t threads = nvox * 32;
    k_zoom<<<(threads + bs - 1) / bs, bs, 0, c.stream>>>(P);
    MRFG_CUDA(cudaGetLastError());
    int err = 0;
    MRFG_CUDA(cudaMemcpyAsync(&err, P.err, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    MRFG_CUDA(cudaStreamSynchronize(c.stream));
    scratch.release();
    MRFG_REQUIRE(err != 1, MRFG_E_RANGE, "objective: lattice index out of range");
    MRFG_REQUIRE(err != 2, MRFG_E_RUNTIME, "quantify: per-voxel memo table full");
    MRFG_REQUIRE(err != 3, MRFG_E_INVALID, "normalize: zero fingerprint");
}

}  // namespace mrfg
