// sim64.cuh -- FP64 lattice Bloch recursion shared by K1/K3/K5.
//
// Reference operand order (bloch.hpp:34-38, bloch.cpp:22-26, 108-123) with
// explicit IEEE round-to-nearest operations (no FMA contraction); the
// per-step transcendentals come from host-libm tables (GridTables), so a
// lattice fingerprint is bit-identical to the reference's.
#pragma once
#include <cstdint>

namespace mrfg {
namespace {
struct Rot64 {
    double r[9];
};

__device__ __forceinline__ void rf_apply64(const double* __restrict__ r, double& x, double& y,
                                           double& z) {
    // bloch.hpp:34-38: {m0 x + m1 y + m2 z, ...}, summed left to right.
    double nx = __dadd_rn(__dadd_rn(__dmul_rn(r[0], x), __dmul_rn(r[1], y)), __dmul_rn(r[2], z));
    double ny = __dadd_rn(__dadd_rn(__dmul_rn(r[3], x), __dmul_rn(r[4], y)), __dmul_rn(r[5], z));
    double nz = __dadd_rn(__dadd_rn(__dmul_rn(r[6], x), __dmul_rn(r[7], y)), __dmul_rn(r[8], z));
    x = nx;
    y = ny;
    z = nz;
}

// bloch.cpp:22-26 with precomputed e1, e2, cos, sin.
__device__ __forceinline__ void relax64(double& x, double& y, double& z, double e1, double e2,
                                        double c, double s) {
    double nx = __dmul_rn(__dsub_rn(__dmul_rn(x, c), __dmul_rn(y, s)), e2);
    double ny = __dmul_rn(__dadd_rn(__dmul_rn(x, s), __dmul_rn(y, c)), e2);
    x = nx;
    y = ny;
    z = __dadd_rn(1.0, __dmul_rn(__dsub_rn(z, 1.0), e1));
}

struct Lattice {
    int64_t n1, n2, ndf;
};

__device__ __forceinline__ void unflatten(int64_t flat, const Lattice& L, int& i1, int& i2,
                                          int& idf) {
    // dictionary.hpp:45-49
    idf = static_cast<int>(flat % L.ndf);
    int64_t rest = flat / L.ndf;
    i2 = static_cast<int>(rest % L.n2);
    i1 = static_cast<int>(rest / L.n2);
}

// Per-step transcendental values of one lattice atom (E1, E2, phasor for
// the te and rest intervals), gathered from the host-libm tables.
struct StepT {
    double e1t, e1r, e2t, e2r, ct, st, cr, sr;
};
__device__ __forceinline__ StepT load_step(const double* __restrict__ e1d,
                                           const double* __restrict__ e2d,
                                           const double* __restrict__ phd, const Lattice& L, int n,
                                           int j, int i1, int i2, int idf) {
    // parameter-major tables: entry (i, j) at i*n + j
    const double2 a = __ldg(reinterpret_cast<const double2*>(e1d + (static_cast<int64_t>(i1) * n + j) * 2));
    const double2 b = __ldg(reinterpret_cast<const double2*>(e2d + (static_cast<int64_t>(i2) * n + j) * 2));
    const double2* P = reinterpret_cast<const double2*>(phd + (static_cast<int64_t>(idf) * n + j) * 4);
    const double2 p0 = __ldg(P), p1 = __ldg(P + 1);
    return {a.x, a.y, b.x, b.y, p0.x, p0.y, p1.x, p1.y};
}

__device__ __forceinline__ void prefetch_l1(const void* p) {
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}
constexpr int kPrefetchSteps = 8;

// Walk one lattice atom through the schedule (bloch.cpp:108-123) calling
// at(j, mx, my) at every echo.  The table gathers run two steps ahead of
// the recursion in registers and eight steps ahead as L1 prefetches (one per
// 128-byte line, every fourth step), so their
// L2 latency hides behind the FP64 dependency chain (measured: the per-step
// gather latency, not the FP64 pipe, bounded K3/K5).  `extra(j)` returns one
// more per-step address to prefetch (the query row), or nullptr.
template <class AT, class PF>
__device__ __forceinline__ void sim64_walk_pf(const double* __restrict__ rf,
                                              const double* __restrict__ e1d,
                                              const double* __restrict__ e2d,
                                              const double* __restrict__ phd, const double inv0[3],
                                              int n, const Lattice& L, int i1, int i2, int idf, AT at,
                                              PF extra) {
    double x = inv0[0], y = inv0[1], z = inv0[2];
    const double* p1 = e1d + static_cast<int64_t>(i1) * n * 2;
    const double* p2 = e2d + static_cast<int64_t>(i2) * n * 2;
    const double* pd = phd + static_cast<int64_t>(idf) * n * 4;
    for (int j = 0; j < kPrefetchSteps && j < n; ++j) {
        prefetch_l1(p1 + j * 2);
        prefetch_l1(p2 + j * 2);
        prefetch_l1(pd + j * 4);
        if (const void* e = extra(j)) prefetch_l1(e);
    }
    StepT c0 = load_step(e1d, e2d, phd, L, n, 0, i1, i2, idf);
    StepT c1 = load_step(e1d, e2d, phd, L, n, n > 1 ? 1 : 0, i1, i2, idf);
    for (int j = 0; j < n; ++j) {
        // one prefetch per 128-byte line: every 4 steps (the 32-byte phasor
        // rows; the 16-byte rows are touched twice per line)
        if ((j & 3) == 0 && j + kPrefetchSteps < n) {
            const int jp = j + kPrefetchSteps;
            prefetch_l1(p1 + jp * 2);
            prefetch_l1(p2 + jp * 2);
            prefetch_l1(pd + jp * 4);
            if (const void* e = extra(jp)) prefetch_l1(e);
        }
        const StepT c2 = load_step(e1d, e2d, phd, L, n, j + 2 < n ? j + 2 : n - 1, i1, i2, idf);
        rf_apply64(rf + 9 * j, x, y, z);
        relax64(x, y, z, c0.e1t, c0.e2t, c0.ct, c0.st);
        at(j, x, y);
        relax64(x, y, z, c0.e1r, c0.e2r, c0.cr, c0.sr);
        c0 = c1;
        c1 = c2;
    }
}

template <class AT>
__device__ __forceinline__ void sim64_walk(const double* __restrict__ rf,
                                           const double* __restrict__ e1d,
                                           const double* __restrict__ e2d,
                                           const double* __restrict__ phd, const double inv0[3],
                                           int n, const Lattice& L, int i1, int i2, int idf, AT at) {
    sim64_walk_pf(rf, e1d, e2d, phd, inv0, n, L, i1, i2, idf, at,
                  [](int) -> const void* { return nullptr; });
}

// One FP64 lattice atom.  mode 0: returns sum |s|^2 (fingerprint.cpp:14-18
// order); mode 1: writes float(m * inv) entries (dictionary.cpp:44-51).
template <int MODE>
__device__ double sim64_lattice(const double* __restrict__ rf, const double* __restrict__ e1d,
                                const double* __restrict__ e2d, const double* __restrict__ phd,
                                const double inv0[3], int n, const Lattice& L, int i1, int i2,
                                int idf, double inv, float* __restrict__ out) {
    double acc = 0.0;
    sim64_walk(rf, e1d, e2d, phd, inv0, n, L, i1, i2, idf, [&](int j, double x, double y) {
        if (MODE == 0) {
            acc = __dadd_rn(acc, __dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)));
        } else {
            out[2 * j] = __double2float_rn(__dmul_rn(x, inv));
            out[2 * j + 1] = __double2float_rn(__dmul_rn(y, inv));
        }
    });
    return acc;
}

}  // namespace
}  // namespace mrfg
