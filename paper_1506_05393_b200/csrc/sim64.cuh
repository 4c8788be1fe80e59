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

// One FP64 lattice atom, table driven.  mode 0: returns sum |s|^2 only;
// mode 1: writes float(m * inv) entries (dictionary.cpp:44-51).
template <int MODE>
__device__ double sim64_lattice(const double* __restrict__ rf, const double* __restrict__ e1d,
                                const double* __restrict__ e2d, const double* __restrict__ phd,
                                const double inv0[3], int n, const Lattice& L, int i1, int i2,
                                int idf, double inv, float* __restrict__ out) {
    double x = inv0[0], y = inv0[1], z = inv0[2];
    double acc = 0.0;
    for (int j = 0; j < n; ++j) {
        rf_apply64(rf + 9 * j, x, y, z);
        const double* E1 = e1d + (static_cast<int64_t>(j) * L.n1 + i1) * 2;
        const double* E2 = e2d + (static_cast<int64_t>(j) * L.n2 + i2) * 2;
        const double* P = phd + (static_cast<int64_t>(j) * L.ndf + idf) * 4;
        relax64(x, y, z, __ldg(E1), __ldg(E2), __ldg(P), __ldg(P + 1));
        if (MODE == 0) {
            acc = __dadd_rn(acc, __dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)));
        } else {
            out[2 * j] = __double2float_rn(__dmul_rn(x, inv));
            out[2 * j + 1] = __double2float_rn(__dmul_rn(y, inv));
        }
        relax64(x, y, z, __ldg(E1 + 1), __ldg(E2 + 1), __ldg(P + 2), __ldg(P + 3));
    }
    return acc;
}

}  // namespace
}  // namespace mrfg
