// subspace.cu -- per-off-resonance subspace screening (EXPERIMENTAL, opt-in:
// MRFG_SUBSPACE=r; off by default and not yet profitable -- see below).
//
// Across off-resonance a lattice dictionary is full rank in time, but the
// fingerprints of ONE off-resonance value, over all (T1, T2), span a much
// smaller subspace (config 2, SVD of 2,500 sampled unit atoms per df: held-out
// residual 1e-3 .. 4e-3 at complex rank 32, 1e-4 .. 8e-4 at 48, <= 3e-4 at 64;
// DESIGN.md 7).  So scan_grid (dictionary.cpp:257-308) can screen df slab by
// df slab in 2r dimensions instead of 2N:
//
//   W_df    orthonormal basis of slab df (r complex vectors -> 2r real rows of
//           the real embedding [re, im, ...]: u_m and J u_m), from pivoted
//           Gram-Schmidt over sampled atoms of the slab (host, once per grid)
//   C  = A W_df^T   atom coefficients (k_project, tensor cores, HBM-bound)
//   QP = Q' W_df^T  query coefficients, both rows of every voxel (same kernel)
//   K2 on (QP, C): <P q, P a> = <q, a> - <q_perp, a_perp>, so
//           |screen - full screen| <= |q_perp| |a_perp| / |a| <= rho_a; the
//           largest rho_a the projection sees is reported in the scan
//           statistics.  The unbiased audit (which widens the margin and
//           rescans when the sampled error exceeds delta/2) and the exact FP64
//           re-rank are unchanged, so the answers are the default path's.
//
// Status: the pipeline (K1 off-resonance-major slabs, projection, K2 on one or
// two K blocks, audit, re-rank) runs end to end with identical answers at
// complex ranks 8 .. 64, but it is not profitable yet (config 2, one B200):
// the bases from pivoted Gram-Schmidt over 4r sampled atoms leave the worst
// atoms of a slab at a residual of 0.07 whatever the rank (the SVD of 2,500
// samples reaches 3e-4 at rank 64), so the audit widens the margin to ~0.05
// (1.2e8 candidates, K3 0.5 s); this mma.sync projection runs at 0.6 TB/s
// (0.7 s per scan) and K2 takes 0.93 s: 2.45 s against 2.77 s.  Missing: a
// better basis (SVD / more samples), a projection kernel at the HBM roofline
// (~0.06 s), an accurate per-atom residual for the analytic certificate.
//
// k_project: out[row][0..63] = sum_k A[row][k] W[n][k] (fp16 in, fp32
// accumulate, fp16 out; columns >= NW stay zero), mma.sync m16n8k16 with a
// K permutation that lets every thread load 16 contiguous bytes per row.
#include <cuda_fp16.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "mrfg_internal.cuh"

namespace mrfg {
namespace {

constexpr int kProjRows = 128;  // rows per block: 8 warps x 16
constexpr int kWPad = 8;        // halves of padding per staged basis row (bank spread)

__device__ __forceinline__ void mma16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// A: rows x kpad (fp16, K-major, rows a multiple of 128); W: NW x kpad; out: rows x opitch.
// The basis goes through shared memory KT columns at a time (KT = kpad when
// the whole basis fits).  inv2 (1/|a|^2 per row, or null): when given,
// rho2max <- max over rows < valid of 1 - |P a|^2 / |a|^2 (float bits, >= 0;
// the fp16 rounding of W and A puts a floor of ~1e-4 under it).
template <int NW>
__global__ void __launch_bounds__(256) k_project(const __half* __restrict__ A, int64_t kpad, int kt,
                                                 const __half* __restrict__ W, __half* __restrict__ out,
                                                 int opitch, const float* __restrict__ inv2, int64_t valid,
                                                 unsigned int* __restrict__ rho2max, int64_t w_stride,
                                                 int64_t o_stride) {
    // blockIdx.y: batch of bases over the same rows (the query projections of all df)
    W += blockIdx.y * w_stride;
    out += blockIdx.y * o_stride;
    extern __shared__ __align__(16) __half wsm[];  // NW x (kt + kWPad)
    const int wp = kt + kWPad;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int64_t r0 = blockIdx.x * static_cast<int64_t>(kProjRows) + warp * 16;
    const __half* a_lo = A + (r0 + g) * kpad + 8 * t;
    const __half* a_hi = A + (r0 + g + 8) * kpad + 8 * t;
    float acc[NW / 8][4];
#pragma unroll
    for (int j = 0; j < NW / 8; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[j][e] = 0.f;
    // 32 K elements per step (thread t holds k0 + 8t .. 8t+7 of rows g, g+8);
    // two steps are in flight
    uint4 lo = *reinterpret_cast<const uint4*>(a_lo), hi = *reinterpret_cast<const uint4*>(a_hi);
    for (int64_t kt0 = 0; kt0 < kpad; kt0 += kt) {
        __syncthreads();
        for (int i = threadIdx.x; i < NW * (kt / 8); i += blockDim.x) {
            const int n = i / (kt / 8), k8 = i % (kt / 8);
            *reinterpret_cast<uint4*>(wsm + n * wp + 8 * k8) =
                *reinterpret_cast<const uint4*>(W + static_cast<int64_t>(n) * kpad + kt0 + 8 * k8);
        }
        __syncthreads();
        for (int k0 = 0; k0 < kt; k0 += 32) {
            uint4 nlo = lo, nhi = hi;
            if (kt0 + k0 + 32 < kpad) {
                nlo = *reinterpret_cast<const uint4*>(a_lo + kt0 + k0 + 32);
                nhi = *reinterpret_cast<const uint4*>(a_hi + kt0 + k0 + 32);
            }
#pragma unroll
            for (int j = 0; j < NW / 8; ++j) {
                const uint4 b = *reinterpret_cast<const uint4*>(wsm + (8 * j + g) * wp + k0 + 8 * t);
                mma16816(acc[j], lo.x, hi.x, lo.y, hi.y, b.x, b.y);
                mma16816(acc[j], lo.z, hi.z, lo.w, hi.w, b.z, b.w);
            }
            lo = nlo;
            hi = nhi;
        }
    }
    // rows g (acc[..][0,1]) and g + 8 (acc[..][2,3]); columns 8 j + 2 t, + 1
    float s_lo = 0.f, s_hi = 0.f;
#pragma unroll
    for (int j = 0; j < NW / 8; ++j) {
        s_lo = fmaf(acc[j][0], acc[j][0], fmaf(acc[j][1], acc[j][1], s_lo));
        s_hi = fmaf(acc[j][2], acc[j][2], fmaf(acc[j][3], acc[j][3], s_hi));
        *reinterpret_cast<__half2*>(out + (r0 + g) * opitch + 8 * j + 2 * t) = __floats2half2_rn(acc[j][0], acc[j][1]);
        *reinterpret_cast<__half2*>(out + (r0 + g + 8) * opitch + 8 * j + 2 * t) =
            __floats2half2_rn(acc[j][2], acc[j][3]);
    }
    if (inv2) {
        s_lo += __shfl_xor_sync(0xffffffffu, s_lo, 1);
        s_lo += __shfl_xor_sync(0xffffffffu, s_lo, 2);
        s_hi += __shfl_xor_sync(0xffffffffu, s_hi, 1);
        s_hi += __shfl_xor_sync(0xffffffffu, s_hi, 2);
        if (t == 0) {
            float worst = 0.f;
            if (r0 + g < valid) worst = fmaxf(worst, 1.f - s_lo * inv2[r0 + g]);
            if (r0 + g + 8 < valid) worst = fmaxf(worst, 1.f - s_hi * inv2[r0 + g + 8]);
            if (worst > 0.f) atomicMax(rho2max, __float_as_uint(worst));
        }
    }
}

template <int NW>
void project_variant(Ctx& c, const __half* A, int64_t rows, int64_t kpad, const __half* W, __half* out, int opitch,
                     const float* inv2, int64_t valid, unsigned int* rho2max, int batch, int64_t w_stride,
                     int64_t o_stride) {
    // the largest K tile (a divisor of kpad, multiple of 32) whose basis tile fits ~128 KB
    int kt = static_cast<int>(kpad);
    while (static_cast<int64_t>(sizeof(__half)) * NW * (kt + kWPad) > 132 * 1024 && kt % 64 == 0) kt /= 2;
    const int smem = static_cast<int>(sizeof(__half) * NW * (kt + kWPad));
    MRFG_CUDA(cudaFuncSetAttribute(k_project<NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    k_project<NW><<<dim3(static_cast<unsigned>(rows / kProjRows), batch), 256, smem, c.stream>>>(
        A, kpad, kt, W, out, opitch, inv2, valid, rho2max, w_stride, o_stride);
    MRFG_CUDA(cudaGetLastError());
}

}  // namespace

// complex rank -> real basis rows (2r) and the operand width K2 sees (a multiple of 64)
int subspace_rank(int r) { return r <= 8 ? 8 : (r <= 16 ? 16 : (r <= 32 ? 32 : (r <= 48 ? 48 : 64))); }
int subspace_cols(int r) { return 2 * subspace_rank(r); }
int subspace_pitch(int r) { return (subspace_cols(r) + 63) / 64 * 64; }

void launch_project(Ctx& c, const __half* A, int64_t rows, int64_t kpad, const __half* W, int nw, __half* out,
                    int opitch, const float* inv2, int64_t valid, unsigned int* rho2max, int batch,
                    int64_t w_stride, int64_t o_stride) {
    MRFG_REQUIRE(rows % kProjRows == 0 && kpad % 64 == 0, MRFG_E_INVALID, "project: bad operand shape");
    switch (nw) {
        case 16: project_variant<16>(c, A, rows, kpad, W, out, opitch, inv2, valid, rho2max, batch, w_stride, o_stride); break;
        case 32: project_variant<32>(c, A, rows, kpad, W, out, opitch, inv2, valid, rho2max, batch, w_stride, o_stride); break;
        case 64: project_variant<64>(c, A, rows, kpad, W, out, opitch, inv2, valid, rho2max, batch, w_stride, o_stride); break;
        case 96: project_variant<96>(c, A, rows, kpad, W, out, opitch, inv2, valid, rho2max, batch, w_stride, o_stride); break;
        case 128: project_variant<128>(c, A, rows, kpad, W, out, opitch, inv2, valid, rho2max, batch, w_stride, o_stride); break;
        default: throw Error{MRFG_E_INVALID, "project: unsupported basis width"};
    }
}

// The bases of every off-resonance slab of the cached grid: W[df][nw][kpad]
// (fp16).  About 5 r sample rows (T1, T2) are produced at ALL their
// off-resonance values by the FP32 operand producer (fp16 rows, as screened),
// copied to the host, and per df orthonormalized by pivoted Gram-Schmidt in
// double precision: the largest remaining residual becomes the next basis
// vector until r are found.
const __half* ensure_subspace(Ctx& c, const GridTables& tc, int r) {
    GridTables& t = const_cast<GridTables&>(tc);
    const int nw = subspace_cols(r);
    const int64_t n = c.n, kp = k_pad_of(n);
    const int64_t ndf = t.grid.df_hz.count, n1 = t.grid.t1_ms.count, n2 = t.grid.t2_ms.count;
    if (t.sub_r == r && t.subw.p) return t.subw.as<__half>();
    // sample atoms of a slab: an s1 x s2 grid over (T1, T2) whose axis VALUES are
    // geometrically spaced, both ends included -- the fingerprints change
    // fastest at short T2 / T1 (an evenly spaced 16-point T2 grid left atoms
    // between its first two points at a residual of 0.07 whatever the rank)
    auto geo = [](const mrfg_axis& ax, int64_t cnt) {
        const int64_t nn = ax.count;
        std::vector<int64_t> idx;
        const double lo = axis_value(ax, 0), hi = axis_value(ax, nn - 1);
        for (int64_t k = 0; k < cnt; ++k) {
            const double v = cnt > 1 && lo > 0 && hi > lo ? lo * std::pow(hi / lo, static_cast<double>(k) / (cnt - 1))
                                                           : lo + (hi - lo) * (cnt > 1 ? double(k) / (cnt - 1) : 0.0);
            int64_t a = 0, b = nn - 1;  // nearest index on the (monotonic) axis
            while (b - a > 1) {
                const int64_t m = (a + b) / 2;
                (axis_value(ax, m) <= v ? a : b) = m;
            }
            const int64_t i = std::fabs(axis_value(ax, b) - v) < std::fabs(axis_value(ax, a) - v) ? b : a;
            if (idx.empty() || idx.back() != i) idx.push_back(i);
        }
        return idx;
    };
    const int64_t want2 = r > 48 ? 28 : 24;
    const std::vector<int64_t> I2 = geo(t.grid.t2_ms, std::min<int64_t>(n2, want2));
    const std::vector<int64_t> I1 = geo(t.grid.t1_ms, std::min<int64_t>(n1, std::max<int64_t>(6, (5 * r + want2 - 1) / want2)));
    const int64_t ns = static_cast<int64_t>(I1.size() * I2.size());
    MRFG_REQUIRE(ns >= r, MRFG_E_INVALID, "subspace: fewer lattice rows than the rank");
    // held-out rows: the index midpoints between neighbouring samples (where an
    // interpolating basis is worst); their residual is the truncation error the
    // scan adds to its screening margin
    auto mids = [](const std::vector<int64_t>& v) {
        std::vector<int64_t> m;
        for (size_t k = 0; k + 1 < v.size(); ++k)
            if (v[k + 1] - v[k] > 1) m.push_back((v[k] + v[k + 1]) / 2);
        if (m.empty()) m.push_back(v[0]);
        return m;
    };
    const std::vector<int64_t> H1 = mids(I1), H2 = mids(I2);
    const int64_t nh = static_cast<int64_t>(H1.size() * H2.size());
    // one launch per sample row: all its off-resonance values (flat stride 1)
    DevBuf samp, sinv;
    samp.ensure(sizeof(__half) * (ns + nh) * ndf * kp);
    sinv.ensure(sizeof(float) * ndf);
    {
        int64_t k = 0;
        for (int64_t i1 : I1)
            for (int64_t i2 : I2) {
                const int64_t row = i1 * n2 + i2;
                launch_bloch_operand(c, t, row * ndf, 1, (row + 1) * ndf, ndf, MRFG_METRIC_CC,
                                     samp.as<__half>() + k * ndf * kp, sinv.as<float>());
                ++k;
            }
        for (int64_t i1 : H1)
            for (int64_t i2 : H2) {
                const int64_t row = i1 * n2 + i2;
                launch_bloch_operand(c, t, row * ndf, 1, (row + 1) * ndf, ndf, MRFG_METRIC_CC,
                                     samp.as<__half>() + k * ndf * kp, sinv.as<float>());
                ++k;
            }
    }
    std::vector<__half> hs(static_cast<size_t>(ns + nh) * ndf * kp);
    MRFG_CUDA(cudaMemcpyAsync(hs.data(), samp.p, sizeof(__half) * hs.size(), cudaMemcpyDeviceToHost, c.stream));
    MRFG_CUDA(cudaStreamSynchronize(c.stream));
    std::vector<__half> hw(static_cast<size_t>(ndf) * nw * kp, __float2half(0.f));
    double rho2_held = 0;
#pragma omp parallel for schedule(dynamic, 2) reduction(max : rho2_held)
    for (int64_t d = 0; d < ndf; ++d) {
        std::vector<double> Br(static_cast<size_t>(r) * n, 0.0), Bi(static_cast<size_t>(r) * n, 0.0);  // the basis
        // sample residuals (re, im planes) and the current basis vector
        std::vector<double> vr(static_cast<size_t>(ns) * n), vi(static_cast<size_t>(ns) * n), br(n), bi(n), res(ns);
        for (int64_t k = 0; k < ns; ++k) {
            const __half* row = hs.data() + (k * ndf + d) * kp;  // sample k at off-resonance d
            double nn = 0;
            for (int64_t j = 0; j < n; ++j) {
                const double x = __half2float(row[2 * j]), y = __half2float(row[2 * j + 1]);
                vr[k * n + j] = x;
                vi[k * n + j] = y;
                nn += x * x + y * y;
            }
            const double inv = nn > 0 ? 1.0 / std::sqrt(nn) : 0.0;
            for (int64_t j = 0; j < n; ++j) {
                vr[k * n + j] *= inv;
                vi[k * n + j] *= inv;
            }
            res[k] = nn > 0 ? 1.0 : 0.0;
        }
        for (int m = 0; m < r; ++m) {
            const int64_t piv = std::max_element(res.begin(), res.end()) - res.begin();
            if (res[piv] < 1e-20) break;  // the samples are exhausted: the remaining rows stay zero
            const double inv = 1.0 / std::sqrt(res[piv]);
            for (int64_t j = 0; j < n; ++j) {
                br[j] = vr[piv * n + j] * inv;
                bi[j] = vi[piv * n + j] * inv;
            }
            for (int64_t k = 0; k < ns; ++k) {
                double* xr = &vr[k * n];
                double* xi = &vi[k * n];
                double dr = 0, di = 0;  // <b, v_k> = sum conj(b) v
                for (int64_t j = 0; j < n; ++j) {
                    dr += br[j] * xr[j] + bi[j] * xi[j];
                    di += br[j] * xi[j] - bi[j] * xr[j];
                }
                double nn = 0;
                for (int64_t j = 0; j < n; ++j) {
                    xr[j] -= dr * br[j] - di * bi[j];
                    xi[j] -= dr * bi[j] + di * br[j];
                    nn += xr[j] * xr[j] + xi[j] * xi[j];
                }
                res[k] = nn;
            }
            res[piv] = 0;
            std::copy(br.begin(), br.end(), Br.begin() + static_cast<size_t>(m) * n);
            std::copy(bi.begin(), bi.end(), Bi.begin() + static_cast<size_t>(m) * n);
            // real embedding: u = (re, im, ...), J u = (-im, re, ...)
            __half* u = hw.data() + (d * nw + 2 * m) * kp;
            __half* ju = u + kp;
            for (int64_t j = 0; j < n; ++j) {
                u[2 * j] = __float2half(static_cast<float>(br[j]));
                u[2 * j + 1] = __float2half(static_cast<float>(bi[j]));
                ju[2 * j] = __float2half(static_cast<float>(-bi[j]));
                ju[2 * j + 1] = __float2half(static_cast<float>(br[j]));
            }
        }
        // residual of the held-out rows: 1 - |B^H a|^2 / |a|^2
        for (int64_t k = 0; k < nh; ++k) {
            const __half* row = hs.data() + ((ns + k) * ndf + d) * kp;
            double nn = 0;
            for (int64_t j = 0; j < 2 * n; ++j) nn += double(__half2float(row[j])) * double(__half2float(row[j]));
            if (!(nn > 0)) continue;
            double pp = 0;
            for (int m = 0; m < r; ++m) {
                const double* xr = &Br[static_cast<size_t>(m) * n];
                const double* xi = &Bi[static_cast<size_t>(m) * n];
                double dr = 0, di = 0;
                for (int64_t j = 0; j < n; ++j) {
                    const double ar = __half2float(row[2 * j]), ai = __half2float(row[2 * j + 1]);
                    dr += xr[j] * ar + xi[j] * ai;
                    di += xr[j] * ai - xi[j] * ar;
                }
                pp += dr * dr + di * di;
            }
            rho2_held = std::max(rho2_held, 1.0 - pp / nn);
        }
    }
    t.sub_rho_held = std::sqrt(std::max(0.0, rho2_held));
    t.subw.ensure(sizeof(__half) * hw.size());
    MRFG_CUDA(cudaMemcpyAsync(t.subw.p, hw.data(), sizeof(__half) * hw.size(), cudaMemcpyHostToDevice, c.stream));
    MRFG_CUDA(cudaStreamSynchronize(c.stream));
    samp.release();
    sinv.release();
    t.sub_r = r;
    return t.subw.as<__half>();
}

}  // namespace mrfg
