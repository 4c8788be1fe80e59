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
// Status: the pipeline (K1 off-resonance-major slabs, projection, K2 on one K
// block, audit, re-rank) runs end to end with identical answers, but this
// kernel holds the whole basis in shared memory, which caps the rank at 16 --
// at that rank the residual reaches 0.17 on config 2, the audit widens the
// margin to ~0.1 and the scan is no faster than the default.  Rank 48-64 needs
// the basis tiled through shared memory.
//
// k_project: out[row][0..63] = sum_k A[row][k] W[n][k] (fp16 in, fp32
// accumulate, fp16 out; columns >= NW stay zero), mma.sync m16n8k16 with a
// K permutation that lets every thread load 16 contiguous bytes per row.
#include <cuda_fp16.h>

#include <algorithm>
#include <cmath>
#include <complex>
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

// A: rows x kpad (fp16, K-major, rows a multiple of 128); W: NW x kpad; out: rows x 64.
// inv2 (1/|a|^2 per row, or null): when given, rho2max <- max over rows < valid of
// 1 - |P a|^2 / |a|^2 (as float bits; values are clamped at 0).
template <int NW>
__global__ void __launch_bounds__(256) k_project(const __half* __restrict__ A, int64_t kpad,
                                                 const __half* __restrict__ W, __half* __restrict__ out,
                                                 const float* __restrict__ inv2, int64_t valid,
                                                 unsigned int* __restrict__ rho2max) {
    extern __shared__ __align__(16) __half wsm[];  // NW x (kpad + kWPad)
    const int64_t wp = kpad + kWPad;
    for (int64_t i = threadIdx.x; i < NW * (kpad / 8); i += blockDim.x) {
        const int64_t n = i / (kpad / 8), k8 = i % (kpad / 8);
        *reinterpret_cast<uint4*>(wsm + n * wp + 8 * k8) = *reinterpret_cast<const uint4*>(W + n * kpad + 8 * k8);
    }
    __syncthreads();
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
    for (int64_t k0 = 0; k0 < kpad; k0 += 32) {
        uint4 nlo = lo, nhi = hi;
        if (k0 + 32 < kpad) {
            nlo = *reinterpret_cast<const uint4*>(a_lo + k0 + 32);
            nhi = *reinterpret_cast<const uint4*>(a_hi + k0 + 32);
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
    // rows g (acc[..][0,1]) and g + 8 (acc[..][2,3]); columns 8 j + 2 t, + 1
    float s_lo = 0.f, s_hi = 0.f;
#pragma unroll
    for (int j = 0; j < NW / 8; ++j) {
        s_lo = fmaf(acc[j][0], acc[j][0], fmaf(acc[j][1], acc[j][1], s_lo));
        s_hi = fmaf(acc[j][2], acc[j][2], fmaf(acc[j][3], acc[j][3], s_hi));
        *reinterpret_cast<__half2*>(out + (r0 + g) * 64 + 8 * j + 2 * t) = __floats2half2_rn(acc[j][0], acc[j][1]);
        *reinterpret_cast<__half2*>(out + (r0 + g + 8) * 64 + 8 * j + 2 * t) =
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

}  // namespace

int subspace_cols(int r) { return r <= 8 ? 16 : 32; }

void launch_project(Ctx& c, const __half* A, int64_t rows, int64_t kpad, const __half* W, int nw, __half* out,
                    const float* inv2, int64_t valid, unsigned int* rho2max) {
    MRFG_REQUIRE(rows % kProjRows == 0 && kpad % 32 == 0 && (nw == 16 || nw == 32), MRFG_E_INVALID,
                 "project: bad operand shape");
    const int smem = static_cast<int>(sizeof(__half) * nw * (kpad + kWPad));
    const unsigned grid = static_cast<unsigned>(rows / kProjRows);
    if (nw == 16) {
        MRFG_CUDA(cudaFuncSetAttribute(k_project<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        k_project<16><<<grid, 256, smem, c.stream>>>(A, kpad, W, out, inv2, valid, rho2max);
    } else {
        MRFG_CUDA(cudaFuncSetAttribute(k_project<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        k_project<32><<<grid, 256, smem, c.stream>>>(A, kpad, W, out, inv2, valid, rho2max);
    }
    MRFG_CUDA(cudaGetLastError());
}

// The bases of every off-resonance slab of the cached grid: W[df][nw][kpad]
// (fp16).  Per df, kSamples atoms spread over the (T1, T2) rows are produced
// by the FP32 operand producer (fp16 rows, as screened), copied to the host,
// and orthonormalized by pivoted Gram-Schmidt in double precision: the
// largest remaining residual becomes the next basis vector until r are found.
const __half* ensure_subspace(Ctx& c, const GridTables& tc, int r) {
    GridTables& t = const_cast<GridTables&>(tc);
    const int nw = subspace_cols(r);
    const int64_t n = c.n, kp = k_pad_of(n);
    const int64_t ndf = t.grid.df_hz.count, nrows = t.grid.t1_ms.count * t.grid.t2_ms.count;
    if (t.sub_r == r && t.subw.p) return t.subw.as<__half>();
    constexpr int kSamples = 64;
    const int64_t step = std::max<int64_t>(1, (nrows - 1) / (kSamples - 1));
    const int64_t ns = std::min<int64_t>(kSamples, (nrows + step - 1) / step);
    MRFG_REQUIRE(ns >= r, MRFG_E_INVALID, "subspace: fewer lattice rows than the rank");
    const int64_t srows = 256;  // operand producer granularity
    DevBuf samp, sinv;
    samp.ensure(sizeof(__half) * srows * kp * ndf);
    sinv.ensure(sizeof(float) * srows);
    for (int64_t d = 0; d < ndf; ++d)
        launch_bloch_operand(c, t, d, step * ndf, nrows * ndf, srows, MRFG_METRIC_CC,
                             samp.as<__half>() + d * srows * kp, sinv.as<float>());
    std::vector<__half> hs(static_cast<size_t>(srows) * kp * ndf);
    MRFG_CUDA(cudaMemcpyAsync(hs.data(), samp.p, sizeof(__half) * hs.size(), cudaMemcpyDeviceToHost, c.stream));
    MRFG_CUDA(cudaStreamSynchronize(c.stream));
    std::vector<__half> hw(static_cast<size_t>(ndf) * nw * kp, __float2half(0.f));
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t d = 0; d < ndf; ++d) {
        std::vector<std::complex<double>> v(static_cast<size_t>(ns) * n), b(static_cast<size_t>(r) * n);
        std::vector<double> res(ns);
        for (int64_t k = 0; k < ns; ++k) {
            const __half* row = hs.data() + (d * srows + k) * kp;
            double nn = 0;
            for (int64_t j = 0; j < n; ++j) {
                const std::complex<double> z(__half2float(row[2 * j]), __half2float(row[2 * j + 1]));
                v[k * n + j] = z;
                nn += std::norm(z);
            }
            const double inv = nn > 0 ? 1.0 / std::sqrt(nn) : 0.0;
            for (int64_t j = 0; j < n; ++j) v[k * n + j] *= inv;
            res[k] = nn > 0 ? 1.0 : 0.0;
        }
        for (int m = 0; m < r; ++m) {
            const int64_t piv = std::max_element(res.begin(), res.end()) - res.begin();
            if (res[piv] < 1e-20) break;  // the samples are exhausted: the remaining rows stay zero
            const double inv = 1.0 / std::sqrt(res[piv]);
            std::complex<double>* bm = &b[static_cast<size_t>(m) * n];
            for (int64_t j = 0; j < n; ++j) bm[j] = v[piv * n + j] * inv;
            for (int64_t k = 0; k < ns; ++k) {
                std::complex<double> dot = 0;
                for (int64_t j = 0; j < n; ++j) dot += std::conj(bm[j]) * v[k * n + j];
                double nn = 0;
                for (int64_t j = 0; j < n; ++j) {
                    v[k * n + j] -= dot * bm[j];
                    nn += std::norm(v[k * n + j]);
                }
                res[k] = nn;
            }
            res[piv] = 0;
            // real embedding: u = (re, im, ...), J u = (-im, re, ...)
            __half* u = hw.data() + (d * nw + 2 * m) * kp;
            __half* ju = u + kp;
            for (int64_t j = 0; j < n; ++j) {
                u[2 * j] = __float2half(static_cast<float>(bm[j].real()));
                u[2 * j + 1] = __float2half(static_cast<float>(bm[j].imag()));
                ju[2 * j] = __float2half(static_cast<float>(-bm[j].imag()));
                ju[2 * j + 1] = __float2half(static_cast<float>(bm[j].real()));
            }
        }
    }
    t.subw.ensure(sizeof(__half) * hw.size());
    MRFG_CUDA(cudaMemcpyAsync(t.subw.p, hw.data(), sizeof(__half) * hw.size(), cudaMemcpyHostToDevice, c.stream));
    MRFG_CUDA(cudaStreamSynchronize(c.stream));
    samp.release();
    sinv.release();
    t.sub_r = r;
    return t.subw.as<__half>();
}

}  // namespace mrfg
