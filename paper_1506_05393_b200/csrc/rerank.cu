// rerank.cu -- K3: exact re-rank of screened candidates, per-voxel argmax,
// cross-GPU merge (C1), cc_map and query preparation.
//
// Exactness: the reference scores a unit FP64 query against FP32-quantized
// unit FP64 fingerprints (dictionary.cpp:37-53, 117-143, 145-150).  The
// re-rank recomputes each surviving candidate through that very pipeline in
// FP64 (sim64.cuh, host-libm tables), so its scores are bit-identical to the
// reference's and the argmax -- including the lowest-flat tie rule of
// dictionary.cpp:291-294 -- is the reference's.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>

#include "mrfg_internal.cuh"
#include "sim64.cuh"

namespace mrfg {
namespace {

// prep_query (dictionary.cpp:145-150) -> normalize (fingerprint.cpp:28-37),
// then the fp16 screening rows (see match_sm100.cu).  A query flagged
// unit_norm (unit[v] != 0) is used as given (`fp.unit_norm ? fp :
// normalize(fp)`); its screening rows are still scaled to unit length.
__global__ void k_prepare_queries(const double* __restrict__ raw, int n, int64_t nq,
                                  int64_t k_pad, double* __restrict__ q64,
                                  __half* __restrict__ qprime, int* __restrict__ bad,
                                  const uint8_t* __restrict__ unit) {
    int64_t v = blockIdx.x;
    if (v >= nq) return;
    __shared__ double s_inv;
    const double* src = raw + v * 2 * n;
    const bool as_is = unit != nullptr && unit[v] != 0;
    if (threadIdx.x == 0) {
        double acc = 0;  // sequential, the reference's summation order
        for (int j = 0; j < n; ++j)
            acc = __dadd_rn(acc, __dadd_rn(__dmul_rn(src[2 * j], src[2 * j]),
                                           __dmul_rn(src[2 * j + 1], src[2 * j + 1])));
        double nn = sqrt(acc);
        if (nn == 0) atomicExch(bad, 1);
        s_inv = nn == 0 ? 0.0 : 1.0 / nn;
    }
    __syncthreads();
    const double inv = s_inv;
    __half* re_row = qprime + (2 * v) * k_pad;
    __half* im_row = qprime + (2 * v + 1) * k_pad;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
        const double ur = __dmul_rn(src[2 * j], inv), ui = __dmul_rn(src[2 * j + 1], inv);
        q64[v * 2 * n + 2 * j] = as_is ? src[2 * j] : ur;
        q64[v * 2 * n + 2 * j + 1] = as_is ? src[2 * j + 1] : ui;
        re_row[2 * j] = __double2half(ur);
        re_row[2 * j + 1] = __double2half(ui);
        im_row[2 * j] = __double2half(ui);
        im_row[2 * j + 1] = __double2half(-ur);
    }
}

__device__ __forceinline__ float threshold_final(float best, float delta, int metric) {
    float t = best - delta;
    if (metric == MRFG_METRIC_CC) return t > 0.f ? t * t : 0.f;
    return t;
}

__global__ void k_filter(const CandRec* __restrict__ cand, int64_t n, const float* __restrict__ best,
                         float delta, int metric, int64_t* __restrict__ list,
                         unsigned long long* __restrict__ count) {
    int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    CandRec r = cand[i];
    if (r.s >= threshold_final(best[r.voxel], delta, metric)) {
        unsigned long long k = atomicAdd(count, 1ull);
        list[k] = i;
    }
}

// Sort key of a selected candidate: voxel above flat, so a warp's lanes
// re-rank one voxel's neighbouring atoms -- the query row is a broadcast load
// and the parameter-major table rows are shared or adjacent (the gathers,
// not the FP64 pipe, bound the walk).
constexpr int kFlatBits = 40;
constexpr float kRescreenEps = 1e-5f;  // certification margin of the FP32 re-screen
__global__ void k_rerank_keys(const CandRec* __restrict__ cand, const int64_t* __restrict__ list,
                              int64_t n, unsigned long long* __restrict__ keys) {
    int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (k >= n) return;
    const CandRec r = cand[list[k]];
    keys[k] = (static_cast<unsigned long long>(r.voxel) << kFlatBits) |
              static_cast<unsigned long long>(r.flat);
}

__device__ __forceinline__ unsigned long long order_key(double x) {
    long long b = __double_as_longlong(x);
    return b >= 0 ? static_cast<unsigned long long>(b) ^ 0x8000000000000000ull
                  : ~static_cast<unsigned long long>(b);
}
__device__ __forceinline__ double key_value(unsigned long long k) {
    long long b = (k & 0x8000000000000000ull) ? static_cast<long long>(k ^ 0x8000000000000000ull)
                                              : static_cast<long long>(~k);
    return __longlong_as_double(b);
}

struct Tab64 {
    const double *rf, *e1d, *e2d, *phd;
    double inv0[3];
    int n;
    Lattice L;
};

// Exact reference score of lattice atom `flat` against unit FP64 query q.
__device__ double exact_score(const Tab64& T, const double* __restrict__ q, int64_t flat,
                              int metric) {
    int i1, i2, idf;
    unflatten(flat, T.L, i1, i2, idf);
    double acc = sim64_lattice<0>(T.rf, T.e1d, T.e2d, T.phd, T.inv0, T.n, T.L, i1, i2, idf, 0.0,
                                  nullptr);
    const double inv = 1.0 / sqrt(acc);
    // second pass: float entries streamed straight into the score
    double re = 0.0, im = 0.0, dd = 0.0;
    sim64_walk_pf(T.rf, T.e1d, T.e2d, T.phd, T.inv0, T.n, T.L, i1, i2, idf, [&](int j, double x, double y) {
        const double er = static_cast<double>(__double2float_rn(__dmul_rn(x, inv)));
        const double ei = static_cast<double>(__double2float_rn(__dmul_rn(y, inv)));
        const double qr = q[2 * j], qi = q[2 * j + 1];
        if (metric == MRFG_METRIC_CC) {
            // dictionary.cpp:121-124
            re = __dadd_rn(re, __dadd_rn(__dmul_rn(qr, er), __dmul_rn(qi, ei)));
            im = __dadd_rn(im, __dsub_rn(__dmul_rn(qi, er), __dmul_rn(qr, ei)));
        } else {
            // dictionary.cpp:133-136
            const double dr = __dsub_rn(qr, er), di = __dsub_rn(qi, ei);
            dd = __dadd_rn(dd, __dadd_rn(__dmul_rn(dr, dr), __dmul_rn(di, di)));
        }
    }, [&](int jj) -> const void* { return q + 2 * jj; });
    if (metric == MRFG_METRIC_CC) {
        double v = sqrt(__dadd_rn(__dmul_rn(re, re), __dmul_rn(im, im)));
        return v < 1.0 ? v : 1.0;  // dictionary.cpp:126
    }
    return -sqrt(dd);
}

__global__ void k_rerank(Tab64 T, const double* __restrict__ q64, const CandRec* __restrict__ cand,
                         const int64_t* __restrict__ list, int64_t n, int metric,
                         double* __restrict__ score, unsigned long long* __restrict__ vkey,
                         unsigned int* __restrict__ err_max) {
    int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (k >= n) return;
    const CandRec r = cand[list[k]];
    const double sc = exact_score(T, q64 + static_cast<int64_t>(r.voxel) * 2 * T.n, r.flat, metric);
    score[k] = sc;
    atomicMax(vkey + r.voxel, order_key(sc));
    if (metric == MRFG_METRIC_CC && err_max) {
        const float e = fabsf(sqrtf(r.s) - static_cast<float>(sc));
        atomicMax(err_max, __float_as_uint(e));
    }
}

// Single-walk variant of k_rerank: the FP64 echoes of the one walk are kept
// in a lane-interleaved scratch (a warp's 32 lanes store step j as 512
// contiguous bytes, streaming cache hints), then the scoring pass reads them
// back instead of re-walking: the walk -- L1-wavefront bound on its table
// gathers -- runs once per candidate instead of twice.  Same operations in the
// same order as exact_score, so the score is the same bits.  Persistent
// threads (grid-stride over the sorted list) bound the scratch.
__global__ void __launch_bounds__(64) k_rerank1(Tab64 T, const double* __restrict__ q64,
                                                const CandRec* __restrict__ cand,
                                                const int64_t* __restrict__ list, int64_t n, int metric,
                                                double2* __restrict__ scratch, double* __restrict__ score,
                                                unsigned long long* __restrict__ vkey,
                                                unsigned int* __restrict__ err_max) {
    const int64_t tid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    const int64_t nthreads = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int lane = threadIdx.x & 31;
    double2* my = scratch + (tid >> 5) * static_cast<int64_t>(T.n) * 32 + lane;
    // whole warps iterate together (lanes past the end idle in the last round)
    const int64_t rounds = (n + nthreads - 1) / nthreads;
    for (int64_t rd = 0; rd < rounds; ++rd) {
        const int64_t k = tid + rd * nthreads;
        if (k >= n) break;
        const CandRec r = cand[list[k]];
        const double* q = q64 + static_cast<int64_t>(r.voxel) * 2 * T.n;
        int i1, i2, idf;
        unflatten(r.flat, T.L, i1, i2, idf);
        double acc = 0.0;
        sim64_walk(T.rf, T.e1d, T.e2d, T.phd, T.inv0, T.n, T.L, i1, i2, idf, [&](int j, double x, double y) {
            acc = __dadd_rn(acc, __dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)));
            __stcs(my + static_cast<int64_t>(j) * 32, make_double2(x, y));
        });
        const double inv = 1.0 / sqrt(acc);
        double re = 0.0, im = 0.0, dd = 0.0;
        // scoring pass: the echoes stream back 8 steps per batch of loads
        // (memory-level parallelism: the scratch is DRAM-resident at large N)
        constexpr int U = 8;
        for (int j0 = 0; j0 < T.n; j0 += U) {
            double2 m[U];
#pragma unroll
            for (int u = 0; u < U; ++u)
                m[u] = j0 + u < T.n ? __ldcs(my + static_cast<int64_t>(j0 + u) * 32) : make_double2(0.0, 0.0);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int j = j0 + u;
                if (j >= T.n) break;
                const double er = static_cast<double>(__double2float_rn(__dmul_rn(m[u].x, inv)));
                const double ei = static_cast<double>(__double2float_rn(__dmul_rn(m[u].y, inv)));
                const double qr = q[2 * j], qi = q[2 * j + 1];
                if (metric == MRFG_METRIC_CC) {
                    re = __dadd_rn(re, __dadd_rn(__dmul_rn(qr, er), __dmul_rn(qi, ei)));
                    im = __dadd_rn(im, __dsub_rn(__dmul_rn(qi, er), __dmul_rn(qr, ei)));
                } else {
                    const double dr = __dsub_rn(qr, er), di = __dsub_rn(qi, ei);
                    dd = __dadd_rn(dd, __dadd_rn(__dmul_rn(dr, dr), __dmul_rn(di, di)));
                }
            }
        }
        double sc;
        if (metric == MRFG_METRIC_CC) {
            const double v = sqrt(__dadd_rn(__dmul_rn(re, re), __dmul_rn(im, im)));
            sc = v < 1.0 ? v : 1.0;
        } else {
            sc = -sqrt(dd);
        }
        score[k] = sc;
        atomicMax(vkey + r.voxel, order_key(sc));
        if (metric == MRFG_METRIC_CC && err_max)
            atomicMax(err_max, __float_as_uint(fabsf(sqrtf(r.s) - static_cast<float>(sc))));
    }
}

// Certified FP32 re-screen (lattice scans, CC metric).  Every selected
// candidate is walked once in FP32 over the float copies of the host-libm
// tables (one thread per candidate, (voxel, flat) order), partial sums folded
// into FP64 every 16 steps -- the K5 screening arithmetic, audited there at
// <= 2.5e-7 from the exact score.  With eps = 1e-5 the exact argmax a* keeps
// s32(a*) >= e(a*) - eps >= e(a) - eps >= s32(a) - 2 eps for every a, so only
// candidates within 2 eps of their voxel's FP32 maximum go on to the FP64
// re-rank (config 5: 7.1 M -> ~1e4).  The fp16 screening error is measured
// against these scores.
struct Tab32 {
    const StepU* su;
    const float4* e1f;
    const float2* e2f;
    const float4* phf;
    float inv0[3];
    int n;
    Lattice L;
};

// One candidate's FP32 re-screen score (the K5 screening arithmetic).
__device__ float rescreen32_score(const Tab32& T, const double* __restrict__ q64, int64_t flat) {
    int i1, i2, idf;
    unflatten(flat, T.L, i1, i2, idf);
    const int n = T.n;
    const float4* e1p = T.e1f + static_cast<int64_t>(i1) * n;
    const float2* e2p = T.e2f + static_cast<int64_t>(i2) * n;
    const float4* php = T.phf + static_cast<int64_t>(idf) * n;
    const double2* q = reinterpret_cast<const double2*>(q64);
    float x = T.inv0[0], y = T.inv0[1], z = T.inv0[2];
    double re = 0.0, im = 0.0, nn = 0.0;
    float pr = 0.f, pi = 0.f, pn = 0.f;
    for (int j = 0; j < n; ++j) {
        const StepU& u = T.su[j];
        const float4 ra = __ldg(reinterpret_cast<const float4*>(u.r));
        const float4 rb = __ldg(reinterpret_cast<const float4*>(u.r) + 1);
        const float r8 = __ldg(u.r + 8);
        const float4 e1 = __ldg(e1p + j), ph = __ldg(php + j);
        const float2 e2 = __ldg(e2p + j);
        const double2 qd = __ldg(q + j);
        const float qr = static_cast<float>(qd.x), qi = static_cast<float>(qd.y);
        const float nx = fmaf(ra.x, x, fmaf(ra.y, y, ra.z * z));
        const float ny = fmaf(ra.w, x, fmaf(rb.x, y, rb.y * z));
        const float nz = fmaf(rb.z, x, fmaf(rb.w, y, r8 * z));
        x = (nx * ph.x - ny * ph.y) * e2.x;
        y = (nx * ph.y + ny * ph.x) * e2.x;
        z = fmaf(nz, e1.x, e1.y);
        pr = fmaf(qr, x, fmaf(qi, y, pr));
        pi = fmaf(qi, x, fmaf(-qr, y, pi));
        pn = fmaf(x, x, fmaf(y, y, pn));
        const float rx = (x * ph.z - y * ph.w) * e2.y;
        y = (x * ph.w + y * ph.z) * e2.y;
        x = rx;
        z = fmaf(z, e1.z, e1.w);
        if ((j & 15) == 15) {
            re += pr;
            im += pi;
            nn += pn;
            pr = pi = pn = 0.f;
        }
    }
    re += pr;
    im += pi;
    nn += pn;
    return static_cast<float>(fmin(sqrt(re * re + im * im) / sqrt(nn), 1.0));
}

__global__ void __launch_bounds__(128) k_rescreen32(Tab32 T, const double* __restrict__ q64,
                                                    const CandRec* __restrict__ cand,
                                                    const int64_t* __restrict__ list, int64_t cnt,
                                                    float* __restrict__ s32, unsigned* __restrict__ vmax,
                                                    unsigned* __restrict__ err_max) {
    const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (k >= cnt) return;
    const CandRec r = cand[list[k]];
    const float sc = rescreen32_score(T, q64 + static_cast<int64_t>(r.voxel) * 2 * T.n, r.flat);
    s32[k] = sc;
    atomicMax(vmax + r.voxel, __float_as_uint(sc));  // scores >= 0: int order = float order
    atomicMax(err_max, __float_as_uint(fabsf(sqrtf(r.s) - sc)));
}

// max |s32 - exact| over the FP64 survivors of the FP32 stage (k: compacted index)
__global__ void k_err32(const float* __restrict__ s32c, const double* __restrict__ score, int64_t n,
                        unsigned* __restrict__ err) {
    const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (k >= n) return;
    atomicMax(err, __float_as_uint(static_cast<float>(fabs(static_cast<double>(s32c[k]) - score[k]))));
}

__global__ void k_flag32(const CandRec* __restrict__ cand, const int64_t* __restrict__ list, int64_t cnt,
                         const float* __restrict__ s32, const unsigned* __restrict__ vmax, float margin,
                         unsigned char* __restrict__ flags) {
    const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (k >= cnt) return;
    const CandRec r = cand[list[k]];
    flags[k] = s32[k] >= __uint_as_float(vmax[r.voxel]) - margin ? 1 : 0;
}

// brute_force_search over a stored dictionary: the reference scores the
// FP64 unit query against the stored float32 entry (dictionary.cpp:117-143).
__device__ double exact_score_entry(const double* __restrict__ q, const float* __restrict__ e, int n,
                                    int metric) {
    double re = 0.0, im = 0.0, dd = 0.0;
    auto acc = [&](int j, float erf, float eif) {
        const double er = static_cast<double>(erf), ei = static_cast<double>(eif);
        const double qr = q[2 * j], qi = q[2 * j + 1];
        if (metric == MRFG_METRIC_CC) {
            re = __dadd_rn(re, __dadd_rn(__dmul_rn(qr, er), __dmul_rn(qi, ei)));
            im = __dadd_rn(im, __dsub_rn(__dmul_rn(qi, er), __dmul_rn(qr, ei)));
        } else {
            const double dr = __dsub_rn(qr, er), di = __dsub_rn(qi, ei);
            dd = __dadd_rn(dd, __dadd_rn(__dmul_rn(dr, dr), __dmul_rn(di, di)));
        }
    };
    int j = 0;
    // whole 32-byte sectors per lane (4 steps = two float4 loads) when the
    // entry row is 16-byte aligned (n even); the lanes of a warp read
    // different rows, so 8-byte loads used a quarter of every sector
    if ((reinterpret_cast<uintptr_t>(e) & 15) == 0) {
        const float4* e4 = reinterpret_cast<const float4*>(e);
        for (; j + 4 <= n; j += 4) {
            const float4 a = __ldg(e4 + j / 2), b = __ldg(e4 + j / 2 + 1);
            acc(j, a.x, a.y);
            acc(j + 1, a.z, a.w);
            acc(j + 2, b.x, b.y);
            acc(j + 3, b.z, b.w);
        }
    }
    for (; j < n; ++j) acc(j, e[2 * j], e[2 * j + 1]);
    if (metric == MRFG_METRIC_CC) {
        const double v = sqrt(__dadd_rn(__dmul_rn(re, re), __dmul_rn(im, im)));
        return v < 1.0 ? v : 1.0;
    }
    return -sqrt(dd);
}

__global__ void k_rerank_dict(const float* __restrict__ dict, int n, const double* __restrict__ q64,
                              const CandRec* __restrict__ cand, const int64_t* __restrict__ list,
                              int64_t cnt, int metric, double* __restrict__ score,
                              unsigned long long* __restrict__ vkey, unsigned int* __restrict__ err_max) {
    int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (k >= cnt) return;
    const CandRec r = cand[list[k]];
    const double sc = exact_score_entry(q64 + static_cast<int64_t>(r.voxel) * 2 * n, dict + r.flat * 2 * n,
                                        n, metric);
    score[k] = sc;
    atomicMax(vkey + r.voxel, order_key(sc));
    if (metric == MRFG_METRIC_CC) atomicMax(err_max, __float_as_uint(fabsf(sqrtf(r.s) - static_cast<float>(sc))));
}

// Stored float32 entries -> fp16 screening operand rows (+ 1/|e|^2 or 1/|e|):
// one warp per atom, coalesced row reads.
__global__ void k_dict_operand(const float* __restrict__ dict, int64_t first, int64_t count,
                               int64_t stride, int n, int64_t k_pad, int inv_mode,
                               __half* __restrict__ a, float* __restrict__ inv2, int64_t rows) {
    const int64_t r = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / 32;
    const int lane = threadIdx.x % 32;
    if (r >= rows) return;
    __half* dst = a + r * k_pad;
    float acc = 0.f;
    if (r < count) {
        const float* src = dict + (first + r * stride) * 2 * n;
        for (int64_t c = lane; c < k_pad; c += 32) {
            const float v = c < 2 * n ? src[c] : 0.f;
            acc = fmaf(v, v, acc);
            dst[c] = __float2half_rn(v);
        }
    } else {
        for (int64_t c = lane; c < k_pad; c += 32) dst[c] = __float2half_rn(0.f);
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) inv2[r] = (r < count && acc > 0.f) ? (inv_mode == 0 ? 1.f / acc : rsqrtf(acc)) : 0.f;
}

__global__ void k_select_flat(const CandRec* __restrict__ cand, const int64_t* __restrict__ list,
                              int64_t n, const double* __restrict__ score,
                              const unsigned long long* __restrict__ vkey,
                              unsigned long long* __restrict__ vflat) {
    int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (k >= n) return;
    const CandRec r = cand[list[k]];
    if (order_key(score[k]) == vkey[r.voxel])
        atomicMin(vflat + r.voxel, static_cast<unsigned long long>(r.flat));
}

__global__ void k_write_matches(const unsigned long long* __restrict__ vkey,
                                const unsigned long long* __restrict__ vflat, int64_t nq,
                                mrfg_match* __restrict__ out, int* __restrict__ missing) {
    int64_t v = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (v >= nq) return;
    if (vkey[v] == 0ull) {
        atomicExch(missing, 1);
        out[v].flat = -1;
        out[v].score = -1e300;
        return;
    }
    out[v].flat = static_cast<int64_t>(vflat[v]);
    out[v].score = key_value(vkey[v]);
}

__global__ void k_merge(const mrfg_match* __restrict__ in, int nranks, int64_t nq,
                        mrfg_match* __restrict__ out) {
    int64_t v = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (v >= nq) return;
    mrfg_match b = in[v];
    for (int r = 1; r < nranks; ++r) {
        mrfg_match m = in[static_cast<int64_t>(r) * nq + v];
        if (m.flat < 0) continue;
        if (b.flat < 0 || m.score > b.score || (m.score == b.score && m.flat < b.flat)) b = m;
    }
    out[v] = b;
}

__global__ void k_cc_map(Tab64 T, const double* __restrict__ q, int64_t first, int64_t count,
                         float* __restrict__ out) {
    int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (k >= count) return;
    out[k] = static_cast<float>(exact_score(T, q, first + k, MRFG_METRIC_CC));  // dictionary.cpp:325-327
}

Tab32 tab32_of(Ctx& c, const GridTables& t) {
    Tab32 T32;
    T32.su = t.stepu.as<StepU>();
    T32.e1f = t.e1f.as<float4>();
    T32.e2f = t.e2f.as<float2>();
    T32.phf = t.phf.as<float4>();
    T32.inv0[0] = static_cast<float>(c.inv64[2]);
    T32.inv0[1] = static_cast<float>(c.inv64[5]);
    T32.inv0[2] = static_cast<float>(c.inv64[8]);
    T32.n = static_cast<int>(c.n);
    T32.L = {t.grid.t1_ms.count, t.grid.t2_ms.count, t.grid.df_hz.count};
    return T32;
}

// Unbiased screening audit (metric cc): for every sampled (voxel, atom) pair,
// whatever its screening score, the exact reference score, the fp16 screening
// error |sqrt(s) - exact| and (lattice scans) the FP32 re-screen error
// |s32 - exact|.  Errors are rounded up to float.
__global__ void __launch_bounds__(64) k_audit(Tab64 T, Tab32 T32, const float* __restrict__ dict,
                                              const double* __restrict__ q64, const CandRec* __restrict__ rec,
                                              int64_t n, unsigned* __restrict__ err16,
                                              unsigned* __restrict__ err32) {
    const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (k >= n) return;
    const CandRec r = rec[k];
    const double* q = q64 + static_cast<int64_t>(r.voxel) * 2 * T.n;
    const double ex = dict ? exact_score_entry(q, dict + r.flat * 2 * T.n, T.n, MRFG_METRIC_CC)
                           : exact_score(T, q, r.flat, MRFG_METRIC_CC);
    atomicMax(err16, __float_as_uint(__double2float_ru(fabs(sqrt(static_cast<double>(r.s)) - ex))));
    if (!dict) {
        const float s32 = rescreen32_score(T32, q, r.flat);
        atomicMax(err32, __float_as_uint(__double2float_ru(fabs(static_cast<double>(s32) - ex))));
    }
}

Tab64 tab64_of(Ctx& c, const GridTables& t) {
    Tab64 T;
    T.rf = c.rf64_d.as<double>();
    T.e1d = t.e1d.as<double>();
    T.e2d = t.e2d.as<double>();
    T.phd = t.phd.as<double>();
    T.inv0[0] = c.inv64[2];
    T.inv0[1] = c.inv64[5];
    T.inv0[2] = c.inv64[8];
    T.n = static_cast<int>(c.n);
    T.L = {t.grid.t1_ms.count, t.grid.t2_ms.count, t.grid.df_hz.count};
    return T;
}

}  // namespace

void launch_prepare_queries(Ctx& c, const double* d_raw, int64_t nq, int64_t qrows, double* d_q64,
                            __half* d_qprime, int* d_bad, const uint8_t* d_unit) {
    const int64_t kp = k_pad_of(c.n);
    MRFG_CUDA(cudaMemsetAsync(d_qprime, 0, sizeof(__half) * qrows * kp, c.stream));
    k_prepare_queries<<<nq, 128, 0, c.stream>>>(d_raw, static_cast<int>(c.n), nq, kp, d_q64, d_qprime,
                                                d_bad, d_unit);
    MRFG_CUDA(cudaGetLastError());
}

// Returns the number of re-ranked candidates; throws when a voxel ends
// without any (cannot happen unless the candidate buffer overflowed), unless
// allow_missing (a score floor from another scan was applied).
int64_t rerank_and_select(Ctx& c, const GridTables* t, const float* d_dict, const double* d_q64,
                          int64_t nq, int metric, const float* d_best, float delta, CandRec* d_cand,
                          int64_t ncand, mrfg_match* d_out, double* err_max, bool allow_missing,
                          int64_t* stats_n32, bool allow_fp32, double* err32_max) {
    // scratch layout: list, list2 (ncand i64) | keys, keys2 (ncand u64) |
    //                 score (ncand f64) | vkey, vflat (nq u64) | counters | sort temp
    const int vbits = std::max(1, 64 - __builtin_clzll(static_cast<unsigned long long>(std::max<int64_t>(nq, 2) - 1)));
    const int end_bit = kFlatBits + vbits;
    size_t sort_tmp = 0;
    MRFG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, sort_tmp, static_cast<unsigned long long*>(nullptr),
                                              static_cast<unsigned long long*>(nullptr),
                                              static_cast<int64_t*>(nullptr), static_cast<int64_t*>(nullptr),
                                              std::max<int64_t>(ncand, 1), 0, end_bit, c.stream));
    // Sized for the next power of two of the candidate count: the count
    // varies by a few 1e4 between identical scans (the running maxima race
    // the GEMM epilogue), and a regrow (cudaFree + cudaMalloc of ~0.5 GB in
    // the timed scan) was measured to cost up to 200 ms.
    int64_t cap = int64_t(1) << 20;
    while (cap < ncand) cap *= 2;
    size_t sort_cap_tmp = 0;
    MRFG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, sort_cap_tmp, static_cast<unsigned long long*>(nullptr),
                                              static_cast<unsigned long long*>(nullptr),
                                              static_cast<int64_t*>(nullptr), static_cast<int64_t*>(nullptr),
                                              cap, 0, end_bit, c.stream));
    sort_tmp = std::max(sort_tmp, sort_cap_tmp);
    size_t sel_tmp = 0;  // order-preserving compaction for the FP32 stage
    MRFG_CUDA(cub::DeviceSelect::Flagged(nullptr, sel_tmp, static_cast<int64_t*>(nullptr),
                                         static_cast<unsigned char*>(nullptr), static_cast<int64_t*>(nullptr),
                                         static_cast<unsigned long long*>(nullptr), cap, c.stream));
    sort_tmp = std::max(sort_tmp, sel_tmp);
    const size_t head = 53 * static_cast<size_t>(cap) + 20 * nq + 64;
    size_t need = head + sort_tmp + 256;
    c.rerank.ensure(need);
    char* base = c.rerank.as<char>();
    int64_t* list = reinterpret_cast<int64_t*>(base);
    int64_t* list2 = list + cap;
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(list2 + cap);
    unsigned long long* keys2 = keys + cap;
    double* score = reinterpret_cast<double*>(keys2 + cap);
    unsigned long long* vkey = reinterpret_cast<unsigned long long*>(score + cap);
    unsigned long long* vflat = vkey + nq;
    unsigned long long* cnt = vflat + nq;
    int* missing = reinterpret_cast<int*>(cnt + 1);
    unsigned int* d_err = reinterpret_cast<unsigned int*>(missing + 1);
    unsigned long long* cnt32 = reinterpret_cast<unsigned long long*>(cnt + 2);
    float* s32 = reinterpret_cast<float*>(base + 40 * static_cast<size_t>(cap) + 16 * nq + 64);
    unsigned* vmax = reinterpret_cast<unsigned*>(s32 + cap);
    unsigned char* flags = reinterpret_cast<unsigned char*>(vmax + nq);
    float* s32c = reinterpret_cast<float*>(flags + cap);  // 4-byte aligned: cap, nq multiples of 4 apart
    unsigned* d_err32 = reinterpret_cast<unsigned*>(cnt32 + 2);
    void* d_sort_tmp = base + (head + 255) / 256 * 256;
    MRFG_CUDA(cudaMemsetAsync(vkey, 0, sizeof(unsigned long long) * nq, c.stream));
    MRFG_CUDA(cudaMemsetAsync(vflat, 0xFF, sizeof(unsigned long long) * nq, c.stream));
    MRFG_CUDA(cudaMemsetAsync(cnt, 0, 40, c.stream));
    const int bs = 256;
    if (ncand > 0)
        k_filter<<<(ncand + bs - 1) / bs, bs, 0, c.stream>>>(d_cand, ncand, d_best, delta, metric,
                                                             list, cnt);
    MRFG_CUDA(cudaGetLastError());
    unsigned long long nsel = 0;
    MRFG_CUDA(cudaMemcpyAsync(&nsel, cnt, sizeof nsel, cudaMemcpyDeviceToHost, c.stream));
    MRFG_CUDA(cudaStreamSynchronize(c.stream));
    const int rb = 64;
    const char* sort_env = std::getenv("MRFG_RERANK_SORT");  // "0": keep screening order
    if (nsel > 0 && !(sort_env && sort_env[0] == '0')) {
        // (voxel, flat) order for the gathers; the argmax does not depend on it
        k_rerank_keys<<<(nsel + bs - 1) / bs, bs, 0, c.stream>>>(d_cand, list, nsel, keys);
        MRFG_CUDA(cudaGetLastError());
        size_t tmp = sort_tmp;
        MRFG_CUDA(cub::DeviceRadixSort::SortPairs(d_sort_tmp, tmp, keys, keys2, list, list2,
                                                  static_cast<int64_t>(nsel), 0, end_bit, c.stream));
        list = list2;
    }
    // certified FP32 re-screen (lattice scans, CC): only near-ties go to FP64
    const char* r32_env = std::getenv("MRFG_RERANK_FP32");  // "0": every candidate in FP64
    int64_t n32 = 0;
    if (nsel > 0 && t != nullptr && metric == MRFG_METRIC_CC && allow_fp32 && !(r32_env && r32_env[0] == '0')) {
        n32 = static_cast<int64_t>(nsel);
        const Tab32 T32 = tab32_of(c, *t);
        MRFG_CUDA(cudaMemsetAsync(vmax, 0, sizeof(unsigned) * nq, c.stream));
        k_rescreen32<<<(nsel + 127) / 128, 128, 0, c.stream>>>(T32, d_q64, d_cand, list, nsel, s32, vmax, d_err);
        MRFG_CUDA(cudaGetLastError());
        k_flag32<<<(nsel + bs - 1) / bs, bs, 0, c.stream>>>(d_cand, list, nsel, s32, vmax, 2.0f * kRescreenEps,
                                                            flags);
        MRFG_CUDA(cudaGetLastError());
        int64_t* out_list = list == list2 ? reinterpret_cast<int64_t*>(keys) : list2;
        size_t tmp = sort_tmp;
        MRFG_CUDA(cub::DeviceSelect::Flagged(d_sort_tmp, tmp, list, flags, out_list, cnt32,
                                             static_cast<int64_t>(nsel), c.stream));
        // the survivors' FP32 scores, aligned with the compacted list (their
        // error against the exact scores is checked after the FP64 re-rank)
        tmp = sort_tmp;
        MRFG_CUDA(cub::DeviceSelect::Flagged(d_sort_tmp, tmp, s32, flags, s32c, cnt32 + 1,
                                             static_cast<int64_t>(nsel), c.stream));
        MRFG_CUDA(cudaMemcpyAsync(&nsel, cnt32, sizeof nsel, cudaMemcpyDeviceToHost, c.stream));
        MRFG_CUDA(cudaStreamSynchronize(c.stream));
        list = out_list;
    }
    if (stats_n32) *stats_n32 = n32;
    if (nsel > 0) {
        if (d_dict) {
            k_rerank_dict<<<(nsel + rb - 1) / rb, rb, 0, c.stream>>>(
                d_dict, static_cast<int>(c.n), d_q64, d_cand, list, nsel, metric, score, vkey, d_err);
        } else {
            // one walk per candidate (k_rerank1) while its echo scratch stays
            // small (measured: config 2, N = 1000, 1.5 GB: 91 -> 64 ms); at
            // config 5's N = 3000 (4.5 GB, DRAM-resident) the re-walk is as fast
            // (681 vs 703 ms), so k_rerank walks twice.  MRFG_RERANK_WALK=1/2 forces.
            int per_sm = 0;
            MRFG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_rerank1, rb, 0));
            const int64_t blocks = std::min<int64_t>((nsel + rb - 1) / rb,
                                                     int64_t(std::max(per_sm, 1)) * c.num_sms);
            const size_t scratch = sizeof(double2) * c.n * blocks * rb;
            const char* e = std::getenv("MRFG_RERANK_WALK");
            const bool one = e ? e[0] == '1' : scratch <= (size_t(2) << 30);
            if (!one) {
                k_rerank<<<(nsel + rb - 1) / rb, rb, 0, c.stream>>>(tab64_of(c, *t), d_q64, d_cand, list,
                                                                    nsel, metric, score, vkey,
                                                                    n32 ? nullptr : d_err);
                MRFG_CUDA(cudaGetLastError());
            } else {
            c.rerank_scratch.ensure(scratch);
            k_rerank1<<<static_cast<unsigned>(blocks), rb, 0, c.stream>>>(
                tab64_of(c, *t), d_q64, d_cand, list, nsel, metric, c.rerank_scratch.as<double2>(), score, vkey,
                n32 ? nullptr : d_err);
            }
        }
        MRFG_CUDA(cudaGetLastError());
        k_select_flat<<<(nsel + bs - 1) / bs, bs, 0, c.stream>>>(d_cand, list, nsel, score, vkey,
                                                                 vflat);
        MRFG_CUDA(cudaGetLastError());
        if (n32) {
            k_err32<<<(nsel + bs - 1) / bs, bs, 0, c.stream>>>(s32c, score, nsel, d_err32);
            MRFG_CUDA(cudaGetLastError());
        }
    }
    k_write_matches<<<(nq + bs - 1) / bs, bs, 0, c.stream>>>(vkey, vflat, nq, d_out, missing);
    MRFG_CUDA(cudaGetLastError());
    int h_missing[2] = {0, 0};
    unsigned h_err32 = 0;
    MRFG_CUDA(cudaMemcpyAsync(h_missing, missing, 2 * sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    MRFG_CUDA(cudaMemcpyAsync(&h_err32, d_err32, sizeof h_err32, cudaMemcpyDeviceToHost, c.stream));
    MRFG_CUDA(cudaStreamSynchronize(c.stream));
    if (err32_max) {
        float e;
        std::memcpy(&e, &h_err32, sizeof e);
        *err32_max = e;
    }
    if (err_max) {
        float e;
        std::memcpy(&e, &h_missing[1], sizeof e);
        *err_max = e;
    }
    // without a floor every query keeps its best atom (unless the candidate
    // buffer overflowed); with one, flat -1 marks "nothing above the floor"
    MRFG_REQUIRE(!h_missing[0] || allow_missing, MRFG_E_RUNTIME, "scan: a query ended without candidates");
    return static_cast<int64_t>(nsel);
}

void audit_screen(Ctx& c, const GridTables* t, const float* d_dict, const double* d_q64, const CandRec* d_rec,
                  int64_t n, double* err16, double* err32) {
    *err16 = 0;
    *err32 = 0;
    if (n <= 0) return;
    c.misc2.ensure(64);
    unsigned* d_e = c.misc2.as<unsigned>();
    MRFG_CUDA(cudaMemsetAsync(d_e, 0, 8, c.stream));
    Tab64 T{};
    Tab32 T32{};
    if (t) {
        T = tab64_of(c, *t);
        T32 = tab32_of(c, *t);
    } else {
        T.n = static_cast<int>(c.n);
    }
    k_audit<<<static_cast<unsigned>((n + 63) / 64), 64, 0, c.stream>>>(T, T32, t ? nullptr : d_dict, d_q64, d_rec,
                                                                        n, d_e, d_e + 1);
    MRFG_CUDA(cudaGetLastError());
    unsigned h[2] = {0, 0};
    MRFG_CUDA(cudaMemcpyAsync(h, d_e, sizeof h, cudaMemcpyDeviceToHost, c.stream));
    MRFG_CUDA(cudaStreamSynchronize(c.stream));
    float f[2];
    std::memcpy(f, h, sizeof f);
    *err16 = f[0];
    *err32 = f[1];
}

void launch_dict_operand(Ctx& c, const float* d_dict, int64_t first, int64_t count, int64_t rows,
                         int64_t stride, int metric, __half* d_a, float* d_inv2) {
    const int bs = 256;
    k_dict_operand<<<(rows * 32 + bs - 1) / bs, bs, 0, c.stream>>>(
        d_dict, first, count, stride, static_cast<int>(c.n), k_pad_of(c.n),
        metric == MRFG_METRIC_CC ? 0 : 1, d_a, d_inv2, rows);
    MRFG_CUDA(cudaGetLastError());
}

void launch_merge(Ctx& c, const mrfg_match* d_in, int nranks, int64_t nq, mrfg_match* d_out) {
    const int bs = 256;
    k_merge<<<(nq + bs - 1) / bs, bs, 0, c.stream>>>(d_in, nranks, nq, d_out);
    MRFG_CUDA(cudaGetLastError());
}

void launch_cc_map(Ctx& c, const GridTables& t, const double* d_q64, int64_t first, int64_t count,
                   float* d_out) {
    const int bs = 64;
    k_cc_map<<<(count + bs - 1) / bs, bs, 0, c.stream>>>(tab64_of(c, t), d_q64, first, count, d_out);
    MRFG_CUDA(cudaGetLastError());
}

}  // namespace mrfg
