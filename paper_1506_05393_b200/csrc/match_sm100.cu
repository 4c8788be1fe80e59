// match_sm100.cu -- K2: fused complex-correlation screening GEMM on tcgen05.
//
// Replaces the scan loop of scan_grid / brute_force_search (reference
// proj/src/dictionary.cpp:283-299, 241-255; score cc_against_entry :117-127).
// The complex correlation of unit query q_v with atom d_a,
//     z = sum_j q_vj conj(d_aj),
// is a real GEMM over K = 2N: atoms are stored as interleaved (re, im) rows
// (the reference's dictionary layout) and each voxel contributes two rows
//     row 2v   = ( qr_0,  qi_0, qr_1,  qi_1, ...)  -> Re z
//     row 2v+1 = ( qi_0, -qr_0, qi_1, -qr_1, ...)  -> Im z
// so S = A (atoms x 2N) . B^T (2N x 2V) lands Re/Im of each voxel in adjacent
// accumulator columns.  fp16 operands, FP32 accumulation in TMEM.
//
// Kernel shape: persistent, one CTA per SM, 256 threads:
//   warp 0 : TMA producer (A tile 128x64, B tile 256x64, SWIZZLE_128B, 4 stages)
//   warp 1 : single-thread tcgen05.mma issuer, M=128 N=256 K=16, cta_group::1
//   warp 2 : TMEM allocator (512 columns = two 128x256 FP32 accumulators)
//   warps 4-7 : epilogue -- tcgen05.ld of its 32 TMEM lanes (one atom per
//              thread), score = |z|^2 / |d|^2 (approx CC^2), compare with the
//              per-voxel threshold (running max - delta)^2 and append the
//              rare survivors to a global candidate list for the exact
//              FP64 re-rank (rerank.cu).  The epilogue of tile i overlaps
//              the MMAs of tile i+1 (double-buffered TMEM).
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "mrfg_internal.cuh"

namespace mrfg {
namespace {

constexpr int BM = 128;  // atoms per tile (TMEM lanes)
constexpr int BN = 256;  // query rows per tile = 128 voxels
constexpr int BK = 64;   // fp16 elements per 128-byte swizzle row
constexpr int STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;
constexpr int B_BYTES = BN * BK * 2;
constexpr int NTHREADS = 256;

struct alignas(1024) Smem {
    uint8_t a[STAGES][A_BYTES];
    uint8_t b[STAGES][B_BYTES];
    uint64_t full[STAGES], empty[STAGES], tfull[2], tempty[2];
    uint32_t tmem_base;
    float thr[2][128];
    float bst[2][128];
    uint32_t hv[2][128];
};
constexpr size_t SMEM_BYTES = sizeof(Smem) + 1024;

struct Dev {
    const float* inv2;
    int64_t vox_base;  // global index of this launch's voxel 0 (candidate records)
    int64_t n_at, n_vt, nkb, last_sub;
    int64_t ga;  // tile raster: 1 = atom-major; > 1 = groups of ga atom tiles per query tile
    int64_t valid_atoms, valid_begin, nvox, flat_base, flat_stride;
    float* best;
    CandRec* cand;
    unsigned long long* cand_count;
    int64_t cand_cap;
    float delta;
    int metric;
    CandRec* audit;
    unsigned long long* audit_count;
    int64_t audit_cap;
    uint32_t audit_thr;
    // two-level audit sample (same expected fraction audit_thr / 2^32 of all
    // pairs, still independent of the scores): atoms whose hash has its top
    // audit_shift bits clear, then pairs whose mixed hash is below
    // audit_thr << audit_shift -- the per-pair hash is computed for 1/2^shift
    // of the atom rows only (it was half of the epilogue's per-pair work)
    uint32_t audit_shift, audit_thr_pairs;
};

// Tile t -> (atom tile, query tile).  ga = 1: atom-major (the query operand
// is L2-resident, each atom tile is read once).  ga > 1 (query operand far
// larger than L2, configs 3/5): the ga concurrently running CTAs (pairs) take
// ga different atom tiles of the SAME query tile, so every query tile is
// fetched from HBM once per ga atom tiles and the group's atom tiles stay in
// L2 while it sweeps the query tiles.
__device__ __forceinline__ void tile_coords(int64_t t, int64_t n_at, int64_t n_vt, int64_t ga, int64_t& at,
                                            int64_t& vt) {
    if (ga <= 1) {
        at = t / n_vt;
        vt = t % n_vt;
        return;
    }
    const int64_t per = ga * n_vt, g0 = t / per * ga, rem = t % per;
    const int64_t gsz = n_at - g0 < ga ? n_at - g0 : ga;  // the last group may be smaller
    vt = rem / gsz;
    at = g0 + rem % gsz;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(b)), "r"(parity)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, void* dst, uint64_t* bar,
                                            int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tc_mma_f16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                           uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// UMMA shared-memory descriptor, K-major SWIZZLE_128B canonical layout:
// rows of 128 B, 8-row core groups 1024 B apart (SBO), version 1 (sm_100).
__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr & 0x3FFFF) >> 4);
    d |= static_cast<uint64_t>(1) << 16;   // LBO (unused for swizzled K-major)
    d |= static_cast<uint64_t>(64) << 32;  // SBO = 1024 B
    d |= static_cast<uint64_t>(1) << 46;   // descriptor version (sm_100)
    d |= static_cast<uint64_t>(2) << 61;   // SWIZZLE_128B
    return d;
}
// Instruction descriptor: D=F32, A=B=F16, both K-major, N=256, M=128.
constexpr uint32_t IDESC = (1u << 4) | (static_cast<uint32_t>(BN >> 3) << 17) |
                           (static_cast<uint32_t>(BM >> 4) << 24);

#define TMEM_LD_X64(taddr, r)                                                                 \
    asm volatile(                                                                             \
        "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13," \
        "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,"  \
        "%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,"  \
        "%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"                                              \
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),  \
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),           \
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),        \
          "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),        \
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),        \
          "=r"(r[31]), "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]),        \
          "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]),        \
          "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]),        \
          "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]),        \
          "=r"(r[55]), "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]),        \
          "=r"(r[61]), "=r"(r[62]), "=r"(r[63])                                                \
        : "r"(taddr))

__device__ __forceinline__ void atomic_max_float(float* addr, float v) {
    if (v >= 0.f)
        atomicMax(reinterpret_cast<int*>(addr), __float_as_int(v));
    else
        atomicMin(reinterpret_cast<unsigned*>(addr), __float_as_uint(v));
}

__device__ __forceinline__ float screen_score(float re, float im, float inv, int metric) {
    // metric cc: |z|^2/|d|^2 (squared CC); euclidean: Re z/|d| (monotone in
    // -|q-d| for unit vectors).
    return metric == MRFG_METRIC_CC ? (re * re + im * im) * inv : re * inv;
}
__device__ __forceinline__ float threshold_of(float best, float delta, int metric) {
    float t = best - delta;
    if (metric == MRFG_METRIC_CC) return t > 0.f ? t * t : 0.f;
    return t;
}
__device__ __forceinline__ float unsquare(float s, int metric) {
    return metric == MRFG_METRIC_CC ? sqrtf(s) : s;
}

__device__ __forceinline__ void push_candidate(const Dev& p, int64_t v, int64_t atom, float s) {
    if (p.cand != nullptr) {
        unsigned long long idx = atomicAdd(p.cand_count, 1ull);
        if (idx < static_cast<unsigned long long>(p.cand_cap)) {
            CandRec rec;
            rec.voxel = static_cast<uint32_t>(p.vox_base + v);
            rec.s = s;
            rec.flat = p.flat_base + atom * p.flat_stride;
            p.cand[idx] = rec;
        }
    }
}

__device__ __noinline__ void record_hit(const Dev& p, float bst, int64_t v, int64_t atom, float sc) {
    push_candidate(p, v, atom, sc);
    const float su = unsquare(sc, p.metric);
    if (su > bst) atomic_max_float(p.best + v, su);
}

// Warp-aggregated candidate append for one 32-column block of the epilogue:
// lane l holds the hit mask of its atom over the block's 32 voxels.  One
// atomicAdd per warp reserves the warp's slots (warp prefix sum of the
// per-lane counts) instead of one contended atomic per hit on the single
// global counter (config 3 records 1.2e8 candidates); returns this lane's
// first slot.
__device__ __noinline__ unsigned long long reserve_hits(const Dev& p, uint32_t hits) {
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int mine = __popc(hits);
    int incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(full, incl, o);
        if (lane >= o) incl += t;
    }
    unsigned long long base = 0;
    if (lane == 31 && p.cand != nullptr && incl > 0)
        base = atomicAdd(p.cand_count, static_cast<unsigned long long>(incl));
    base = __shfl_sync(full, base, 31);
    return base + static_cast<unsigned long long>(incl - mine);
}

// One audit-sampled pair (rare): recorded whatever its score, valid voxels only.
__device__ __noinline__ void record_audit(const Dev& p, int64_t v, int64_t atom, float sc) {
    if (v >= p.nvox) return;
    const unsigned long long idx = atomicAdd(p.audit_count, 1ull);
    if (idx < static_cast<unsigned long long>(p.audit_cap)) {
        CandRec rec;
        rec.voxel = static_cast<uint32_t>(p.vox_base + v);
        rec.s = sc;
        rec.flat = p.flat_base + atom * p.flat_stride;
        p.audit[idx] = rec;
    }
}

// One reserved hit: the candidate record and the running maximum.
__device__ __noinline__ void store_hit(const Dev& p, float bst, int64_t v, int64_t atom, float sc,
                                       unsigned long long idx) {
    if (p.cand != nullptr && idx < static_cast<unsigned long long>(p.cand_cap)) {
        CandRec rec;
        rec.voxel = static_cast<uint32_t>(p.vox_base + v);
        rec.s = sc;
        rec.flat = p.flat_base + atom * p.flat_stride;
        p.cand[idx] = rec;
    }
    const float su = unsquare(sc, p.metric);
    if (su > bst) atomic_max_float(p.best + v, su);
}

__global__ void __launch_bounds__(NTHREADS, 1)
    k_match_sm100(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                  Dev p) {
    extern __shared__ uint8_t smem_raw[];
    Smem& s = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                       ~static_cast<uintptr_t>(1023));
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int64_t n_tiles = p.n_at * p.n_vt;

    if (warp == 0 && lane == 0) {
        for (int i = 0; i < STAGES; ++i) {
            mbar_init(&s.full[i], 1);
            mbar_init(&s.empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&s.tfull[i], 1);
            mbar_init(&s.tempty[i], 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_a)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_b)) : "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&s.tmem_base)),
                     "r"(512)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s.tmem_base;

    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
                int64_t at64, vt64;
                tile_coords(t, p.n_at, p.n_vt, p.ga, at64, vt64);
                const int at = static_cast<int>(at64), vt = static_cast<int>(vt64);
                for (int kb = 0; kb < p.nkb; ++kb) {
                    mbar_wait(&s.empty[stage], phase ^ 1);
                    mbar_expect_tx(&s.full[stage], A_BYTES + B_BYTES);
                    tma_load_2d(&tma_a, s.a[stage], &s.full[stage], kb * BK, at * BM);
                    tma_load_2d(&tma_b, s.b[stage], &s.full[stage], kb * BK, vt * BN);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
                mbar_wait(&s.tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d = tmem + static_cast<uint32_t>(acc * BN);
                for (int kb = 0; kb < p.nkb; ++kb) {
                    mbar_wait(&s.full[stage], phase);
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(s.a[stage]), b0 = smem_u32(s.b[stage]);
                    const int nsub = kb == p.nkb - 1 ? static_cast<int>(p.last_sub) : BK / 16;
                    for (int k = 0; k < nsub; ++k) {
                        tc_mma_f16(d, smem_desc_sw128(a0 + 32 * k), smem_desc_sw128(b0 + 32 * k), IDESC,
                                   (kb | k) != 0);
                    }
                    tc_commit(&s.empty[stage]);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                tc_commit(&s.tfull[acc]);
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
            }
        }
    } else if (warp >= 4) {
        // ------------------------------------------------ epilogue
        const int ew = warp - 4;  // == warp % 4: TMEM lane quarter
        const int row = ew * 32 + lane;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
            int64_t at, vt;
            tile_coords(t, p.n_at, p.n_vt, p.ga, at, vt);
            {
                const int64_t v = vt * 128 + row;
                float b = v < p.nvox ? __ldcg(p.best + v) : 1e30f;
                // padding voxel columns can never screen in
                s.thr[acc][row] = v < p.nvox ? threshold_of(b, p.delta, p.metric) : __int_as_float(0x7f800000);
                s.bst[acc][row] = b;
                s.hv[acc][row] = audit_hash_voxel(static_cast<uint64_t>(p.vox_base + v));
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");
            mbar_wait(&s.tfull[acc], acc_phase);
            tc_fence_after();
            const int64_t atom = at * BM + row;
            const bool avalid = atom >= p.valid_begin && atom < p.valid_atoms;
            const float inv = __ldg(p.inv2 + atom);
            const uint32_t ha = audit_hash_flat(static_cast<uint64_t>(p.flat_base + atom * p.flat_stride));
            const bool asamp = p.audit_thr != 0u && avalid && (p.audit_shift == 0u || (ha >> (32u - p.audit_shift)) == 0u);
            const uint32_t tbase = tmem + (static_cast<uint32_t>(ew * 32) << 16) +
                                   static_cast<uint32_t>(acc * BN);
#pragma unroll 1
            for (int q = 0; q < 4; ++q) {
                uint32_t r[64];
                TMEM_LD_X64(tbase + q * 64, r);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                float sc[32];
                uint32_t hits = 0;
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    sc[i] = screen_score(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]), inv,
                                         p.metric);
                    hits |= (sc[i] >= s.thr[acc][q * 32 + i] ? 1u : 0u) << i;
                }
                if (!avalid) hits = 0;
                if (__any_sync(0xffffffffu, hits != 0)) {
                    unsigned long long slot = reserve_hits(p, hits);
#pragma unroll
                    for (int i = 0; i < 32; ++i)
                        if ((hits >> i) & 1u)
                            store_hit(p, s.bst[acc][q * 32 + i], vt * 128 + q * 32 + i, atom, sc[i], slot++);
                }
                if (asamp) {
                    uint32_t samp = 0;
#pragma unroll
                    for (int i = 0; i < 32; ++i)
                        samp |= (audit_mix(ha, s.hv[acc][q * 32 + i]) < p.audit_thr_pairs ? 1u : 0u) << i;
                    if (samp) {
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            if ((samp >> i) & 1u) record_audit(p, vt * 128 + q * 32 + i, atom, sc[i]);
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&s.tempty[acc]);
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1;
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512)
                     : "memory");
    }
}

// ------------------------------------------------------------------------
// CTA-pair variant: tcgen05.mma.cta_group::2, M = 256 atoms per pair.
// Each CTA of the cluster owns 128 atom rows (A) and half of the 256 query
// rows (B); the leader's single thread issues the pair-wide MMA, the tensor
// cores of both SMs read both B halves, and each CTA's TMEM receives its
// 128 atoms x 256 columns.  Per SM the smem/L2 operand traffic per MMA step
// drops from (128 + 256) to (128 + 128) rows.
constexpr int STAGES2 = 6;
constexpr int B2_BYTES = (BN / 2) * BK * 2;
struct alignas(1024) Smem2 {
    uint8_t a[STAGES2][A_BYTES];
    uint8_t b[STAGES2][B2_BYTES];
    uint64_t full[STAGES2], empty[STAGES2], tfull[2], tempty[2];
    uint32_t tmem_base;
    float thr[2][128];
    float bst[2][128];
    uint32_t hv[2][128];
};
constexpr size_t SMEM2_BYTES = sizeof(Smem2) + 1024;
constexpr uint32_t IDESC2 = (1u << 4) | (static_cast<uint32_t>(BN >> 3) << 17) |
                            (static_cast<uint32_t>(256 >> 4) << 24);

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t map_to_rank(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
// Remote arrive with the default (CTA-scope) semantics: the data it guards is
// either TMA-tracked (transaction bytes) or TMEM (ordered by the tcgen05
// fences), so no GPU-scope fence is needed -- `.release.cluster` here compiled
// to MEMBAR.ALL.GPU per pipeline stage and starved the pair's MMA.
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(const CUtensorMap* map, void* dst, uint64_t* bar, int c0,
                                                 int c1) {
    // both CTAs load their half; the transaction bytes land on the leader's barrier
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar) & 0xFEFFFFFFu)
        : "memory");
}
__device__ __forceinline__ void tc_mma_f16_pair(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                                uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void tc_commit_pair(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(static_cast<uint16_t>(3))
        : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NTHREADS, 1)
    k_match_sm100_2cta(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                       Dev p) {
    extern __shared__ uint8_t smem_raw[];
    Smem2& s = *reinterpret_cast<Smem2*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                         ~static_cast<uintptr_t>(1023));
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    const int64_t cid = blockIdx.x / 2, ncl = gridDim.x / 2;
    const int64_t n_at = p.n_at / 2, n_vt = p.n_vt;  // 256-atom pair tiles
    const int64_t n_tiles = n_at * n_vt;

    if (warp == 0 && lane == 0) {
        for (int i = 0; i < STAGES2; ++i) {
            mbar_init(&s.full[i], 2);  // leader's arrive_expect_tx + the peer's arrive
            mbar_init(&s.empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&s.tfull[i], 1);
            mbar_init(&s.tempty[i], 8);  // 4 epilogue warps x 2 CTAs
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_a)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_b)) : "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&s.tmem_base)),
                     "r"(512)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = s.tmem_base;

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int64_t t = cid; t < n_tiles; t += ncl) {
                int64_t at64, vt64;
                tile_coords(t, n_at, n_vt, p.ga, at64, vt64);
                const int at = static_cast<int>(at64), vt = static_cast<int>(vt64);
                for (int kb = 0; kb < p.nkb; ++kb) {
                    mbar_wait(&s.empty[stage], phase ^ 1);
                    if (leader)
                        mbar_expect_tx(&s.full[stage], 2 * (A_BYTES + B2_BYTES));
                    else
                        mbar_arrive_cluster(map_to_rank(smem_u32(&s.full[stage]), 0));
                    tma_load_2d_pair(&tma_a, s.a[stage], &s.full[stage], kb * BK,
                                     at * 256 + static_cast<int>(rank) * 128);
                    tma_load_2d_pair(&tma_b, s.b[stage], &s.full[stage], kb * BK,
                                     vt * BN + static_cast<int>(rank) * (BN / 2));
                    if (++stage == STAGES2) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (leader && lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int64_t t = cid; t < n_tiles; t += ncl) {
                mbar_wait(&s.tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d = tmem + static_cast<uint32_t>(acc * BN);
                for (int kb = 0; kb < p.nkb; ++kb) {
                    mbar_wait(&s.full[stage], phase);
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(s.a[stage]), b0 = smem_u32(s.b[stage]);
                    const int nsub = kb == p.nkb - 1 ? static_cast<int>(p.last_sub) : BK / 16;
                    for (int k = 0; k < nsub; ++k)
                        tc_mma_f16_pair(d, smem_desc_sw128(a0 + 32 * k), smem_desc_sw128(b0 + 32 * k), IDESC2,
                                        (kb | k) != 0);
                    tc_commit_pair(&s.empty[stage]);
                    if (++stage == STAGES2) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                tc_commit_pair(&s.tfull[acc]);
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
            }
        }
    } else if (warp >= 4) {
        const int ew = warp - 4;
        const int row = ew * 32 + lane;
        const uint32_t tempty_leader[2] = {map_to_rank(smem_u32(&s.tempty[0]), 0),
                                           map_to_rank(smem_u32(&s.tempty[1]), 0)};
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int64_t t = cid; t < n_tiles; t += ncl) {
            int64_t at, vt;
            tile_coords(t, n_at, n_vt, p.ga, at, vt);
            {
                const int64_t v = vt * 128 + row;
                float b = v < p.nvox ? __ldcg(p.best + v) : 1e30f;
                s.thr[acc][row] = v < p.nvox ? threshold_of(b, p.delta, p.metric) : __int_as_float(0x7f800000);
                s.bst[acc][row] = b;
                s.hv[acc][row] = audit_hash_voxel(static_cast<uint64_t>(p.vox_base + v));
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");
            mbar_wait(&s.tfull[acc], acc_phase);
            tc_fence_after();
            const int64_t atom = at * 256 + static_cast<int64_t>(rank) * 128 + row;
            const bool avalid = atom >= p.valid_begin && atom < p.valid_atoms;
            const float inv = __ldg(p.inv2 + atom);
            const uint32_t ha = audit_hash_flat(static_cast<uint64_t>(p.flat_base + atom * p.flat_stride));
            const bool asamp = p.audit_thr != 0u && avalid && (p.audit_shift == 0u || (ha >> (32u - p.audit_shift)) == 0u);
            const uint32_t tbase = tmem + (static_cast<uint32_t>(ew * 32) << 16) +
                                   static_cast<uint32_t>(acc * BN);
#pragma unroll 1
            for (int q = 0; q < 4; ++q) {
                uint32_t r[64];
                TMEM_LD_X64(tbase + q * 64, r);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                float sc[32];
                uint32_t hits = 0;
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    sc[i] = screen_score(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]), inv,
                                         p.metric);
                    hits |= (sc[i] >= s.thr[acc][q * 32 + i] ? 1u : 0u) << i;
                }
                if (!avalid) hits = 0;
                if (__any_sync(0xffffffffu, hits != 0)) {
                    unsigned long long slot = reserve_hits(p, hits);
#pragma unroll
                    for (int i = 0; i < 32; ++i)
                        if ((hits >> i) & 1u)
                            store_hit(p, s.bst[acc][q * 32 + i], vt * 128 + q * 32 + i, atom, sc[i], slot++);
                }
                if (asamp) {
                    uint32_t samp = 0;
#pragma unroll
                    for (int i = 0; i < 32; ++i)
                        samp |= (audit_mix(ha, s.hv[acc][q * 32 + i]) < p.audit_thr_pairs ? 1u : 0u) << i;
                    if (samp) {
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            if ((samp >> i) & 1u) record_audit(p, vt * 128 + q * 32 + i, atom, sc[i]);
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(tempty_leader[acc]);
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1;
        }
    }

    tc_fence_before();
    cluster_sync_all();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512)
                     : "memory");
    }
}

// CUDA-core version of the same fused screening (tests: validates the
// tcgen05 descriptors/layouts against identical fp16 operands).
__global__ void k_match_simt(const __half* __restrict__ a, const __half* __restrict__ b,
                             int64_t k_pad, Dev p, int64_t atoms, float* __restrict__ debug) {
    int64_t atom = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    int64_t v = blockIdx.y;
    if (atom >= atoms || v >= p.nvox) return;
    float re = 0.f, im = 0.f;
    for (int64_t k = 0; k < k_pad; ++k) {
        float x = __half2float(a[atom * k_pad + k]);
        re = fmaf(x, __half2float(b[(2 * v) * k_pad + k]), re);
        im = fmaf(x, __half2float(b[(2 * v + 1) * k_pad + k]), im);
    }
    float sc = screen_score(re, im, p.inv2[atom], p.metric);
    if (debug) debug[atom * p.nvox + v] = sc;
    if (atom >= p.valid_atoms || atom < p.valid_begin) return;
    float b0 = __ldcg(p.best + v);
    if (sc >= threshold_of(b0, p.delta, p.metric)) {
        push_candidate(p, v, atom, sc);
        atomic_max_float(p.best + v, unsquare(sc, p.metric));
    }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encoder(Ctx& c) {
    if (!c.encode_fn) {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        MRFG_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        MRFG_REQUIRE(fn != nullptr && q == cudaDriverEntryPointSuccess, MRFG_E_CUDA,
                     "cuTensorMapEncodeTiled unavailable");
        c.encode_fn = fn;
    }
    return reinterpret_cast<EncodeTiledFn>(c.encode_fn);
}

CUtensorMap make_map(Ctx& c, const __half* base, int64_t rows, int64_t k_pad, int box_rows) {
    CUtensorMap m;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(k_pad), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(k_pad * 2)};
    cuuint32_t box[2] = {BK, static_cast<cuuint32_t>(box_rows)};
    cuuint32_t es[2] = {1, 1};
    CUresult r = get_encoder(c)(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<__half*>(base),
                                dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    MRFG_REQUIRE(r == CUDA_SUCCESS, MRFG_E_CUDA, "cuTensorMapEncodeTiled failed");
    return m;
}

Dev dev_of(const MatchParams& p, int64_t k_valid) {
    Dev d;
    d.inv2 = p.inv2;
    d.vox_base = p.vox_base;
    d.n_at = p.atoms / BM;
    d.n_vt = p.q_rows / BN;
    d.nkb = p.k_pad / BK;
    int64_t last = k_valid - (d.nkb - 1) * BK;  // valid elements of the last K block
    d.last_sub = (last + 15) / 16;
    if (d.last_sub < 1) d.last_sub = 1;
    d.valid_atoms = p.valid_atoms;
    d.valid_begin = p.valid_begin;
    d.nvox = p.nvox;
    d.flat_base = p.flat_base;
    d.flat_stride = p.flat_stride;
    d.best = p.best;
    d.cand = p.cand;
    d.cand_count = p.cand_count;
    d.cand_cap = p.cand_cap;
    d.delta = p.delta;
    d.metric = p.metric;
    d.ga = 1;
    d.audit = p.audit;
    d.audit_count = p.audit_count;
    d.audit_cap = p.audit_cap;
    d.audit_thr = (p.audit != nullptr && p.audit_count != nullptr) ? p.audit_thr : 0u;
    d.audit_shift = 0;
    while (d.audit_shift < 8 && (static_cast<uint64_t>(d.audit_thr) << (d.audit_shift + 1)) <= 0xffffffffull &&
           d.audit_thr != 0u)
        ++d.audit_shift;
    d.audit_thr_pairs = d.audit_thr << d.audit_shift;
    return d;
}

// Raster group size (MRFG_K2_GROUP; default 1 = atom-major).  Measured on
// config 3 (2.1 GB query operand): one group per wave of concurrent CTA pairs
// (74) ran the GEMM at 802 vs 940 TFLOP/s atom-major, config 5 977 vs 1011.
int64_t group_of(const MatchParams&, int64_t) {
    if (const char* e = std::getenv("MRFG_K2_GROUP")) return std::max<int64_t>(1, std::atoll(e));
    return 1;
}

}  // namespace

// K2 variant: the CTA-pair kernel when the chunk is a multiple of 256 atoms
// (MRFG_K2_PAIR=0 forces the single-CTA kernel).
static bool use_pair_kernel() {
    const char* e = std::getenv("MRFG_K2_PAIR");
    return !(e && e[0] == '0');
}

void launch_match(Ctx& c, const MatchParams& p) {
    MRFG_REQUIRE(p.atoms % BM == 0 && p.q_rows % BN == 0 && p.k_pad % BK == 0, MRFG_E_INVALID,
                 "match: operand shapes not tile aligned");
    // the shared-memory opt-in is per device (a process may drive several
    // GPUs), so it is set on every launch, like the K1/K5 attributes
    MRFG_CUDA(cudaFuncSetAttribute(k_match_sm100, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(SMEM_BYTES)));
    MRFG_CUDA(cudaFuncSetAttribute(k_match_sm100_2cta, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(SMEM2_BYTES)));
    Dev d = dev_of(p, p.k_valid > 0 ? p.k_valid : 2 * c.n);
    if (use_pair_kernel() && p.atoms % 256 == 0) {
        CUtensorMap ma = make_map(c, p.a, p.atoms, p.k_pad, 128);
        CUtensorMap mb = make_map(c, p.b, p.q_rows, p.k_pad, BN / 2);
        const int64_t tiles = (p.atoms / 256) * d.n_vt;
        const int64_t pairs = std::min<int64_t>(tiles, c.num_sms / 2);
        d.ga = group_of(p, pairs);
        k_match_sm100_2cta<<<static_cast<int>(2 * pairs), NTHREADS, SMEM2_BYTES, c.stream>>>(ma, mb, d);
        MRFG_CUDA(cudaGetLastError());
        return;
    }
    CUtensorMap ma = make_map(c, p.a, p.atoms, p.k_pad, BM);
    CUtensorMap mb = make_map(c, p.b, p.q_rows, p.k_pad, BN);
    int64_t tiles = d.n_at * d.n_vt;
    int grid = static_cast<int>(tiles < c.num_sms ? tiles : c.num_sms);
    d.ga = group_of(p, grid);
    k_match_sm100<<<grid, NTHREADS, SMEM_BYTES, c.stream>>>(ma, mb, d);
    MRFG_CUDA(cudaGetLastError());
}

void launch_match_simt(Ctx& c, const MatchParams& p) {
    Dev d = dev_of(p, p.k_valid > 0 ? p.k_valid : 2 * c.n);
    dim3 grid(static_cast<unsigned>((p.atoms + 127) / 128), static_cast<unsigned>(p.nvox));
    k_match_simt<<<grid, 128, 0, c.stream>>>(p.a, p.b, p.k_pad, d, p.atoms, p.debug_scores);
    MRFG_CUDA(cudaGetLastError());
}

}  // namespace mrfg
