// mrfg_internal.cuh -- shared declarations of the sm_100a DGS path.
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "mrfg.h"

namespace mrfg {

// ------------------------------------------------------------------ errors
struct Error {
    int code;
    std::string msg;
};
void set_error(const std::string& msg);
#define MRFG_CUDA(call)                                                                  \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess)                                                           \
            throw ::mrfg::Error{MRFG_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)}; \
    } while (0)
#define MRFG_REQUIRE(cond, code, msg)                          \
    do {                                                       \
        if (!(cond)) throw ::mrfg::Error{(code), (msg)};       \
    } while (0)

// ---------------------------------------------------------- device buffers
// Owning, move-only device allocation (grow-only via ensure).  The owner
// frees on destruction; callers keep the right device current.
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes) {
        o.p = nullptr;
        o.bytes = 0;
    }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            release();
            p = o.p;
            bytes = o.bytes;
            o.p = nullptr;
            o.bytes = 0;
        }
        return *this;
    }
    ~DevBuf() { release(); }
    void ensure(size_t n) {
        if (n <= bytes) return;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        MRFG_CUDA(cudaMalloc(&p, n));
        bytes = n;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    template <class T>
    T* as() const { return static_cast<T*>(p); }
};

// Per-(context, grid) transcendental tables.  FP64 values are computed on
// the HOST with the same libm calls and operand order as the reference
// (bloch.cpp:17-21), so the FP64 device recursion reproduces the reference
// bit-for-bit; the FP32 tables are those values rounded.
// Per-step data every FP32 producer thread shares (staged in shared memory):
// RF matrix, te/rest [s], and the off-resonance pitch phasors
// w = e^{i 2 pi ddf te}, e^{i 2 pi ddf rest} (host FP64 -> FP32).
struct StepU {
    float r[9];
    float te, rest;
    float wtc, wts, wrc, wrs;
    float pad;
};
static_assert(sizeof(StepU) == 64, "StepU is 4 x 16 B");

struct GridTables {
    mrfg_grid grid{};
    std::vector<double> v1, v2;  // explicit T1/T2 values of the cached grid (empty: evenly spaced)
    DevBuf kt;  // float log2(e)/T1 [n1] then log2(e)/T2 [n2], 1/s (K1 row producers)
    DevBuf stepu;  // n x StepU
    DevBuf stepx;  // x-axis schedules: n x 2 float4 (r4, r5, r7, r8), (wtc, wts, wrc, wrs) (K5 screening)
    bool valid = false;
    // Parameter-major (lattice index i, step j):
    // FP32: e1[i*n+j] = (E1te, 1-E1te, E1rest, 1-E1rest); e2[i*n+j] = (E2te, E2rest);
    //       ph[i*n+j] = (cos te, sin te, cos rest, sin rest)
    DevBuf e1f, e2f, phf;
    // FP64, same index order: e1d[(i*n+j)*2 + {0,1}] = (E1te, E1rest); e2d likewise;
    // phd[(i*n+j)*4 + {0..3}] = (cos te, sin te, cos rest, sin rest)
    DevBuf e1d, e2d, phd;
    // subspace screening (MRFG_SUBSPACE=r): per-df bases W[df][cols][k_pad] (fp16), built on first use
    DevBuf subw;
    int sub_r = 0;
    double sub_rho_held = 0;  // largest relative residual |a - P a| / |a| over the held-out rows, all df
};

struct Ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int num_sms = 148;
    int64_t n = 0;  // schedule length
    std::vector<double> flip_deg, phase_deg, tr_ms, te_ms;
    std::vector<double> rf64;       // n x 9 (bloch.cpp:101)
    std::vector<double> te_s, rest_s;
    double inv64[9];                // kInvert (bloch.cpp:113)
    bool rf_xaxis = false;          // every RF rotation is about x (phases 0/180 deg): K1 specialization
    bool te_sym = false;            // te == rest at every TR (TE = TR/2): K1 symmetric-echo specialization
    DevBuf rf64_d, rf32_d;          // n x 9 doubles; n x 12 floats (9 RF, te, rest, pad)
    GridTables tab;                 // cache for the last grid
    // scratch
    DevBuf zoom;  // K5 per-warp scratch (grow-only: no allocation inside a timed call)
    DevBuf q64, qprime, best, cand, cand_count, atoms_a, inv2, seed_a, seed_inv2, rerank,
        params, out64, misc, rerank_scratch, misc2, audit,
        // persistent buffers of the host-buffer entry points (no per-call cudaMalloc)
        h_raw, h_res, h_dict, h_zdict, h_trace, zidx, zib,
        sub_c, sub_q, sub_rho;  // subspace screening: atom / query coefficients, max residual
    // producer stream + events for the K1/K2 overlap (created on first use)
    cudaStream_t aux = nullptr;
    cudaEvent_t ev[8] = {};
    void ensure_aux() {
        if (aux) return;
        MRFG_CUDA(cudaStreamCreateWithFlags(&aux, cudaStreamNonBlocking));
        for (auto& e : ev) MRFG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    // tensor-map encoder (driver entry point)
    void* encode_fn = nullptr;
};

// ------------------------------------------------------------ host helpers
void host_rf_matrix(double alpha, double phi, double out[9]);  // bloch.cpp:63-66
const GridTables& ensure_tables(Ctx& c, const mrfg_grid& g, bool need64);
// AxisSpec::value (dictionary.hpp:22), or the explicit value
inline double axis_value(const mrfg_axis& a, int64_t i) {
    return a.values ? a.values[i] : a.min + static_cast<double>(i) * a.step;
}
inline bool grid_explicit(const mrfg_grid& g) {
    return g.t1_ms.values || g.t2_ms.values || g.df_hz.values;
}
inline int64_t grid_total(const mrfg_grid& g) {
    return g.t1_ms.count * g.t2_ms.count * g.df_hz.count;
}
inline int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }
inline int64_t k_pad_of(int64_t n) { return round_up(2 * n, 64); }  // fp16 elements per GEMM row

// --------------------------------------------------------------- launchers
// K1 (bloch.cu)
void launch_simulate64(Ctx& c, const double* d_params, int64_t count, int normalize, double* d_out);
void launch_simulate32(Ctx& c, const double* d_params, int64_t count, int normalize, double* d_out);
void launch_generate(Ctx& c, const GridTables& t, int64_t first, int64_t count, int precision,
                     float* d_out);
// Rows r in [0, rows) simulate flat first + r*stride (zero rows past valid_end);
// inv2 gets 1/|s|^2 (metric cc) or 1/|s| (euclidean).
void launch_bloch_operand(Ctx& c, const GridTables& t, int64_t first, int64_t stride,
                          int64_t valid_end, int64_t rows, int metric, __half* d_a,
                          float* d_inv2);
// Row-tiled K1 over flats [vb, ve) (out 0: fp16 operand + inv; 1: raw float
// entries; 2: |s|^2; 3: FP32 cc_map score against the unit query d_q32 into
// d_inv2[flat - vb]).  Returns base_flat (operand row = flat - base_flat);
// for out 0 the buffer rows outside the range, up to `rows`, are zeroed.
int64_t launch_bloch_rows(Ctx& c, const GridTables& t, int64_t vb, int64_t ve, int metric, int out,
                          int64_t rows, __half* d_a, float* d_outf, float* d_inv2,
                          const float2* d_q32 = nullptr);
void launch_bloch_norms(Ctx& c, const GridTables& t, int64_t first, int64_t count, float* d_norm2);
// subspace screening (subspace.cu)
int subspace_rank(int r);   // supported complex ranks: 8, 16, 32, 48, 64
int subspace_cols(int r);   // real basis rows, 2 r
int subspace_pitch(int r);  // coefficient row pitch (multiple of 64: K2's K blocks)
const __half* ensure_subspace(Ctx& c, const GridTables& t, int r);
void launch_project(Ctx& c, const __half* A, int64_t rows, int64_t kpad, const __half* W, int nw, __half* out,
                    int opitch, const float* inv2, int64_t valid, unsigned int* rho2max, int batch = 1,
                    int64_t w_stride = 0, int64_t o_stride = 0);
bool bloch_dfquad_ok(const Ctx& c);
void launch_bloch_dfquad(Ctx& c, const GridTables& t, int idf0, int64_t row_lo, int64_t nrows, int64_t pitch,
                         int metric, __half* d_a, float* d_inv2);

// K2 (match_sm100.cu)
struct CandRec {
    uint32_t voxel;
    float s;       // screening score (CC or Re-part units)
    int64_t flat;
};
struct MatchParams {
    const __half* a;    // atoms x k_pad (fp16, K-major)
    const float* inv2;  // atoms
    const __half* b;    // q_rows x k_pad (fp16, K-major): rows 2v (re), 2v+1 (im)
    int64_t atoms;      // multiple of 128
    int64_t q_rows;     // multiple of 256
    int64_t k_pad;      // multiple of 64
    int64_t k_valid = 0;  // valid K elements (0: 2 * timepoints); subspace operands: 2 * rank
    int64_t valid_atoms;  // local atoms in [valid_begin, valid_atoms) are real
    int64_t valid_begin;
    int64_t nvox;
    int64_t flat_base, flat_stride;  // global flat of local atom r = flat_base + r*flat_stride
    int64_t vox_base;   // global index of voxel 0 of b / best (voxel batches)
    float* best;        // nvox running max (screening units)
    CandRec* cand;      // may be null (seed pass)
    unsigned long long* cand_count;
    int64_t cand_cap;
    float delta;
    int metric;
    float* debug_scores;  // optional dense atoms x nvox output (tests)
    // Unbiased screening audit: every (voxel, atom) pair whose hash falls
    // below audit_thr (a fraction audit_thr / 2^32 of all screened pairs,
    // independent of its score) is appended here with its screening score.
    CandRec* audit;
    unsigned long long* audit_count;
    int64_t audit_cap;
    uint32_t audit_thr;
};
// The audit sample's hash: one mix of the pair's global flat and voxel.
__host__ __device__ inline uint32_t audit_hash_voxel(uint64_t v) {
    uint32_t h = static_cast<uint32_t>(v) * 0x85EBCA77u + 0x165667B1u;
    return h ^ (h >> 13);
}
__host__ __device__ inline uint32_t audit_hash_flat(uint64_t f) {
    uint32_t h = static_cast<uint32_t>(f) * 0x9E3779B1u ^ static_cast<uint32_t>(f >> 32) * 0xC2B2AE3Du;
    return h ^ (h >> 16);
}
__host__ __device__ inline uint32_t audit_mix(uint32_t ha, uint32_t hv) {
    uint32_t h = (ha ^ hv) * 0x7FEB352Du;
    return h ^ (h >> 15);
}
void launch_match(Ctx& c, const MatchParams& p);
// CUDA-core reference of the same fused screening (tests only, small sizes).
void launch_match_simt(Ctx& c, const MatchParams& p);

// K3 (rerank.cu)
void launch_prepare_queries(Ctx& c, const double* d_raw, int64_t nq, int64_t qrows, double* d_q64,
                            __half* d_qprime, int* d_bad, const uint8_t* d_unit = nullptr);
// Exact re-rank: lattice atoms re-simulated through the FP64 tables (t), or
// stored float32 dictionary entries (d_dict != nullptr, flat = row).
int64_t rerank_and_select(Ctx& c, const GridTables* t, const float* d_dict, const double* d_q64,
                          int64_t nq, int metric, const float* d_best, float delta, CandRec* d_cand,
                          int64_t ncand, mrfg_match* d_out, double* err_max = nullptr,
                          bool allow_missing = false, int64_t* stats_n32 = nullptr,
                          bool allow_fp32 = true, double* err32_max = nullptr);
// Unbiased screening audit over K2's sampled pairs (metric cc): max fp16
// screening error and (lattice) max FP32 re-screen error against the exact scores.
void audit_screen(Ctx& c, const GridTables* t, const float* d_dict, const double* d_q64, const CandRec* d_rec,
                  int64_t n, double* err16, double* err32);
// Stored float32 rows first + r*stride (r < count) -> fp16 operand (rows, zero
// padded) + inv.
void launch_dict_operand(Ctx& c, const float* d_dict, int64_t first, int64_t count, int64_t rows,
                         int64_t stride, int metric, __half* d_a, float* d_inv2);
void launch_merge(Ctx& c, const mrfg_match* d_in, int nranks, int64_t nq, mrfg_match* d_out);
void launch_cc_map(Ctx& c, const GridTables& t, const double* d_q64, int64_t first, int64_t count,
                   float* d_out);

// K5 (zoom.cu)
void run_quantify(Ctx& c, const mrfg_grid& lattice, const mrfg_zoom_config& cfg,
                  const double* d_fps, int64_t nvox, const int64_t* h_bounds /* nvox x 6 or null */,
                  const double* h_init /* nvox x 2 or null */, mrfg_quant* d_out,
                  // neighbour-seeded slice (d_fps/d_out: the raster): nrows rows of
                  // masked voxels, vox_list[row_start[r] .. row_start[r+1])
                  int64_t nrows = 0, const int64_t* h_row_start = nullptr,
                  const int64_t* h_vox_list = nullptr,
                  // the caller's dictionary payload (device, or null) and the
                  // StageLog outputs (device, nvox x MRFG_TRACE_MAX / nvox, or null)
                  const float* d_dict = nullptr, int64_t dict_entries = 0, mrfg_stage* d_trace = nullptr,
                  int* d_trace_len = nullptr,
                  // several schedules in one launch: voxel v of schedule d_vox_ib[v]
                  // (device), contexts sched[0 .. nsched) of the same length
                  const int* d_vox_ib = nullptr, Ctx* const* sched = nullptr, int nsched = 0);

}  // namespace mrfg
