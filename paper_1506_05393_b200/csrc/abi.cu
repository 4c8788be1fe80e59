// abi.cu -- the C ABI of include/mrfg.h: context, host tables and the
// orchestration of the streamed simulate-and-match scan.
#include <omp.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "mrfg_internal.cuh"

namespace mrfg {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }

template <class F>
static int guard(F&& f) {
    try {
        f();
        return MRFG_OK;
    } catch (const Error& e) {
        g_err = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "out of host memory";
        return MRFG_E_NOMEM;
    } catch (const std::exception& e) {
        g_err = e.what();
        return MRFG_E_RUNTIME;
    }
}

// ----------------------------------------------------------- host physics
// bloch.cpp:31-53 / 63-66: Rz(phi) Rx(-alpha) Rz(-phi), row-major products
// summed left to right (bloch.hpp:25-32) -- the reference's exact doubles.
static void rot(int axis, double theta, double r[9]) {
    double c = std::cos(theta), s = std::sin(theta);
    const double x[9] = {1, 0, 0, 0, c, -s, 0, s, c};
    const double z[9] = {c, -s, 0, s, c, 0, 0, 0, 1};
    std::memcpy(r, axis == 0 ? x : z, sizeof(x));
}
static void mul3(const double* a, const double* b, double* r) {
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            r[3 * i + j] = a[3 * i] * b[j] + a[3 * i + 1] * b[3 + j] + a[3 * i + 2] * b[6 + j];
}
void host_rf_matrix(double alpha, double phi, double out[9]) {
    double a[9], b[9], c[9], ab[9];
    rot(2, phi, a);
    rot(0, -alpha, b);
    rot(2, -phi, c);
    mul3(a, b, ab);
    mul3(ab, c, out);
}

static bool same_axis(const mrfg_axis& a, const mrfg_axis& b, const std::vector<double>& bv) {
    if (a.min != b.min || a.step != b.step || a.count != b.count || (a.values == nullptr) != bv.empty())
        return false;
    return a.values == nullptr || std::memcmp(a.values, bv.data(), sizeof(double) * a.count) == 0;
}
static bool same_grid(const mrfg_grid& a, const GridTables& t) {
    return same_axis(a.t1_ms, t.grid.t1_ms, t.v1) && same_axis(a.t2_ms, t.grid.t2_ms, t.v2) &&
           a.df_hz.min == t.grid.df_hz.min && a.df_hz.step == t.grid.df_hz.step &&
           a.df_hz.count == t.grid.df_hz.count && a.df_hz.values == nullptr;
}

static void check_grid(const mrfg_grid& g) {
    const mrfg_axis* ax[3] = {&g.t1_ms, &g.t2_ms, &g.df_hz};
    for (auto* a : ax) MRFG_REQUIRE(a->count > 0, MRFG_E_INVALID, "grid: empty axis");
    MRFG_REQUIRE(g.df_hz.values == nullptr, MRFG_E_INVALID,
                 "grid: explicit axis values are supported on the T1 and T2 axes only");
    for (const mrfg_axis* a : {&g.t1_ms, &g.t2_ms}) {
        if (a->values) {
            for (int64_t i = 0; i < a->count; ++i)
                MRFG_REQUIRE(a->values[i] > 0 && std::isfinite(a->values[i]), MRFG_E_INVALID,
                             "simulate: T1 and T2 must be positive");
        } else {
            MRFG_REQUIRE(a->min > 0 && a->min + (a->count - 1) * a->step > 0, MRFG_E_INVALID,
                         "simulate: T1 and T2 must be positive");
        }
    }
}

// Per-axis transcendental tables: host libm, reference operand order
// (bloch.cpp:17-21).  Cached per context for the last grid.
const GridTables& ensure_tables(Ctx& c, const mrfg_grid& g, bool /*need64*/) {
    if (c.tab.valid && same_grid(g, c.tab)) return c.tab;
    check_grid(g);
    c.tab.sub_r = 0;  // the subspace bases belong to the grid
    const int64_t n = c.n, n1 = g.t1_ms.count, n2 = g.t2_ms.count, nd = g.df_hz.count;
    std::vector<double> e1(n * n1 * 2), e2(n * n2 * 2), ph(n * nd * 4);
    std::vector<float> e1f(n * n1 * 4), e2f(n * n2 * 2), phf(n * nd * 4);
    const double kTwoPi = 6.283185307179586476925286766559;
    // Layout: parameter-major, [i][j] (one lattice value's n steps contiguous),
    // so a walker over j streams memory (K3/K4/K5 gather scattered points).
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n1; ++i) {
        const double inv = 1.0 / (axis_value(g.t1_ms, i) * 1e-3);
        for (int64_t j = 0; j < n; ++j) {
            const double a = std::exp(-c.te_s[j] * inv), b = std::exp(-c.rest_s[j] * inv);
            e1[(i * n + j) * 2] = a;
            e1[(i * n + j) * 2 + 1] = b;
            float* f = &e1f[(i * n + j) * 4];
            f[0] = static_cast<float>(a);
            f[1] = static_cast<float>(1.0 - a);
            f[2] = static_cast<float>(b);
            f[3] = static_cast<float>(1.0 - b);
        }
    }
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n2; ++i) {
        const double inv = 1.0 / (axis_value(g.t2_ms, i) * 1e-3);
        for (int64_t j = 0; j < n; ++j) {
            const double a = std::exp(-c.te_s[j] * inv), b = std::exp(-c.rest_s[j] * inv);
            e2[(i * n + j) * 2] = a;
            e2[(i * n + j) * 2 + 1] = b;
            e2f[(i * n + j) * 2] = static_cast<float>(a);
            e2f[(i * n + j) * 2 + 1] = static_cast<float>(b);
        }
    }
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < nd; ++i) {
        const double df = g.df_hz.min + static_cast<double>(i) * g.df_hz.step;
        for (int64_t j = 0; j < n; ++j) {
            const double at = kTwoPi * df * c.te_s[j], ar = kTwoPi * df * c.rest_s[j];
            double* p = &ph[(i * n + j) * 4];
            p[0] = std::cos(at);
            p[1] = std::sin(at);
            p[2] = std::cos(ar);
            p[3] = std::sin(ar);
            float* f = &phf[(i * n + j) * 4];
            for (int k = 0; k < 4; ++k) f[k] = static_cast<float>(p[k]);
        }
    }
    std::vector<StepU> su(n);
    for (int64_t j = 0; j < n; ++j) {
        StepU& u = su[j];
        for (int k = 0; k < 9; ++k) u.r[k] = static_cast<float>(c.rf64[9 * j + k]);
        u.te = static_cast<float>(c.te_s[j]);
        u.rest = static_cast<float>(c.rest_s[j]);
        const double at = kTwoPi * g.df_hz.step * c.te_s[j], ar = kTwoPi * g.df_hz.step * c.rest_s[j];
        u.wtc = static_cast<float>(std::cos(at));
        u.wts = static_cast<float>(std::sin(at));
        u.wrc = static_cast<float>(std::cos(ar));
        u.wrs = static_cast<float>(std::sin(ar));
        u.pad = 0.f;
    }
    GridTables& t = c.tab;
    t.valid = false;
    // 1 KB of zeroed tail padding: table walkers may load a few steps past the
    // last row's end (look-ahead of the final block; the values are unused)
    auto up = [&](DevBuf& b, const void* src, size_t bytes) {
        b.ensure(bytes + 1024);
        MRFG_CUDA(cudaMemsetAsync(static_cast<char*>(b.p) + bytes, 0, 1024, c.stream));
        MRFG_CUDA(cudaMemcpyAsync(b.p, src, bytes, cudaMemcpyHostToDevice, c.stream));
    };
    up(t.e1d, e1.data(), e1.size() * 8);
    up(t.e2d, e2.data(), e2.size() * 8);
    up(t.phd, ph.data(), ph.size() * 8);
    up(t.e1f, e1f.data(), e1f.size() * 4);
    up(t.e2f, e2f.data(), e2f.size() * 4);
    up(t.phf, phf.data(), phf.size() * 4);
    up(t.stepu, su.data(), su.size() * sizeof(StepU));
    // x-axis schedules: the K5 screening step rows, 2 x float4 per step:
    // (r4, r5, r7, r8) -- the RF entries that are not 0 or 1 -- and the
    // one-df-step phasors (wtc, wts, wrc, wrs)
    if (c.rf_xaxis) {
        std::vector<float> sx(8 * n);
        for (int64_t j = 0; j < n; ++j) {
            const StepU& u = su[j];
            const float v[8] = {u.r[4], u.r[5], u.r[7], u.r[8], u.wtc, u.wts, u.wrc, u.wrs};
            std::memcpy(&sx[8 * j], v, sizeof v);
        }
        up(t.stepx, sx.data(), sx.size() * 4);
    }
    // K1 row producers: log2(e)/T per lattice index (ex2 arguments), FP64 -> FP32
    std::vector<float> kt(n1 + n2);
    for (int64_t i = 0; i < n1; ++i) kt[i] = static_cast<float>(1.4426950408889634 / (axis_value(g.t1_ms, i) * 1e-3));
    for (int64_t i = 0; i < n2; ++i)
        kt[n1 + i] = static_cast<float>(1.4426950408889634 / (axis_value(g.t2_ms, i) * 1e-3));
    up(t.kt, kt.data(), kt.size() * sizeof(float));
    MRFG_CUDA(cudaStreamSynchronize(c.stream));
    t.grid = g;
    t.v1.assign(g.t1_ms.values ? g.t1_ms.values : nullptr, g.t1_ms.values ? g.t1_ms.values + n1 : nullptr);
    t.v2.assign(g.t2_ms.values ? g.t2_ms.values : nullptr, g.t2_ms.values ? g.t2_ms.values + n2 : nullptr);
    t.grid.t1_ms.values = t.v1.empty() ? nullptr : t.v1.data();  // owned copies, not the caller's
    t.grid.t2_ms.values = t.v2.empty() ? nullptr : t.v2.data();
    t.valid = true;
    return t;
}

// dst[k] = src[idx[k]] for rows of `row` doubles (K5 voxel groups)
__global__ void k_gather_rows(const double* __restrict__ src, const int64_t* __restrict__ idx, int64_t row,
                              double* __restrict__ dst) {
    const double* s = src + idx[blockIdx.x] * row;
    double* d = dst + static_cast<int64_t>(blockIdx.x) * row;
    for (int64_t t = threadIdx.x; t < row; t += blockDim.x) d[t] = s[t];
}

__global__ void k_fill(float* p, int64_t n, float v) {
    int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < n) p[i] = v;
}

// Screening maxima from an earlier scan's exact CC scores, rounded down
// (a kept atom then still satisfies s >= e - eps >= floor - delta).
__global__ void k_floor(const mrfg_match* __restrict__ m, int64_t nq, float* __restrict__ best) {
    const int64_t v = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (v >= nq || m[v].flat < 0) return;
    const float f = __double2float_rd(m[v].score);
    if (f > best[v]) best[v] = f;
}

static void fill(Ctx& c, float* p, int64_t n, float v) {
    if (n <= 0) return;
    k_fill<<<(n + 255) / 256, 256, 0, c.stream>>>(p, n, v);
    MRFG_CUDA(cudaGetLastError());
}

struct EventTimer {
    cudaStream_t s;
    std::vector<cudaEvent_t> evs;
    explicit EventTimer(cudaStream_t st) : s(st) {}
    ~EventTimer() {
        for (auto e : evs) cudaEventDestroy(e);
    }
    int mark() {
        cudaEvent_t e;
        MRFG_CUDA(cudaEventCreate(&e));
        MRFG_CUDA(cudaEventRecord(e, s));
        evs.push_back(e);
        return static_cast<int>(evs.size()) - 1;
    }
    double ms(int a, int b) {
        float m = 0;
        MRFG_CUDA(cudaEventElapsedTime(&m, evs[a], evs[b]));
        return m;
    }
};

// The streamed brute-force scan on device-resident queries.  Atoms come from
// the lattice (grid != nullptr: K1 simulates them chunk by chunk) or from a
// stored float32 dictionary (d_dict: converted to the fp16 operand per chunk).
// Returns false (nothing written) when the unbiased audit finds a screening
// error above delta/2: the caller repeats the scan with a wider margin.
static bool scan_dev_once(Ctx& c, const mrfg_grid* grid, const float* d_dict, int64_t dict_atoms,
                          int64_t fb, int64_t fe, const double* d_raw, int64_t nq, int metric,
                          const mrfg_scan_opts* o, double delta, mrfg_match* d_out, mrfg_scan_stats* st,
                          float* seed_out = nullptr) {
    MRFG_REQUIRE(nq > 0, MRFG_E_INVALID, "scan_grid: no queries");  // dictionary.cpp:260
    MRFG_REQUIRE(metric == MRFG_METRIC_CC || metric == MRFG_METRIC_EUCLIDEAN, MRFG_E_INVALID,
                 "scan_grid: unknown metric");
    const int64_t total = grid ? grid_total(*grid) : dict_atoms;
    if (fb == 0 && fe == 0) fe = total;
    MRFG_REQUIRE(0 <= fb && fb < fe && fe <= total, MRFG_E_INVALID, "scan_grid: bad flat range");
    const GridTables* tp = grid ? &ensure_tables(c, *grid, true) : nullptr;
    // K1 tiles whole lattice rows (ndf atoms): a chunk is crows rows.  A stored
    // dictionary is chunked in flat order directly (ndf = 1).
    const int64_t ndf = grid ? grid->df_hz.count : 1;
    // Default lattice chunk: ONE full wave of the K1 producer (2 resident
    // blocks of 256 threads per SM, 4 atoms per thread, whole rows) -- the
    // 524,288-atom chunk ran K1 as 1.73 waves (config 2: 128 vs 118 ms per step)
    int64_t chunk = (o && o->chunk_atoms > 0) ? o->chunk_atoms : 524288;
    if (grid && !(o && o->chunk_atoms > 0)) {
        const int64_t threads_per_row = (ndf + 3) / 4;
        chunk = std::max<int64_t>(1, int64_t(c.num_sms) * 2 * 256 / threads_per_row) * ndf;
    }
    const int64_t crows = std::max<int64_t>(1, chunk / ndf);
    // Per-off-resonance subspace screening (subspace.cu): CC scans of whole
    // lattice rows with the atom-pair producer.  Default: complex rank 48 when
    // the range is large enough to pay for the projections (>= 4e6 atoms and
    // >= 4,096 lattice rows: also the atom shards of an 8-GPU config-2 scan); MRFG_SUBSPACE=0 turns it off, =r forces rank r.
    int sub_r = 0;
    const bool sub_ok = grid && metric == MRFG_METRIC_CC && fb % ndf == 0 && fe % ndf == 0 && bloch_dfquad_ok(c) &&
                        !seed_out && (fe - fb) / ndf >= 256 && grid->t1_ms.count * grid->t2_ms.count >= 640;
    if (const char* e = std::getenv("MRFG_SUBSPACE"))
        sub_r = std::atoi(e);
    else if (sub_ok && fe - fb >= 4000000 && (fe - fb) / ndf >= 4096)
        sub_r = 48;  // held-out residual 5e-4 on config 2 (rank 32: 3e-3, a margin of 8.6e-3 and an overflow pass)
    const bool sub_auto = std::getenv("MRFG_SUBSPACE") == nullptr;
    if (sub_r > 0) sub_r = subspace_rank(sub_r);
    if (!sub_ok) sub_r = 0;
    // a lattice whose slabs do not compress (held-out residual above 2e-3 at the
    // default rank: the margin and the candidate lists would grow) keeps the
    // full-length screening
    if (sub_r && sub_auto) {
        ensure_subspace(c, *tp, sub_r);
        if (tp->sub_rho_held > 2e-3) sub_r = 0;
    }
    const int sub_nw = sub_r ? subspace_cols(sub_r) : 0, sub_kc = sub_r ? subspace_pitch(sub_r) : 0;
    const __half* sub_w = sub_r ? ensure_subspace(c, *tp, sub_r) : nullptr;  // cached per grid
    // the truncation adds at most |q_perp| |a_perp| / |a| <= rho to the screening
    // error: the default margin grows by twice the held-out residual
    if (sub_r && !(o && o->delta > 0)) delta += 2.0 * tp->sub_rho_held;
    int64_t cap = (o && o->cand_capacity > 0) ? o->cand_capacity : (int64_t(1) << (sub_r ? 26 : 25));
    const int64_t seed_atoms = (o && o->seed_atoms > 0) ? o->seed_atoms : 16384;
    const int64_t n = c.n, kp = k_pad_of(n), qrows = round_up(2 * nq, 256);
    const int64_t range = fe - fb;

    EventTimer tm(c.stream);
    const int e_start = tm.mark();
    c.q64.ensure(sizeof(double) * 2 * n * nq);
    c.qprime.ensure(sizeof(__half) * qrows * kp);
    c.best.ensure(sizeof(float) * nq + 64);
    int* d_bad = reinterpret_cast<int*>(c.best.as<char>() + sizeof(float) * nq);
    MRFG_CUDA(cudaMemsetAsync(d_bad, 0, sizeof(int), c.stream));
    const uint8_t* d_unit = nullptr;
    if (o && o->unit_queries) {  // Fingerprint::unit_norm flags (host) -> device
        c.misc2.ensure(64 + nq);
        d_unit = c.misc2.as<uint8_t>() + 64;
        MRFG_CUDA(cudaMemcpyAsync(const_cast<uint8_t*>(d_unit), o->unit_queries, nq, cudaMemcpyHostToDevice,
                                  c.stream));
    }
    launch_prepare_queries(c, d_raw, nq, qrows, c.q64.as<double>(), c.qprime.as<__half>(), d_bad, d_unit);
    int h_bad = 0;
    MRFG_CUDA(cudaMemcpyAsync(&h_bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    MRFG_CUDA(cudaStreamSynchronize(c.stream));
    MRFG_REQUIRE(!h_bad, MRFG_E_INVALID, "normalize: zero fingerprint");
    float* best = c.best.as<float>();
    fill(c, best, nq, -3.0f);
    const bool floored = o && o->floor_matches && metric == MRFG_METRIC_CC;
    if (floored) {  // earlier scans' exact scores (rounded down) seed the maxima
        k_floor<<<static_cast<unsigned>((nq + 255) / 256), 256, 0, c.stream>>>(o->floor_matches, nq, best);
        MRFG_CUDA(cudaGetLastError());
    }

    const int64_t arows = round_up(std::min(crows * ndf, round_up(range, ndf) + ndf), 256);  // pair tiles
    c.atoms_a.ensure(sizeof(__half) * 2 * arows * kp);  // double-buffered operand
    c.inv2.ensure(sizeof(float) * 2 * arows);
    c.ensure_aux();
    c.cand_count.ensure(64);
    auto* d_count = c.cand_count.as<unsigned long long>();

    MatchParams mp{};
    mp.a = c.atoms_a.as<__half>();
    mp.inv2 = c.inv2.as<float>();
    mp.b = c.qprime.as<__half>();
    mp.q_rows = qrows;
    mp.k_pad = kp;
    mp.nvox = nq;
    mp.best = best;
    mp.cand_count = d_count;
    mp.delta = static_cast<float>(delta);
    mp.metric = metric;

    double gemm_ms = 0, bloch_ms = 0, project_ms = 0, sub_rho2 = 0;
    int64_t gemm_launches = 0, chunks = 0;
    // Voxel batch: query rows of <= ~40 MB (L2 is 126 MB).  Measured on config 3
    // (stored dictionary): the GEMM runs at 1,255 / 1,039 / 890 TFLOP/s with
    // 33 MB / 134 MB / 2.1 GB of query rows.  MRFG_VOX_BATCH overrides (0 = all).
    int64_t vox_batch = std::max<int64_t>(128, (int64_t(40) << 20) / (4 * kp) / 128 * 128);
    if (const char* e = std::getenv("MRFG_VOX_BATCH")) {
        const int64_t v = std::atoll(e);
        vox_batch = v > 0 ? std::max<int64_t>(128, v / 128 * 128) : nq;
    }
    if (vox_batch >= nq) vox_batch = nq;
    // Seed pass: a strided sample of the range raises the running maxima
    // before the stream starts (no candidates are recorded).
    {
        int64_t stride = std::max<int64_t>(1, range / seed_atoms);
        int64_t cnt = (range + stride - 1) / stride;
        int64_t rows = round_up(std::min(cnt, arows), 256);
        int a0 = tm.mark();
        if (tp)
            launch_bloch_operand(c, *tp, fb, stride, fe, rows, metric, c.atoms_a.as<__half>(),
                                 c.inv2.as<float>());
        else
            launch_dict_operand(c, d_dict, fb, std::min(cnt, rows), rows, stride, metric,
                                c.atoms_a.as<__half>(), c.inv2.as<float>());
        int a1 = tm.mark();
        mp.atoms = rows;
        mp.valid_atoms = std::min(cnt, rows);
        mp.flat_base = fb;
        mp.flat_stride = stride;
        mp.cand = nullptr;
        mp.cand_cap = 0;
        launch_match(c, mp);
        int a2 = tm.mark();
        MRFG_CUDA(cudaStreamSynchronize(c.stream));
        bloch_ms += tm.ms(a0, a1);
        gemm_ms += tm.ms(a1, a2);
        ++gemm_launches;
    }
    if (seed_out) {  // seed maxima only (mrfg_scan_seed_dev)
        MRFG_CUDA(cudaMemcpyAsync(seed_out, best, sizeof(float) * nq, cudaMemcpyDeviceToDevice, c.stream));
        if (st) {
            st->atoms = range;
            st->voxels = nq;
            st->bloch_ms = bloch_ms;
            st->gemm_ms = gemm_ms;
            st->gemm_launches = gemm_launches;
        }
        return true;
    }
    // Unbiased audit: a hash sample of ALL screened pairs, about audit_target
    // of them per scan (MRFG_AUDIT=0 disables, =k sets the target).
    int64_t audit_target = 16384;
    if (const char* e = std::getenv("MRFG_AUDIT")) audit_target = std::atoll(e);
    const int64_t audit_cap = 4 * std::max<int64_t>(audit_target, 1024);
    const bool audit_on = audit_target > 0 && metric == MRFG_METRIC_CC;
    if (audit_on) {
        c.audit.ensure(sizeof(CandRec) * audit_cap + 64);
        const double pairs = static_cast<double>(nq) * static_cast<double>(range);
        const double frac = std::min(1.0, static_cast<double>(audit_target) / pairs);
        mp.audit = c.audit.as<CandRec>();
        mp.audit_count = reinterpret_cast<unsigned long long*>(c.audit.as<char>() + sizeof(CandRec) * audit_cap);
        mp.audit_cap = audit_cap;
        mp.audit_thr = static_cast<uint32_t>(std::min(4294967295.0, std::floor(frac * 4294967296.0)));
        if (mp.audit_thr == 0) mp.audit_thr = 1;
    }
    int64_t overflow_passes = 0;
    unsigned long long ncand = 0;
    for (int pass = 0; pass < 2; ++pass) {
        c.cand.ensure(sizeof(CandRec) * cap);
        MRFG_CUDA(cudaMemsetAsync(d_count, 0, sizeof(unsigned long long), c.stream));
        if (audit_on) MRFG_CUDA(cudaMemsetAsync(mp.audit_count, 0, sizeof(unsigned long long), c.stream));
        mp.cand = c.cand.as<CandRec>();
        mp.cand_cap = cap;
        // Two operand buffers: with MRFG_OVERLAP=1 the producer (K1 or the
        // dictionary conversion) fills chunk i+1 on the aux stream while K2
        // consumes chunk i (the persistent GEMM leaves room for one producer CTA
        // per SM).  Measured on B200: K2 runs under sw_power_cap, so concurrent
        // CUDA-core work lowers the SM clock and the GEMM loses what K1 gains
        // (3.05 s vs 2.99 s per config-2 slice with the scalar K1; with the
        // packed-pair K1: 2.900 vs 2.940 s, but K1's own duration stretches to
        // 355 ms, so the Bloch rate is no longer measurable per kernel); the
        // default is one stream.
        static const bool overlap = [] {
            const char* e = std::getenv("MRFG_OVERLAP");
            return e && e[0] == '1';
        }();
        const cudaStream_t S = c.stream, A = overlap ? c.aux : c.stream;
        EventTimer ta(A);
        std::vector<int> pm, gm, pj;
        MRFG_CUDA(cudaEventRecord(c.ev[0], S));
        MRFG_CUDA(cudaStreamWaitEvent(A, c.ev[0], 0));
        int64_t i = 0;
        if (sub_r) {
            // df-major: K1 produces the four off-resonance slabs of a quad (all
            // lattice rows each), every slab is projected onto its basis and
            // screened by K2 in 2r dimensions against that df's query coefficients
            const int64_t row_lo = fb / ndf, nrows = (fe - fb) / ndf, pitch = round_up(nrows, 256);
            c.atoms_a.ensure(sizeof(__half) * 4 * pitch * kp);
            c.inv2.ensure(sizeof(float) * 4 * pitch);
            c.sub_c.ensure(sizeof(__half) * 4 * pitch * sub_kc);
            c.sub_q.ensure(sizeof(__half) * ndf * qrows * sub_kc);
            c.sub_rho.ensure(64);
            __half* abuf = c.atoms_a.as<__half>();
            float* ibuf = c.inv2.as<float>();
            __half* cbuf = c.sub_c.as<__half>();
            __half* qbuf = c.sub_q.as<__half>();
            auto* rho = c.sub_rho.as<unsigned int>();
            MRFG_CUDA(cudaMemsetAsync(abuf, 0, sizeof(__half) * 4 * pitch * kp, S));
            MRFG_CUDA(cudaMemsetAsync(ibuf, 0, sizeof(float) * 4 * pitch, S));
            MRFG_CUDA(cudaMemsetAsync(cbuf, 0, sizeof(__half) * 4 * pitch * sub_kc, S));
            MRFG_CUDA(cudaMemsetAsync(qbuf, 0, sizeof(__half) * ndf * qrows * sub_kc, S));
            MRFG_CUDA(cudaMemsetAsync(rho, 0, sizeof(unsigned int), S));
            pj.push_back(tm.mark());
            // the query coefficients of every df in one launch (grid.y = df)
            launch_project(c, c.qprime.as<__half>(), qrows, kp, sub_w, sub_nw, qbuf, sub_kc, nullptr, 0, nullptr,
                           static_cast<int>(ndf), sub_nw * kp, qrows * sub_kc);
            pj.push_back(tm.mark());
            for (int64_t q0 = 0; q0 < ndf; q0 += 4, ++i) {
                pm.push_back(tm.mark());
                launch_bloch_dfquad(c, *tp, static_cast<int>(q0), row_lo, nrows, pitch, metric, abuf, ibuf);
                pm.push_back(tm.mark());
                for (int64_t m = 0; m < 4 && q0 + m < ndf; ++m) {
                    const int64_t d = q0 + m;
                    pj.push_back(tm.mark());
                    launch_project(c, abuf + m * pitch * kp, pitch, kp, sub_w + d * sub_nw * kp, sub_nw,
                                   cbuf + m * pitch * sub_kc, sub_kc, ibuf + m * pitch, nrows, rho);
                    pj.push_back(tm.mark());
                    mp.a = cbuf + m * pitch * sub_kc;
                    mp.inv2 = ibuf + m * pitch;
                    mp.atoms = pitch;
                    mp.k_pad = sub_kc;
                    mp.k_valid = sub_nw;
                    mp.valid_begin = 0;
                    mp.valid_atoms = nrows;
                    mp.flat_base = row_lo * ndf + d;
                    mp.flat_stride = ndf;
                    mp.b = qbuf + d * qrows * sub_kc;
                    mp.q_rows = qrows;
                    mp.nvox = nq;
                    mp.best = best;
                    mp.vox_base = 0;
                    gm.push_back(tm.mark());
                    launch_match(c, mp);
                    gm.push_back(tm.mark());
                }
                ++chunks;
            }
            mp.k_pad = kp;
            mp.k_valid = 0;
            unsigned int rbits = 0;
            MRFG_CUDA(cudaMemcpyAsync(&rbits, rho, sizeof rbits, cudaMemcpyDeviceToHost, S));
            MRFG_CUDA(cudaStreamSynchronize(S));
            float r2;
            std::memcpy(&r2, &rbits, sizeof r2);
            sub_rho2 = r2;
            for (size_t k = 0; k + 1 < pj.size(); k += 2) project_ms += tm.ms(pj[k], pj[k + 1]);
            // pm holds tm marks here (one stream)
            for (size_t k = 0; k + 1 < pm.size(); k += 2) bloch_ms += tm.ms(pm[k], pm[k + 1]);
            pm.clear();
        }
        for (int64_t r0 = fb / ndf; !sub_r && r0 * ndf < fe; r0 += crows, ++i) {
            const int64_t vb = std::max(fb, r0 * ndf), ve = std::min(fe, (r0 + crows) * ndf);
            const int64_t base = r0 * ndf;
            const int64_t rows = round_up(ve - base, 256);
            const int b = static_cast<int>(i & 1);
            __half* abuf = c.atoms_a.as<__half>() + b * arows * kp;
            float* ibuf = c.inv2.as<float>() + b * arows;
            if (i >= 2) MRFG_CUDA(cudaStreamWaitEvent(A, c.ev[2 + b], 0));  // GEMM(i-2) released b
            pm.push_back(ta.mark());
            c.stream = A;
            if (tp)
                launch_bloch_rows(c, *tp, vb, ve, metric, 0, rows, abuf, nullptr, ibuf);
            else  // rows [vb-base, ve-base) hold the entries
                launch_dict_operand(c, d_dict, base, ve - base, rows, 1, metric, abuf, ibuf);
            c.stream = S;
            pm.push_back(ta.mark());
            MRFG_CUDA(cudaEventRecord(c.ev[4 + b], A));
            MRFG_CUDA(cudaStreamWaitEvent(S, c.ev[4 + b], 0));
            mp.a = abuf;
            mp.inv2 = ibuf;
            mp.atoms = rows;
            mp.valid_begin = vb - base;
            mp.valid_atoms = ve - base;
            mp.flat_base = base;
            mp.flat_stride = 1;
            // voxel batches whose query rows stay L2-resident (the chunk's atom
            // operand is re-read from HBM per batch instead of every query
            // tile per atom tile)
            for (int64_t v0 = 0; v0 < nq; v0 += vox_batch) {
                const int64_t nvb = std::min(vox_batch, nq - v0);
                mp.b = c.qprime.as<__half>() + 2 * v0 * kp;
                mp.q_rows = round_up(2 * nvb, 256);
                mp.nvox = nvb;
                mp.best = best + v0;
                mp.vox_base = v0;
                gm.push_back(tm.mark());
                launch_match(c, mp);
                gm.push_back(tm.mark());
            }
            MRFG_CUDA(cudaEventRecord(c.ev[2 + b], S));
            ++chunks;
        }
        MRFG_CUDA(cudaMemcpyAsync(&ncand, d_count, sizeof ncand, cudaMemcpyDeviceToHost, S));
        MRFG_CUDA(cudaStreamSynchronize(S));
        MRFG_CUDA(cudaStreamSynchronize(A));
        for (size_t k = 0; k + 1 < pm.size(); k += 2) bloch_ms += ta.ms(pm[k], pm[k + 1]);
        for (size_t k = 0; k + 1 < gm.size(); k += 2) {
            gemm_ms += tm.ms(gm[k], gm[k + 1]);
            ++gemm_launches;
        }
        mp.a = c.atoms_a.as<__half>();
        mp.inv2 = c.inv2.as<float>();
        mp.b = c.qprime.as<__half>();
        mp.q_rows = qrows;
        mp.nvox = nq;
        mp.best = best;
        mp.vox_base = 0;
        if (ncand <= static_cast<unsigned long long>(cap)) break;
        // Overflow: the running maxima are now final, so a second pass records
        // a subset of the first pass's candidates; size the buffer for all.
        MRFG_REQUIRE(pass == 0, MRFG_E_RUNTIME, "scan: candidate buffer overflow");
        cap = static_cast<int64_t>(ncand);
        ++overflow_passes;
    }
    // the audit: exact scores of the sampled pairs (fp16 screen and FP32
    // re-screen errors); a margin the sample contradicts is widened by a rescan
    double a16 = 0, a32 = 0;
    int64_t nsamp = 0;
    int ra0 = tm.mark();
    if (audit_on) {
        unsigned long long h = 0;
        MRFG_CUDA(cudaMemcpyAsync(&h, mp.audit_count, sizeof h, cudaMemcpyDeviceToHost, c.stream));
        MRFG_CUDA(cudaStreamSynchronize(c.stream));
        nsamp = static_cast<int64_t>(std::min<unsigned long long>(h, static_cast<unsigned long long>(audit_cap)));
        audit_screen(c, tp, d_dict, c.q64.as<double>(), mp.audit, nsamp, &a16, &a32);
        if (a16 > 0.5 * delta) {
            if (st) st->screen_err_audit_max = a16;
            return false;
        }
    }
    int ra1 = tm.mark();
    double err_max = 0, err32 = 0;
    int r0 = tm.mark();
    int64_t n32 = 0;
    // the FP32 stage certifies with margin kRescreenEps = 1e-5: needs its
    // audited error below half of it, else every candidate is re-ranked in FP64
    const bool fp32_ok = !audit_on || a32 <= 0.5e-5;
    int64_t nsel = rerank_and_select(c, tp, d_dict, c.q64.as<double>(), nq, metric, best,
                                     static_cast<float>(delta), c.cand.as<CandRec>(),
                                     static_cast<int64_t>(ncand), d_out, &err_max, floored, &n32, fp32_ok,
                                     &err32);
    int r1 = tm.mark();
    MRFG_CUDA(cudaStreamSynchronize(c.stream));
    if (st) {
        st->atoms = range;
        st->voxels = nq;
        st->chunks = chunks;
        st->candidates = static_cast<int64_t>(ncand);
        st->reranked = nsel;
        st->overflow_passes = overflow_passes;
        st->bloch_ms = bloch_ms;
        st->gemm_ms = gemm_ms;
        st->rerank_ms = tm.ms(r0, r1);
        st->total_ms = tm.ms(e_start, r1);
        st->gemm_launches = gemm_launches;
        st->gemm_kernel_ms_avg = gemm_launches ? gemm_ms / gemm_launches : 0;
        st->screen_err_max = err_max;
        st->rescreened32 = n32;
        st->screen_err_audit_max = a16;
        st->rescreen_err_audit_max = a32;
        st->audit_samples = nsamp;
        st->delta_used = delta;
        st->rescreen_err_max = err32;
        st->chunk_atoms = sub_r ? (fe - fb) / ndf : crows * ndf;
        st->project_ms = project_ms;
        st->subspace_rank = sub_r;
        st->subspace_residual_max = sub_r ? tp->sub_rho_held : 0.0;
        st->subspace_residual_device = sub_rho2 > 0 ? std::sqrt(sub_rho2) : 0.0;
        st->rerank_ms += tm.ms(ra0, ra1);
    }
    return true;
}

// Default screening margin: twice the analytic bound on |fp16 screen CC -
// exact CC| (2u + u^2 + FP32 accumulation over 2N terms + the
// K1 FP32 error, u = 2^-11).
constexpr double kDefaultDelta = 2.5e-3;

static void scan_dev(Ctx& c, const mrfg_grid* grid, const float* d_dict, int64_t dict_atoms, int64_t fb,
                     int64_t fe, const double* d_raw, int64_t nq, int metric, const mrfg_scan_opts* o,
                     mrfg_match* d_out, mrfg_scan_stats* st) {
    double delta = (o && o->delta > 0) ? o->delta : kDefaultDelta;
    for (int64_t rescans = 0;; ++rescans) {
        mrfg_scan_stats tmp{};
        mrfg_scan_stats* sp = st ? st : &tmp;
        if (scan_dev_once(c, grid, d_dict, dict_atoms, fb, fe, d_raw, nq, metric, o, delta, d_out, sp)) {
            sp->rescans = rescans;
            return;
        }
        MRFG_REQUIRE(rescans < 3, MRFG_E_RUNTIME, "scan: screening audit failed after widening the margin");
        delta = std::max(2 * delta, 4 * sp->screen_err_audit_max);
    }
}

}  // namespace mrfg

using namespace mrfg;

struct mrfg_ctx {
    Ctx c;
};

extern "C" {

const char* mrfg_last_error(void) { return g_err.c_str(); }
const char* mrfg_version(void) { return "mrfg 0.1 (sm_100a)"; }

void mrfg_zoom_config_default(mrfg_zoom_config* c) {
    std::memset(c, 0, sizeof(*c));
    c->metric = MRFG_METRIC_CC;
    c->final_metric = MRFG_METRIC_CC;
    c->omega_hz = 70;
    c->df_coarse_hz = 60;
    c->df_refine_hz = 3;
    c->df_window_hz = 150;
    c->plateau_eps = 1e-7;
    c->heavy_noise_cc = 0.1;
    c->fallback_coarse_hz = 30;
    c->fallback_window_hz = 300;
    c->n2d = 2;
    c->t1t2_2d_steps_ms[0] = 200;
    c->t1t2_2d_steps_ms[1] = 100;
    c->n1d = 4;
    c->t1t2_1d_steps_ms[0] = 100;
    c->t1t2_1d_steps_ms[1] = 50;
    c->t1t2_1d_steps_ms[2] = 20;
    c->t1t2_1d_steps_ms[3] = 10;
    c->final_2d_step_ms = 1;
    c->init_t1_ms = 1000;
    c->init_t2_ms = 500;
    c->prior_window_t1_ms = 3000;
    c->prior_window_t2_ms = 800;
    c->prior_window_df_hz = 150;
}

int mrfg_create(const double* flip_deg, const double* phase_deg, const double* tr_ms,
                const double* te_ms, int64_t n, int device, mrfg_ctx** out) {
    return guard([&] {
        MRFG_REQUIRE(out != nullptr, MRFG_E_INVALID, "mrfg_create: null output");
        MRFG_REQUIRE(n > 0, MRFG_E_INVALID, "generate: empty schedule");
        for (int64_t i = 0; i < n; ++i)
            MRFG_REQUIRE(te_ms[i] >= 0 && te_ms[i] <= tr_ms[i], MRFG_E_INVALID,
                         "BlochSimulator: schedule needs 0 <= te <= tr");
        int ndev = 0;
        MRFG_CUDA(cudaGetDeviceCount(&ndev));
        MRFG_REQUIRE(device >= 0 && device < ndev, MRFG_E_CUDA, "mrfg_create: no such CUDA device");
        cudaDeviceProp prop;
        MRFG_CUDA(cudaGetDeviceProperties(&prop, device));
        MRFG_REQUIRE(prop.major == 10, MRFG_E_CUDA,
                     std::string("mrfg requires an sm_100 (Blackwell B200) device, found ") + prop.name);
        auto* h = new mrfg_ctx();
        Ctx& c = h->c;
        c.device = device;
        MRFG_CUDA(cudaSetDevice(device));
        MRFG_CUDA(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
        c.own_stream = true;
        c.num_sms = prop.multiProcessorCount;
        c.n = n;
        c.flip_deg.assign(flip_deg, flip_deg + n);
        c.phase_deg.assign(phase_deg, phase_deg + n);
        c.tr_ms.assign(tr_ms, tr_ms + n);
        c.te_ms.assign(te_ms, te_ms + n);
        c.rf64.resize(9 * n);
        c.te_s.resize(n);
        c.rest_s.resize(n);
        std::vector<float> rf32(12 * n, 0.f);
        for (int64_t i = 0; i < n; ++i) {
            // ScheduleEntry accessors (sequence.hpp:20-23), bloch.cpp:101-103
            host_rf_matrix(flip_deg[i] * 0.017453292519943295, phase_deg[i] * 0.017453292519943295,
                           &c.rf64[9 * i]);
            c.te_s[i] = te_ms[i] * 1e-3;
            c.rest_s[i] = tr_ms[i] * 1e-3 - te_ms[i] * 1e-3;
            for (int k = 0; k < 9; ++k) rf32[12 * i + k] = static_cast<float>(c.rf64[9 * i + k]);
            rf32[12 * i + 9] = static_cast<float>(c.te_s[i]);  // per-step intervals (s) in the pad
            rf32[12 * i + 10] = static_cast<float>(c.rest_s[i]);
        }
        // x-axis pulses: the x row and column are (1, 0, 0) up to FP64 dust
        // (rot(Z, pi) carries sin(pi) = 1.2e-16), far below FP32 resolution
        c.rf_xaxis = n > 0;
        for (int64_t i = 0; i < n && c.rf_xaxis; ++i) {
            const double* r = &c.rf64[9 * i];
            c.rf_xaxis = std::fabs(r[0] - 1.0) <= 1e-12 && std::fabs(r[1]) <= 1e-12 && std::fabs(r[2]) <= 1e-12 &&
                         std::fabs(r[3]) <= 1e-12 && std::fabs(r[6]) <= 1e-12;
        }
        // symmetric echo: the te and rest intervals are equal in FP64 (TE = TR/2:
        // tr*1e-3 - (tr/2)*1e-3 == (tr/2)*1e-3 exactly), so every table value
        // and StepU field of the two stages is identical
        c.te_sym = n > 0;
        for (int64_t i = 0; i < n && c.te_sym; ++i) c.te_sym = c.te_s[i] == c.rest_s[i];
        double inv[9];
        host_rf_matrix(3.14159265358979323846, 0, inv);  // bloch.cpp:113
        // kInvert * (0,0,1) = third column
        std::memcpy(c.inv64, inv, sizeof inv);
        c.rf64_d.ensure(sizeof(double) * 9 * n);
        c.rf32_d.ensure(sizeof(float) * 12 * n);
        MRFG_CUDA(cudaMemcpy(c.rf64_d.p, c.rf64.data(), sizeof(double) * 9 * n, cudaMemcpyHostToDevice));
        MRFG_CUDA(cudaMemcpy(c.rf32_d.p, rf32.data(), sizeof(float) * 12 * n, cudaMemcpyHostToDevice));
        *out = h;
    });
}

int mrfg_destroy(mrfg_ctx* h) {
    return guard([&] {
        if (!h) return;
        Ctx& c = h->c;
        cudaSetDevice(c.device);
        cudaStreamSynchronize(c.stream);
        for (DevBuf* b : {&c.zoom, &c.rf64_d, &c.rf32_d, &c.tab.e1f, &c.tab.e2f, &c.tab.phf, &c.tab.e1d,
                          &c.tab.e2d, &c.tab.phd, &c.tab.stepu, &c.tab.kt, &c.q64, &c.qprime, &c.best,
                          &c.cand, &c.cand_count, &c.atoms_a, &c.inv2, &c.seed_a, &c.seed_inv2, &c.rerank,
                          &c.params, &c.out64, &c.misc, &c.rerank_scratch, &c.misc2, &c.audit, &c.h_raw,
                          &c.h_res, &c.h_dict})
            b->release();
        if (c.own_stream) cudaStreamDestroy(c.stream);
        if (c.aux) {
            cudaStreamSynchronize(c.aux);
            cudaStreamDestroy(c.aux);
            for (auto e : c.ev) cudaEventDestroy(e);
        }
        delete h;
    });
}

int64_t mrfg_length(const mrfg_ctx* h) { return h ? h->c.n : 0; }

int mrfg_set_stream(mrfg_ctx* h, void* s) {
    return guard([&] {
        Ctx& c = h->c;
        if (c.own_stream) MRFG_CUDA(cudaStreamDestroy(c.stream));
        c.stream = static_cast<cudaStream_t>(s);
        c.own_stream = false;
    });
}

int mrfg_synchronize(mrfg_ctx* h) {
    return guard([&] { MRFG_CUDA(cudaStreamSynchronize(h->c.stream)); });
}

int mrfg_simulate_dev(mrfg_ctx* h, const double* d_params, int64_t count, int precision,
                      int normalize, double* d_out) {
    return guard([&] {
        Ctx& c = h->c;
        MRFG_CUDA(cudaSetDevice(c.device));
        if (count <= 0) return;
        if (precision == 64)
            launch_simulate64(c, d_params, count, normalize, d_out);
        else
            launch_simulate32(c, d_params, count, normalize, d_out);
    });
}

int mrfg_simulate(mrfg_ctx* h, const double* params, int64_t count, int precision, int normalize,
                  double* out) {
    return guard([&] {
        Ctx& c = h->c;
        MRFG_CUDA(cudaSetDevice(c.device));
        for (int64_t k = 0; k < count; ++k)
            MRFG_REQUIRE(params[3 * k] > 0 && params[3 * k + 1] > 0, MRFG_E_INVALID,
                         "simulate: T1 and T2 must be positive");  // bloch.cpp:109-110
        if (count <= 0) return;
        c.params.ensure(sizeof(double) * 3 * count);
        c.out64.ensure(sizeof(double) * 2 * c.n * count);
        MRFG_CUDA(cudaMemcpyAsync(c.params.p, params, sizeof(double) * 3 * count,
                                  cudaMemcpyHostToDevice, c.stream));
        if (precision == 64)
            launch_simulate64(c, c.params.as<double>(), count, normalize, c.out64.as<double>());
        else
            launch_simulate32(c, c.params.as<double>(), count, normalize, c.out64.as<double>());
        MRFG_CUDA(cudaMemcpyAsync(out, c.out64.p, sizeof(double) * 2 * c.n * count,
                                  cudaMemcpyDeviceToHost, c.stream));
        MRFG_CUDA(cudaStreamSynchronize(c.stream));
    });
}

int mrfg_generate_dev(mrfg_ctx* h, const mrfg_grid* grid, int64_t first, int64_t count,
                      int precision, float* d_out) {
    return guard([&] {
        Ctx& c = h->c;
        MRFG_CUDA(cudaSetDevice(c.device));
        MRFG_REQUIRE(first >= 0 && count >= 0 && first + count <= grid_total(*grid), MRFG_E_INVALID,
                     "generate: flat range outside the grid");
        const GridTables& t = ensure_tables(c, *grid, precision == 64);
        launch_generate(c, t, first, count, precision, d_out);
    });
}

int mrfg_generate(mrfg_ctx* h, const mrfg_grid* grid, int64_t first, int64_t count, int precision,
                  float* out) {
    return guard([&] {
        Ctx& c = h->c;
        MRFG_CUDA(cudaSetDevice(c.device));
        MRFG_REQUIRE(first >= 0 && count >= 0 && first + count <= grid_total(*grid), MRFG_E_INVALID,
                     "generate: flat range outside the grid");
        const GridTables& t = ensure_tables(c, *grid, precision == 64);
        const int64_t per = std::max<int64_t>(1, (int64_t(256) << 20) / (8 * c.n));
        c.misc.ensure(sizeof(float) * 2 * c.n * std::min(per, std::max<int64_t>(count, 1)));
        for (int64_t f = 0; f < count; f += per) {
            int64_t k = std::min(per, count - f);
            launch_generate(c, t, first + f, k, precision, c.misc.as<float>());
            MRFG_CUDA(cudaMemcpyAsync(out + f * 2 * c.n, c.misc.p, sizeof(float) * 2 * c.n * k,
                                      cudaMemcpyDeviceToHost, c.stream));
            MRFG_CUDA(cudaStreamSynchronize(c.stream));
        }
    });
}

int mrfg_bloch_norms_dev(mrfg_ctx* h, const mrfg_grid* grid, int64_t first, int64_t count,
                         float* d_norm2) {
    return guard([&] {
        Ctx& c = h->c;
        MRFG_CUDA(cudaSetDevice(c.device));
        const GridTables& t = ensure_tables(c, *grid, false);
        launch_bloch_norms(c, t, first, count, d_norm2);
    });
}

int mrfg_scan_grid_dev(mrfg_ctx* h, const mrfg_grid* grid, int64_t fb, int64_t fe,
                       const double* d_queries, int64_t nq, int metric, const mrfg_scan_opts* o,
                       mrfg_match* d_out, mrfg_scan_stats* st) {
    return guard([&] {
        Ctx& c = h->c;
        MRFG_CUDA(cudaSetDevice(c.device));
        scan_dev(c, grid, nullptr, 0, fb, fe, d_queries, nq, metric, o, d_out, st);
    });
}

int mrfg_scan_seed_dev(mrfg_ctx* h, const mrfg_grid* grid, const float* d_dict, int64_t natoms, int64_t fb,
                       int64_t fe, const double* d_queries, int64_t nq, int metric, const mrfg_scan_opts* o,
                       float* d_seed, mrfg_scan_stats* st) {
    return guard([&] {
        Ctx& c = h->c;
        MRFG_CUDA(cudaSetDevice(c.device));
        MRFG_REQUIRE((grid != nullptr) != (d_dict != nullptr), MRFG_E_INVALID,
                     "scan_seed: give either a grid or a dictionary");
        const double delta = (o && o->delta > 0) ? o->delta : kDefaultDelta;
        scan_dev_once(c, grid, d_dict, grid ? 0 : natoms, fb, fe, d_queries, nq, metric, o, delta, nullptr, st,
                      d_seed);
    });
}

int mrfg_scan_dict_dev(mrfg_ctx* h, const float* d_dict, int64_t natoms, int64_t fb, int64_t fe,
                       const double* d_queries, int64_t nq, int metric, const mrfg_scan_opts* o,
                       mrfg_match* d_out, mrfg_scan_stats* st) {
    return guard([&] {
        Ctx& c = h->c;
        MRFG_CUDA(cudaSetDevice(c.device));
        MRFG_REQUIRE(natoms > 0, MRFG_E_INVALID, "brute_force_search: empty dictionary");
        scan_dev(c, nullptr, d_dict, natoms, fb, fe, d_queries, nq, metric, o, d_out, st);
    });
}

// The host-buffer entry points stage through per-context device buffers
// (grow-only, kept between calls: no cudaMalloc/cudaFree per call).
int mrfg_scan_dict(mrfg_ctx* h, const float* dict, int64_t natoms, const double* queries,
                   int64_t nq, int metric, const mrfg_scan_opts* o, mrfg_match* out,
                   mrfg_scan_stats* st) {
    return guard([&] {
        Ctx& c = h->c;
        MRFG_CUDA(cudaSetDevice(c.device));
        MRFG_REQUIRE(nq > 0, MRFG_E_INVALID, "scan_grid: no queries");
        MRFG_REQUIRE(natoms > 0, MRFG_E_INVALID, "brute_force_search: empty dictionary");
        c.h_raw.ensure(sizeof(double) * 2 * c.n * nq);
        c.h_res.ensure(sizeof(mrfg_match) * nq);
        c.h_dict.ensure(sizeof(float) * 2 * c.n * natoms);
        MRFG_CUDA(cudaMemcpyAsync(c.h_dict.p, dict, sizeof(float) * 2 * c.n * natoms, cudaMemcpyHostToDevice,
                                  c.stream));
        MRFG_CUDA(cudaMemcpyAsync(c.h_raw.p, queries, sizeof(double) * 2 * c.n * nq, cudaMemcpyHostToDevice,
                                  c.stream));
        scan_dev(c, nullptr, c.h_dict.as<float>(), natoms, 0, natoms, c.h_raw.as<double>(), nq, metric, o,
                 c.h_res.as<mrfg_match>(), st);
        MRFG_CUDA(cudaMemcpyAsync(out, c.h_res.p, sizeof(mrfg_match) * nq, cudaMemcpyDeviceToHost, c.stream));
        MRFG_CUDA(cudaStreamSynchronize(c.stream));
    });
}

int mrfg_scan_grid(mrfg_ctx* h, const mrfg_grid* grid, int64_t fb, int64_t fe,
                   const double* queries, int64_t nq, int metric, const mrfg_scan_opts* o,
                   mrfg_match* out, mrfg_scan_stats* st) {
    return guard([&] {
        Ctx& c = h->c;
        MRFG_CUDA(cudaSetDevice(c.device));
        MRFG_REQUIRE(nq > 0, MRFG_E_INVALID, "scan_grid: no queries");
        c.h_raw.ensure(sizeof(double) * 2 * c.n * nq);
        c.h_res.ensure(sizeof(mrfg_match) * nq);
        MRFG_CUDA(cudaMemcpyAsync(c.h_raw.p, queries, sizeof(double) * 2 * c.n * nq, cudaMemcpyHostToDevice,
                                  c.stream));
        scan_dev(c, grid, nullptr, 0, fb, fe, c.h_raw.as<double>(), nq, metric, o, c.h_res.as<mrfg_match>(), st);
        MRFG_CUDA(cudaMemcpyAsync(out, c.h_res.p, sizeof(mrfg_match) * nq, cudaMemcpyDeviceToHost, c.stream));
        MRFG_CUDA(cudaStreamSynchronize(c.stream));
    });
}

int mrfg_merge_matches_dev(mrfg_ctx* h, const mrfg_match* d_in, int nranks, int64_t nq,
                           mrfg_match* d_out) {
    return guard([&] {
        Ctx& c = h->c;
        MRFG_CUDA(cudaSetDevice(c.device));
        MRFG_REQUIRE(nranks >= 1 && nq >= 0, MRFG_E_INVALID, "merge: bad shape");
        if (nq) launch_merge(c, d_in, nranks, nq, d_out);
    });
}

int mrfg_screen_scores(mrfg_ctx* h, const mrfg_grid* grid, int64_t first, int64_t count,
                       const double* queries, int64_t nq, int metric, int use_simt, float* out) {
    return guard([&] {
        Ctx& c = h->c;
        MRFG_CUDA(cudaSetDevice(c.device));
        MRFG_REQUIRE(nq > 0 && count > 0 && first >= 0 && first + count <= grid_total(*grid),
                     MRFG_E_INVALID, "screen_scores: bad shape");
        const GridTables& t = ensure_tables(c, *grid, false);
        const int64_t n = c.n, kp = k_pad_of(n), qrows = round_up(2 * nq, 256);
        // use_simt bit 0: CUDA-core screening GEMM; bit 1: the production
        // row producer (launch_bloch_rows, K1) instead of the table producer
        const bool prod = (use_simt & 2) != 0;
        const int64_t base = prod ? first / grid->df_hz.count * grid->df_hz.count : first;
        const int64_t rows = round_up(first + count - base, 256);
        DevBuf raw, q64, qp, best, a, inv, cand, cnt;
        raw.ensure(sizeof(double) * 2 * n * nq);
        q64.ensure(sizeof(double) * 2 * n * nq);
        qp.ensure(sizeof(__half) * qrows * kp);
        best.ensure(sizeof(float) * nq + 64);
        a.ensure(sizeof(__half) * rows * kp);
        inv.ensure(sizeof(float) * rows);
        const int64_t cap = count * nq;
        cand.ensure(sizeof(CandRec) * cap);
        cnt.ensure(16);
        int* bad = reinterpret_cast<int*>(best.as<char>() + sizeof(float) * nq);
        MRFG_CUDA(cudaMemcpyAsync(raw.p, queries, sizeof(double) * 2 * n * nq, cudaMemcpyHostToDevice, c.stream));
        MRFG_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), c.stream));
        MRFG_CUDA(cudaMemsetAsync(cnt.p, 0, 16, c.stream));
        launch_prepare_queries(c, raw.as<double>(), nq, qrows, q64.as<double>(), qp.as<__half>(), bad);
        fill(c, best.as<float>(), nq, -3.0f);
        if (prod) {
            const int64_t b2 = launch_bloch_rows(c, t, first, first + count, metric, 0, rows, a.as<__half>(),
                                                 nullptr, inv.as<float>());
            MRFG_REQUIRE(b2 == base, MRFG_E_RUNTIME, "screen_scores: producer base mismatch");
        } else {
            launch_bloch_operand(c, t, first, 1, first + count, rows, metric, a.as<__half>(), inv.as<float>());
        }
        MatchParams mp{};
        mp.a = a.as<__half>();
        mp.inv2 = inv.as<float>();
        mp.b = qp.as<__half>();
        mp.atoms = rows;
        mp.q_rows = qrows;
        mp.k_pad = kp;
        mp.valid_atoms = first + count - base;
        mp.valid_begin = first - base;
        mp.nvox = nq;
        mp.flat_base = base - first;
        mp.flat_stride = 1;
        mp.best = best.as<float>();
        mp.cand = cand.as<CandRec>();
        mp.cand_count = cnt.as<unsigned long long>();
        mp.cand_cap = cap;
        mp.delta = 1e30f;  // every (atom, voxel) pair becomes a candidate
        mp.metric = metric;
        if (use_simt & 1)
            launch_match_simt(c, mp);
        else
            launch_match(c, mp);
        unsigned long long got = 0;
        MRFG_CUDA(cudaMemcpyAsync(&got, cnt.p, sizeof got, cudaMemcpyDeviceToHost, c.stream));
        std::vector<CandRec> h_c(cap);
        MRFG_CUDA(cudaMemcpyAsync(h_c.data(), cand.p, sizeof(CandRec) * cap, cudaMemcpyDeviceToHost, c.stream));
        MRFG_CUDA(cudaStreamSynchronize(c.stream));
        MRFG_REQUIRE(got == static_cast<unsigned long long>(cap), MRFG_E_RUNTIME,
                     "screen_scores: expected every pair to be screened in");
        for (int64_t i = 0; i < nq * count; ++i) out[i] = std::nanf("");
        for (const CandRec& r : h_c) out[r.flat * nq + r.voxel] = r.s;
        for (DevBuf* b : {&raw, &q64, &qp, &best, &a, &inv, &cand, &cnt}) b->release();
    });
}

}  // extern "C"

namespace mrfg {
// cc_map over flats [first, first+count), results delivered in pieces of at
// most `per` scores to sink(offset, device pointer, k) on the ctx stream.
// precision 64: the reference pipeline in FP64 (bit-identical float scores);
// 32: the fused FP32 simulate-and-correlate row kernel (K1 OUT 3).
template <class Sink>
static void cc_map_run(Ctx& c, const mrfg_grid* grid, const double* query, int64_t first, int64_t count,
                       int precision, Sink&& sink) {
    MRFG_REQUIRE(precision == 32 || precision == 64, MRFG_E_INVALID, "cc_map: precision must be 32 or 64");
    MRFG_REQUIRE(first >= 0 && count >= 0 && first + count <= grid_total(*grid), MRFG_E_INVALID,
                 "cc_map: flat range outside the grid");
    const GridTables& t = ensure_tables(c, *grid, precision == 64);
    const int64_t kp = k_pad_of(c.n);
    DevBuf raw, q64, qp, flag, res, q32;
    raw.ensure(sizeof(double) * 2 * c.n);
    q64.ensure(sizeof(double) * 2 * c.n);
    qp.ensure(sizeof(__half) * 256 * kp);
    flag.ensure(sizeof(int));
    const int64_t per = int64_t(1) << 24;
    res.ensure(sizeof(float) * std::min(per, std::max<int64_t>(count, 1)));
    MRFG_CUDA(cudaMemcpyAsync(raw.p, query, sizeof(double) * 2 * c.n, cudaMemcpyHostToDevice, c.stream));
    MRFG_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(int), c.stream));
    launch_prepare_queries(c, raw.as<double>(), 1, 256, q64.as<double>(), qp.as<__half>(), flag.as<int>());
    int bad = 0;
    MRFG_CUDA(cudaMemcpyAsync(&bad, flag.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    MRFG_CUDA(cudaStreamSynchronize(c.stream));
    MRFG_REQUIRE(!bad, MRFG_E_INVALID, "normalize: zero fingerprint");
    if (precision == 32) {  // the FP64 unit query (prep_query) rounded to FP32
        std::vector<double> h64(2 * c.n);
        MRFG_CUDA(cudaMemcpy(h64.data(), q64.p, sizeof(double) * 2 * c.n, cudaMemcpyDeviceToHost));
        std::vector<float> h32(h64.begin(), h64.end());
        q32.ensure(sizeof(float) * 2 * c.n);
        MRFG_CUDA(cudaMemcpyAsync(q32.p, h32.data(), sizeof(float) * 2 * c.n, cudaMemcpyHostToDevice, c.stream));
        MRFG_CUDA(cudaStreamSynchronize(c.stream));
    }
    for (int64_t f = 0; f < count; f += per) {
        const int64_t k = std::min(per, count - f);
        if (precision == 64)
            launch_cc_map(c, t, q64.as<double>(), first + f, k, res.as<float>());
        else
            launch_bloch_rows(c, t, first + f, first + f + k, MRFG_METRIC_CC, 3, k, nullptr, nullptr,
                              res.as<float>(), q32.as<float2>());
        MRFG_CUDA(cudaGetLastError());
        sink(f, res.as<float>(), k);
    }
    for (DevBuf* b : {&raw, &q64, &qp, &flag, &res, &q32}) b->release();
}

// .mrfd / .mrfc header (dictionary.cpp:62-112): magic, u32 version 1, 32-byte
// schedule digest, 3 x (f64 min, f64 step, u64 count), u64 entry length.
static void write_header(FILE* f, const char magic[4], const uint8_t digest[32], const mrfg_grid& g,
                         uint64_t entry_len) {
    const uint32_t version = 1;
    bool ok = fwrite(magic, 1, 4, f) == 4 && fwrite(&version, 4, 1, f) == 1 && fwrite(digest, 1, 32, f) == 32;
    for (const mrfg_axis* ax : {&g.t1_ms, &g.t2_ms, &g.df_hz}) {
        const uint64_t cnt = static_cast<uint64_t>(ax->count);
        ok = ok && fwrite(&ax->min, 8, 1, f) == 1 && fwrite(&ax->step, 8, 1, f) == 1 && fwrite(&cnt, 8, 1, f) == 1;
    }
    ok = ok && fwrite(&entry_len, 8, 1, f) == 1;
    MRFG_REQUIRE(ok, MRFG_E_RUNTIME, "write failed");
}

struct FileCloser {
    FILE* f;
    ~FileCloser() {
        if (f) fclose(f);
    }
};

// Payload writer overlapping the device with the disk: piece i is copied to
// pinned buffer i % 2 on the stream while a host thread writes piece i - 1.
struct PipelinedWriter {
    FILE* f;
    Ctx& c;
    void* pin[2] = {nullptr, nullptr};
    size_t cap = 0;
    int cur = 0;
    std::thread th;
    bool failed = false;
    PipelinedWriter(FILE* f_, Ctx& c_, size_t bytes) : f(f_), c(c_), cap(bytes) {
        MRFG_CUDA(cudaMallocHost(&pin[0], bytes));
        MRFG_CUDA(cudaMallocHost(&pin[1], bytes));
    }
    void put(const void* d_src, size_t bytes) {
        MRFG_CUDA(cudaMemcpyAsync(pin[cur], d_src, bytes, cudaMemcpyDeviceToHost, c.stream));
        MRFG_CUDA(cudaStreamSynchronize(c.stream));
        join();
        void* buf = pin[cur];
        th = std::thread([this, buf, bytes] { failed |= fwrite(buf, 1, bytes, f) != bytes; });
        cur ^= 1;
    }
    void join() {
        if (th.joinable()) th.join();
    }
    ~PipelinedWriter() {
        join();
        for (void* p : pin)
            if (p) cudaFreeHost(p);
    }
};
}  // namespace mrfg

extern "C" {

int mrfg_cc_map(mrfg_ctx* h, const mrfg_grid* grid, const double* query, int64_t first,
                int64_t count, float* out) {
    return mrfg_cc_map_ex(h, grid, query, first, count, 64, out);
}

int mrfg_cc_map_ex(mrfg_ctx* h, const mrfg_grid* grid, const double* query, int64_t first,
                   int64_t count, int precision, float* out) {
    return guard([&] {
        Ctx& c = h->c;
        MRFG_CUDA(cudaSetDevice(c.device));
        cc_map_run(c, grid, query, first, count, precision, [&](int64_t f, const float* d, int64_t k) {
            MRFG_CUDA(cudaMemcpyAsync(out + f, d, sizeof(float) * k, cudaMemcpyDeviceToHost, c.stream));
            MRFG_CUDA(cudaStreamSynchronize(c.stream));
        });
    });
}

int mrfg_cc_map_to_file(mrfg_ctx* h, const mrfg_grid* grid, const double* query, const uint8_t* digest,
                        const char* path, int precision) {
    return guard([&] {
        Ctx& c = h->c;
        MRFG_CUDA(cudaSetDevice(c.device));
        check_grid(*grid);
        MRFG_REQUIRE(!grid_explicit(*grid), MRFG_E_INVALID,
                     "the .mrfd/.mrfc header stores evenly spaced axes only (explicit axis values)");
        FileCloser fc{fopen(path, "wb")};
        MRFG_REQUIRE(fc.f, MRFG_E_RUNTIME, std::string("cannot open for write: ") + path);
        write_header(fc.f, "MRFC", digest, *grid, static_cast<uint64_t>(c.n));
        {
            PipelinedWriter w(fc.f, c, sizeof(float) * (size_t(1) << 24));
            cc_map_run(c, grid, query, 0, grid_total(*grid), precision,
                       [&](int64_t, const float* d, int64_t k) { w.put(d, sizeof(float) * k); });
            w.join();
            MRFG_REQUIRE(!w.failed, MRFG_E_RUNTIME, std::string("write failed: ") + path);
        }
        MRFG_REQUIRE(fflush(fc.f) == 0, MRFG_E_RUNTIME, std::string("write failed: ") + path);
    });
}

int mrfg_save_generated(mrfg_ctx* h, const mrfg_grid* grid, const uint8_t* digest, const char* path,
                        int64_t chunk_entries, int precision) {
    return guard([&] {
        Ctx& c = h->c;
        MRFG_CUDA(cudaSetDevice(c.device));
        MRFG_REQUIRE(chunk_entries > 0, MRFG_E_INVALID, "chunk_entries must be > 0");
        MRFG_REQUIRE(precision == 32 || precision == 64, MRFG_E_INVALID, "generate: precision must be 32 or 64");
        check_grid(*grid);
        MRFG_REQUIRE(!grid_explicit(*grid), MRFG_E_INVALID,
                     "the .mrfd/.mrfc header stores evenly spaced axes only (explicit axis values)");
        FileCloser fc{fopen(path, "wb")};
        MRFG_REQUIRE(fc.f, MRFG_E_RUNTIME, std::string("cannot open for write: ") + path);
        write_header(fc.f, "MRFD", digest, *grid, static_cast<uint64_t>(c.n));
        const GridTables& t = ensure_tables(c, *grid, precision == 64);
        // the payload does not depend on chunk_entries (bit-identical entries);
        // device pieces of <= 256 MB keep the disk busy while the GPU generates
        const int64_t total = grid_total(*grid);
        const int64_t per = std::max<int64_t>(1, (int64_t(256) << 20) / (8 * c.n));
        const size_t piece = sizeof(float) * 2 * c.n * std::min(per, std::max<int64_t>(total, 1));
        DevBuf dev[2];
        dev[0].ensure(piece);
        dev[1].ensure(piece);
        {
            PipelinedWriter w(fc.f, c, piece);
            int b = 0;
            for (int64_t f = 0; f < total; f += per, b ^= 1) {
                const int64_t k = std::min(per, total - f);
                launch_generate(c, t, f, k, precision, dev[b].as<float>());
                MRFG_CUDA(cudaGetLastError());
                w.put(dev[b].p, sizeof(float) * 2 * c.n * k);
            }
            w.join();
            MRFG_REQUIRE(!w.failed, MRFG_E_RUNTIME, std::string("write failed: ") + path);
        }
        MRFG_REQUIRE(fflush(fc.f) == 0, MRFG_E_RUNTIME, std::string("write failed: ") + path);
    });
}

// ---------------------------------------------------------------- noise
// Host restatements of the Experiment-4 noise tooling (fingerprint.cpp:80-145),
// operand order identical to the reference (bit-identical sigma / output).
namespace {
double fp_norm2(const double* v, int64_t n) {  // fingerprint.cpp:14-18
    double acc = 0;
    for (int64_t j = 0; j < n; ++j) acc += v[2 * j] * v[2 * j] + v[2 * j + 1] * v[2 * j + 1];
    return std::sqrt(acc);
}
double fp_cc(const double* a, const double* b, int64_t n) {  // fingerprint.cpp:39-55 (not unit)
    double re = 0, im = 0;
    for (int64_t j = 0; j < n; ++j) {
        re += a[2 * j] * b[2 * j] + a[2 * j + 1] * b[2 * j + 1];
        im += a[2 * j + 1] * b[2 * j] - a[2 * j] * b[2 * j + 1];
    }
    double num = std::sqrt(re * re + im * im);
    const double na = fp_norm2(a, n), nb = fp_norm2(b, n);
    MRFG_REQUIRE(na != 0 && nb != 0, MRFG_E_INVALID, "cc: zero fingerprint");
    num /= na * nb;
    return num < 1.0 ? num : 1.0;
}
struct CalibrateFail {};
double calibrate(const double* fp, int64_t n, double target, uint64_t seed) {  // fingerprint.cpp:80-105
    MRFG_REQUIRE(target > 0 && target < 1, MRFG_E_INVALID, "calibrate_noise: target must be in (0,1)");
    MRFG_REQUIRE(n > 0, MRFG_E_INVALID, "cc: empty input");
    std::vector<double> noisy(2 * n);
    auto cc_at = [&](double sigma) {
        mrfg_add_noise(fp, n, sigma, seed, noisy.data());
        return fp_cc(fp, noisy.data(), n);
    };
    double lo = 0;
    double hi = fp_norm2(fp, n) / std::sqrt(static_cast<double>(n));
    double c = cc_at(hi);
    for (int i = 0; i < 80 && c > target; ++i) {
        if (std::abs(c - target) <= 0.02) return hi;
        hi *= 2;
        c = cc_at(hi);
    }
    if (c > target) throw Error{MRFG_E_RUNTIME, "calibrate_noise: cannot bracket target"};
    for (int i = 0; i < 60; ++i) {
        double mid = 0.5 * (lo + hi);
        double cm = cc_at(mid);
        if (std::abs(cm - target) <= 0.02) return mid;
        (cm > target ? lo : hi) = mid;
    }
    throw Error{MRFG_E_RUNTIME, "calibrate_noise: no sigma within tolerance after 60 steps"};
}
}  // namespace

int mrfg_calibrate_noise(const double* fp, int64_t n, double target_cc, uint64_t seed, double* sigma) {
    return guard([&] { *sigma = calibrate(fp, n, target_cc, seed); });
}

int mrfg_make_calibrated_noise(const double* fp, int64_t n, double target_cc, uint64_t seed,
                               double* sigma, uint64_t* seed_used, double* noisy) {
    return guard([&] {  // fingerprint.cpp:107-120: up to 8 deterministic realizations
        for (int attempt = 0;; ++attempt) {
            const uint64_t sd = attempt == 0 ? seed : mrfg_rng_at(seed, 99, attempt);
            try {
                const double sg = calibrate(fp, n, target_cc, sd);
                *sigma = sg;
                *seed_used = sd;
                mrfg_add_noise(fp, n, sg, sd, noisy);
                return;
            } catch (const Error& e) {
                if (e.code != MRFG_E_RUNTIME || attempt >= 7) throw;
            }
        }
    });
}

int mrfg_smooth(const double* fp, int64_t n, int k, double* out) {
    return guard([&] {  // fingerprint.cpp:122-145
        MRFG_REQUIRE(k == 3 || k == 5, MRFG_E_INVALID, "smooth: kernel must be 3 or 5");
        MRFG_REQUIRE(n > 0, MRFG_E_INVALID, "smooth: empty input");
        const double sigma = (k == 3) ? 0.85 : 1.0;
        const int hh = k / 2;
        double w[5];
        for (int j = -hh; j <= hh; ++j) w[j + hh] = std::exp(-0.5 * j * j / (sigma * sigma));
        for (int64_t i = 0; i < n; ++i) {
            double re = 0, im = 0, wsum = 0;
            for (int j = -hh; j <= hh; ++j) {
                const int64_t t = i + j;
                if (t < 0 || t >= n) continue;
                re += w[j + hh] * fp[2 * t];
                im += w[j + hh] * fp[2 * t + 1];
                wsum += w[j + hh];
            }
            out[2 * i] = re / wsum;
            out[2 * i + 1] = im / wsum;
        }
    });
}

int mrfg_write_header(const char* path, const char* magic, const mrfg_grid* grid, const uint8_t* digest,
                      int64_t entry_len) {
    return guard([&] {
        FileCloser fc{fopen(path, "wb")};
        MRFG_REQUIRE(fc.f, MRFG_E_RUNTIME, std::string("cannot open for write: ") + path);
        write_header(fc.f, magic, digest, *grid, static_cast<uint64_t>(entry_len));
    });
}

int mrfg_read_header(const char* path, const char* magic, mrfg_grid* grid, uint8_t* digest,
                     int64_t* entry_len, int64_t* payload_offset) {
    return guard([&] {
        FileCloser fc{fopen(path, "rb")};
        MRFG_REQUIRE(fc.f, MRFG_E_RUNTIME, std::string("cannot open: ") + path);
        char m[4];
        uint32_t version = 0;
        MRFG_REQUIRE(fread(m, 1, 4, fc.f) == 4 && std::memcmp(m, magic, 4) == 0, MRFG_E_RUNTIME,
                     std::string("bad magic in ") + path);
        MRFG_REQUIRE(fread(&version, 4, 1, fc.f) == 1 && version == 1, MRFG_E_RUNTIME,
                     std::string("unsupported version in ") + path);
        bool ok = fread(digest, 1, 32, fc.f) == 32;
        for (mrfg_axis* ax : {&grid->t1_ms, &grid->t2_ms, &grid->df_hz}) {
            uint64_t cnt = 0;
            ok = ok && fread(&ax->min, 8, 1, fc.f) == 1 && fread(&ax->step, 8, 1, fc.f) == 1 &&
                 fread(&cnt, 8, 1, fc.f) == 1;
            ax->count = static_cast<int64_t>(cnt);
        }
        uint64_t el = 0;
        ok = ok && fread(&el, 8, 1, fc.f) == 1;
        MRFG_REQUIRE(ok, MRFG_E_RUNTIME, std::string("truncated header in ") + path);
        MRFG_REQUIRE(grid_total(*grid) != 0 && el != 0, MRFG_E_RUNTIME,
                     std::string("degenerate dimensions in ") + path);
        *entry_len = static_cast<int64_t>(el);
        if (payload_offset) *payload_offset = ftell(fc.f);
    });
}

namespace {
// mrfg_zoom_io on the device: the dictionary payload (host payloads are
// uploaded into a persistent buffer) and the trace outputs.
struct ZoomDevIo {
    const float* dict = nullptr;
    int64_t entries = 0;
    mrfg_stage* trace = nullptr;
    int* trace_len = nullptr;
};
ZoomDevIo zoom_io_upload(Ctx& c, const mrfg_zoom_io* io, int64_t nvox) {
    ZoomDevIo d;
    if (!io) return d;
    if (io->dict) {
        MRFG_REQUIRE(io->dict_entries > 0, MRFG_E_INVALID, "objective: dictionary does not match the lattice");
        if (io->dict_on_device) {
            d.dict = io->dict;
        } else {
            const size_t b = sizeof(float) * 2 * c.n * io->dict_entries;
            c.h_zdict.ensure(b);
            MRFG_CUDA(cudaMemcpyAsync(c.h_zdict.p, io->dict, b, cudaMemcpyHostToDevice, c.stream));
            d.dict = c.h_zdict.as<float>();
        }
        d.entries = io->dict_entries;
    }
    if (io->trace) {
        MRFG_REQUIRE(io->trace_len, MRFG_E_INVALID, "quantify: trace without trace_len");
        c.h_trace.ensure((sizeof(mrfg_stage) * MRFG_TRACE_MAX + sizeof(int)) * nvox);
        d.trace = c.h_trace.as<mrfg_stage>();
        d.trace_len = reinterpret_cast<int*>(d.trace + MRFG_TRACE_MAX * nvox);
    }
    return d;
}
// Device trace records of voxels [0, nvox) -> the caller's host records of
// voxels dst[k] (identity when dst is null).
void zoom_trace_download(Ctx& c, const mrfg_zoom_io* io, const ZoomDevIo& d, int64_t nvox, const int64_t* dst) {
    if (!d.trace) return;
    std::vector<mrfg_stage> rec(static_cast<size_t>(MRFG_TRACE_MAX * nvox));
    std::vector<int> len(static_cast<size_t>(nvox));
    MRFG_CUDA(cudaMemcpyAsync(rec.data(), d.trace, sizeof(mrfg_stage) * rec.size(), cudaMemcpyDeviceToHost, c.stream));
    MRFG_CUDA(cudaMemcpyAsync(len.data(), d.trace_len, sizeof(int) * len.size(), cudaMemcpyDeviceToHost, c.stream));
    MRFG_CUDA(cudaStreamSynchronize(c.stream));
    for (int64_t k = 0; k < nvox; ++k) {
        const int64_t o = dst ? dst[k] : k;
        std::memcpy(io->trace + o * MRFG_TRACE_MAX, rec.data() + k * MRFG_TRACE_MAX,
                    sizeof(mrfg_stage) * MRFG_TRACE_MAX);
        io->trace_len[o] = len[k];
    }
}
void fill_axis_values(const mrfg_grid& g, mrfg_quant& q) {  // AxisSpec::value (dictionary.hpp:22)
    q.t1_ms = g.t1_ms.min + static_cast<double>(q.i1) * g.t1_ms.step;
    q.t2_ms = g.t2_ms.min + static_cast<double>(q.i2) * g.t2_ms.step;
    q.df_hz = g.df_hz.min + static_cast<double>(q.idf) * g.df_hz.step;
}
}  // namespace

int mrfg_quantify_ex(mrfg_ctx* h, const mrfg_grid* lattice, const mrfg_zoom_config* cfg, const double* fps,
                     int64_t nvox, const int64_t* bounds, const double* init_ms, const mrfg_zoom_io* io,
                     mrfg_quant* out) {
    return guard([&] {
        Ctx& c = h->c;
        MRFG_CUDA(cudaSetDevice(c.device));
        MRFG_REQUIRE(nvox >= 0, MRFG_E_INVALID, "quantify: negative voxel count");
        if (nvox == 0) return;
        if (bounds)
            for (int64_t k = 0; k < nvox; ++k)
                MRFG_REQUIRE(bounds[6 * k] <= bounds[6 * k + 1] && bounds[6 * k + 2] <= bounds[6 * k + 3] &&
                                 bounds[6 * k + 4] <= bounds[6 * k + 5],
                             MRFG_E_INVALID, "zoom_2d: empty range");  // zoom.cpp:176,287
        c.h_raw.ensure(sizeof(double) * 2 * c.n * nvox);
        c.h_res.ensure(sizeof(mrfg_quant) * nvox);
        MRFG_CUDA(cudaMemcpyAsync(c.h_raw.p, fps, sizeof(double) * 2 * c.n * nvox, cudaMemcpyHostToDevice,
                                  c.stream));
        const ZoomDevIo d = zoom_io_upload(c, io, nvox);
        run_quantify(c, *lattice, *cfg, c.h_raw.as<double>(), nvox, bounds, init_ms, c.h_res.as<mrfg_quant>(), 0,
                     nullptr, nullptr, d.dict, d.entries, d.trace, d.trace_len);
        MRFG_CUDA(cudaMemcpyAsync(out, c.h_res.p, sizeof(mrfg_quant) * nvox, cudaMemcpyDeviceToHost, c.stream));
        MRFG_CUDA(cudaStreamSynchronize(c.stream));
        zoom_trace_download(c, io, d, nvox, nullptr);
        for (int64_t k = 0; k < nvox; ++k) fill_axis_values(*lattice, out[k]);
    });
}

int mrfg_quantify_b1(mrfg_ctx* const* ctxs, int nb, const mrfg_grid* lattice, const mrfg_zoom_config* cfg,
                     const int64_t* steps, int nsteps, int64_t init_ib, const double* fps, int64_t nvox,
                     mrfg_quant* out, int64_t* ib_out) {
    return guard([&] {
        MRFG_REQUIRE(nb > 0 && ctxs, MRFG_E_INVALID, "quantify_b1: no B1 values");
        MRFG_REQUIRE(nvox >= 0, MRFG_E_INVALID, "quantify: negative voxel count");
        for (int k = 0; k < nsteps; ++k)
            MRFG_REQUIRE(steps[k] > 0, MRFG_E_INVALID, "zoom_1d: step must be positive");  // zoom.cpp:258
        const int64_t n = ctxs[0]->c.n;
        for (int k = 0; k < nb; ++k)
            MRFG_REQUIRE(ctxs[k] && ctxs[k]->c.n == n && ctxs[k]->c.device == ctxs[0]->c.device, MRFG_E_INVALID,
                         "quantify_b1: contexts differ in length or device");
        if (nvox == 0) return;
        const int64_t n2 = 2 * n;
        // the fingerprints go to the device once; each round gathers its
        // voxel groups there (k_gather_rows) instead of re-uploading them
        MRFG_CUDA(cudaSetDevice(ctxs[0]->c.device));
        DevBuf d_all;
        d_all.ensure(sizeof(double) * n2 * nvox);
        MRFG_CUDA(cudaMemcpy(d_all.p, fps, sizeof(double) * n2 * nvox, cudaMemcpyHostToDevice));
        auto clampi = [&](int64_t v) { return v < 0 ? int64_t(0) : (v >= nb ? int64_t(nb - 1) : v); };
        // per-voxel memo of the inner searches and the outer walk's state
        std::vector<mrfg_quant> res(static_cast<size_t>(nvox * nb));
        std::vector<uint8_t> have(static_cast<size_t>(nvox * nb), 0), acq(static_cast<size_t>(nvox * nb), 0);
        struct Walk {
            int64_t x = 0;
            double fx = 0;
            int si = 0, phase = 0;  // 0 start, 1 left flank, 2 right flank, 3 done
            int64_t evals = 0;
        };
        std::vector<Walk> w(static_cast<size_t>(nvox));
        for (auto& v : w) v.x = clampi(init_ib);
        // g(ib) in the walk's order: the first read acquires (counts) the value
        auto read = [&](int64_t v, int64_t ib) {
            const size_t k = static_cast<size_t>(v * nb + ib);
            if (!acq[k]) {
                acq[k] = 1;
                w[v].evals += res[k].evaluations;
            }
            return res[k].score;
        };
        // advance voxel v's walk (zoom.cpp:252-282) as far as the memo allows;
        // returns the B1 indices it needs next (first: the one it waits on)
        auto advance = [&](int64_t v, std::vector<int64_t>& need) {
            Walk& s = w[v];
            auto ready = [&](int64_t ib) { return have[static_cast<size_t>(v * nb + ib)] != 0; };
            for (;;) {
                if (s.phase == 0) {
                    if (!ready(s.x)) {
                        need.push_back(s.x);
                        if (nsteps) {  // speculative: the first step's flanks
                            need.push_back(clampi(s.x - steps[0]));
                            need.push_back(clampi(s.x + steps[0]));
                        }
                        return;
                    }
                    s.fx = read(v, s.x);
                    s.phase = 1;
                }
                if (s.si >= nsteps) {
                    s.phase = 3;
                    return;
                }
                const int64_t st = steps[s.si];
                if (s.phase == 1) {
                    const int64_t xl = clampi(s.x - st);
                    if (xl != s.x) {
                        if (!ready(xl)) {
                            need.push_back(xl);
                            need.push_back(clampi(s.x + st));  // speculative: the right flank
                            return;
                        }
                        const double fl = read(v, xl);
                        if (fl > s.fx) {
                            s.x = xl;
                            s.fx = fl;
                            continue;
                        }
                    }
                    s.phase = 2;
                }
                const int64_t xr = clampi(s.x + st);
                if (xr != s.x) {
                    if (!ready(xr)) {
                        need.push_back(xr);
                        return;
                    }
                    const double fr = read(v, xr);
                    if (fr > s.fx) {
                        s.x = xr;
                        s.fx = fr;
                        s.phase = 1;
                        continue;
                    }
                }
                s.phase = 1;
                ++s.si;
            }
        };
        // each round: the (voxel, B1) pairs the walks need, in ONE K5 launch
        // (voxel k of the launch uses schedule ib[k]: rf_b / sut_b per B1)
        MRFG_REQUIRE(nb <= 16, MRFG_E_INVALID, "quantify_b1: at most 16 B1 values");
        Ctx& c0 = ctxs[0]->c;
        std::vector<Ctx*> sched(static_cast<size_t>(nb));
        for (int k = 0; k < nb; ++k) sched[k] = &ctxs[k]->c;
        std::vector<int64_t> iv;
        std::vector<int> ibv;
        std::vector<uint8_t> pend(static_cast<size_t>(nvox * nb), 0);
        for (;;) {
            iv.clear();
            ibv.clear();
            std::vector<int64_t> need;
            for (int64_t v = 0; v < nvox; ++v) {
                if (w[v].phase == 3) continue;
                need.clear();
                advance(v, need);
                for (int64_t ib : need) {
                    const size_t key = static_cast<size_t>(v * nb + ib);
                    if (!have[key] && !pend[key]) {
                        pend[key] = 1;
                        iv.push_back(v);
                        ibv.push_back(static_cast<int>(ib));
                    }
                }
            }
            if (iv.empty()) break;
            const int64_t m = static_cast<int64_t>(iv.size());
            std::vector<mrfg_quant> r(iv.size());
            MRFG_CUDA(cudaSetDevice(c0.device));
            c0.zidx.ensure(sizeof(int64_t) * m);
            c0.zib.ensure(sizeof(int) * m);
            c0.h_raw.ensure(sizeof(double) * n2 * m);
            c0.h_res.ensure(sizeof(mrfg_quant) * m);
            MRFG_CUDA(cudaMemcpyAsync(c0.zidx.p, iv.data(), sizeof(int64_t) * m, cudaMemcpyHostToDevice, c0.stream));
            MRFG_CUDA(cudaMemcpyAsync(c0.zib.p, ibv.data(), sizeof(int) * m, cudaMemcpyHostToDevice, c0.stream));
            k_gather_rows<<<static_cast<unsigned>(m), 256, 0, c0.stream>>>(d_all.as<double>(), c0.zidx.as<int64_t>(),
                                                                           n2, c0.h_raw.as<double>());
            MRFG_CUDA(cudaGetLastError());
            run_quantify(c0, *lattice, *cfg, c0.h_raw.as<double>(), m, nullptr, nullptr, c0.h_res.as<mrfg_quant>(), 0,
                         nullptr, nullptr, nullptr, 0, nullptr, nullptr, c0.zib.as<int>(), sched.data(), nb);
            MRFG_CUDA(cudaMemcpyAsync(r.data(), c0.h_res.p, sizeof(mrfg_quant) * m, cudaMemcpyDeviceToHost, c0.stream));
            MRFG_CUDA(cudaStreamSynchronize(c0.stream));
            for (int64_t k = 0; k < m; ++k) {
                const size_t key = static_cast<size_t>(iv[k] * nb + ibv[k]);
                res[key] = r[k];
                have[key] = 1;
            }
        }
        for (int64_t v = 0; v < nvox; ++v) {
            out[v] = res[static_cast<size_t>(v * nb + w[v].x)];
            out[v].evaluations = w[v].evals;
            ib_out[v] = w[v].x;
        }
    });
}

int mrfg_quantify_bounded(mrfg_ctx* h, const mrfg_grid* lattice, const mrfg_zoom_config* cfg,
                          const double* fps, int64_t nvox, const int64_t* bounds,
                          const double* init_ms, mrfg_quant* out) {
    return mrfg_quantify_ex(h, lattice, cfg, fps, nvox, bounds, init_ms, nullptr, out);
}

int mrfg_quantify_dev(mrfg_ctx* h, const mrfg_grid* lattice, const mrfg_zoom_config* cfg,
                      const double* d_fps, int64_t nvox, mrfg_quant* d_out) {
    return guard([&] {
        Ctx& c = h->c;
        MRFG_CUDA(cudaSetDevice(c.device));
        MRFG_REQUIRE(nvox >= 0, MRFG_E_INVALID, "quantify: negative voxel count");
        if (nvox) run_quantify(c, *lattice, *cfg, d_fps, nvox, nullptr, nullptr, d_out);
    });
}

int mrfg_quantify(mrfg_ctx* h, const mrfg_grid* lattice, const mrfg_zoom_config* cfg,
                  const double* fps, int64_t nvox, mrfg_quant* out) {
    return mrfg_quantify_bounded(h, lattice, cfg, fps, nvox, nullptr, nullptr, out);
}

namespace {
// Prior window around a finished voxel (zoom.cpp:595-610): the prior's
// parameters round-trip through seconds exactly like QuantResult::params.
void prior_of(const mrfg_grid& g, const mrfg_zoom_config& cfg, const mrfg_quant& pr, int64_t* b,
              double* init) {
    auto snap = [](double v, const mrfg_axis& ax) { return std::lround((v - ax.min) / ax.step); };
    auto units = [](double s, double fine) {
        long u = std::lround(s / fine);
        return u > 0 ? u : 1L;
    };
    const double t1 = (g.t1_ms.min + static_cast<double>(pr.i1) * g.t1_ms.step) * 1e-3 * 1e3;
    const double t2 = (g.t2_ms.min + static_cast<double>(pr.i2) * g.t2_ms.step) * 1e-3 * 1e3;
    const double df = g.df_hz.min + static_cast<double>(pr.idf) * g.df_hz.step;
    init[0] = t1;
    init[1] = t2;
    const long p1 = snap(t1, g.t1_ms), p2 = snap(t2, g.t2_ms), pdf = snap(df, g.df_hz);
    const long w1 = units(cfg.prior_window_t1_ms, g.t1_ms.step);
    const long w2 = units(cfg.prior_window_t2_ms, g.t2_ms.step);
    const long wdf = units(cfg.prior_window_df_hz, g.df_hz.step);
    b[0] = std::max<int64_t>(0, p1 - w1);
    b[1] = std::min<int64_t>(g.t1_ms.count - 1, p1 + w1);
    b[2] = std::max<int64_t>(0, p2 - w2);
    b[3] = std::min<int64_t>(g.t2_ms.count - 1, p2 + w2);
    b[4] = std::max<int64_t>(0, pdf - wdf);
    b[5] = std::min<int64_t>(g.df_hz.count - 1, pdf + wdf);
}
void full_bounds(const mrfg_grid& g, int64_t* b) {
    b[0] = 0;
    b[1] = g.t1_ms.count - 1;
    b[2] = 0;
    b[3] = g.t2_ms.count - 1;
    b[4] = 0;
    b[5] = g.df_hz.count - 1;
}
}  // namespace

int mrfg_quantify_slice_ex(mrfg_ctx* h, const mrfg_grid* lattice, const mrfg_zoom_config* cfg,
                           const double* fps, const uint8_t* mask, int nx, int ny, int use_prior,
                           const mrfg_zoom_io* io, mrfg_quant* out, double* seconds) {
    return guard([&] {
        Ctx& c = h->c;
        MRFG_CUDA(cudaSetDevice(c.device));
        MRFG_REQUIRE(nx > 0 && ny > 0, MRFG_E_INVALID,
                     "quantify_slice: inconsistent raster dimensions");  // zoom.cpp:561-562
        MRFG_REQUIRE(use_prior >= 0 && use_prior <= 2, MRFG_E_INVALID, "quantify_slice: bad prior mode");
        auto t0 = std::chrono::steady_clock::now();
        const int64_t nv = static_cast<int64_t>(nx) * ny, n2 = 2 * c.n;
        std::memset(out, 0, sizeof(mrfg_quant) * nv);
        if (io && io->trace) {
            std::memset(io->trace, 0, sizeof(mrfg_stage) * MRFG_TRACE_MAX * nv);
            std::memset(io->trace_len, 0, sizeof(int32_t) * nv);
        }
        // masked voxels in raster order (zoom.cpp:579-581)
        std::vector<int64_t> masked;
        for (int64_t i = 0; i < nv; ++i)
            if (mask[i]) masked.push_back(i);
        // the rows kernel stages the schedule in shared memory (72 B/TR)
        const bool rows_fit = (sizeof(StepU) + sizeof(float2)) * c.n + 256 * 32 + 16 <= 200 * 1024;
        if (use_prior == 0 || (use_prior == 1 && !rows_fit)) {
            if (masked.empty()) return;
            if (use_prior == 0) {  // independent voxels (zoom.cpp:616-624)
                std::vector<double> packed(n2 * masked.size());
                for (size_t k = 0; k < masked.size(); ++k)
                    std::memcpy(&packed[n2 * k], fps + n2 * masked[k], sizeof(double) * n2);
                const int64_t m = static_cast<int64_t>(masked.size());
                c.h_raw.ensure(sizeof(double) * n2 * m);
                c.h_res.ensure(sizeof(mrfg_quant) * m);
                MRFG_CUDA(cudaMemcpyAsync(c.h_raw.p, packed.data(), sizeof(double) * n2 * m, cudaMemcpyHostToDevice,
                                          c.stream));
                const ZoomDevIo d = zoom_io_upload(c, io, m);
                run_quantify(c, *lattice, *cfg, c.h_raw.as<double>(), m, nullptr, nullptr, c.h_res.as<mrfg_quant>(),
                             0, nullptr, nullptr, d.dict, d.entries, d.trace, d.trace_len);
                std::vector<mrfg_quant> res(masked.size());
                MRFG_CUDA(cudaMemcpyAsync(res.data(), c.h_res.p, sizeof(mrfg_quant) * m, cudaMemcpyDeviceToHost,
                                          c.stream));
                MRFG_CUDA(cudaStreamSynchronize(c.stream));
                zoom_trace_download(c, io, d, m, masked.data());
                for (size_t k = 0; k < masked.size(); ++k) {
                    out[masked[k]] = res[k];
                    fill_axis_values(*lattice, out[masked[k]]);
                }
            } else {
                // strict raster with a schedule too long for the rows kernel:
                // one voxel in flight, driven from the host (zoom.cpp:589-615)
                bool have = false;
                int64_t prev = -1;
                for (int64_t i : masked) {
                    int64_t b[6];
                    double init[2];
                    if (have) {
                        prior_of(*lattice, *cfg, out[prev], b, init);
                    } else {
                        full_bounds(*lattice, b);
                        init[0] = cfg->init_t1_ms;
                        init[1] = cfg->init_t2_ms;
                    }
                    mrfg_zoom_io one{};
                    if (io) {
                        one = *io;
                        if (io->trace) {
                            one.trace = io->trace + i * MRFG_TRACE_MAX;
                            one.trace_len = io->trace_len + i;
                        }
                    }
                    const int rc = mrfg_quantify_ex(h, lattice, cfg, fps + n2 * i, 1, b, init, io ? &one : nullptr,
                                                    &out[i]);
                    if (rc) throw Error{rc, g_err};
                    prev = i;
                    have = true;
                }
            }
        } else {
            // ONE launch of the row kernel.  use_prior 1: the strict raster
            // (zoom.cpp:589-615) as a single row -- each masked voxel seeded
            // and windowed by the previous one, on one SM with all its warps
            // evaluating the running voxel's rounds.  use_prior 2: the row
            // relaxation SPEC.md:449 permits -- rows of masked voxels in
            // parallel, a row's first voxel seeded by the first voxel of the
            // previous non-empty row, every other voxel by its left neighbour.
            std::vector<int64_t> row_start(1, 0), vox;
            if (use_prior == 1) {
                vox = masked;
                if (!vox.empty()) row_start.push_back(static_cast<int64_t>(vox.size()));
            } else {
                for (int y = 0; y < ny; ++y) {
                    for (int x = 0; x < nx; ++x)
                        if (mask[static_cast<int64_t>(y) * nx + x]) vox.push_back(static_cast<int64_t>(y) * nx + x);
                    if (static_cast<int64_t>(vox.size()) > row_start.back())
                        row_start.push_back(static_cast<int64_t>(vox.size()));
                }
            }
            const int64_t R = static_cast<int64_t>(row_start.size()) - 1;
            if (R > 0) {
                DevBuf& d_fps = c.h_raw;
                DevBuf& d_res = c.h_res;
                d_fps.ensure(sizeof(double) * n2 * nv);
                d_res.ensure(sizeof(mrfg_quant) * nv);
                MRFG_CUDA(cudaMemcpyAsync(d_fps.p, fps, sizeof(double) * n2 * nv, cudaMemcpyHostToDevice, c.stream));
                MRFG_CUDA(cudaMemsetAsync(d_res.p, 0, sizeof(mrfg_quant) * nv, c.stream));
                const ZoomDevIo d = zoom_io_upload(c, io, nv);
                if (d.trace) MRFG_CUDA(cudaMemsetAsync(d.trace_len, 0, sizeof(int) * nv, c.stream));
                run_quantify(c, *lattice, *cfg, d_fps.as<double>(), nv, nullptr, nullptr, d_res.as<mrfg_quant>(), R,
                             row_start.data(), vox.data(), d.dict, d.entries, d.trace, d.trace_len);
                MRFG_CUDA(cudaMemcpyAsync(out, d_res.p, sizeof(mrfg_quant) * nv, cudaMemcpyDeviceToHost, c.stream));
                MRFG_CUDA(cudaStreamSynchronize(c.stream));
                if (d.trace) {
                    std::vector<mrfg_stage> rec(static_cast<size_t>(MRFG_TRACE_MAX * nv));
                    std::vector<int> len(static_cast<size_t>(nv));
                    MRFG_CUDA(cudaMemcpy(rec.data(), d.trace, sizeof(mrfg_stage) * rec.size(), cudaMemcpyDeviceToHost));
                    MRFG_CUDA(cudaMemcpy(len.data(), d.trace_len, sizeof(int) * nv, cudaMemcpyDeviceToHost));
                    for (int64_t v : vox) {
                        std::memcpy(io->trace + v * MRFG_TRACE_MAX, rec.data() + v * MRFG_TRACE_MAX,
                                    sizeof(mrfg_stage) * MRFG_TRACE_MAX);
                        io->trace_len[v] = len[v];
                    }
                }
                for (int64_t v : vox) fill_axis_values(*lattice, out[v]);
            }
        }
        if (seconds)
            *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    });
}

int mrfg_quantify_slice(mrfg_ctx* h, const mrfg_grid* lattice, const mrfg_zoom_config* cfg,
                        const double* fps, const uint8_t* mask, int nx, int ny, int use_prior,
                        mrfg_quant* out, double* seconds) {
    return mrfg_quantify_slice_ex(h, lattice, cfg, fps, mask, nx, ny, use_prior, nullptr, out, seconds);
}

}  // extern "C"
