/*
 * mrfg.h -- C ABI of the B200-native MRF dictionary generating-and-searching
 * (DGS) path.  Implemented in paper_1506_05393_b200/csrc (sm_100a CUDA + C++),
 * built as paper_1506_05393_b200/libmrfg.so.
 *
 * This is the drop-in boundary: the reference's C++ entry points in
 * /root/reference/proj/include/mrf/ keep their signatures in include/mrf/*.hpp
 * (implemented by paper_1506_05393_b200/csrc/host/mrf_api.cpp, libmrf_b200.so)
 * and forward to the functions below.  Each function cites the reference
 * interface it replaces.  Conventions:
 *   - every function returns 0 on success, a negative MRFG_E* code on error,
 *     and mrfg_last_error() (thread-local) describes the failure -- the C++
 *     shim turns these back into the reference's exceptions;
 *   - plain pointers and sizes only; "_dev" entry points take CUDA device
 *     pointers and run asynchronously on the context's stream, every other
 *     entry point takes caller-owned HOST buffers and is synchronous;
 *   - complex vectors are interleaved (re, im) -- the reference's dictionary
 *     entry layout (dictionary.hpp:72-80);
 *   - units follow the reference: schedules deg/ms (sequence.hpp:14-24),
 *     lattices ms/ms/Hz (dictionary.hpp:17-56), tissue params s/s/Hz
 *     (fingerprint.hpp:12-17).
 * There is no CPU fallback: without an sm_100 device every compute entry
 * point fails with MRFG_E_CUDA.
 */
#ifndef MRFG_H
#define MRFG_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    MRFG_OK = 0,
    MRFG_E_INVALID = -1,  /* std::invalid_argument in the reference */
    MRFG_E_RANGE = -2,    /* std::out_of_range (zoom.cpp:126-130) */
    MRFG_E_RUNTIME = -3,  /* std::runtime_error */
    MRFG_E_CUDA = -4,     /* device error / no sm_100 device */
    MRFG_E_NOMEM = -5
};

enum { MRFG_METRIC_CC = 0, MRFG_METRIC_EUCLIDEAN = 1 }; /* Metric, dictionary.hpp:98 */

typedef struct mrfg_ctx mrfg_ctx;

/* AxisSpec (dictionary.hpp:17-24): values min + k*step, k < count.
 * `values` (optional, may be NULL): count explicit axis values that replace
 * min + k*step -- e.g. the log-spaced T1/T2 axes of BASELINE configs[2],
 * which a ParameterGrid cannot express (the reference builds those
 * dictionaries from explicit TissueParams, value[k] ms * 1e-3 s).  Supported
 * on the T1 and T2 axes of generate / scan_grid / cc_map; the df axis and
 * ZOOM lattices must be evenly spaced.  Tables are computed from the values
 * with host libm, so FP64 entries equal the reference's simulate() of the
 * same TissueParams bit for bit. */
typedef struct { double min, step; int64_t count; const double* values; } mrfg_axis;
/* ParameterGrid (dictionary.hpp:34-56): T1 outer, T2 middle, df inner;
 * flat = (i1*n2 + i2)*ndf + idf. */
typedef struct { mrfg_axis t1_ms, t2_ms, df_hz; } mrfg_grid;

/* Match (dictionary.hpp:100-104) reduced to the lattice point and score. */
typedef struct { int64_t flat; double score; } mrfg_match;

/* Screening/streaming knobs of the brute-force path (no reference analogue;
 * zero fields take defaults). */
typedef struct {
    double delta;          /* screening margin in CC units (default 2.5e-3: twice the analytic
                              bound on the fp16 screening error) */
    int64_t chunk_atoms;   /* atoms simulated per streamed chunk (default: lattice scans one full
                              wave of the K1 producer in whole rows, ~300 K atoms on 148 SMs;
                              stored dictionaries 524288) */
    int64_t cand_capacity; /* candidate buffer entries (default 1<<25) */
    int64_t seed_atoms;    /* strided pre-pass atoms that seed the running max (default 16384) */
    /* Optional (device, *_dev calls, metric cc): nq matches of an earlier scan
     * over OTHER atoms (another B1 slab, another shard).  Their scores seed the
     * screening maxima, so only atoms that can still win are re-ranked; a
     * query with no atom above its floor returns flat -1 (merge skips it). */
    const mrfg_match* floor_matches;
    /* Optional HOST array of nq flags: 1 = the query is already unit norm
     * (Fingerprint::unit_norm) and is scored as given, without the FP64
     * normalization of prep_query (dictionary.cpp:145-150). */
    const uint8_t* unit_queries;
} mrfg_scan_opts;

/* What one scan did (device-timed with CUDA events on the ctx stream). */
typedef struct {
    int64_t atoms, voxels, chunks, candidates, reranked, overflow_passes;
    double bloch_ms, gemm_ms, rerank_ms, total_ms;
    double gemm_kernel_ms_avg; /* average duration of one K2 launch */
    int64_t gemm_launches;
    double screen_err_max;     /* max |screen CC - exact CC| over re-ranked candidates (cc;
                                  measured against the FP32 re-screen, +-1e-5, when it runs) */
    int64_t rescreened32;      /* candidates scored by the certified FP32 walk before the
                                  FP64 re-rank (0 when that stage is off); reranked = FP64 */
    /* Unbiased screening audit (metric cc): a hash-sampled subset of ALL
     * screened (voxel, atom) pairs, whatever their screening score, is scored
     * exactly.  screen_err_audit_max = max |fp16 screen CC - exact CC| over it;
     * rescreen_err_audit_max = max |FP32 re-screen - exact| (lattice scans).
     * A scan whose audit exceeds delta/2 is repeated with a wider margin
     * (rescans); one whose FP32 re-screen error exceeds half its margin
     * re-ranks every candidate in FP64. */
    double screen_err_audit_max, rescreen_err_audit_max, delta_used;
    int64_t audit_samples, rescans;
    double rescreen_err_max;   /* max |FP32 re-screen - exact| over the FP64 survivors */
    int64_t chunk_atoms;       /* atoms per streamed chunk (whole lattice rows) */
    /* Per-off-resonance subspace screening (csrc/subspace.cu; default for large
     * lattice scans, MRFG_SUBSPACE=0 off): complex rank used (0: full-length
     * screening), time of the projection kernels, the largest relative
     * residual |a - P a| / |a| over the held-out rows of the basis
     * construction (the default margin grows by twice it), and the device
     * estimate 1 - |P a|^2 / |a|^2 over every screened atom (its fp16 noise
     * floor is ~0.02). */
    double project_ms;
    int64_t subspace_rank;
    double subspace_residual_max;
    double subspace_residual_device;
} mrfg_scan_stats;

/* ZoomConfig (zoom.hpp:23-52) as a POD; the step lists hold up to 8 values.
 * dict_mode selects the reference's dictionary lookups (zoom.cpp:94-123):
 * 0 = every entry simulated (FP64); 1 = df dictionary: entries first acquired
 * during the off-resonance search (stage 1) are the dictionary's float
 * entries (quantify's df_dict, built by make_df_dictionary); 2 = full
 * dictionary: every entry is a float dictionary entry (quantify's full_dict).
 * The payload is passed through mrfg_zoom_io (mrfg_quantify_ex) and read as
 * given; the entry points without it score the entries generate() would
 * produce, float(normalize(simulate)) (dictionary.cpp:37-53), reproduced
 * bit-exactly.  The caller validates the dictionary against the schedule and
 * lattice (zoom.cpp:50-69). */
typedef struct {
    int32_t metric, final_metric, smooth_k, n2d, n1d, dict_mode;
    double omega_hz, df_coarse_hz, df_refine_hz, df_window_hz, plateau_eps, heavy_noise_cc,
        fallback_coarse_hz, fallback_window_hz;
    double t1t2_2d_steps_ms[8];
    double t1t2_1d_steps_ms[8];
    double final_2d_step_ms, init_t1_ms, init_t2_ms, prior_window_t1_ms, prior_window_t2_ms,
        prior_window_df_hz;
} mrfg_zoom_config;

/* QuantResult (zoom.hpp:61-67) with the lattice indices. */
typedef struct {
    int64_t i1, i2, idf;
    double t1_ms, t2_ms, df_hz, pd, score;
    int64_t evaluations;
} mrfg_quant;

/* StageLog (zoom.hpp:54-59): one record per stage note of quantify_impl
 * (log_stage, zoom.cpp:441-451, and search_df's notes, zoom.cpp:179-249):
 * unique evaluations the stage added, its best objective value (exact, the
 * reference's), and its lattice point.  Stage names map to these codes. */
enum {
    MRFG_STAGE_DF_COARSE = 0,    /* "df.coarse" */
    MRFG_STAGE_DF_REFINE,        /* "df.refine" */
    MRFG_STAGE_DF_TRANSLATE,     /* "df.translate" */
    MRFG_STAGE_DF_REREFINE,      /* "df.rerefine" */
    MRFG_STAGE_DF_PLATEAU_STOP,  /* "df.plateau_stop" */
    MRFG_STAGE_DF_FINEST,        /* "df.finest" */
    MRFG_STAGE_DF_FALLBACK,      /* "df.fallback" */
    MRFG_STAGE_T1T2_2D,          /* "t1t2.2d" */
    MRFG_STAGE_DF_SWEEP,         /* "df.sweep" */
    MRFG_STAGE_T1_1D,            /* "t1.1d" */
    MRFG_STAGE_T2_1D,            /* "t2.1d" */
    MRFG_STAGE_T1T2_FINAL        /* "t1t2.final" */
};
/* Upper bound on the records of one voxel: 2 x 19 search_df notes + fallback
 * + 2-D + sweep + 2 x 8 1-D + final = 58. */
#define MRFG_TRACE_MAX 64
typedef struct {
    int32_t stage, pad;
    int64_t evaluations;
    double best, t1_ms, t2_ms, df_hz;
} mrfg_stage;

/* Optional inputs/outputs of mrfg_quantify_ex / mrfg_quantify_slice_ex.
 * dict: the caller's dictionary payload, dict_entries x 2N float (re, im)
 *   in the reference's entry layout -- the df slab of make_df_dictionary
 *   (cfg->dict_mode 1: entry idf) or the full lattice dictionary (dict_mode 2:
 *   flat (i1*n2 + i2)*ndf + idf).  K5 scores these bytes as given, exactly as
 *   Objective::acquire reads d->entry(flat) (zoom.cpp:101-113); NULL with
 *   dict_mode != 0 scores the entries generate() would produce
 *   (float(normalize(simulate)), dictionary.cpp:44-51).  dict_on_device: the
 *   pointer is device memory.
 * trace / trace_len: nvox x MRFG_TRACE_MAX records and nvox counts (host
 *   memory; device memory for the _dev form), or NULL. */
typedef struct {
    const float* dict;
    int64_t dict_entries;
    int32_t dict_on_device, pad;
    mrfg_stage* trace;
    int32_t* trace_len;
} mrfg_zoom_io;

/* ------------------------------------------------------------------ misc */
const char* mrfg_last_error(void);
const char* mrfg_version(void);
/* Fill cfg with the reference's ZoomConfig defaults (zoom.hpp:23-52). */
void mrfg_zoom_config_default(mrfg_zoom_config* cfg);

/* ----------------------------------------------- host-side input synthesis
 * Restatements of the reference's input generators (host C++, no GPU). */
/* build_schedule (sequence.hpp:51, sequence.cpp:77-92) */
int mrfg_reference_schedule(int64_t n, uint64_t seed, double* flip_deg, double* phase_deg,
                            double* tr_ms, double* te_ms);
/* BASELINE.json schedule generator, %.9g-canonical. */
int mrfg_baseline_schedule(int64_t n, uint64_t seed, double* flip_deg, double* phase_deg,
                           double* tr_ms, double* te_ms);
/* add_noise (fingerprint.hpp:53, fingerprint.cpp:68-78) */
int mrfg_add_noise(const double* fp, int64_t n, double sigma, uint64_t seed, double* out);
/* rng::at / uniform01 / gaussian (rng.hpp:24-41) */
uint64_t mrfg_rng_at(uint64_t seed, uint64_t stream, uint64_t index);
double mrfg_rng_uniform01(uint64_t seed, uint64_t stream, uint64_t index);
double mrfg_rng_gaussian(uint64_t seed, uint64_t stream, uint64_t index);
/* Endpoint-exclusive axis count (dictionary.cpp:25-33): 0 and MRFG_E_INVALID
 * when the range is empty or the step non-positive. */
int mrfg_axis_count(double min, double max, double step, int64_t* count);

/* --------------------------------------------------------------- context
 * BlochSimulator(const Schedule&) (bloch.hpp:83, bloch.cpp:95-106): validates
 * 0 <= te <= tr, composes the RF rotations once, uploads the schedule. */
int mrfg_create(const double* flip_deg, const double* phase_deg, const double* tr_ms,
                const double* te_ms, int64_t n, int device, mrfg_ctx** out);
int mrfg_destroy(mrfg_ctx* ctx);
int64_t mrfg_length(const mrfg_ctx* ctx); /* BlochSimulator::length (bloch.hpp:89) */
/* Run on a caller-provided cudaStream_t (e.g. torch's current stream). */
int mrfg_set_stream(mrfg_ctx* ctx, void* cuda_stream);
int mrfg_synchronize(mrfg_ctx* ctx);

/* ------------------------------------------------------------ K1 Bloch
 * BlochSimulator::simulate (bloch.hpp:86-87, bloch.cpp:108-123) for a batch of
 * tissue points params[3*k..] = (t1_s, t2_s, df_hz).  precision 64 is the
 * reference's FP64 recursion (bit-exact with it); 32 is the FP32 FMA kernel.
 * normalize != 0 scales each fingerprint to unit L2 norm (fingerprint.cpp:28-37). */
int mrfg_simulate(mrfg_ctx* ctx, const double* params, int64_t count, int precision,
                  int normalize, double* out /* count x 2N */);
int mrfg_simulate_dev(mrfg_ctx* ctx, const double* d_params, int64_t count, int precision,
                      int normalize, double* d_out);
/* generate / generate_range (dictionary.hpp:85, dictionary.cpp:37-60,184-194):
 * unit-norm float32 entries of flats [first, first+count) of the grid. */
int mrfg_generate(mrfg_ctx* ctx, const mrfg_grid* grid, int64_t first, int64_t count,
                  int precision, float* out /* count x 2N */);
int mrfg_generate_dev(mrfg_ctx* ctx, const mrfg_grid* grid, int64_t first, int64_t count,
                      int precision, float* d_out);
/* FP32 Bloch throughput kernel alone (bench): simulates flats [first,
 * first+count) and accumulates only per-atom norms into d_norm2 (count). */
int mrfg_bloch_norms_dev(mrfg_ctx* ctx, const mrfg_grid* grid, int64_t first, int64_t count,
                         float* d_norm2);

/* ---------------------------------------------------- K2/K3 brute force
 * scan_grid (dictionary.hpp:120-122, dictionary.cpp:257-308): streamed
 * simulate-and-match of flats [flat_begin, flat_end) (the whole grid when
 * both are 0), per-query argmax with the lowest-flat tie rule.  Queries are
 * raw (they are normalized in FP64 as prep_query does, dictionary.cpp:145-150);
 * scores are the reference's FP64 score of the FP32-quantized entry. */
int mrfg_scan_grid(mrfg_ctx* ctx, const mrfg_grid* grid, int64_t flat_begin, int64_t flat_end,
                   const double* queries, int64_t nq, int metric, const mrfg_scan_opts* opts,
                   mrfg_match* out, mrfg_scan_stats* stats);
int mrfg_scan_grid_dev(mrfg_ctx* ctx, const mrfg_grid* grid, int64_t flat_begin,
                       int64_t flat_end, const double* d_queries, int64_t nq, int metric,
                       const mrfg_scan_opts* opts, mrfg_match* d_out, mrfg_scan_stats* stats);
/* K4 -- brute_force_search (dictionary.hpp:108-109, dictionary.cpp:241-255)
 * over a stored dictionary of natoms unit float32 entries (2N interleaved,
 * generate()'s layout): same screening GEMM, exact FP64 re-rank against the
 * stored entries (dictionary.cpp:117-143).  The _dev form takes a device
 * dictionary and a flat range [flat_begin, flat_end) (both 0: all), so a
 * dictionary sharded across GPUs needs no copy. */
int mrfg_scan_dict(mrfg_ctx* ctx, const float* dict, int64_t natoms, const double* queries,
                   int64_t nq, int metric, const mrfg_scan_opts* opts, mrfg_match* out,
                   mrfg_scan_stats* stats);
int mrfg_scan_dict_dev(mrfg_ctx* ctx, const float* d_dict, int64_t natoms, int64_t flat_begin,
                       int64_t flat_end, const double* d_queries, int64_t nq, int metric,
                       const mrfg_scan_opts* opts, mrfg_match* d_out, mrfg_scan_stats* stats);
/* Seed pass only (multi-GPU / multi-device sharding): the screening maxima
 * (CC units, float, nq) of a strided sample of flats [flat_begin, flat_end)
 * of the lattice (grid) or of a device dictionary (d_dict, natoms) -- the
 * maxima a scan of that range starts from.  Maxima of all shards, reduced by
 * max and passed back as floor_matches (flat 0, score = maximum), seed every
 * shard's screening with the GLOBAL sample, so per-shard candidate and
 * re-rank work does not grow with the number of shards; the screening
 * certificate holds for any seed. */
int mrfg_scan_seed_dev(mrfg_ctx* ctx, const mrfg_grid* grid, const float* d_dict, int64_t natoms,
                       int64_t flat_begin, int64_t flat_end, const double* d_queries, int64_t nq, int metric,
                       const mrfg_scan_opts* opts, float* d_seed, mrfg_scan_stats* stats);
/* C1: merge per-rank matches gathered as d_in[rank*nq + q] (max score,
 * lowest flat on ties) -- the reduction after the NCCL allgather. */
int mrfg_merge_matches_dev(mrfg_ctx* ctx, const mrfg_match* d_in, int nranks, int64_t nq,
                           mrfg_match* d_out);

/* Test support: dense K2 screening scores (|z|^2/|d|^2 for cc, Re z/|d| for
 * euclidean) of flats [first, first+count) against nq queries, out[a*nq+v],
 * through the tcgen05 kernel (use_simt = 0) or its CUDA-core twin (1). */
int mrfg_screen_scores(mrfg_ctx* ctx, const mrfg_grid* grid, int64_t first, int64_t count,
                       const double* queries, int64_t nq, int metric, int use_simt, float* out);

/* cc_map (dictionary.hpp:127-129, dictionary.cpp:310-331): float CC of one
 * query against flats [first, first+count). */
int mrfg_cc_map(mrfg_ctx* ctx, const mrfg_grid* grid, const double* query, int64_t first,
                int64_t count, float* out);

/* cc_map with a precision choice: 64 = the reference pipeline in FP64
 * (bit-identical float scores, = mrfg_cc_map); 32 = the fused FP32
 * simulate-and-correlate row kernel (K1 OUT 3: |score - reference| ~1e-5,
 * about 1000x the FP64 throughput). */
int mrfg_cc_map_ex(mrfg_ctx* ctx, const mrfg_grid* grid, const double* query, int64_t first,
                   int64_t count, int precision, float* out);

/* -------------------------------------------------------- .mrfd / .mrfc files
 * Layout (README.md:160-170, dictionary.cpp:62-112): little-endian magic
 * "MRFD"/"MRFC", u32 version 1, 32-byte schedule digest (SHA-256 of the
 * schedule CSV, dictionary.cpp:163-171 -- the caller supplies it), three axes
 * as (f64 min, f64 step, u64 count), u64 entry length, then the payload:
 * float32 (re, im) unit entries (MRFD) or float32 scores (MRFC) in flat order.
 * I/O failures -> MRFG_E_RUNTIME (std::runtime_error in the reference). */
/* save_generated (dictionary.hpp:94-96, dictionary.cpp:216-239): streams the
 * GPU-generated dictionary to `path` (device generation overlaps the disk
 * writes); precision 64 = bit-identical entries.  The payload does not depend
 * on chunk_entries (> 0 required, as in the reference). */
int mrfg_save_generated(mrfg_ctx* ctx, const mrfg_grid* grid, const uint8_t* digest,
                        const char* path, int64_t chunk_entries, int precision);
/* cc_map_to_file (dictionary.hpp:130-132, dictionary.cpp:333-347): the whole
 * lattice's cc_map as an .mrfc file (entry length = schedule length). */
int mrfg_cc_map_to_file(mrfg_ctx* ctx, const mrfg_grid* grid, const double* query,
                        const uint8_t* digest, const char* path, int precision);
/* write_header (dictionary.cpp:72-82): creates/truncates `path`; the caller
 * appends the payload (save, dictionary.cpp:196-203). */
int mrfg_write_header(const char* path, const char* magic, const mrfg_grid* grid,
                      const uint8_t* digest, int64_t entry_len);
/* read_header (dictionary.cpp:90-112) with its errors (bad magic, version,
 * truncated header, degenerate dimensions); *payload_offset = header bytes. */
int mrfg_read_header(const char* path, const char* magic, mrfg_grid* grid, uint8_t* digest,
                     int64_t* entry_len, int64_t* payload_offset);

/* ---------------------------------------------------------------- noise
 * Host restatements (fingerprint.cpp:80-145): calibrate_noise
 * (fingerprint.hpp:45-50), make_calibrated_noise (:52-61), smooth (:63-66).
 * fp/out: n interleaved complex samples. */
int mrfg_calibrate_noise(const double* fp, int64_t n, double target_cc, uint64_t seed,
                         double* sigma);
int mrfg_make_calibrated_noise(const double* fp, int64_t n, double target_cc, uint64_t seed,
                               double* sigma, uint64_t* seed_used, double* noisy);
int mrfg_smooth(const double* fp, int64_t n, int k, double* out);

/* ----------------------------------------------------------- K5 MRF-ZOOM
 * quantify_impl per voxel (zoom.cpp:416-523) on a lattice (the finest
 * search pitch, zoom.hpp:17-21).  mrfg_quantify: independent voxels with full
 * bounds (quantify, zoom.cpp:533-539; quantify_slice without priors,
 * zoom.cpp:616-624).  mrfg_quantify_slice adds the neighbour-prior raster mode
 * (zoom.cpp:589-615) when use_prior != 0. */
int mrfg_quantify(mrfg_ctx* ctx, const mrfg_grid* lattice, const mrfg_zoom_config* cfg,
                  const double* fps, int64_t nvox, mrfg_quant* out);
/* use_prior: 0 = independent voxels (zoom.cpp:616-624); 1 = the reference's
 * strict raster order, each voxel seeded and windowed by the previous masked
 * voxel (zoom.cpp:589-615; one voxel in flight, exact); 2 = the row-wavefront
 * relaxation SPEC.md:449 permits (rows in parallel, a row's first voxel takes
 * its prior from the first masked voxel of the nearest row above). */
int mrfg_quantify_slice(mrfg_ctx* ctx, const mrfg_grid* lattice, const mrfg_zoom_config* cfg,
                        const double* fps, const uint8_t* mask, int nx, int ny, int use_prior,
                        mrfg_quant* out, double* seconds);
/* mrfg_quantify_bounded / mrfg_quantify_slice with dictionary payloads and
 * the stage trace (mrfg_zoom_io, may be NULL).  In the slice form with
 * use_prior = 1 the strict raster runs as ONE launch (the voxel chain on one
 * SM, every warp of the block evaluating the running voxel's rounds). */
int mrfg_quantify_ex(mrfg_ctx* ctx, const mrfg_grid* lattice, const mrfg_zoom_config* cfg,
                     const double* fps, int64_t nvox, const int64_t* bounds, const double* init_ms,
                     const mrfg_zoom_io* io, mrfg_quant* out);
int mrfg_quantify_slice_ex(mrfg_ctx* ctx, const mrfg_grid* lattice, const mrfg_zoom_config* cfg,
                           const double* fps, const uint8_t* mask, int nx, int ny, int use_prior,
                           const mrfg_zoom_io* io, mrfg_quant* out, double* seconds);
/* Four-parameter MRF-ZOOM (BASELINE configs[4]; the reference has no B1
 * axis, fingerprint.hpp:12-17).  ctxs[ib] is a context of the schedule whose
 * excitation flips are scaled by the ib-th B1 value (same device, same
 * length).  Per voxel: an outer zoom_1d (zoom.cpp:252-282) over the B1
 * index -- steps in index units, coarse to fine, from init_ib -- whose
 * objective is the score of the three-parameter quantify (K5) under
 * ctxs[ib], memoized per voxel and B1 value.  Each round of the outer walks
 * is ONE K5 launch over every (voxel, B1) pair the walks need, each voxel with
 * its B1 schedule's RF rows (the E1/E2/phasor tables do not depend on B1);
 * the flanks a walk may probe next are evaluated speculatively and only the
 * probes the walk takes count.  At most 16 B1 values.  out: quantify's result at the
 * chosen B1 with evaluations summed over the B1 values the walk acquired;
 * ib_out: the chosen index.  The oracle is oracle_api.h orc_quantify_b1. */
int mrfg_quantify_b1(mrfg_ctx* const* ctxs, int nb, const mrfg_grid* lattice, const mrfg_zoom_config* cfg,
                     const int64_t* steps, int nsteps, int64_t init_ib, const double* fps, int64_t nvox,
                     mrfg_quant* out, int64_t* ib_out);
/* mrfg_quantify on device-resident fingerprints (nvox x 2N FP64) and results
 * (async on the ctx stream; t1_ms/t2_ms/df_hz of d_out are left 0 -- the
 * lattice indices are filled). */
int mrfg_quantify_dev(mrfg_ctx* ctx, const mrfg_grid* lattice, const mrfg_zoom_config* cfg,
                      const double* d_fps, int64_t nvox, mrfg_quant* d_out);
/* quantify_impl with explicit per-voxel lattice bounds (lo1,hi1,lo2,hi2,lodf,hidf)
 * and initial T1/T2 [ms] (zoom.cpp:416-429); either array may be NULL (full
 * bounds / cfg->init_*). */
int mrfg_quantify_bounded(mrfg_ctx* ctx, const mrfg_grid* lattice, const mrfg_zoom_config* cfg,
                          const double* fps, int64_t nvox, const int64_t* bounds,
                          const double* init_ms, mrfg_quant* out);

#ifdef __cplusplus
}
#endif
#endif
