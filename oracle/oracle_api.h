/*
 * oracle_api.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Common C API of the two CPU oracles used by tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs:
 *
 *   oracle/liboracle.so     plain-C restatement of the reference algorithm
 *                           (oracle/mrf_oracle.c; every function cites the
 *                           reference file:line it follows);
 *   oracle/_ref/libmrf_ref.so  the reference library itself, compiled from
 *                           /root/reference/proj/src by oracle/Makefile and
 *                           wrapped by oracle/ref_capi.cpp.
 *
 * Nothing in the product (paper_1506_05393_b200/) links or calls this.
 * Units follow the reference: schedules in deg/ms (sequence.hpp:14-24),
 * lattices in ms/ms/Hz (dictionary.hpp:17-56), tissue params in s/s/Hz
 * (fingerprint.hpp:12-17).  Complex vectors are interleaved (re, im) doubles.
 */
#ifndef MRF_ORACLE_API_H
#define MRF_ORACLE_API_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct { double min, step; int64_t count; } orc_axis;           /* AxisSpec */
typedef struct { orc_axis t1_ms, t2_ms, df_hz; } orc_grid;                /* ParameterGrid */
typedef struct {
    int64_t n;
    const double *flip_deg, *phase_deg, *tr_ms, *te_ms;
} orc_sched;                                                             /* Schedule */

/* ZoomConfig (zoom.hpp:23-52) as a POD; step lists hold up to 8 entries. */
typedef struct {
    int32_t metric, final_metric, smooth_k, n2d, n1d;
    int32_t dict_mode; /* 0 none, 1 df dictionary (stage 1), 2 full dictionary (zoom.cpp:94-123) */
    double omega_hz, df_coarse_hz, df_refine_hz, df_window_hz, plateau_eps, heavy_noise_cc,
        fallback_coarse_hz, fallback_window_hz;
    double t1t2_2d_steps_ms[8];
    double t1t2_1d_steps_ms[8];
    double final_2d_step_ms, init_t1_ms, init_t2_ms, prior_window_t1_ms, prior_window_t2_ms,
        prior_window_df_hz;
} orc_zoom_cfg;

/* QuantResult (zoom.hpp:61-67) plus the lattice indices. */
typedef struct {
    int64_t i1, i2, idf;
    double t1_ms, t2_ms, df_hz, pd, score;
    int64_t evaluations;
} orc_quant;

/* 0 = ok; otherwise a negative code and orc_last_error() explains. */
const char* orc_last_error(void);
const char* orc_impl_name(void); /* "restatement" or "reference" */

int orc_build_schedule(int64_t n, uint64_t seed, double* flip_deg, double* phase_deg,
                       double* tr_ms, double* te_ms);
int orc_baseline_schedule(int64_t n, uint64_t seed, double* flip_deg, double* phase_deg,
                          double* tr_ms, double* te_ms);
int orc_simulate(const orc_sched* s, double t1_s, double t2_s, double df_hz, double* out);
int orc_add_noise(const double* fp, int64_t n, double sigma, uint64_t seed, double* out);
double orc_cc(const double* a, const double* b, int64_t n);
/* cc(normalize(a), normalize(b)): both unit-flagged, no denominator
 * (fingerprint.cpp:39-55 with unit_norm set by normalize, :28-37). */
double orc_cc_unit(const double* a, const double* b, int64_t n);
int orc_generate(const orc_sched* s, const orc_grid* g, int64_t first, int64_t count,
                 float* out);
/* scan_grid: per-query lowest-flat argmax.  second_score (may be NULL) is the
 * best score over all other flats (restatement only; the reference wrapper
 * writes NaN). */
int orc_scan_grid(const orc_sched* s, const orc_grid* g, const double* queries, int64_t nq,
                  int metric, int threads, int64_t* best_flat, double* best_score,
                  double* second_score);
/* scan_grid with Fingerprint::unit_norm flags (unit may be NULL): flagged
 * queries are used as given (prep_query, dictionary.cpp:145-150). */
int orc_scan_grid_ex(const orc_sched* s, const orc_grid* g, const double* queries, const uint8_t* unit,
                     int64_t nq, int metric, int threads, int64_t* best_flat, double* best_score,
                     double* second_score);
/* fingerprint.cpp:80-145: calibrate_noise, make_calibrated_noise, smooth. */
int orc_calibrate_noise(const double* fp, int64_t n, double target, uint64_t seed, double* sigma);
int orc_make_calibrated_noise(const double* fp, int64_t n, double target, uint64_t seed,
                              double* sigma, uint64_t* seed_used, double* noisy);
int orc_smooth(const double* fp, int64_t n, int k, double* out);
/* Reference library only (oracle/_ref): the file writers of dictionary.cpp. */
int orc_ref_save_generated(const orc_sched* s, const orc_grid* g, const char* path);
int orc_ref_cc_map_to_file(const orc_sched* s, const orc_grid* g, const double* fp,
                           const char* path);
/* Reference library only: exhaustive argmax over T1 values x T2 values x a
 * linear df axis, built from mrf::generate rows and mrf::brute_force_search
 * (see ref_capi.cpp).  Flat order (i1*n2 + i2)*ndf + idf; lowest flat on ties. */
int orc_ref_scan_rows(const orc_sched* s, const double* t1_ms, int64_t n1, const double* t2_ms,
                      int64_t n2, const orc_axis* df, const double* queries, int64_t nq,
                      int metric, int threads, int64_t* best_flat, double* best_score);
int orc_quantify(const orc_sched* s, const orc_grid* lattice, const orc_zoom_cfg* cfg,
                 const double* fp, orc_quant* out);
int orc_quantify_slice(const orc_sched* s, const orc_grid* lattice, const orc_zoom_cfg* cfg,
                       const double* fps, const uint8_t* mask, int nx, int ny, int use_prior,
                       int threads, orc_quant* out);

/* StageLog (zoom.hpp:54-59): one record per stage note of quantify_impl
 * (zoom.cpp:441-451 log_stage; search_df's notes, zoom.cpp:179-249).  Stage
 * names map to codes in this order (the same as mrfg.h's MRFG_STAGE_*). */
enum {
    ORC_STAGE_DF_COARSE, ORC_STAGE_DF_REFINE, ORC_STAGE_DF_TRANSLATE, ORC_STAGE_DF_REREFINE,
    ORC_STAGE_DF_PLATEAU_STOP, ORC_STAGE_DF_FINEST, ORC_STAGE_DF_FALLBACK, ORC_STAGE_T1T2_2D,
    ORC_STAGE_DF_SWEEP, ORC_STAGE_T1_1D, ORC_STAGE_T2_1D, ORC_STAGE_T1T2_FINAL
};
typedef struct {
    int32_t stage, pad;
    int64_t evaluations; /* unique evaluations this stage added */
    double best;
    double t1_ms, t2_ms, df_hz;
} orc_stage;

/* quantify (zoom.cpp:533-539) with an explicit dictionary payload and the
 * stage trace.  dict: NULL (cfg->dict_mode 1/2 then use the dictionary
 * generate() / make_df_dictionary() would build) or dict_entries x 2N float
 * (re, im) entries: the df slab (dict_mode 1; entry idf) or the full lattice
 * dictionary (dict_mode 2; flat order).  trace: trace_cap records or NULL. */
int orc_quantify_ex(const orc_sched* s, const orc_grid* lattice, const orc_zoom_cfg* cfg,
                    const double* fp, const float* dict, int64_t dict_entries, orc_stage* trace,
                    int trace_cap, int* trace_len, orc_quant* out);

/* Four-parameter MRF-ZOOM (BASELINE configs[4]; no reference counterpart --
 * the reference has no B1 axis, fingerprint.hpp:12-17).  B1 scales every
 * excitation flip (scheds[ib] = the schedule with flip_deg * b1[ib]; the
 * inversion stays ideal).  Parameter-separable extension of the reference's
 * search: an OUTER zoom_1d (zoom.cpp:252-282) over the B1 index, whose
 * objective g(ib) is the score of the reference's own three-parameter
 * quantify (zoom.cpp:533-539) under scheds[ib], memoized per ib; steps are
 * B1-index units (coarse to fine), init_ib the starting index.  The answer
 * is quantify's result at the chosen ib; evaluations = the inner unique
 * evaluations summed over the B1 values acquired. */
int orc_quantify_b1(const orc_sched* scheds, int nb, const orc_grid* lattice, const orc_zoom_cfg* cfg,
                    const int64_t* steps, int nsteps, int64_t init_ib, const double* fp, orc_quant* out,
                    int64_t* ib_out);

#ifdef __cplusplus
}
#endif
#endif
