/*
 * mrf_oracle.c -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * Plain-C restatement of the reference MRF dictionary generating-and-searching
 * path (arxiv 1506.05393 reference, /root/reference/proj).  Every function
 * cites the reference file:line it restates; floating-point expression order
 * follows the reference so that, compiled without FMA contraction (see
 * oracle/Makefile: -ffp-contract=off, default x86-64 ISA), results are
 * bit-identical to the reference library.  tests/test_oracle.py pins this
 * restatement against the reference library (oracle/_ref) and against the
 * reference's recorded runs (tests/golden/).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU legs load this.
 */
#define _GNU_SOURCE
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "oracle_api.h"

static __thread char g_err[256];
static int fail(const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return -1;
}
const char* orc_last_error(void) { return g_err; }
const char* orc_impl_name(void) { return "restatement"; }

/* ---------------------------------------------------------------- rng.hpp */
/* proj/include/mrf/rng.hpp:13-22 */
static const uint64_t kGolden = 0x9E3779B97F4A7C15ull;
static uint64_t mix64(uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}
/* rng.hpp:24-27 */
static uint64_t rng_at(uint64_t seed, uint64_t stream, uint64_t index) {
    uint64_t s = mix64(seed + kGolden * (stream + 1));
    return mix64(s + kGolden * (index + 1));
}
/* rng.hpp:30-32 */
static double uniform01(uint64_t seed, uint64_t stream, uint64_t index) {
    return (double)(rng_at(seed, stream, index) >> 11) * 0x1.0p-53;
}
/* rng.hpp:36-41 */
static double gaussian(uint64_t seed, uint64_t stream, uint64_t index) {
    double u1 = uniform01(seed, stream, 2 * index);
    double u2 = uniform01(seed, stream, 2 * index + 1);
    double r = sqrt(-2.0 * log1p(-u1));
    return r * cos(6.283185307179586476925286766559 * u2);
}

/* --------------------------------------------------------------- util.hpp */
/* util.hpp:19-23 */
static double quantize9(double x) {
    char buf[40];
    snprintf(buf, sizeof buf, "%.9g", x);
    return strtod(buf, NULL);
}

/* ----------------------------------------------------------- sequence.cpp */
static const double kDeg2Rad = 0.017453292519943295;
/* sequence.cpp:17-20 */
static double lattice_grad(uint64_t seed, int64_t i) {
    return 2.0 * uniform01(seed, 1, (uint64_t)i) - 1.0;
}
/* sequence.cpp:23-32 */
static double perlin1d(uint64_t seed, double x) {
    double fx = floor(x);
    int64_t i0 = (int64_t)fx;
    double t = x - fx;
    double n0 = lattice_grad(seed, i0) * t;
    double n1 = lattice_grad(seed, i0 + 1) * (t - 1.0);
    double u = t * t * t * (t * (6.0 * t - 15.0) + 10.0);
    return n0 + u * (n1 - n0);
}
/* sequence.cpp:36-50 */
static void remap(double* v, int64_t n, double lo, double hi) {
    if (n == 0) return;
    double mn = v[0], mx = v[0];
    for (int64_t i = 0; i < n; ++i) {
        mn = v[i] < mn ? v[i] : mn;
        mx = v[i] > mx ? v[i] : mx;
    }
    if (mx == mn) {
        for (int64_t i = 0; i < n; ++i) v[i] = lo;
        return;
    }
    double scale = (hi - lo) / (mx - mn);
    for (int64_t i = 0; i < n; ++i) v[i] = lo + (v[i] - mn) * scale;
}

/* sequence.cpp:52-92: perlin flips, 0/90/180/90 phases, remapped-gaussian TRs. */
int orc_build_schedule(int64_t n, uint64_t seed, double* flip_deg, double* phase_deg,
                       double* tr_ms, double* te_ms) {
    double* flips = malloc(sizeof(double) * (size_t)(n ? n : 1));
    double* trs = malloc(sizeof(double) * (size_t)(n ? n : 1));
    for (int64_t k = 0; k < n; ++k) flips[k] = perlin1d(seed, (double)k / 16.0);
    remap(flips, n, 0.0, 79.0 * kDeg2Rad);
    for (int64_t k = 0; k < n; ++k) trs[k] = gaussian(seed, 2, (uint64_t)k);
    remap(trs, n, 0.0, 6e-3);
    for (int64_t k = 0; k < n; ++k) trs[k] += 14e-3;
    const double cycle[4] = {0.0, 90.0 * kDeg2Rad, 180.0 * kDeg2Rad, 90.0 * kDeg2Rad};
    for (int64_t k = 0; k < n; ++k) {
        flip_deg[k] = quantize9(flips[k] / kDeg2Rad);
        phase_deg[k] = quantize9(cycle[k % 4] / kDeg2Rad);
        tr_ms[k] = quantize9(trs[k] * 1e3);
        te_ms[k] = quantize9(trs[k] * 1e3 / 2.0);
    }
    free(flips);
    free(trs);
    return 0;
}

/* BASELINE.json schedule generator; not in the reference,
 * which ingests it through load_schedule_csv (sequence.cpp:112-140). */
int orc_baseline_schedule(int64_t n, uint64_t seed, double* flip_deg, double* phase_deg,
                          double* tr_ms, double* te_ms) {
    for (int64_t j = 0; j < n; ++j) {
        double fa = 10.0 + 50.0 * fabs(sin(2.0 * M_PI * (double)j / 250.0)) +
                    2.0 * gaussian(seed, 1, (uint64_t)j);
        double tr = quantize9(10.5 + 3.5 * uniform01(seed, 2, (uint64_t)j));
        flip_deg[j] = quantize9(fa);
        phase_deg[j] = (j % 2) ? 180.0 : 0.0;
        tr_ms[j] = tr;
        te_ms[j] = quantize9(tr / 2.0);
    }
    return 0;
}

/* -------------------------------------------------------------- bloch.cpp */
typedef struct { double m[9]; } M3;
typedef struct { double x, y, z; } V3;

/* bloch.hpp:25-32: row-major product, left-to-right sums. */
static M3 m3_mul(const M3* a, const M3* o) {
    M3 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            r.m[3 * i + j] = a->m[3 * i] * o->m[j] + a->m[3 * i + 1] * o->m[3 + j] +
                             a->m[3 * i + 2] * o->m[6 + j];
    return r;
}
/* bloch.hpp:34-38 */
static V3 m3_apply(const M3* a, V3 v) {
    V3 r = {a->m[0] * v.x + a->m[1] * v.y + a->m[2] * v.z,
            a->m[3] * v.x + a->m[4] * v.y + a->m[5] * v.z,
            a->m[6] * v.x + a->m[7] * v.y + a->m[8] * v.z};
    return r;
}
/* bloch.cpp:31-53 (axis 0=X, 2=Z) */
static M3 rot(int axis, double theta) {
    double c = cos(theta), s = sin(theta);
    M3 r = {{1, 0, 0, 0, 1, 0, 0, 0, 1}};
    if (axis == 0) {
        double t[9] = {1, 0, 0, 0, c, -s, 0, s, c};
        memcpy(r.m, t, sizeof t);
    } else if (axis == 1) {
        double t[9] = {c, 0, s, 0, 1, 0, -s, 0, c};
        memcpy(r.m, t, sizeof t);
    } else {
        double t[9] = {c, -s, 0, s, c, 0, 0, 0, 1};
        memcpy(r.m, t, sizeof t);
    }
    return r;
}
/* bloch.cpp:63-66: simplified model Rz(phi) Rx(-alpha) Rz(-phi), left-assoc. */
static M3 rf_matrix(double alpha, double phi) {
    M3 a = rot(2, phi), b = rot(0, -alpha), c = rot(2, -phi);
    M3 ab = m3_mul(&a, &b);
    return m3_mul(&ab, &c);
}
/* bloch.cpp:15-27 */
static void relax_precess(V3* m, double dt, double inv_t1, double inv_t2, double df) {
    const double kTwoPi = 6.283185307179586476925286766559;
    double e2 = exp(-dt * inv_t2);
    double e1 = exp(-dt * inv_t1);
    double a = kTwoPi * df * dt;
    double c = cos(a);
    double s = sin(a);
    double x = (m->x * c - m->y * s) * e2;
    double y = (m->x * s + m->y * c) * e2;
    m->x = x;
    m->y = y;
    m->z = 1.0 + (m->z - 1.0) * e1;
}

typedef struct {
    int64_t n;
    M3* rf;
    double *te, *rest;
} Sim;

/* bloch.cpp:95-106 (BlochSimulator constructor). */
static int sim_init(Sim* sim, const orc_sched* s) {
    sim->n = s->n;
    sim->rf = malloc(sizeof(M3) * (size_t)(s->n ? s->n : 1));
    sim->te = malloc(sizeof(double) * (size_t)(s->n ? s->n : 1));
    sim->rest = malloc(sizeof(double) * (size_t)(s->n ? s->n : 1));
    for (int64_t i = 0; i < s->n; ++i) {
        if (s->te_ms[i] < 0 || s->te_ms[i] > s->tr_ms[i])
            return fail("BlochSimulator: schedule needs 0 <= te <= tr");
        sim->rf[i] = rf_matrix(s->flip_deg[i] * 0.017453292519943295,
                               s->phase_deg[i] * 0.017453292519943295);
        sim->te[i] = s->te_ms[i] * 1e-3;
        sim->rest[i] = s->tr_ms[i] * 1e-3 - s->te_ms[i] * 1e-3;
    }
    return 0;
}
static void sim_free(Sim* sim) {
    free(sim->rf);
    free(sim->te);
    free(sim->rest);
}
/* bloch.cpp:108-123 (BlochSimulator::simulate). */
static void sim_run(const Sim* sim, double t1, double t2, double df, double* out) {
    double inv_t1 = 1.0 / t1;
    double inv_t2 = 1.0 / t2;
    M3 inv = rf_matrix(3.14159265358979323846, 0);
    V3 m = {0, 0, 1};
    m = m3_apply(&inv, m);
    for (int64_t i = 0; i < sim->n; ++i) {
        m = m3_apply(&sim->rf[i], m);
        relax_precess(&m, sim->te[i], inv_t1, inv_t2, df);
        out[2 * i] = m.x;
        out[2 * i + 1] = m.y;
        relax_precess(&m, sim->rest[i], inv_t1, inv_t2, df);
    }
}

int orc_simulate(const orc_sched* s, double t1_s, double t2_s, double df_hz, double* out) {
    if (t1_s <= 0 || t2_s <= 0) return fail("simulate: T1 and T2 must be positive");
    Sim sim;
    int rc = sim_init(&sim, s);
    if (rc == 0) sim_run(&sim, t1_s, t2_s, df_hz, out);
    sim_free(&sim);
    return rc;
}

/* -------------------------------------------------------- fingerprint.cpp */
/* fingerprint.cpp:14-18 */
static double norm2(const double* v, int64_t n) {
    double acc = 0;
    for (int64_t j = 0; j < n; ++j) acc += v[2 * j] * v[2 * j] + v[2 * j + 1] * v[2 * j + 1];
    return sqrt(acc);
}
/* fingerprint.cpp:28-37 */
static int normalize(const double* v, int64_t n, double* out) {
    double nn = norm2(v, n);
    if (nn == 0) return fail("normalize: zero fingerprint");
    double inv = 1.0 / nn;
    for (int64_t j = 0; j < n; ++j) {
        out[2 * j] = v[2 * j] * inv;
        out[2 * j + 1] = v[2 * j + 1] * inv;
    }
    return 0;
}
/* fingerprint.cpp:39-55 (neither input flagged unit-norm) */
double orc_cc(const double* a, const double* b, int64_t n) {
    double re = 0, im = 0;
    for (int64_t j = 0; j < n; ++j) {
        re += a[2 * j] * b[2 * j] + a[2 * j + 1] * b[2 * j + 1];
        im += a[2 * j + 1] * b[2 * j] - a[2 * j] * b[2 * j + 1];
    }
    double num = sqrt(re * re + im * im);
    double na = norm2(a, n), nb = norm2(b, n);
    if (na == 0 || nb == 0) return NAN;
    num /= na * nb;
    return num < 1.0 ? num : 1.0;
}
double orc_cc_unit(const double* a, const double* b, int64_t n) {
    double* na = malloc(sizeof(double) * 2 * (size_t)n);
    double* nb = malloc(sizeof(double) * 2 * (size_t)n);
    double out = NAN;
    if (normalize(a, n, na) == 0 && normalize(b, n, nb) == 0) {
        double re = 0, im = 0;
        for (int64_t j = 0; j < n; ++j) {
            re += na[2 * j] * nb[2 * j] + na[2 * j + 1] * nb[2 * j + 1];
            im += na[2 * j + 1] * nb[2 * j] - na[2 * j] * nb[2 * j + 1];
        }
        double num = sqrt(re * re + im * im);
        out = num < 1.0 ? num : 1.0;
    }
    free(na);
    free(nb);
    return out;
}

/* fingerprint.cpp:68-78 */
int orc_add_noise(const double* fp, int64_t n, double sigma, uint64_t seed, double* out) {
    if (sigma < 0) return fail("add_noise: sigma must be >= 0");
    for (int64_t j = 0; j < n; ++j) {
        double nr = gaussian(seed, 3, 2 * (uint64_t)j);
        double ni = gaussian(seed, 3, 2 * (uint64_t)j + 1);
        out[2 * j] = fp[2 * j] + sigma * nr;
        out[2 * j + 1] = fp[2 * j + 1] + sigma * ni;
    }
    return 0;
}
/* fingerprint.cpp:122-145 */
static void smooth(const double* v, int64_t n, int k, double* out) {
    double sigma = (k == 3) ? 0.85 : 1.0;
    int h = k / 2;
    double w[5];
    for (int j = -h; j <= h; ++j) w[j + h] = exp(-0.5 * j * j / (sigma * sigma));
    for (int64_t i = 0; i < n; ++i) {
        double re = 0, im = 0, wsum = 0;
        for (int j = -h; j <= h; ++j) {
            int64_t t = i + j;
            if (t < 0 || t >= n) continue;
            re += w[j + h] * v[2 * t];
            im += w[j + h] * v[2 * t + 1];
            wsum += w[j + h];
        }
        out[2 * i] = re / wsum;
        out[2 * i + 1] = im / wsum;
    }
}

int orc_smooth(const double* fp, int64_t n, int k, double* out) {
    if (k != 3 && k != 5) return fail("smooth: kernel must be 3 or 5");
    if (n == 0) return fail("smooth: empty input");
    smooth(fp, n, k, out);
    return 0;
}
/* fingerprint.cpp:80-105.  Returns 0 (sigma set), -1 invalid argument,
 * -3 (runtime: cannot bracket / no sigma in 60 steps). */
static int calibrate(const double* fp, int64_t n, double target, uint64_t seed, double* sigma) {
    if (!(target > 0 && target < 1)) return fail("calibrate_noise: target must be in (0,1)");
    double* noisy = malloc(sizeof(double) * 2 * (size_t)n);
    int rc = -3;
    double lo = 0, hi = norm2(fp, n) / sqrt((double)n);
    orc_add_noise(fp, n, hi, seed, noisy);
    double c = orc_cc(fp, noisy, n);
    int done = 0;
    for (int i = 0; i < 80 && c > target; ++i) {
        if (fabs(c - target) <= 0.02) { *sigma = hi; rc = 0; done = 1; break; }
        hi *= 2;
        orc_add_noise(fp, n, hi, seed, noisy);
        c = orc_cc(fp, noisy, n);
    }
    if (!done && c > target) {
        fail("calibrate_noise: cannot bracket target");
        done = 1;
        rc = -3;
    }
    for (int i = 0; !done && i < 60; ++i) {
        double mid = 0.5 * (lo + hi);
        orc_add_noise(fp, n, mid, seed, noisy);
        double cm = orc_cc(fp, noisy, n);
        if (fabs(cm - target) <= 0.02) { *sigma = mid; rc = 0; done = 1; break; }
        if (cm > target) lo = mid; else hi = mid;
    }
    if (!done) fail("calibrate_noise: no sigma within tolerance after 60 steps");
    free(noisy);
    return rc;
}
int orc_calibrate_noise(const double* fp, int64_t n, double target, uint64_t seed, double* sigma) {
    return calibrate(fp, n, target, seed, sigma);
}
/* fingerprint.cpp:107-120 */
int orc_make_calibrated_noise(const double* fp, int64_t n, double target, uint64_t seed,
                              double* sigma, uint64_t* seed_used, double* noisy) {
    for (int attempt = 0;; ++attempt) {
        uint64_t s = attempt == 0 ? seed : rng_at(seed, 99, (uint64_t)attempt);
        int rc = calibrate(fp, n, target, s, sigma);
        if (rc == 0) {
            *seed_used = s;
            return orc_add_noise(fp, n, *sigma, s, noisy);
        }
        if (rc != -3 || attempt >= 7) return rc;
    }
}

/* --------------------------------------------------------- dictionary.cpp */
/* dictionary.hpp:22, 51-56: value(k) = min + k*step; params_at converts ms->s. */
static double axis_value(const orc_axis* a, int64_t k) { return a->min + (double)k * a->step; }

/* dictionary.cpp:37-53: simulate, FP64 normalize, quantize to float32. */
static void entry_f32(const Sim* sim, const orc_grid* g, int64_t flat, double* buf, float* dst) {
    int64_t ndf = g->df_hz.count, n2 = g->t2_ms.count;
    int64_t idf = flat % ndf, rest = flat / ndf;
    int64_t i1 = rest / n2, i2 = rest % n2;
    sim_run(sim, axis_value(&g->t1_ms, i1) * 1e-3, axis_value(&g->t2_ms, i2) * 1e-3,
            axis_value(&g->df_hz, idf), buf);
    double acc = 0;
    for (int64_t j = 0; j < sim->n; ++j)
        acc += buf[2 * j] * buf[2 * j] + buf[2 * j + 1] * buf[2 * j + 1];
    double inv = 1.0 / sqrt(acc);
    for (int64_t j = 0; j < sim->n; ++j) {
        dst[2 * j] = (float)(buf[2 * j] * inv);
        dst[2 * j + 1] = (float)(buf[2 * j + 1] * inv);
    }
}

int orc_generate(const orc_sched* s, const orc_grid* g, int64_t first, int64_t count,
                 float* out) {
    Sim sim;
    if (sim_init(&sim, s)) {
        sim_free(&sim);
        return -1;
    }
#pragma omp parallel
    {
        double* buf = malloc(sizeof(double) * 2 * (size_t)s->n);
#pragma omp for schedule(static)
        for (int64_t k = 0; k < count; ++k) entry_f32(&sim, g, first + k, buf, out + k * 2 * s->n);
        free(buf);
    }
    sim_free(&sim);
    return 0;
}

/* dictionary.cpp:117-127 */
static double cc_against_entry(const double* q, const float* e, int64_t n) {
    double re = 0, im = 0;
    for (int64_t j = 0; j < n; ++j) {
        double er = e[2 * j], ei = e[2 * j + 1];
        re += q[2 * j] * er + q[2 * j + 1] * ei;
        im += q[2 * j + 1] * er - q[2 * j] * ei;
    }
    double v = sqrt(re * re + im * im);
    return v < 1.0 ? v : 1.0;
}
/* dictionary.cpp:129-138 */
static double dist_against_entry(const double* q, const float* e, int64_t n) {
    double acc = 0;
    for (int64_t j = 0; j < n; ++j) {
        double dr = q[2 * j] - e[2 * j];
        double di = q[2 * j + 1] - e[2 * j + 1];
        acc += dr * dr + di * di;
    }
    return sqrt(acc);
}

/* dictionary.cpp:257-308 (scan_grid), scored per dictionary.cpp:140-143 with
 * the strict '>' lowest-flat tie rule (:291-294).  Chunked generation keeps
 * memory bounded; queries are scanned in parallel (the reference scans them
 * serially, which changes nothing but time). */
int orc_scan_grid(const orc_sched* s, const orc_grid* g, const double* queries, int64_t nq,
                  int metric, int threads, int64_t* best_flat, double* best_score,
                  double* second_score) {
    return orc_scan_grid_ex(s, g, queries, NULL, nq, metric, threads, best_flat, best_score, second_score);
}

/* prep_query (dictionary.cpp:145-150): `fp.unit_norm ? fp : normalize(fp)`. */
int orc_scan_grid_ex(const orc_sched* s, const orc_grid* g, const double* queries, const uint8_t* unit,
                     int64_t nq, int metric, int threads, int64_t* best_flat, double* best_score,
                     double* second_score) {
    if (nq <= 0) return fail("scan_grid: no queries");
    Sim sim;
    if (sim_init(&sim, s)) {
        sim_free(&sim);
        return -1;
    }
    int64_t n = s->n;
    double* q = malloc(sizeof(double) * 2 * (size_t)(n * nq));
    for (int64_t iq = 0; iq < nq; ++iq) {
        if (unit && unit[iq]) {
            memcpy(q + iq * 2 * n, queries + iq * 2 * n, sizeof(double) * 2 * (size_t)n);
            continue;
        }
        if (normalize(queries + iq * 2 * n, n, q + iq * 2 * n)) {
            free(q);
            sim_free(&sim);
            return -1;
        }
    }
    double* best = malloc(sizeof(double) * (size_t)nq);
    double* second = malloc(sizeof(double) * (size_t)nq);
    for (int64_t iq = 0; iq < nq; ++iq) {
        best[iq] = -1e300;
        second[iq] = -1e300;
        best_flat[iq] = 0;
    }
    int64_t total = g->t1_ms.count * g->t2_ms.count * g->df_hz.count;
    const int64_t chunk = 4096;
    float* buf = malloc(sizeof(float) * 2 * (size_t)(n * chunk));
    if (threads < 1) threads = 1;
    for (int64_t begin = 0; begin < total; begin += chunk) {
        int64_t end = begin + chunk < total ? begin + chunk : total;
#pragma omp parallel num_threads(threads)
        {
            double* sbuf = malloc(sizeof(double) * 2 * (size_t)n);
#pragma omp for schedule(static)
            for (int64_t f = begin; f < end; ++f) entry_f32(&sim, g, f, sbuf, buf + (f - begin) * 2 * n);
            free(sbuf);
#pragma omp for schedule(static)
            for (int64_t iq = 0; iq < nq; ++iq) {
                const double* qq = q + iq * 2 * n;
                double b = best[iq], sc = second[iq];
                int64_t bf = best_flat[iq];
                for (int64_t f = begin; f < end; ++f) {
                    const float* e = buf + (f - begin) * 2 * n;
                    double v = metric == 0 ? cc_against_entry(qq, e, n) : -dist_against_entry(qq, e, n);
                    if (v > b) {
                        sc = b;
                        b = v;
                        bf = f;
                    } else if (v > sc) {
                        sc = v;
                    }
                }
                best[iq] = b;
                second[iq] = sc;
                best_flat[iq] = bf;
            }
        }
    }
    for (int64_t iq = 0; iq < nq; ++iq) {
        best_score[iq] = best[iq];
        if (second_score) second_score[iq] = second[iq];
    }
    free(buf);
    free(best);
    free(second);
    free(q);
    sim_free(&sim);
    return 0;
}

/* ---------------------------------------------------------------- zoom.cpp */
/* Objective (zoom.cpp:41-150): memo over lattice keys i1<<42|i2<<21|idf
 * (zoom.cpp:14-19); each unique key costs one FP64 simulation + normalize
 * (zoom.cpp:114-122); both metric scores are derived from the same entry, so
 * metric switches are free (zoom.cpp:94-138). */
typedef struct {
    uint64_t key;
    double cc, euc;
    int used;
} Slot;

typedef struct {
    const Sim* sim;
    const orc_grid* g;
    int smooth_k;
    int64_t n;
    double* query; /* normalized (smoothed) */
    double *buf, *buf2;
    Slot* tab;
    int64_t cap, size;
    int64_t evals;
    int err;
    int dict_mode; /* 0 none, 1 df dictionary during stage 1, 2 full dictionary */
    int in_stage1;
    double* buf3;
    const float* dict; /* caller's dictionary payload (NULL: the generated entries) */
} Obj;

static uint64_t key_of(int64_t i1, int64_t i2, int64_t idf) {
    return ((uint64_t)i1 << 42) | ((uint64_t)i2 << 21) | (uint64_t)idf;
}
static uint64_t hash64(uint64_t k) { return mix64(k + kGolden); }

static Slot* obj_find(Obj* o, uint64_t key) {
    uint64_t h = hash64(key) & (uint64_t)(o->cap - 1);
    for (;;) {
        Slot* sl = &o->tab[h];
        if (!sl->used || sl->key == key) return sl;
        h = (h + 1) & (uint64_t)(o->cap - 1);
    }
}
static void obj_grow(Obj* o) {
    Slot* old = o->tab;
    int64_t oc = o->cap;
    o->cap *= 2;
    o->tab = calloc((size_t)o->cap, sizeof(Slot));
    for (int64_t i = 0; i < oc; ++i)
        if (old[i].used) *obj_find(o, old[i].key) = old[i];
    free(old);
}

/* zoom.cpp:125-138 (eval), with acquire (zoom.cpp:94-123) and
 * score_from_entry (zoom.cpp:74-92). */
static double obj_eval(Obj* o, int64_t i1, int64_t i2, int64_t idf, int metric) {
    if (i1 < 0 || i2 < 0 || idf < 0 || i1 >= o->g->t1_ms.count || i2 >= o->g->t2_ms.count ||
        idf >= o->g->df_hz.count) {
        o->err = 1;
        fail("objective: lattice index out of range");
        return -1e300;
    }
    uint64_t key = key_of(i1, i2, idf);
    Slot* sl = obj_find(o, key);
    if (!sl->used) {
        int64_t n = o->n;
        sim_run(o->sim, axis_value(&o->g->t1_ms, i1) * 1e-3, axis_value(&o->g->t2_ms, i2) * 1e-3,
                axis_value(&o->g->df_hz, idf), o->buf);
        const double* e;
        if (o->dict_mode == 2 || (o->dict_mode == 1 && o->in_stage1)) {
            /* dictionary entry (zoom.cpp:101-110): d->entry(flat) with flat the
             * lattice flat (full dictionary) or idf (df slab), as given -- or,
             * without a payload, the generated float entry
             * float(normalize(simulate)) (dictionary.cpp:44-51); then, with
             * smoothing, normalize(smooth(entry)) */
            if (o->dict) {
                const int64_t flat = o->dict_mode == 2
                                         ? (i1 * o->g->t2_ms.count + i2) * o->g->df_hz.count + idf
                                         : idf;
                const float* raw = o->dict + flat * 2 * n;
                for (int64_t j = 0; j < 2 * n; ++j) o->buf3[j] = (double)raw[j];
            } else {
                normalize(o->buf, n, o->buf3);
                for (int64_t j = 0; j < 2 * n; ++j) o->buf3[j] = (double)(float)o->buf3[j];
            }
            if (o->smooth_k) {
                smooth(o->buf3, n, o->smooth_k, o->buf2);
                normalize(o->buf2, n, o->buf3);
            }
            e = o->buf3;
        } else {
            const double* src = o->buf;
            if (o->smooth_k) {
                smooth(o->buf, n, o->smooth_k, o->buf2);
                src = o->buf2;
            }
            normalize(src, n, o->buf);
            e = o->buf;
        }
        double re = 0, im = 0, acc = 0;
        for (int64_t j = 0; j < n; ++j) {
            re += o->query[2 * j] * e[2 * j] + o->query[2 * j + 1] * e[2 * j + 1];
            im += o->query[2 * j + 1] * e[2 * j] - o->query[2 * j] * e[2 * j + 1];
        }
        for (int64_t j = 0; j < n; ++j) {
            double dr = o->query[2 * j] - e[2 * j];
            double di = o->query[2 * j + 1] - e[2 * j + 1];
            acc += dr * dr + di * di;
        }
        double v = sqrt(re * re + im * im);
        sl->used = 1;
        sl->key = key;
        sl->cc = v < 1.0 ? v : 1.0;
        sl->euc = -sqrt(acc);
        o->evals++;
        if (++o->size * 2 > o->cap) {
            double cc = sl->cc, eu = sl->euc;
            obj_grow(o);
            sl = obj_find(o, key);
            (void)cc;
            (void)eu;
        }
    }
    return metric == 0 ? sl->cc : sl->euc;
}

/* zoom.cpp:160-169 */
typedef struct {
    int64_t idx;
    double val;
} Best;
static void offer(Best* b, int64_t i, double v) {
    if (v > b->val) {
        b->val = v;
        b->idx = i;
    }
}

typedef struct {
    int64_t coarse, refine, finest, window_half, omega;
    double plateau_eps, heavy_cc;
    int64_t fallback_coarse, fallback_window_half;
    int allow_fallback;
} DfParams; /* zoom.hpp:115-126 */

/* StageLog recording (zoom.cpp:441-451 log_stage): evaluations added since
 * the previous note, the stage's best value and its lattice point. */
typedef struct {
    orc_stage* out;
    int cap, n;
    int64_t last;
} Trace;
static void note(Trace* t, const Obj* o, int stage, int64_t i1, int64_t i2, int64_t idf, double best) {
    if (!t || !t->out) return;
    if (t->n < t->cap) {
        orc_stage* r = &t->out[t->n];
        r->stage = stage;
        r->pad = 0;
        r->evaluations = o->evals - t->last;
        r->best = best;
        r->t1_ms = axis_value(&o->g->t1_ms, i1);
        r->t2_ms = axis_value(&o->g->t2_ms, i2);
        r->df_hz = axis_value(&o->g->df_hz, idf);
    }
    t->n++;
    t->last = o->evals;
}

typedef struct {
    Obj* o;
    int64_t i1, i2;
    int metric;
    Trace* tr;
} DfCtx;
#define DF_NOTE(c, st, b) note((c)->tr, (c)->o, (st), (c)->i1, (c)->i2, (b).idx, (b).val)
static double f_df(DfCtx* c, int64_t idf) { return obj_eval(c->o, c->i1, c->i2, idf, c->metric); }

static int64_t clampl(int64_t v, int64_t lo, int64_t hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* zoom.cpp:182-187 */
static void df_scan(DfCtx* c, int64_t lo, int64_t hi, int64_t a, int64_t b, int64_t step, Best* bst) {
    a = clampl(a, lo, hi);
    b = clampl(b, lo, hi);
    for (int64_t x = a; x <= b; x += step) offer(bst, x, f_df(c, x));
    if ((b - a) % step != 0) offer(bst, b, f_df(c, b));
}

/* zoom.cpp:191-199 */
static int plateau(const double* marks, int nm, double eps) {
    if (nm < 3) return 0;
    double mn = marks[nm - 3], mx = mn;
    for (int j = nm - 3; j < nm; ++j) {
        mn = marks[j] < mn ? marks[j] : mn;
        mx = marks[j] > mx ? marks[j] : mx;
    }
    return mx - mn < eps;
}

/* zoom.cpp:189-241 (the `run` lambda) */
static Best df_run(DfCtx* c, int64_t lo, int64_t hi, const DfParams* p, int64_t coarse,
                   int64_t window_half) {
    double marks[16];
    int nm = 0;
    Best cur = {-1, -1e300};
    df_scan(c, lo, hi, lo, hi, coarse, &cur);
    DF_NOTE(c, ORC_STAGE_DF_COARSE, cur);
    marks[nm++] = cur.val;
    {
        Best r = cur;
        df_scan(c, lo, hi, cur.idx - window_half, cur.idx + window_half, p->refine, &r);
        cur = r;
    }
    DF_NOTE(c, ORC_STAGE_DF_REFINE, cur);
    marks[nm++] = cur.val;
    for (int round = 0; round < 8; ++round) {
        Best t = cur;
        for (int64_t k = 1; cur.idx + k * p->omega <= hi; ++k) {
            int64_t q = cur.idx + k * p->omega;
            offer(&t, q, f_df(c, q));
        }
        for (int64_t k = 1; cur.idx - k * p->omega >= lo; ++k) {
            int64_t q = cur.idx - k * p->omega;
            offer(&t, q, f_df(c, q));
        }
        DF_NOTE(c, ORC_STAGE_DF_TRANSLATE, t);
        if (t.idx == cur.idx) break;
        Best r = t;
        df_scan(c, lo, hi, t.idx - window_half, t.idx + window_half, p->refine, &r);
        cur = r;
        DF_NOTE(c, ORC_STAGE_DF_REREFINE, cur);
        marks[nm++] = cur.val;
        if (plateau(marks, nm, p->plateau_eps)) {
            DF_NOTE(c, ORC_STAGE_DF_PLATEAU_STOP, cur);
            return cur;
        }
    }
    if (plateau(marks, nm, p->plateau_eps)) {
        DF_NOTE(c, ORC_STAGE_DF_PLATEAU_STOP, cur);
        return cur;
    }
    Best fin = cur;
    df_scan(c, lo, hi, cur.idx - p->omega / 2, cur.idx + p->omega / 2, p->finest, &fin);
    DF_NOTE(c, ORC_STAGE_DF_FINEST, fin);
    return fin;
}

/* zoom.cpp:173-250 (search_df) */
static int64_t search_df(DfCtx* c, int64_t lo, int64_t hi, const DfParams* p) {
    Best mainb = df_run(c, lo, hi, p, p->coarse, p->window_half);
    if (p->allow_fallback && mainb.val < p->heavy_cc) {
        Best fb = df_run(c, lo, hi, p, p->fallback_coarse, p->fallback_window_half);
        DF_NOTE(c, ORC_STAGE_DF_FALLBACK, fb);
        if (fb.val > mainb.val) return fb.idx;
    }
    return mainb.idx;
}

/* 1-D objective along T1 (axis 0) or T2 (axis 1), zoom.cpp:494-499 */
typedef struct {
    Obj* o;
    int axis;
    int64_t i1, i2, idf;
    int metric;
} LineCtx;
static double f_line(LineCtx* c, int64_t a) {
    return c->axis == 0 ? obj_eval(c->o, a, c->i2, c->idf, c->metric)
                        : obj_eval(c->o, c->i1, a, c->idf, c->metric);
}

/* zoom.cpp:252-282 (zoom_1d) */
static int64_t zoom_1d(LineCtx* c, int64_t lo, int64_t hi, int64_t init, const int64_t* steps, int ns) {
    int64_t x = clampl(init, lo, hi);
    double fx = f_line(c, x);
    for (int si = 0; si < ns; ++si) {
        int64_t s = steps[si];
        for (;;) {
            int64_t xl = clampl(x - s, lo, hi);
            if (xl != x) {
                double fl = f_line(c, xl);
                if (fl > fx) {
                    x = xl;
                    fx = fl;
                    continue;
                }
            }
            int64_t xr = clampl(x + s, lo, hi);
            if (xr != x) {
                double fr = f_line(c, xr);
                if (fr > fx) {
                    x = xr;
                    fx = fr;
                    continue;
                }
            }
            break;
        }
    }
    return x;
}

/* zoom.cpp:284-399 (zoom_2d); f(a,b) = obj.eval(a, b, idf, metric). */
static void zoom_2d(Obj* o, int64_t idf, int metric, int64_t lo1, int64_t hi1, int64_t lo2,
                    int64_t hi2, int64_t* px, int64_t* py, const int64_t* s1v, const int64_t* s2v,
                    int ns) {
#define F2(a, b) obj_eval(o, (a), (b), idf, metric)
    int64_t x = clampl(*px, lo1, hi1);
    int64_t y = clampl(*py, lo2, hi2);
    double fc = F2(x, y);
    int64_t bx = x, by = y;
    double bf = fc;
#define NOTE(ax, ay, v)    \
    do {                   \
        if ((v) > bf) {    \
            bf = (v);      \
            bx = (ax);     \
            by = (ay);     \
        }                  \
    } while (0)
    for (int si = 0; si < ns; ++si) {
        int64_t s1 = s1v[si], s2 = s2v[si];
        int64_t cap = 4 * ((hi1 - lo1) / s1 + (hi2 - lo2) / s2) + 16;
        int converged = 0;
        for (int64_t iter = 0; iter < cap && !converged; ++iter) {
            int64_t xl = clampl(x - s1, lo1, hi1);
            int64_t xr = clampl(x + s1, lo1, hi1);
            int64_t yd = clampl(y - s2, lo2, hi2);
            int64_t yu = clampl(y + s2, lo2, hi2);
            double fl = fc, fd = fc;
            if (xl != x) {
                fl = F2(xl, y);
                NOTE(xl, y, fl);
            }
            if (yd != y) {
                fd = F2(x, yd);
                NOTE(x, yd, fd);
            }
            int lw = xl != x && fl > fc;
            int dw = yd != y && fd > fc;
            if (lw && dw) {
                x = xl;
                y = yd;
                fc = F2(x, y);
                NOTE(x, y, fc);
                continue;
            }
            if (!lw && !dw) {
                double fr = fc, fu = fc;
                if (xr != x) {
                    fr = F2(xr, y);
                    NOTE(xr, y, fr);
                }
                if (yu != y) {
                    fu = F2(x, yu);
                    NOTE(x, yu, fu);
                }
                int rw = xr != x && fr > fc;
                int uw = yu != y && fu > fc;
                if (rw && uw) {
                    x = xr;
                    y = yu;
                    fc = F2(x, y);
                    NOTE(x, y, fc);
                    continue;
                }
                if (rw) {
                    x = xr;
                    fc = fr;
                    continue;
                }
                if (uw) {
                    y = yu;
                    fc = fu;
                    continue;
                }
                converged = 1;
                continue;
            }
            if (lw) {
                double fu = fc;
                if (yu != y) {
                    fu = F2(x, yu);
                    NOTE(x, yu, fu);
                }
                if (yu != y && fu > fc) {
                    x = xl;
                    y = yu;
                    fc = F2(x, y);
                    NOTE(x, y, fc);
                    continue;
                }
                x = xl;
                fc = fl;
                continue;
            }
            double fr = fc;
            if (xr != x) {
                fr = F2(xr, y);
                NOTE(xr, y, fr);
            }
            if (xr != x && fr > fc) {
                x = xr;
                y = yd;
                fc = F2(x, y);
                NOTE(x, y, fc);
                continue;
            }
            y = yd;
            fc = fd;
        }
        if (!converged) {
            x = bx;
            y = by;
            fc = bf;
        }
    }
    *px = x;
    *py = y;
#undef F2
#undef NOTE
}

/* zoom.cpp:407-414 */
static int64_t snap_index(double value, const orc_axis* ax) { return lround((value - ax->min) / ax->step); }
static int64_t step_units(double step_value, double finest) {
    int64_t u = lround(step_value / finest);
    return u > 0 ? u : 1;
}

typedef struct {
    int64_t lo1, hi1, lo2, hi2, lodf, hidf;
} Bounds; /* zoom.cpp:403-405 */

/* zoom.cpp:416-523 (quantify_impl) */
static int quantify_impl(const Sim* sim, const orc_grid* g, const Bounds* b,
                         const orc_zoom_cfg* cfg, double init_t1, double init_t2,
                         const double* fp, const float* dict, Trace* tr, orc_quant* out) {
    int64_t n = sim->n;
    Obj o;
    memset(&o, 0, sizeof o);
    o.sim = sim;
    o.g = g;
    o.n = n;
    o.smooth_k = cfg->smooth_k;
    o.query = malloc(sizeof(double) * 2 * (size_t)n);
    o.buf = malloc(sizeof(double) * 2 * (size_t)n);
    o.buf2 = malloc(sizeof(double) * 2 * (size_t)n);
    o.buf3 = malloc(sizeof(double) * 2 * (size_t)n);
    o.dict_mode = cfg->dict_mode;
    o.dict = dict;
    o.cap = 4096;
    o.tab = calloc((size_t)o.cap, sizeof(Slot));
    int rc = 0;
    {
        const double* q = fp;
        if (cfg->smooth_k) {
            smooth(fp, n, cfg->smooth_k, o.buf2);
            q = o.buf2;
        }
        if (normalize(q, n, o.query)) rc = -1;
    }
    if (rc == 0) {
        int64_t i1 = clampl(snap_index(init_t1, &g->t1_ms), b->lo1, b->hi1);
        int64_t i2 = clampl(snap_index(init_t2, &g->t2_ms), b->lo2, b->hi2);
        int metric = cfg->metric;
        DfParams prm;
        prm.coarse = step_units(cfg->df_coarse_hz, g->df_hz.step);
        prm.refine = step_units(cfg->df_refine_hz, g->df_hz.step);
        prm.finest = 1;
        prm.window_half = step_units(cfg->df_window_hz / 2, g->df_hz.step);
        prm.omega = step_units(cfg->omega_hz, g->df_hz.step);
        prm.plateau_eps = cfg->plateau_eps;
        prm.heavy_cc = metric == 0 ? cfg->heavy_noise_cc : -1e300;
        prm.fallback_coarse = step_units(cfg->fallback_coarse_hz, g->df_hz.step);
        prm.fallback_window_half = step_units(cfg->fallback_window_hz / 2, g->df_hz.step);
        prm.allow_fallback = 1;
        /* Stage 1 (zoom.cpp:465-469) */
        DfCtx dc = {&o, i1, i2, metric, tr};
        o.in_stage1 = 1;
        int64_t idf = search_df(&dc, b->lodf, b->hidf, &prm);
        o.in_stage1 = 0;
        /* Stage 2 (zoom.cpp:472-479) */
        int64_t s1v[8], s2v[8];
        for (int k = 0; k < cfg->n2d; ++k) {
            s1v[k] = step_units(cfg->t1t2_2d_steps_ms[k], g->t1_ms.step);
            s2v[k] = step_units(cfg->t1t2_2d_steps_ms[k], g->t2_ms.step);
        }
        zoom_2d(&o, idf, metric, b->lo1, b->hi1, b->lo2, b->hi2, &i1, &i2, s1v, s2v, cfg->n2d);
        note(tr, &o, ORC_STAGE_T1T2_2D, i1, i2, idf, obj_eval(&o, i1, i2, idf, metric));
        /* Stage 3 (zoom.cpp:482-489) */
        {
            Best bb = {-1, -1e300};
            int64_t a = clampl(idf - prm.omega / 2, b->lodf, b->hidf);
            int64_t z = clampl(idf + prm.omega / 2, b->lodf, b->hidf);
            for (int64_t k = a; k <= z; ++k) offer(&bb, k, obj_eval(&o, i1, i2, k, metric));
            idf = bb.idx;
            note(tr, &o, ORC_STAGE_DF_SWEEP, i1, i2, idf, bb.val);
        }
        /* Stage 4 (zoom.cpp:492-501) */
        for (int k = 0; k < cfg->n1d; ++k) {
            double s = cfg->t1t2_1d_steps_ms[k];
            int64_t u1 = step_units(s, g->t1_ms.step);
            LineCtx lc1 = {&o, 0, i1, i2, idf, metric};
            i1 = zoom_1d(&lc1, b->lo1, b->hi1, i1, &u1, 1);
            note(tr, &o, ORC_STAGE_T1_1D, i1, i2, idf, obj_eval(&o, i1, i2, idf, metric));
            int64_t u2 = step_units(s, g->t2_ms.step);
            LineCtx lc2 = {&o, 1, i1, i2, idf, metric};
            i2 = zoom_1d(&lc2, b->lo2, b->hi2, i2, &u2, 1);
            note(tr, &o, ORC_STAGE_T2_1D, i1, i2, idf, obj_eval(&o, i1, i2, idf, metric));
        }
        /* Stage 5 (zoom.cpp:505-512) */
        {
            int64_t f1 = step_units(cfg->final_2d_step_ms, g->t1_ms.step);
            int64_t f2 = step_units(cfg->final_2d_step_ms, g->t2_ms.step);
            zoom_2d(&o, idf, cfg->final_metric, b->lo1, b->hi1, b->lo2, b->hi2, &i1, &i2, &f1, &f2, 1);
            note(tr, &o, ORC_STAGE_T1T2_FINAL, i1, i2, idf, obj_eval(&o, i1, i2, idf, cfg->final_metric));
        }
        /* zoom.cpp:514-519 */
        out->score = obj_eval(&o, i1, i2, idf, metric);
        out->i1 = i1;
        out->i2 = i2;
        out->idf = idf;
        out->t1_ms = axis_value(&g->t1_ms, i1);
        out->t2_ms = axis_value(&g->t2_ms, i2);
        out->df_hz = axis_value(&g->df_hz, idf);
        sim_run(sim, axis_value(&g->t1_ms, i1) * 1e-3, axis_value(&g->t2_ms, i2) * 1e-3,
                axis_value(&g->df_hz, idf), o.buf);
        out->pd = norm2(fp, n) / norm2(o.buf, n); /* estimate_pd, fingerprint.cpp:147-152 */
        out->evaluations = o.evals;
        if (o.err) rc = -1;
    }
    free(o.query);
    free(o.buf);
    free(o.buf2);
    free(o.buf3);
    free(o.tab);
    return rc;
}

static Bounds full_bounds(const orc_grid* g) {
    Bounds b = {0, g->t1_ms.count - 1, 0, g->t2_ms.count - 1, 0, g->df_hz.count - 1};
    return b;
}

static int check_lattice(const orc_grid* g) {
    const orc_axis* ax[3] = {&g->t1_ms, &g->t2_ms, &g->df_hz};
    for (int i = 0; i < 3; ++i)
        if (ax[i]->count <= 0 || ax[i]->count >= (1LL << 21))
            return fail("objective: lattice axis empty or too fine");
    return 0;
}

/* zoom.cpp:533-539 (quantify) */
int orc_quantify(const orc_sched* s, const orc_grid* lattice, const orc_zoom_cfg* cfg,
                 const double* fp, orc_quant* out) {
    if (check_lattice(lattice)) return -1;
    Sim sim;
    int rc = sim_init(&sim, s);
    Bounds b = full_bounds(lattice);
    if (rc == 0)
        rc = quantify_impl(&sim, lattice, &b, cfg, cfg->init_t1_ms, cfg->init_t2_ms, fp, NULL, NULL, out);
    sim_free(&sim);
    return rc;
}

int orc_quantify_ex(const orc_sched* s, const orc_grid* lattice, const orc_zoom_cfg* cfg,
                    const double* fp, const float* dict, int64_t dict_entries, orc_stage* trace,
                    int trace_cap, int* trace_len, orc_quant* out) {
    if (check_lattice(lattice)) return -1;
    if (dict) {
        const int64_t need = cfg->dict_mode == 2
                                 ? lattice->t1_ms.count * lattice->t2_ms.count * lattice->df_hz.count
                                 : lattice->df_hz.count;
        if (cfg->dict_mode == 0 || dict_entries != need)
            return fail("objective: dictionary does not match the lattice");
    }
    Sim sim;
    int rc = sim_init(&sim, s);
    Bounds b = full_bounds(lattice);
    Trace tr = {trace, trace_cap, 0, 0};
    if (rc == 0)
        rc = quantify_impl(&sim, lattice, &b, cfg, cfg->init_t1_ms, cfg->init_t2_ms, fp, dict, &tr, out);
    if (trace_len) *trace_len = tr.n;
    sim_free(&sim);
    return rc;
}

/* zoom.cpp:555-629 (quantify_slice); off-mask voxels come back zeroed. */
int orc_quantify_slice(const orc_sched* s, const orc_grid* g, const orc_zoom_cfg* cfg,
                       const double* fps, const uint8_t* mask, int nx, int ny, int use_prior,
                       int threads, orc_quant* out) {
    if (nx <= 0 || ny <= 0) return fail("quantify_slice: inconsistent raster dimensions");
    if (check_lattice(g)) return -1;
    Sim sim;
    if (sim_init(&sim, s)) {
        sim_free(&sim);
        return -1;
    }
    int64_t nvox = (int64_t)nx * ny, n = s->n;
    memset(out, 0, sizeof(orc_quant) * (size_t)nvox);
    int rc = 0;
    if (use_prior) {
        int have = 0;
        orc_quant prior;
        memset(&prior, 0, sizeof prior);
        for (int64_t i = 0; i < nvox && rc == 0; ++i) {
            if (!mask[i]) continue;
            Bounds b = full_bounds(g);
            double it1 = cfg->init_t1_ms, it2 = cfg->init_t2_ms;
            if (have) {
                /* zoom.cpp:595-610: prior.params.t1 * 1e3 round-trips through seconds */
                double pt1 = (prior.t1_ms * 1e-3) * 1e3, pt2 = (prior.t2_ms * 1e-3) * 1e3;
                it1 = pt1;
                it2 = pt2;
                int64_t p1 = snap_index(pt1, &g->t1_ms);
                int64_t p2 = snap_index(pt2, &g->t2_ms);
                int64_t pdf = snap_index(prior.df_hz, &g->df_hz);
                int64_t w1 = step_units(cfg->prior_window_t1_ms, g->t1_ms.step);
                int64_t w2 = step_units(cfg->prior_window_t2_ms, g->t2_ms.step);
                int64_t wdf = step_units(cfg->prior_window_df_hz, g->df_hz.step);
                b.lo1 = b.lo1 > p1 - w1 ? b.lo1 : p1 - w1;
                b.hi1 = b.hi1 < p1 + w1 ? b.hi1 : p1 + w1;
                b.lo2 = b.lo2 > p2 - w2 ? b.lo2 : p2 - w2;
                b.hi2 = b.hi2 < p2 + w2 ? b.hi2 : p2 + w2;
                b.lodf = b.lodf > pdf - wdf ? b.lodf : pdf - wdf;
                b.hidf = b.hidf < pdf + wdf ? b.hidf : pdf + wdf;
            }
            rc = quantify_impl(&sim, g, &b, cfg, it1, it2, fps + i * 2 * n, NULL, NULL, &out[i]);
            prior = out[i];
            have = 1;
        }
    } else {
        if (threads < 1) threads = 1;
        int bad = 0;
#pragma omp parallel for num_threads(threads) schedule(dynamic, 1) reduction(| : bad)
        for (int64_t i = 0; i < nvox; ++i) {
            if (!mask[i]) continue;
            Bounds b = full_bounds(g);
            if (quantify_impl(&sim, g, &b, cfg, cfg->init_t1_ms, cfg->init_t2_ms, fps + i * 2 * n, NULL,
                              NULL, &out[i]))
                bad = 1;
        }
        if (bad) rc = -1;
    }
    sim_free(&sim);
    return rc;
}

/* Four-parameter ZOOM (oracle_api.h): outer zoom_1d over the B1 index with
 * the memoized objective g(ib) = quantify(fp, scheds[ib]).score; the inner
 * search is quantify_impl above (zoom.cpp:416-523), the outer walk zoom_1d's
 * probe order (zoom.cpp:252-282: left flank first, strict improvement,
 * clamped, ties keep the centre). */
int orc_quantify_b1(const orc_sched* scheds, int nb, const orc_grid* lattice, const orc_zoom_cfg* cfg,
                    const int64_t* steps, int nsteps, int64_t init_ib, const double* fp, orc_quant* out,
                    int64_t* ib_out) {
    if (nb <= 0) return fail("quantify_b1: no B1 values");
    if (check_lattice(lattice)) return -1;
    for (int k = 0; k < nsteps; ++k)
        if (steps[k] <= 0) return fail("zoom_1d: step must be positive");
    orc_quant* res = calloc((size_t)nb, sizeof(orc_quant));
    int* have = calloc((size_t)nb, sizeof(int));
    int64_t evals = 0;
    int rc = 0;
#define G(ib) (have[ib] ? 0 : (rc = rc ? rc : orc_quantify(&scheds[ib], lattice, cfg, fp, &res[ib]), \
                                 have[ib] = 1, evals += res[ib].evaluations, 0), res[ib].score)
    int64_t x = clampl(init_ib, 0, nb - 1);
    double fx = G(x);
    for (int si = 0; si < nsteps && rc == 0; ++si) {
        const int64_t st = steps[si];
        for (;;) {
            const int64_t xl = clampl(x - st, 0, nb - 1);
            if (xl != x) {
                const double fl = G(xl);
                if (fl > fx) {
                    x = xl;
                    fx = fl;
                    continue;
                }
            }
            const int64_t xr = clampl(x + st, 0, nb - 1);
            if (xr != x) {
                const double fr = G(xr);
                if (fr > fx) {
                    x = xr;
                    fx = fr;
                    continue;
                }
            }
            break;
        }
    }
#undef G
    if (rc == 0) {
        *out = res[x];
        out->evaluations = evals;
        *ib_out = x;
    }
    free(res);
    free(have);
    return rc;
}
