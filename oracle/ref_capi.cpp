// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrapper exposing the UNMODIFIED reference library (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/libmrf_ref.so)
// through oracle/oracle_api.h, so the tests can pin the C restatement
// (oracle/mrf_oracle.c) against the reference itself and bench.py can time
// the reference's own CPU path.  Every entry calls the reference's public API
// (proj/include/mrf/*.hpp); the only harness logic is unit conversion and the
// BASELINE.json schedule formula (which the reference ingests through
// load_schedule_csv in real use).
#include <atomic>
#include <cmath>
#include <exception>
#include <mutex>
#include <thread>
#include <complex>
#include <cstring>
#include <string>
#include <vector>

#include "mrf/bloch.hpp"
#include "mrf/dictionary.hpp"
#include "mrf/fingerprint.hpp"
#include "mrf/rng.hpp"
#include "mrf/sequence.hpp"
#include "mrf/util.hpp"
#include "mrf/zoom.hpp"
#include "oracle_api.h"

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

mrf::Schedule to_sched(const orc_sched* s) {
    mrf::Schedule out;
    out.entries.resize(static_cast<std::size_t>(s->n));
    for (int64_t i = 0; i < s->n; ++i)
        out.entries[i] = {s->flip_deg[i], s->phase_deg[i], s->tr_ms[i], s->te_ms[i]};
    return out;
}

mrf::ParameterGrid to_grid(const orc_grid* g) {
    mrf::ParameterGrid p;
    p.t1_ms = {g->t1_ms.min, g->t1_ms.step, static_cast<std::size_t>(g->t1_ms.count)};
    p.t2_ms = {g->t2_ms.min, g->t2_ms.step, static_cast<std::size_t>(g->t2_ms.count)};
    p.df_hz = {g->df_hz.min, g->df_hz.step, static_cast<std::size_t>(g->df_hz.count)};
    return p;
}

// Half-open ranges whose endpoint-exclusive count (dictionary.cpp:25-33)
// reproduces the axis count exactly.
mrf::AxisRange to_range(const orc_axis& a) {
    return {a.min, a.min + static_cast<double>(a.count) * a.step, a.step};
}

mrf::Fingerprint to_fp(const double* v, int64_t n) {
    mrf::Fingerprint fp;
    fp.s.resize(static_cast<std::size_t>(n));
    for (int64_t j = 0; j < n; ++j) fp.s[j] = {v[2 * j], v[2 * j + 1]};
    return fp;
}

mrf::ZoomConfig to_cfg(const orc_zoom_cfg* c) {
    mrf::ZoomConfig z;
    z.metric = c->metric ? mrf::Metric::euclidean : mrf::Metric::cc;
    z.final_metric = c->final_metric ? mrf::Metric::euclidean : mrf::Metric::cc;
    z.smooth_k = c->smooth_k;
    z.omega_hz = c->omega_hz;
    z.df_coarse_hz = c->df_coarse_hz;
    z.df_refine_hz = c->df_refine_hz;
    z.df_window_hz = c->df_window_hz;
    z.plateau_eps = c->plateau_eps;
    z.heavy_noise_cc = c->heavy_noise_cc;
    z.fallback_coarse_hz = c->fallback_coarse_hz;
    z.fallback_window_hz = c->fallback_window_hz;
    z.t1t2_2d_steps_ms.assign(c->t1t2_2d_steps_ms, c->t1t2_2d_steps_ms + c->n2d);
    z.t1t2_1d_steps_ms.assign(c->t1t2_1d_steps_ms, c->t1t2_1d_steps_ms + c->n1d);
    z.final_2d_step_ms = c->final_2d_step_ms;
    z.init_t1_ms = c->init_t1_ms;
    z.init_t2_ms = c->init_t2_ms;
    z.prior_window_t1_ms = c->prior_window_t1_ms;
    z.prior_window_t2_ms = c->prior_window_t2_ms;
    z.prior_window_df_hz = c->prior_window_df_hz;
    return z;
}

int64_t snap(double v, const orc_axis& a) { return std::lround((v - a.min) / a.step); }

void fill_quant(const orc_grid* g, double t1_ms, double t2_ms, double df_hz, double pd,
                double score, std::size_t evals, orc_quant* out) {
    out->t1_ms = t1_ms;
    out->t2_ms = t2_ms;
    out->df_hz = df_hz;
    out->i1 = snap(t1_ms, g->t1_ms);
    out->i2 = snap(t2_ms, g->t2_ms);
    out->idf = snap(df_hz, g->df_hz);
    out->pd = pd;
    out->score = score;
    out->evaluations = static_cast<int64_t>(evals);
}
}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }
const char* orc_impl_name(void) { return "reference"; }

int orc_build_schedule(int64_t n, uint64_t seed, double* flip, double* phase, double* tr,
                       double* te) {
    return guard([&] {
        mrf::Schedule s = mrf::build_schedule(static_cast<std::size_t>(n), seed);
        for (int64_t i = 0; i < n; ++i) {
            flip[i] = s.entries[i].flip_deg;
            phase[i] = s.entries[i].phase_deg;
            tr[i] = s.entries[i].tr_ms;
            te[i] = s.entries[i].te_ms;
        }
    });
}

int orc_baseline_schedule(int64_t n, uint64_t seed, double* flip, double* phase, double* tr,
                          double* te) {
    return guard([&] {
        for (int64_t j = 0; j < n; ++j) {
            double fa = 10.0 + 50.0 * std::fabs(std::sin(2.0 * M_PI * static_cast<double>(j) / 250.0)) +
                        2.0 * mrf::rng::gaussian(seed, 1, static_cast<std::uint64_t>(j));
            double trv = mrf::quantize9(10.5 + 3.5 * mrf::rng::uniform01(seed, 2, static_cast<std::uint64_t>(j)));
            flip[j] = mrf::quantize9(fa);
            phase[j] = (j % 2) ? 180.0 : 0.0;
            tr[j] = trv;
            te[j] = mrf::quantize9(trv / 2.0);
        }
    });
}

int orc_simulate(const orc_sched* s, double t1_s, double t2_s, double df_hz, double* out) {
    return guard([&] {
        mrf::BlochSimulator sim(to_sched(s));
        std::vector<std::complex<double>> buf(sim.length());
        sim.simulate({t1_s, t2_s, df_hz, 1.0}, buf.data());
        for (std::size_t j = 0; j < buf.size(); ++j) {
            out[2 * j] = buf[j].real();
            out[2 * j + 1] = buf[j].imag();
        }
    });
}

int orc_add_noise(const double* fp, int64_t n, double sigma, uint64_t seed, double* out) {
    return guard([&] {
        mrf::Fingerprint r = mrf::add_noise(to_fp(fp, n), sigma, seed);
        for (int64_t j = 0; j < n; ++j) {
            out[2 * j] = r.s[j].real();
            out[2 * j + 1] = r.s[j].imag();
        }
    });
}

double orc_cc(const double* a, const double* b, int64_t n) {
    try {
        return mrf::cc(to_fp(a, n), to_fp(b, n));
    } catch (const std::exception& e) {
        g_err = e.what();
        return NAN;
    }
}

double orc_cc_unit(const double* a, const double* b, int64_t n) {
    try {
        return mrf::cc(mrf::normalize(to_fp(a, n)), mrf::normalize(to_fp(b, n)));
    } catch (const std::exception& e) {
        g_err = e.what();
        return NAN;
    }
}

int orc_calibrate_noise(const double* fp, int64_t n, double target, uint64_t seed, double* sigma) {
    try {
        *sigma = mrf::calibrate_noise(to_fp(fp, n), target, seed);
        return 0;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return -3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

int orc_make_calibrated_noise(const double* fp, int64_t n, double target, uint64_t seed,
                              double* sigma, uint64_t* seed_used, double* noisy) {
    try {
        mrf::CalibratedNoise r = mrf::make_calibrated_noise(to_fp(fp, n), target, seed);
        *sigma = r.sigma;
        *seed_used = r.seed;
        std::memcpy(noisy, r.noisy.s.data(), sizeof(double) * 2 * static_cast<std::size_t>(n));
        return 0;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return -3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

int orc_smooth(const double* fp, int64_t n, int k, double* out) {
    return guard([&] {
        mrf::Fingerprint r = mrf::smooth(to_fp(fp, n), k);
        std::memcpy(out, r.s.data(), sizeof(double) * 2 * static_cast<std::size_t>(n));
    });
}

int orc_ref_save_generated(const orc_sched* s, const orc_grid* g, const char* path) {
    return guard([&] { mrf::save_generated(to_grid(g), to_sched(s), path, 8); });
}

int orc_ref_cc_map_to_file(const orc_sched* s, const orc_grid* g, const double* fp, const char* path) {
    return guard([&] { mrf::cc_map_to_file(to_fp(fp, s->n), to_grid(g), to_sched(s), path, 8); });
}

int orc_generate(const orc_sched* s, const orc_grid* g, int64_t first, int64_t count, float* out) {
    return guard([&] {
        // The reference materializes the whole lattice; generate() of a grid
        // then slice [first, first+count).
        mrf::Dictionary d = mrf::generate(to_grid(g), to_sched(s), 8);
        std::memcpy(out, d.data.data() + first * 2 * s->n,
                    sizeof(float) * static_cast<std::size_t>(count * 2 * s->n));
    });
}

int orc_scan_grid(const orc_sched* s, const orc_grid* g, const double* queries, int64_t nq,
                  int metric, int threads, int64_t* best_flat, double* best_score,
                  double* second_score) {
    return orc_scan_grid_ex(s, g, queries, nullptr, nq, metric, threads, best_flat, best_score, second_score);
}

int orc_scan_grid_ex(const orc_sched* s, const orc_grid* g, const double* queries, const uint8_t* unit,
                     int64_t nq, int metric, int threads, int64_t* best_flat, double* best_score,
                     double* second_score) {
    return guard([&] {
        std::vector<mrf::Fingerprint> qs;
        for (int64_t i = 0; i < nq; ++i) {
            qs.push_back(to_fp(queries + i * 2 * s->n, s->n));
            qs.back().unit_norm = unit != nullptr && unit[i] != 0;
        }
        mrf::ParameterGrid grid = to_grid(g);
        mrf::ScanOutcome out = mrf::scan_grid(grid, to_sched(s), qs,
                                              metric ? mrf::Metric::euclidean : mrf::Metric::cc,
                                              threads);
        for (int64_t i = 0; i < nq; ++i) {
            const auto& p = out.matches[i].params;
            int64_t i1 = snap(p.t1 * 1e3, g->t1_ms), i2 = snap(p.t2 * 1e3, g->t2_ms),
                    idf = snap(p.df, g->df_hz);
            best_flat[i] = static_cast<int64_t>(grid.flatten(i1, i2, idf));
            best_score[i] = out.matches[i].score;
            if (second_score) second_score[i] = NAN;
        }
    });
}

int orc_quantify(const orc_sched* s, const orc_grid* lattice, const orc_zoom_cfg* cfg,
                 const double* fp, orc_quant* out) {
    return guard([&] {
        mrf::SearchRanges r{to_range(lattice->t1_ms), to_range(lattice->t2_ms),
                            to_range(lattice->df_hz)};
        // dictionary lookup modes: the reference's own dictionaries
        // (make_df_dictionary, zoom.cpp:541-553; generate over the lattice)
        const mrf::Schedule sc = to_sched(s);
        const mrf::ZoomConfig zc = to_cfg(cfg);
        mrf::Dictionary dict;
        const mrf::Dictionary *df = nullptr, *full = nullptr;
        if (cfg->dict_mode == 1) {
            dict = mrf::make_df_dictionary(r, zc, sc, 1);
            df = &dict;
        } else if (cfg->dict_mode == 2) {
            dict = mrf::generate(mrf::grid_from_ranges(r.t1_ms, r.t2_ms, r.df_hz), sc, 1);
            full = &dict;
        }
        mrf::QuantResult q = mrf::quantify(to_fp(fp, s->n), r, zc, sc, df, full);
        fill_quant(lattice, q.params.t1 * 1e3, q.params.t2 * 1e3, q.params.df, q.params.pd,
                   q.score, q.evaluations, out);
    });
}

int orc_quantify_ex(const orc_sched* s, const orc_grid* lattice, const orc_zoom_cfg* cfg,
                    const double* fp, const float* dict, int64_t dict_entries, orc_stage* trace,
                    int trace_cap, int* trace_len, orc_quant* out) {
    return guard([&] {
        mrf::SearchRanges r{to_range(lattice->t1_ms), to_range(lattice->t2_ms),
                            to_range(lattice->df_hz)};
        const mrf::Schedule sc = to_sched(s);
        const mrf::ZoomConfig zc = to_cfg(cfg);
        // the reference's own dictionaries (grid, digest, entry length), whose
        // payload is then replaced by the caller's entries when given
        mrf::Dictionary dict_obj;
        const mrf::Dictionary *df = nullptr, *full = nullptr;
        if (cfg->dict_mode == 1) {
            dict_obj = mrf::make_df_dictionary(r, zc, sc, 1);
            df = &dict_obj;
        } else if (cfg->dict_mode == 2) {
            dict_obj = mrf::generate(mrf::grid_from_ranges(r.t1_ms, r.t2_ms, r.df_hz), sc, 1);
            full = &dict_obj;
        }
        if (dict) {
            if (cfg->dict_mode == 0 ||
                static_cast<std::size_t>(dict_entries) * dict_obj.entry_len * 2 != dict_obj.data.size())
                throw std::invalid_argument("objective: dictionary does not match the lattice");
            dict_obj.data.assign(dict, dict + dict_obj.data.size());
        }
        mrf::QuantResult q = mrf::quantify(to_fp(fp, s->n), r, zc, sc, df, full);
        fill_quant(lattice, q.params.t1 * 1e3, q.params.t2 * 1e3, q.params.df, q.params.pd,
                   q.score, q.evaluations, out);
        static const char* kNames[] = {"df.coarse",  "df.refine", "df.translate", "df.rerefine",
                                       "df.plateau_stop", "df.finest", "df.fallback", "t1t2.2d",
                                       "df.sweep", "t1.1d", "t2.1d", "t1t2.final"};
        int k = 0;
        for (const mrf::StageLog& lg : q.trace) {
            if (trace && k < trace_cap) {
                int code = -1;
                for (int c = 0; c < 12; ++c)
                    if (lg.stage == kNames[c]) code = c;
                if (code < 0) throw std::runtime_error("unknown stage name " + lg.stage);
                trace[k] = orc_stage{code, 0, static_cast<int64_t>(lg.evaluations), lg.best, lg.t1_ms,
                                     lg.t2_ms, lg.df_hz};
            }
            ++k;
        }
        if (trace_len) *trace_len = k;
    });
}

int orc_quantify_b1(const orc_sched* scheds, int nb, const orc_grid* lattice, const orc_zoom_cfg* cfg,
                    const int64_t* steps, int nsteps, int64_t init_ib, const double* fp, orc_quant* out,
                    int64_t* ib_out) {
    // the reference's own zoom_1d (zoom.cpp:252-282) over the B1 index, its
    // objective the reference's own quantify under each B1 schedule, memoized
    return guard([&] {
        if (nb <= 0) throw std::invalid_argument("quantify_b1: no B1 values");
        mrf::SearchRanges r{to_range(lattice->t1_ms), to_range(lattice->t2_ms), to_range(lattice->df_hz)};
        const mrf::ZoomConfig zc = to_cfg(cfg);
        const mrf::Fingerprint q = to_fp(fp, scheds[0].n);
        std::vector<mrf::QuantResult> res(static_cast<std::size_t>(nb));
        std::vector<bool> have(static_cast<std::size_t>(nb), false);
        std::size_t evals = 0;
        auto g = [&](long ib) {
            if (!have[ib]) {
                res[ib] = mrf::quantify(q, r, zc, to_sched(&scheds[ib]));
                have[ib] = true;
                evals += res[ib].evaluations;
            }
            return res[ib].score;
        };
        std::vector<long> st(steps, steps + nsteps);
        const long ib = mrf::zoom_1d(g, 0, nb - 1, static_cast<long>(init_ib), st);
        const mrf::QuantResult& b = res[ib];
        fill_quant(lattice, b.params.t1 * 1e3, b.params.t2 * 1e3, b.params.df, b.params.pd, b.score, evals, out);
        *ib_out = ib;
    });
}

int orc_quantify_slice(const orc_sched* s, const orc_grid* g, const orc_zoom_cfg* cfg,
                       const double* fps, const uint8_t* mask, int nx, int ny, int use_prior,
                       int threads, orc_quant* out) {
    return guard([&] {
        std::size_t nv = static_cast<std::size_t>(nx) * static_cast<std::size_t>(ny);
        std::vector<mrf::Fingerprint> v(nv);
        std::vector<std::uint8_t> m(mask, mask + nv);
        for (std::size_t i = 0; i < nv; ++i)
            if (m[i]) v[i] = to_fp(fps + i * 2 * s->n, s->n);
        mrf::SearchRanges r{to_range(g->t1_ms), to_range(g->t2_ms), to_range(g->df_hz)};
        const mrf::Schedule sc = to_sched(s);
        const mrf::ZoomConfig zc = to_cfg(cfg);
        mrf::Dictionary dfd;
        if (cfg->dict_mode == 1) dfd = mrf::make_df_dictionary(r, zc, sc, 1);
        mrf::SliceResult res = mrf::quantify_slice(v, m, nx, ny, r, zc, sc, use_prior != 0, threads,
                                                   cfg->dict_mode == 1 ? &dfd : nullptr);
        std::memset(out, 0, sizeof(orc_quant) * nv);
        for (std::size_t i = 0; i < nv; ++i)
            if (m[i])
                fill_quant(g, res.t1_ms[i], res.t2_ms[i], res.df_hz[i], res.pd[i], res.score[i],
                           res.evaluations[i], &out[i]);
    });
}

/* Reference answers at BASELINE scale (test infrastructure for the scale
 * fixtures).  The lattice is T1 values x T2 values x a linear df axis, given
 * as explicit value arrays (linear axes pass min + k*step, which is what
 * AxisSpec::value computes; config 3 passes its log-spaced values).  Each
 * (T1, T2) row of atoms is produced by the reference's own mrf::generate on
 * the one-row subgrid {t1[i1], 1, 1} x {t2[i2], 1, 1} x df (value(0) = min
 * exactly, so every TissueParams equals the full lattice's), rows are
 * gathered into T1 slabs, and every query is scored by the reference's own
 * mrf::brute_force_search over each slab (an index-space Dictionary).  Slabs
 * are visited in flat order and a later slab wins only with a strictly higher
 * score: the reference's lowest-flat tie rule (dictionary.cpp:241-255,
 * :291-294).  Work is spread over `threads` host threads (rows for
 * generation, queries for the search). */
int orc_ref_scan_rows(const orc_sched* s, const double* t1_ms, int64_t n1, const double* t2_ms,
                      int64_t n2, const orc_axis* df, const double* queries, int64_t nq,
                      int metric, int threads, int64_t* best_flat, double* best_score) {
    return guard([&] {
        const mrf::Schedule sc = to_sched(s);
        const std::size_t n = static_cast<std::size_t>(s->n);
        const std::size_t ndf = static_cast<std::size_t>(df->count);
        const std::size_t row = ndf * 2 * n;
        std::vector<mrf::Fingerprint> qs;
        for (int64_t i = 0; i < nq; ++i) qs.push_back(to_fp(queries + i * 2 * s->n, s->n));
        std::vector<double> best(static_cast<std::size_t>(nq), -1e300);
        std::vector<int64_t> bflat(static_cast<std::size_t>(nq), 0);
        mrf::Dictionary slab;
        slab.grid.t1_ms = {0.0, 1.0, 1};
        slab.grid.t2_ms = {0.0, 1.0, static_cast<std::size_t>(n2)};
        slab.grid.df_hz = {0.0, 1.0, ndf};
        slab.entry_len = n;
        slab.data.resize(static_cast<std::size_t>(n2) * row);
        const int T = threads > 0 ? threads : 1;
        auto pool = [&](int64_t count, auto&& fn) {
            std::atomic<int64_t> next{0};
            std::vector<std::thread> ts;
            std::exception_ptr err;
            std::mutex mu;
            for (int t = 0; t < T; ++t)
                ts.emplace_back([&] {
                    try {
                        for (int64_t k; (k = next.fetch_add(1)) < count;) fn(k);
                    } catch (...) {
                        std::lock_guard<std::mutex> lk(mu);
                        if (!err) err = std::current_exception();
                    }
                });
            for (auto& t : ts) t.join();
            if (err) std::rethrow_exception(err);
        };
        const mrf::Metric m = metric ? mrf::Metric::euclidean : mrf::Metric::cc;
        for (int64_t i1 = 0; i1 < n1; ++i1) {
            pool(n2, [&](int64_t i2) {
                mrf::ParameterGrid g;
                g.t1_ms = {t1_ms[i1], 1.0, 1};
                g.t2_ms = {t2_ms[i2], 1.0, 1};
                g.df_hz = {df->min, df->step, ndf};
                mrf::Dictionary d = mrf::generate(g, sc, 1);
                std::memcpy(slab.data.data() + static_cast<std::size_t>(i2) * row, d.data.data(),
                            row * sizeof(float));
            });
            pool(nq, [&](int64_t q) {
                mrf::Match r = mrf::brute_force_search(qs[static_cast<std::size_t>(q)], slab, m);
                if (r.score > best[q]) {
                    best[q] = r.score;
                    const int64_t i2 = std::lround(r.params.t2 * 1e3);
                    const int64_t idf = std::lround(r.params.df);
                    bflat[q] = (i1 * n2 + i2) * static_cast<int64_t>(ndf) + idf;
                }
            });
        }
        for (int64_t q = 0; q < nq; ++q) {
            best_flat[q] = bflat[q];
            best_score[q] = best[q];
        }
    });
}

}  // extern "C"
