// mrf_api.cpp -- the reference's C++ interface (include/mrf_b200/mrf.hpp) on top
// of the C ABI (include/mrfg.h).  Built as libmrf_b200.so.
//
// Heavy work (simulation, dictionary generation, brute-force search, cc_map,
// MRF-ZOOM) is forwarded to the sm_100a kernels; the small host pieces the
// reference's callers also use (schedule I/O, normalize/cc/estimate_pd on single
// fingerprints, the generic search_df/zoom_1d/zoom_2d over caller objectives)
// are host restatements with the reference's operand order.  ABI status codes
// become the reference's exceptions.
#include <openssl/evp.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <exception>
#include <stdexcept>
#include <thread>

#include "mrf_b200/mrf.hpp"
#include "mrfg.h"

namespace mrf {
namespace {

int device() {
    const char* e = std::getenv("MRFG_DEVICE");
    return e ? std::atoi(e) : 0;
}

// Devices the drop-in spreads its work over: MRFG_DEVICES="0,1,...,7" (one
// context per listed device; a device may repeat), else the single
// MRFG_DEVICE.  The reference's `workers` selects host threads and never
// changes results (parallel.hpp:12-15); the device list likewise never
// changes results: atom shards are merged by (max score, lowest flat), voxel
// shards are independent.
std::vector<int> devices() {
    std::vector<int> out;
    if (const char* e = std::getenv("MRFG_DEVICES")) {
        std::string v(e);
        std::size_t pos = 0;
        while (pos < v.size()) {
            const std::size_t c = v.find(',', pos);
            const std::string tok = v.substr(pos, c == std::string::npos ? std::string::npos : c - pos);
            if (!tok.empty()) out.push_back(std::atoi(tok.c_str()));
            if (c == std::string::npos) break;
            pos = c + 1;
        }
    }
    if (out.empty()) out.push_back(device());
    return out;
}

// fn(k) on one host thread per shard; the first exception is rethrown.
template <class F>
void on_shards(std::size_t count, F&& fn) {
    if (count == 1) {
        fn(std::size_t{0});
        return;
    }
    std::vector<std::thread> th;
    std::vector<std::exception_ptr> err(count);
    for (std::size_t k = 0; k < count; ++k)
        th.emplace_back([&, k] {
            try {
                fn(k);
            } catch (...) {
                err[k] = std::current_exception();
            }
        });
    for (auto& t : th) t.join();
    for (auto& e : err)
        if (e) std::rethrow_exception(e);
}

[[noreturn]] void raise(int rc) {
    const std::string msg = mrfg_last_error();
    if (rc == MRFG_E_INVALID) throw std::invalid_argument(msg);
    if (rc == MRFG_E_RANGE) throw std::out_of_range(msg);
    throw std::runtime_error(msg);
}
void check(int rc) {
    if (rc != MRFG_OK) raise(rc);
}

struct CtxGuard {
    mrfg_ctx* h = nullptr;
    ~CtxGuard() {
        if (h) mrfg_destroy(h);
    }
};

mrfg_ctx* create(const Schedule& s, int dev = device()) {
    const std::size_t n = s.size();
    std::vector<double> f(n), p(n), tr(n), te(n);
    for (std::size_t i = 0; i < n; ++i) {
        f[i] = s.entries[i].flip_deg;
        p[i] = s.entries[i].phase_deg;
        tr[i] = s.entries[i].tr_ms;
        te[i] = s.entries[i].te_ms;
    }
    mrfg_ctx* h = nullptr;
    check(mrfg_create(f.data(), p.data(), tr.data(), te.data(), static_cast<int64_t>(n), dev, &h));
    return h;
}

// A context for stored-dictionary searches: only the entry length matters.
mrfg_ctx* create_len(std::size_t n) {
    Schedule s;
    s.entries.assign(n, ScheduleEntry{0.0, 0.0, 1.0, 0.5});
    return create(s);
}

mrfg_axis to_axis(const AxisSpec& a) { return {a.min, a.step, static_cast<int64_t>(a.count), nullptr}; }
mrfg_grid to_grid(const ParameterGrid& g) { return {to_axis(g.t1_ms), to_axis(g.t2_ms), to_axis(g.df_hz)}; }

mrfg_zoom_config to_cfg(const ZoomConfig& z) {
    mrfg_zoom_config c;
    mrfg_zoom_config_default(&c);
    c.metric = z.metric == Metric::cc ? MRFG_METRIC_CC : MRFG_METRIC_EUCLIDEAN;
    c.final_metric = z.final_metric == Metric::cc ? MRFG_METRIC_CC : MRFG_METRIC_EUCLIDEAN;
    c.smooth_k = z.smooth_k;
    c.omega_hz = z.omega_hz;
    c.df_coarse_hz = z.df_coarse_hz;
    c.df_refine_hz = z.df_refine_hz;
    c.df_window_hz = z.df_window_hz;
    c.plateau_eps = z.plateau_eps;
    c.heavy_noise_cc = z.heavy_noise_cc;
    c.fallback_coarse_hz = z.fallback_coarse_hz;
    c.fallback_window_hz = z.fallback_window_hz;
    if (z.t1t2_2d_steps_ms.size() > 8 || z.t1t2_1d_steps_ms.size() > 8)
        throw std::invalid_argument("ZoomConfig: at most 8 steps per stage on the GPU");
    c.n2d = static_cast<int32_t>(z.t1t2_2d_steps_ms.size());
    c.n1d = static_cast<int32_t>(z.t1t2_1d_steps_ms.size());
    std::copy(z.t1t2_2d_steps_ms.begin(), z.t1t2_2d_steps_ms.end(), c.t1t2_2d_steps_ms);
    std::copy(z.t1t2_1d_steps_ms.begin(), z.t1t2_1d_steps_ms.end(), c.t1t2_1d_steps_ms);
    c.final_2d_step_ms = z.final_2d_step_ms;
    c.init_t1_ms = z.init_t1_ms;
    c.init_t2_ms = z.init_t2_ms;
    c.prior_window_t1_ms = z.prior_window_t1_ms;
    c.prior_window_t2_ms = z.prior_window_t2_ms;
    c.prior_window_df_hz = z.prior_window_df_hz;
    return c;
}

const double* interleaved(const Fingerprint& fp) {
    return reinterpret_cast<const double*>(fp.s.data());  // std::complex<double> is 2 doubles
}

std::string g9(double x) {
    char b[40];
    std::snprintf(b, sizeof b, "%.9g", x);
    return b;
}

double norm2(const Fingerprint& fp) {  // fingerprint.cpp:14-18
    double acc = 0;
    for (const auto& v : fp.s) acc += v.real() * v.real() + v.imag() * v.imag();
    return std::sqrt(acc);
}

std::vector<std::string> split_csv(const std::string& line) {
    std::vector<std::string> out;
    std::string cur;
    for (char ch : line) {
        if (ch == ',') {
            out.push_back(cur);
            cur.clear();
        } else if (ch != '\r') {
            cur += ch;
        }
    }
    out.push_back(cur);
    return out;
}

double parse_num(const std::string& s) {
    const char* p = s.c_str();
    char* end = nullptr;
    double v = std::strtod(p, &end);
    while (end && *end == ' ') ++end;
    if (end == p || (end && *end != '\0')) throw std::runtime_error("bad numeric field: '" + s + "'");
    return v;
}

QuantResult to_result(const ParameterGrid& lat, const mrfg_quant& q, double seconds) {
    QuantResult r;
    r.params = lat.params_at(static_cast<std::size_t>(q.i1), static_cast<std::size_t>(q.i2),
                             static_cast<std::size_t>(q.idf));
    r.params.pd = q.pd;
    r.score = q.score;
    r.evaluations = static_cast<std::size_t>(q.evaluations);
    r.seconds = seconds;
    return r;
}

// StageLog names (zoom.cpp:179-249, :441-512) by mrfg_stage code.
const char* const kStageNames[] = {"df.coarse", "df.refine", "df.translate", "df.rerefine", "df.plateau_stop",
                                   "df.finest", "df.fallback", "t1t2.2d", "df.sweep", "t1.1d", "t2.1d",
                                   "t1t2.final"};
std::vector<StageLog> to_trace(const mrfg_stage* rec, int count) {
    std::vector<StageLog> out;
    for (int k = 0; k < std::min(count, MRFG_TRACE_MAX); ++k) {
        StageLog lg;
        lg.stage = kStageNames[rec[k].stage];
        lg.evaluations = static_cast<std::size_t>(rec[k].evaluations);
        lg.best = rec[k].best;
        lg.t1_ms = rec[k].t1_ms;
        lg.t2_ms = rec[k].t2_ms;
        lg.df_hz = rec[k].df_hz;
        out.push_back(std::move(lg));
    }
    return out;
}

// df_dict validation of zoom.cpp:61-69 and :430-437.  The slab's payload is
// passed to the GPU, which scores its entries as given for stage-1
// acquisitions (mrfg_zoom_config.dict_mode = 1, zoom.cpp:101-113).
void check_df_dict(const Dictionary* d, const ParameterGrid& lat, const ZoomConfig& cfg,
                   const Schedule& sched) {
    if (!d) return;
    auto close = [](double a, double b) {
        return std::abs(a - b) <= 1e-9 * std::max({1.0, std::abs(a), std::abs(b)});
    };
    if (d->digest != schedule_digest(sched))
        throw std::invalid_argument("objective: df dictionary from another schedule");
    if (d->grid.t1_ms.count != 1 || d->grid.t2_ms.count != 1)
        throw std::invalid_argument("objective: df dictionary must fix T1 and T2");
    if (!close(d->grid.df_hz.min, lat.df_hz.min) || !close(d->grid.df_hz.step, lat.df_hz.step) ||
        d->grid.df_hz.count != lat.df_hz.count)
        throw std::invalid_argument("lattice mismatch: df axis");
    if (d->entry_len != sched.size())
        throw std::invalid_argument("objective: df dictionary entry length mismatch");
    auto snap = [](double v, const AxisSpec& a) { return std::lround((v - a.min) / a.step); };
    long i1 = std::clamp(snap(cfg.init_t1_ms, lat.t1_ms), 0L, static_cast<long>(lat.t1_ms.count) - 1);
    long i2 = std::clamp(snap(cfg.init_t2_ms, lat.t2_ms), 0L, static_cast<long>(lat.t2_ms.count) - 1);
    if (!close(d->grid.t1_ms.value(0), lat.t1_ms.value(static_cast<std::size_t>(i1))))
        throw std::invalid_argument("lattice mismatch: df dictionary T1 vs initial value");
    if (!close(d->grid.t2_ms.value(0), lat.t2_ms.value(static_cast<std::size_t>(i2))))
        throw std::invalid_argument("lattice mismatch: df dictionary T2 vs initial value");
}

// full_dict validation (zoom.cpp:50-58); its payload is scored as given for
// every acquisition (mrfg_zoom_config.dict_mode = 2).
void check_full_dict(const Dictionary* d, const ParameterGrid& lat, const Schedule& sched) {
    if (!d) return;
    auto close = [](double a, double b) {
        return std::abs(a - b) <= 1e-9 * std::max({1.0, std::abs(a), std::abs(b)});
    };
    auto axis = [&](const AxisSpec& a, const AxisSpec& b, const char* what) {
        if (!close(a.min, b.min) || !close(a.step, b.step) || a.count != b.count)
            throw std::invalid_argument(std::string("lattice mismatch: ") + what);
    };
    if (d->digest != schedule_digest(sched))
        throw std::invalid_argument("objective: dictionary built from another schedule");
    axis(d->grid.t1_ms, lat.t1_ms, "t1 axis");
    axis(d->grid.t2_ms, lat.t2_ms, "t2 axis");
    axis(d->grid.df_hz, lat.df_hz, "df axis");
    if (d->entry_len != sched.size()) throw std::invalid_argument("objective: dictionary entry length mismatch");
}

}  // namespace

// ------------------------------------------------------------------ sequence
Schedule build_schedule(std::size_t n, std::uint64_t seed) {
    std::vector<double> f(n), p(n), tr(n), te(n);
    check(mrfg_reference_schedule(static_cast<int64_t>(n), seed, f.data(), p.data(), tr.data(), te.data()));
    Schedule s;
    s.seed = seed;
    s.entries.resize(n);
    for (std::size_t i = 0; i < n; ++i) s.entries[i] = {f[i], p[i], tr[i], te[i]};
    return s;
}

std::string to_csv(const Schedule& sched) {
    std::string out = "idx,flip_deg,phase_deg,tr_ms,te_ms\n";
    for (std::size_t k = 0; k < sched.size(); ++k) {
        const ScheduleEntry& e = sched.entries[k];
        out += std::to_string(k) + ',' + g9(e.flip_deg) + ',' + g9(e.phase_deg) + ',' + g9(e.tr_ms) + ',' +
               g9(e.te_ms) + '\n';
    }
    return out;
}

void save_csv(const Schedule& sched, const std::filesystem::path& path) {
    std::ofstream f(path, std::ios::binary);
    if (!f) throw std::runtime_error("cannot open for write: " + path.string());
    f << to_csv(sched);
    if (!f) throw std::runtime_error("write failed: " + path.string());
}

Schedule load_schedule_csv(const std::filesystem::path& path) {  // sequence.cpp:112-140
    std::ifstream f(path, std::ios::binary);
    if (!f) throw std::runtime_error("cannot open schedule: " + path.string());
    std::string line;
    if (!std::getline(f, line) ||
        split_csv(line) != std::vector<std::string>{"idx", "flip_deg", "phase_deg", "tr_ms", "te_ms"})
        throw std::runtime_error("bad schedule header in " + path.string());
    Schedule s;
    std::size_t expect = 0;
    while (std::getline(f, line)) {
        if (line.empty()) continue;
        auto c = split_csv(line);
        if (c.size() != 5) throw std::runtime_error("bad schedule row in " + path.string() + ": " + line);
        if (static_cast<std::size_t>(parse_num(c[0])) != expect)
            throw std::runtime_error("non-sequential idx in " + path.string());
        ScheduleEntry e{parse_num(c[1]), parse_num(c[2]), parse_num(c[3]), parse_num(c[4])};
        if (e.tr_ms <= 0 || e.te_ms < 0 || e.te_ms > e.tr_ms)
            throw std::runtime_error("invalid timing in " + path.string() + ": " + line);
        s.entries.push_back(e);
        ++expect;
    }
    return s;
}

// --------------------------------------------------------------- fingerprint
Fingerprint normalize(const Fingerprint& fp) {  // fingerprint.cpp:28-37
    const double nn = norm2(fp);
    if (nn == 0) throw std::invalid_argument("normalize: zero fingerprint");
    Fingerprint out;
    out.s.reserve(fp.size());
    const double inv = 1.0 / nn;
    for (const auto& v : fp.s) out.s.emplace_back(v.real() * inv, v.imag() * inv);
    out.unit_norm = true;
    return out;
}

double cc(const Fingerprint& a, const Fingerprint& b) {  // fingerprint.cpp:39-55
    if (a.size() != b.size()) throw std::invalid_argument("cc: length mismatch");
    if (a.size() == 0) throw std::invalid_argument("cc: empty input");
    double re = 0, im = 0;
    for (std::size_t j = 0; j < a.size(); ++j) {
        re += a.s[j].real() * b.s[j].real() + a.s[j].imag() * b.s[j].imag();
        im += a.s[j].imag() * b.s[j].real() - a.s[j].real() * b.s[j].imag();
    }
    double num = std::sqrt(re * re + im * im);
    if (!(a.unit_norm && b.unit_norm)) {
        const double na = norm2(a), nb = norm2(b);
        if (na == 0 || nb == 0) throw std::invalid_argument("cc: zero fingerprint");
        num /= na * nb;
    }
    return num < 1.0 ? num : 1.0;
}

double euclidean(const Fingerprint& a, const Fingerprint& b) {  // fingerprint.cpp:57-66
    if (a.size() != b.size()) throw std::invalid_argument("euclidean: length mismatch");
    if (a.size() == 0) throw std::invalid_argument("euclidean: empty input");
    double acc = 0;
    for (std::size_t j = 0; j < a.size(); ++j) {
        const double dr = a.s[j].real() - b.s[j].real(), di = a.s[j].imag() - b.s[j].imag();
        acc += dr * dr + di * di;
    }
    return std::sqrt(acc);
}

Fingerprint add_noise(const Fingerprint& fp, double sigma, std::uint64_t seed) {
    Fingerprint out;
    out.s.resize(fp.size());
    check(mrfg_add_noise(interleaved(fp), static_cast<int64_t>(fp.size()), sigma, seed,
                         reinterpret_cast<double*>(out.s.data())));
    return out;
}

double calibrate_noise(const Fingerprint& fp, double target_cc, std::uint64_t seed) {
    double sigma = 0;
    check(mrfg_calibrate_noise(interleaved(fp), static_cast<int64_t>(fp.size()), target_cc, seed, &sigma));
    return sigma;
}

CalibratedNoise make_calibrated_noise(const Fingerprint& fp, double target_cc, std::uint64_t seed) {
    CalibratedNoise r;
    r.noisy.s.resize(fp.size());
    uint64_t used = 0;
    check(mrfg_make_calibrated_noise(interleaved(fp), static_cast<int64_t>(fp.size()), target_cc, seed,
                                     &r.sigma, &used, reinterpret_cast<double*>(r.noisy.s.data())));
    r.seed = used;
    return r;
}

Fingerprint smooth(const Fingerprint& fp, int k) {
    Fingerprint out;
    out.s.resize(fp.size());
    check(mrfg_smooth(interleaved(fp), static_cast<int64_t>(fp.size()), k,
                      reinterpret_cast<double*>(out.s.data())));
    return out;
}

void save_csv(const Fingerprint& fp, const std::filesystem::path& path) {  // fingerprint.cpp:154-161
    std::ofstream f(path, std::ios::binary);
    if (!f) throw std::runtime_error("cannot open for write: " + path.string());
    f << "idx,re,im\n";
    for (std::size_t j = 0; j < fp.size(); ++j)
        f << j << ',' << g9(fp.s[j].real()) << ',' << g9(fp.s[j].imag()) << '\n';
    if (!f) throw std::runtime_error("write failed: " + path.string());
}

Fingerprint load_fingerprint_csv(const std::filesystem::path& path) {  // fingerprint.cpp:163-183
    std::ifstream f(path, std::ios::binary);
    if (!f) throw std::runtime_error("cannot open fingerprint: " + path.string());
    std::string line;
    if (!std::getline(f, line) || split_csv(line) != std::vector<std::string>{"idx", "re", "im"})
        throw std::runtime_error("bad fingerprint header in " + path.string());
    Fingerprint fp;
    std::size_t expect = 0;
    while (std::getline(f, line)) {
        if (line.empty()) continue;
        auto cols = split_csv(line);
        if (cols.size() != 3) throw std::runtime_error("bad fingerprint row in " + path.string());
        if (static_cast<std::size_t>(parse_num(cols[0])) != expect)
            throw std::runtime_error("non-sequential idx in " + path.string());
        fp.s.emplace_back(parse_num(cols[1]), parse_num(cols[2]));
        ++expect;
    }
    if (fp.size() == 0) throw std::runtime_error("empty fingerprint: " + path.string());
    return fp;
}

double estimate_pd(const Fingerprint& acquired, const Fingerprint& matched_ideal) {
    if (acquired.size() != matched_ideal.size()) throw std::invalid_argument("estimate_pd: length mismatch");
    if (acquired.size() == 0) throw std::invalid_argument("estimate_pd: empty input");
    const double ni = norm2(matched_ideal);
    if (ni == 0) throw std::invalid_argument("estimate_pd: zero ideal fingerprint");
    return norm2(acquired) / ni;
}

// --------------------------------------------------------------------- bloch
// Host primitives (bloch.cpp:11-93), FP64 in the reference's operand order
// (this file is compiled without FMA contraction, like the reference).
Matrix3 Matrix3::operator*(const Matrix3& o) const {  // bloch.hpp:26-33
    Matrix3 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            r.m[3 * i + j] = m[3 * i] * o.m[j] + m[3 * i + 1] * o.m[3 + j] + m[3 * i + 2] * o.m[6 + j];
    return r;
}

Magnetization Matrix3::operator*(const Magnetization& v) const {  // bloch.hpp:35-38
    return {m[0] * v.x + m[1] * v.y + m[2] * v.z, m[3] * v.x + m[4] * v.y + m[5] * v.z,
            m[6] * v.x + m[7] * v.y + m[8] * v.z};
}

Matrix3 rot(Axis axis, double theta) {  // bloch.cpp:31-53: counterclockwise about a lab axis
    const double c = std::cos(theta), s = std::sin(theta);
    Matrix3 r;
    int a = 0, b = 1;  // the rotated coordinate pair
    if (axis == Axis::X) a = 1, b = 2;
    if (axis == Axis::Y) a = 2, b = 0;  // about y: (z, x) -> r[x][z] = s, r[z][x] = -s
    r.m[4 * a] = c;
    r.m[4 * b] = c;
    r.m[3 * b + a] = s;
    r.m[3 * a + b] = -s;
    return r;
}

Magnetization relax_step(const Magnetization& m, double dt, double t1, double t2) {  // bloch.cpp:55-61
    if (dt < 0 || t1 <= 0 || t2 <= 0)
        throw std::invalid_argument("relax_step: dt must be >= 0 and T1, T2 > 0");
    const double e2 = std::exp(-dt / t2), e1 = std::exp(-dt / t1);
    return {m.x * e2, m.y * e2, 1.0 + (m.z - 1.0) * e1};
}

Matrix3 rf_matrix(const RfPulse& pulse, bool simplified) {  // bloch.cpp:63-78
    if (simplified) return rot(Axis::Z, pulse.phi) * rot(Axis::X, -pulse.alpha) * rot(Axis::Z, -pulse.phi);
    if (pulse.alpha == 0)
        throw std::invalid_argument("rf_matrix: full rotation model is undefined for a zero flip angle");
    if (pulse.tau <= 0) throw std::invalid_argument("rf_matrix: full rotation model needs tau > 0");
    const double beta = std::atan(pulse.tau * pulse.delta_omega / pulse.alpha);
    const double rate = pulse.alpha / pulse.tau;
    const double alpha_eff = -pulse.tau * std::sqrt(pulse.delta_omega * pulse.delta_omega + rate * rate);
    return rot(Axis::Z, pulse.phi) * rot(Axis::Y, beta) * rot(Axis::X, alpha_eff) * rot(Axis::Y, -beta) *
           rot(Axis::Z, -pulse.phi);
}

namespace {
// relax_precess (bloch.cpp:15-27): rotate by 2 pi df dt, scale by E2; recover z.
void relax_precess_host(Magnetization& m, double dt, double inv_t1, double inv_t2, double df) {
    const double e2 = std::exp(-dt * inv_t2), e1 = std::exp(-dt * inv_t1);
    const double a = 6.283185307179586476925286766559 * df * dt;
    const double c = std::cos(a), s = std::sin(a);
    const double x = (m.x * c - m.y * s) * e2, y = (m.x * s + m.y * c) * e2;
    m.x = x;
    m.y = y;
    m.z = 1.0 + (m.z - 1.0) * e1;
}
}  // namespace

std::pair<std::complex<double>, Magnetization> evolve_tr(const Magnetization& m, const RfPulse& pulse, double tr,
                                                         double te, const TissueParams& p) {  // bloch.cpp:80-93
    if (te < 0 || te > tr) throw std::invalid_argument("evolve_tr: need 0 <= te <= tr");
    if (p.t1 <= 0 || p.t2 <= 0) throw std::invalid_argument("evolve_tr: T1 and T2 must be positive");
    Magnetization cur = rf_matrix(pulse) * m;
    relax_precess_host(cur, te, 1.0 / p.t1, 1.0 / p.t2, p.df);
    const std::complex<double> echo(cur.x, cur.y);
    relax_precess_host(cur, tr - te, 1.0 / p.t1, 1.0 / p.t2, p.df);
    return {echo, cur};
}

BlochSimulator::BlochSimulator(const Schedule& sched) : ctx_(create(sched)), n_(sched.size()), sched_(sched) {}

BlochSimulator::BlochSimulator(const BlochSimulator& o) : ctx_(create(o.sched_)), n_(o.n_), sched_(o.sched_) {}

BlochSimulator& BlochSimulator::operator=(const BlochSimulator& o) {
    if (this != &o) {
        mrfg_ctx* c = create(o.sched_);
        if (ctx_) mrfg_destroy(ctx_);
        ctx_ = c;
        n_ = o.n_;
        sched_ = o.sched_;
    }
    return *this;
}

BlochSimulator::~BlochSimulator() {
    if (ctx_) mrfg_destroy(ctx_);
}

void BlochSimulator::simulate(const TissueParams& p, std::complex<double>* out) const {
    const double prm[3] = {p.t1, p.t2, p.df};
    check(mrfg_simulate(ctx_, prm, 1, 64, 0, reinterpret_cast<double*>(out)));
}

Fingerprint BlochSimulator::simulate(const TissueParams& p) const {
    Fingerprint fp;
    fp.s.resize(n_);
    simulate(p, fp.s.data());
    return fp;
}

std::vector<std::complex<double>> BlochSimulator::simulate_batch(const std::vector<TissueParams>& params) const {
    std::vector<double> prm(3 * params.size());
    for (std::size_t k = 0; k < params.size(); ++k) {
        prm[3 * k] = params[k].t1;
        prm[3 * k + 1] = params[k].t2;
        prm[3 * k + 2] = params[k].df;
    }
    std::vector<std::complex<double>> out(n_ * params.size());
    if (!params.empty())
        check(mrfg_simulate(ctx_, prm.data(), static_cast<int64_t>(params.size()), 64, 0,
                            reinterpret_cast<double*>(out.data())));
    return out;
}

Fingerprint simulate_fingerprint(const TissueParams& p, const Schedule& sched) {
    return BlochSimulator(sched).simulate(p);
}

// ---------------------------------------------------------------- dictionary
ParameterGrid grid_from_ranges(const AxisRange& t1, const AxisRange& t2, const AxisRange& df) {
    auto axis = [](const AxisRange& r, const char* name) {
        if (!(r.step > 0)) throw std::invalid_argument(std::string(name) + ": step must be > 0");
        if (!(r.max > r.min)) throw std::invalid_argument(std::string(name) + ": need max > min");
        int64_t c = 0;
        if (mrfg_axis_count(r.min, r.max, r.step, &c) != MRFG_OK)
            throw std::invalid_argument(std::string(name) + ": empty axis");
        return AxisSpec{r.min, r.step, static_cast<std::size_t>(c)};
    };
    return {axis(t1, "t1"), axis(t2, "t2"), axis(df, "df")};
}

Digest schedule_digest(const Schedule& sched) {  // dictionary.cpp:163-171
    const std::string csv = to_csv(sched);
    Digest d{};
    unsigned int n = 0;
    if (EVP_Digest(csv.data(), csv.size(), d.data(), &n, EVP_sha256(), nullptr) != 1 || n != d.size())
        throw std::runtime_error("SHA-256 digest failed");
    return d;
}

std::string digest_hex(const Digest& d) {
    static const char* hex = "0123456789abcdef";
    std::string s;
    for (auto b : d) {
        s += hex[b >> 4];
        s += hex[b & 0xF];
    }
    return s;
}

Dictionary generate(const ParameterGrid& grid, const Schedule& sched, int) {
    if (sched.size() == 0) throw std::invalid_argument("generate: empty schedule");
    CtxGuard c{create(sched)};
    Dictionary d;
    d.grid = grid;
    d.digest = schedule_digest(sched);
    d.entry_len = sched.size();
    d.data.resize(grid.total() * 2 * d.entry_len);
    const mrfg_grid g = to_grid(grid);
    check(mrfg_generate(c.h, &g, 0, static_cast<int64_t>(grid.total()), 64, d.data.data()));
    return d;
}

void save(const Dictionary& dict, const std::filesystem::path& path) {  // dictionary.cpp:196-203
    const mrfg_grid g = to_grid(dict.grid);
    check(mrfg_write_header(path.c_str(), "MRFD", &g, dict.digest.data(), static_cast<int64_t>(dict.entry_len)));
    std::ofstream f(path, std::ios::binary | std::ios::app);
    if (!f) throw std::runtime_error("cannot open for write: " + path.string());
    f.write(reinterpret_cast<const char*>(dict.data.data()),
            static_cast<std::streamsize>(dict.data.size() * sizeof(float)));
    if (!f) throw std::runtime_error("write failed: " + path.string());
}

Dictionary load(const std::filesystem::path& path) {  // dictionary.cpp:205-220
    mrfg_grid g{};
    Dictionary d;
    int64_t el = 0, off = 0;
    check(mrfg_read_header(path.c_str(), "MRFD", &g, d.digest.data(), &el, &off));
    auto axis = [](const mrfg_axis& a) { return AxisSpec{a.min, a.step, static_cast<std::size_t>(a.count)}; };
    d.grid = {axis(g.t1_ms), axis(g.t2_ms), axis(g.df_hz)};
    d.entry_len = static_cast<std::size_t>(el);
    d.data.resize(d.grid.total() * 2 * d.entry_len);
    std::ifstream f(path, std::ios::binary);
    f.seekg(off);
    f.read(reinterpret_cast<char*>(d.data.data()), static_cast<std::streamsize>(d.data.size() * sizeof(float)));
    if (f.gcount() != static_cast<std::streamsize>(d.data.size() * sizeof(float)))
        throw std::runtime_error("truncated payload in " + path.string());
    return d;
}

void save_generated(const ParameterGrid& grid, const Schedule& sched, const std::filesystem::path& path,
                    int, std::size_t chunk_entries) {  // dictionary.cpp:216-239
    if (chunk_entries == 0) throw std::invalid_argument("chunk_entries must be > 0");
    if (sched.size() == 0) throw std::invalid_argument("generate: empty schedule");
    CtxGuard c{create(sched)};
    const mrfg_grid g = to_grid(grid);
    const Digest dg = schedule_digest(sched);
    check(mrfg_save_generated(c.h, &g, dg.data(), path.c_str(), static_cast<int64_t>(chunk_entries), 64));
}

Match brute_force_search(const Fingerprint& fp, const Dictionary& dict, Metric metric) {
    if (fp.size() != dict.entry_len)
        throw std::invalid_argument("query length does not match dictionary entries");
    CtxGuard c{create_len(dict.entry_len)};
    mrfg_match m;
    // prep_query (dictionary.cpp:145-150): a unit_norm query is used as given
    const uint8_t unit = fp.unit_norm ? 1 : 0;
    mrfg_scan_opts o{};
    o.unit_queries = &unit;
    check(mrfg_scan_dict(c.h, dict.data.data(), static_cast<int64_t>(dict.grid.total()), interleaved(fp), 1,
                         metric == Metric::cc ? MRFG_METRIC_CC : MRFG_METRIC_EUCLIDEAN, &o, &m, nullptr));
    const auto u = dict.grid.unflatten(static_cast<std::size_t>(m.flat));
    return {dict.grid.params_at(u.i1, u.i2, u.idf), m.score, dict.grid.total()};
}

ScanOutcome scan_grid(const ParameterGrid& grid, const Schedule& sched,
                      const std::vector<Fingerprint>& queries, Metric metric, int,
                      std::size_t chunk_entries) {
    if (queries.empty()) throw std::invalid_argument("scan_grid: no queries");
    if (chunk_entries == 0) throw std::invalid_argument("chunk_entries must be > 0");
    for (const auto& q : queries)
        if (q.size() != sched.size())
            throw std::invalid_argument("query length does not match dictionary entries");
    const std::size_t n = sched.size(), nq = queries.size();
    std::vector<double> flat(2 * n * nq);
    std::vector<uint8_t> unit(nq);  // prep_query: unit_norm queries are used as given
    for (std::size_t k = 0; k < nq; ++k) {
        std::memcpy(&flat[2 * n * k], interleaved(queries[k]), 16 * n);
        unit[k] = queries[k].unit_norm ? 1 : 0;
    }
    const mrfg_grid g = to_grid(grid);
    // atom shards: contiguous T1 slabs, one per listed device
    const std::vector<int> devs = devices();
    const std::size_t row = grid.t2_ms.count * grid.df_hz.count;
    const std::size_t rows_per = (grid.t1_ms.count + devs.size() - 1) / devs.size();
    std::vector<std::vector<mrfg_match>> part(devs.size(), std::vector<mrfg_match>(nq, mrfg_match{-1, 0.0}));
    std::vector<mrfg_scan_stats> sts(devs.size());
    on_shards(devs.size(), [&](std::size_t k) {
        const std::size_t fb = std::min(grid.total(), k * rows_per * row);
        const std::size_t fe = std::min(grid.total(), (k + 1) * rows_per * row);
        if (fe <= fb) return;
        CtxGuard c{create(sched, devs[k])};
        mrfg_scan_opts o{};
        o.unit_queries = unit.data();
        check(mrfg_scan_grid(c.h, &g, static_cast<int64_t>(fb), static_cast<int64_t>(fe), flat.data(),
                             static_cast<int64_t>(nq), metric == Metric::cc ? MRFG_METRIC_CC : MRFG_METRIC_EUCLIDEAN,
                             &o, part[k].data(), &sts[k]));
    });
    // merge: highest score, lowest flat on ties (dictionary.cpp:291-294)
    std::vector<mrfg_match> m(nq, mrfg_match{-1, 0.0});
    for (const auto& pm : part)
        for (std::size_t q = 0; q < nq; ++q)
            if (pm[q].flat >= 0 && (m[q].flat < 0 || pm[q].score > m[q].score ||
                                    (pm[q].score == m[q].score && pm[q].flat < m[q].flat)))
                m[q] = pm[q];
    mrfg_scan_stats st{};
    for (const auto& x : sts) {  // the shards run concurrently: the slowest one's times
        st.gemm_ms = std::max(st.gemm_ms, x.gemm_ms);
        st.rerank_ms = std::max(st.rerank_ms, x.rerank_ms);
        st.bloch_ms = std::max(st.bloch_ms, x.bloch_ms);
    }
    ScanOutcome out;
    for (std::size_t k = 0; k < nq; ++k) {
        const auto u = grid.unflatten(static_cast<std::size_t>(m[k].flat));
        out.matches.push_back({grid.params_at(u.i1, u.i2, u.idf), m[k].score, grid.total()});
    }
    // the scan is one batched GPU pass: its match time is shared evenly
    out.scan_seconds.assign(nq, (st.gemm_ms + st.rerank_ms) * 1e-3 / static_cast<double>(nq));
    out.generate_seconds = st.bloch_ms * 1e-3;
    return out;
}

void cc_map(const Fingerprint& fp, const ParameterGrid& grid, const Schedule& sched,
            const std::function<void(std::size_t, std::span<const float>)>& sink, int,
            std::size_t chunk_entries) {
    if (chunk_entries == 0) throw std::invalid_argument("chunk_entries must be > 0");
    if (fp.size() != sched.size())
        throw std::invalid_argument("query length does not match dictionary entries");
    CtxGuard c{create(sched)};
    const mrfg_grid g = to_grid(grid);
    std::vector<float> scores;
    for (std::size_t begin = 0; begin < grid.total(); begin += chunk_entries) {
        const std::size_t end = std::min(grid.total(), begin + chunk_entries);
        scores.resize(end - begin);
        check(mrfg_cc_map(c.h, &g, interleaved(fp), static_cast<int64_t>(begin),
                          static_cast<int64_t>(end - begin), scores.data()));
        sink(begin, {scores.data(), scores.size()});
    }
}

void cc_map_to_file(const Fingerprint& fp, const ParameterGrid& grid, const Schedule& sched,
                    const std::filesystem::path& path, int) {  // dictionary.cpp:333-347
    if (fp.size() != sched.size())
        throw std::invalid_argument("query length does not match dictionary entries");
    CtxGuard c{create(sched)};
    const mrfg_grid g = to_grid(grid);
    const Digest dg = schedule_digest(sched);
    check(mrfg_cc_map_to_file(c.h, &g, interleaved(fp), dg.data(), path.c_str(), 64));
}

// ---------------------------------------------------------------------- zoom
// Generic forms over caller objectives (zoom.cpp:173-399), host-side.
long search_df(const std::function<double(long)>& f, long lo, long hi, const DfSearchParams& prm,
               const std::function<void(const char*, long, double)>& stage) {
    if (lo > hi) throw std::invalid_argument("search_df: empty range");
    if (prm.coarse <= 0 || prm.refine <= 0 || prm.finest <= 0 || prm.omega <= 0)
        throw std::invalid_argument("search_df: steps must be positive");
    struct B {
        long idx = -1;
        double val = -1e300;
        void offer(long i, double v) {
            if (v > val) {
                val = v;
                idx = i;
            }
        }
    };
    auto note = [&](const char* name, const B& b) {
        if (stage) stage(name, b.idx, b.val);
    };
    auto sweep = [&](long a, long b, long step, B& best) {
        a = std::clamp(a, lo, hi);
        b = std::clamp(b, lo, hi);
        for (long x = a; x <= b; x += step) best.offer(x, f(x));
        if ((b - a) % step != 0) best.offer(b, f(b));
    };
    auto run = [&](long coarse, long wh) -> B {
        std::vector<double> marks;
        auto flat3 = [&] {
            if (marks.size() < 3) return false;
            auto [mn, mx] = std::minmax_element(marks.end() - 3, marks.end());
            return *mx - *mn < prm.plateau_eps;
        };
        B cur;
        sweep(lo, hi, coarse, cur);
        note("df.coarse", cur);
        marks.push_back(cur.val);
        B r = cur;
        sweep(cur.idx - wh, cur.idx + wh, prm.refine, r);
        cur = r;
        note("df.refine", cur);
        marks.push_back(cur.val);
        for (int round = 0; round < 8; ++round) {
            B t = cur;
            for (long k = 1; cur.idx + k * prm.omega <= hi; ++k) t.offer(cur.idx + k * prm.omega, f(cur.idx + k * prm.omega));
            for (long k = 1; cur.idx - k * prm.omega >= lo; ++k) t.offer(cur.idx - k * prm.omega, f(cur.idx - k * prm.omega));
            note("df.translate", t);
            if (t.idx == cur.idx) break;
            B rr = t;
            sweep(t.idx - wh, t.idx + wh, prm.refine, rr);
            cur = rr;
            note("df.rerefine", cur);
            marks.push_back(cur.val);
            if (flat3()) {
                note("df.plateau_stop", cur);
                return cur;
            }
        }
        if (flat3()) {
            note("df.plateau_stop", cur);
            return cur;
        }
        B fin = cur;
        sweep(cur.idx - prm.omega / 2, cur.idx + prm.omega / 2, prm.finest, fin);
        note("df.finest", fin);
        return fin;
    };
    B m = run(prm.coarse, prm.window_half);
    if (prm.allow_fallback && m.val < prm.heavy_cc) {
        B fb = run(prm.fallback_coarse, prm.fallback_window_half);
        note("df.fallback", fb);
        if (fb.val > m.val) return fb.idx;
    }
    return m.idx;
}

long zoom_1d(const std::function<double(long)>& f, long lo, long hi, long init, std::span<const long> steps) {
    if (lo > hi) throw std::invalid_argument("zoom_1d: empty range");
    long x = std::clamp(init, lo, hi);
    double fx = f(x);
    for (long s : steps) {
        if (s <= 0) throw std::invalid_argument("zoom_1d: step must be positive");
        bool moved = true;
        while (moved) {
            moved = false;
            for (long cand : {std::clamp(x - s, lo, hi), std::clamp(x + s, lo, hi)}) {
                if (cand == x) continue;
                const double fc = f(cand);
                if (fc > fx) {
                    x = cand;
                    fx = fc;
                    moved = true;
                    break;
                }
            }
        }
    }
    return x;
}

std::pair<long, long> zoom_2d(const std::function<double(long, long)>& f, long lo1, long hi1, long lo2,
                              long hi2, long init1, long init2, std::span<const std::pair<long, long>> steps) {
    if (lo1 > hi1 || lo2 > hi2) throw std::invalid_argument("zoom_2d: empty range");
    long x = std::clamp(init1, lo1, hi1), y = std::clamp(init2, lo2, hi2);
    double fc = f(x, y);
    long bx = x, by = y;
    double bf = fc;
    auto seen = [&](long px, long py, double v) {
        if (v > bf) {
            bf = v;
            bx = px;
            by = py;
        }
    };
    auto probe = [&](long px, long py) {
        const double v = f(px, py);
        seen(px, py, v);
        return v;
    };
    for (auto [s1, s2] : steps) {
        if (s1 <= 0 || s2 <= 0) throw std::invalid_argument("zoom_2d: step must be positive");
        const long cap = 4 * ((hi1 - lo1) / s1 + (hi2 - lo2) / s2) + 16;
        bool done = false;
        for (long it = 0; it < cap && !done; ++it) {
            const long xl = std::clamp(x - s1, lo1, hi1), xr = std::clamp(x + s1, lo1, hi1);
            const long yd = std::clamp(y - s2, lo2, hi2), yu = std::clamp(y + s2, lo2, hi2);
            const double fl = xl != x ? probe(xl, y) : fc;
            const double fd = yd != y ? probe(x, yd) : fc;
            const bool lw = xl != x && fl > fc, dw = yd != y && fd > fc;
            if (lw && dw) {
                x = xl;
                y = yd;
                fc = probe(x, y);
            } else if (!lw && !dw) {
                const double fr = xr != x ? probe(xr, y) : fc;
                const double fu = yu != y ? probe(x, yu) : fc;
                const bool rw = xr != x && fr > fc, uw = yu != y && fu > fc;
                if (rw && uw) {
                    x = xr;
                    y = yu;
                    fc = probe(x, y);
                } else if (rw) {
                    x = xr;
                    fc = fr;
                } else if (uw) {
                    y = yu;
                    fc = fu;
                } else {
                    done = true;
                }
            } else if (lw) {
                const double fu = yu != y ? probe(x, yu) : fc;
                if (yu != y && fu > fc) {
                    x = xl;
                    y = yu;
                    fc = probe(x, y);
                } else {
                    x = xl;
                    fc = fl;
                }
            } else {
                const double fr = xr != x ? probe(xr, y) : fc;
                if (xr != x && fr > fc) {
                    x = xr;
                    y = yd;
                    fc = probe(x, y);
                } else {
                    y = yd;
                    fc = fd;
                }
            }
        }
        if (!done) {
            x = bx;
            y = by;
            fc = bf;
        }
    }
    return {x, y};
}

// ------------------------------------------------------------------ Objective
// zoom.cpp:41-156: lattice-key memo; acquisitions simulate on the GPU in FP64
// (bit-identical entries) or read the caller's dictionary entry.
namespace {
constexpr long kMaxAxis = 1L << 21;
std::uint64_t key_of(long i1, long i2, long idf) {  // zoom.cpp:14-19
    return (static_cast<std::uint64_t>(i1) << 42) | (static_cast<std::uint64_t>(i2) << 21) |
           static_cast<std::uint64_t>(idf);
}
void check_close_axis(const AxisSpec& a, const AxisSpec& b, const char* what) {  // zoom.cpp:27-37
    auto close = [](double x, double y) {
        return std::abs(x - y) <= 1e-9 * std::max({1.0, std::abs(x), std::abs(y)});
    };
    if (!close(a.min, b.min) || !close(a.step, b.step) || a.count != b.count)
        throw std::invalid_argument(std::string("lattice mismatch: ") + what);
}
}  // namespace

Objective::Objective(const Fingerprint& query, const ParameterGrid& lattice, const Schedule& sched,
                     const Options& opt)
    : lattice_(lattice), sim_(sched), opt_(opt) {
    if (query.size() != sched.size())
        throw std::invalid_argument("objective: query length does not match schedule");
    for (const AxisSpec* ax : {&lattice.t1_ms, &lattice.t2_ms, &lattice.df_hz})
        if (ax->count == 0 || ax->count >= static_cast<std::size_t>(kMaxAxis))
            throw std::invalid_argument("objective: lattice axis empty or too fine");
    query_ = normalize(opt_.smooth_k ? smooth(query, opt_.smooth_k) : query).s;
    if (opt_.full_dict) {
        if (opt_.full_dict->digest != schedule_digest(sched))
            throw std::invalid_argument("objective: dictionary built from another schedule");
        check_close_axis(opt_.full_dict->grid.t1_ms, lattice.t1_ms, "t1 axis");
        check_close_axis(opt_.full_dict->grid.t2_ms, lattice.t2_ms, "t2 axis");
        check_close_axis(opt_.full_dict->grid.df_hz, lattice.df_hz, "df axis");
        if (opt_.full_dict->entry_len != sched.size())
            throw std::invalid_argument("objective: dictionary entry length mismatch");
    }
    if (opt_.df_dict) {
        if (opt_.df_dict->digest != schedule_digest(sched))
            throw std::invalid_argument("objective: df dictionary from another schedule");
        if (opt_.df_dict->grid.t1_ms.count != 1 || opt_.df_dict->grid.t2_ms.count != 1)
            throw std::invalid_argument("objective: df dictionary must fix T1 and T2");
        check_close_axis(opt_.df_dict->grid.df_hz, lattice.df_hz, "df axis");
        if (opt_.df_dict->entry_len != sched.size())
            throw std::invalid_argument("objective: df dictionary entry length mismatch");
    }
}

Objective::~Objective() = default;

double Objective::score_from_entry(const std::vector<std::complex<double>>& e, Metric metric) const {
    if (metric == Metric::cc) {  // zoom.cpp:74-84
        double re = 0, im = 0;
        for (std::size_t j = 0; j < query_.size(); ++j) {
            re += query_[j].real() * e[j].real() + query_[j].imag() * e[j].imag();
            im += query_[j].imag() * e[j].real() - query_[j].real() * e[j].imag();
        }
        const double v = std::sqrt(re * re + im * im);
        return v < 1.0 ? v : 1.0;
    }
    double acc = 0;  // zoom.cpp:85-91
    for (std::size_t j = 0; j < query_.size(); ++j) {
        const double dr = query_[j].real() - e[j].real(), di = query_[j].imag() - e[j].imag();
        acc += dr * dr + di * di;
    }
    return -std::sqrt(acc);
}

const std::vector<std::complex<double>>& Objective::acquire(long i1, long i2, long idf, bool df_stage) {
    const std::uint64_t k = key_of(i1, i2, idf);  // zoom.cpp:94-123
    if (auto it = entries_.find(k); it != entries_.end()) return it->second;
    std::vector<std::complex<double>> entry;
    if (opt_.full_dict || (df_stage && opt_.df_dict)) {
        const Dictionary* d = opt_.full_dict ? opt_.full_dict : opt_.df_dict;
        const std::size_t flat = opt_.full_dict ? d->grid.flatten(static_cast<std::size_t>(i1),
                                                                  static_cast<std::size_t>(i2),
                                                                  static_cast<std::size_t>(idf))
                                                : static_cast<std::size_t>(idf);
        auto raw = d->entry(flat);
        Fingerprint f;
        f.s.reserve(d->entry_len);
        for (std::size_t j = 0; j < d->entry_len; ++j) f.s.emplace_back(raw[2 * j], raw[2 * j + 1]);
        entry = opt_.smooth_k ? normalize(smooth(f, opt_.smooth_k)).s : std::move(f.s);
    } else {
        Fingerprint f = sim_.simulate(lattice_.params_at(static_cast<std::size_t>(i1), static_cast<std::size_t>(i2),
                                                          static_cast<std::size_t>(idf)));
        entry = normalize(opt_.smooth_k ? smooth(f, opt_.smooth_k) : f).s;
    }
    ++evals_;
    return entries_.emplace(k, std::move(entry)).first->second;
}

double Objective::eval(long i1, long i2, long idf, Metric metric) {  // zoom.cpp:125-138
    if (i1 < 0 || i2 < 0 || idf < 0 || i1 >= static_cast<long>(lattice_.t1_ms.count) ||
        i2 >= static_cast<long>(lattice_.t2_ms.count) || idf >= static_cast<long>(lattice_.df_hz.count))
        throw std::out_of_range("objective: lattice index out of range");
    auto& memo = metric == Metric::cc ? memo_cc_ : memo_euc_;
    const std::uint64_t k = key_of(i1, i2, idf);
    if (auto it = memo.find(k); it != memo.end()) return it->second;
    const double s = score_from_entry(acquire(i1, i2, idf, false), metric);
    memo.emplace(k, s);
    return s;
}

double Objective::eval_df_stage(long i1, long i2, long idf, Metric metric) {  // zoom.cpp:140-150
    if (idf < 0 || idf >= static_cast<long>(lattice_.df_hz.count))
        throw std::out_of_range("objective: lattice index out of range");
    auto& memo = metric == Metric::cc ? memo_cc_ : memo_euc_;
    const std::uint64_t k = key_of(i1, i2, idf);
    if (auto it = memo.find(k); it != memo.end()) return it->second;
    const double s = score_from_entry(acquire(i1, i2, idf, true), metric);
    memo.emplace(k, s);
    return s;
}

Fingerprint Objective::ideal_at(long i1, long i2, long idf) const {  // zoom.cpp:152-156
    return sim_.simulate(lattice_.params_at(static_cast<std::size_t>(i1), static_cast<std::size_t>(i2),
                                            static_cast<std::size_t>(idf)));
}

std::vector<QuantResult> quantify_batch(const std::vector<Fingerprint>& fps, const SearchRanges& ranges,
                                        const ZoomConfig& cfg, const Schedule& sched, const Dictionary* df_dict,
                                        const Dictionary* full_dict) {
    const ParameterGrid lat = grid_from_ranges(ranges.t1_ms, ranges.t2_ms, ranges.df_hz);
    check_full_dict(full_dict, lat, sched);
    check_df_dict(df_dict, lat, cfg, sched);
    for (const auto& fp : fps)
        if (fp.size() != sched.size())
            throw std::invalid_argument("objective: query length does not match schedule");
    std::vector<QuantResult> out;
    if (fps.empty()) return out;
    const std::size_t n = sched.size();
    std::vector<double> flat(2 * n * fps.size());
    for (std::size_t k = 0; k < fps.size(); ++k) std::memcpy(&flat[2 * n * k], interleaved(fps[k]), 16 * n);
    const mrfg_grid g = to_grid(lat);
    mrfg_zoom_config zc = to_cfg(cfg);
    zc.dict_mode = full_dict ? 2 : (df_dict ? 1 : 0);
    const Dictionary* d = full_dict ? full_dict : df_dict;
    std::vector<mrfg_quant> q(fps.size());
    std::vector<mrfg_stage> rec(MRFG_TRACE_MAX * fps.size());
    std::vector<int32_t> len(fps.size());
    const auto t0 = std::chrono::steady_clock::now();
    // voxel shards: contiguous blocks, one per listed device
    const std::vector<int> devs = devices();
    const std::size_t per = (fps.size() + devs.size() - 1) / devs.size();
    on_shards(devs.size(), [&](std::size_t k) {
        const std::size_t vb = std::min(fps.size(), k * per), ve = std::min(fps.size(), (k + 1) * per);
        if (ve <= vb) return;
        CtxGuard c{create(sched, devs[k])};
        mrfg_zoom_io io{};
        io.dict = d ? d->data.data() : nullptr;
        io.dict_entries = d ? static_cast<int64_t>(d->data.size() / (2 * n)) : 0;
        io.trace = rec.data() + MRFG_TRACE_MAX * vb;
        io.trace_len = len.data() + vb;
        check(mrfg_quantify_ex(c.h, &g, &zc, flat.data() + 2 * n * vb, static_cast<int64_t>(ve - vb), nullptr,
                               nullptr, &io, q.data() + vb));
    });
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    for (std::size_t k = 0; k < q.size(); ++k) {
        out.push_back(to_result(lat, q[k], secs / static_cast<double>(fps.size())));
        out.back().trace = to_trace(rec.data() + MRFG_TRACE_MAX * k, len[k]);
    }
    return out;
}

QuantResult quantify(const Fingerprint& fp, const SearchRanges& ranges, const ZoomConfig& cfg,
                     const Schedule& sched, const Dictionary* df_dict, const Dictionary* full_dict) {
    return quantify_batch({fp}, ranges, cfg, sched, df_dict, full_dict).at(0);
}

Dictionary make_df_dictionary(const SearchRanges& ranges, const ZoomConfig& cfg, const Schedule& sched,
                              int workers) {  // zoom.cpp:541-553
    const ParameterGrid lat = grid_from_ranges(ranges.t1_ms, ranges.t2_ms, ranges.df_hz);
    auto snap = [](double v, const AxisSpec& a) { return std::lround((v - a.min) / a.step); };
    const long i1 = std::clamp(snap(cfg.init_t1_ms, lat.t1_ms), 0L, static_cast<long>(lat.t1_ms.count) - 1);
    const long i2 = std::clamp(snap(cfg.init_t2_ms, lat.t2_ms), 0L, static_cast<long>(lat.t2_ms.count) - 1);
    const double t1 = lat.t1_ms.value(static_cast<std::size_t>(i1)), t2 = lat.t2_ms.value(static_cast<std::size_t>(i2));
    return generate(grid_from_ranges({t1, t1 + lat.t1_ms.step, lat.t1_ms.step},
                                     {t2, t2 + lat.t2_ms.step, lat.t2_ms.step}, ranges.df_hz),
                    sched, workers);
}

SliceResult quantify_slice(const std::vector<Fingerprint>& fps, const std::vector<std::uint8_t>& mask, int nx,
                           int ny, const SearchRanges& ranges, const ZoomConfig& cfg, const Schedule& sched,
                           bool use_prior, int, const Dictionary* df_dict) {
    const auto nv = static_cast<std::size_t>(nx) * static_cast<std::size_t>(ny);
    if (nx <= 0 || ny <= 0 || fps.size() != nv || mask.size() != nv)
        throw std::invalid_argument("quantify_slice: inconsistent raster dimensions");
    const ParameterGrid lat = grid_from_ranges(ranges.t1_ms, ranges.t2_ms, ranges.df_hz);
    check_df_dict(df_dict, lat, cfg, sched);
    if (!use_prior && devices().size() > 1) {
        // independent voxels (zoom.cpp:616-624): voxel shards over the devices
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<Fingerprint> sel;
        std::vector<std::size_t> idx;
        for (std::size_t i = 0; i < nv; ++i)
            if (mask[i]) {
                sel.push_back(fps[i]);
                idx.push_back(i);
            }
        const std::vector<QuantResult> r = quantify_batch(sel, ranges, cfg, sched, df_dict, nullptr);
        SliceResult out;
        out.nx = nx;
        out.ny = ny;
        for (auto* v : {&out.t1_ms, &out.t2_ms, &out.df_hz, &out.pd, &out.score}) v->assign(nv, 0);
        out.evaluations.assign(nv, 0);
        for (std::size_t k = 0; k < idx.size(); ++k) {
            const std::size_t i = idx[k];
            out.t1_ms[i] = r[k].params.t1 * 1e3;  // zoom.cpp:581-586
            out.t2_ms[i] = r[k].params.t2 * 1e3;
            out.df_hz[i] = r[k].params.df;
            out.pd[i] = r[k].params.pd;
            out.score[i] = r[k].score;
            out.evaluations[i] = r[k].evaluations;
            out.total_evaluations += r[k].evaluations;
        }
        out.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        return out;
    }
    CtxGuard c{create(sched)};
    const std::size_t n = sched.size();
    std::vector<double> flat(2 * n * nv, 0.0);
    for (std::size_t i = 0; i < nv; ++i)
        if (mask[i]) {
            if (fps[i].size() != n) throw std::invalid_argument("objective: query length does not match schedule");
            std::memcpy(&flat[2 * n * i], interleaved(fps[i]), 16 * n);
        }
    const mrfg_grid g = to_grid(lat);
    mrfg_zoom_config zc = to_cfg(cfg);
    zc.dict_mode = df_dict ? 1 : 0;
    std::vector<mrfg_quant> q(nv);
    double secs = 0;
    mrfg_zoom_io io{};
    io.dict = df_dict ? df_dict->data.data() : nullptr;
    io.dict_entries = df_dict ? static_cast<int64_t>(df_dict->data.size() / (2 * n)) : 0;
    check(mrfg_quantify_slice_ex(c.h, &g, &zc, flat.data(), mask.data(), nx, ny, use_prior ? 1 : 0, &io, q.data(),
                                 &secs));
    if (use_prior && df_dict) {
        // quantify_impl's df_dict check (zoom.cpp:430-437) for every voxel
        // after the first: its initial T1/T2 are the previous voxel's answer
        // (zoom.cpp:593-597), clamped into its prior window; the reference
        // throws at the first voxel whose start is not the slab's T1/T2.
        auto close = [](double a, double b) {
            return std::abs(a - b) <= 1e-9 * std::max({1.0, std::abs(a), std::abs(b)});
        };
        auto snap = [](double v, const AxisSpec& a) { return std::lround((v - a.min) / a.step); };
        auto units = [](double st, double fine) { return std::max(1L, std::lround(st / fine)); };
        long prev = -1;
        for (std::size_t i = 0; i < nv; ++i) {
            if (!mask[i]) continue;
            if (prev >= 0) {
                const double t1 = lat.t1_ms.value(static_cast<std::size_t>(q[prev].i1)) * 1e-3 * 1e3;
                const double t2 = lat.t2_ms.value(static_cast<std::size_t>(q[prev].i2)) * 1e-3 * 1e3;
                const long p1 = snap(t1, lat.t1_ms), p2 = snap(t2, lat.t2_ms);
                const long w1 = units(cfg.prior_window_t1_ms, lat.t1_ms.step);
                const long w2 = units(cfg.prior_window_t2_ms, lat.t2_ms.step);
                const long lo1 = std::max(0L, p1 - w1), hi1 = std::min<long>(lat.t1_ms.count - 1, p1 + w1);
                const long lo2 = std::max(0L, p2 - w2), hi2 = std::min<long>(lat.t2_ms.count - 1, p2 + w2);
                const long i1 = std::clamp(p1, lo1, hi1), i2 = std::clamp(p2, lo2, hi2);
                if (!close(df_dict->grid.t1_ms.value(0), lat.t1_ms.value(static_cast<std::size_t>(i1))))
                    throw std::invalid_argument("lattice mismatch: df dictionary T1 vs initial value");
                if (!close(df_dict->grid.t2_ms.value(0), lat.t2_ms.value(static_cast<std::size_t>(i2))))
                    throw std::invalid_argument("lattice mismatch: df dictionary T2 vs initial value");
            }
            prev = static_cast<long>(i);
        }
    }
    SliceResult out;
    out.nx = nx;
    out.ny = ny;
    out.t1_ms.assign(nv, 0);
    out.t2_ms.assign(nv, 0);
    out.df_hz.assign(nv, 0);
    out.pd.assign(nv, 0);
    out.score.assign(nv, 0);
    out.evaluations.assign(nv, 0);
    for (std::size_t i = 0; i < nv; ++i) {
        if (!mask[i]) continue;
        const QuantResult r = to_result(lat, q[i], 0);
        out.t1_ms[i] = r.params.t1 * 1e3;  // zoom.cpp:581-586
        out.t2_ms[i] = r.params.t2 * 1e3;
        out.df_hz[i] = r.params.df;
        out.pd[i] = r.params.pd;
        out.score[i] = r.score;
        out.evaluations[i] = r.evaluations;
        out.total_evaluations += r.evaluations;
    }
    out.seconds = secs;
    return out;
}

}  // namespace mrf
