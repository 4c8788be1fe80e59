// synth.cpp -- host-side input synthesis for the DGS path (C ABI, no GPU).
//
// Restates the reference's input generators so the product can build the
// BASELINE.json workloads without the reference: the counter RNG
// (proj/include/mrf/rng.hpp:13-41), %.9g canonicalisation (util.hpp:19-23),
// build_schedule (sequence.cpp:17-92), add_noise (fingerprint.cpp:68-78) and
// the endpoint-exclusive axis rule (dictionary.cpp:25-33).  Compiled without
// FMA contraction so the doubles equal the reference's.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "mrfg.h"

namespace {

thread_local std::string g_synth_err;

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;
constexpr double kDeg2Rad = 0.017453292519943295;

uint64_t mix64(uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}

double quantize9(double x) {
    char buf[40];
    std::snprintf(buf, sizeof buf, "%.9g", x);
    return std::strtod(buf, nullptr);
}

double perlin1d(uint64_t seed, double x) {
    double fx = std::floor(x);
    auto i0 = static_cast<int64_t>(fx);
    double t = x - fx;
    double n0 = (2.0 * mrfg_rng_uniform01(seed, 1, static_cast<uint64_t>(i0)) - 1.0) * t;
    double n1 = (2.0 * mrfg_rng_uniform01(seed, 1, static_cast<uint64_t>(i0 + 1)) - 1.0) * (t - 1.0);
    double u = t * t * t * (t * (6.0 * t - 15.0) + 10.0);
    return n0 + u * (n1 - n0);
}

void remap(std::vector<double>& v, double lo, double hi) {
    if (v.empty()) return;
    double mn = v[0], mx = v[0];
    for (double x : v) {
        mn = x < mn ? x : mn;
        mx = x > mx ? x : mx;
    }
    if (mx == mn) {
        for (double& x : v) x = lo;
        return;
    }
    double scale = (hi - lo) / (mx - mn);
    for (double& x : v) x = lo + (x - mn) * scale;
}

}  // namespace

extern "C" {

uint64_t mrfg_rng_at(uint64_t seed, uint64_t stream, uint64_t index) {
    uint64_t s = mix64(seed + kGolden * (stream + 1));
    return mix64(s + kGolden * (index + 1));
}

double mrfg_rng_uniform01(uint64_t seed, uint64_t stream, uint64_t index) {
    return static_cast<double>(mrfg_rng_at(seed, stream, index) >> 11) * 0x1.0p-53;
}

double mrfg_rng_gaussian(uint64_t seed, uint64_t stream, uint64_t index) {
    double u1 = mrfg_rng_uniform01(seed, stream, 2 * index);
    double u2 = mrfg_rng_uniform01(seed, stream, 2 * index + 1);
    double r = std::sqrt(-2.0 * std::log1p(-u1));
    return r * std::cos(6.283185307179586476925286766559 * u2);
}

int mrfg_reference_schedule(int64_t n, uint64_t seed, double* flip_deg, double* phase_deg,
                            double* tr_ms, double* te_ms) {
    if (n < 0) return MRFG_E_INVALID;
    std::vector<double> flips(n), trs(n);
    for (int64_t k = 0; k < n; ++k) flips[k] = perlin1d(seed, static_cast<double>(k) / 16.0);
    remap(flips, 0.0, 79.0 * kDeg2Rad);
    for (int64_t k = 0; k < n; ++k) trs[k] = mrfg_rng_gaussian(seed, 2, static_cast<uint64_t>(k));
    remap(trs, 0.0, 6e-3);
    for (double& x : trs) x += 14e-3;
    const double cycle[4] = {0.0, 90.0 * kDeg2Rad, 180.0 * kDeg2Rad, 90.0 * kDeg2Rad};
    for (int64_t k = 0; k < n; ++k) {
        flip_deg[k] = quantize9(flips[k] / kDeg2Rad);
        phase_deg[k] = quantize9(cycle[k % 4] / kDeg2Rad);
        tr_ms[k] = quantize9(trs[k] * 1e3);
        te_ms[k] = quantize9(trs[k] * 1e3 / 2.0);
    }
    return MRFG_OK;
}

int mrfg_baseline_schedule(int64_t n, uint64_t seed, double* flip_deg, double* phase_deg,
                           double* tr_ms, double* te_ms) {
    if (n < 0) return MRFG_E_INVALID;
    for (int64_t j = 0; j < n; ++j) {
        double fa = 10.0 + 50.0 * std::fabs(std::sin(2.0 * M_PI * static_cast<double>(j) / 250.0)) +
                    2.0 * mrfg_rng_gaussian(seed, 1, static_cast<uint64_t>(j));
        double tr = quantize9(10.5 + 3.5 * mrfg_rng_uniform01(seed, 2, static_cast<uint64_t>(j)));
        flip_deg[j] = quantize9(fa);
        phase_deg[j] = (j % 2) ? 180.0 : 0.0;
        tr_ms[j] = tr;
        te_ms[j] = quantize9(tr / 2.0);
    }
    return MRFG_OK;
}

int mrfg_add_noise(const double* fp, int64_t n, double sigma, uint64_t seed, double* out) {
    if (sigma < 0) return MRFG_E_INVALID;  // fingerprint.cpp:69
    for (int64_t j = 0; j < n; ++j) {
        double nr = mrfg_rng_gaussian(seed, 3, 2 * static_cast<uint64_t>(j));
        double ni = mrfg_rng_gaussian(seed, 3, 2 * static_cast<uint64_t>(j) + 1);
        out[2 * j] = fp[2 * j] + sigma * nr;
        out[2 * j + 1] = fp[2 * j + 1] + sigma * ni;
    }
    return MRFG_OK;
}

int mrfg_axis_count(double min, double max, double step, int64_t* count) {
    *count = 0;
    if (!(step > 0) || !(max > min)) return MRFG_E_INVALID;
    double q = (max - min) / step;
    auto c = static_cast<int64_t>(std::floor(q + q * 1e-12 + 1e-12));
    if (c < 1) return MRFG_E_INVALID;
    *count = c;
    return MRFG_OK;
}

}  // extern "C"
