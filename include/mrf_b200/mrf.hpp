// mrf_b200/mrf.hpp -- drop-in C++ interface for the DGS path on B200.
//
// Declares, in namespace mrf, the entry points and value types of the
// reference library (/root/reference/proj/include/mrf/{sequence,fingerprint,
// bloch,dictionary,zoom}.hpp) with the SAME signatures and semantics, so code
// written against the reference compiles unchanged after replacing its
// includes with this one header and linking libmrf_b200.so (+ libmrfg.so).
// Each function cites the reference declaration it replaces.  The compute runs
// on an sm_100 GPU through the C ABI of include/mrfg.h (device: env
// MRFG_DEVICE, default 0); errors come back as the reference's exceptions.
// `workers` arguments are accepted for signature compatibility (the GPU grid
// replaces the host thread pool; results never depended on them).
#pragma once

#include <array>
#include <complex>
#include <cstdint>
#include <filesystem>
#include <functional>
#include <span>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

struct mrfg_ctx;

namespace mrf {

// ---------------------------------------------------------- sequence.hpp:14-56
struct ScheduleEntry {
    double flip_deg = 0, phase_deg = 0, tr_ms = 0, te_ms = 0;
    double flip_rad() const { return flip_deg * 0.017453292519943295; }
    double phase_rad() const { return phase_deg * 0.017453292519943295; }
    double tr_s() const { return tr_ms * 1e-3; }
    double te_s() const { return te_ms * 1e-3; }
};
struct Schedule {
    std::vector<ScheduleEntry> entries;
    std::uint64_t seed = 0;
    std::size_t size() const { return entries.size(); }
};
Schedule build_schedule(std::size_t n, std::uint64_t seed);              // sequence.hpp:51
std::string to_csv(const Schedule& sched);                              // sequence.hpp:56
void save_csv(const Schedule& sched, const std::filesystem::path& path);
Schedule load_schedule_csv(const std::filesystem::path& path);

// ------------------------------------------------------- fingerprint.hpp:12-75
struct TissueParams {
    double t1 = 0, t2 = 0, df = 0, pd = 1.0;
};
struct Fingerprint {
    std::vector<std::complex<double>> s;
    bool unit_norm = false;
    std::size_t size() const { return s.size(); }
};
Fingerprint normalize(const Fingerprint& fp);                           // fingerprint.hpp:34
double cc(const Fingerprint& a, const Fingerprint& b);                  // fingerprint.hpp:40
double euclidean(const Fingerprint& a, const Fingerprint& b);           // fingerprint.hpp:43
Fingerprint add_noise(const Fingerprint& fp, double sigma, std::uint64_t seed);  // :47
double estimate_pd(const Fingerprint& acquired, const Fingerprint& matched_ideal);  // :71
double calibrate_noise(const Fingerprint& fp, double target_cc, std::uint64_t seed);  // :45-50
struct CalibratedNoise {                                                // :52-61
    double sigma = 0;
    std::uint64_t seed = 0;
    Fingerprint noisy;
};
CalibratedNoise make_calibrated_noise(const Fingerprint& fp, double target_cc, std::uint64_t seed);
Fingerprint smooth(const Fingerprint& fp, int k);                       // :63-66
void save_csv(const Fingerprint& fp, const std::filesystem::path& path);  // :73-74
Fingerprint load_fingerprint_csv(const std::filesystem::path& path);

// ------------------------------------------------------------- bloch.hpp:12-74
// Host primitives of the Bloch model (FP64, the reference's operand order:
// bit-identical results).  They are the per-TR building blocks the GPU
// kernels run fused; here for code that composes them directly.
struct Magnetization {
    double x = 0, y = 0, z = 1;
};
struct Matrix3 {  // row-major (bloch.hpp:22-41)
    double m[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
    static Matrix3 identity() { return {}; }
    Matrix3 operator*(const Matrix3& o) const;
    Magnetization operator*(const Magnetization& v) const;
};
enum class Axis { X, Y, Z };
struct RfPulse {  // bloch.hpp:48-53: flip, phase (rad), duration (s), off-resonance (rad/s)
    double alpha = 0, phi = 0, tau = 0, delta_omega = 0;
};
Matrix3 rot(Axis axis, double theta);                                    // bloch.hpp:56
Magnetization relax_step(const Magnetization& m, double dt, double t1, double t2);  // bloch.hpp:60
// Simplified Rz(phi) Rx(-alpha) Rz(-phi), or the full off-resonant-axis form
// (bloch.hpp:62-69); std::invalid_argument for the full form's undefined cases.
Matrix3 rf_matrix(const RfPulse& pulse, bool simplified = true);
std::pair<std::complex<double>, Magnetization> evolve_tr(const Magnetization& m, const RfPulse& pulse,
                                                         double tr, double te,
                                                         const TissueParams& p);  // bloch.hpp:71-74

// ------------------------------------------------------------- bloch.hpp:79-102
// Holds one GPU context (the schedule's RF rotations composed once, as the
// reference's constructor does); copies create their own context.
class BlochSimulator {
  public:
    explicit BlochSimulator(const Schedule& sched);
    ~BlochSimulator();
    BlochSimulator(const BlochSimulator& o);
    BlochSimulator& operator=(const BlochSimulator& o);
    void simulate(const TissueParams& p, std::complex<double>* out) const;
    Fingerprint simulate(const TissueParams& p) const;
    // Batched form (GPU-native): params.size() fingerprints, row-major.
    std::vector<std::complex<double>> simulate_batch(const std::vector<TissueParams>& params) const;
    std::size_t length() const { return n_; }
    mrfg_ctx* native() const { return ctx_; }

  private:
    mrfg_ctx* ctx_ = nullptr;
    std::size_t n_ = 0;
    Schedule sched_;
};
Fingerprint simulate_fingerprint(const TissueParams& p, const Schedule& sched);  // bloch.hpp:102

// -------------------------------------------------------- dictionary.hpp:16-132
struct AxisSpec {
    double min = 0, step = 1;
    std::size_t count = 0;
    double value(std::size_t k) const { return min + static_cast<double>(k) * step; }
};
struct AxisRange {
    double min = 0, max = 0, step = 1;
};
struct ParameterGrid {
    AxisSpec t1_ms, t2_ms, df_hz;
    std::size_t total() const { return t1_ms.count * t2_ms.count * df_hz.count; }
    std::size_t flatten(std::size_t i1, std::size_t i2, std::size_t idf) const {
        return (i1 * t2_ms.count + i2) * df_hz.count + idf;
    }
    struct Index3 {
        std::size_t i1, i2, idf;
    };
    Index3 unflatten(std::size_t flat) const {
        const std::size_t idf = flat % df_hz.count, rest = flat / df_hz.count;
        return {rest / t2_ms.count, rest % t2_ms.count, idf};
    }
    TissueParams params_at(std::size_t i1, std::size_t i2, std::size_t idf) const {
        return {t1_ms.value(i1) * 1e-3, t2_ms.value(i2) * 1e-3, df_hz.value(idf), 1.0};
    }
};
ParameterGrid grid_from_ranges(const AxisRange& t1_ms, const AxisRange& t2_ms,
                               const AxisRange& df_hz);                 // dictionary.hpp:61
using Digest = std::array<std::uint8_t, 32>;
Digest schedule_digest(const Schedule& sched);                          // dictionary.hpp:67
std::string digest_hex(const Digest& d);
struct Dictionary {
    ParameterGrid grid;
    Digest digest{};
    std::size_t entry_len = 0;
    std::vector<float> data;
    std::span<const float> entry(std::size_t flat) const {
        return {data.data() + flat * 2 * entry_len, 2 * entry_len};
    }
};
Dictionary generate(const ParameterGrid& grid, const Schedule& sched, int workers = 1);  // :85
// .mrfd files (dictionary.hpp:87-96): save / load / save_generated (GPU generation
// streamed to disk; byte-identical to the reference's files).
void save(const Dictionary& dict, const std::filesystem::path& path);
Dictionary load(const std::filesystem::path& path);
void save_generated(const ParameterGrid& grid, const Schedule& sched,
                    const std::filesystem::path& path, int workers = 1,
                    std::size_t chunk_entries = 1 << 15);
enum class Metric { cc, euclidean };
struct Match {
    TissueParams params;
    double score = 0;
    std::size_t evaluations = 0;
};
Match brute_force_search(const Fingerprint& fp, const Dictionary& dict,
                         Metric metric = Metric::cc);                   // dictionary.hpp:108
struct ScanOutcome {
    std::vector<Match> matches;
    std::vector<double> scan_seconds;
    double generate_seconds = 0;
};
ScanOutcome scan_grid(const ParameterGrid& grid, const Schedule& sched,
                      const std::vector<Fingerprint>& queries, Metric metric = Metric::cc,
                      int workers = 1, std::size_t chunk_entries = 1 << 15);  // :120-122
void cc_map(const Fingerprint& fp, const ParameterGrid& grid, const Schedule& sched,
            const std::function<void(std::size_t first_flat, std::span<const float>)>& sink,
            int workers = 1, std::size_t chunk_entries = 1 << 15);        // :127-129
void cc_map_to_file(const Fingerprint& fp, const ParameterGrid& grid, const Schedule& sched,
                    const std::filesystem::path& path, int workers = 1);  // :130-132

// -------------------------------------------------------------- zoom.hpp:17-178
struct SearchRanges {
    AxisRange t1_ms{100, 5500, 1};
    AxisRange t2_ms{50, 1200, 1};
    AxisRange df_hz{-300, 300, 1};
};
struct ZoomConfig {
    Metric metric = Metric::cc;
    Metric final_metric = Metric::cc;
    int smooth_k = 0;
    double omega_hz = 70, df_coarse_hz = 60, df_refine_hz = 3, df_window_hz = 150;
    double plateau_eps = 1e-7, heavy_noise_cc = 0.1, fallback_coarse_hz = 30,
           fallback_window_hz = 300;
    std::vector<double> t1t2_2d_steps_ms{200, 100};
    std::vector<double> t1t2_1d_steps_ms{100, 50, 20, 10};
    double final_2d_step_ms = 1;
    double init_t1_ms = 1000, init_t2_ms = 500;
    double prior_window_t1_ms = 3000, prior_window_t2_ms = 800, prior_window_df_hz = 150;
};
struct StageLog {
    std::string stage;
    std::size_t evaluations = 0;
    double best = 0;
    double t1_ms = 0, t2_ms = 0, df_hz = 0;
};
struct QuantResult {
    TissueParams params;
    double score = 0;
    std::size_t evaluations = 0;
    double seconds = 0;
    std::vector<StageLog> trace;  // recorded by K5 (exact bests, the reference's stages)
};
struct DfSearchParams {
    long coarse = 60, refine = 3, finest = 1, window_half = 75, omega = 70;
    double plateau_eps = 1e-7, heavy_cc = 0.1;
    long fallback_coarse = 30, fallback_window_half = 150;
    bool allow_fallback = true;
};
// Generic host forms over caller objectives (zoom.hpp:127-143).
long search_df(const std::function<double(long)>& f, long lo, long hi, const DfSearchParams& prm,
               const std::function<void(const char*, long, double)>& stage = {});
long zoom_1d(const std::function<double(long)>& f, long lo, long hi, long init,
             std::span<const long> steps);
std::pair<long, long> zoom_2d(const std::function<double(long, long)>& f, long lo1, long hi1,
                              long lo2, long hi2, long init1, long init2,
                              std::span<const std::pair<long, long>> steps);
// Memoizing objective over a search lattice (zoom.hpp:72-110): each unique
// point costs one FP64 simulation on the GPU (bit-identical to the
// reference's) or one dictionary lookup; repeats and metric switches are
// free.  The K5 kernel runs the same objective fused on the device; this
// class serves callers that drive search_df / zoom_1d / zoom_2d themselves.
class Objective {
  public:
    struct Options {
        int smooth_k = 0;
        const Dictionary* full_dict = nullptr;  // every point is a lookup
        const Dictionary* df_dict = nullptr;    // first-stage lookups only
    };
    Objective(const Fingerprint& query, const ParameterGrid& lattice, const Schedule& sched,
              const Options& opt);
    ~Objective();
    double eval(long i1, long i2, long idf, Metric metric);
    double eval_df_stage(long i1, long i2, long idf, Metric metric);
    std::size_t evaluations() const { return evals_; }
    const ParameterGrid& lattice() const { return lattice_; }
    Fingerprint ideal_at(long i1, long i2, long idf) const;

  private:
    double score_from_entry(const std::vector<std::complex<double>>& entry, Metric metric) const;
    const std::vector<std::complex<double>>& acquire(long i1, long i2, long idf, bool df_stage);
    ParameterGrid lattice_;
    BlochSimulator sim_;
    Options opt_;
    std::vector<std::complex<double>> query_;
    std::size_t evals_ = 0;
    std::unordered_map<std::uint64_t, std::vector<std::complex<double>>> entries_;
    std::unordered_map<std::uint64_t, double> memo_cc_, memo_euc_;
};

QuantResult quantify(const Fingerprint& fp, const SearchRanges& ranges, const ZoomConfig& cfg,
                     const Schedule& sched, const Dictionary* df_dict = nullptr,
                     const Dictionary* full_dict = nullptr);            // zoom.hpp:148-151
// Batched form (GPU-native): one call, many fingerprints; same dictionary
// options and validation as quantify.
std::vector<QuantResult> quantify_batch(const std::vector<Fingerprint>& fps,
                                        const SearchRanges& ranges, const ZoomConfig& cfg,
                                        const Schedule& sched, const Dictionary* df_dict = nullptr,
                                        const Dictionary* full_dict = nullptr);
Dictionary make_df_dictionary(const SearchRanges& ranges, const ZoomConfig& cfg,
                              const Schedule& sched, int workers = 1);  // zoom.hpp:157-158
struct SliceResult {
    int nx = 0, ny = 0;
    std::vector<double> t1_ms, t2_ms, df_hz, pd, score;
    std::vector<std::size_t> evaluations;
    std::size_t total_evaluations = 0;
    double seconds = 0;
};
SliceResult quantify_slice(const std::vector<Fingerprint>& fps, const std::vector<std::uint8_t>& mask,
                           int nx, int ny, const SearchRanges& ranges, const ZoomConfig& cfg,
                           const Schedule& sched, bool use_prior, int workers = 1,
                           const Dictionary* df_dict = nullptr);        // zoom.hpp:174-178

}  // namespace mrf
