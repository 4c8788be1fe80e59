// Compiled twice by tests/test_cpp_shim.py -- against the drop-in
// (-I include/mrf_b200, libmrf_b200.so) and against the reference's own
// sources (-I /root/reference/proj/include) -- and the two outputs diffed:
// the host Bloch primitives of bloch.hpp:12-74 must agree bit for bit,
// including the exceptions of the full rotation model and evolve_tr.
#include <cstdio>
#include <stdexcept>

#include "mrf/bloch.hpp"

using namespace mrf;

static void put(const char* tag, double v) { std::printf("%s %a\n", tag, v); }
static void put_m(const char* tag, const Matrix3& m) {
    for (double v : m.m) put(tag, v);
}

int main() {
    const double th[] = {0.0, 0.3, -1.2, 3.14159, 7.5};
    for (double t : th) {
        put_m("rotx", rot(Axis::X, t));
        put_m("roty", rot(Axis::Y, t));
        put_m("rotz", rot(Axis::Z, t));
    }
    const RfPulse pulses[] = {{0.5, 0.0, 1e-3, 0.0}, {1.2, 3.14159265358979, 1e-3, 0.0},
                              {0.7, 1.5707963267948966, 2e-3, 300.0}, {3.1, 0.4, 5e-4, -1200.0}};
    for (const RfPulse& p : pulses) {
        put_m("rf", rf_matrix(p));
        put_m("rf_full", rf_matrix(p, false));
        Matrix3 a = rf_matrix(p) * rf_matrix(p, false);
        put_m("prod", a);
        Magnetization m = a * Magnetization{0.1, -0.2, 0.9};
        put("mv", m.x), put("mv", m.y), put("mv", m.z);
    }
    Magnetization m{0.3, 0.4, -0.5};
    for (double dt : {0.0, 1e-3, 0.05, 2.0}) {
        Magnetization r = relax_step(m, dt, 1.1, 0.08);
        put("relax", r.x), put("relax", r.y), put("relax", r.z);
    }
    Magnetization cur{0, 0, -1};
    TissueParams tp{0.9, 0.07, 37.5, 1.0};
    for (int j = 0; j < 50; ++j) {
        RfPulse p{0.17 + 0.01 * j, (j % 2) ? 3.141592653589793 : 0.0, 0.0, 0.0};
        auto [echo, next] = evolve_tr(cur, p, 0.012 + 1e-4 * j, 0.006, tp);
        put("echo", echo.real()), put("echo", echo.imag());
        cur = next;
    }
    put("z", cur.z);
    auto expect_throw = [](const char* tag, auto fn) {
        try {
            fn();
            std::printf("%s no-throw\n", tag);
        } catch (const std::invalid_argument& e) {
            std::printf("%s invalid_argument %s\n", tag, e.what());
        }
    };
    expect_throw("zero_flip", [] { rf_matrix(RfPulse{0.0, 0.0, 1e-3, 10.0}, false); });
    expect_throw("zero_tau", [] { rf_matrix(RfPulse{0.5, 0.0, 0.0, 10.0}, false); });
    expect_throw("relax_dt", [] { relax_step(Magnetization{}, -1.0, 1.0, 1.0); });
    expect_throw("relax_t1", [] { relax_step(Magnetization{}, 1.0, 0.0, 1.0); });
    expect_throw("evolve_te", [] { evolve_tr(Magnetization{}, RfPulse{}, 0.01, 0.02, TissueParams{1, 1, 0, 1}); });
    expect_throw("evolve_t2", [] { evolve_tr(Magnetization{}, RfPulse{}, 0.01, 0.005, TissueParams{1, 0, 0, 1}); });
    return 0;
}
