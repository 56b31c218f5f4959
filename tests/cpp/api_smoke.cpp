// C++ host API smoke test (built and run by tests/test_cpp_api.py on the GPU).
// Mirrors test_transform.cpp:66-72 (round trip) and test_apps.cpp:53-95.
#include <cmath>
#include <cstdio>
#include <random>
#include <string>

#include "shearlet_b200.hpp"

using namespace shearlet_b200;

int main() {
    auto sys = build_system_2d(64, 64, ScaleProfile::from_levels({0, 0, 1, 1}));
    std::mt19937_64 rng(22);
    std::vector<double> f(64 * 64);
    for (double& x : f) x = 2.0 * (static_cast<double>(rng()) * 0x1.0p-64) - 1.0;
    const auto c = forward(f, sys);
    const auto r = inverse(c, sys);
    double num = 0, den = 0;
    for (size_t i = 0; i < f.size(); ++i) {
        num += (r[i] - f[i]) * (r[i] - f[i]);
        den += f[i] * f[i];
    }
    const double err = std::sqrt(num / den);
    int fails = 0;
    if (!(err <= 1e-10)) { std::printf("round trip %g\n", err); ++fails; }
    if (sys.redundancy() != 25) { std::printf("R %zu\n", sys.redundancy()); ++fails; }
    try {
        (void)forward(std::vector<double>(16 * 16), sys);
        ++fails;
    } catch (const ShapeError&) {
    }
    try {
        (void)hard_threshold(c, ThresholdSchedule{{1.0}, 0.1, true}, sys);
        ++fails;
    } catch (const ConfigError&) {
    }
    const auto same = hard_threshold(c, ThresholdSchedule{{1, 1, 1, 1}, 0.0, true}, sys);
    if (same != c) { std::printf("sigma 0 not identity\n"); ++fails; }
    const auto [A, B] = sys.frame_bounds();
    if (!(A > 0 && B >= A)) ++fails;
    // SHCF round trip and a custom filter bank (a symmetric 3x3 diamond fan + a 5-tap QMF)
    const auto bytes = serialize(c, sys);
    if (deserialize(bytes, sys) != c) { std::printf("shcf round trip\n"); ++fails; }
    auto bytes_bad = bytes;
    bytes_bad[0] = 'X';
    try {
        (void)deserialize(bytes_bad, sys);
        ++fails;
    } catch (const FormatError&) {
    }
    auto sys2 = build_system_2d(32, 32, ScaleProfile::from_levels({0, 1}),
                                FanFilter{{0, 0.25, 0, 0.25, 0.5, 0.25, 0, 0.25, 0}, 3, 3, 1, 1, "custom"},
                                QmfPair::from_lowpass(Taps1d{{-0.125, 0.25, 0.75, 0.25, -0.125}, 2}));
    std::vector<double> g(32 * 32);
    for (double& x : g) x = 2.0 * (static_cast<double>(rng()) * 0x1.0p-64) - 1.0;
    const auto r2 = inverse(forward(g, sys2), sys2);
    double n2 = 0, d2 = 0;
    for (size_t i = 0; i < g.size(); ++i) {
        n2 += (r2[i] - g[i]) * (r2[i] - g[i]);
        d2 += g[i] * g[i];
    }
    if (!(std::sqrt(n2 / d2) <= 1e-10)) { std::printf("custom bank round trip %g\n", std::sqrt(n2 / d2)); ++fails; }
    // descriptor round trip, SVOL round trip, Q_opt of an exact recovery
    const std::string text = describe(sys);
    auto sys3 = build_from_descriptor(text);
    if (describe(sys3) != text || sys3.redundancy() != sys.redundancy()) { std::printf("descriptor\n"); ++fails; }
    std::vector<double> vol(8 * 9 * 10);
    for (double& x : vol) x = static_cast<double>(rng() % 1000) / 7.0;
    save_svol(vol, {8, 9, 10}, "/tmp/api_smoke.svol");
    std::array<std::size_t, 3> vd{};
    if (load_svol("/tmp/api_smoke.svol", &vd) != vol || vd[2] != 10) { std::printf("svol\n"); ++fails; }
    std::vector<double> truth(64 * 64, 0.0);
    for (int i = 20; i < 30; ++i) truth[static_cast<std::size_t>(i) * 64 + 32] = 1.0;
    std::vector<double> recovered(truth.size());
    for (std::size_t i = 0; i < truth.size(); ++i) recovered[i] = 200.0 * truth[i];
    const auto [qmin, dbest] = quality_q_opt(recovered, truth, 64, 64, gaussian_kernel(2.0));
    if (!(qmin < 1e-12) || dbest != 1) { std::printf("q_opt %g %d\n", qmin, dbest); ++fails; }
    // inpainting with every pixel observed converges to the input
    InpaintConfig ic;
    ic.iterations = 4;
    const auto inp = inpaint(f, std::vector<double>(f.size(), 1.0), sys, ic);
    double ni = 0, di = 0;
    for (size_t i = 0; i < f.size(); ++i) {
        ni += (inp[i] - f[i]) * (inp[i] - f[i]);
        di += f[i] * f[i];
    }
    if (!(std::sqrt(ni / di) < 0.5)) { std::printf("inpaint %g\n", std::sqrt(ni / di)); ++fails; }
    std::printf("cpp api: err %.2e R %zu A %.6f B %.6f fails %d\n", err, sys.redundancy(), A, B, fails);
    return fails;
}
