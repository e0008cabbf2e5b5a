// tests/cpp/engine_facade.cpp — a C++ caller of the drop-in boundary:
// builds the circular dam break on the host, runs it through
// swamp::Engine (include/swamp/engine.hpp -> libswamp_gpu.so) and prints one
// JSON line. Compiled by tests/test_abi.py; run on the GPU by the gpu tier.
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <vector>

#include "swamp/engine.hpp"

int main(int argc, char** argv) {
    swamp::SimConfig cfg;
    cfg.L = argc > 1 ? std::atoi(argv[1]) : 7;
    cfg.epsilon = 1e-3;
    cfg.width = 40.0;
    cfg.x0 = cfg.y0 = -20.0;
    cfg.t_end = 0.5;
    const int side = 1 << cfg.L;
    const double dx = cfg.width / side;
    std::vector<double> h(size_t(side) * side), qx(h.size(), 0.0), qy(h.size(), 0.0), z(h.size(), 0.0);
    for (int j = 0; j < side; ++j)
        for (int i = 0; i < side; ++i) {
            const double x = cfg.x0 + (i + 0.5) * dx, y = cfg.y0 + (j + 0.5) * dx;
            h[size_t(j) * side + i] = (x * x + y * y < 2.5 * 2.5) ? 2.5 : 0.5;
        }
    // config validation errors are exceptions
    bool rejected = false;
    try {
        swamp::SimConfig bad = cfg;
        bad.L = 20;
        bad.validate();
    } catch (const std::invalid_argument&) {
        rejected = true;
    }
    swamp::Engine eng(cfg, h, qx, qy, z);
    const swamp::StepReport r = eng.run();
    const swamp::LeafAssembly a = eng.leaves();
    long covered = 0;
    for (auto zi : a.leaves) covered += 1L << (2 * (cfg.L - swamp::zorder::level_of(zi)));
    std::vector<double> fh, fqx, fqy;
    eng.finest(fh, fqx, fqy);
    double mass = 0;
    for (double v : fh) mass += v;
    std::printf("{\"t\": %.17g, \"steps\": %lld, \"leaves\": %zu, \"covered\": %ld, \"finest\": %d, "
                "\"mass\": %.17g, \"rejected_bad_L\": %s}\n",
                eng.time(), (long long)r.step, a.leaves.size(), covered, side * side, mass * dx * dx,
                rejected ? "true" : "false");
    return (covered == long(side) * side && rejected) ? 0 : 1;
}
