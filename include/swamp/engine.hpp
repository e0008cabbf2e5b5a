// swamp/engine.hpp — C++ solver/config facade over the C-ABI (swamp_gpu.h).
//
// The reference's engine interface exists only as a specification
// (SPEC.md:373-455): SimConfig, SimState, StepReport, initialise,
// step_adaptive, step_uniform, run. This header gives a C++ caller those
// names, backed by libswamp_gpu.so (sm_100a). Errors are rethrown as
// std::runtime_error (device / numerical failures, with step/stage context —
// SPEC.md:403) or std::invalid_argument (config validation, SPEC.md:552,
// mirroring io.load_config's rejection).
//
// Header-only; link with -lswamp_gpu. Not thread-safe: one control thread
// per Engine.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../swamp_gpu.h"
#include "zorder.hpp"

namespace swamp {

enum class Boundary : int32_t { Reflective = SWAMP_BC_REFLECTIVE, Transmissive = SWAMP_BC_TRANSMISSIVE, Inflow = SWAMP_BC_INFLOW };
enum class Band : int32_t { None = SWAMP_BAND_NONE, Parents = SWAMP_BAND_PARENTS, Neighbours = SWAMP_BAND_NEIGHBOURS };

// SimConfig with the spec defaults.
struct SimConfig {
    int L = 8;
    double epsilon = 1e-3;
    double width = 1.0;
    double x0 = 0.0, y0 = 0.0;
    double cfl = 0.5;
    double g = 9.80665;
    double manning = 0.0;
    double h_dry = 1e-6;
    double t_end = 1.0;
    double dt_fallback = 1e-3;
    Boundary bc[4] = {Boundary::Reflective, Boundary::Reflective, Boundary::Reflective, Boundary::Reflective};
    Band band = Band::Neighbours;
    bool inflow_is_eta = false;
    std::vector<double> inflow_t, inflow_v, output_times;
    std::vector<uint8_t> inactive;  // 4^L finest cells (south row first), empty = all active (D16)

    void validate() const {
        if (L < 1 || L > zorder::kMaxLevel) throw std::invalid_argument("SimConfig: L outside [1, 13]");
        if (!(epsilon >= 0.0)) throw std::invalid_argument("SimConfig: epsilon must be >= 0");
        if (!(width > 0.0)) throw std::invalid_argument("SimConfig: width must be > 0");
        if (!(cfl > 0.0 && cfl <= 1.0)) throw std::invalid_argument("SimConfig: CFL must be in (0, 1]");
        if (!(h_dry > 0.0)) throw std::invalid_argument("SimConfig: h_dry must be > 0");
        if (inflow_t.size() != inflow_v.size()) throw std::invalid_argument("SimConfig: inflow series size mismatch");
    }

    swamp_config to_c() const {
        validate();
        swamp_config c{};
        c.L = L;
        c.band_mode = static_cast<int32_t>(band);
        c.epsilon = epsilon;
        c.width = width;
        c.x0 = x0;
        c.y0 = y0;
        c.cfl = cfl;
        c.g = g;
        c.manning = manning;
        c.h_dry = h_dry;
        c.t_end = t_end;
        c.dt_fallback = dt_fallback;
        for (int k = 0; k < 4; ++k) c.bc[k] = static_cast<int32_t>(bc[k]);
        c.inflow_mode = inflow_is_eta ? SWAMP_INFLOW_ETA : SWAMP_INFLOW_DEPTH;
        c.inflow_n = static_cast<int32_t>(inflow_t.size());
        c.inflow_t = inflow_t.empty() ? nullptr : inflow_t.data();
        c.inflow_v = inflow_v.empty() ? nullptr : inflow_v.data();
        c.n_outputs = static_cast<int32_t>(output_times.size());
        c.output_times = output_times.empty() ? nullptr : output_times.data();
        c.inactive = inactive.empty() ? nullptr : inactive.data();
        return c;
    }
};

using StepReport = swamp_step_report;

// LeafAssembly
struct LeafAssembly {
    std::vector<zorder::ZIndex> leaves;
    std::vector<uint32_t> west, east, north, south;
    static bool is_boundary(uint32_t d) { return d >= SWAMP_BOUNDARY_BASE; }
};

// The SimState owner on one B200.
class Engine {
public:
    // initialise: finest-level rasters, row-major, south row first.
    Engine(const SimConfig& cfg, const std::vector<double>& h, const std::vector<double>& qx,
           const std::vector<double>& qy, const std::vector<double>& z, int device = 0, bool uniform = false)
        : cfg_(cfg) {
        const size_t n = size_t(1) << (2 * cfg.L);
        if (h.size() != n || qx.size() != n || qy.size() != n || z.size() != n)
            throw std::invalid_argument("initialise: fields must hold 4^L values");
        const swamp_config c = cfg_.to_c();
        const int st = uniform ? swamp_gpu_create_uniform(&c, h.data(), qx.data(), qy.data(), z.data(), device, &g_)
                               : swamp_gpu_create(&c, h.data(), qx.data(), qy.data(), z.data(), device, &g_);
        if (st != SWAMP_OK) throw std::runtime_error("initialise failed: status " + std::to_string(st));
        uniform_ = uniform;
    }
    ~Engine() {
        if (g_) swamp_gpu_destroy(g_);
    }
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;
    Engine(Engine&& o) noexcept : cfg_(std::move(o.cfg_)), g_(std::exchange(o.g_, nullptr)), uniform_(o.uniform_) {}

    StepReport step_adaptive() {
        StepReport r{};
        check(swamp_gpu_step(g_, &r), "step_adaptive");
        return r;
    }
    StepReport step_uniform(int64_t n = 1) {
        StepReport r{};
        check(swamp_gpu_step_uniform(g_, n, &r), "step_uniform");
        return r;
    }
    StepReport advance(int64_t n) {
        StepReport r{};
        check(swamp_gpu_advance(g_, n, &r), "advance");
        return r;
    }
    // n steps back to back, every step's report (swamp_gpu_advance_reports)
    std::vector<StepReport> advance_reports(int64_t n) {
        std::vector<StepReport> r(static_cast<size_t>(n > 0 ? n : 0));
        if (n > 0) check(swamp_gpu_advance_reports(g_, n, r.data()), "advance_reports");
        return r;
    }
    StepReport run() {  // SPEC.md:417-420 (no outputs)
        StepReport r{};
        check(swamp_gpu_run(g_, &r), "run");
        return r;
    }
    double time() const {
        double t = 0;
        check(swamp_gpu_info(g_, &t, nullptr, nullptr, nullptr), "info");
        return t;
    }
    LeafAssembly leaves() const {
        int64_t n = 0;
        check(swamp_gpu_copy_leaves(g_, nullptr, nullptr, nullptr, nullptr, nullptr, 0, &n), "leaves");
        LeafAssembly a;
        a.leaves.resize(n);
        a.west.resize(n);
        a.east.resize(n);
        a.north.resize(n);
        a.south.resize(n);
        check(swamp_gpu_copy_leaves(g_, a.leaves.data(), a.west.data(), a.east.data(), a.north.data(), a.south.data(),
                                    n, &n),
              "leaves");
        return a;
    }
    // zero-detail expansion to the finest grid
    void finest(std::vector<double>& h, std::vector<double>& qx, std::vector<double>& qy) const {
        const size_t n = size_t(1) << (2 * cfg_.L);
        h.resize(n);
        qx.resize(n);
        qy.resize(n);
        check(swamp_gpu_export_finest(g_, h.data(), qx.data(), qy.data()), "export_finest");
    }
    const SimConfig& config() const { return cfg_; }

private:
    void check(int st, const char* what) const {
        if (st == SWAMP_OK) return;
        int32_t code = 0, q = 0, stage = 0;
        uint32_t z = 0;
        char msg[256] = {0};
        swamp_gpu_last_error(g_, &code, &z, &q, &stage, msg, sizeof msg);
        throw std::runtime_error(std::string(what) + ": status " + std::to_string(st) + " (z=" + std::to_string(z) +
                                 ", quantity=" + std::to_string(q) + ", stage=" + std::to_string(stage) + ") " + msg);
    }
    SimConfig cfg_;
    swamp_gpu* g_ = nullptr;
    bool uniform_ = false;
};

}  // namespace swamp
