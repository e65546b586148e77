// paramd_b200/gpu_msm_field.hpp -- drop-in B200 MsmField (and the pair-only
// SimpleCutoffField / WolfField: GpuSimpleCutoffField, GpuWolfField) for the reference
// library `paramd` (arXiv 1309.1889).  Header-only C++ over the C ABI in msmb.h.
//
// The reference's plugin interface is paramd::ForceField
// (include/paramd/force_field.hpp:14-21): a field evaluates potentials and
// forces from positions and charges.  GpuMsmField implements it with the
// sm_100a kernels of libmsmb.so, so any reference code that takes a
// ForceField -- propagate (src/integrate.cpp:13-36), energy_report
// (src/integrate.cpp:47-55), parareal_run (src/parareal.cpp:182-239) -- runs its
// MSM evaluations on the GPU unchanged:
//
//     auto ff = std::make_shared<paramd::GpuMsmField>(cfg, units);   // was MsmField
//     paramd::PropagatorSpec spec{ff, dt, steps};
//     paramd::ParticleSystem out = paramd::propagate(spec, s, units);
//
// Each evaluate() uploads positions/charges and downloads results (the plugin
// contract is host-side ParticleSystems).  For the device-resident hot path use
// paramd_b200::propagate / paramd_b200::parareal_run below: same signatures and
// semantics, the whole trajectory stays in HBM.
//
// Errors are rethrown as the reference's exception types with the reference's
// messages (include/paramd/errors.hpp:12-49).
#pragma once
#include <cstring>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../msmb.h"
#include "paramd/errors.hpp"
#include "paramd/force_field.hpp"
#include "paramd/integrate.hpp"
#include "paramd/parareal.hpp"

namespace paramd {

namespace detail_b200 {
[[noreturn]] inline void rethrow(const msmb_field* h, int rc) {
    int kind = rc;
    int64_t i = -1, j = -1;
    int step = -1;
    char msg[1024] = {0};
    msmb_last_error(h, &kind, &i, &j, &step, msg, sizeof msg);
    const std::string m(msg);
    switch (rc) {
        case MSMB_ERR_CONFIG: throw ConfigError(m);
        case MSMB_ERR_DOMAIN: throw DomainError(m);
        case MSMB_ERR_COVERAGE: throw CoverageError(m);
        case MSMB_ERR_COINCIDENT: throw CoincidentParticlesError(m);
        case MSMB_ERR_HIERARCHY: throw HierarchyError(m);
        case MSMB_ERR_RUNTIME: throw RuntimeFault(m);
        default: throw Error("msmb: " + m);
    }
}

inline msmb_msm_config to_c(const MsmConfig& c) {
    return msmb_msm_config{c.cutoff_a, c.spacing_h, c.levels_l, c.interp_order_p, c.smoothing_m};
}
inline msmb_units to_c(const UnitsConfig& u) { return msmb_units{u.coulomb_constant, u.energy_to_native}; }
}  // namespace detail_b200

/// Common part of the B200 fields: one msmb_field handle (libmsmb.so).
class GpuFieldBase : public ForceField {
  public:
    ~GpuFieldBase() override { msmb_destroy(h_); }
    GpuFieldBase(const GpuFieldBase&) = delete;
    GpuFieldBase& operator=(const GpuFieldBase&) = delete;

    PotentialResult evaluate(const ParticleSystem& s) const override {
        const std::size_t n = s.size();
        PotentialResult r;
        r.per_particle_potential.assign(n, 0.0);
        r.per_particle_force.assign(n, Vec3{});
        std::vector<double> sp(n), lp(n);
        const double box[3] = {s.box.x, s.box.y, s.box.z};
        static_assert(sizeof(Vec3) == 3 * sizeof(double), "Vec3 must be {double x,y,z}");
        const int rc = msmb_evaluate(h_, static_cast<int64_t>(n),
                                     reinterpret_cast<const double*>(s.positions.data()),
                                     s.charges.data(), box, r.per_particle_potential.data(),
                                     sp.data(), lp.data(),
                                     reinterpret_cast<double*>(r.per_particle_force.data()),
                                     &r.total_energy);
        if (rc) detail_b200::rethrow(h_, rc);
        if (msmb_field_kind(h_) == MSMB_FIELD_MSM) { // the cutoff fields leave them empty
            r.short_part = std::move(sp);
            r.long_part = std::move(lp);
        }
        return r;
    }
    double cost_flops_per_step(std::size_t n) const override {
        return msmb_cost_flops_per_step(h_, static_cast<int64_t>(n));
    }
    msmb_field* handle() const { return h_; }

  protected:
    GpuFieldBase() = default;
    msmb_field* h_ = nullptr;
};

/// paramd::MsmField (force_field.hpp:62-73) evaluated on a B200.
class GpuMsmField final : public GpuFieldBase {
  public:
    GpuMsmField(MsmConfig config, UnitsConfig units, int device = 0)
        : config_(config), units_(units) {
        const msmb_msm_config c = detail_b200::to_c(config);
        const msmb_units u = detail_b200::to_c(units);
        const int rc = msmb_create(&c, &u, device, &h_);
        if (rc) detail_b200::rethrow(nullptr, rc);
    }
    std::string name() const override { return "msm"; }
    const MsmConfig& config() const { return config_; }

  private:
    MsmConfig config_;
    UnitsConfig units_;
};

namespace detail_b200 {
inline msmb_field* make_pair_field(int kind, const CutoffParams& p, const UnitsConfig& units,
                                   double flops_per_particle, int device) {
    const msmb_cutoff_params c{p.cutoff, p.wolf_alpha.has_value() ? 1 : 0, p.wolf_alpha.value_or(0.0),
                               flops_per_particle};
    const msmb_units u = to_c(units);
    msmb_field* h = nullptr;
    const int rc = msmb_create_cutoff(kind, &c, &u, device, &h);
    if (rc) rethrow(nullptr, rc);
    return h;
}
}  // namespace detail_b200

/// paramd::SimpleCutoffField (force_field.hpp:34-46; simple_cutoff,
/// src/electrostatics.cpp:66-89) evaluated on a B200.
class GpuSimpleCutoffField final : public GpuFieldBase {
  public:
    GpuSimpleCutoffField(CutoffParams params, UnitsConfig units, double flops_per_particle = 301.0,
                         int device = 0) {
        h_ = detail_b200::make_pair_field(MSMB_FIELD_CUTOFF, params, units, flops_per_particle, device);
    }
    std::string name() const override { return "cutoff"; }
};

/// paramd::WolfField (force_field.hpp:48-60; wolf_summation,
/// src/electrostatics.cpp:91-129) evaluated on a B200.
class GpuWolfField final : public GpuFieldBase {
  public:
    GpuWolfField(CutoffParams params, UnitsConfig units, double flops_per_particle = 350.0,
                 int device = 0) {
        h_ = detail_b200::make_pair_field(MSMB_FIELD_WOLF, params, units, flops_per_particle, device);
    }
    std::string name() const override { return "wolf"; }
};

/// paramd::DirectCoulombField (force_field.hpp:23-32; direct_coulomb,
/// src/electrostatics.cpp:43-64): the exact O(N^2) sum, all pairs on a B200.
class GpuDirectCoulombField final : public GpuFieldBase {
  public:
    explicit GpuDirectCoulombField(UnitsConfig units, int device = 0) {
        const msmb_units u = detail_b200::to_c(units);
        const int rc = msmb_create_direct(&u, device, &h_);
        if (rc) detail_b200::rethrow(nullptr, rc);
    }
    std::string name() const override { return "direct"; }
};

/// paramd::PairRepulsionOverlay (force_field.hpp:75-97; force_field.cpp:45-68) over a
/// B200 base field: one GPU handle evaluating the base field plus the all-pairs
/// repulsion (the base object itself is unchanged).
class GpuPairRepulsionOverlay final : public GpuFieldBase {
  public:
    GpuPairRepulsionOverlay(std::shared_ptr<const GpuFieldBase> base, double epsilon = 0.1, double sigma = 1.0)
        : base_(std::move(base)) {
        const int rc = msmb_create_overlay(base_->handle(), epsilon, sigma, &h_);
        if (rc) detail_b200::rethrow(nullptr, rc);
    }
    std::string name() const override { return base_->name() + "+rep"; }

  private:
    std::shared_ptr<const GpuFieldBase> base_;
};

}  // namespace paramd

namespace paramd_b200 {

/// The reference's Executor plug-in (include/paramd/parareal.hpp:15-31, used for the
/// fine sweep at src/parareal.cpp:151) over GPUs: holds replicas of the fine field,
/// one per device.  paramd_b200::parareal_run deals the fine slices of every
/// iteration to the fine field and the replicas (msmb_parareal_run_ex); as a plain
/// Executor it runs parallel_for with one std::async worker per replica, like
/// AsyncExecutor (src/parareal.cpp:16-36).
class GpuExecutor final : public paramd::Executor {
  public:
    explicit GpuExecutor(std::vector<std::shared_ptr<const paramd::GpuFieldBase>> fine_replicas)
        : replicas_(std::move(fine_replicas)) {}
    void parallel_for(std::size_t count, const std::function<void(std::size_t)>& fn) const override {
        paramd::AsyncExecutor(static_cast<int>(replicas_.size() > 0 ? replicas_.size() : 1)).parallel_for(count, fn);
    }
    const std::vector<std::shared_ptr<const paramd::GpuFieldBase>>& replicas() const { return replicas_; }

  private:
    std::vector<std::shared_ptr<const paramd::GpuFieldBase>> replicas_;
};

namespace detail {
inline const paramd::GpuFieldBase* gpu_field(const std::shared_ptr<const paramd::ForceField>& ff, const char* who) {
    auto* gf = dynamic_cast<const paramd::GpuFieldBase*>(ff.get());
    // no silent CPU fall-through: a host field handed to the device path is a wiring error
    if (!gf) throw paramd::ConfigError(std::string(who) + ": force field is not a B200 field");
    return gf;
}
}  // namespace detail

/// paramd::propagate (src/integrate.cpp:13-36), device-resident.  The spec's field
/// must be a B200 field (GpuMsmField, GpuSimpleCutoffField, ...): any other field is
/// rejected with ConfigError (there is no CPU fallback on this path).
inline paramd::ParticleSystem propagate(const paramd::PropagatorSpec& spec,
                                        const paramd::ParticleSystem& s,
                                        const paramd::UnitsConfig& units) {
    spec.validate();
    const paramd::GpuFieldBase* gf = detail::gpu_field(spec.force_field, "paramd_b200::propagate");
    units.validate();
    paramd::ParticleSystem out = s;
    const double box[3] = {s.box.x, s.box.y, s.box.z};
    const msmb_units u = paramd::detail_b200::to_c(units);
    const int rc = msmb_propagate_ex(gf->handle(), static_cast<int64_t>(s.size()),
                                     reinterpret_cast<double*>(out.positions.data()),
                                     reinterpret_cast<double*>(out.velocities.data()),
                                     out.charges.data(), out.masses.data(), box, spec.dt,
                                     spec.steps_per_slice, &u);
    if (rc) paramd::detail_b200::rethrow(gf->handle(), rc);
    return out;
}

/// paramd::parareal_run (src/parareal.cpp:182-239) with device-resident states.
/// Both propagators must use B200 fields (e.g. GpuMsmField fine, GpuSimpleCutoffField
/// coarse); a GpuExecutor spreads the fine sweep over its replicas (GPUs).  The
/// report carries the reference's rows and point_iterations.
inline paramd::PararealResult parareal_run(const paramd::ParticleSystem& v, int total_points,
                                           const paramd::PararealConfig& cfg,
                                           const paramd::Executor& exec = paramd::sequential_executor()) {
    cfg.validate();
    const paramd::GpuFieldBase* F = detail::gpu_field(cfg.fine.force_field, "paramd_b200::parareal_run (fine)");
    const paramd::GpuFieldBase* G = detail::gpu_field(cfg.coarse.force_field, "paramd_b200::parareal_run (coarse)");
    std::vector<msmb_field*> reps;
    if (auto* ge = dynamic_cast<const GpuExecutor*>(&exec))
        for (const auto& r : ge->replicas()) reps.push_back(r->handle());
    msmb_parareal_config c{};
    c.window_points = cfg.window_points;
    c.max_iter = cfg.max_iter;
    c.tol = cfg.tol;
    c.fine = msmb_propagator{F->handle(), cfg.fine.dt, cfg.fine.steps_per_slice};
    c.coarse = msmb_propagator{G->handle(), cfg.coarse.dt, cfg.coarse.steps_per_slice};
    c.units = paramd::detail_b200::to_c(cfg.units);
    c.has_skip_threshold = cfg.skip_threshold.has_value();
    c.skip_threshold = cfg.skip_threshold.value_or(0.0);
    c.short_circuit = cfg.short_circuit;
    const std::size_t n = v.size();
    const std::size_t tp_n = static_cast<std::size_t>(total_points > 0 ? total_points : 1);
    std::vector<double> tp(3 * n * tp_n), tv(tp.size());
    int64_t rep[6] = {0, 0, 0, 0, 0, 0};
    const double box[3] = {v.box.x, v.box.y, v.box.z};
    // rows: at most max_iter * window_points per window, windows <= total_points
    std::vector<msmb_parareal_row> rows(static_cast<std::size_t>(cfg.max_iter) *
                                        static_cast<std::size_t>(cfg.window_points) * tp_n);
    int64_t nrows = 0;
    std::vector<int> piters(tp_n, 0);
    const int rc = msmb_parareal_run_ex(&c, reps.data(), static_cast<int>(reps.size()), static_cast<int64_t>(n),
                                        reinterpret_cast<const double*>(v.positions.data()),
                                        reinterpret_cast<const double*>(v.velocities.data()),
                                        v.charges.data(), v.masses.data(), box, total_points,
                                        tp.data(), tv.data(), rep, rows.data(), static_cast<int64_t>(rows.size()),
                                        &nrows, piters.data());
    auto report = [&]() {
        paramd::ConvergenceReport r;
        r.counts.g_evals = static_cast<std::size_t>(rep[0]);
        r.counts.f_evals = static_cast<std::size_t>(rep[1]);
        r.counts.f_skipped = static_cast<std::size_t>(rep[2]);
        r.windows = static_cast<int>(rep[3]);
        r.converged = rep[4] != 0;
        for (int64_t i = 0; i < nrows && i < static_cast<int64_t>(rows.size()); ++i)
            r.rows.push_back({rows[i].window, rows[i].point, rows[i].iteration, rows[i].delta_rms,
                              rows[i].converged != 0});
        r.point_iterations.assign(piters.begin(), piters.begin() + static_cast<std::ptrdiff_t>(rep[5]));
        return r;
    };
    if (rc == MSMB_ERR_NONCONVERGENCE) {
        char msg[512] = {0};
        msmb_last_error(F->handle(), nullptr, nullptr, nullptr, nullptr, msg, sizeof msg);
        throw paramd::NonConvergenceError(msg, report());
    }
    if (rc) paramd::detail_b200::rethrow(F->handle(), rc);
    paramd::PararealResult out;
    for (int k = 0; k < total_points; ++k) {
        paramd::ParticleSystem st = v;
        std::memcpy(st.positions.data(), tp.data() + 3 * n * k, 3 * n * sizeof(double));
        std::memcpy(st.velocities.data(), tv.data() + 3 * n * k, 3 * n * sizeof(double));
        out.trajectory.push_back(std::move(st));
    }
    out.report = report();
    return out;
}

}  // namespace paramd_b200
