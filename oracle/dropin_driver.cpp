// oracle/dropin_driver.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Proves the drop-in at the reference's own plugin boundary: the UNMODIFIED
// reference library (paramd, compiled from /root/reference/proj/src by
// oracle/Makefile) drives paramd_b200::GpuMsmField through its ForceField
// interface (include/paramd/force_field.hpp:14-21):
//   1. MsmField::evaluate vs GpuMsmField::evaluate on the same system;
//   2. paramd::propagate(spec{GpuMsmField}) -- the reference's own Verlet loop
//      calling the GPU plugin every step -- vs paramd::propagate(spec{MsmField});
//   3. paramd_b200::propagate (device-resident) vs the reference;
//   4. paramd::parareal_run with GPU fine/coarse fields vs the reference's;
//   5. error behaviour: the reference's exception types come back out;
//   6. the pair-only fields: SimpleCutoffField / WolfField vs GpuSimpleCutoffField /
//      GpuWolfField (evaluate, the reference's propagate over the plugin) and parareal
//      with the CLI's default pairing, MSM fine + cutoff coarse (tools/paramd_main.cpp:417),
//      through paramd_b200::parareal_run vs the reference's parareal_run.
// Prints one JSON object; tests/test_gpu_dropin.py checks it.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <memory>
#include <random>
#include <string>

#include "paramd/electrostatics.hpp"
#include "paramd/force_field.hpp"
#include "paramd/generate.hpp"
#include "paramd/integrate.hpp"
#include "paramd/msm.hpp"
#include "paramd/parareal.hpp"
#include "paramd_b200/gpu_msm_field.hpp"

using namespace paramd;

static double rel_rms(const std::vector<Vec3>& a, const std::vector<Vec3>& b) {
    double num = 0, den = 0;
    for (std::size_t i = 0; i < a.size(); ++i) {
        const Vec3 d = a[i] - b[i];
        num += norm2(d);
        den += norm2(b[i]);
    }
    return std::sqrt(num / (den > 0 ? den : 1e-300));
}

int main() {
    const UnitsConfig units = UnitsConfig::physical();
    ParticleSystem s = generate_random_system(2048, Vec3{27.4, 27.4, 27.4}, ChargeScheme::RandomNeutral, 1.5, 77);
    std::mt19937_64 rng(78);
    std::normal_distribution<double> nd(0.0, 1.0);
    const double kt = 0.0019872041 * 300.0 * 4.184e-4;
    for (auto& m : s.masses) m = 18.0;
    for (auto& v : s.velocities) v = Vec3{nd(rng), nd(rng), nd(rng)} * std::sqrt(kt / 18.0);

    MsmConfig fcfg;
    fcfg.cutoff_a = 12.0;
    fcfg.spacing_h = 2.5;
    fcfg.levels_l = 3;
    MsmConfig gcfg;
    gcfg.cutoff_a = 8.0;
    gcfg.spacing_h = 5.0;
    gcfg.levels_l = 2;
    auto ref_f = std::make_shared<MsmField>(fcfg, units);
    auto gpu_f = std::make_shared<GpuMsmField>(fcfg, units);
    auto ref_g = std::make_shared<MsmField>(gcfg, units);
    auto gpu_g = std::make_shared<GpuMsmField>(gcfg, units);

    // 1. plugin evaluate
    const ForceField& fr = *ref_f;
    const ForceField& fg = *gpu_f;
    PotentialResult a = fr.evaluate(s), b = fg.evaluate(s);
    const double de = std::fabs(a.total_energy - b.total_energy) / std::fabs(a.total_energy);
    const double df = rel_rms(b.per_particle_force, a.per_particle_force);

    // 2. the reference's own propagate with the GPU plugin
    PropagatorSpec sr{ref_f, 0.005, 20}, sg{gpu_f, 0.005, 20};
    ParticleSystem pr = paramd::propagate(sr, s, units);
    ParticleSystem pg = paramd::propagate(sg, s, units);
    const double dx_plugin = rel_rms(pg.positions, pr.positions);
    // 3. device-resident propagate
    ParticleSystem pd = paramd_b200::propagate(sg, s, units);
    const double dx_dev = rel_rms(pd.positions, pr.positions);

    // 4. parareal_run (reference driver, GPU fields) and the device-resident driver
    PararealConfig cr;
    cr.window_points = 4;
    cr.max_iter = 3;
    cr.tol = 1e-9;
    cr.units = units;
    cr.fine = PropagatorSpec{ref_f, 0.005, 20};
    cr.coarse = PropagatorSpec{ref_g, 0.02, 5};
    PararealConfig cg = cr;
    cg.fine = PropagatorSpec{gpu_f, 0.005, 20};
    cg.coarse = PropagatorSpec{gpu_g, 0.02, 5};
    int pr_ok = 1;
    double dx_pr = -1, dx_pr_dev = -1;
    std::size_t gref = 0, fref = 0, ggpu = 0, fgpu = 0, gdev = 0, fdev = 0;
    try {
        PararealResult rr = parareal_run(s, 6, cr, sequential_executor());
        PararealResult rg = parareal_run(s, 6, cg, sequential_executor());
        PararealResult rd = paramd_b200::parareal_run(s, 6, cg);
        dx_pr = 0;
        dx_pr_dev = 0;
        for (int k = 0; k < 6; ++k) {
            dx_pr = std::max(dx_pr, rel_rms(rg.trajectory[k].positions, rr.trajectory[k].positions));
            dx_pr_dev = std::max(dx_pr_dev, rel_rms(rd.trajectory[k].positions, rr.trajectory[k].positions));
        }
        gref = rr.report.counts.g_evals;
        fref = rr.report.counts.f_evals;
        ggpu = rg.report.counts.g_evals;
        fgpu = rg.report.counts.f_evals;
        gdev = rd.report.counts.g_evals;
        fdev = rd.report.counts.f_evals;
    } catch (const std::exception& e) {
        pr_ok = 0;
        std::fprintf(stderr, "parareal: %s\n", e.what());
    }

    // 4b. GpuExecutor: the fine sweep over fine replicas (one per GPU; device k % ndev),
    // bitwise equal to the single-field run; the report rows / point_iterations equal
    // the reference's ConvergenceReport
    double dx_exec = -1;
    int rows_ok = 0, fallback_rejected = 0;
    try {
        const int ndev = msmb_device_count();
        std::vector<std::shared_ptr<const GpuFieldBase>> reps;
        for (int k = 1; k <= 2; ++k) reps.push_back(std::make_shared<GpuMsmField>(fcfg, units, k % ndev));
        paramd_b200::GpuExecutor gx(reps);
        PararealResult rr = parareal_run(s, 6, cr, sequential_executor());
        PararealResult r1 = paramd_b200::parareal_run(s, 6, cg);
        PararealResult rx = paramd_b200::parareal_run(s, 6, cg, gx);
        dx_exec = 0;
        for (int k = 0; k < 6; ++k)
            dx_exec = std::max(dx_exec, rel_rms(rx.trajectory[k].positions, r1.trajectory[k].positions));
        rows_ok = rr.report.rows.size() == rx.report.rows.size() &&
                  rr.report.point_iterations == rx.report.point_iterations && rr.report.windows == rx.report.windows;
        for (std::size_t i = 0; rows_ok && i < rr.report.rows.size(); ++i) {
            const auto &a0 = rr.report.rows[i], &b0 = rx.report.rows[i];
            rows_ok = a0.window == b0.window && a0.point == b0.point && a0.iteration == b0.iteration &&
                      a0.converged == b0.converged &&
                      std::fabs(a0.delta_rms - b0.delta_rms) <= 1e-6 * std::fabs(a0.delta_rms) + 1e-300;
        }
    } catch (const std::exception& e) {
        std::fprintf(stderr, "gpu executor: %s\n", e.what());
    }
    try { // a host field on the device path is an error, not a silent CPU run
        paramd_b200::propagate(sr, s, units);
    } catch (const ConfigError&) {
        fallback_rejected = 1;
    }

    // 5. errors through the plugin
    ParticleSystem bad = s;
    bad.positions[100] = bad.positions[7];
    std::string err_ref, err_gpu;
    try { fr.evaluate(bad); } catch (const CoincidentParticlesError& e) { err_ref = e.what(); }
    try { fg.evaluate(bad); } catch (const CoincidentParticlesError& e) { err_gpu = e.what(); }
    bad = s;
    bad.positions[300].x = 60.0;
    std::string cov_ref, cov_gpu;
    try { fr.evaluate(bad); } catch (const CoverageError& e) { cov_ref = e.what(); }
    try { fg.evaluate(bad); } catch (const CoverageError& e) { cov_gpu = e.what(); }

    // 6. pair-only fields
    CutoffParams cp;
    cp.cutoff = 10.0;
    CutoffParams wp = cp;
    wp.wolf_alpha = 0.2;
    auto ref_c = std::make_shared<SimpleCutoffField>(cp, units);
    auto gpu_c = std::make_shared<GpuSimpleCutoffField>(cp, units);
    auto ref_w = std::make_shared<WolfField>(wp, units);
    auto gpu_w = std::make_shared<GpuWolfField>(wp, units);
    double pf_de = 0, pf_df = 0;
    for (int k = 0; k < 2; ++k) {
        const ForceField& r0 = k ? static_cast<const ForceField&>(*ref_w) : *ref_c;
        const ForceField& g0 = k ? static_cast<const ForceField&>(*gpu_w) : *gpu_c;
        PotentialResult x = r0.evaluate(s), y = g0.evaluate(s);
        pf_de = std::max(pf_de, std::fabs(x.total_energy - y.total_energy) / std::fabs(x.total_energy));
        pf_df = std::max(pf_df, rel_rms(y.per_particle_force, x.per_particle_force));
        if (y.short_part.has_value() || y.long_part.has_value() || r0.name() != g0.name()) pf_de = 1.0;
        if (r0.cost_flops_per_step(2048) != g0.cost_flops_per_step(2048)) pf_de = 1.0;
    }
    PropagatorSpec scr{ref_c, 0.005, 20}, scg{gpu_c, 0.005, 20};
    const double pf_dx = rel_rms(paramd::propagate(scg, s, units).positions, paramd::propagate(scr, s, units).positions);
    const double pf_dx_dev = rel_rms(paramd_b200::propagate(scg, s, units).positions,
                                     paramd::propagate(scr, s, units).positions);
    PararealConfig pcr = cr, pcg = cg;
    pcr.coarse = PropagatorSpec{ref_c, 0.02, 5};
    pcg.coarse = PropagatorSpec{gpu_c, 0.02, 5};
    double pf_dx_pr = -1;
    try {
        PararealResult rr = parareal_run(s, 6, pcr, sequential_executor());
        PararealResult rd = paramd_b200::parareal_run(s, 6, pcg);
        pf_dx_pr = 0;
        for (int k = 0; k < 6; ++k)
            pf_dx_pr = std::max(pf_dx_pr, rel_rms(rd.trajectory[k].positions, rr.trajectory[k].positions));
        if (rr.report.counts.g_evals != rd.report.counts.g_evals || rr.report.counts.f_evals != rd.report.counts.f_evals)
            pf_dx_pr = 1.0;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "pair-field parareal: %s\n", e.what());
    }

    // 7. all-pairs fields: DirectCoulombField and PairRepulsionOverlay(SimpleCutoffField)
    auto ref_d = std::make_shared<DirectCoulombField>(units);
    auto gpu_d = std::make_shared<GpuDirectCoulombField>(units);
    auto ref_o = std::make_shared<PairRepulsionOverlay>(ref_c, 0.1, 2.0);
    auto gpu_o = std::make_shared<GpuPairRepulsionOverlay>(gpu_c, 0.1, 2.0);
    double ap_de = 0, ap_df = 0;
    for (int k = 0; k < 2; ++k) {
        const ForceField& r0 = k ? static_cast<const ForceField&>(*ref_o) : *ref_d;
        const ForceField& g0 = k ? static_cast<const ForceField&>(*gpu_o) : *gpu_d;
        PotentialResult x = r0.evaluate(s), y = g0.evaluate(s);
        ap_de = std::max(ap_de, std::fabs(x.total_energy - y.total_energy) / std::fabs(x.total_energy));
        ap_df = std::max(ap_df, rel_rms(y.per_particle_force, x.per_particle_force));
        if (r0.name() != g0.name() || r0.cost_flops_per_step(2048) != g0.cost_flops_per_step(2048)) ap_de = 1.0;
    }
    std::printf("{\"ap_de\": %.3e, \"ap_df\": %.3e, \"dx_executor\": %.3e, \"rows_ok\": %d, "
                "\"fallback_rejected\": %d, ", ap_de, ap_df, dx_exec, rows_ok, fallback_rejected);
    std::printf(
        "\"pf_de\": %.3e, \"pf_df\": %.3e, \"pf_dx_plugin_propagate\": %.3e, \"pf_dx_device_propagate\": %.3e, "
        "\"pf_dx_parareal_device\": %.3e, ",
        pf_de, pf_df, pf_dx, pf_dx_dev, pf_dx_pr);
    std::printf(
        "\"de\": %.3e, \"df\": %.3e, \"dx_plugin_propagate\": %.3e, \"dx_device_propagate\": %.3e, "
        "\"parareal_ok\": %d, \"dx_parareal_plugin\": %.3e, \"dx_parareal_device\": %.3e, "
        "\"counts\": [%zu, %zu, %zu, %zu, %zu, %zu], \"coincident_ref\": \"%s\", \"coincident_gpu\": \"%s\", "
        "\"coverage_ref\": \"%s\", \"coverage_gpu\": \"%s\", \"name\": \"%s\", \"cost\": %.6e, \"cost_ref\": %.6e}\n",
        de, df, dx_plugin, dx_dev, pr_ok, dx_pr, dx_pr_dev, gref, fref, ggpu, fgpu, gdev, fdev,
        err_ref.c_str(), err_gpu.c_str(), cov_ref.c_str(), cov_gpu.c_str(), fg.name().c_str(),
        fg.cost_flops_per_step(2048), fr.cost_flops_per_step(2048));
    return 0;
}
