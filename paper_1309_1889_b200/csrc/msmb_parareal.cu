// Device-resident parareal driver: the reference's parareal_init /
// parareal_iterate / parareal_run (src/parareal.cpp:94-239) with every
// lambda / g / delta state kept in HBM.  Propagations go through the fine and
// coarse msmb_field handles (each a CUDA-graph Verlet propagate); the state
// algebra (state_sub / state_add / rms_pos_change, src/parareal.cpp:58-90) runs
// as sm_100a kernels.  Only the rows the algorithm reads are kept (the last two
// lambda rows, the last g and delta rows), which is observationally identical
// to the reference's full history.
//
// The Executor of the reference (src/parareal.cpp:11-36) only changes where fine
// slices run; results are independent of it (pure propagators).  With one fine
// field the fine slices run back to back on its stream; msmb_parareal_run_ex takes
// several fine fields (replicas of F, one per GPU) and runs the fine sweep of an
// iteration on all of them at once, one host worker per field pulling slice
// indices from a shared counter -- the reference's AsyncExecutor::parallel_for
// (src/parareal.cpp:16-36) with GPUs as workers.  Each worker propagates its
// slice on its own device and copies the end state back (peer copy over NVLink);
// the state algebra and the coarse sweep stay on the first fine field's device.
// The multi-process (one process per GPU, NCCL) split of the same sweep is
// paper_1309_1889_b200/parallel.py over the raw device-state entry points at the
// end of this file.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <thread>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "msmb_engine.cuh"

namespace msmb {

struct Delta {
    DBuf buf; // 6n: dpos (3n AoS) then dvel (3n AoS)
    double rms_pos = 0.0;
    double* dpos() const { return buf.as<double>(); }
    double* dvel(int64_t n) const { return buf.as<double>() + 3 * size_t(n); }
};

struct PR {
    const msmb_parareal_config* cfg;
    std::vector<msmb_field*> fines; // fine-field replicas ([0] = cfg->fine.field)
    int device = 0;                 // device of the rows (fines[0]'s)
    std::vector<msmb_parareal_row> rows; // ConvergenceReport::rows (parareal.cpp:208)
    int64_t n;
    cudaStream_t st; // fine field's stream for the algebra
    DBuf partial;
    int nblk;
    int64_t g_evals = 0, f_evals = 0, f_skipped = 0;
    StateBuf proto; // q, m, box
};

static void ckp(cudaError_t e, const char* w) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(w) + ": " + cudaGetErrorString(e));
}

static std::unique_ptr<StateBuf> new_state(PR& P) {
    auto s = std::make_unique<StateBuf>();
    ckp(s->alloc(P.n), "cudaMalloc state");
    for (int ax = 0; ax < 3; ++ax) s->box[ax] = P.proto.box[ax];
    return s;
}

static void copy_state(PR& P, StateBuf& dst, const StateBuf& src) {
    ckp(cudaMemcpyAsync(dst.buf.p, src.buf.p, src.buf.bytes, cudaMemcpyDeviceToDevice, P.st), "copy");
    for (int ax = 0; ax < 3; ++ax) dst.box[ax] = src.box[ax];
}

static double host_sum(PR& P) {
    std::vector<double> h(size_t(P.nblk));
    ckp(cudaMemcpyAsync(h.data(), P.partial.p, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, P.st), "D2H");
    ckp(cudaStreamSynchronize(P.st), "sync");
    double s = 0.0;
    for (double v : h) s += v;
    return s;
}

static double rms_change(PR& P, const StateBuf& a, const StateBuf& b) { // parareal.cpp:86-90
    launch_rms_change(P.st, P.n, a.dev(), b.dev(), P.partial.as<double>(), P.nblk);
    return std::sqrt(host_sum(P) / (3.0 * double(P.n)));
}

static std::unique_ptr<Delta> state_sub(PR& P, const StateBuf& a, const StateBuf& b) { // :58-73
    auto d = std::make_unique<Delta>();
    ckp(d->buf.alloc(sizeof(double) * 6 * size_t(P.n > 0 ? P.n : 1)), "cudaMalloc delta");
    launch_state_sub(P.st, P.n, a.dev(), b.dev(), d->dpos(), d->dvel(P.n), P.partial.as<double>(), P.nblk);
    d->rms_pos = std::sqrt(host_sum(P) / (3.0 * double(P.n)));
    return d;
}

static std::unique_ptr<Delta> copy_delta(PR& P, const Delta& src) {
    auto d = std::make_unique<Delta>();
    ckp(d->buf.alloc(src.buf.bytes), "cudaMalloc delta");
    ckp(cudaMemcpyAsync(d->buf.p, src.buf.p, src.buf.bytes, cudaMemcpyDeviceToDevice, P.st), "copy");
    d->rms_pos = src.rms_pos;
    return d;
}

static std::unique_ptr<StateBuf> state_add(PR& P, const StateBuf& base, const Delta& d) { // :75-82
    auto o = new_state(P);
    copy_state(P, *o, base); // charges, masses
    DevState od = o->dev();
    launch_state_add(P.st, P.n, base.dev(), d.dpos(), d.dvel(P.n), od);
    return o;
}

// propagate(spec, in, units) into a new state.  The field's scratch system is
// the working buffer so its captured CUDA graphs are reused across calls.
// `f` may live on another device than the rows (a fine replica): the copies are
// cudaMemcpyDefault (peer copies under UVA) and `out` is allocated on P.device.
static int prop(PR& P, const msmb_propagator& sp, const StateBuf& in, std::unique_ptr<StateBuf>& out,
                msmb_field* f = nullptr) {
    if (!f) f = sp.field;
    std::lock_guard<std::recursive_mutex> lk(f->mu);
    ckp(cudaSetDevice(P.device), "cudaSetDevice");
    ckp(cudaStreamSynchronize(P.st), "sync");
    out = new_state(P);
    ckp(cudaSetDevice(f->device), "cudaSetDevice");
    if (f->scratch.n != P.n || !f->scratch.buf.p) ckp(f->scratch.alloc(P.n), "alloc scratch");
    ckp(cudaMemcpyAsync(f->scratch.buf.p, in.buf.p, in.buf.bytes, cudaMemcpyDefault, f->stream), "copy");
    for (int ax = 0; ax < 3; ++ax) f->scratch.box[ax] = in.box[ax];
    const int rc = engine_propagate(f, f->scratch, sp.dt, sp.steps_per_slice,
                                    P.cfg->units.energy_to_native);
    if (rc == MSMB_OK) {
        ckp(cudaMemcpyAsync(out->buf.p, f->scratch.buf.p, in.buf.bytes, cudaMemcpyDefault, f->stream), "copy");
        ckp(cudaStreamSynchronize(f->stream), "sync");
    }
    ckp(cudaSetDevice(P.device), "cudaSetDevice");
    return rc;
}

using Row = std::vector<std::unique_ptr<StateBuf>>;
using DRow = std::vector<std::unique_ptr<Delta>>;

struct Window {
    int points = 0;
    int rows = 0;             // rows created so far (reference w.rows())
    Row lam_prev2, lam_prev;  // lambda rows rows-2 and rows-1
    Row lam0;                 // only [0] (the window's initial condition) is kept
    Row g_prev;               // g row rows-1
    DRow d_prev;              // delta row rows-1
    int msmb_rc = 0;
};

static int pr_init(PR& P, const StateBuf& v, int t, Window& w) { // parareal.cpp:94-115
    w = Window{};
    w.points = t;
    w.lam_prev.resize(size_t(t) + 1);
    w.g_prev.resize(size_t(t) + 1);
    w.d_prev.resize(size_t(t) + 1);
    w.lam_prev[0] = new_state(P);
    copy_state(P, *w.lam_prev[0], v);
    w.lam0.resize(1);
    w.lam0[0] = new_state(P);
    copy_state(P, *w.lam0[0], v);
    for (int n = 1; n <= t; ++n) {
        const int rc = prop(P, P.cfg->coarse, *w.lam_prev[n - 1], w.lam_prev[n]);
        if (rc) return rc;
        P.g_evals++;
        w.g_prev[n] = new_state(P);
        copy_state(P, *w.g_prev[n], *w.lam_prev[n]);
    }
    w.rows = 1;
    return MSMB_OK;
}

static int pr_iterate(PR& P, Window& w) { // parareal.cpp:117-180
    const int t = w.points;
    const int prev = w.rows - 1;
    std::vector<char> skip(size_t(t) + 1, 0);
    if (P.cfg->has_skip_threshold && w.rows >= 2) // metastable_skip_indices :117-127
        for (int n = 1; n <= t; ++n)
            if (rms_change(P, *w.lam_prev[n - 1], *w.lam_prev2[n - 1]) < P.cfg->skip_threshold) skip[n] = 1;
    DRow deltas(size_t(t) + 1);
    for (int n = 1; n <= t; ++n)
        if (skip[n]) {
            deltas[n] = copy_delta(P, *w.d_prev[n]);
            P.f_skipped++;
        }
    // the executor's work list (parareal.cpp:146-155): fine slices, over the fine replicas
    std::vector<int> work;
    for (int n = 1; n <= t; ++n)
        if (!skip[n]) work.push_back(n);
    Row fres(size_t(t) + 1);
    std::vector<int> frc(size_t(t) + 1, MSMB_OK);
    std::vector<Error> ferr(size_t(t) + 1);
    std::vector<std::string> fexc(size_t(t) + 1);
    std::atomic<size_t> next{0};
    std::atomic<int> stop{0};
    auto worker = [&](msmb_field* f) {
        for (;;) {
            const size_t k = next.fetch_add(1);
            if (k >= work.size() || stop.load()) return;
            const int n = work[k];
            try {
                frc[n] = prop(P, P.cfg->fine, *w.lam_prev[n - 1], fres[n], f);
                if (frc[n]) ferr[n] = f->last;
            } catch (const std::exception& ex) {
                frc[n] = MSMB_ERR_CUDA;
                fexc[n] = ex.what();
            }
            if (frc[n]) stop.store(1);
        }
    };
    if (P.fines.size() > 1 && work.size() > 1) {
        std::vector<std::thread> th;
        for (msmb_field* f : P.fines) th.emplace_back(worker, f);
        for (auto& x : th) x.join();
        ckp(cudaSetDevice(P.device), "cudaSetDevice");
    } else {
        worker(P.fines[0]);
    }
    // a failure is the one a sequential executor meets first: the lowest slice index
    for (int n : work)
        if (frc[n]) {
            if (!fexc[n].empty()) throw std::runtime_error(fexc[n]);
            P.fines[0]->last = ferr[n];
            return frc[n];
        }
    for (int n : work) {
        if (!fres[n]) return MSMB_ERR_INTERNAL; // not reached: every slice ran or one failed
        deltas[n] = state_sub(P, *fres[n], *w.g_prev[n]);
        P.f_evals++;
    }
    Row row(size_t(t) + 1), grow(size_t(t) + 1);
    row[0] = new_state(P);
    copy_state(P, *row[0], *w.lam0[0]);
    for (int n = 1; n <= t; ++n) {
        std::unique_ptr<StateBuf> g;
        if (prev == 0 && n == 1) {
            g = new_state(P);
            copy_state(P, *g, *w.g_prev[1]);
        } else {
            const int rc = prop(P, P.cfg->coarse, *row[n - 1], g);
            if (rc) return rc;
            P.g_evals++;
        }
        row[n] = state_add(P, *g, *deltas[n]);
        grow[n] = std::move(g);
    }
    w.lam_prev2 = std::move(w.lam_prev);
    w.lam_prev = std::move(row);
    w.g_prev = std::move(grow);
    w.d_prev = std::move(deltas);
    w.rows++;
    ckp(cudaStreamSynchronize(P.st), "sync");
    return MSMB_OK;
}

static Error validate(const msmb_parareal_config* c) { // parareal.cpp:43-56
    auto E = [](const char* m) { return Error{MSMB_ERR_CONFIG, -1, -1, -1, m}; };
    if (c->window_points < 1) return E("window_points must be >= 1");
    if (c->max_iter < 1) return E("max_iter must be >= 1");
    if (!(c->tol > 0.0)) return E("tol must be > 0");
    const msmb_propagator* sp[2] = {&c->fine, &c->coarse};
    for (auto* s : sp) { // PropagatorSpec::validate, integrate.cpp:7-11
        if (!s->field) return E("propagator has no force field");
        if (!(s->dt > 0.0)) return E("dt must be > 0");
        if (s->steps_per_slice < 1) return E("steps_per_slice must be >= 1");
    }
    Error e = validate_units(c->units);
    if (e.kind) return e;
    const double sf = c->fine.dt * c->fine.steps_per_slice, sg = c->coarse.dt * c->coarse.steps_per_slice;
    if (std::fabs(sf - sg) > 1e-12 * std::max(std::fabs(sf), std::fabs(sg)))
        return E("fine and coarse propagators span different slice lengths");
    if (c->has_skip_threshold && !(c->skip_threshold >= 0.0)) return E("skip threshold must be >= 0");
    return Error{};
}

static int setup(PR& P, const msmb_parareal_config* cfg, int64_t n, const double* pos,
                 const double* vel, const double* q, const double* mass, const double* box) {
    P.cfg = cfg;
    P.n = n;
    msmb_field* f = cfg->fine.field;
    if (P.fines.empty()) P.fines.push_back(f);
    P.device = f->device;
    P.st = f->stream;
    P.nblk = reduce_blocks(n);
    ckp(P.partial.alloc(sizeof(double) * size_t(P.nblk)), "alloc");
    ckp(P.proto.alloc(n), "alloc");
    for (int ax = 0; ax < 3; ++ax) P.proto.box[ax] = box[ax];
    // upload through the fine field's host entry point machinery
    std::vector<double> soa(size_t(n) * 8);
    for (int64_t i = 0; i < n; ++i) {
        for (int ax = 0; ax < 3; ++ax) {
            soa[size_t(ax) * n + i] = pos[3 * i + ax];
            soa[size_t(3 + ax) * n + i] = vel[3 * i + ax];
        }
        soa[size_t(6) * n + i] = q[i];
        soa[size_t(7) * n + i] = mass[i];
    }
    ckp(cudaMemcpyAsync(P.proto.buf.p, soa.data(), sizeof(double) * soa.size(), cudaMemcpyHostToDevice, P.st),
        "H2D");
    ckp(cudaStreamSynchronize(P.st), "sync"); // before other fields' streams read proto
    return MSMB_OK;
}

static void download(PR& P, const StateBuf& s, double* pos, double* vel) {
    std::vector<double> soa(size_t(P.n) * 6);
    ckp(cudaStreamSynchronize(P.st), "sync");
    ckp(cudaMemcpy(soa.data(), s.buf.p, sizeof(double) * soa.size(), cudaMemcpyDeviceToHost), "D2H");
    for (int64_t i = 0; i < P.n; ++i)
        for (int ax = 0; ax < 3; ++ax) {
            if (pos) pos[3 * i + ax] = soa[size_t(ax) * P.n + i];
            if (vel) vel[3 * i + ax] = soa[size_t(3 + ax) * P.n + i];
        }
}

} // namespace msmb

using namespace msmb;

static int pr_fail(const msmb_parareal_config* cfg, const Error& e) {
    if (cfg && cfg->fine.field) cfg->fine.field->last = e;
    return e.kind;
}

static int pr_propagate_error(const msmb_parareal_config* cfg, int rc) {
    // a propagation failed: surface the failing field's error on the fine handle
    if (cfg->coarse.field && cfg->coarse.field->last.kind == rc && cfg->fine.field != cfg->coarse.field &&
        cfg->fine.field->last.kind != rc)
        cfg->fine.field->last = cfg->coarse.field->last;
    return rc;
}

extern "C" int msmb_parareal_window(const msmb_parareal_config* cfg, int64_t n, const double* pos_xyz,
                                    const double* vel_xyz, const double* q, const double* mass,
                                    const double box[3], int t_points, int k_iters, double* row_pos,
                                    double* row_vel, double* delta_rms, int64_t* counts) {
    Error e = validate(cfg);
    if (e.kind) return pr_fail(cfg, e);
    try {
        cudaSetDevice(cfg->fine.field->device);
        PR P;
        setup(P, cfg, n, pos_xyz, vel_xyz, q, mass, box);
        Window w;
        int rc = pr_init(P, P.proto, t_points, w);
        for (int k = 0; rc == MSMB_OK && k < k_iters; ++k) rc = pr_iterate(P, w);
        if (rc) return pr_propagate_error(cfg, rc);
        for (int i = 0; i <= t_points; ++i)
            download(P, *w.lam_prev[i], row_pos ? row_pos + 3 * n * i : nullptr,
                     row_vel ? row_vel + 3 * n * i : nullptr);
        if (delta_rms) {
            delta_rms[0] = 0.0;
            for (int i = 1; i <= t_points; ++i) delta_rms[i] = w.d_prev[i] ? w.d_prev[i]->rms_pos : 0.0;
        }
        if (counts) {
            counts[0] = P.g_evals;
            counts[1] = P.f_evals;
            counts[2] = P.f_skipped;
        }
        cfg->fine.field->last = Error{};
        return MSMB_OK;
    } catch (const std::exception& ex) {
        return pr_fail(cfg, Error{MSMB_ERR_CUDA, -1, -1, -1, ex.what()});
    }
}

// parareal_run (parareal.cpp:182-239) over the fine replicas `fines` (fines[0] is
// cfg->fine.field).  rows / point_iterations: the ConvergenceReport's history.
static int run_impl(const msmb_parareal_config* cfg, std::vector<msmb_field*> fines, int64_t n,
                    const double* pos_xyz, const double* vel_xyz, const double* q, const double* mass,
                    const double box[3], int total_points, double* traj_pos, double* traj_vel, int64_t* report,
                    msmb_parareal_row* rows, int64_t rows_cap, int64_t* rows_written, int* point_iterations,
                    int report_len = 5) {
    Error e = validate(cfg);
    if (e.kind) return pr_fail(cfg, e);
    if (total_points < 1) return pr_fail(cfg, Error{MSMB_ERR_CONFIG, -1, -1, -1, "total_points must be >= 1"});
    for (msmb_field* f : fines) {
        if (!f) return pr_fail(cfg, Error{MSMB_ERR_CONFIG, -1, -1, -1, "propagator has no force field"});
        const msmb_field* F = fines[0];
        const bool same = f->kind == F->kind && f->rep == F->rep && f->cfg.cutoff_a == F->cfg.cutoff_a &&
                          f->cfg.spacing_h == F->cfg.spacing_h && f->cfg.levels_l == F->cfg.levels_l &&
                          f->cut.cutoff == F->cut.cutoff && f->cut.wolf_alpha == F->cut.wolf_alpha &&
                          f->units.coulomb_constant == F->units.coulomb_constant;
        if (!same)
            return pr_fail(cfg, Error{MSMB_ERR_CONFIG, -1, -1, -1, "fine replicas must be the fine field's kind and parameters"});
    }
    if (rows_written) *rows_written = 0;
    try {
        cudaSetDevice(cfg->fine.field->device);
        PR P;
        P.fines = std::move(fines);
        setup(P, cfg, n, pos_xyz, vel_xyz, q, mass, box);
        auto current = new_state(P);
        copy_state(P, *current, P.proto);
        int remaining = total_points, window_idx = 0, out_idx = 0, rc = MSMB_OK;
        auto fill_report = [&](int converged) {
            if (report) {
                report[0] = P.g_evals;
                report[1] = P.f_evals;
                report[2] = P.f_skipped;
                report[3] = window_idx;
                report[4] = converged;
                if (report_len > 5) report[5] = out_idx; // output points (point_iterations entries)
            }
            const int64_t nr = std::min<int64_t>(int64_t(P.rows.size()), rows ? rows_cap : 0);
            for (int64_t i = 0; i < nr; ++i) rows[i] = P.rows[size_t(i)];
            if (rows_written) *rows_written = int64_t(P.rows.size()); // may exceed rows_cap
        };
        while (remaining > 0 && rc == MSMB_OK) { // parareal.cpp:193-235
            ++window_idx;
            const int t = std::min(cfg->window_points, remaining);
            Window w;
            rc = pr_init(P, *current, t, w);
            int prefix = 0;
            for (int k = 0; rc == MSMB_OK && k < cfg->max_iter; ++k) {
                rc = pr_iterate(P, w);
                if (rc) break;
                prefix = 0;
                bool unbroken = true;
                for (int m = 1; m <= t; ++m) {
                    const double change = rms_change(P, *w.lam_prev[m], *w.lam_prev2[m]);
                    const bool ok = change <= cfg->tol;
                    P.rows.push_back(msmb_parareal_row{window_idx, m, k, w.d_prev[m]->rms_pos, ok ? 1 : 0});
                    if (unbroken && ok)
                        prefix = m;
                    else
                        unbroken = false;
                }
                if (cfg->short_circuit && prefix == t) break;
            }
            if (rc) break;
            if (prefix == 0) {
                fill_report(0);
                return pr_fail(cfg, Error{MSMB_ERR_NONCONVERGENCE, -1, -1, -1,
                                          "window " + std::to_string(window_idx) +
                                              " did not converge within max_iter=" +
                                              std::to_string(cfg->max_iter)});
            }
            for (int m = 1; m <= prefix; ++m, ++out_idx) {
                download(P, *w.lam_prev[m], traj_pos ? traj_pos + 3 * n * out_idx : nullptr,
                         traj_vel ? traj_vel + 3 * n * out_idx : nullptr);
                if (point_iterations) point_iterations[out_idx] = w.rows - 1; // iterations_done()
            }
            copy_state(P, *current, *w.lam_prev[prefix]);
            remaining -= prefix;
        }
        if (rc) return pr_propagate_error(cfg, rc);
        fill_report(1);
        cfg->fine.field->last = Error{};
        return MSMB_OK;
    } catch (const std::exception& ex) {
        return pr_fail(cfg, Error{MSMB_ERR_CUDA, -1, -1, -1, ex.what()});
    }
}

extern "C" int msmb_parareal_run(const msmb_parareal_config* cfg, int64_t n, const double* pos_xyz,
                                 const double* vel_xyz, const double* q, const double* mass,
                                 const double box[3], int total_points, double* traj_pos,
                                 double* traj_vel, int64_t* report) {
    return run_impl(cfg, {cfg ? cfg->fine.field : nullptr}, n, pos_xyz, vel_xyz, q, mass, box, total_points,
                    traj_pos, traj_vel, report, nullptr, 0, nullptr, nullptr);
}

extern "C" int msmb_parareal_run_ex(const msmb_parareal_config* cfg, msmb_field* const* fine_replicas,
                                    int n_replicas, int64_t n, const double* pos_xyz, const double* vel_xyz,
                                    const double* q, const double* mass, const double box[3], int total_points,
                                    double* traj_pos, double* traj_vel, int64_t* report, msmb_parareal_row* rows,
                                    int64_t rows_cap, int64_t* rows_written, int* point_iterations) {
    std::vector<msmb_field*> fines{cfg ? cfg->fine.field : nullptr};
    for (int k = 0; k < n_replicas; ++k)
        if (fine_replicas && fine_replicas[k] != fines[0]) fines.push_back(fine_replicas[k]);
    return run_impl(cfg, std::move(fines), n, pos_xyz, vel_xyz, q, mass, box, total_points, traj_pos, traj_vel,
                    report, rows, rows_cap, rows_written, point_iterations, 6);
}

// ---- raw device states (multi-process drivers, paper_1309_1889_b200/parallel.py) ----
namespace {

DevState raw_state(const double* p, int64_t n) {
    DevState s{};
    s.n = n;
    double* b = const_cast<double*>(p);
    s.x = b;
    s.y = b + n;
    s.z = b + 2 * n;
    s.vx = b + 3 * n;
    s.vy = b + 4 * n;
    s.vz = b + 5 * n;
    s.q = s.m = nullptr;
    return s;
}

// the block partials summed on the host in block order (host_sum above)
double partial_sum(msmb_field* f, int nblk) {
    std::vector<double> h(static_cast<size_t>(nblk), 0.0);
    ckp(cudaMemcpyAsync(h.data(), f->reduce.p, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, f->stream),
        "D2H");
    ckp(cudaStreamSynchronize(f->stream), "sync");
    double s = 0.0;
    for (double v : h) s += v;
    return s;
}

template <class Fn>
int raw_call(msmb_field* f, int64_t n, Fn&& fn) {
    if (!f) return MSMB_ERR_CONFIG;
    std::lock_guard<std::recursive_mutex> lk(f->mu);
    try {
        cudaSetDevice(f->device);
        const int nblk = reduce_blocks(n);
        if (f->reduce.bytes < sizeof(double) * size_t(nblk)) ckp(f->reduce.alloc(sizeof(double) * size_t(nblk)), "alloc");
        fn(nblk);
        ckp(cudaGetLastError(), "kernel launch");
        ckp(cudaStreamSynchronize(f->stream), "sync");
        f->last = Error{};
        return MSMB_OK;
    } catch (const std::exception& ex) {
        f->last = Error{MSMB_ERR_CUDA, -1, -1, -1, ex.what()};
        return MSMB_ERR_CUDA;
    }
}

} // namespace

extern "C" int msmb_state_sub_device(msmb_field* f, int64_t n, const double* a, const double* b,
                                     double* delta, double* rms_pos) {
    return raw_call(f, n, [&](int nblk) {
        if (n > 0) {
            f->launches += launch_state_sub(f->stream, n, raw_state(a, n), raw_state(b, n), delta, delta + 3 * n,
                                            f->reduce.as<double>(), nblk);
        }
        const double s = n > 0 ? partial_sum(f, nblk) : 0.0;
        if (rms_pos) *rms_pos = std::sqrt(s / (3.0 * double(n)));
    });
}

extern "C" int msmb_state_add_device(msmb_field* f, int64_t n, const double* base, const double* delta,
                                     double* out) {
    return raw_call(f, n, [&](int) {
        if (n == 0) return;
        DevState o = raw_state(out, n);
        f->launches += launch_state_add(f->stream, n, raw_state(base, n), delta, delta + 3 * n, o);
    });
}

extern "C" int msmb_state_rms_change_device(msmb_field* f, int64_t n, const double* a, const double* b,
                                            double* rms) {
    return raw_call(f, n, [&](int nblk) {
        if (n > 0) f->launches += launch_rms_change(f->stream, n, raw_state(a, n), raw_state(b, n),
                                                    f->reduce.as<double>(), nblk);
        const double s = n > 0 ? partial_sum(f, nblk) : 0.0;
        if (rms) *rms = std::sqrt(s / (3.0 * double(n)));
    });
}

extern "C" int msmb_system_set_state_device(msmb_system* s, const double* state) {
    if (!s) return MSMB_ERR_CONFIG;
    return raw_call(s->f, s->st.n, [&](int) {
        if (s->st.n > 0)
            ckp(cudaMemcpyAsync(s->st.buf.p, state, sizeof(double) * 6 * size_t(s->st.n), cudaMemcpyDeviceToDevice,
                                s->f->stream), "D2D");
    });
}

extern "C" int msmb_system_get_state_device(const msmb_system* s, double* state) {
    if (!s) return MSMB_ERR_CONFIG;
    return raw_call(s->f, s->st.n, [&](int) {
        if (s->st.n > 0)
            ckp(cudaMemcpyAsync(state, s->st.buf.p, sizeof(double) * 6 * size_t(s->st.n), cudaMemcpyDeviceToDevice,
                                s->f->stream), "D2D");
    });
}
