// Spatial decomposition of one MSM force + velocity-Verlet step over parts (one
// part per GPU).  Every part holds the whole replicated
// particle state.  A part computes only the work it owns (msmb::Part):
//   * the short-range pair sum of the i-clusters in its x-range of pair columns
//     (the reference's short_range, src/msm_phases.cpp:224-252);
//   * anterpolation of its level-0 planes (src/msm_phases.cpp:39-61);
//   * the lattice cutoff of its output planes on every non-top level
//     (src/msm_phases.cpp:93-134);
//   * interpolation, long-range forces and the Verlet update of the atoms binned
//     into its pair columns (src/msm_phases.cpp:195-222, src/msm.cpp:16-48,
//     src/integrate.cpp:23-34).
// Binning, restriction, the top level and prolongation are O(N) or tiny and are
// replicated.
//
// One step is four phases with an exchange between consecutive phases:
//   0  bin + sort + clusters, owned pair lists, owned anterpolation
//      -> level-0 charge planes; the owned pair sum is left running   exchange #1
//   1  restriction, owned lattice-cutoff planes -> level potentials exchange #2
//   2  top level, prolongation, owned interpolation + forces + energy share,
//      owned Verlet update -> particle state                       exchange #3
//   3  import the exchanged state
// Each exchange buffer holds IEEE bit patterns as int64.  Entries a part does not
// own are INT64_MIN, so an element-wise MAX all-reduce (NCCL / gloo) delivers
// every owner's exact bits to every part.  Every owned value is computed exactly
// as the single-GPU path computes it: the same clusters and lists, the same
// per-point and per-tile sums, the same lattice source split.  So a decomposed
// trajectory equals the single-GPU one bit for bit, for any part count.  Only
// the energy, a sum of per-part shares, is rounded differently.
//
// The driver (one process per GPU, torch.distributed) is
// paper_1309_1889_b200/parallel.py:SpatialDecomposition.
#include <cuda_runtime.h>

#include <climits>
#include <cstring>
#include <stdexcept>
#include <string>

#include "msmb_engine.cuh"

using namespace msmb;

namespace {

void ckd(cudaError_t e, const char* w) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(w) + ": " + cudaGetErrorString(e));
}

// owned planes [pl0, pl1) of level k of `src` into the exchange buffer (same offsets)
void export_planes(cudaStream_t st, const Geometry& g, const Part& P, int k, const double* src, long long* x) {
    const LevelGeom& lv = g.lv[k];
    const size_t plane = size_t(lv.dims[1]) * lv.dims[2];
    const size_t off = lv.offset + size_t(P.pl0[k]) * plane;
    const size_t cnt = size_t(P.pl1[k] - P.pl0[k]) * plane;
    if (cnt) ckd(cudaMemcpyAsync(x + off, src + off, cnt * sizeof(double), cudaMemcpyDeviceToDevice, st), "D2D");
}

// The pair sum overlaps the long-range chain and the exchanges: phase 0 checks the
// binning (and the pair-list capacity) synchronously, then leaves the pair kernel
// running on the field's main stream; the chain of phases 1 and 2 runs on its side
// stream; phase 2 joins both before interpolation.
int phase0(msmb_field* f, Workspace& W, DevState& s, long long* xbuf, int rebuild, double* rebuilt) {
    const Geometry& g = W.g;
    cudaStream_t st = f->stream, sd = f->side_hi;
    for (int attempt = 0; attempt < 8; ++attempt) {
        ensure_const_table(f, W);
        int rb0 = 0;
        ckd(cudaMemcpy(&rb0, W.c.flag + 2, sizeof(int), cudaMemcpyDeviceToHost), "D2H");
        int nl = launch_reset_err(st, W.err, 0);
        nl += launch_bin(st, g, s, W.a, W.c, W.err);
        nl += launch_sort(st, g, s, W.a, W.c, W.err);
        // the list is rebuilt when invalid or after a skin/2 move, as on one GPU (`rebuild`,
        // the caller's `kicks`, is ignored: the same schedule as msmb_propagate)
        (void)rebuild;
        nl += launch_clusters(st, g, s.n, s, W.a, W.c, W.err, W.cap, W.part, attempt > 0 ? 1 : 0);
        nl += launch_err_brute(st, s.n, s, W.a, W.err);
        nl += launch_finalize(st, s, W.err);
        f->launches += nl;
        ckd(cudaGetLastError(), "kernel launch");
        const ErrRec r = read_err(f, W);
        if (r.kind == kOverflowKind) {
            grow_cap(W, r);
            continue;
        }
        // binning, sorting and error detection are replicated: every part fails alike
        if (r.kind) return engine_set_error(f, error_from_rec(r));
        int rb1 = 0;
        ckd(cudaMemcpy(&rb1, W.c.flag + 2, sizeof(int), cudaMemcpyDeviceToHost), "D2H");
        if (rebuilt) *rebuilt = rb1 != rb0 ? 1.0 : 0.0;
        f->launches += launch_anterp(st, g, W.a, W.c, W.L, W.err, W.part);
        ckd(cudaEventRecord(f->fork_ev, st), "record");
        f->launches += launch_pairs(st, g, s.n, s, W.a, W.c, W.err, W.cap, W.part); // joined in phase 2
        ckd(cudaStreamWaitEvent(sd, f->fork_ev, 0), "wait");
        if (W.part.nparts > 1) { // one part: the charges stay where phase 1 reads them
            const LevelGeom& l0 = g.lv[0];
            f->launches += launch_fill_i64(sd, xbuf, int64_t(l0.size), LLONG_MIN);
            export_planes(sd, g, W.part, 0, W.L.charge, xbuf);
        }
        ckd(cudaGetLastError(), "kernel launch");
        ckd(cudaStreamSynchronize(sd), "sync");
        return MSMB_OK;
    }
    return engine_set_error(f, Error{MSMB_ERR_INTERNAL, -1, -1, -1, "pair list did not converge"});
}

int phase1(msmb_field* f, Workspace& W, const long long* xin, long long* xbuf) {
    const Geometry& g = W.g;
    cudaStream_t sd = f->side_hi;
    const bool x = W.part.nparts > 1;
    if (x) ckd(cudaMemcpyAsync(W.L.charge, xin, sizeof(double) * g.lv[0].size, cudaMemcpyDeviceToDevice, sd), "D2D");
    ensure_const_table(f, W);
    f->launches += launch_restrict_all(sd, g, W.L, W.err);
    // the FFT path transforms whole levels (replicated); the direct path only owned planes
    f->launches += W.lattice_fft ? launch_lattice_fft(sd, W.fft, W.err) : launch_lattice(sd, g, W.L, W.err, W.part);
    if (x) {
        f->launches += launch_fill_i64(sd, xbuf, int64_t(g.lattice_total), LLONG_MIN);
        for (int k = 0; k + 1 < g.levels; ++k) export_planes(sd, g, W.part, k, W.L.pot, xbuf);
    }
    ckd(cudaGetLastError(), "kernel launch");
    ckd(cudaStreamSynchronize(sd), "sync");
    return MSMB_OK;
}

int phase2(msmb_field* f, Workspace& W, DevState& s, const long long* xin, long long* xbuf, double dt, int kicks,
           int drift, double conv, double* energy) {
    const Geometry& g = W.g;
    cudaStream_t st = f->stream, sd = f->side_hi;
    const bool x = W.part.nparts > 1;
    if (x) ckd(cudaMemcpyAsync(W.L.pot, xin, sizeof(double) * g.lattice_total, cudaMemcpyDeviceToDevice, sd), "D2D");
    f->launches += W.fft_top.n ? launch_lattice_fft(sd, W.fft_top, W.err) : launch_top(sd, g, W.L, W.err);
    f->launches += launch_prolong_all(sd, g, W.L, W.err);
    ckd(cudaEventRecord(f->join_ev, sd), "record");
    ckd(cudaStreamWaitEvent(st, f->join_ev, 0), "join"); // pair sum (phase 0) + long-range chain
    DevOut o = W.o;
    o.phi = o.phis = o.phil = nullptr;
    if (s.n) ckd(cudaMemsetAsync(o.e, 0, sizeof(double) * size_t(s.n), st), "memset"); // unowned e_i = 0
    f->launches += launch_interp(st, g, s.n, W.a, W.c, W.L, o, W.err, 1, W.part);
    f->launches += launch_verlet_part(st, g, W.c, W.a, s, o, dt, conv, kicks, drift, W.part, W.err);
    if (x) {
        f->launches += launch_fill_i64(st, xbuf, 6 * s.n, LLONG_MIN);
        f->launches += launch_export_state(st, g, W.c, W.a, s, xbuf, W.part);
    }
    ckd(cudaGetLastError(), "kernel launch");
    double e = 0.0;
    if (s.n) ckd(cudaMemcpyAsync(&e, W.o.energy, sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
    const ErrRec r = read_err(f, W); // synchronizes the main stream
    record_counters(f, W, r);
    if (r.kind) return engine_set_error(f, error_from_rec(r));
    if (energy) *energy = e;
    return MSMB_OK;
}

// phase 3: positions (x, y, z = the first 3 n doubles of the state); phase 4: velocities
int phase34(msmb_field* f, Workspace& W, DevState& s, const long long* xbuf, int which) {
    const size_t off = which == 4 ? 3 * size_t(s.n) : 0;
    if (s.n && W.part.nparts > 1)
        ckd(cudaMemcpyAsync(s.x + off, xbuf + off, sizeof(double) * 3 * size_t(s.n), cudaMemcpyDeviceToDevice,
                            f->stream),
            "D2D");
    ckd(cudaStreamSynchronize(f->stream), "sync");
    return MSMB_OK;
}

} // namespace

extern "C" int msmb_dd_plan(const msmb_msm_config* cfg, const msmb_units* units, const double box[3], int64_t n,
                            int nparts, int part, int* out, int cap) {
    if (!cfg || !units || !box || nparts < 1 || part < 0 || part >= nparts) return MSMB_ERR_CONFIG;
    Geometry g;
    Error e = build_geometry(*cfg, *units, box, n, g);
    if (e.kind) return e.kind;
    const Part P = make_part(g, nparts, part);
    // [ncx, cx0, cx1, levels, (d0_k, pl0_k, pl1_k) per level]
    const int need = 4 + 3 * g.levels;
    if (!out || cap < need) return MSMB_ERR_CONFIG;
    out[0] = g.ncx;
    out[1] = P.cx0;
    out[2] = P.cx1;
    out[3] = g.levels;
    for (int k = 0; k < g.levels; ++k) {
        out[4 + 3 * k] = g.lv[k].dims[0];
        out[5 + 3 * k] = P.pl0[k];
        out[6 + 3 * k] = P.pl1[k];
    }
    return MSMB_OK;
}

extern "C" int msmb_dd_set_part(msmb_field* f, int nparts, int part) {
    if (!f) return MSMB_ERR_CONFIG;
    std::lock_guard<std::recursive_mutex> lk(f->mu);
    if (f->kind != MSMB_FIELD_MSM)
        return engine_set_error(f, Error{MSMB_ERR_CONFIG, -1, -1, -1, "this entry point needs an MSM field"});
    if (nparts < 1 || part < 0 || part >= nparts)
        return engine_set_error(f, Error{MSMB_ERR_CONFIG, -1, -1, -1, "invalid decomposition part"});
    f->dd_nparts = nparts;
    f->dd_part = part;
    if (f->ws) f->ws->part = make_part(f->ws->g, nparts, part);
    return MSMB_OK;
}

extern "C" int msmb_set_pair_skin(msmb_field* f, double skin) {
    if (!f || !(skin >= 0.0)) return MSMB_ERR_CONFIG;
    std::lock_guard<std::recursive_mutex> lk(f->mu);
    f->pair_skin = skin;
    f->ws.reset(); // rebuilt on the next call
    return MSMB_OK;
}

extern "C" int msmb_set_list_reuse(msmb_field* f, int reuse) {
    if (!f) return MSMB_ERR_CONFIG;
    std::lock_guard<std::recursive_mutex> lk(f->mu);
    f->list_reuse = reuse ? 1 : 0;
    return MSMB_OK;
}

extern "C" int msmb_set_lattice_method(msmb_field* f, int direct) {
    if (!f) return MSMB_ERR_CONFIG;
    std::lock_guard<std::recursive_mutex> lk(f->mu);
    if (f->kind != MSMB_FIELD_MSM)
        return engine_set_error(f, Error{MSMB_ERR_CONFIG, -1, -1, -1, "this entry point needs an MSM field"});
    f->lattice_direct = direct ? 1 : 0;
    f->ws.reset(); // rebuilt on the next call with the chosen method
    return MSMB_OK;
}

extern "C" int msmb_dd_sizes(msmb_field* f, msmb_system* sys, int64_t* out) {
    if (!f || !sys || !out) return MSMB_ERR_CONFIG;
    std::lock_guard<std::recursive_mutex> lk(f->mu);
    if (f->kind != MSMB_FIELD_MSM)
        return engine_set_error(f, Error{MSMB_ERR_CONFIG, -1, -1, -1, "this entry point needs an MSM field"});
    try {
        cudaSetDevice(f->device);
        Error e = ensure_workspace(f, sys->st.n, sys->st.box);
        if (e.kind) return engine_set_error(f, e);
        out[0] = int64_t(f->ws->g.lv[0].size);
        out[1] = int64_t(f->ws->g.lattice_total);
        out[2] = 6 * sys->st.n;
        return MSMB_OK;
    } catch (const std::exception& ex) {
        return engine_set_error(f, Error{MSMB_ERR_CUDA, -1, -1, -1, ex.what()});
    }
}

extern "C" int msmb_dd_phase(msmb_field* f, msmb_system* sys, int phase, double dt, int kicks, int drift,
                             const msmb_units* units, const void* xin, void* xout, double* energy) {
    if (!f || !sys || (phase > 0 && !xin) || (phase < 3 && !xout)) return MSMB_ERR_CONFIG;
    std::lock_guard<std::recursive_mutex> lk(f->mu);
    if (f->kind != MSMB_FIELD_MSM)
        return engine_set_error(f, Error{MSMB_ERR_CONFIG, -1, -1, -1, "this entry point needs an MSM field"});
    try {
        cudaSetDevice(f->device);
        f->last = Error{};
        const msmb_units u = units ? *units : f->units;
        Error e = validate_units(u);
        if (e.kind) return engine_set_error(f, e);
        e = ensure_workspace(f, sys->st.n, sys->st.box);
        if (e.kind) return engine_set_error(f, e);
        Workspace& W = *f->ws;
        DevState s = sys->st.dev();
        const long long* xi = static_cast<const long long*>(xin);
        long long* xo = static_cast<long long*>(xout);
        switch (phase) {
            case 0: return phase0(f, W, s, xo, kicks, energy); // *energy = 1: the list was rebuilt
            case 1: return phase1(f, W, xi, xo);
            case 2: return phase2(f, W, s, xi, xo, dt, kicks, drift, u.energy_to_native, energy);
            case 3:
            case 4: return phase34(f, W, s, xi, phase);
            default: return engine_set_error(f, Error{MSMB_ERR_CONFIG, -1, -1, -1, "invalid phase"});
        }
    } catch (const std::exception& ex) {
        return engine_set_error(f, Error{MSMB_ERR_CUDA, -1, -1, -1, ex.what()});
    }
}
