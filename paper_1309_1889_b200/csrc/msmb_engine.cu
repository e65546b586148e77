// Host engine + C ABI (include/msmb.h).
//
// One msmb_field == one paramd::MsmField (include/paramd/force_field.hpp:62-73)
// bound to one GPU.  An evaluation is a fixed sequence of sm_100a kernels on the
// field's stream (see msmb_kernels.cu for the stage map); a velocity-Verlet
// propagate (src/integrate.cpp:13-36) is the initial evaluation followed by
// `steps` replays of a CUDA graph holding {kick(+kick)+drift, evaluation}.
// Errors are detected on the device (ErrRec) and surface after the call with
// the reference's exception type, message and particle indices; kernels of a
// failed evaluation and of every later step become no-ops, so the state a
// caller gets back on error is the untouched input (the reference throws).
#include <cuda_runtime.h>

#include <chrono>
#include <nvtx3/nvToolsExt.h>

#include <cstdlib>
#include <cstring>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>

#include "msmb_engine.cuh"

namespace msmb {

size_t conv_smem_bytes(const ConvTable& t);
cudaError_t conv_prepare(size_t bytes);

struct CudaErr : std::runtime_error {
    cudaError_t code;
    CudaErr(cudaError_t c, const std::string& w) : std::runtime_error(w), code(c) {}
};

static void ck(cudaError_t e, const char* where) {
    if (e != cudaSuccess) throw CudaErr(e, std::string(where) + ": " + cudaGetErrorString(e));
}

Workspace::~Workspace() {
    std::lock_guard<std::recursive_mutex> dl(device_mutex());
    if (gx_eval) cudaGraphExecDestroy(gx_eval);
    if (gx_step1) cudaGraphExecDestroy(gx_step1);
    if (gx_step2) cudaGraphExecDestroy(gx_step2);
    if (err) cudaFree(err);
    if (err_host) cudaFreeHost(err_host);
}

// ---- stage timer ------------------------------------------------------------------
int StageTimer::stage_index(const char* name) {
    for (size_t i = 0; i < names.size(); ++i)
        if (names[i] == name) return int(i);
    names.emplace_back(name);
    ms.push_back(0.0);
    launches.push_back(0);
    return int(names.size() - 1);
}

cudaEvent_t StageTimer::ev() {
    if (!pool.empty()) {
        cudaEvent_t e = pool.back();
        pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

void StageTimer::resolve() {
    for (auto& p : pending) {
        float t = 0.f;
        if (cudaEventSynchronize(p.b) == cudaSuccess && cudaEventElapsedTime(&t, p.a, p.b) == cudaSuccess)
            ms[p.stage] += t;
        launches[p.stage] += p.nl;
        pool.push_back(p.a);
        pool.push_back(p.b);
    }
    pending.clear();
}

StageTimer::~StageTimer() {
    for (auto& p : pending) {
        cudaEventDestroy(p.a);
        cudaEventDestroy(p.b);
    }
    for (auto e : pool) cudaEventDestroy(e);
}

// ---- errors -----------------------------------------------------------------------
int engine_set_error(msmb_field* f, const Error& e) {
    f->last = e;
    // a failed evaluation may have left a partial pair list: rebuild at the next one
    if (f->ws && f->ws->c.flag) { // the list and the cell sort must be rebuilt (kernels skipped work)
        cudaMemsetAsync(f->ws->c.flag + 3, 0, sizeof(int), f->stream);
        cudaMemsetAsync(f->ws->c.flag + 6, 0, sizeof(int), f->stream);
    }
    return e.kind;
}

int cuda_fail(msmb_field* f, cudaError_t e, const char* where) {
    Error er;
    er.kind = MSMB_ERR_CUDA;
    er.msg = std::string(where) + ": " + cudaGetErrorString(e);
    if (f) f->last = er;
    return MSMB_ERR_CUDA;
}

Error error_from_rec(const ErrRec& r) {
    Error e;
    e.kind = r.kind;
    e.step = r.step;
    e.i = r.err_i;
    e.j = r.err_j;
    char buf[256];
    switch (r.kind) {
        case MSMB_ERR_COVERAGE:
            snprintf(buf, sizeof buf, "particle %lld outside grid coverage", (long long)r.err_i);
            e.msg = buf;
            break;
        case MSMB_ERR_COINCIDENT:
            snprintf(buf, sizeof buf, "particles %lld and %lld coincide", (long long)r.err_i,
                     (long long)r.err_j);
            e.msg = buf;
            break;
        case MSMB_ERR_DOMAIN:
            if (r.err_i >= 0 && r.err_j < 0) { // pair-only fields: infinite coordinate (msmb.h)
                snprintf(buf, sizeof buf, "particle %lld has a non-finite position", (long long)r.err_i);
                e.msg = buf;
            } else {
                e.msg = "kernel_g_star: r must be > 0";
            }
            break;
        default:
            e.msg = "internal error";
    }
    return e;
}

// ---- workspace --------------------------------------------------------------------
template <class T>
static T* walloc(Workspace& W, size_t count) {
    auto b = std::make_unique<DBuf>();
    ck(b->alloc(sizeof(T) * (count ? count : 1)), "cudaMalloc");
    T* p = b->as<T>();
    W.bufs.push_back(std::move(b));
    return p;
}

template <class T>
static T* wupload(Workspace& W, const std::vector<T>& v) {
    T* p = walloc<T>(W, v.size());
    if (!v.empty()) ck(cudaMemcpy(p, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice), "upload");
    return p;
}

// Both new buffers are allocated before the old ones are released and swapped in
// only when both succeeded, so a failed growth leaves the workspace consistent
// (old capacity, old pointers, graphs still valid).
static void alloc_plist(Workspace& W, int cap) {
    DBuf pl, pm;
    ck(pl.alloc(sizeof(int) * size_t(W.maxclu) * size_t(cap)), "cudaMalloc plist");
    ck(pm.alloc(sizeof(unsigned) * 32 * size_t(W.maxclu) * size_t(cap)), "cudaMalloc pmask");
    std::swap(W.plist_buf.p, pl.p);
    std::swap(W.plist_buf.bytes, pl.bytes);
    std::swap(W.pmask_buf.p, pm.p);
    std::swap(W.pmask_buf.bytes, pm.bytes);
    W.c.plist = W.plist_buf.as<int>();
    W.c.pmask = W.pmask_buf.as<unsigned>();
    W.cap = cap;
}

static std::atomic<uint64_t> g_ws_uid{1};
static std::mutex g_const_mu;
static uint64_t g_const_owner[64] = {0}; // per device: uid of the workspace whose stencil is in c_lat_*

// k_lattice<true> reads the level-0 stencil from constant memory, which is shared by
// every field of the process on a device: make sure it holds this workspace's table.
void ensure_const_table(msmb_field* f, Workspace& W) {
    if (!W.L.lat_const) return;
    std::lock_guard<std::mutex> lk(g_const_mu);
    const int d = f->device & 63;
    if (g_const_owner[d] == W.uid) return;
    ck(lattice_upload_const(W.g, f->stream), "cudaMemcpyToSymbol");
    g_const_owner[d] = W.uid;
}

static bool make_levels(msmb_field* f, Workspace& W, Error& e);

// per-atom outputs, state backup/staging and the error record
static void alloc_outputs(Workspace& Wr, int64_t n) {
    Workspace* W = &Wr;
    const size_t N = size_t(n > 0 ? n : 1);
    DevOut& o = W->o;
    o.fx = walloc<double>(*W, N);
    o.fy = walloc<double>(*W, N);
    o.fz = walloc<double>(*W, N);
    o.phi = walloc<double>(*W, N);
    o.phis = walloc<double>(*W, N);
    o.phil = walloc<double>(*W, N);
    o.e = walloc<double>(*W, N);
    o.partial = walloc<double>(*W, size_t(reduce_blocks(n)));
    o.energy = walloc<double>(*W, 1);
    ck(W->backup.alloc(sizeof(double) * 6 * N), "cudaMalloc backup");
    ck(W->staging.alloc(sizeof(double) * 3 * N), "cudaMalloc staging");
    ck(W->staging2.alloc(sizeof(double) * 3 * N), "cudaMalloc staging");
    ck(cudaMalloc(&W->err, sizeof(ErrRec)), "cudaMalloc err");
    ck(cudaMallocHost(&W->err_host, sizeof(ErrRec)), "cudaMallocHost err");
}

static std::unique_ptr<Workspace> make_workspace(msmb_field* f, int64_t n, const double* box,
                                                 Error& e) {
    auto W = std::make_unique<Workspace>();
    W->uid = g_ws_uid++;
    const size_t NN = size_t(n > 0 ? n : 1);
    if (f->rep_on || f->kind == MSMB_FIELD_DIRECT) { // all-pairs buffers (msmb_direct.cu)
        W->ap.S = allpairs_splits(n);
        W->ap.part = W->ap.S > 1 ? walloc<double>(*W, size_t(W->ap.S) * 5 * NN) : nullptr;
        W->ap.e_rep = walloc<double>(*W, NN);
    }
    if (f->kind == MSMB_FIELD_DIRECT) { // no binning, no grid: only the outputs
        Geometry& g = W->g;
        g.kind = MSMB_FIELD_DIRECT;
        g.units = f->units;
        for (int ax = 0; ax < 3; ++ax) g.box[ax] = box[ax];
        W->n = n;
        alloc_outputs(*W, n);
        ck(cudaDeviceSynchronize(), "sync");
        return W;
    }
    e = f->kind == MSMB_FIELD_MSM ? build_geometry(f->cfg, f->units, box, n, W->g)
                                  : build_pair_geometry(f->kind, f->cut, f->units, box, n, W->g);
    if (e.kind) return nullptr;
    const bool msm = f->kind == MSMB_FIELD_MSM;
    Geometry& g = W->g;
    if (f->pair_skin >= 0.0) g.skin = f->pair_skin;
    W->n = n;
    W->whole = make_part(g, 1, 0);
    W->part = make_part(g, f->dd_nparts, f->dd_part);
    const size_t N = size_t(n > 0 ? n : 1);
    DevAtoms& a = W->a;
    a.key = walloc<int>(*W, N);
    a.rank = walloc<int>(*W, N);
    a.perm = walloc<int>(*W, N);
    a.outlist = walloc<int>(*W, N);
    a.aw = msm ? walloc<double>(*W, N * 12) : nullptr;
    a.phis = walloc<double>(*W, N);
    a.fsx = walloc<double>(*W, N);
    a.fsy = walloc<double>(*W, N);
    a.fsz = walloc<double>(*W, N);
    a.cl_perm = walloc<int>(*W, N);
    a.cl_inv = walloc<int>(*W, N);
    a.xc = walloc<double>(*W, N);
    a.yc = walloc<double>(*W, N);
    a.zc = walloc<double>(*W, N);
    a.qc = walloc<double>(*W, N);
    a.ref = walloc<double>(*W, 3 * N);
    {
        const int64_t maxclu_est = n / 32 + g.ncols + 1; // as launch_pairs
        const int sp = pair_split(maxclu_est);
        a.pair_part = sp > 1 ? walloc<double>(*W, size_t(sp) * 4 * N) : nullptr;
    }
    DevCells& c = W->c;
    c.count = walloc<int>(*W, size_t(g.ncells + 1));
    c.start = walloc<int>(*W, size_t(g.ncells + 1));
    c.nat = walloc<int2>(*W, g.lv[0].size);
    c.col_cnt = walloc<int>(*W, size_t(g.ncols + 1));
    c.col_off = walloc<int>(*W, size_t(g.ncols + 1));
    W->maxclu = n / 32 + g.ncols + 1;
    c.clu = walloc<int2>(*W, size_t(W->maxclu));
    c.blo = walloc<float4>(*W, size_t(W->maxclu));
    c.bhi = walloc<float4>(*W, size_t(W->maxclu));
    c.nclu = walloc<int>(*W, 1);
    c.pcnt = walloc<int>(*W, size_t(W->maxclu));
    c.dcnt = walloc<int>(*W, size_t(W->maxclu));
    c.dlist = walloc<int>(*W, size_t(W->maxclu) * size_t(std::max(g.dense_cap, 32)));
    ck(cudaMemset(c.dcnt, 0, sizeof(int) * size_t(W->maxclu)), "memset");
    c.scan_tmp = walloc<int>(*W, size_t((std::max(g.ncells, g.ncols) + 1 + 4095) / 4096 + 8));
    c.colstart = walloc<int>(*W, size_t(g.ncols + 1));
    c.flag = walloc<int>(*W, 10);
    ck(cudaMemset(c.nclu, 0, sizeof(int)), "memset");
    ck(cudaMemset(c.flag, 0, 10 * sizeof(int)), "memset");
    ck(cudaMemset(c.colstart, 0, sizeof(int) * size_t(g.ncols + 1)), "memset");
    alloc_plist(*W, g.pair_cap);
    alloc_outputs(*W, n);
    if (msm && !make_levels(f, *W, e)) return nullptr;
    // wupload's pageable cudaMemcpy may return before its DMA lands, and the
    // field's streams are non-blocking (not ordered after the legacy stream)
    ck(cudaDeviceSynchronize(), "sync uploads");
    return W;
}

// The MSM grid hierarchy: level lattices, transfer and stencil tables, FFT plans.
static bool make_levels(msmb_field* f, Workspace& Wr, Error& e) {
    Workspace* W = &Wr;
    const Geometry& g = W->g;
    DevLevels& L = W->L;
    L.charge = walloc<double>(*W, g.lattice_total);
    L.pot = walloc<double>(*W, g.lattice_total);
    L.anterp_part = walloc<double>(*W, anterp_tile_part_doubles(g));
    for (int k = 0; k + 1 < g.levels; ++k)
        for (int ax = 0; ax < 3; ++ax) {
            const TransferAxis& T = g.tr[k][ax];
            L.tr_base[k][ax] = wupload(*W, T.base);
            L.tr_w[k][ax] = wupload(*W, T.w);
            L.tr_rcnt[k][ax] = wupload(*W, T.rcnt);
            L.tr_ridx[k][ax] = wupload(*W, T.ridx);
            L.tr_rw[k][ax] = wupload(*W, T.rw);
        }
    size_t smem = 0;
    for (int k = 0; k < g.levels; ++k) {
        const ConvTable& t = (k == g.levels - 1) ? g.top : g.lattice[k];
        std::vector<int4> rows(t.rows.size());
        for (size_t i = 0; i < rows.size(); ++i)
            rows[i] = make_int4(t.rows[i].dx, t.rows[i].dy, t.rows[i].m, t.rows[i].tap_off);
        L.rows[k] = wupload(*W, rows);
        L.dxb[k] = wupload(*W, t.dx_begin);
        L.taps[k] = wupload(*W, t.taps);
        smem = std::max(smem, conv_smem_bytes(t));
    }
    if (g.levels >= 2) {
        L.lat_rowidx = wupload(*W, g.lat.rowidx);
        std::vector<int2> rc(g.lat.rowchunks.size());
        for (size_t i = 0; i < rc.size(); ++i) rc[i] = make_int2(g.lat.rowchunks[i].x, g.lat.rowchunks[i].y);
        L.lat_rowchunks = wupload(*W, rc);
        L.lat_taps = wupload(*W, g.lat.taps);
        L.lat_S = lattice_splits(g);
        L.lat_const = lattice_const_fits(g) ? 1 : 0;
        L.lat_partial = L.lat_S > 1 ? walloc<double>(*W, size_t(L.lat_S) * g.lattice_total) : nullptr;
        ck(lattice_prepare(lattice_smem_bytes(g)), "cudaFuncSetAttribute");
    }
    // FFT lattice cutoff + large top level: plans, twiddles, kernel spectra (msmb_fft.cu)
    W->lattice_fft = !f->lattice_direct && g.levels >= 2;
    if (W->lattice_fft) {
        std::vector<int> Ms;
        std::vector<double2> tw;
        auto tw_of = [&](int M) {
            size_t off = 0;
            for (size_t i = 0; i < Ms.size(); off += size_t(Ms[i]), ++i)
                if (Ms[i] == M) return int(off);
            Ms.push_back(M);
            for (int m = 0; m < M; ++m) {
                const long double ang = -2.0L * 3.141592653589793238462643383279502884L * m / M;
                tw.push_back(make_double2(double(cosl(ang)), double(sinl(ang))));
            }
            return int(off);
        };
        // job lists: cutoff levels 0..l-2 (pad d + R) and, if large, the top (pad 2d - 1)
        auto plan = [&](FftJobs& J, int k0, int k1, bool top) {
            J = FftJobs{};
            J.n = k1 - k0;
            size_t boff = 0;
            for (int k = k0; k < k1; ++k) {
                FftLevel& lv = J.lv[k - k0];
                for (int ax = 0; ax < 3; ++ax) {
                    lv.d[ax] = g.lv[k].dims[ax];
                    const int M = fft_len(top ? 2 * lv.d[ax] - 1 : lv.d[ax] + g.lat.R);
                    lv.ax[ax] = fft_axis(M, tw_of(M));
                    J.maxM = std::max(J.maxM, M);
                }
                lv.boff = lv.soff = boff;
                boff += size_t(lv.ax[0].M) * lv.ax[1].M * lv.ax[2].M;
                lv.q = L.charge + g.lv[k].offset;
                lv.u = L.pot + g.lv[k].offset;
            }
            // lines per FFT tile: 4 (64-thread CTAs of ~9 KB), which fit beside the pair
            // kernel's CTAs; C2-S 0.842 ms/step vs 0.849 with 16-line tiles of 256
            // threads (2 lines: 0.842, 1: 0.855).  MSMB_FFT_LINES overrides (timing knob;
            // results do not depend on it)
            int lines = 4;
            if (const char* e = std::getenv("MSMB_FFT_LINES")) lines = std::max(1, std::min(16, atoi(e)));
            J.L = std::max(1, std::min(lines, 2048 / std::max(J.maxM, 1)));
            J.buf = walloc<double2>(*W, boff);
            J.spec = walloc<double>(*W, boff);
            return boff;
        };
        const int lt = g.levels - 1;
        plan(W->fft, 0, lt, false);
        const bool big_top = int64_t(g.lv[lt].size) > kTopFftMin;
        if (big_top) plan(W->fft_top, lt, lt + 1, true);
        const double2* twd = wupload(*W, tw);
        W->fft.tw = twd;
        W->fft_top.tw = twd;
        ck(cudaDeviceSynchronize(), "sync uploads");
        ck(fft_prepare(size_t(2) * std::max(W->fft.L * W->fft.maxM, W->fft_top.L * W->fft_top.maxM) *
                       sizeof(double2)),
           "cudaFuncSetAttribute");
        std::vector<FftKernel> K(size_t(W->fft.n));
        for (int k = 0; k < W->fft.n; ++k)
            K[k] = FftKernel{0, L.lat_rowidx, L.lat_taps, {g.lat.R, g.lat.R, g.lat.R}, g.lat.TW, std::ldexp(1.0, -k)};
        launch_fft_spectrum(f->stream, W->fft, K.data());
        if (big_top) {
            const ConvTable& t = g.top;
            const FftKernel KT{1, nullptr, L.taps[lt], {t.Rx, t.Ry, t.Rz}, (2 * t.Rz + 1 + kConvL - 1) / kConvL * kConvL,
                               1.0};
            launch_fft_spectrum(f->stream, W->fft_top, &KT);
        }
        ck(cudaGetLastError(), "fft spectrum");
    }
    if (smem > 227 * 1024) {
        e.kind = MSMB_ERR_CONFIG;
        e.msg = "msm: top level of " + std::to_string(g.lv[g.levels - 1].size) +
                " points exceeds this build's shared-memory stencil tile";
        return false;
    }
    ck(conv_prepare(smem), "cudaFuncSetAttribute");
    ck(top_prepare(g), "cudaFuncSetAttribute");
    return true;
}

Error ensure_workspace(msmb_field* f, int64_t n, const double* box) {
    std::lock_guard<std::recursive_mutex> dl(device_mutex()); // allocations + device syncs
    Error e;
    if (f->ws && f->ws->n == n && f->ws->g.box[0] == box[0] && f->ws->g.box[1] == box[1] &&
        f->ws->g.box[2] == box[2])
        return e;
    f->ws.reset();
    f->ws = make_workspace(f, n, box, e);
    return e;
}

// ---- one evaluation ------------------------------------------------------------------
// One engine stage: an NVTX range (named like the stage, visible to ncu --nvtx and
// Nsight Systems on eager launches and graph captures) and, when stage timing is
// on, CUDA events around its launches.
struct StageScope {
    msmb_field* f;
    int stage = -1;
    cudaEvent_t a = nullptr;
    bool open = true;
    StageScope(msmb_field* ff, const char* name) : f(ff) {
        nvtxRangePushA(name);
        if (!f->timer.on) return;
        stage = f->timer.stage_index(name);
        a = f->timer.ev();
        cudaEventRecord(a, f->stream);
    }
    void done(int nl) {
        f->launches += nl;
        if (open) nvtxRangePop(), open = false;
        if (stage < 0) return;
        cudaEvent_t b = f->timer.ev();
        cudaEventRecord(b, f->stream);
        f->timer.pending.push_back({stage, a, b, nl});
    }
    ~StageScope() {
        if (open) nvtxRangePop();
    }
};

static thread_local bool t_capturing = false; // graph captures skip the pair statistics

static const char* kStages[] = {"bin", "sort", "clusters", "pairs", "anterp", "restrict",
                                "lattice", "top", "prolong", "interp", "finalize", "overlay"};
constexpr int kNumStages = 12;
constexpr int kBenchStages = 11; // stage names msmb_bench_propagate reports (msmb.h)

static int stage_id(const char* name) {
    for (int i = 0; i < kNumStages; ++i)
        if (!strcmp(kStages[i], name)) return i;
    return -1;
}

// The long-range chain (anterpolation .. prolongation) depends only on the binned,
// sorted atoms, and the short-range pair sum only on the cluster lists, so after
// the sort the chain is forked onto the field's side stream and
// joined before interpolation, which consumes both (a fork/join in the captured
// graphs).  The two branches write disjoint buffers; every reduction keeps its
// fixed order, so results do not depend on how the branches interleave.  With
// per-stage timing on, everything runs on one stream so the stage events are
// exclusive.
// `rebuild`: force a pair-list rebuild; otherwise the list is rebuilt only when it
// is not valid (never built, capacity grown, a failed evaluation, another part's
// columns) or once some atom moved more than skin/2 since it was built
// (launch_clusters) -- also across calls: a call that starts within skin/2 of the
// last build reuses its list.
// MSMB_TIMELINE=1: globaltimer stamps at the fork/join points of every evaluation
// (diagnostic only; msmb_bench_propagate prints the per-step averages to stderr)
void launch_stamp(cudaStream_t st, int idx);
void read_stamps(unsigned long long* h);
static const bool g_exp_stamps = std::getenv("MSMB_TIMELINE") != nullptr;
// MSMB_EXP_CHAIN (timing experiments only; results are wrong): 0 = no long-range chain,
// 1 = anterpolation only, 2 = everything but anterpolation, 3 = anterpolation + restriction,
// 4 = ... + lattice, 5 = ... + top (everything but prolongation)
static const int g_exp_chain = std::getenv("MSMB_EXP_CHAIN") ? std::atoi(std::getenv("MSMB_EXP_CHAIN")) : -1;
static int enqueue_eval(msmb_field* f, Workspace& W, DevState& s, bool outputs, bool rebuild = false) {
    cudaStream_t st = f->stream;
    const bool fork = !f->timer.on;
    cudaStream_t lr = fork ? f->side : st;
    const Geometry& g = W.g;
    int total = 0;
    auto run = [&](const char* name, auto&& fn) {
        StageScope sc(f, name);
        const int nl = fn();
        sc.done(nl);
        total += nl;
    };
    // PairRepulsionOverlay (force_field.cpp:45-68): after the base field's outputs,
    // all-pairs repulsion forces added to F, its energy added to the total
    // Nested overlays compose like the reference's decorators: the innermost term is
    // added first (each PairRepulsionOverlay::evaluate adds its term to its base's result).
    auto overlay = [&](DevOut& o, size_t first) {
        for (size_t t = first; t < f->rep.size(); ++t)
            run("overlay", [&] {
                int nl = launch_allpairs(st, s, g.units.coulomb_constant, 0, 1, f->rep[t].first, f->rep[t].second,
                                         W.ap, o, W.err);
                if (o.e) nl += launch_energy_sum(st, s.n, W.ap.e_rep, o.partial, 1.0, o.energy, 1, W.err);
                return nl;
            });
    };
    if (g.kind == MSMB_FIELD_DIRECT) { // direct_coulomb (electrostatics.cpp:43-64): all pairs
        DevOut o = W.o;
        if (!outputs) o.phi = o.phis = o.phil = o.e = nullptr;
        run("pairs", [&] {
            const bool rep1 = !f->rep.empty(); // the innermost overlay is fused into the direct sum
            int nl = launch_allpairs(st, s, g.units.coulomb_constant, 1, rep1 ? 1 : 0, rep1 ? f->rep[0].first : 0.0,
                                     rep1 ? f->rep[0].second : 1.0, W.ap, o, W.err);
            if (o.e) nl += launch_energy_sum(st, s.n, o.e, o.partial, g.units.coulomb_constant, o.energy, 0, W.err);
            if (o.e && rep1)
                nl += launch_energy_sum(st, s.n, W.ap.e_rep, o.partial, 1.0, o.energy, 1, W.err);
            return nl;
        });
        overlay(o, 1);
        run("finalize", [&] { return launch_finalize(st, s, W.err, 1); });
        return total;
    }
    if (g_exp_stamps) launch_stamp(st, 0);
    run("bin", [&] { return launch_bin(st, g, s, W.a, W.c, W.err); });
    if (g.kind != MSMB_FIELD_MSM) { // pair-only field: no grid hierarchy
        run("sort", [&] { return launch_sort(st, g, s, W.a, W.c, W.err); });
        run("clusters", [&] { return launch_clusters(st, g, s.n, s, W.a, W.c, W.err, W.cap, W.whole, rebuild ? 1 : 0); });
        run("pairs", [&] { return launch_pairs(st, g, s.n, s, W.a, W.c, W.err, W.cap, W.whole, !t_capturing); });
        DevOut o = W.o;
        if (!outputs) o.phi = o.phis = o.phil = o.e = nullptr;
        run("interp", [&] { return launch_pair_out(st, g, s.n, W.a, W.c, o, W.err, outputs ? 1 : 0, W.whole); });
        overlay(o, 0);
        run("finalize", [&] { return launch_finalize(st, s, W.err, 1); });
        return total;
    }
    // Forked evaluation.  Main stream: binning, the rebuild decision and the frozen-order
    // gather (they need the binning's coverage list, not the cell sort), then the pair kernel's
    // skin instance (it exits at once on a rebuild evaluation).  Stream la: the cell sort, then
    // the anterpolation; stream lr: the rest of the long-range chain.  Stream sr: after the
    // sort and the decision, the list rebuild and the pair kernel's rebuild instance (every
    // kernel exits at once on a skin evaluation).  So on a skin step the pair sum starts ~35 us
    // earlier (it no longer waits for the sort and the four exiting rebuild launches), and on
    // a rebuild step the rebuild runs beside the anterpolation.  Each output is written by one
    // kernel in a fixed order: results do not depend on the interleaving.
    cudaStream_t la = fork ? f->side_a : st; // cell sort + anterpolation, then the rest of the chain on lr
    cudaStream_t sr = fork ? f->side_r : st; // list rebuild + the pair kernel's rebuild instance
    if (fork) {
        ck(cudaEventRecord(f->fork_ev, st), "fork");
        ck(cudaStreamWaitEvent(la, f->fork_ev, 0), "fork");
    }
    run("sort", [&] { return launch_sort(la, g, s, W.a, W.c, W.err); });
    if (fork) {
        ck(cudaEventRecord(f->sort_ev, la), "fork");
        run("clusters", [&] {
            return launch_clusters(st, g, s.n, s, W.a, W.c, W.err, W.cap, W.whole, rebuild ? 1 : 0, 1, 1);
        });
        ck(cudaEventRecord(f->disp_ev, st), "fork");
        ck(cudaStreamWaitEvent(sr, f->disp_ev, 0), "fork");
        ck(cudaStreamWaitEvent(sr, f->sort_ev, 0), "fork");
    } else {
        run("clusters", [&] { return launch_clusters(st, g, s.n, s, W.a, W.c, W.err, W.cap, W.whole, rebuild ? 1 : 0); });
    }
    if (g_exp_stamps) { launch_stamp(st, 1); launch_stamp(la, 2); }
    if (g_exp_chain != 0 && g_exp_chain != 2)
        run("anterp", [&] { return launch_anterp(la, g, s, W.a, W.c, W.L, W.err, W.whole); });
    if (g_exp_stamps) launch_stamp(la, 7);
    if (fork) {
        ck(cudaEventRecord(f->mid_ev, la), "fork");
        ck(cudaStreamWaitEvent(lr, f->mid_ev, 0), "fork");
    }
    const bool full = g_exp_chain < 0 || g_exp_chain == 2;
    if (full || g_exp_chain >= 3) run("restrict", [&] { return launch_restrict_all(lr, g, W.L, W.err); });
    if (g_exp_stamps) launch_stamp(lr, 8);
    if (full || g_exp_chain >= 4)
        run("lattice", [&] {
            return W.lattice_fft ? launch_lattice_fft(lr, W.fft, W.err) : launch_lattice(lr, g, W.L, W.err, W.whole);
        });
    if (g_exp_stamps) launch_stamp(lr, 9);
    if (full || g_exp_chain >= 5)
        run("top", [&] {
            return W.fft_top.n ? launch_lattice_fft(lr, W.fft_top, W.err) : launch_top(lr, g, W.L, W.err);
        });
    if (g_exp_stamps) launch_stamp(lr, 10);
    if (full) run("prolong", [&] { return launch_prolong_all(lr, g, W.L, W.err); });
    if (g_exp_stamps) launch_stamp(lr, 3);
    if (fork) ck(cudaEventRecord(f->join_ev, lr), "join");
    if (g_exp_stamps) launch_stamp(st, 4);
    // (Measured, C2-S ms/step: pair kernel right away 0.751; after the cell sort 0.748; after
    // the anterpolation, which then runs alone in 55 us instead of ~245, 0.775.)
    run("pairs", [&] {
        return launch_pairs(st, g, s.n, s, W.a, W.c, W.err, W.cap, W.whole, !t_capturing, fork ? 1 : 0);
    });
    if (g_exp_stamps) launch_stamp(st, 5);
    if (fork) {
        run("clusters", [&] {
            return launch_clusters(sr, g, s.n, s, W.a, W.c, W.err, W.cap, W.whole, rebuild ? 1 : 0, 1, 2);
        });
        run("pairs", [&] {
            return launch_pairs(sr, g, s.n, s, W.a, W.c, W.err, W.cap, W.whole, !t_capturing, 2);
        });
        ck(cudaEventRecord(f->reb_ev, sr), "join");
        ck(cudaStreamWaitEvent(st, f->reb_ev, 0), "join");
        ck(cudaStreamWaitEvent(st, f->join_ev, 0), "join");
    }
    DevOut o = W.o;
    if (!outputs) o.phi = o.phis = o.phil = o.e = nullptr;
    run("interp", [&] { return launch_interp(st, g, s.n, W.a, W.c, W.L, o, W.err, outputs ? 1 : 0, W.whole); });
    overlay(o, 0);
    run("finalize", [&] { return launch_finalize(st, s, W.err); });
    if (g_exp_stamps) launch_stamp(st, 6);
    return total;
}

ErrRec read_err(msmb_field* f, Workspace& W) {
    ck(cudaMemcpyAsync(W.err_host, W.err, sizeof(ErrRec), cudaMemcpyDeviceToHost, f->stream),
       "read err");
    ck(cudaStreamSynchronize(f->stream), "cudaStreamSynchronize");
    f->timer.resolve();
    return *W.err_host;
}

void record_counters(msmb_field* f, const Workspace& W, const ErrRec& r) {
    f->counters[0] = int64_t(r.pairs / 2);
    f->counters[1] = int64_t(r.candidates);
    int nclu = 0;
    if (W.c.nclu) cudaMemcpy(&nclu, W.c.nclu, sizeof(int), cudaMemcpyDeviceToHost);
    f->counters[2] = nclu;
    f->counters[3] = W.g.lattice_taps_clipped;
    f->counters[4] = W.g.top_taps;
    f->counters[5] = W.launches_eval;
    int rebuilds = 0;
    if (W.c.flag) cudaMemcpy(&rebuilds, W.c.flag + 2, sizeof(int), cudaMemcpyDeviceToHost);
    f->counters[6] = rebuilds;
    // warps per i-cluster of the pair kernel: 1 = the large-system instance (k_pairs_mw<K, false>)
    f->counters[7] = (W.g.kind == MSMB_FIELD_MSM || W.g.kind == MSMB_FIELD_CUTOFF || W.g.kind == MSMB_FIELD_WOLF) &&
                             W.a.pair_part
                         ? pair_split(W.maxclu)
                         : 1;
}

void grow_cap(Workspace& W, const ErrRec& r) {
    std::lock_guard<std::recursive_mutex> dl(device_mutex());
    const int need = std::max(r.overflow, W.cap);
    const int cap = std::max(need + need / 4 + 32, W.cap * 2);
    alloc_plist(W, cap);
    ck(cudaMemset(W.c.flag + 3, 0, sizeof(int)), "memset"); // the list must be rebuilt
    ck(cudaDeviceSynchronize(), "sync");
}

// Every evaluate / propagate call starts from a freshly built pair list, so its
// results are a pure function of its input (the reference's evaluate is pure and
// bitwise repeatable): the summation order follows the list, and a
// list carried over from an earlier call would make the last bits depend on the
// call history -- e.g. on which parareal rank or fine replica ran a slice.
// msmb_set_list_reuse(f, 1) opts into carrying the list across calls.
static void fresh_list(msmb_field* f, Workspace& W) {
    if (!f->list_reuse && W.c.flag) ck(cudaMemsetAsync(W.c.flag + 3, 0, sizeof(int), f->stream), "memset");
}

// Evaluate the system in `s` (device), outputs left in W.o.
static int eval_device(msmb_field* f, StateBuf& sb, bool outputs) {
    Error e = ensure_workspace(f, sb.n, sb.box);
    if (e.kind) return engine_set_error(f, e);
    Workspace& W = *f->ws;
    DevState s = sb.dev();
    fresh_list(f, W);
    for (int attempt = 0; attempt < 8; ++attempt) {
        ensure_const_table(f, W);
        f->launches += launch_reset_err(f->stream, W.err, 0);
        W.launches_eval = enqueue_eval(f, W, s, outputs);
        ck(cudaGetLastError(), "kernel launch");
        const ErrRec r = read_err(f, W);
        if (r.kind == kOverflowKind) {
            grow_cap(W, r);
            continue;
        }
        record_counters(f, W, r);
        if (r.kind) return engine_set_error(f, error_from_rec(r));
        return MSMB_OK;
    }
    return engine_set_error(f, Error{MSMB_ERR_INTERNAL, -1, -1, -1, "pair list did not converge"});
}

static void destroy_graphs(Workspace& W) {
    if (W.gx_eval) cudaGraphExecDestroy(W.gx_eval);
    if (W.gx_step1) cudaGraphExecDestroy(W.gx_step1);
    if (W.gx_step2) cudaGraphExecDestroy(W.gx_step2);
    W.gx_eval = W.gx_step1 = W.gx_step2 = nullptr;
    W.graph_key = nullptr;
}

template <class Fn>
static cudaGraphExec_t capture(msmb_field* f, Fn&& fn);

// The three step graphs of a propagate call (cached per state buffer, dt and
// pair-list capacity): evaluation, first step (kick + drift + evaluation), and
// later steps (fused kick + kick + drift + evaluation).
static void ensure_graphs(msmb_field* f, Workspace& W, DevState& s, double dt, double conv) {
    if (W.graph_key == s.x && W.graph_dt == dt && W.graph_conv == conv && W.graph_cap == W.cap) return;
    destroy_graphs(W);
    int nl = 0;
    W.gx_eval = capture(f, [&] { nl = enqueue_eval(f, W, s, false); });
    W.launches_eval = nl;
    W.gx_step1 = capture(f, [&] {
        nl = launch_kick_drift(f->stream, s, W.o, dt, conv, 1, W.err);
        nl += enqueue_eval(f, W, s, false, false);
    });
    W.gx_step2 = capture(f, [&] {
        if (g_exp_stamps) launch_stamp(f->stream, 11);
        nl = launch_kick_drift(f->stream, s, W.o, dt, conv, 2, W.err);
        nl += enqueue_eval(f, W, s, false, false);
    });
    W.launches_step = nl;
    f->launches -= 3 * int64_t(W.launches_eval); // captures are not launches
    W.graph_key = s.x;
    W.graph_dt = dt;
    W.graph_conv = conv;
    W.graph_cap = W.cap;
}

template <class Fn>
static cudaGraphExec_t capture(msmb_field* f, Fn&& fn) {
    std::lock_guard<std::recursive_mutex> dl(device_mutex()); // no other thread allocates meanwhile
    struct Flag {
        Flag() { t_capturing = true; }
        ~Flag() { t_capturing = false; }
    } flag_scope;
    cudaGraph_t graph = nullptr;
    ck(cudaStreamBeginCapture(f->stream, cudaStreamCaptureModeThreadLocal), "BeginCapture");
    try {
        fn();
    } catch (...) { // never leave the stream (and this thread) in capture mode
        cudaStreamEndCapture(f->stream, &graph);
        if (graph) cudaGraphDestroy(graph);
        cudaGetLastError();
        throw;
    }
    ck(cudaStreamEndCapture(f->stream, &graph), "EndCapture");
    cudaGraphExec_t ex;
    ck(cudaGraphInstantiateWithFlags(&ex, graph, cudaGraphInstantiateFlagUseNodePriority),
       "GraphInstantiate");
    cudaGraphDestroy(graph);
    return ex;
}

int engine_propagate(msmb_field* f, StateBuf& sb, double dt, int steps, double conv, cudaEvent_t vel_ready) {
    if (!(dt > 0.0)) return engine_set_error(f, Error{MSMB_ERR_CONFIG, -1, -1, -1, "dt must be > 0"});
    if (steps < 1)
        return engine_set_error(f, Error{MSMB_ERR_CONFIG, -1, -1, -1, "steps_per_slice must be >= 1"});
    Error e = validate_units(f->units);
    if (e.kind) return engine_set_error(f, e);
    e = ensure_workspace(f, sb.n, sb.box);
    if (e.kind) return engine_set_error(f, e);
    Workspace& W = *f->ws;
    DevState s = sb.dev();
    const size_t N = size_t(sb.n > 0 ? sb.n : 1);
    double* bk = W.backup.as<double>();
    // keep the input state: restored on error and on pair-list retries (the velocities once
    // they are there: vel_ready)
    ck(cudaMemcpyAsync(bk, s.x, sizeof(double) * (vel_ready ? 3 : 6) * N, cudaMemcpyDeviceToDevice, f->stream),
       "backup");
    fresh_list(f, W);
    for (int attempt = 0; attempt < 8; ++attempt) {
        ensure_const_table(f, W);
        const bool graphs = !f->timer.on;
        if (graphs) ensure_graphs(f, W, s, dt, conv);
        f->launches += launch_reset_err(f->stream, W.err, 0);
        if (graphs) {
            ck(cudaGraphLaunch(W.gx_eval, f->stream), "GraphLaunch");
            f->launches += W.launches_eval;
            if (vel_ready) { // the initial evaluation needed positions and charges only
                ck(cudaStreamWaitEvent(f->stream, vel_ready, 0), "wait");
                ck(cudaMemcpyAsync(bk + 3 * N, s.vx, sizeof(double) * 3 * N, cudaMemcpyDeviceToDevice, f->stream),
                   "backup");
                vel_ready = nullptr;
            }
            for (int st = 1; st <= steps; ++st) {
                ck(cudaGraphLaunch(st == 1 ? W.gx_step1 : W.gx_step2, f->stream), "GraphLaunch");
                f->launches += W.launches_step;
            }
        } else {
            enqueue_eval(f, W, s, false);
            if (vel_ready) {
                ck(cudaStreamWaitEvent(f->stream, vel_ready, 0), "wait");
                ck(cudaMemcpyAsync(bk + 3 * N, s.vx, sizeof(double) * 3 * N, cudaMemcpyDeviceToDevice, f->stream),
                   "backup");
                vel_ready = nullptr;
            }
            for (int st = 1; st <= steps; ++st) {
                StageScope sc(f, "verlet");
                sc.done(launch_kick_drift(f->stream, s, W.o, dt, conv, st == 1 ? 1 : 2, W.err));
                enqueue_eval(f, W, s, false, false);
            }
        }
        {
            StageScope sc(f, "verlet");
            sc.done(launch_kick(f->stream, s, W.o, dt, conv, W.err));
        }
        ck(cudaGetLastError(), "kernel launch");
        const ErrRec r = read_err(f, W);
        if (r.kind == kOverflowKind || r.kind) {
            ck(cudaMemcpyAsync(s.x, bk, sizeof(double) * 6 * N, cudaMemcpyDeviceToDevice, f->stream),
               "restore");
            ck(cudaStreamSynchronize(f->stream), "sync");
        }
        if (r.kind == kOverflowKind) {
            grow_cap(W, r);
            continue;
        }
        record_counters(f, W, r);
        if (r.kind) return engine_set_error(f, error_from_rec(r));
        return MSMB_OK;
    }
    return engine_set_error(f, Error{MSMB_ERR_INTERNAL, -1, -1, -1, "pair list did not converge"});
}

// ---- host <-> device state ------------------------------------------------------------
static void upload_vec3(msmb_field* f, const double* host, double* x, double* y, double* z,
                        int64_t n, Workspace* W, DBuf& tmp) {
    if (n == 0) return;
    double* stg;
    if (W && W->staging.bytes >= sizeof(double) * 3 * size_t(n))
        stg = W->staging.as<double>();
    else {
        if (tmp.bytes < sizeof(double) * 3 * size_t(n)) ck(tmp.alloc(sizeof(double) * 3 * size_t(n)), "alloc");
        stg = tmp.as<double>();
    }
    ck(cudaMemcpyAsync(stg, host, sizeof(double) * 3 * size_t(n), cudaMemcpyHostToDevice, f->stream), "H2D");
    f->launches += launch_aos_to_soa(f->stream, n, stg, x, y, z);
}

static void download_vec3(msmb_field* f, double* host, const double* x, const double* y,
                          const double* z, int64_t n, Workspace* W, DBuf& tmp) {
    if (n == 0 || !host) return;
    double* stg;
    if (W && W->staging.bytes >= sizeof(double) * 3 * size_t(n))
        stg = W->staging.as<double>();
    else {
        if (tmp.bytes < sizeof(double) * 3 * size_t(n)) ck(tmp.alloc(sizeof(double) * 3 * size_t(n)), "alloc");
        stg = tmp.as<double>();
    }
    f->launches += launch_soa_to_aos(f->stream, n, x, y, z, stg);
    ck(cudaMemcpyAsync(host, stg, sizeof(double) * 3 * size_t(n), cudaMemcpyDeviceToHost, f->stream), "D2H");
}

static int fill_state(msmb_field* f, StateBuf& sb, int64_t n, const double* pos, const double* vel,
                      const double* q, const double* mass, const double* box) {
    if (sb.n != n || !sb.buf.p) ck(sb.alloc(n), "cudaMalloc state");
    for (int ax = 0; ax < 3; ++ax) sb.box[ax] = box[ax];
    DevState s = sb.dev();
    DBuf tmp;
    Workspace* W = (f->ws && f->ws->n == n) ? f->ws.get() : nullptr;
    upload_vec3(f, pos, s.x, s.y, s.z, n, W, tmp);
    if (vel)
        upload_vec3(f, vel, s.vx, s.vy, s.vz, n, W, tmp);
    else if (n)
        ck(cudaMemsetAsync(s.vx, 0, sizeof(double) * 3 * size_t(n), f->stream), "memset");
    if (n) ck(cudaMemcpyAsync(s.q, q, sizeof(double) * size_t(n), cudaMemcpyHostToDevice, f->stream), "H2D q");
    if (n && mass)
        ck(cudaMemcpyAsync(s.m, mass, sizeof(double) * size_t(n), cudaMemcpyHostToDevice, f->stream), "H2D m");
    ck(cudaStreamSynchronize(f->stream), "sync");
    return MSMB_OK;
}

static void copy_outputs(msmb_field* f, int64_t n, double* phi, double* phi_short, double* phi_long,
                         double* force, double* energy) {
    Workspace& W = *f->ws;
    DBuf tmp;
    auto d2h = [&](double* h, const double* d) {
        if (h && n) ck(cudaMemcpyAsync(h, d, sizeof(double) * size_t(n), cudaMemcpyDeviceToHost, f->stream), "D2H");
    };
    d2h(phi, W.o.phi);
    d2h(phi_short, W.o.phis);
    d2h(phi_long, W.o.phil);
    if (force) download_vec3(f, force, W.o.fx, W.o.fy, W.o.fz, n, &W, tmp);
    if (energy) {
        if (n)
            ck(cudaMemcpyAsync(energy, W.o.energy, sizeof(double), cudaMemcpyDeviceToHost, f->stream), "D2H");
        else
            *energy = 0.0;
    }
    ck(cudaStreamSynchronize(f->stream), "sync");
}

__global__ void k_fp64_peak(double* out, int iters, double seed) {
    double a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = seed + threadIdx.x * 1e-9 + k;
    const double m = 0.9999999999, c = 1e-12;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = fma(a[k], m, c);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
    if (s == 1234.5678) out[threadIdx.x] = s;
}

} // namespace msmb

using namespace msmb;

// =======================================================================================
// C ABI
// =======================================================================================
#define GUARD_BEGIN try {
#define GUARD_END(f)                                                                     \
    }                                                                                    \
    catch (const CudaErr& ex) {                                                          \
        Error er;                                                                        \
        er.kind = MSMB_ERR_CUDA;                                                         \
        er.msg = ex.what();                                                              \
        if (f) (f)->last = er;                                                           \
        return MSMB_ERR_CUDA;                                                            \
    }                                                                                    \
    catch (const std::exception& ex) {                                                   \
        Error er;                                                                        \
        er.kind = MSMB_ERR_INTERNAL;                                                     \
        er.msg = ex.what();                                                              \
        if (f) (f)->last = er;                                                           \
        return MSMB_ERR_INTERNAL;                                                        \
    }

static thread_local Error g_create_error;

extern "C" {

int msmb_abi_version(void) { return MSMB_ABI_VERSION; }

int msmb_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

static int field_new(int device, msmb_field** out);

int msmb_create(const msmb_msm_config* cfg, const msmb_units* units, int device, msmb_field** out) {
    *out = nullptr;
    Error e = validate_config(*cfg);
    if (!e.kind) e = validate_units(*units);
    if (e.kind) {
        g_create_error = e;
        return e.kind;
    }
    const int rc = field_new(device, out);
    if (rc) return rc;
    (*out)->cfg = *cfg;
    (*out)->units = *units;
    return MSMB_OK;
}

int msmb_create_cutoff(int kind, const msmb_cutoff_params* params, const msmb_units* units, int device,
                       msmb_field** out) {
    *out = nullptr;
    Error e = validate_cutoff(kind, *params);
    if (!e.kind) e = validate_units(*units);
    if (e.kind) {
        g_create_error = e;
        return e.kind;
    }
    const int rc = field_new(device, out);
    if (rc) return rc;
    msmb_field* f = *out;
    f->kind = kind;
    f->cut = *params;
    f->units = *units;
    f->cfg = msmb_msm_config{params->cutoff, params->cutoff / 4.0, 1, 3, 2}; // binning only
    return MSMB_OK;
}

int msmb_field_kind(const msmb_field* f) { return f ? f->kind : -1; }

int msmb_create_direct(const msmb_units* units, int device, msmb_field** out) {
    *out = nullptr;
    Error e = validate_units(*units);
    if (e.kind) {
        g_create_error = e;
        return e.kind;
    }
    const int rc = field_new(device, out);
    if (rc) return rc;
    (*out)->kind = MSMB_FIELD_DIRECT;
    (*out)->units = *units;
    return MSMB_OK;
}

int msmb_create_overlay(const msmb_field* base, double epsilon, double sigma, msmb_field** out) {
    *out = nullptr;
    if (!base) {
        g_create_error = Error{MSMB_ERR_CONFIG, -1, -1, -1, "overlay needs a base field"};
        return MSMB_ERR_CONFIG;
    }
    const int rc = field_new(base->device, out);
    if (rc) return rc;
    msmb_field* f = *out;
    std::lock_guard<std::recursive_mutex> lk(const_cast<msmb_field*>(base)->mu); // a consistent snapshot
    f->kind = base->kind;
    f->cut = base->cut;
    f->cfg = base->cfg;
    f->units = base->units;
    f->lattice_direct = base->lattice_direct;
    f->pair_skin = base->pair_skin;
    f->rep = base->rep; // nested overlays add their terms (force_field.cpp:45-68)
    f->rep.emplace_back(epsilon, sigma);
    f->rep_on = 1;
    return MSMB_OK;
}

static int field_new(int device, msmb_field** out) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0 || device < 0 || device >= ndev) {
        g_create_error = Error{MSMB_ERR_CUDA, -1, -1, -1, "no usable CUDA device (this library has no CPU fallback)"};
        return MSMB_ERR_CUDA;
    }
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, device);
    if (prop.major < 10) {
        g_create_error = Error{MSMB_ERR_CUDA, -1, -1, -1,
                               std::string("device ") + prop.name + " is not sm_100 (B200); this build targets sm_100a only"};
        return MSMB_ERR_CUDA;
    }
    auto* f = new msmb_field();
    f->device = device;
    cudaSetDevice(device);
    int prio_lo = 0, prio_hi = 0;
    cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
    // side (long-range chain) stream priority relative to the main (pair-sum) stream:
    // high, so the chain's CTAs are dispatched as pair CTAs retire instead of after the
    // pair kernel's last one.  C2-S round 2 with the 4-line FFT tiles: 0.842 ms/step
    // vs 0.849 at equal priority (round 1, 256-thread FFT tiles: equal was best).
    // MSMB_SIDE_PRIO = high | equal | low is the knob.
    int side_prio = prio_hi, main_prio = prio_lo;
    if (const char* e = std::getenv("MSMB_SIDE_PRIO")) {
        if (!strcmp(e, "equal")) side_prio = prio_lo, main_prio = prio_lo;
        if (!strcmp(e, "high")) side_prio = prio_hi, main_prio = prio_lo;
        if (!strcmp(e, "low")) side_prio = prio_lo, main_prio = prio_hi;
    }
    // the anterpolation's stream: the chain's priority (MSMB_ANTERP_PRIO=main: the main
    // stream's; measured equal on C2-S, 0.836 ms/step: at main priority the
    // anterpolation waits behind the pair kernel and the chain ends after it)
    int anterp_prio = side_prio;
    if (const char* e = std::getenv("MSMB_ANTERP_PRIO"))
        if (!strcmp(e, "main")) anterp_prio = main_prio;
    if (cudaStreamCreateWithPriority(&f->stream, cudaStreamNonBlocking, main_prio) != cudaSuccess ||
        cudaStreamCreateWithPriority(&f->side, cudaStreamNonBlocking, side_prio) != cudaSuccess ||
        cudaStreamCreateWithPriority(&f->side_a, cudaStreamNonBlocking, anterp_prio) != cudaSuccess ||
        cudaStreamCreateWithPriority(&f->side_r, cudaStreamNonBlocking, main_prio) != cudaSuccess ||
        cudaStreamCreateWithFlags(&f->copy, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&f->vel_ev, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&f->sort_ev, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&f->disp_ev, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&f->reb_ev, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&f->fork_ev, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&f->join_ev, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&f->mid_ev, cudaEventDisableTiming) != cudaSuccess) {
        if (f->stream) cudaStreamDestroy(f->stream);
        if (f->side) cudaStreamDestroy(f->side);
        if (f->side_a) cudaStreamDestroy(f->side_a);
        if (f->side_r) cudaStreamDestroy(f->side_r);
        if (f->copy) cudaStreamDestroy(f->copy);
        if (f->vel_ev) cudaEventDestroy(f->vel_ev);
        if (f->sort_ev) cudaEventDestroy(f->sort_ev);
        if (f->disp_ev) cudaEventDestroy(f->disp_ev);
        if (f->reb_ev) cudaEventDestroy(f->reb_ev);
        if (f->fork_ev) cudaEventDestroy(f->fork_ev);
        if (f->join_ev) cudaEventDestroy(f->join_ev);
        if (f->mid_ev) cudaEventDestroy(f->mid_ev);
        delete f;
        g_create_error = Error{MSMB_ERR_CUDA, -1, -1, -1, "cudaStreamCreate failed"};
        return MSMB_ERR_CUDA;
    }
    *out = f;
    return MSMB_OK;
}

static void field_free(msmb_field* f) {
    cudaSetDevice(f->device);
    cudaStreamSynchronize(f->stream);
    f->ws.reset();
    f->scratch.buf.reset();
    cudaStreamDestroy(f->stream);
    cudaStreamDestroy(f->side);
    cudaStreamDestroy(f->side_a);
    cudaStreamDestroy(f->side_r);
    cudaStreamDestroy(f->copy);
    cudaEventDestroy(f->vel_ev);
    cudaEventDestroy(f->sort_ev);
    cudaEventDestroy(f->disp_ev);
    cudaEventDestroy(f->reb_ev);
    cudaEventDestroy(f->fork_ev);
    cudaEventDestroy(f->join_ev);
    cudaEventDestroy(f->mid_ev);
    delete f;
}

// A field outlives every msmb_system created from it: destroying a field that
// still has systems only marks it; the last msmb_system_destroy frees it.
void msmb_destroy(msmb_field* f) {
    if (!f) return;
    {
        std::lock_guard<std::recursive_mutex> lk(f->mu);
        if (f->refs > 0) {
            f->destroy_pending = true;
            return;
        }
    }
    field_free(f);
}

int msmb_last_error(const msmb_field* f, int* kind, int64_t* idx_i, int64_t* idx_j, int* step,
                    char* msg, int cap) {
    const Error& e = f ? f->last : g_create_error;
    if (kind) *kind = e.kind;
    if (idx_i) *idx_i = e.i;
    if (idx_j) *idx_j = e.j;
    if (step) *step = e.step;
    if (msg && cap > 0) {
        strncpy(msg, e.msg.c_str(), size_t(cap - 1));
        msg[cap - 1] = 0;
    }
    return e.kind;
}

double msmb_cost_flops_per_step(const msmb_field* f, int64_t n) {
    const double rep = 30.0 * double(n) * double(f->rep.size()); // PairRepulsionOverlay, force_field.cpp:70-72
    if (f->kind == MSMB_FIELD_DIRECT) return 20.0 * double(n) * double(n) + rep; // force_field.cpp:17-19
    if (f->kind != MSMB_FIELD_MSM) { // force_field.cpp:25-35
        const double fpp = f->cut.flops_per_particle > 0.0 ? f->cut.flops_per_particle
                                                           : (f->kind == MSMB_FIELD_WOLF ? 350.0 : 301.0);
        return fpp * double(n) + rep;
    }
    return host_flops_simplified(f->cfg.cutoff_a, f->cfg.spacing_h, double(n)) + rep;
}

int msmb_evaluate(msmb_field* f, int64_t n, const double* pos_xyz, const double* q,
                  const double box[3], double* phi, double* phi_short, double* phi_long,
                  double* force_xyz, double* energy) {
    std::lock_guard<std::recursive_mutex> lk(f->mu);
    GUARD_BEGIN
    f->last = Error{};
    cudaSetDevice(f->device);
    Error e = f->kind == MSMB_FIELD_MSM ? validate_config(f->cfg) : Error{};
    if (!e.kind) e = validate_units(f->units);
    if (e.kind) return engine_set_error(f, e);
    e = ensure_workspace(f, n, box);
    if (e.kind) return engine_set_error(f, e);
    fill_state(f, f->scratch, n, pos_xyz, nullptr, q, nullptr, box);
    const int rc = eval_device(f, f->scratch, true);
    if (rc) return rc;
    copy_outputs(f, n, phi, phi_short, phi_long, force_xyz, energy);
    return MSMB_OK;
    GUARD_END(f)
}

// energy_report (src/integrate.cpp:47-55): kinetic energy on the device, then the
// field's evaluation.  out = [kinetic, potential, total].
int msmb_energy_report(msmb_field* f, int64_t n, const double* pos_xyz, const double* vel_xyz, const double* q,
                       const double* mass, const double box[3], const msmb_units* units, double* out) {
    std::lock_guard<std::recursive_mutex> lk(f->mu);
    GUARD_BEGIN
    f->last = Error{};
    cudaSetDevice(f->device);
    const msmb_units u = units ? *units : f->units;
    Error e = validate_units(u); // energy_report validates its units first
    if (!e.kind && f->kind == MSMB_FIELD_MSM) e = validate_config(f->cfg);
    if (!e.kind) e = validate_units(f->units);
    if (e.kind) return engine_set_error(f, e);
    e = ensure_workspace(f, n, box);
    if (e.kind) return engine_set_error(f, e);
    fill_state(f, f->scratch, n, pos_xyz, vel_xyz, q, mass, box);
    Workspace& W = *f->ws;
    double ke = 0.0;
    if (n > 0) {
        f->launches += launch_reset_err(f->stream, W.err, 0);
        f->launches += launch_kinetic(f->stream, f->scratch.dev(), W.o.e, W.o.partial, 1.0, W.o.energy, W.err);
        ck(cudaMemcpyAsync(&ke, W.o.energy, sizeof(double), cudaMemcpyDeviceToHost, f->stream), "D2H");
        ck(cudaStreamSynchronize(f->stream), "sync");
    }
    const int rc = eval_device(f, f->scratch, true);
    if (rc) return rc;
    double pot = 0.0;
    copy_outputs(f, n, nullptr, nullptr, nullptr, nullptr, &pot);
    out[0] = ke / u.energy_to_native;
    out[1] = pot;
    out[2] = out[0] + out[1];
    return MSMB_OK;
    GUARD_END(f)
}

int msmb_propagate_ex(msmb_field* f, int64_t n, double* pos_xyz, double* vel_xyz, const double* q,
                      const double* mass, const double box[3], double dt, int steps,
                      const msmb_units* units) {
    std::lock_guard<std::recursive_mutex> lk(f->mu);
    GUARD_BEGIN
    f->last = Error{};
    cudaSetDevice(f->device);
    // PropagatorSpec::validate (src/integrate.cpp:7-11), then UnitsConfig::validate
    if (!(dt > 0.0)) return engine_set_error(f, Error{MSMB_ERR_CONFIG, -1, -1, -1, "dt must be > 0"});
    if (steps < 1)
        return engine_set_error(f, Error{MSMB_ERR_CONFIG, -1, -1, -1, "steps_per_slice must be >= 1"});
    const msmb_units u = units ? *units : f->units;
    Error e = validate_units(u);
    if (e.kind) return engine_set_error(f, e);
    e = ensure_workspace(f, n, box);
    if (e.kind) return engine_set_error(f, e);
    // Positions and charges go up on the engine's stream; velocities and masses on the copy stream,
    // beside the initial evaluation (which needs neither).  The final state comes back through the
    // two staging buffers with one synchronisation.
    StateBuf& sb = f->scratch;
    if (sb.n != n || !sb.buf.p) ck(sb.alloc(n), "cudaMalloc state");
    for (int ax = 0; ax < 3; ++ax) sb.box[ax] = box[ax];
    DevState s = sb.dev();
    Workspace& W = *f->ws;
    const size_t N3 = sizeof(double) * 3 * size_t(n);
    cudaEvent_t vel_ready = nullptr;
    if (n > 0) {
        double* stg = W.staging.as<double>();
        double* stg2 = W.staging2.as<double>();
        ck(cudaMemcpyAsync(stg, pos_xyz, N3, cudaMemcpyHostToDevice, f->stream), "H2D");
        f->launches += launch_aos_to_soa(f->stream, n, stg, s.x, s.y, s.z);
        ck(cudaMemcpyAsync(s.q, q, sizeof(double) * size_t(n), cudaMemcpyHostToDevice, f->stream), "H2D q");
        if (vel_xyz) {
            ck(cudaMemcpyAsync(stg2, vel_xyz, N3, cudaMemcpyHostToDevice, f->copy), "H2D");
            f->launches += launch_aos_to_soa(f->copy, n, stg2, s.vx, s.vy, s.vz);
        } else {
            ck(cudaMemsetAsync(s.vx, 0, N3, f->copy), "memset");
        }
        if (mass) ck(cudaMemcpyAsync(s.m, mass, sizeof(double) * size_t(n), cudaMemcpyHostToDevice, f->copy), "H2D m");
        ck(cudaEventRecord(f->vel_ev, f->copy), "record");
        vel_ready = f->vel_ev;
    }
    int rc;
    try {
        rc = engine_propagate(f, sb, dt, steps, u.energy_to_native, vel_ready);
    } catch (...) {
        cudaStreamSynchronize(f->copy); // the host buffers must outlive the copies
        throw;
    }
    ck(cudaStreamSynchronize(f->copy), "sync");
    if (rc) return rc;
    if (n > 0) {
        double* stg = W.staging.as<double>();
        double* stg2 = W.staging2.as<double>();
        f->launches += launch_soa_to_aos(f->stream, n, s.x, s.y, s.z, stg);
        ck(cudaMemcpyAsync(pos_xyz, stg, N3, cudaMemcpyDeviceToHost, f->stream), "D2H");
        if (vel_xyz) {
            f->launches += launch_soa_to_aos(f->stream, n, s.vx, s.vy, s.vz, stg2);
            ck(cudaMemcpyAsync(vel_xyz, stg2, N3, cudaMemcpyDeviceToHost, f->stream), "D2H");
        }
        ck(cudaStreamSynchronize(f->stream), "sync");
    }
    return MSMB_OK;
    GUARD_END(f)
}

int msmb_propagate(msmb_field* f, int64_t n, double* pos_xyz, double* vel_xyz, const double* q,
                   const double* mass, const double box[3], double dt, int steps) {
    return msmb_propagate_ex(f, n, pos_xyz, vel_xyz, q, mass, box, dt, steps, nullptr);
}

void* msmb_host_alloc(int64_t bytes) {
    void* p = nullptr;
    if (cudaHostAlloc(&p, size_t(bytes > 0 ? bytes : 8), cudaHostAllocDefault) != cudaSuccess) return nullptr;
    return p;
}

void msmb_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

int msmb_system_create(msmb_field* f, int64_t n, const double* pos_xyz, const double* vel_xyz,
                       const double* q, const double* mass, const double box[3], msmb_system** out) {
    std::lock_guard<std::recursive_mutex> lk(f->mu);
    *out = nullptr;
    GUARD_BEGIN
    cudaSetDevice(f->device);
    auto* s = new msmb_system();
    s->f = f;
    try {
        fill_state(f, s->st, n, pos_xyz, vel_xyz, q, mass, box);
    } catch (...) {
        delete s;
        throw;
    }
    f->refs++;
    *out = s;
    return MSMB_OK;
    GUARD_END(f)
}

void msmb_system_destroy(msmb_system* s) {
    if (!s) return;
    msmb_field* f = s->f;
    bool free_field = false;
    {
        std::lock_guard<std::recursive_mutex> lk(f->mu);
        cudaSetDevice(f->device);
        cudaStreamSynchronize(f->stream);
        if (f->ws && f->ws->graph_key == s->st.dev().x) destroy_graphs(*f->ws);
        delete s;
        f->refs--;
        free_field = f->destroy_pending && f->refs == 0;
    }
    if (free_field) field_free(f);
}

int msmb_system_upload(msmb_system* s, const double* pos_xyz, const double* vel_xyz) {
    msmb_field* f = s->f;
    std::lock_guard<std::recursive_mutex> lk(f->mu);
    GUARD_BEGIN
    cudaSetDevice(f->device);
    DevState d = s->st.dev();
    DBuf tmp;
    Workspace* W = (f->ws && f->ws->n == s->st.n) ? f->ws.get() : nullptr;
    if (pos_xyz) upload_vec3(f, pos_xyz, d.x, d.y, d.z, s->st.n, W, tmp);
    if (vel_xyz) upload_vec3(f, vel_xyz, d.vx, d.vy, d.vz, s->st.n, W, tmp);
    ck(cudaStreamSynchronize(f->stream), "sync");
    return MSMB_OK;
    GUARD_END(f)
}

int msmb_system_download(const msmb_system* s, double* pos_xyz, double* vel_xyz) {
    msmb_field* f = s->f;
    std::lock_guard<std::recursive_mutex> lk(f->mu);
    GUARD_BEGIN
    cudaSetDevice(f->device);
    DevState d = s->st.dev();
    DBuf tmp;
    Workspace* W = (f->ws && f->ws->n == s->st.n) ? f->ws.get() : nullptr;
    download_vec3(f, pos_xyz, d.x, d.y, d.z, s->st.n, W, tmp);
    ck(cudaStreamSynchronize(f->stream), "sync");
    download_vec3(f, vel_xyz, d.vx, d.vy, d.vz, s->st.n, W, tmp);
    ck(cudaStreamSynchronize(f->stream), "sync");
    return MSMB_OK;
    GUARD_END(f)
}

int msmb_system_copy(msmb_system* dst, const msmb_system* src) {
    msmb_field* f = dst->f;
    std::lock_guard<std::recursive_mutex> lk(f->mu);
    GUARD_BEGIN
    cudaSetDevice(f->device);
    if (dst->st.n != src->st.n) ck(dst->st.alloc(src->st.n), "alloc");
    for (int ax = 0; ax < 3; ++ax) dst->st.box[ax] = src->st.box[ax];
    ck(cudaMemcpyAsync(dst->st.buf.p, src->st.buf.p, src->st.buf.bytes, cudaMemcpyDeviceToDevice,
                       f->stream),
       "copy");
    ck(cudaStreamSynchronize(f->stream), "sync");
    return MSMB_OK;
    GUARD_END(f)
}

int msmb_system_propagate(msmb_field* f, msmb_system* s, double dt, int steps) {
    std::lock_guard<std::recursive_mutex> lk(f->mu);
    GUARD_BEGIN
    f->last = Error{};
    cudaSetDevice(f->device);
    return engine_propagate(f, s->st, dt, steps, f->units.energy_to_native);
    GUARD_END(f)
}

int msmb_system_propagate_ex(msmb_field* f, msmb_system* s, double dt, int steps, const msmb_units* units) {
    if (!units) return msmb_system_propagate(f, s, dt, steps);
    std::lock_guard<std::recursive_mutex> lk(f->mu);
    GUARD_BEGIN
    f->last = Error{};
    Error e = validate_units(*units);
    if (e.kind) return engine_set_error(f, e);
    cudaSetDevice(f->device);
    return engine_propagate(f, s->st, dt, steps, units->energy_to_native);
    GUARD_END(f)
}

int msmb_system_evaluate(msmb_field* f, msmb_system* s, double* phi, double* phi_short,
                         double* phi_long, double* force_xyz, double* energy) {
    std::lock_guard<std::recursive_mutex> lk(f->mu);
    GUARD_BEGIN
    f->last = Error{};
    cudaSetDevice(f->device);
    const int rc = eval_device(f, s->st, true);
    if (rc) return rc;
    copy_outputs(f, s->st.n, phi, phi_short, phi_long, force_xyz, energy);
    return MSMB_OK;
    GUARD_END(f)
}

int msmb_bench_propagate(msmb_field* f, msmb_system* sys, double dt, int steps, int flush_l2,
                         double* step_ms, double* stage_ms, const char** stage_names,
                         int64_t* launches) {
    std::lock_guard<std::recursive_mutex> lk(f->mu);
    GUARD_BEGIN
    f->last = Error{};
    cudaSetDevice(f->device);
    if (!(dt > 0.0)) return engine_set_error(f, Error{MSMB_ERR_CONFIG, -1, -1, -1, "dt must be > 0"});
    if (steps < 1)
        return engine_set_error(f, Error{MSMB_ERR_CONFIG, -1, -1, -1, "steps_per_slice must be >= 1"});
    StateBuf& sb = sys->st;
    Error e = ensure_workspace(f, sb.n, sb.box);
    if (e.kind) return engine_set_error(f, e);
    Workspace& W = *f->ws;
    DevState s = sb.dev();
    const size_t N = size_t(sb.n > 0 ? sb.n : 1);
    const double conv = f->units.energy_to_native;
    const size_t flush_bytes = size_t(256) << 20; // 2x the 126 MB L2
    if (flush_l2 && W.flush.bytes < flush_bytes) ck(W.flush.alloc(flush_bytes), "cudaMalloc flush");
    if (f->timer.on) f->timer.on = false;
    ensure_graphs(f, W, s, dt, conv);
    double* bk = W.backup.as<double>();
    ck(cudaMemcpyAsync(bk, s.x, sizeof(double) * 6 * N, cudaMemcpyDeviceToDevice, f->stream), "backup");
    cudaEvent_t ea, eb;
    ck(cudaEventCreate(&ea), "event");
    ck(cudaEventCreate(&eb), "event");
    std::vector<double> acc(kNumStages, 0.0);
    const int64_t l0 = f->launches;
    int flush_k = 0;
    auto timed = [&](auto&& launch, bool stages) -> double {
        if (flush_l2) ck(cudaMemsetAsync(W.flush.p, (flush_k++) & 0xff, W.flush.bytes, f->stream), "flush");
        ck(cudaEventRecord(ea, f->stream), "record");
        launch();
        ck(cudaEventRecord(eb, f->stream), "record");
        ck(cudaEventSynchronize(eb), "sync");
        float ms = 0.f;
        ck(cudaEventElapsedTime(&ms, ea, eb), "elapsed");
        (void)stages;
        return double(ms);
    };
    ensure_const_table(f, W);
    f->launches += launch_reset_err(f->stream, W.err, 0);
    step_ms[0] = timed([&] {
        ck(cudaGraphLaunch(W.gx_eval, f->stream), "GraphLaunch");
        f->launches += W.launches_eval;
    }, true);
    double stamp_acc[16] = {0};
    for (int st = 1; st <= steps; ++st) {
        step_ms[st] = timed([&] {
            const auto c0 = std::chrono::steady_clock::now();
            ck(cudaGraphLaunch(st == 1 ? W.gx_step1 : W.gx_step2, f->stream), "GraphLaunch");
            stamp_acc[13] += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - c0).count();
            f->launches += W.launches_step;
        }, true);
        if (g_exp_stamps) {
            unsigned long long h[16];
            read_stamps(h);
            for (int k = 1; k <= 10; ++k) stamp_acc[k] += double(h[k] - h[0]) * 1e-3;
            if (st > 1) stamp_acc[11] += double(h[0] - h[11]) * 1e-3, stamp_acc[12] += step_ms[st] * 1e3 - double(h[6] - h[11]) * 1e-3;
        }
    }
    if (g_exp_stamps && steps > 0)
        fprintf(stderr, "timeline (us from evaluation start): sort_end %.1f chain_start %.1f chain_end %.1f clusters_end %.1f pairs_end %.1f eval_end %.1f\n",
                stamp_acc[1] / steps, stamp_acc[2] / steps, stamp_acc[3] / steps, stamp_acc[4] / steps, stamp_acc[5] / steps, stamp_acc[6] / steps);
    if (g_exp_stamps && steps > 1)
        fprintf(stderr, "graph: first stamp -> evaluation start (kick/drift) %.1f us; step event time minus first..last stamp %.1f us; cudaGraphLaunch host time %.1f us\n",
                stamp_acc[11] / (steps - 1), stamp_acc[12] / (steps - 1), stamp_acc[13] / steps);
    if (g_exp_stamps && steps > 0)
        fprintf(stderr, "chain: anterp_end %.1f restrict_end %.1f lattice_end %.1f top_end %.1f\n", stamp_acc[7] / steps,
                stamp_acc[8] / steps, stamp_acc[9] / steps, stamp_acc[10] / steps);
    step_ms[steps + 1] = timed([&] { f->launches += launch_kick(f->stream, s, W.o, dt, conv, W.err); }, false);
    cudaEventDestroy(ea);
    cudaEventDestroy(eb);
    const ErrRec r = read_err(f, W);
    if (launches) *launches = f->launches - l0;
    for (int i = 0; i < kBenchStages; ++i) { // the ABI's 11 (msmb.h); "overlay" is reported by msmb_stage_times
        if (stage_ms) stage_ms[i] = acc[i];
        if (stage_names) stage_names[i] = kStages[i];
    }
    if (r.kind) {
        ck(cudaMemcpyAsync(s.x, bk, sizeof(double) * 6 * N, cudaMemcpyDeviceToDevice, f->stream), "restore");
        ck(cudaStreamSynchronize(f->stream), "sync");
        if (r.kind == kOverflowKind) {
            grow_cap(W, r);
            return msmb_bench_propagate(f, sys, dt, steps, flush_l2, step_ms, stage_ms, stage_names, launches);
        }
        return engine_set_error(f, error_from_rec(r));
    }
    record_counters(f, W, r);
    return MSMB_OK;
    GUARD_END(f)
}

int msmb_measure_fp64_peak(int device, double seconds, double* tflops) {
    cudaSetDevice(device);
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return MSMB_ERR_CUDA;
    const int blocks = prop.multiProcessorCount * 8, threads = 256, iters = 4096;
    double* out = nullptr;
    if (cudaMalloc(&out, sizeof(double) * threads) != cudaSuccess) return MSMB_ERR_CUDA;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_fp64_peak<<<blocks, threads>>>(out, iters, 1.0); // warm-up
    cudaDeviceSynchronize();
    double best = 0.0, elapsed = 0.0;
    int reps = 0;
    while (elapsed < seconds * 1e3 || reps < 3) {
        cudaEventRecord(a);
        for (int k = 0; k < 8; ++k) k_fp64_peak<<<blocks, threads>>>(out, iters, 1.0 + k);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        elapsed += ms;
        ++reps;
        const double fl = 8.0 * 2.0 * 8.0 * double(iters) * blocks * threads; // 8 launches, FMA = 2
        best = std::max(best, fl / (ms * 1e-3) / 1e12);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(out);
    *tflops = best;
    return cudaGetLastError() == cudaSuccess ? MSMB_OK : MSMB_ERR_CUDA;
}

int msmb_set_stage_timing(msmb_field* f, int enable) {
    std::lock_guard<std::recursive_mutex> lk(f->mu);
    f->timer.on = enable != 0;
    return MSMB_OK;
}

int msmb_stage_times(msmb_field* f, double* ms, int64_t* launches, const char** names, int cap) {
    std::lock_guard<std::recursive_mutex> lk(f->mu);
    const int n = std::min<int>(cap, int(f->timer.names.size()));
    for (int i = 0; i < n; ++i) {
        if (ms) ms[i] = f->timer.ms[i];
        if (launches) launches[i] = f->timer.launches[i];
        if (names) names[i] = f->timer.names[i].c_str();
    }
    return n;
}

void msmb_reset_stage_times(msmb_field* f) {
    std::lock_guard<std::recursive_mutex> lk(f->mu);
    for (auto& m : f->timer.ms) m = 0.0;
    for (auto& l : f->timer.launches) l = 0;
}

int msmb_work_counters(msmb_field* f, int64_t* out, int cap) {
    const int n = std::min(cap, 8);
    for (int i = 0; i < n; ++i) out[i] = f->counters[i];
    return n;
}

int64_t msmb_kernel_launches(const msmb_field* f) { return f->launches; }

int msmb_grid_geometry(const msmb_msm_config* cfg, const double box[3], int* dims, double* spacing,
                       double* origin) {
    msmb_units u{332.0636, 4.184e-4};
    Geometry g;
    Error e = build_geometry(*cfg, u, box, 1, g);
    if (e.kind) {
        g_create_error = e;
        return e.kind;
    }
    for (int k = 0; k < g.levels; ++k) {
        for (int ax = 0; ax < 3; ++ax) {
            dims[3 * k + ax] = g.lv[k].dims[ax];
            origin[3 * k + ax] = g.lv[k].origin[ax];
        }
        spacing[k] = g.lv[k].spacing;
    }
    return MSMB_OK;
}

static int msm_only(msmb_field* f) {
    return engine_set_error(f, Error{MSMB_ERR_CONFIG, -1, -1, -1, "this entry point needs an MSM field"});
}

int msmb_debug_levels(msmb_field* f, double* level_charge, double* level_potential) {
    std::lock_guard<std::recursive_mutex> lk(f->mu);
    if (f->kind != MSMB_FIELD_MSM) return msm_only(f);
    GUARD_BEGIN
    if (!f->ws) return MSMB_ERR_INTERNAL;
    cudaSetDevice(f->device);
    const size_t bytes = sizeof(double) * f->ws->g.lattice_total;
    ck(cudaStreamSynchronize(f->stream), "sync");
    if (level_charge) ck(cudaMemcpy(level_charge, f->ws->L.charge, bytes, cudaMemcpyDeviceToHost), "D2H");
    if (level_potential) ck(cudaMemcpy(level_potential, f->ws->L.pot, bytes, cudaMemcpyDeviceToHost), "D2H");
    return MSMB_OK;
    GUARD_END(f)
}

int msmb_debug_cells(msmb_field* f, int64_t n, const double* pos_xyz, const double box[3],
                     int32_t* cells_xyz, int32_t* covered) {
    std::lock_guard<std::recursive_mutex> lk(f->mu);
    GUARD_BEGIN
    cudaSetDevice(f->device);
    Error e = ensure_workspace(f, n, box);
    if (e.kind) return engine_set_error(f, e);
    std::vector<double> q(size_t(n), 0.0);
    fill_state(f, f->scratch, n, pos_xyz, nullptr, q.data(), nullptr, box);
    DBuf dc, dv;
    ck(dc.alloc(sizeof(int) * 3 * size_t(n > 0 ? n : 1)), "alloc");
    ck(dv.alloc(sizeof(int) * size_t(n > 0 ? n : 1)), "alloc");
    f->launches += launch_debug_cells(f->stream, f->ws->g, f->scratch.dev(), dc.as<int>(), dv.as<int>());
    ck(cudaStreamSynchronize(f->stream), "sync");
    if (n) {
        ck(cudaMemcpy(cells_xyz, dc.p, sizeof(int) * 3 * size_t(n), cudaMemcpyDeviceToHost), "D2H");
        ck(cudaMemcpy(covered, dv.p, sizeof(int) * size_t(n), cudaMemcpyDeviceToHost), "D2H");
    }
    return MSMB_OK;
    GUARD_END(f)
}

int msmb_debug_stage(msmb_field* f, int stage, int k, const double box[3], const double* in,
                     double* out, int64_t n, const double* pos_xyz) {
    std::lock_guard<std::recursive_mutex> lk(f->mu);
    if (f->kind != MSMB_FIELD_MSM) return msm_only(f);
    GUARD_BEGIN
    cudaSetDevice(f->device);
    Error e = ensure_workspace(f, n, box);
    if (e.kind) return engine_set_error(f, e);
    Workspace& W = *f->ws;
    const Geometry& g = W.g;
    ensure_const_table(f, W);
    f->launches += launch_reset_err(f->stream, W.err, 0);
    auto up = [&](double* d, const double* h, size_t cnt) { // stream-ordered before the stage kernel
        ck(cudaMemcpyAsync(d, h, sizeof(double) * cnt, cudaMemcpyHostToDevice, f->stream), "H2D");
        ck(cudaStreamSynchronize(f->stream), "sync");
    };
    auto down = [&](double* h, const double* d, size_t cnt) {
        ck(cudaStreamSynchronize(f->stream), "sync");
        ck(cudaMemcpy(h, d, sizeof(double) * cnt, cudaMemcpyDeviceToHost), "D2H");
    };
    switch (stage) {
        case 0: // restrict k -> k+1
            if (k < 0 || k + 1 >= g.levels) return MSMB_ERR_HIERARCHY;
            up(W.L.charge + g.lv[k].offset, in, g.lv[k].size);
            f->launches += launch_restrict(f->stream, g, k, W.L, W.err);
            down(out, W.L.charge + g.lv[k + 1].offset, g.lv[k + 1].size);
            break;
        case 1: { // lattice cutoff on level k (runs all non-top levels; reads level k only)
            if (k < 0 || k + 1 >= g.levels) return MSMB_ERR_HIERARCHY;
            up(W.L.charge + g.lv[k].offset, in, g.lv[k].size);
            f->launches += W.lattice_fft ? launch_lattice_fft(f->stream, W.fft, W.err)
                                         : launch_lattice(f->stream, g, W.L, W.err, W.whole);
            down(out, W.L.pot + g.lv[k].offset, g.lv[k].size);
            break;
        }
        case 2: { // top level
            const int t = g.levels - 1;
            up(W.L.charge + g.lv[t].offset, in, g.lv[t].size);
            f->launches += W.fft_top.n ? launch_lattice_fft(f->stream, W.fft_top, W.err)
                                       : launch_top(f->stream, g, W.L, W.err, true);
            down(out, W.L.pot + g.lv[t].offset, g.lv[t].size);
            break;
        }
        case 3: // prolongate k+1 -> k; `in` = coarse potential, `out` = fine potential (in/out)
            if (k < 0 || k + 1 >= g.levels) return MSMB_ERR_HIERARCHY;
            up(W.L.pot + g.lv[k + 1].offset, in, g.lv[k + 1].size);
            up(W.L.pot + g.lv[k].offset, out, g.lv[k].size);
            f->launches += launch_prolong(f->stream, g, k, W.L, W.err);
            down(out, W.L.pot + g.lv[k].offset, g.lv[k].size);
            break;
        case 4: { // interpolate level-0 potential at particles
            std::vector<double> q(size_t(n), 0.0);
            fill_state(f, f->scratch, n, pos_xyz, nullptr, q.data(), nullptr, box);
            up(W.L.pot + g.lv[0].offset, in, g.lv[0].size);
            f->launches += launch_debug_interp(f->stream, g, f->scratch.dev(), W.L.pot + g.lv[0].offset, W.o.phil);
            down(out, W.o.phil, size_t(n));
            break;
        }
        // ---- the production kernels of an evaluation (tolerance tests) ----
        case 5: // restriction chain: in = level-0 charges, out = every level's charges
            up(W.L.charge + g.lv[0].offset, in, g.lv[0].size);
            f->launches += launch_restrict_all(f->stream, g, W.L, W.err);
            down(out, W.L.charge, g.lattice_total);
            break;
        case 6: { // top level as an evaluation runs it (warp kernel or FFT job)
            const int t = g.levels - 1;
            up(W.L.charge + g.lv[t].offset, in, g.lv[t].size);
            f->launches += W.fft_top.n ? launch_lattice_fft(f->stream, W.fft_top, W.err)
                                       : launch_top(f->stream, g, W.L, W.err, false);
            down(out, W.L.pot + g.lv[t].offset, g.lv[t].size);
            break;
        }
        case 7: // prolongation chain: in = every level's potential before it, out = after
            up(W.L.pot, in, g.lattice_total);
            f->launches += launch_prolong_all(f->stream, g, W.L, W.err);
            down(out, W.L.pot, g.lattice_total);
            break;
        default:
            return MSMB_ERR_CONFIG;
    }
    ck(cudaGetLastError(), "launch");
    return MSMB_OK;
    GUARD_END(f)
}

// The production binning kernel (k_bin, the one every evaluation runs): the level-0
// cell triple of every particle, decoded from its sorted-cell key; covered = 0 for a
// particle outside grid coverage (key -1).
int msmb_debug_bin_keys(msmb_field* f, int64_t n, const double* pos_xyz, const double box[3],
                        int32_t* cells_xyz, int32_t* covered) {
    std::lock_guard<std::recursive_mutex> lk(f->mu);
    if (f->kind != MSMB_FIELD_MSM) return msm_only(f);
    GUARD_BEGIN
    cudaSetDevice(f->device);
    Error e = ensure_workspace(f, n, box);
    if (e.kind) return engine_set_error(f, e);
    Workspace& W = *f->ws;
    const Geometry& g = W.g;
    std::vector<double> q(size_t(n), 0.0);
    fill_state(f, f->scratch, n, pos_xyz, nullptr, q.data(), nullptr, box);
    f->launches += launch_reset_err(f->stream, W.err, 0);
    f->launches += launch_bin(f->stream, g, f->scratch.dev(), W.a, W.c, W.err);
    std::vector<int> key(size_t(n > 0 ? n : 1));
    ck(cudaStreamSynchronize(f->stream), "sync");
    if (n) ck(cudaMemcpy(key.data(), W.a.key, sizeof(int) * size_t(n), cudaMemcpyDeviceToHost), "D2H");
    const int d2 = g.lv[0].dims[2], cw = g.cw, ncy = g.ncy;
    for (int64_t i = 0; i < n; ++i) {
        int k = key[size_t(i)];
        covered[i] = k >= 0;
        if (k < 0) {
            cells_xyz[3 * i] = cells_xyz[3 * i + 1] = cells_xyz[3 * i + 2] = 0;
            continue;
        }
        const int cyr = k % cw;
        k /= cw;
        const int cxr = k % cw;
        k /= cw;
        const int cz = k % d2;
        const int col = k / d2;
        cells_xyz[3 * i] = (col / ncy) * cw + cxr;
        cells_xyz[3 * i + 1] = (col % ncy) * cw + cyr;
        cells_xyz[3 * i + 2] = cz;
    }
    return MSMB_OK;
    GUARD_END(f)
}

} // extern "C"
