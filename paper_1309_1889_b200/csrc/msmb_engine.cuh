// Host-side engine objects shared by msmb_engine.cu and msmb_parareal.cu.
#pragma once
#include <cuda_runtime.h>

#include <memory>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "msmb_kernels.cuh"

namespace msmb {

// Several host threads may drive fields of one process (the parareal executor's fine
// replicas, a caller sharing fields between threads).  A thread that captures a CUDA
// graph must not see another thread allocate, free or synchronize the device in the
// middle of its capture (the capture is invalidated), so graph capture and every
// device allocation / free / device-wide synchronization take this lock.
inline std::recursive_mutex& device_mutex() {
    static std::recursive_mutex m;
    return m;
}

// RAII device buffer
struct DBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() { reset(); }
    void reset() {
        if (p) {
            std::lock_guard<std::recursive_mutex> lk(device_mutex());
            cudaFree(p);
        }
        p = nullptr;
        bytes = 0;
    }
    cudaError_t alloc(size_t b) {
        std::lock_guard<std::recursive_mutex> lk(device_mutex());
        reset();
        if (b == 0) b = 8;
        bytes = b;
        return cudaMalloc(&p, b);
    }
    template <class T>
    T* as() const { return static_cast<T*>(p); }
};

// A device-resident particle system (SoA)
struct StateBuf {
    int64_t n = 0;
    DBuf buf; // 8 arrays of n doubles: x y z vx vy vz q m
    double box[3] = {0, 0, 0};
    cudaError_t alloc(int64_t nn) {
        n = nn;
        return buf.alloc(sizeof(double) * 8 * size_t(nn > 0 ? nn : 1));
    }
    DevState dev() const {
        DevState s;
        s.n = n;
        double* b = buf.as<double>();
        const size_t N = size_t(n > 0 ? n : 1);
        s.x = b;
        s.y = b + N;
        s.z = b + 2 * N;
        s.vx = b + 3 * N;
        s.vy = b + 4 * N;
        s.vz = b + 5 * N;
        s.q = b + 6 * N;
        s.m = b + 7 * N;
        return s;
    }
};

struct Workspace {
    Geometry g;
    int64_t n = 0;
    int64_t maxclu = 0;
    int cap = 0;
    DevAtoms a{};
    DevCells c{};
    DevLevels L{};
    DevOut o{};
    std::vector<std::unique_ptr<DBuf>> bufs; // owns everything above
    DBuf plist_buf;
    DBuf pmask_buf;
    DBuf backup;   // 6n doubles: initial x,y,z,vx,vy,vz of a propagate call
    DBuf staging;  // 3n doubles: AoS transfers
    DBuf staging2; // 3n doubles: the velocities' AoS transfers of msmb_propagate (copy stream)
    ErrRec* err = nullptr;
    ErrRec* err_host = nullptr; // pinned
    // graph cache
    cudaGraphExec_t gx_eval = nullptr, gx_step1 = nullptr, gx_step2 = nullptr;
    const double* graph_key = nullptr;
    double graph_dt = 0;
    double graph_conv = 0;               // energy_to_native baked into the kick kernels
    int graph_cap = 0;
    int launches_eval = 0, launches_step = 0;
    std::vector<std::string> stage_names;
    DBuf flush;                          // > L2, written between timed steps
    uint64_t uid = 0;                    // identifies whose stencil is in constant memory
    FftJobs fft{};                       // FFT lattice cutoff plan (msmb_fft.cu)
    FftJobs fft_top{};                   // FFT top level (n = 0: k_top_direct / k_conv)
    bool lattice_fft = true;             // false: direct stencil (k_lattice)
    AllPairsBuf ap{};                    // direct Coulomb / repulsion overlay (msmb_direct.cu)
    Part whole;                          // the whole system (single-GPU path)
    Part part;                           // this field's part of a spatial decomposition (msmb_dd.cu)
    ~Workspace();
};

struct StageTimer {
    bool on = false;
    std::vector<std::string> names;
    std::vector<double> ms;
    std::vector<int64_t> launches;
    struct Pending {
        int stage;
        cudaEvent_t a, b;
        int nl;
    };
    std::vector<Pending> pending;
    std::vector<cudaEvent_t> pool;
    int stage_index(const char* name);
    cudaEvent_t ev();
    void resolve();
    ~StageTimer();
};

} // namespace msmb

struct msmb_field {
    int kind = MSMB_FIELD_MSM;       // msmb_field_kind
    msmb_cutoff_params cut{};        // pair-only fields (msmb_create_cutoff)
    int rep_on = 0;                  // PairRepulsionOverlay terms (msmb_create_overlay), innermost first
    std::vector<std::pair<double, double>> rep; // (epsilon, sigma) per nested overlay (force_field.cpp:45-68)
    msmb_msm_config cfg{};
    msmb_units units{};
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t side = nullptr;             // long-range chain, forked from `stream`
    cudaStream_t side_a = nullptr;           // the chain's anterpolation (at the main stream's priority)
    cudaStream_t side_r = nullptr;           // pair-list rebuild + the pair kernel's rebuild instance
    cudaStream_t copy = nullptr;             // msmb_propagate: velocity / mass upload beside the first evaluation
    cudaEvent_t vel_ev = nullptr;
    cudaEvent_t fork_ev = nullptr, join_ev = nullptr, mid_ev = nullptr;
    cudaEvent_t sort_ev = nullptr, disp_ev = nullptr, reb_ev = nullptr;
    std::recursive_mutex mu;
    std::unique_ptr<msmb::Workspace> ws;
    msmb::Error last;
    msmb::StageTimer timer;
    int64_t launches = 0;
    int64_t counters[8] = {0};      // msmb_work_counters
    msmb::StateBuf scratch; // device system for the host-pointer entry points
    msmb::DBuf reduce;      // block partials of the raw-state reductions
    int refs = 0;           // live msmb_system objects bound to this field
    int dd_nparts = 1, dd_part = 0; // spatial decomposition part (msmb_dd_set_part)
    int lattice_direct = 0;         // msmb_set_lattice_method: 1 = direct stencil sum
    double pair_skin = -1.0;        // msmb_set_pair_skin (A); < 0 = default
    int list_reuse = 0;             // msmb_set_list_reuse: keep the pair list across calls
    bool destroy_pending = false;
};

struct msmb_system {
    msmb_field* f = nullptr;
    msmb::StateBuf st;
};

namespace msmb {
// engine entry points used by the parareal driver and the spatial decomposition
// (caller holds f->mu)
// vel_ready: the velocities and masses of `s` are still being uploaded on another stream; the call
// waits for the event after launching the initial evaluation (which needs neither)
int engine_propagate(msmb_field* f, StateBuf& s, double dt, int steps, double conv, cudaEvent_t vel_ready = nullptr);
int engine_set_error(msmb_field* f, const Error& e);
int cuda_fail(msmb_field* f, cudaError_t e, const char* where);
Error ensure_workspace(msmb_field* f, int64_t n, const double* box);
void ensure_const_table(msmb_field* f, Workspace& W);
ErrRec read_err(msmb_field* f, Workspace& W);
void record_counters(msmb_field* f, const Workspace& W, const ErrRec& r);
void grow_cap(Workspace& W, const ErrRec& r);
Error error_from_rec(const ErrRec& r);
} // namespace msmb
