// Spatial slab decomposition of MSM force + velocity-Verlet propagation over GPUs
// (configs[2] C3 and configs[3] C4), one part per GPU.
//
// The reference has no decomposition (SPEC.md:504 lists it as a non-goal); this is
// the B200 build's scale-out of propagate (src/integrate.cpp:13-36) over
// msm_potential (src/msm.cpp:52-90).  The x-axis is cut into slabs of pair columns
// (msmb::Part: columns [cx0, cx1) and, per grid level k, x-planes [pl0_k, pl1_k)).
//
// Particles.  A part OWNS the atoms binned into its columns at the last pair-list
// rebuild (it integrates them and computes their forces) and keeps HALO copies of
// the atoms of the neighbouring columns its work reads: the columns the pair lists
// of its clusters reach (a + skin + the list's slack) and the cells its level-0
// planes anterpolate from.  Between rebuilds the owned and halo sets are frozen, as
// the cluster order is: no atom moves more than skin/2, so the sets stay complete.
// Per step only the halo positions travel (owner -> reader, ncclSend/Recv of packed
// (x, y, z)).  At a rebuild (the same global decision as one GPU: some atom moved
// more than skin/2) atoms MIGRATE to the part owning their new column (full state),
// then the halo sets are selected anew (two variable-size exchanges).
//
// Grid.  Every level is stored at full size on every part, but a part computes
// only its own planes: anterpolation of level-0 planes, restriction into its
// coarse planes, the lattice cutoff (direct stencil, msm_phases.cpp:93-134) of its
// planes on each level, prolongation into its planes.  Between those stages the
// planes a part READS but does not own are fetched from their owners: charges on
// [pl0 - R, pl1 + R) (R = ceil(2a/h), msm_phases.cpp:99-100) plus the restriction
// window, potentials on the prolongation window and, for level 0, the
// interpolation window of the owned atoms (msm_phases.cpp:195-222).  A plane range
// is contiguous in the row-major lattice (x slowest), so each exchange is one
// ncclSend/Recv per peer and range, straight from / into the lattice buffers.  Where
// a level is thinner than its halo the same rule fetches from every owner it
// needs (e.g. the top level is gathered whole and computed on every part).
//
// Bit-identity.  Storage stays globally indexed (atom i of the caller is atom i
// here), so every owned value is computed exactly as on one GPU: the same cells
// and within-cell order, the same clusters and pair lists (complete columns), the
// same per-point sums, the same lattice source split.  With the direct lattice
// method on the single-GPU run, a decomposed trajectory equals the single-GPU one
// bit for bit for any part count (tests/test_slab.py); the energy is a sum of
// per-part shares.
//
// Transport.  With an NCCL communicator (one process per GPU) the exchanges are
// ncclSend/ncclRecv inside ncclGroupStart/End and the decisions are ncclAllReduce /
// ncclAllGather, all on the part's stream.  Without one, all parts live in this
// process (local mode, the tests and single-process runs) and the exchanges are
// stream-ordered copies between the parts' buffers.  NCCL is loaded at run time
// (dlopen of libnccl.so.2, which the process may already hold through PyTorch).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "msmb_engine.cuh"

using namespace msmb;

namespace {

void cks(cudaError_t e, const char* w) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(w) + ": " + cudaGetErrorString(e));
}

// ---------------------------------------------------------------- NCCL at run time
struct Nccl {
    bool ok = false;
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

Nccl& nccl() {
    static Nccl n;
    static bool tried = false;
    if (tried) return n;
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        n.why = "libnccl.so.2 not found";
        return n;
    }
    auto sym = [&](auto& fp, const char* name) {
        fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
        return fp != nullptr;
    };
    n.ok = sym(n.GetUniqueId, "ncclGetUniqueId") && sym(n.CommInitRank, "ncclCommInitRank") &&
           sym(n.CommDestroy, "ncclCommDestroy") && sym(n.Send, "ncclSend") && sym(n.Recv, "ncclRecv") &&
           sym(n.GroupStart, "ncclGroupStart") && sym(n.GroupEnd, "ncclGroupEnd") &&
           sym(n.AllReduce, "ncclAllReduce") && sym(n.AllGather, "ncclAllGather") &&
           sym(n.GetErrorString, "ncclGetErrorString");
    if (!n.ok) n.why = "libnccl.so.2 lacks a needed symbol";
    return n;
}

void ckn(ncclResult_t r, const char* w) {
    if (r != ncclSuccess)
        throw std::runtime_error(std::string(w) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "nccl"));
}

// ---------------------------------------------------------------- kernels
__device__ __forceinline__ int column_of(double x, double o, double inv_h, int d0, int cw, int ncx) {
    const double t = __dmul_rn(__dsub_rn(x, o), inv_h); // the binning formula (msm_phases.cpp:23,42)
    int c = (t >= 0.0) ? int(fmin(floor(t), double(d0 - 1))) : 0; // NaN and below: column 0
    c /= cw;
    return c < ncx ? c : ncx - 1;
}

// owner rank of column c: the part whose [cx0, cx1) holds it
__device__ __forceinline__ int owner_of(int c, const int* __restrict__ cx1s, int nparts) {
    int r = 0;
    while (r + 1 < nparts && c >= cx1s[r]) ++r;
    return r;
}

struct ColP {
    double o, inv_h;
    int d0, cw, ncx;
};

// mark[i] = v for the atoms i in list[0..n)
__global__ void k_mark(const int* __restrict__ list, int64_t n, int* mark, int v) {
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t < n) mark[list[t]] = v;
}

// mark[i] = 1 for the atoms whose column is in [c0, c1) (replicated initial state)
__global__ void k_mark_columns(int64_t n, const double* __restrict__ x, ColP p, int c0, int c1, int* mark) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int c = column_of(x[i], p.o, p.inv_h, p.d0, p.cw, p.ncx);
    mark[i] = (c >= c0 && c < c1) ? 1 : 0;
}

// out[scan[i]] = i where mark[i] (ascending: the caller's atom order)
__global__ void k_compact(int64_t n, const int* __restrict__ mark, const int* __restrict__ scan, int* out) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n && mark[i]) out[scan[i]] = int(i);
}

// per owned atom: its column's owner (migration) -- dest[t]
__global__ void k_dest(const int* __restrict__ owned, int64_t n, const double* __restrict__ x, ColP p,
                       const int* __restrict__ cx1s, int nparts, int* dest, int* count) {
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const int r = owner_of(column_of(x[owned[t]], p.o, p.inv_h, p.d0, p.cw, p.ncx), cx1s, nparts);
    dest[t] = r;
    atomicAdd(&count[r], 1);
}

// per owned atom and peer: is its column in the peer's local range (halo selection)
__global__ void k_halo_flag(const int* __restrict__ owned, int64_t n, const double* __restrict__ x, ColP p, int c0,
                            int c1, int* flag) {
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const int c = column_of(x[owned[t]], p.o, p.inv_h, p.d0, p.cw, p.ncx);
    flag[t] = (c >= c0 && c < c1) ? 1 : 0;
}

// list entries whose flag equals `want`: out[scan[t]] = list[t] (order kept)
__global__ void k_select(const int* __restrict__ list, int64_t n, const int* __restrict__ flag, int want,
                         const int* __restrict__ scan, int* out) {
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t < n && flag[t] == want) out[scan[t]] = list[t];
}

__global__ void k_eq(const int* __restrict__ a, int64_t n, int v, int* out) {
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t < n) out[t] = a[t] == v ? 1 : 0;
}

// packed records: ids as doubles (exact below 2^53) + `nv` state arrays
__global__ void k_pack(const int* __restrict__ ids, int64_t n, DevState s, int nv, double* out) {
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const int i = ids[t];
    const double* src[6] = {s.x, s.y, s.z, s.vx, s.vy, s.vz};
    double* o = out + t * (nv + 1);
    o[0] = double(i);
    for (int k = 0; k < nv; ++k) o[1 + k] = src[k][i];
}

__global__ void k_unpack(const double* __restrict__ in, int64_t n, DevState s, int nv, int* ids, int* mark) {
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const double* r = in + t * (nv + 1);
    const int i = int(r[0]);
    double* dst[6] = {s.x, s.y, s.z, s.vx, s.vy, s.vz};
    for (int k = 0; k < nv; ++k) dst[k][i] = r[1 + k];
    if (ids) ids[t] = i;
    if (mark) mark[i] = 1;
}

// per-step halo refresh: positions only, in the frozen order of the lists
__global__ void k_pack_pos(const int* __restrict__ ids, int64_t n, const double* __restrict__ x,
                           const double* __restrict__ y, const double* __restrict__ z, double* out) {
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const int i = ids[t];
    out[3 * t] = x[i];
    out[3 * t + 1] = y[i];
    out[3 * t + 2] = z[i];
}

__global__ void k_unpack_pos(const int* __restrict__ ids, int64_t n, const double* __restrict__ in, double* x,
                             double* y, double* z) {
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const int i = ids[t];
    x[i] = in[3 * t];
    y[i] = in[3 * t + 1];
    z[i] = in[3 * t + 2];
}

// velocity Verlet of the owned atoms (src/integrate.cpp:24-33, the reference's
// operation order, as k_kick_drift / k_kick); the step counter advances once per drift
__global__ void k_verlet_owned(const int* __restrict__ owned, int64_t n, DevState s, const double* __restrict__ fx,
                               const double* __restrict__ fy, const double* __restrict__ fz, double dt, double hdc,
                               int kicks, int drift, ErrRec* err) {
    if (__ldcg(&err->kind) != 0) return;
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t == 0 && drift) err->pairs = 0, err->candidates = 0, err->cur_step += 1;
    if (t >= n) return;
    const int i = owned[t];
    const double c = __ddiv_rn(hdc, s.m[i]);
    double a = s.vx[i], b = s.vy[i], d = s.vz[i];
    const double Fx = fx[i], Fy = fy[i], Fz = fz[i];
    for (int k = 0; k < kicks; ++k) {
        a = __dadd_rn(a, __dmul_rn(Fx, c));
        b = __dadd_rn(b, __dmul_rn(Fy, c));
        d = __dadd_rn(d, __dmul_rn(Fz, c));
    }
    s.vx[i] = a;
    s.vy[i] = b;
    s.vz[i] = d;
    if (drift) {
        s.x[i] = __dadd_rn(s.x[i], __dmul_rn(a, dt));
        s.y[i] = __dadd_rn(s.y[i], __dmul_rn(b, dt));
        s.z[i] = __dadd_rn(s.z[i], __dmul_rn(d, dt));
    }
}

// skin/2 displacement test of the owned atoms since the last rebuild (k_disp)
__global__ void k_disp_owned(const int* __restrict__ owned, int64_t n, const double* __restrict__ x,
                             const double* __restrict__ y, const double* __restrict__ z,
                             const double* __restrict__ ref, int64_t N, double half_skin2, int* flag) {
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const int i = owned[t];
    const double dx = x[i] - ref[i], dy = y[i] - ref[N + i], dz = z[i] - ref[2 * N + i];
    if (!(dx * dx + dy * dy + dz * dz <= half_skin2)) *flag = 1;
}

__global__ void k_gather_e(const int* __restrict__ owned, int64_t n, const double* __restrict__ e, double* out) {
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t < n) out[t] = e[owned[t]];
}

int nb256(int64_t n) { return int(std::max<int64_t>(1, (n + 255) / 256)); }

// ---------------------------------------------------------------- plans
struct Range {
    int lo = 0, hi = 0;
    int size() const { return std::max(0, hi - lo); }
};
Range isect(Range a, Range b) { return Range{std::max(a.lo, b.lo), std::min(a.hi, b.hi)}; }

struct Op { // one peer's share of an exchange: send [s, s+sb) and receive into [r, r+rb)
    int peer = -1;
    const void* s = nullptr;
    size_t sb = 0;
    void* r = nullptr;
    size_t rb = 0;
};

} // namespace

namespace msmb {

// One part (GPU) of a decomposition.
struct SlabPart {
    msmb_field* f = nullptr;
    int rank = 0, nparts = 1;
    StateBuf st;      // the whole system, globally indexed; only local atoms are current
    Part P;
    std::vector<Range> cols, lcols; // owned / local column ranges of every part
    // plane ranges per level of every part: owned, charge need, potential need
    std::vector<std::vector<Range>> own, qneed, uneed;
    // atom sets (ascending indices)
    DBuf owned, local, mark_own, mark_loc, scan, tmp, dest, flag, cnt, sel;
    int64_t n_owned = 0, n_local = 0;
    // halo refresh plan: to peer p the owned atoms in p's local columns, from p its atoms here
    std::vector<int64_t> hsend_off, hrecv_off; // [nparts + 1]
    DBuf hsend_ids, hrecv_ids, hsend_buf, hrecv_buf;
    // exchange scratch (migration / halo selection)
    DBuf xsend, xrecv;
    DBuf ebuf, dflag; // owned e_i, displacement flag
    ErrRec rec{};
    int64_t bytes_step = 0, bytes_rebuild = 0, migrated = 0;
    std::vector<Op> ops;
    cudaStream_t stream() const { return f->stream; }
    Workspace& W() const { return *f->ws; }
};

} // namespace msmb

struct msmb_slab {
    std::vector<std::unique_ptr<SlabPart>> parts; // this process's parts
    int nparts = 1;
    ncclComm_t comm = nullptr;
    bool own_comm = false;
    bool local() const { return comm == nullptr; }
    int64_t rebuilds = 0;
    msmb::Error last;
};

namespace {

void set_err(msmb_slab* g, const Error& e) {
    g->last = e;
    for (auto& p : g->parts) p->f->last = e;
}

// ---------------------------------------------------------------- transport
// Each part has filled p->ops (at most one Op per peer); run them all.
void exchange(msmb_slab* g, int64_t& bytes_acc) {
    if (g->local()) {
        for (auto& p : g->parts) cks(cudaStreamSynchronize(p->stream()), "sync");
        for (auto& p : g->parts) {
            for (const Op& op : p->ops) {
                if (!op.rb) continue;
                SlabPart* q = g->parts[size_t(op.peer)].get();
                const Op* m = nullptr;
                for (const Op& o2 : q->ops)
                    if (o2.peer == p->rank) m = &o2;
                if (!m || m->sb != op.rb) throw std::runtime_error("slab: unmatched exchange");
                cks(cudaMemcpyAsync(op.r, m->s, op.rb, cudaMemcpyDefault, p->stream()), "copy");
                p->bytes_step += int64_t(op.rb);
            }
        }
        for (auto& p : g->parts) cks(cudaStreamSynchronize(p->stream()), "sync");
    } else {
        SlabPart* p = g->parts[0].get();
        Nccl& N = nccl();
        ckn(N.GroupStart(), "ncclGroupStart");
        for (const Op& op : p->ops) {
            if (op.sb) ckn(N.Send(op.s, op.sb, ncclUint8, op.peer, g->comm, p->stream()), "ncclSend");
            if (op.rb) ckn(N.Recv(op.r, op.rb, ncclUint8, op.peer, g->comm, p->stream()), "ncclRecv");
            p->bytes_step += int64_t(op.rb);
        }
        ckn(N.GroupEnd(), "ncclGroupEnd");
    }
    (void)bytes_acc;
    for (auto& p : g->parts) p->ops.clear();
}

// host-visible max over every part of every rank of per-part values
int64_t allmax(msmb_slab* g, const std::vector<int64_t>& mine) {
    int64_t m = LLONG_MIN;
    for (int64_t v : mine) m = std::max(m, v);
    if (!g->local()) {
        SlabPart* p = g->parts[0].get();
        int64_t* d = p->tmp.as<int64_t>();
        cks(cudaMemcpyAsync(d, &m, sizeof m, cudaMemcpyHostToDevice, p->stream()), "H2D");
        ckn(nccl().AllReduce(d, d, 1, ncclInt64, ncclMax, g->comm, p->stream()), "ncclAllReduce");
        cks(cudaMemcpyAsync(&m, d, sizeof m, cudaMemcpyDeviceToHost, p->stream()), "D2H");
        cks(cudaStreamSynchronize(p->stream()), "sync");
    }
    return m;
}

// all parts' `count` values of `per` int64s each, in rank order
std::vector<int64_t> allgather(msmb_slab* g, const std::vector<std::vector<int64_t>>& mine, int per) {
    std::vector<int64_t> out(size_t(g->nparts) * per);
    if (g->local()) {
        for (size_t r = 0; r < mine.size(); ++r)
            for (int k = 0; k < per; ++k) out[r * per + k] = mine[r][size_t(k)];
        return out;
    }
    SlabPart* p = g->parts[0].get();
    int64_t* d = p->tmp.as<int64_t>();
    cks(cudaMemcpyAsync(d + size_t(p->rank) * per, mine[0].data(), sizeof(int64_t) * per, cudaMemcpyHostToDevice,
                        p->stream()),
        "H2D");
    ckn(nccl().AllGather(d + size_t(p->rank) * per, d, size_t(per), ncclInt64, g->comm, p->stream()), "AllGather");
    cks(cudaMemcpyAsync(out.data(), d, sizeof(int64_t) * out.size(), cudaMemcpyDeviceToHost, p->stream()), "D2H");
    cks(cudaStreamSynchronize(p->stream()), "sync");
    return out;
}

ColP colp(const Geometry& g) {
    return ColP{g.lv[0].origin[0], g.inv_h0, g.lv[0].dims[0], g.cw, g.ncx};
}

// ---------------------------------------------------------------- plans (host, static)
void make_plans(SlabPart& p) {
    const Geometry& g = p.W().g;
    const int P = p.nparts, L = g.levels;
    p.cols.resize(size_t(P));
    p.lcols.resize(size_t(P));
    p.own.assign(size_t(L), std::vector<Range>(size_t(P)));
    p.qneed = p.own;
    p.uneed = p.own;
    const int R = g.lat.R;
    // pair lists reach ceil(cut / colw) + 1 columns beyond a cluster's box (k_pairlist), a
    // cluster box lies within its column at the rebuild: one more column of slack
    const double cut = g.screen_cut + g.skin;
    const int Dp = int(std::ceil(cut / g.colw)) + 2;
    for (int r = 0; r < P; ++r) {
        const Part Q = make_part(g, P, r);
        p.cols[r] = Range{Q.cx0, Q.cx1};
        // level-0 planes [pl0, pl1) anterpolate from cells [pl0 - 2, pl1 + 1); an atom drifts
        // by less than one cell between rebuilds
        const int a0 = std::max(0, Q.pl0[0] - 3), a1 = std::min(g.lv[0].dims[0], Q.pl1[0] + 2);
        int lc0 = Q.cx0 - Dp, lc1 = Q.cx1 + Dp;
        if (Q.pl1[0] > Q.pl0[0]) {
            lc0 = std::min(lc0, a0 / g.cw);
            lc1 = std::max(lc1, (a1 - 1) / g.cw + 1);
        }
        p.lcols[r] = Range{std::max(0, lc0), std::min(g.ncx, lc1)};
        for (int k = 0; k < L; ++k) {
            const int d0 = g.lv[k].dims[0];
            p.own[k][r] = Range{Q.pl0[k], Q.pl1[k]};
            if (k == L - 1) { // top: gathered whole, computed on every part
                p.qneed[k][r] = Range{0, d0};
                p.uneed[k][r] = Range{0, d0};
                continue;
            }
            // charges: the lattice cutoff of owned planes reads [pl0 - R, pl1 + R); the
            // restriction into owned coarse planes reads the fine planes feeding them
            Range q{Q.pl0[k] - R, Q.pl1[k] + R};
            const TransferAxis& T = g.tr[k][0];
            const Range oc{Q.pl0[k + 1], Q.pl1[k + 1]};
            for (int i = 0; i < d0; ++i)
                if (T.base[size_t(i)] + 3 >= oc.lo && T.base[size_t(i)] < oc.hi && oc.size() > 0)
                    q.lo = std::min(q.lo, i), q.hi = std::max(q.hi, i + 1);
            p.qneed[k][r] = isect(q, Range{0, d0});
        }
        // potentials: prolongation into owned fine planes of level k reads the coarse planes
        // base..base+3 of level k+1; interpolation of owned atoms reads level-0 planes of the
        // cells of owned columns (+-1 cell of drift): [cx0 cw - 2, cx1 cw + 3)
        for (int k = 0; k + 1 < L; ++k) {
            const TransferAxis& T = g.tr[k][0];
            Range u{INT_MAX, INT_MIN};
            for (int i = Q.pl0[k]; i < Q.pl1[k]; ++i)
                u.lo = std::min(u.lo, T.base[size_t(i)]), u.hi = std::max(u.hi, T.base[size_t(i)] + 4);
            if (u.lo > u.hi) u = Range{0, 0};
            if (k + 1 < L - 1) p.uneed[k + 1][r] = isect(u, Range{0, g.lv[k + 1].dims[0]});
        }
        p.uneed[0][r] = isect(Range{Q.cx0 * g.cw - 2, Q.cx1 * g.cw + 3}, Range{0, g.lv[0].dims[0]});
    }
}

// ops fetching the planes `need[k][me]` of level k (buffer `base` = charges or
// potentials) from their owners, and serving the owned planes others need
void plane_ops(SlabPart& p, int k, double* base, const std::vector<std::vector<Range>>& need) {
    const Geometry& g = p.W().g;
    const LevelGeom& lv = g.lv[k];
    const size_t plane = size_t(lv.dims[1]) * lv.dims[2];
    double* lat = base + lv.offset;
    for (int q = 0; q < p.nparts; ++q) {
        if (q == p.rank) continue;
        const Range s = isect(p.own[k][p.rank], need[k][q]); // mine, q reads
        const Range r = isect(p.own[k][q], need[k][p.rank]); // q's, I read
        if (!s.size() && !r.size()) continue;
        Op op;
        op.peer = q;
        op.s = lat + size_t(s.lo) * plane;
        op.sb = sizeof(double) * plane * size_t(s.size());
        op.r = lat + size_t(r.lo) * plane;
        op.rb = sizeof(double) * plane * size_t(r.size());
        p.ops.push_back(op);
    }
}

void ensure_buf(DBuf& b, size_t bytes) {
    if (b.bytes < bytes) cks(b.alloc(bytes), "cudaMalloc");
}

// sorted list of the marked atoms
int64_t compact(SlabPart& p, const int* mark, DBuf& out) {
    const int64_t N = p.st.n;
    cudaStream_t st = p.stream();
    int* scan = p.scan.as<int>();
    launch_scan_exclusive(st, mark, scan, p.W().c.scan_tmp, N + 1);
    int cnt = 0;
    cks(cudaMemcpyAsync(&cnt, scan + N, sizeof(int), cudaMemcpyDeviceToHost, st), "D2H");
    cks(cudaStreamSynchronize(st), "sync");
    ensure_buf(out, sizeof(int) * size_t(std::max(cnt, 1)));
    k_compact<<<nb256(N), 256, 0, st>>>(N, mark, scan, out.as<int>());
    return cnt;
}

// halo selection: for every peer q, my owned atoms in q's local columns (flag + scan)
void halo_send_lists(SlabPart& p, std::vector<int64_t>& counts) {
    cudaStream_t st = p.stream();
    const ColP cp = colp(p.W().g);
    counts.assign(size_t(p.nparts), 0);
    std::vector<int> ids;
    p.hsend_off.assign(size_t(p.nparts) + 1, 0);
    ensure_buf(p.flag, sizeof(int) * size_t(p.n_owned + 1));
    ensure_buf(p.sel, sizeof(int) * size_t(p.n_owned + 1) * size_t(std::max(1, p.nparts - 1)));
    int64_t off = 0;
    for (int q = 0; q < p.nparts; ++q) {
        p.hsend_off[size_t(q)] = off;
        if (q == p.rank || p.n_owned == 0) continue;
        int* flag = p.flag.as<int>();
        k_halo_flag<<<nb256(p.n_owned), 256, 0, st>>>(p.owned.as<int>(), p.n_owned, p.st.dev().x, cp,
                                                      p.lcols[q].lo, p.lcols[q].hi, flag);
        cks(cudaMemsetAsync(flag + p.n_owned, 0, sizeof(int), st), "memset");
        launch_scan_exclusive(st, flag, p.scan.as<int>(), p.W().c.scan_tmp, p.n_owned + 1);
        int c = 0;
        cks(cudaMemcpyAsync(&c, p.scan.as<int>() + p.n_owned, sizeof(int), cudaMemcpyDeviceToHost, st), "D2H");
        cks(cudaStreamSynchronize(st), "sync");
        k_select<<<nb256(p.n_owned), 256, 0, st>>>(p.owned.as<int>(), p.n_owned, flag, 1, p.scan.as<int>(),
                                                   p.sel.as<int>() + off);
        counts[size_t(q)] = c;
        off += c;
    }
    p.hsend_off[size_t(p.nparts)] = off;
    ensure_buf(p.hsend_ids, sizeof(int) * size_t(std::max<int64_t>(off, 1)));
    if (off) cks(cudaMemcpyAsync(p.hsend_ids.p, p.sel.p, sizeof(int) * size_t(off), cudaMemcpyDeviceToDevice, st), "D2D");
    cks(cudaStreamSynchronize(st), "sync");
}

// ---------------------------------------------------------------- (re)decomposition
// Setup: every part holds the caller's whole initial state, so ownership and halos
// are local computations (the same rule on every part).
void setup_sets(msmb_slab* g) {
    for (auto& pp : g->parts) {
        SlabPart& p = *pp;
        const int64_t N = p.st.n;
        cudaStream_t st = p.stream();
        const ColP cp = colp(p.W().g);
        int* mo = p.mark_own.as<int>();
        k_mark_columns<<<nb256(N), 256, 0, st>>>(N, p.st.dev().x, cp, p.cols[p.rank].lo, p.cols[p.rank].hi, mo);
        cks(cudaMemsetAsync(mo + N, 0, sizeof(int), st), "memset");
        p.n_owned = compact(p, mo, p.owned);
    }
    // the halo sets then follow from the owned sets exactly as at a rebuild (select_halos)
}

// The halo sets and refresh lists from the owned sets: every owner sends (id, x, y, z)
// of its atoms in each peer's local columns; receivers record them.
void select_halos(msmb_slab* g) {
    nvtxRangePushA("slab halo selection");
    struct Pop { ~Pop() { nvtxRangePop(); } } pop_at_exit;
    std::vector<std::vector<int64_t>> counts(g->parts.size());
    for (size_t i = 0; i < g->parts.size(); ++i) halo_send_lists(*g->parts[i], counts[i]);
    const int P = g->nparts;
    const std::vector<int64_t> all = allgather(g, counts, P); // all[s * P + r]: s sends to r
    for (auto& pp : g->parts) {
        SlabPart& p = *pp;
        cudaStream_t st = p.stream();
        p.hrecv_off.assign(size_t(P) + 1, 0);
        int64_t off = 0;
        for (int s = 0; s < P; ++s) {
            p.hrecv_off[size_t(s)] = off;
            if (s != p.rank) off += all[size_t(s) * P + p.rank];
        }
        p.hrecv_off[size_t(P)] = off;
        const int64_t ns = p.hsend_off[size_t(P)];
        ensure_buf(p.hrecv_ids, sizeof(int) * size_t(std::max<int64_t>(off, 1)));
        ensure_buf(p.hsend_buf, sizeof(double) * 4 * size_t(std::max<int64_t>(ns, 1)));
        ensure_buf(p.hrecv_buf, sizeof(double) * 4 * size_t(std::max<int64_t>(off, 1)));
        if (ns) k_pack<<<nb256(ns), 256, 0, st>>>(p.hsend_ids.as<int>(), ns, p.st.dev(), 3, p.hsend_buf.as<double>());
        for (int q = 0; q < P; ++q) {
            if (q == p.rank) continue;
            Op op;
            op.peer = q;
            op.s = p.hsend_buf.as<double>() + 4 * p.hsend_off[size_t(q)];
            op.sb = sizeof(double) * 4 * size_t(p.hsend_off[size_t(q) + 1] - p.hsend_off[size_t(q)]);
            op.r = p.hrecv_buf.as<double>() + 4 * p.hrecv_off[size_t(q)];
            op.rb = sizeof(double) * 4 * size_t(p.hrecv_off[size_t(q) + 1] - p.hrecv_off[size_t(q)]);
            if (op.sb || op.rb) p.ops.push_back(op);
        }
    }
    int64_t dummy = 0;
    exchange(g, dummy);
    for (auto& pp : g->parts) {
        SlabPart& p = *pp;
        cudaStream_t st = p.stream();
        const int64_t N = p.st.n, nr = p.hrecv_off[size_t(P)];
        int* ml = p.mark_loc.as<int>();
        cks(cudaMemsetAsync(ml, 0, sizeof(int) * size_t(N + 1), st), "memset");
        k_mark<<<nb256(p.n_owned), 256, 0, st>>>(p.owned.as<int>(), p.n_owned, ml, 1);
        if (nr) k_unpack<<<nb256(nr), 256, 0, st>>>(p.hrecv_buf.as<double>(), nr, p.st.dev(), 3, p.hrecv_ids.as<int>(), ml);
        p.n_local = compact(p, ml, p.local);
        p.bytes_rebuild += int64_t(sizeof(double) * 4 * nr);
    }
}

// Migration at a rebuild: owned atoms whose column now belongs to another part move
// there with their whole state (x, y, z, vx, vy, vz); then the owned sets are rebuilt.
void migrate(msmb_slab* g) {
    nvtxRangePushA("slab migrate");
    struct Pop { ~Pop() { nvtxRangePop(); } } pop_at_exit;
    const int P = g->nparts;
    std::vector<std::vector<int64_t>> counts(g->parts.size());
    for (size_t pi = 0; pi < g->parts.size(); ++pi) {
        SlabPart& p = *g->parts[pi];
        cudaStream_t st = p.stream();
        ensure_buf(p.dest, sizeof(int) * size_t(p.n_owned + 1));
        ensure_buf(p.cnt, sizeof(int) * size_t(P));
        int* dcount = p.cnt.as<int>(); // atoms per destination part
        std::vector<int> hb(static_cast<size_t>(P));
        for (int r = 0; r < P; ++r) hb[size_t(r)] = p.cols[size_t(r)].hi;
        DBuf bounds;
        cks(bounds.alloc(sizeof(int) * size_t(P)), "cudaMalloc");
        cks(cudaMemcpyAsync(bounds.p, hb.data(), sizeof(int) * size_t(P), cudaMemcpyHostToDevice, st), "H2D");
        cks(cudaMemsetAsync(dcount, 0, sizeof(int) * size_t(P), st), "memset");
        if (p.n_owned)
            k_dest<<<nb256(p.n_owned), 256, 0, st>>>(p.owned.as<int>(), p.n_owned, p.st.dev().x, colp(p.W().g),
                                                     bounds.as<int>(), P, p.dest.as<int>(), dcount);
        std::vector<int> hc(static_cast<size_t>(P));
        cks(cudaMemcpyAsync(hc.data(), dcount, sizeof(int) * size_t(P), cudaMemcpyDeviceToHost, st), "D2H");
        cks(cudaStreamSynchronize(st), "sync");
        counts[pi].assign(size_t(P), 0);
        for (int r = 0; r < P; ++r)
            if (r != p.rank) counts[pi][size_t(r)] = hc[size_t(r)];
        // pack the leavers per destination (order kept: ascending index)
        int64_t nleave = 0;
        for (int r = 0; r < P; ++r) nleave += counts[pi][size_t(r)];
        ensure_buf(p.xsend, sizeof(double) * 7 * size_t(std::max<int64_t>(nleave, 1)));
        ensure_buf(p.sel, sizeof(int) * size_t(std::max<int64_t>(p.n_owned, 1) + 1));
        ensure_buf(p.flag, sizeof(int) * size_t(p.n_owned + 1));
        int64_t off = 0;
        for (int r = 0; r < P; ++r) {
            const int64_t c = counts[pi][size_t(r)];
            if (r == p.rank || c == 0) continue;
            int* flag = p.flag.as<int>();
            k_eq<<<nb256(p.n_owned), 256, 0, st>>>(p.dest.as<int>(), p.n_owned, r, flag);
            cks(cudaMemsetAsync(flag + p.n_owned, 0, sizeof(int), st), "memset");
            launch_scan_exclusive(st, flag, p.scan.as<int>(), p.W().c.scan_tmp, p.n_owned + 1);
            k_select<<<nb256(p.n_owned), 256, 0, st>>>(p.owned.as<int>(), p.n_owned, flag, 1, p.scan.as<int>(),
                                                       p.sel.as<int>());
            k_pack<<<nb256(c), 256, 0, st>>>(p.sel.as<int>(), c, p.st.dev(), 6, p.xsend.as<double>() + 7 * off);
            // the leavers are no longer owned here
            k_mark<<<nb256(c), 256, 0, st>>>(p.sel.as<int>(), c, p.mark_own.as<int>(), 0);
            off += c;
        }
        cks(cudaStreamSynchronize(st), "sync");
        p.migrated += nleave;
    }
    const std::vector<int64_t> all = allgather(g, counts, P);
    for (auto& pp : g->parts) {
        SlabPart& p = *pp;
        int64_t nin = 0;
        for (int s = 0; s < P; ++s)
            if (s != p.rank) nin += all[size_t(s) * P + p.rank];
        ensure_buf(p.xrecv, sizeof(double) * 7 * size_t(std::max<int64_t>(nin, 1)));
        int64_t so = 0, ro = 0;
        for (int q = 0; q < P; ++q) {
            if (q == p.rank) continue;
            const int64_t sc = all[size_t(p.rank) * P + q], rc = all[size_t(q) * P + p.rank];
            if (sc || rc) {
                Op op;
                op.peer = q;
                op.s = p.xsend.as<double>() + 7 * so;
                op.sb = sizeof(double) * 7 * size_t(sc);
                op.r = p.xrecv.as<double>() + 7 * ro;
                op.rb = sizeof(double) * 7 * size_t(rc);
                p.ops.push_back(op);
            }
            so += sc;
            ro += rc;
        }
        p.bytes_rebuild += int64_t(sizeof(double) * 7 * size_t(nin));
    }
    int64_t dummy = 0;
    exchange(g, dummy);
    for (auto& pp : g->parts) {
        SlabPart& p = *pp;
        cudaStream_t st = p.stream();
        int64_t nin = 0;
        for (int s = 0; s < P; ++s)
            if (s != p.rank) nin += all[size_t(s) * P + p.rank];
        if (nin) k_unpack<<<nb256(nin), 256, 0, st>>>(p.xrecv.as<double>(), nin, p.st.dev(), 6, nullptr, p.mark_own.as<int>());
        cks(cudaMemsetAsync(p.mark_own.as<int>() + p.st.n, 0, sizeof(int), st), "memset");
        p.n_owned = compact(p, p.mark_own.as<int>(), p.owned);
    }
}

// ---------------------------------------------------------------- one evaluation
// The engine's evaluation restricted to the part's work, with the plane exchanges
// between the grid stages (stream-ordered on every part).
void evaluate(msmb_slab* g, bool rebuild) {
    nvtxRangePushA("slab evaluate");
    struct Pop { ~Pop() { nvtxRangePop(); } } pop_at_exit;
    const int L = g->parts[0]->W().g.levels;
    for (auto& pp : g->parts) {
        SlabPart& p = *pp;
        Workspace& W = p.W();
        const Geometry& G = W.g;
        cudaStream_t st = p.stream();
        DevState s = p.st.dev();
        ensure_const_table(p.f, W);
        // a new local atom set: the cell sort cannot be reused (atoms left cells)
        if (rebuild) cks(cudaMemsetAsync(W.c.flag + 6, 0, sizeof(int), st), "memset");
        int nl = launch_bin(st, G, s, W.a, W.c, W.err, p.local.as<int>(), p.n_local);
        nl += launch_sort(st, G, s, W.a, W.c, W.err, p.local.as<int>(), p.n_local);
        nl += launch_clusters(st, G, s.n, s, W.a, W.c, W.err, W.cap, W.part, rebuild ? 1 : 0, 0);
        nl += launch_pairs(st, G, s.n, s, W.a, W.c, W.err, W.cap, W.part);
        nl += launch_anterp(st, G, s, W.a, W.c, W.L, W.err, W.part);
        p.f->launches += nl;
        plane_ops(p, 0, W.L.charge, p.qneed);
    }
    int64_t acc = 0;
    exchange(g, acc);
    for (int k = 0; k + 1 < L; ++k) {
        for (auto& pp : g->parts) {
            SlabPart& p = *pp;
            Workspace& W = p.W();
            p.f->launches += launch_restrict_planes(p.stream(), W.g, k, W.L, W.err, W.part.pl0[k + 1], W.part.pl1[k + 1]);
            plane_ops(p, k + 1, W.L.charge, p.qneed);
        }
        exchange(g, acc);
    }
    for (auto& pp : g->parts) {
        SlabPart& p = *pp;
        Workspace& W = p.W();
        p.f->launches += W.lattice_fft ? launch_lattice_fft(p.stream(), W.fft, W.err) // one part: whole levels
                                       : launch_lattice(p.stream(), W.g, W.L, W.err, W.part);
        p.f->launches += W.fft_top.n ? launch_lattice_fft(p.stream(), W.fft_top, W.err)
                                     : launch_top(p.stream(), W.g, W.L, W.err);
    }
    for (int k = L - 2; k >= 0; --k) {
        if (k + 1 < L - 1) { // the top level is complete on every part
            for (auto& pp : g->parts) plane_ops(*pp, k + 1, pp->W().L.pot, pp->uneed);
            exchange(g, acc);
        }
        for (auto& pp : g->parts) {
            SlabPart& p = *pp;
            Workspace& W = p.W();
            p.f->launches += launch_prolong_planes(p.stream(), W.g, k, W.L, W.err, W.part.pl0[k], W.part.pl1[k]);
        }
    }
    for (auto& pp : g->parts) plane_ops(*pp, 0, pp->W().L.pot, pp->uneed);
    exchange(g, acc);
    for (auto& pp : g->parts) {
        SlabPart& p = *pp;
        Workspace& W = p.W();
        const Geometry& G = W.g;
        cudaStream_t st = p.stream();
        DevState s = p.st.dev();
        DevOut o = W.o;
        o.phi = o.phis = o.phil = nullptr;
        int nl = launch_interp(st, G, s.n, W.a, W.c, W.L, o, W.err, 0, W.part);
        // the part's energy share: its atoms' e_i in index order (fixed tree)
        if (p.n_owned) {
            k_gather_e<<<nb256(p.n_owned), 256, 0, st>>>(p.owned.as<int>(), p.n_owned, o.e, p.ebuf.as<double>());
            nl += 1 + launch_energy_sum(st, p.n_owned, p.ebuf.as<double>(), W.o.partial, G.units.coulomb_constant,
                                        W.o.energy, 0, W.err);
        } else {
            cks(cudaMemsetAsync(W.o.energy, 0, sizeof(double), st), "memset");
        }
        nl += launch_finalize(st, s, W.err);
        p.f->launches += nl;
    }
}

// ---------------------------------------------------------------- a propagate call
void halo_refresh(msmb_slab* g) {
    nvtxRangePushA("slab halo refresh");
    struct Pop { ~Pop() { nvtxRangePop(); } } pop_at_exit;
    for (auto& pp : g->parts) {
        SlabPart& p = *pp;
        const int64_t ns = p.hsend_off[size_t(p.nparts)];
        DevState s = p.st.dev();
        if (ns)
            k_pack_pos<<<nb256(ns), 256, 0, p.stream()>>>(p.hsend_ids.as<int>(), ns, s.x, s.y, s.z,
                                                          p.hsend_buf.as<double>());
        for (int q = 0; q < p.nparts; ++q) {
            if (q == p.rank) continue;
            Op op;
            op.peer = q;
            op.s = p.hsend_buf.as<double>() + 3 * p.hsend_off[size_t(q)];
            op.sb = sizeof(double) * 3 * size_t(p.hsend_off[size_t(q) + 1] - p.hsend_off[size_t(q)]);
            op.r = p.hrecv_buf.as<double>() + 3 * p.hrecv_off[size_t(q)];
            op.rb = sizeof(double) * 3 * size_t(p.hrecv_off[size_t(q) + 1] - p.hrecv_off[size_t(q)]);
            if (op.sb || op.rb) p.ops.push_back(op);
        }
    }
    int64_t acc = 0;
    exchange(g, acc);
    for (auto& pp : g->parts) {
        SlabPart& p = *pp;
        const int64_t nr = p.hrecv_off[size_t(p.nparts)];
        DevState s = p.st.dev();
        if (nr)
            k_unpack_pos<<<nb256(nr), 256, 0, p.stream()>>>(p.hrecv_ids.as<int>(), nr, p.hrecv_buf.as<double>(), s.x,
                                                            s.y, s.z);
    }
}

ErrRec combine_errors(msmb_slab* g) {
    std::vector<std::vector<int64_t>> mine;
    const int per = int((sizeof(ErrRec) + 7) / 8);
    for (auto& pp : g->parts) {
        SlabPart& p = *pp;
        cks(cudaMemcpyAsync(&p.rec, p.W().err, sizeof(ErrRec), cudaMemcpyDeviceToHost, p.stream()), "D2H");
        cks(cudaStreamSynchronize(p.stream()), "sync");
        std::vector<int64_t> v(size_t(per), 0);
        std::memcpy(v.data(), &p.rec, sizeof(ErrRec));
        mine.push_back(v);
    }
    const std::vector<int64_t> all = allgather(g, mine, per);
    // the error an undivided run meets first: the earliest failing step; within it a
    // pair error (lexicographically first pair) before coverage (lowest particle)
    ErrRec best{};
    bool have = false;
    unsigned long long pairs = 0;
    for (int r = 0; r < g->nparts; ++r) {
        ErrRec e;
        std::memcpy(&e, all.data() + size_t(r) * per, sizeof(ErrRec));
        pairs += e.pairs;
        if (!e.kind) continue;
        auto pair_err = [](const ErrRec& x) { return x.kind == MSMB_ERR_COINCIDENT || x.kind == MSMB_ERR_DOMAIN; };
        bool better = !have;
        if (have) {
            if (e.kind == kOverflowKind || best.kind == kOverflowKind)
                better = e.kind == kOverflowKind && best.kind != kOverflowKind;
            else if (e.step != best.step)
                better = e.step < best.step;
            else if (pair_err(e) != pair_err(best))
                better = pair_err(e);
            else if (pair_err(e))
                better = e.pair_key < best.pair_key;
            else
                better = e.err_i < best.err_i;
        }
        if (better) best = e, have = true;
    }
    best.pairs = pairs;
    return best;
}

} // namespace

// ================================================================= C ABI
extern "C" {

int msmb_nccl_unique_id(void* id128) {
    Nccl& N = nccl();
    if (!N.ok) return MSMB_ERR_CUDA;
    ncclUniqueId id;
    if (N.GetUniqueId(&id) != ncclSuccess) return MSMB_ERR_CUDA;
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(id128, &id, sizeof id);
    return MSMB_OK;
}

int msmb_slab_create(msmb_field* const* fields, int nfields, int nparts, int rank, const void* nccl_id,
                     void* nccl_comm, msmb_slab** out) {
    if (!out) return MSMB_ERR_CONFIG;
    *out = nullptr;
    if (!fields || nfields < 1 || nparts < 1) return MSMB_ERR_CONFIG;
    for (int i = 0; i < nfields; ++i) {
        if (!fields[i] || fields[i]->kind != MSMB_FIELD_MSM || !fields[i]->rep.empty()) return MSMB_ERR_CONFIG;
        for (int j = 0; j < i; ++j)
            if (fields[j] == fields[i]) return MSMB_ERR_CONFIG; // one field (workspace) per part
    }
    // one field: the NCCL transport (also with a single part when an id or communicator is
    // given -- a one-rank communicator exercises the same code path)
    const bool dist = nfields == 1 && (nparts > 1 || nccl_id || nccl_comm);
    if (!dist && nfields != nparts) return MSMB_ERR_CONFIG;
    if (dist && (rank < 0 || rank >= nparts || (!nccl_id && !nccl_comm))) return MSMB_ERR_CONFIG;
    auto g = std::make_unique<msmb_slab>();
    g->nparts = nparts;
    try {
        if (dist) {
            if (nccl_comm) {
                g->comm = static_cast<ncclComm_t>(nccl_comm);
            } else {
                Nccl& N = nccl();
                if (!N.ok) {
                    fields[0]->last = Error{MSMB_ERR_CUDA, -1, -1, -1, "NCCL unavailable: " + N.why};
                    return MSMB_ERR_CUDA;
                }
                ncclUniqueId id;
                std::memcpy(&id, nccl_id, sizeof id);
                cudaSetDevice(fields[0]->device);
                ckn(N.CommInitRank(&g->comm, nparts, id, rank), "ncclCommInitRank");
                g->own_comm = true;
            }
        }
        for (int i = 0; i < nfields; ++i) {
            auto p = std::make_unique<SlabPart>();
            p->f = fields[i];
            p->rank = dist ? rank : i;
            p->nparts = nparts;
            g->parts.push_back(std::move(p));
        }
    } catch (const std::exception& ex) {
        fields[0]->last = Error{MSMB_ERR_CUDA, -1, -1, -1, ex.what()};
        return MSMB_ERR_CUDA;
    }
    *out = g.release();
    return MSMB_OK;
}

void msmb_slab_destroy(msmb_slab* g) {
    if (!g) return;
    for (auto& p : g->parts) {
        cudaSetDevice(p->f->device);
        cudaStreamSynchronize(p->f->stream);
    }
    if (g->own_comm && g->comm) nccl().CommDestroy(g->comm);
    delete g;
}

// propagate(spec, s, units) over the decomposition: every part passes the caller's
// whole system (host AoS, as msmb_propagate); on success every part's pos/vel hold
// the whole final state.  step_ms (optional, steps + 2 entries): device time of the
// initial evaluation, of every step and of the closing kick on this process's first part.
int msmb_slab_propagate(msmb_slab* g, int64_t n, double* pos_xyz, double* vel_xyz, const double* q,
                        const double* mass, const double box[3], double dt, int steps, const msmb_units* units,
                        double* energy, double* step_ms) {
    if (!g) return MSMB_ERR_CONFIG;
    msmb_field* f0 = g->parts[0]->f;
    std::vector<std::unique_lock<std::recursive_mutex>> locks;
    for (auto& p : g->parts) locks.emplace_back(p->f->mu);
    g->last = Error{};
    if (!(dt > 0.0)) return set_err(g, Error{MSMB_ERR_CONFIG, -1, -1, -1, "dt must be > 0"}), MSMB_ERR_CONFIG;
    if (steps < 1)
        return set_err(g, Error{MSMB_ERR_CONFIG, -1, -1, -1, "steps_per_slice must be >= 1"}), MSMB_ERR_CONFIG;
    const msmb_units u = units ? *units : f0->units;
    Error e = validate_units(u);
    if (!e.kind) e = validate_config(f0->cfg);
    if (e.kind) return set_err(g, e), e.kind;
    try {
        std::vector<double> soa(size_t(n) * 8);
        for (int64_t i = 0; i < n; ++i) {
            for (int ax = 0; ax < 3; ++ax) {
                soa[size_t(ax) * n + i] = pos_xyz[3 * i + ax];
                soa[size_t(3 + ax) * n + i] = vel_xyz[3 * i + ax];
            }
            soa[size_t(6) * n + i] = q[i];
            soa[size_t(7) * n + i] = mass[i];
        }
        for (int attempt = 0; attempt < 8; ++attempt) {
            // ---- workspaces, plans, the initial sets
            for (auto& pp : g->parts) {
                SlabPart& p = *pp;
                cks(cudaSetDevice(p.f->device), "cudaSetDevice");
                p.f->dd_nparts = g->nparts;
                p.f->dd_part = p.rank;
                p.f->lattice_direct = g->nparts > 1 ? 1 : p.f->lattice_direct; // owned planes: direct stencil
                Error we = ensure_workspace(p.f, n, box);
                if (we.kind) return set_err(g, we), we.kind;
                p.f->ws->part = make_part(p.f->ws->g, g->nparts, p.rank);
                if (g->nparts > 1 && p.f->ws->lattice_fft) { // a workspace built before: rebuild with the direct method
                    p.f->ws.reset();
                    we = ensure_workspace(p.f, n, box);
                    if (we.kind) return set_err(g, we), we.kind;
                    p.f->ws->part = make_part(p.f->ws->g, g->nparts, p.rank);
                }
                if (p.st.n != n || !p.st.buf.p) cks(p.st.alloc(n), "cudaMalloc state");
                for (int ax = 0; ax < 3; ++ax) p.st.box[ax] = box[ax];
                cks(cudaMemcpyAsync(p.st.buf.p, soa.data(), sizeof(double) * soa.size(), cudaMemcpyHostToDevice,
                                    p.stream()),
                    "H2D");
                const size_t N1 = size_t(n) + 1;
                ensure_buf(p.mark_own, sizeof(int) * N1);
                ensure_buf(p.mark_loc, sizeof(int) * N1);
                ensure_buf(p.scan, sizeof(int) * N1);
                ensure_buf(p.tmp, sizeof(int64_t) * size_t(std::max(64, 16 * g->nparts)));
                ensure_buf(p.ebuf, sizeof(double) * N1);
                ensure_buf(p.dflag, sizeof(int) * 4);
                make_plans(p);
                p.bytes_step = p.bytes_rebuild = p.migrated = 0;
                launch_reset_err(p.stream(), p.W().err, 0);
                // the list of the first evaluation is built fresh (a pure function of the input)
                cks(cudaMemsetAsync(p.W().c.flag + 3, 0, sizeof(int), p.stream()), "memset");
                cks(cudaMemsetAsync(p.W().c.flag + 6, 0, sizeof(int), p.stream()), "memset");
                cks(cudaStreamSynchronize(p.stream()), "sync");
            }
            setup_sets(g);
            select_halos(g);
            // ---- the initial evaluation, then the steps
            std::vector<cudaEvent_t> ev;
            auto stamp = [&]() {
                if (!step_ms) return;
                cudaEvent_t x;
                cudaEventCreate(&x);
                cudaEventRecord(x, g->parts[0]->stream());
                ev.push_back(x);
            };
            stamp();
            evaluate(g, true);
            stamp();
            int64_t bytes_max = 0;
            for (int s = 1; s <= steps; ++s) {
                for (auto& pp : g->parts) {
                    SlabPart& p = *pp;
                    p.bytes_step = 0;
                    Workspace& W = p.W();
                    const double hdc = 0.5 * dt * u.energy_to_native;
                    if (p.n_owned)
                        k_verlet_owned<<<nb256(p.n_owned), 256, 0, p.stream()>>>(
                            p.owned.as<int>(), p.n_owned, p.st.dev(), W.o.fx, W.o.fy, W.o.fz, dt, hdc, s == 1 ? 1 : 2,
                            1, W.err);
                    else
                        k_verlet_owned<<<1, 32, 0, p.stream()>>>(p.owned.as<int>(), 0, p.st.dev(), W.o.fx, W.o.fy,
                                                                 W.o.fz, dt, hdc, 1, 1, W.err);
                    // the rebuild rule of one GPU: some atom moved more than skin/2 since the build
                    cks(cudaMemsetAsync(p.dflag.p, 0, sizeof(int), p.stream()), "memset");
                    const double hs = 0.5 * W.g.skin;
                    if (p.n_owned)
                        k_disp_owned<<<nb256(p.n_owned), 256, 0, p.stream()>>>(
                            p.owned.as<int>(), p.n_owned, p.st.dev().x, p.st.dev().y, p.st.dev().z, W.a.ref, n,
                            hs * hs, p.dflag.as<int>());
                }
                std::vector<int64_t> flags;
                for (auto& pp : g->parts) {
                    int v = 0;
                    cks(cudaMemcpyAsync(&v, pp->dflag.p, sizeof(int), cudaMemcpyDeviceToHost, pp->stream()), "D2H");
                    cks(cudaStreamSynchronize(pp->stream()), "sync");
                    flags.push_back(v || !(pp->W().g.skin > 0.0));
                }
                const bool rebuild = allmax(g, flags) > 0;
                if (rebuild) {
                    ++g->rebuilds;
                    migrate(g);
                    select_halos(g);
                } else {
                    halo_refresh(g);
                }
                evaluate(g, rebuild);
                for (auto& pp : g->parts) bytes_max = std::max(bytes_max, pp->bytes_step);
                stamp();
            }
            for (auto& pp : g->parts) { // the closing half-kick
                SlabPart& p = *pp;
                Workspace& W = p.W();
                if (p.n_owned)
                    k_verlet_owned<<<nb256(p.n_owned), 256, 0, p.stream()>>>(
                        p.owned.as<int>(), p.n_owned, p.st.dev(), W.o.fx, W.o.fy, W.o.fz, dt,
                        0.5 * dt * u.energy_to_native, 1, 0, W.err);
            }
            stamp();
            const ErrRec r = combine_errors(g);
            if (step_ms && !ev.empty()) {
                cudaEventSynchronize(ev.back());
                for (size_t i = 0; i + 1 < ev.size(); ++i) {
                    float ms = 0;
                    cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
                    step_ms[i] = ms;
                }
                for (auto x : ev) cudaEventDestroy(x);
            }
            for (auto& pp : g->parts) {
                pp->f->counters[0] = int64_t(r.pairs / 2);
                pp->f->counters[6] = g->rebuilds;
                pp->bytes_step = bytes_max;
            }
            if (r.kind == kOverflowKind) { // some part's pair list overflowed: grow and redo the call
                for (auto& pp : g->parts)
                    if (pp->rec.kind == kOverflowKind) grow_cap(pp->W(), pp->rec);
                // every part must agree on the retry (the combined record is global)
                continue;
            }
            if (r.kind) return set_err(g, error_from_rec(r)), r.kind;
            // ---- the final state: every part's owned atoms, to everyone
            std::vector<std::vector<int64_t>> cnts;
            for (auto& pp : g->parts) cnts.push_back({pp->n_owned});
            const std::vector<int64_t> all = allgather(g, cnts, 1);
            int64_t tot = 0;
            for (int64_t c : all) tot += c;
            if (tot != n) throw std::runtime_error("slab: owned sets do not partition the system");
            std::vector<double> rec(size_t(tot) * 7);
            if (g->local()) {
                int64_t off = 0;
                for (auto& pp : g->parts) {
                    SlabPart& p = *pp;
                    ensure_buf(p.xsend, sizeof(double) * 7 * size_t(std::max<int64_t>(p.n_owned, 1)));
                    if (p.n_owned)
                        k_pack<<<nb256(p.n_owned), 256, 0, p.stream()>>>(p.owned.as<int>(), p.n_owned, p.st.dev(), 6,
                                                                         p.xsend.as<double>());
                    cks(cudaMemcpyAsync(rec.data() + 7 * off, p.xsend.p, sizeof(double) * 7 * size_t(p.n_owned),
                                        cudaMemcpyDeviceToHost, p.stream()),
                        "D2H");
                    cks(cudaStreamSynchronize(p.stream()), "sync");
                    off += p.n_owned;
                }
            } else {
                SlabPart& p = *g->parts[0];
                cudaStream_t st = p.stream();
                int64_t mx = 0;
                for (int64_t c : all) mx = std::max(mx, c);
                ensure_buf(p.xsend, sizeof(double) * 7 * size_t(std::max<int64_t>(mx, 1)));
                ensure_buf(p.xrecv, sizeof(double) * 7 * size_t(std::max<int64_t>(mx, 1)) * size_t(g->nparts));
                cks(cudaMemsetAsync(p.xsend.p, 0, sizeof(double) * 7 * size_t(mx), st), "memset");
                if (p.n_owned)
                    k_pack<<<nb256(p.n_owned), 256, 0, st>>>(p.owned.as<int>(), p.n_owned, p.st.dev(), 6,
                                                             p.xsend.as<double>());
                ckn(nccl().AllGather(p.xsend.p, p.xrecv.p, size_t(7 * mx), ncclDouble, g->comm, st), "AllGather");
                std::vector<double> h(size_t(7 * mx) * size_t(g->nparts));
                cks(cudaMemcpyAsync(h.data(), p.xrecv.p, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, st), "D2H");
                cks(cudaStreamSynchronize(st), "sync");
                int64_t off = 0;
                for (int r2 = 0; r2 < g->nparts; ++r2) {
                    std::memcpy(rec.data() + 7 * off, h.data() + size_t(r2) * 7 * mx, sizeof(double) * 7 * size_t(all[size_t(r2)]));
                    off += all[size_t(r2)];
                }
            }
            for (int64_t t = 0; t < tot; ++t) {
                const double* x = rec.data() + 7 * t;
                const int64_t i = int64_t(x[0]);
                for (int ax = 0; ax < 3; ++ax) {
                    pos_xyz[3 * i + ax] = x[1 + ax];
                    vel_xyz[3 * i + ax] = x[4 + ax];
                }
            }
            // the energy of the last evaluation: the parts' shares summed in rank order
            std::vector<std::vector<int64_t>> es;
            for (auto& pp : g->parts) {
                double ev2 = 0;
                cks(cudaMemcpyAsync(&ev2, pp->W().o.energy, sizeof(double), cudaMemcpyDeviceToHost, pp->stream()), "D2H");
                cks(cudaStreamSynchronize(pp->stream()), "sync");
                int64_t bits;
                std::memcpy(&bits, &ev2, sizeof bits);
                es.push_back({bits});
            }
            const std::vector<int64_t> eall = allgather(g, es, 1);
            double esum = 0.0;
            for (int64_t b : eall) {
                double v;
                std::memcpy(&v, &b, sizeof v);
                esum += v;
            }
            if (energy) *energy = esum;
            return MSMB_OK;
        }
        return set_err(g, Error{MSMB_ERR_INTERNAL, -1, -1, -1, "pair list did not converge"}), MSMB_ERR_INTERNAL;
    } catch (const std::exception& ex) {
        set_err(g, Error{MSMB_ERR_CUDA, -1, -1, -1, ex.what()});
        return MSMB_ERR_CUDA;
    }
}

// [0] bytes received per step (max over steps and this process's parts), [1] bytes of
// the last rebuild exchanges, [2] owned atoms, [3] halo atoms (first part), [4]
// rebuilds, [5] migrated atoms (this process), [6] parts
int msmb_slab_stats(msmb_slab* g, int64_t* out, int cap) {
    if (!g || !out) return 0;
    const SlabPart& p = *g->parts[0];
    int64_t mig = 0, rb = 0;
    for (auto& pp : g->parts) mig += pp->migrated, rb = std::max(rb, pp->bytes_rebuild);
    const int64_t v[7] = {p.bytes_step, rb, p.n_owned, p.n_local - p.n_owned, g->rebuilds, mig, g->nparts};
    const int k = std::min(cap, 7);
    for (int i = 0; i < k; ++i) out[i] = v[i];
    return k;
}

int msmb_slab_last_error(const msmb_slab* g, int* kind, int64_t* idx_i, int64_t* idx_j, int* step, char* msg, int cap) {
    if (!g) return MSMB_ERR_CONFIG;
    return msmb_last_error(g->parts[0]->f, kind, idx_i, idx_j, step, msg, cap);
}

} // extern "C"
