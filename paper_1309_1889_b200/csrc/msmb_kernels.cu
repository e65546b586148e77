// sm_100a kernels for the MSM force / velocity-Verlet / parareal hot path.
//
// Stage map (reference file:line -> kernel):
//   K1  bin + counting sort          src/msm_phases.cpp:21-29 (stencil_at base), msm.cpp:25-27
//                                    -> k_bin, k_sort_decide, k_scan_block/add, k_scatter, k_cellsort (+ coincidence)
//   K2  short-range pairs            src/msm_phases.cpp:224-252, msm_kernels.hpp:30-42
//                                    -> k_flag_reset, k_disp, k_cl_gather (+ out-of-grid pair errors),
//                                       k_colscan, k_bbox, k_pairlist, k_pairmask (rebuilds), k_pairs_mw
//   K3  anterpolation                src/msm_phases.cpp:39-61      -> k_anterp_tile, k_anterp_combine
//   K4  restriction                  src/msm_phases.cpp:63-91      -> k_restrict_tile
//   K5  lattice cutoff               src/msm_phases.cpp:93-134     -> msmb_fft.cu (k_fft_x/y/z); k_lattice (direct)
//   K6  top level                    src/msm_phases.cpp:136-162    -> k_top_warp (FFT job for large tops)
//   K7  prolongation                 src/msm_phases.cpp:164-193    -> k_prolong_tile
//   K8  interpolation + forces + E   src/msm_phases.cpp:195-222, src/msm.cpp:16-48,69-86
//                                    -> k_interp, k_energy1/2, k_finalize
//   K9  velocity Verlet              src/integrate.cpp:23-34       -> k_kick_drift, k_kick
//   K10 parareal state algebra       src/parareal.cpp:58-90        -> msmb_parareal.cu
// Determinism: no floating-point atomics anywhere; every sum has a fixed order.
// Arithmetic that must reproduce the reference bit for bit (cell keys, stencil
// weights, restriction/prolongation/interpolation given equal lattices, Verlet)
// uses explicit round-to-nearest intrinsics (__dmul_rn/__dadd_rn/...), which
// nvcc never contracts into FMA.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstdlib>

#include <map>
#include <mutex>
#include <type_traits>
#include <utility>

#include "msmb_kernels.cuh"

namespace msmb {

cudaError_t smem_grow(const void* func, size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, size_t> cur;
    int dev = 0;
    cudaGetDevice(&dev);
    const size_t want = std::max<size_t>(bytes, 48 * 1024);
    std::lock_guard<std::mutex> lk(mu);
    size_t& have = cur[{dev, func}];
    if (want <= have) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, int(want));
    if (e == cudaSuccess) have = want;
    return e;
}

#define FULLMASK 0xffffffffu

// anterpolation by per-block shared-memory tiles (k_anterp_tile) computing the weights
// itself; 0 = the per-point gather kernels over k_gather's precomputed weights
#ifndef MSMB_ANTERP_TILE
#define MSMB_ANTERP_TILE 1
#endif

// threads per block of the per-atom kernels: small systems (C1: 8,192 atoms) get
// 64-thread blocks so they spread over more SMs (latency-bound, not throughput-bound)
#ifndef MSMB_ATOM_TPB
#define MSMB_ATOM_TPB 256
#endif
static inline int atom_tpb(int64_t n) { return n < 148 * 1024 ? 64 : MSMB_ATOM_TPB; }
static inline int atom_blocks(int64_t n, int tpb) { return int((n + tpb - 1) / tpb) > 0 ? int((n + tpb - 1) / tpb) : 1; }

__device__ __forceinline__ bool failed(const ErrRec* e) {
    // L2 (GPU-coherent) load: kernel boundaries order it after earlier kernels'
    // writes; a stale value inside a kernel only delays an early exit.  (A volatile
    // read compiles to a system-scope LDG.STRONG.SYS, which every thread would pay.)
    return __ldcg(&e->kind) != 0;
}

// basis_phi / basis_phi_deriv (include/paramd/msm_kernels.hpp:71-92), reference op order.
__device__ __forceinline__ double phi_rn(double xi) {
    const double t = fabs(xi);
    if (t >= 2.0) return 0.0;
    if (t <= 1.0)
        return __dadd_rn(1.0, __dmul_rn(__dmul_rn(t, t), __dadd_rn(-2.5, __dmul_rn(1.5, t))));
    const double u = __dsub_rn(2.0, t);
    return __dmul_rn(__dmul_rn(__dmul_rn(-0.5, __dsub_rn(t, 1.0)), u), u);
}

__device__ __forceinline__ double dphi_rn(double xi) {
    const double t = fabs(xi);
    double d;
    if (t >= 2.0)
        d = 0.0;
    else if (t <= 1.0)
        d = __dmul_rn(t, __dadd_rn(-5.0, __dmul_rn(4.5, t)));
    else
        d = __dmul_rn(__dmul_rn(-0.5, __dsub_rn(2.0, t)), __dsub_rn(4.0, __dmul_rn(3.0, t)));
    return xi < 0.0 ? -d : d;
}

struct BinP {
    double o[3];
    double inv_h;
    int d[3];
    int cw, ncx, ncy;
    int clamp;      // pair-only fields: no coverage, cells clamped to 1 .. d-3
};

static float float_ru(double x) { // host: smallest float >= x
    float f = float(x);
    if (double(f) < x) f = std::nextafter(f, 3e38f);
    return f;
}

static BinP make_binp(const Geometry& g) {
    BinP p;
    for (int ax = 0; ax < 3; ++ax) {
        p.o[ax] = g.lv[0].origin[ax];
        p.d[ax] = g.lv[0].dims[ax];
    }
    p.inv_h = g.inv_h0;
    p.cw = g.cw;
    p.ncx = g.ncx;
    p.ncy = g.ncy;
    p.clamp = g.kind != MSMB_FIELD_MSM;
    return p;
}

__device__ __forceinline__ int scell_of(const BinP& p, int cx, int cy, int cz) {
    const int col = (cx / p.cw) * p.ncy + (cy / p.cw);
    return ((col * p.d[2] + cz) * p.cw + (cx % p.cw)) * p.cw + (cy % p.cw);
}

// ============================================================================
// K1: binning (bit-exact level-0 cell triple) + stable counting sort
// ============================================================================
// list != nullptr: bin only the atoms list[0..n) (a spatial-decomposition part's
// owned + halo atoms, msmb_slab.cu); the others keep no key
__global__ void k_bin(int n, const double* __restrict__ x, const double* __restrict__ y,
                      const double* __restrict__ z, BinP p, int* key, int* rank, int* count,
                      int* outlist, ErrRec* err, const int* __restrict__ list, int* moved) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); // k_flag_reset may be admitted (pdl_enter)
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n || failed(err)) return;
    const int i = list ? list[t] : t;
    const double px[3] = {x[i], y[i], z[i]};
    int c[3];
    bool ok = true;
    if (p.clamp) { // pair-only fields: any position is valid; the cell is clamped
        bool nan = false, inf = false;
        for (int ax = 0; ax < 3; ++ax) {
            const double t = __dmul_rn(__dsub_rn(px[ax], p.o[ax]), p.inv_h);
            nan |= isnan(px[ax]);
            inf |= isinf(px[ax]);
            const double f = fmin(fmax(floor(t), 1.0), double(p.d[ax]) - 3.0); // NaN -> 1
            c[ax] = int(f);
        }
        if (inf && !nan) { // rejected (msmb.h): excluded from the cells, reported as DomainError
            if (key[i] != -1) *moved = 1;
            key[i] = -1;
            atomicMin(&err->cov_min, (long long)i);
            const int slot = atomicAdd(&err->cov_count, 1);
            outlist[slot] = i;
            return;
        }
        if (nan) atomicAdd(&err->nan_count, 1);
        if (nan) c[0] = c[1] = c[2] = 1;
        const int sc = scell_of(p, c[0], c[1], c[2]);
        if (key[i] != sc) *moved = 1;
        key[i] = sc;
        rank[i] = atomicAdd(&count[sc], 1);
        return;
    }
    for (int ax = 0; ax < 3; ++ax) {
        // t = (r - origin) * inv_h; base = floor(t) - 1 (src/msm_phases.cpp:23,42-50)
        const double t = __dmul_rn(__dsub_rn(px[ax], p.o[ax]), p.inv_h);
        const double f = floor(t);
        // covered iff 0 <= base && base + 3 <= dims - 1 (src/msm_phases.cpp:24)
        ok = ok && (f >= 1.0) && (f <= double(p.d[ax]) - 3.0);
        c[ax] = ok ? int(f) : 0;
    }
    if (!ok) {
        if (key[i] != -1) *moved = 1;
        key[i] = -1;
        atomicMin(&err->cov_min, (long long)i);
        const int slot = atomicAdd(&err->cov_count, 1);
        outlist[slot] = i;
        return;
    }
    const int sc = scell_of(p, c[0], c[1], c[2]);
    if (key[i] != sc) *moved = 1;
    key[i] = sc;
    rank[i] = atomicAdd(&count[sc], 1);
}

// exclusive scan of int[m] (m = cells + 1), 4096 elements per block
// gate (optional): skip when gate[0] == 0 (the cell sort of k_bin_decide is reused)
__global__ void __launch_bounds__(1024) k_scan_block(const int* __restrict__ in, int* out,
                                                     int* bsum, int64_t m, const int* __restrict__ gate) {
    __shared__ int wsum[32];
    pdl_enter(gridDim.x <= kPdlEarlyMaxBlocks); // k_scan_add has the same grid
    if (gate && !*gate) return;
    const int64_t base = int64_t(blockIdx.x) * 4096 + threadIdx.x * 4;
    int v[4];
    int s = 0;
    for (int k = 0; k < 4; ++k) {
        v[k] = (base + k < m) ? in[base + k] : 0;
        s += v[k];
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int inc = s;
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(FULLMASK, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    if (w == 0) {
        int ws = wsum[lane];
        int wi = ws;
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(FULLMASK, wi, o);
            if (lane >= o) wi += t;
        }
        wsum[lane] = wi - ws;
        if (lane == 31) bsum[blockIdx.x] = wi;
    }
    __syncthreads();
    int run = inc - s + wsum[w];
    for (int k = 0; k < 4; ++k) {
        if (base + k < m) out[base + k] = run;
        run += v[k];
    }
}

// second pass: block b adds the sum of the blocks before it (it reduces bsum[0..b)
// itself: one launch instead of a block-sum scan and an add; at most a few thousand
// block sums even for C3's 11M cells)
__global__ void __launch_bounds__(1024) k_scan_add(int* out, const int* __restrict__ bsum, int64_t m,
                                                   const int* __restrict__ gate) {
    __shared__ int wsum[32];
    pdl_enter();
    if (gate && !*gate) return;
    const int b = blockIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int v = 0;
    for (int k = threadIdx.x; k < b; k += 1024) v += bsum[k];
    v = __reduce_add_sync(FULLMASK, v);
    if (lane == 0) wsum[w] = v;
    __syncthreads();
    const int off = __reduce_add_sync(FULLMASK, wsum[lane]);
    if (off == 0) return;
    const int64_t base = int64_t(b) * 4096;
    for (int k = threadIdx.x; k < 4096; k += 1024)
        if (base + k < m) out[base + k] += off;
}

static int scan_exclusive(cudaStream_t st, const int* in, int* out, int* tmp, int64_t m,
                          const int* gate = nullptr) {
    const int nb = int((m + 4095) / 4096);
    pdl_launch(k_scan_block, dim3(nb), dim3(1024), 0, st, in, out, tmp, m, gate);
    pdl_launch(k_scan_add, dim3(nb), dim3(1024), 0, st, out, tmp, m, gate);
    return 2;
}

// Cell-sort reuse: k_bin sets flag[5] when some atom's cell key differs from its key
// of the previous evaluation; flag[6] says the sorted structures (start, perm, nat)
// are those of the current keys' cells.  The sort runs only when needed (flag[7]);
// between list rebuilds atoms rarely change cells, and the sorted order of the same
// keys is the same order (within a cell: ascending index), so results are unchanged.
__global__ void k_sort_decide(int* flag) {
    pdl_enter(1);
    const int need = flag[5] || !flag[6];
    flag[7] = need;
    flag[6] = 1;
    flag[5] = 0; // for the next evaluation's k_bin (a launch_bin without a sort after it
                 // leaves it set: the next sort then runs, which is always correct)
}

int launch_scan_exclusive(cudaStream_t st, const int* in, int* out, int* tmp, int64_t m) {
    return scan_exclusive(st, in, out, tmp, m);
}

__global__ void k_scatter(int n, const int* __restrict__ key, const int* __restrict__ rank,
                          const int* __restrict__ start, int* perm, const ErrRec* err,
                          const int* __restrict__ list, const int* __restrict__ gate) {
    pdl_enter();
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n || failed(err) || !*gate) return;
    const int i = list ? list[t] : t;
    const int k = key[i];
    if (k >= 0) perm[start[k] + rank[i]] = i;
}

// within-cell order = ascending original index (deterministic; cells are small);
// also publishes each level-0 cell's range in natural (x, y, z) row-major order
__device__ void cell_sort_one(int64_t c, const BinP& p, int s0, int s1, int* perm, int2* nat) {
    {
        int64_t t = c;
        const int oy = int(t % p.cw);
        t /= p.cw;
        const int ox = int(t % p.cw);
        t /= p.cw;
        const int cz = int(t % p.d[2]);
        const int col = int(t / p.d[2]);
        const int cx = (col / p.ncy) * p.cw + ox, cy = (col % p.ncy) * p.cw + oy;
        if (cx < p.d[0] && cy < p.d[1]) nat[(size_t(cx) * p.d[1] + cy) * p.d[2] + cz] = make_int2(s0, s1);
    }
    for (int a = s0 + 1; a < s1; ++a) {
        const int v = perm[a];
        int b = a - 1;
        while (b >= s0 && perm[b] > v) {
            perm[b + 1] = perm[b];
            --b;
        }
        perm[b + 1] = v;
    }
}

// thread per cell: the cell sort (when gate) and, with coincide, the exact-coincidence
// check of every pair of atoms sharing the cell (src/msm_phases.cpp:237-239; the same
// pairs as coincide_check) in every evaluation -- positions change even when the sort
// is reused.  One launch instead of a cell sort and a per-atom check.
__global__ void k_cellsort(int64_t ncells, BinP p, const int* __restrict__ start, int* perm,
                           int2* nat, const double* __restrict__ x, const double* __restrict__ y,
                           const double* __restrict__ z, ErrRec* err, const int* __restrict__ gate,
                           int coincide) {
    pdl_enter();
    const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (c >= ncells || failed(err)) return;
    const int s0 = start[c], s1 = start[c + 1];
    if (*gate) cell_sort_one(c, p, s0, s1, perm, nat);
    if (!coincide) return;
    for (int a = s0; a + 1 < s1; ++a) {
        const int i = perm[a];
        const double px = x[i], py = y[i], pz = z[i];
        for (int b = a + 1; b < s1; ++b) {
            const int j = perm[b];
            if (x[j] == px && y[j] == py && z[j] == pz) {
                const unsigned long long k = ((unsigned long long)min(i, j) << 32) | (unsigned long long)max(i, j);
                atomicMin(&err->pair_key, k);
            }
        }
    }
}

// exactly coincident particles (r2 == 0, src/msm_phases.cpp:237-239) share a cell: every
// evaluation compares each sorted atom with the later atoms of its cell (cells hold
// ~1-2 atoms); runs whether or not the cell sort was reused
__device__ __forceinline__ void coincide_check(int s, int i, const int* __restrict__ key,
                                               const int* __restrict__ start, const int* __restrict__ perm,
                                               const double* __restrict__ x, const double* __restrict__ y,
                                               const double* __restrict__ z, ErrRec* err) {
    const int s1 = start[key[i] + 1];
    const double px = x[i], py = y[i], pz = z[i];
    for (int b = s + 1; b < s1; ++b) {
        const int j = perm[b];
        if (x[j] == px && y[j] == py && z[j] == pz) {
            const unsigned long long k = ((unsigned long long)min(i, j) << 32) | (unsigned long long)max(i, j);
            atomicMin(&err->pair_key, k);
        }
    }
}


// the anterpolation weights of particle i: o[0..3] = q*wx[d], o[4..7] = wy[d], o[8..11] =
// wz[d], exactly as anterpolate's qa / w (msm_phases.cpp:42-53)
__device__ __forceinline__ void anterp_weights(const BinP& p, double px, double py, double pz, double qq,
                                               double* o) {
    const double pp[3] = {px, py, pz};
    double w[3][4];
    for (int ax = 0; ax < 3; ++ax) {
        const double t = __dmul_rn(__dsub_rn(pp[ax], p.o[ax]), p.inv_h);
        const int base = int(floor(t)) - 1;
        for (int d = 0; d < 4; ++d) w[ax][d] = phi_rn(__dsub_rn(t, double(base + d)));
    }
    for (int d = 0; d < 4; ++d) {
        o[d] = __dmul_rn(qq, w[0][d]);
        o[4 + d] = w[1][d];
        o[8 + d] = w[2][d];
    }
}

// sorted copies + the anterpolation weights of every particle:
// aw = {q*wx[0..3], wy[0..3], wz[0..3]} exactly as anterpolate's qa / w (msm_phases.cpp:45-53)
__global__ void k_gather(int n, const int* __restrict__ start_total, const int* __restrict__ perm,
                         const double* __restrict__ x, const double* __restrict__ y,
                         const double* __restrict__ z, const double* __restrict__ q, BinP p,
                         double* aw, ErrRec* err, const int* __restrict__ key, const int* __restrict__ start) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= *start_total || failed(err)) return;
    const int i = perm[s];
    coincide_check(s, i, key, start, perm, x, y, z, err);
    anterp_weights(p, x[i], y[i], z[i], q[i], aw + size_t(s) * 12);
}

int launch_bin(cudaStream_t st, const Geometry& g, const DevState& s, DevAtoms& a, DevCells& c,
               ErrRec* err, const int* list, int64_t nlist) {
    const int n = list ? int(nlist) : int(s.n);
    cudaMemsetAsync(c.count, 0, sizeof(int) * size_t(g.ncells + 1), st); // flag[5]: see k_sort_decide
    if (n > 0)
        k_bin<<<atom_blocks(n, atom_tpb(n)), atom_tpb(n), 0, st>>>(n, s.x, s.y, s.z, make_binp(g), a.key, a.rank,
                                               c.count, a.outlist, err, list, c.flag + 5);
    return n > 0 ? 1 : 0;
}

int launch_sort(cudaStream_t st, const Geometry& g, const DevState& s, DevAtoms& a, DevCells& c,
                ErrRec* err, const int* list, int64_t nlist) {
    const int n = list ? int(nlist) : int(s.n);
    pdl_launch(k_sort_decide, dim3(1), dim3(1), 0, st, c.flag);
    const int* gate = c.flag + 7;
    int l = 1 + scan_exclusive(st, c.count, c.start, c.scan_tmp, g.ncells + 1, gate);
    if (n > 0)
        pdl_launch(k_scatter, dim3(atom_blocks(n, atom_tpb(n))), dim3(atom_tpb(n)), 0, st, n, a.key, a.rank, c.start,
                   a.perm, err, list, gate);
    // also publishes the (possibly empty) natural-order cell ranges read by k_anterp;
    // without precomputed anterpolation weights (k_gather) it runs the coincidence check
    const bool weights = g.kind == MSMB_FIELD_MSM && !MSMB_ANTERP_TILE;
    pdl_launch(k_cellsort, dim3(int((g.ncells + 255) / 256)), dim3(256), 0, st, g.ncells, make_binp(g), c.start, a.perm,
               c.nat, s.x, s.y, s.z, err, gate, weights ? 0 : 1);
    if (n == 0 || !weights) return l + 1;
    k_gather<<<atom_blocks(n, atom_tpb(n)), atom_tpb(n), 0, st>>>(n, c.start + g.ncells, a.perm, s.x, s.y, s.z, s.q,
                                              make_binp(g), a.aw, err, a.key, c.start);
    return l + 3;
}

// ============================================================================
// K2: short-range pairs.  Columns of cw x cw level-0 cells; 32 consecutive
// sorted atoms of a column form a cluster; one warp per i-cluster walks the
// list of j-clusters whose bounding boxes are within the cutoff.
// ============================================================================
// ---- pair-list (Verlet skin) bookkeeping.  flag[0]: rebuild the cluster pair list
// in this evaluation (forced, or some atom moved more than skin/2 since the last
// rebuild); flag[1]: atoms in the cluster order.  Between rebuilds the clusters keep
// their atoms (cl_perm) and only the positions are gathered anew; the pair kernel
// screens with the exact cutoff, so the frozen list only has to be a superset.
// flag[0] = rebuild the pair list in this evaluation: forced, or no valid list
// (flag[3] == 0: never built, capacity grown, an evaluation failed), or the list was
// built for another ownership range (flag[4]: the part's pair-column key)
__global__ void k_flag_reset(int* flag, int force, int key) {
    pdl_enter(1);
    flag[0] = (force || flag[3] == 0 || flag[4] != key) ? 1 : 0;
}

__global__ void k_disp(int64_t n, const double* __restrict__ x, const double* __restrict__ y,
                       const double* __restrict__ z, const double* __restrict__ ref, double half_skin2,
                       int* flag) {
    pdl_enter(1);
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double dx = x[i] - ref[i], dy = y[i] - ref[n + i], dz = z[i] - ref[2 * n + i];
    if (!(dx * dx + dy * dy + dz * dz <= half_skin2)) flag[0] = 1; // same value from every writer
}

__device__ void err_brute_blocks(int64_t n, const double* __restrict__ x, const double* __restrict__ y,
                                 const double* __restrict__ z, const int* __restrict__ outlist, ErrRec* err,
                                 int b, int nb);

// Cluster-order positions, every evaluation: slot s of the frozen cluster order holds
// atom cl_perm[s]; at a rebuild (flag[0]) the order is first re-frozen from the cell
// sort (cl_perm = perm, its inverse, the reference positions of the skin test).
// Blocks past the atom range run the out-of-grid pair-error search (k_err_brute's
// grid-stride loop; it exits at once unless k_bin counted atoms outside coverage):
// one launch instead of three on a skin step.
__global__ void k_cl_gather(int64_t n, const int* __restrict__ start_total, const int* __restrict__ perm,
                            const double* __restrict__ x, const double* __restrict__ y,
                            const double* __restrict__ z, const double* __restrict__ q, int* cl_perm, int* cl_inv,
                            double* ref, int* flag, int key, double* xc, double* yc, double* zc, double* qc,
                            int gather_blocks, const int* __restrict__ outlist, ErrRec* err, int mode) {
    pdl_enter(1);
    // mode 1: the skin evaluations' gather only (exits at a rebuild), mode 2: the rebuild's only
    if (mode && (flag[0] != 0) != (mode == 2)) {
        if (mode == 2 || int(blockIdx.x) < gather_blocks) return;
    }
    if (int(blockIdx.x) >= gather_blocks) {
        err_brute_blocks(n, x, y, z, outlist, err, blockIdx.x - gather_blocks, gridDim.x - gather_blocks);
        return;
    }
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (failed(err)) return;
    int i;
    if (flag[0]) {
        const int tot = *start_total;
        if (s == 0) {
            flag[1] = tot;
            flag[2] += 1; // rebuilds since the workspace was created (diagnostics)
            flag[3] = 1;  // valid until the host invalidates it (capacity growth, errors)
            flag[4] = key;
        }
        if (s >= tot) return;
        i = perm[s];
        cl_perm[s] = i;
        cl_inv[i] = s;
        ref[i] = x[i];
        ref[n + i] = y[i];
        ref[2 * n + i] = z[i];
    } else {
        if (s >= flag[1]) return;
        i = cl_perm[s];
    }
    xc[s] = x[i];
    yc[s] = y[i];
    zc[s] = z[i];
    qc[s] = q[i];
}

// Columns -> clusters (rebuild evaluations only), one block: clusters per column
// (32 consecutive sorted atoms each), their exclusive scan col_off, then the
// clusters (first sorted slot, count), the columns' first slots and the total.
// One launch instead of five (columns, a three-kernel scan, clusters): on skin steps
// they only read flag[0] and exit.
__global__ void __launch_bounds__(1024)
    k_colscan(int64_t ncols, int cells_per_col, const int* __restrict__ start, int* col_cnt, int* col_off,
              int2* clu, int* nclu, int* colstart, const int* __restrict__ flag, const ErrRec* err) {
    if (failed(err) || !flag[0]) return;
    __shared__ int s_w[32];
    __shared__ int s_carry;
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    if (t == 0) s_carry = 0;
    __syncthreads();
    for (int64_t base = 0; base <= ncols; base += 1024) {
        const int64_t col = base + t;
        int cnt = 0;
        if (col < ncols) cnt = (start[(col + 1) * cells_per_col] - start[col * cells_per_col] + 31) / 32;
        if (col <= ncols) col_cnt[col] = cnt;
        int v = cnt; // inclusive warp scan, then across warps
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(FULLMASK, v, o);
            if (lane >= o) v += u;
        }
        if (lane == 31) s_w[w] = v;
        __syncthreads();
        if (w == 0) {
            int x = s_w[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int u = __shfl_up_sync(FULLMASK, x, o);
                if (lane >= o) x += u;
            }
            s_w[lane] = x;
        }
        __syncthreads();
        const int carry = s_carry;
        const int excl = carry + (w > 0 ? s_w[w - 1] : 0) + v - cnt;
        if (col <= ncols) col_off[col] = excl;
        if (col < ncols) {
            const int s0 = start[col * cells_per_col];
            colstart[col] = s0;
            const int na = start[(col + 1) * cells_per_col] - s0;
            for (int k = 0; 32 * k < na; ++k) clu[excl + k] = make_int2(s0 + 32 * k, min(32, na - 32 * k));
        }
        if (col == ncols) {
            *nclu = excl;
            colstart[ncols] = start[ncols * cells_per_col];
        }
        __syncthreads();
        if (t == 0) s_carry = carry + s_w[31];
        __syncthreads();
    }
}

__global__ void k_bbox(const int* __restrict__ nclu, const int2* __restrict__ clu,
                       const double* __restrict__ xs, const double* __restrict__ ys,
                       const double* __restrict__ zs, float4* blo, float4* bhi,
                       const int* __restrict__ flag, const ErrRec* err) {
    const int ic = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (ic >= *nclu || failed(err) || !flag[0]) return;
    const int2 c = clu[ic];
    float lo[3] = {3e38f, 3e38f, 3e38f}, hi[3] = {-3e38f, -3e38f, -3e38f};
    if (lane < c.y) {
        const double p[3] = {xs[c.x + lane], ys[c.x + lane], zs[c.x + lane]};
        for (int ax = 0; ax < 3; ++ax) {
            lo[ax] = __double2float_rd(p[ax]);
            hi[ax] = __double2float_ru(p[ax]);
        }
    }
    for (int o = 16; o; o >>= 1)
        for (int ax = 0; ax < 3; ++ax) {
            lo[ax] = fminf(lo[ax], __shfl_xor_sync(FULLMASK, lo[ax], o));
            hi[ax] = fmaxf(hi[ax], __shfl_xor_sync(FULLMASK, hi[ax], o));
        }
    if (lane == 0) {
        blo[ic] = make_float4(lo[0], lo[1], lo[2], 0.f);
        bhi[ic] = make_float4(hi[0], hi[1], hi[2], 0.f);
    }
}

struct ListP {
    double ox, oy;   // level-0 origin (x, y)
    double colw;     // column width (A)
    int ncx, ncy;
    float cut, cut2;
    double oz, h;    // level-0 origin z, spacing: z-layer window of a column
    int d2, cw;      // z-layers, level-0 cells per column side
    // pair-only fields (clamped binning): atoms outside the box sit in the boundary
    // cells, so the boundary columns / layers extend to infinity
    int clamp, cxmin, cxmax, cymin, cymax, czmin, czmax;
};

__device__ __forceinline__ float gapf(float alo, float ahi, float blo, float bhi) {
    return fmaxf(0.f, fmaxf(blo - ahi, alo - bhi));
}

// Pair list of one i-cluster (one warp): every j-cluster whose fp32 bounding box
// is within the screening cut.  The order is chosen for k_pairs' lane balance:
// columns are visited in mirror groups (|dx|, |dy|) around the i-cluster's
// column, and the (up to 4) columns of a group are interleaved cluster by
// cluster, every other column in reverse z order.  A j-cluster above-left of the
// i-cluster (busy for its upper-left lanes) is thereby followed by one
// below-right (busy for the other lanes), so k_pairs' two-cluster ring keeps
// most lanes busy.  Order only affects speed: the list is complete either way.
constexpr int kListSeg = 128; // group segments longer than this keep column order

__global__ void __launch_bounds__(256)
    k_pairlist(const int* __restrict__ nclu, const float4* __restrict__ blo,
               const float4* __restrict__ bhi, const int* __restrict__ col_off,
               const int* __restrict__ start, ListP p, int* plist, int* pcnt, int cap, int col_a, int col_b,
               const int* __restrict__ flag, ErrRec* err) {
    __shared__ int s_seg[8][kListSeg];
    const int ic = col_off[col_a] + ((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    if (ic >= col_off[col_b] || failed(err) || !flag[0]) return;
    const float4 lo = blo[ic], hi = bhi[ic];
    const double cutd = double(p.cut);
    int cx0 = int(floor((double(lo.x) - cutd - p.ox) / p.colw)) - 1;
    int cx1 = int(floor((double(hi.x) + cutd - p.ox) / p.colw)) + 1;
    int cy0 = int(floor((double(lo.y) - cutd - p.oy) / p.colw)) - 1;
    int cy1 = int(floor((double(hi.y) + cutd - p.oy) / p.colw)) + 1;
    const int xmn = p.clamp ? p.cxmin : 0, xmx = p.clamp ? p.cxmax : p.ncx - 1;
    const int ymn = p.clamp ? p.cymin : 0, ymx = p.clamp ? p.cymax : p.ncy - 1;
    cx0 = min(max(cx0, xmn), xmx);
    cy0 = min(max(cy0, ymn), ymx);
    cx1 = max(min(cx1, xmx), xmn);
    cy1 = max(min(cy1, ymx), ymn);
    const int cxi = min(max(int(floor((0.5 * (double(lo.x) + double(hi.x)) - p.ox) / p.colw)), xmn), xmx);
    const int cyi = min(max(int(floor((0.5 * (double(lo.y) + double(hi.y)) - p.oy) / p.colw)), ymn), ymx);
    const int DX = max(cxi - cx0, cx1 - cxi), DY = max(cyi - cy0, cy1 - cyi);
    // z-layers that can hold atoms within the cut (one extra layer each side):
    // within a column the sorted atoms are ordered by z-layer, so the window is
    // one atom range per column, i.e. one contiguous range of its clusters
    int czA = max(0, int(floor((double(lo.z) - cutd - p.oz) / p.h)) - 1);
    int czB = min(p.d2 - 1, int(floor((double(hi.z) + cutd - p.oz) / p.h)) + 1);
    if (p.clamp) {
        czA = min(max(czA, p.czmin), p.czmax);
        czB = min(max(czB, p.czmin), p.czmax);
    }
    const int lay = p.cw * p.cw;
    const int64_t cpc = int64_t(p.d2) * lay;
    const float oxf = float(p.ox), oyf = float(p.oy), colwf = float(p.colw);
    int count = 0;
    int* out = plist + size_t(ic) * cap;
    for (int dx = 0; dx <= DX; ++dx)
        for (int dy = 0; dy <= DY; ++dy) {
            const int gstart = count;
            int nseg[4] = {0, 0, 0, 0};
            int ncol = 0;
            // (-dx,-dy), (+dx,+dy), (-dx,+dy), (+dx,-dy); duplicates dropped when dx or dy is 0
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const int sx = (v == 0 || v == 2) ? -1 : 1, sy = (v == 0 || v == 3) ? -1 : 1;
                if ((dx == 0 && sx > 0) || (dy == 0 && sy > 0)) continue;
                const int cx = cxi + sx * dx, cy = cyi + sy * dy;
                int emitted = 0;
                if (cx >= cx0 && cx <= cx1 && cy >= cy0 && cy <= cy1) {
                    // column bounds in fp32 (error ~1e-5 A, inside the 1e-3 A margin)
                    float xlo = fmaf(float(cx), colwf, oxf) - 1e-3f, xhi = fmaf(float(cx + 1), colwf, oxf) + 1e-3f;
                    float ylo = fmaf(float(cy), colwf, oyf) - 1e-3f, yhi = fmaf(float(cy + 1), colwf, oyf) + 1e-3f;
                    if (p.clamp) {
                        if (cx <= p.cxmin) xlo = -3e38f;
                        if (cx >= p.cxmax) xhi = 3e38f;
                        if (cy <= p.cymin) ylo = -3e38f;
                        if (cy >= p.cymax) yhi = 3e38f;
                    }
                    const float gx = gapf(lo.x, hi.x, xlo, xhi), gy = gapf(lo.y, hi.y, ylo, yhi);
                    if (gx * gx + gy * gy < p.cut2) {
                        const int col = cx * p.ncy + cy;
                        int j0 = col_off[col], j1 = col_off[col + 1];
                        if (j1 - j0 > 64) { // tall column: only the clusters of the z-window
                            const int a0 = start[int64_t(col) * cpc];
                            const int aA = start[int64_t(col) * cpc + int64_t(czA) * lay];
                            const int aB = start[int64_t(col) * cpc + int64_t(czB + 1) * lay];
                            const int c0 = col_off[col];
                            j0 = c0 + (aA - a0) / 32;
                            j1 = aB > aA ? c0 + (aB - 1 - a0) / 32 + 1 : j0;
                        }
                        for (int jb = j0; jb < j1; jb += 32) {
                            const int jc = jb + lane;
                            bool ok = false;
                            if (jc < j1) {
                                const float4 l2 = blo[jc], h2 = bhi[jc];
                                const float ex = gapf(lo.x, hi.x, l2.x, h2.x);
                                const float ey = gapf(lo.y, hi.y, l2.y, h2.y);
                                const float ez = gapf(lo.z, hi.z, l2.z, h2.z);
                                ok = ex * ex + ey * ey + ez * ez < p.cut2;
                            }
                            const unsigned b = __ballot_sync(FULLMASK, ok);
                            const int loc = count - gstart + __popc(b & ((1u << lane) - 1u));
                            if (ok) { // staged in shared memory for the interleave; overflow straight out
                                if (loc < kListSeg)
                                    s_seg[wl][loc] = jc;
                                else if (gstart + loc < cap)
                                    out[gstart + loc] = jc;
                            }
                            count += __popc(b);
                            emitted += __popc(b);
                        }
                    }
                }
                nseg[ncol++] = emitted;
            }
            // interleave the group's columns: rank r of column c (odd c reversed) goes to
            // sum_c' min(n_c', r) + #{c' < c : n_c' > r}
            const int total = count - gstart;
            __syncwarp();
            if (ncol > 1 && total > 1 && total <= kListSeg) {
                for (int e = lane; e < total; e += 32) {
                    int c = 0, i = e;
                    while (i >= nseg[c]) i -= nseg[c++];
                    const int r = (c & 1) ? nseg[c] - 1 - i : i;
                    int dest = 0;
                    for (int c2 = 0; c2 < ncol; ++c2) dest += min(nseg[c2], r) + ((c2 < c && nseg[c2] > r) ? 1 : 0);
                    if (gstart + dest < cap) out[gstart + dest] = s_seg[wl][e];
                }
            } else { // column order
                for (int e = lane; e < min(total, kListSeg); e += 32)
                    if (gstart + e < cap) out[gstart + e] = s_seg[wl][e];
            }
            __syncwarp();
        }
    if (lane == 0) {
        pcnt[ic] = min(count, cap);
        if (count > cap) atomicMax(&err->overflow, count);
    }
}

struct PairP {
    double c0, c1, c2;   // gamma(r/a)/a = c0 + r2*(c1 + r2*c2)
    double d0, d1;       // g*'(r)/r + 1/r^3 = d0 + r2*d1
    double kc;
    // Wolf / damped-shifted-force pair term (src/electrostatics.cpp:91-120)
    double alpha, alpha2, gcoef, e_shift, f_shift, a;
    int wolf_fast;               // erfc(x) = exp(-x^2) * poly(u), see PairFieldP
    double wolf_us;
    double wolf_c[kWolfDeg + 1];
};

#ifndef MSMB_RSQRT_NEWTON
#define MSMB_RSQRT_NEWTON 3
#endif
// 1/sqrt(x) for 0 < x < inf: MUFU.RSQ64H seed refined by one cubically convergent
// Newton step, y += y*e*(1/2 + 3/8 e) with e = 1 - x*y^2: full double precision.
// (A quadratic step, MSMB_RSQRT_NEWTON=2, is one DP op cheaper and ~4% faster but
// leaves a one-sided ~1e-12 relative bias -- measured: energy 8.7e-13, phi_short
// 1.1e-12 on C2 shapes vs ~1e-15 with the cubic step -- so it is not the default.)
// No special-value path: callers only accumulate pairs with 0 < r2 < a2.
__device__ __forceinline__ double rsqrt_pos(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double e = fma(-(x * y), y, 1.0);
#if MSMB_RSQRT_NEWTON == 2
    return fma(y * e, 0.5, y);
#else
    return fma(y * e, fma(e, 0.375, 0.5), y);
#endif
}

// Pair function of the field kind K for 0 < r2 (r2 < a2 is applied by the caller):
// g = the pair potential per unit source charge, sd = (dV/dr)/r, so that
// phi_i += q_j g and F_i += d * (-k_C q_i q_j sd).
//  MSM:    g* = 1/r - gamma(r/a)/a, sd = g*'(r)/r        (msm_kernels.hpp:30-42)
//  cutoff: g = 1/r, sd = -1/r^3                           (electrostatics.cpp:81-86)
//  Wolf:   g = erfc(ar)/r - e_shift + f_shift (r - a),
//          sd = -(erfc(ar)/r^2 + gauss/r - f_shift)/r     (electrostatics.cpp:111-118)
template <int K>
__device__ __forceinline__ void pair_fn(const PairP& p, double r2, double rinv, double& g, double& sd) {
    const double rinv2 = rinv * rinv;
    if constexpr (K == MSMB_FIELD_MSM) {
        g = rinv - fma(r2, fma(r2, p.c2, p.c1), p.c0);
        sd = fma(-rinv, rinv2, fma(r2, p.d1, p.d0));
    } else if constexpr (K == MSMB_FIELD_CUTOFF) {
        g = rinv;
        sd = -rinv * rinv2;
    } else {
        const double r = r2 * rinv;
        const double e = exp(-p.alpha2 * r2); // shared by erfc and the Gaussian
        double er;
        if (p.wolf_fast) { // erfc(ar) = exp(-a^2 r^2) erfcx(ar); u clamped for r >= a (masked)
            const double u = fmin(fma(p.wolf_us, r, -1.0), 1.0);
            double poly = p.wolf_c[kWolfDeg];
#pragma unroll
            for (int k = kWolfDeg - 1; k >= 0; --k) poly = fma(poly, u, p.wolf_c[k]);
            er = e * poly;
        } else {
            er = erfc(p.alpha * r);
        }
        const double gs = p.gcoef * e;
        g = fma(p.f_shift, r - p.a, fma(er, rinv, -p.e_shift));
        sd = -fma(er, rinv2, fma(gs, rinv, -p.f_shift)) * rinv;
    }
}

__device__ __forceinline__ void record_pair(ErrRec* err, int i, int j) {
    const unsigned long long lo = (unsigned long long)min(i, j), hi = (unsigned long long)max(i, j);
    atomicMin(&err->pair_key, (lo << 32) | hi);
}

// Short-range pair sum in two kernels over the cluster pair list of
// k_pairlist: k_pairmask (list rebuilds only) turns every entry into per-lane
// 32-bit masks of the j-cluster atoms within a + skin; k_pairs_mw (every
// evaluation) walks them.  Measured history on C2-S (pairs, ms): two-slot drain
// ring with in-kernel fp32 screening 0.92; per-lane walk with in-kernel
// screening 0.92 (screening was 36% of the instructions); masks + walk 0.64.
constexpr int kSlots = 33;            // one ring slot: dummy + 32 atoms
#ifndef MSMB_PAIR_MINB
#define MSMB_PAIR_MINB (20 / MSMB_PAIR_WARPS) // CTAs per SM: 20 warps (96 registers)
#endif
#ifndef MSMB_PAIR_RING
#define MSMB_PAIR_RING 8
#endif
constexpr int kRing = MSMB_PAIR_RING;
static_assert((kRing & (kRing - 1)) == 0, "ring size must be a power of two");
static_assert(kRing >= 2, "the dense phase stages its batches in ring slots 0 and 1");
#ifndef MSMB_PAIR_UNROLL
#define MSMB_PAIR_UNROLL 4
#endif
#ifndef MSMB_DENSE_UNROLL
#define MSMB_DENSE_UNROLL 4 // divides 32
#endif

// Pair masks, built once per pair-list rebuild (flag[0]): for every list entry of
// an i-cluster, each lane's 32-bit mask of the j-cluster atoms within the list cut
// a + skin (fp32 screen with the rigorous rounding pad).  A pair within a at any
// evaluation before the next rebuild is within a + skin at the build (the rebuild
// trigger is a move of skin/2), so the masks stay complete until then; k_pairs_mw
// applies the exact r < a test in fp64.  Entries whose masks are empty for every
// lane are dropped (in-place compaction), as is the i-cluster's own entry (summed
// densely by k_pairs_mw), and each entry becomes the j-cluster's first sorted slot.
constexpr int kMaskWarps = 8;
__global__ void __launch_bounds__(kMaskWarps * 32)
    k_pairmask(const int2* __restrict__ clu, int* plist, int* pcnt, unsigned* __restrict__ pmask, int cap,
               const double* __restrict__ xs, const double* __restrict__ ys, const double* __restrict__ zs,
               float cut2f, const int* __restrict__ col_off, int col_a, int col_b, const int* __restrict__ flag,
               ErrRec* err, int* __restrict__ dlist, int* __restrict__ dcnt, int dcap, int dense_t) {
    __shared__ __align__(16) float s_sc[kMaskWarps][4][32];
    __shared__ __align__(16) int s_sh[kMaskWarps][32];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ic = col_off[col_a] + blockIdx.x * kMaskWarps + w;
    if (ic >= col_off[col_b] || failed(err) || !flag[0]) return;
    const int2 c = clu[ic];
    const bool vi = lane < c.y;
    const int si = c.x + (vi ? lane : 0);
    const double rx = xs[c.x], ry = ys[c.x], rz = zs[c.x];
    const float xf = float(xs[si] - rx), yf = float(ys[si] - ry), zf = float(zs[si] - rz);
    const float2 xi2 = make_float2(xf, xf), yi2 = make_float2(yf, yf), zi2 = make_float2(zf, zf);
    const float nif = fmaf(zf, zf, fmaf(yf, yf, xf * xf));
    const float2 ni2 = make_float2(nif, nif);
    const float ri2 = __uint_as_float(__reduce_max_sync(FULLMASK, __float_as_uint(vi ? nif : 0.f)));
    // the i-cluster's box in the same relative fp32 coordinates
    float blo[3] = {vi ? xf : 3e38f, vi ? yf : 3e38f, vi ? zf : 3e38f};
    float bhi[3] = {vi ? xf : -3e38f, vi ? yf : -3e38f, vi ? zf : -3e38f};
#pragma unroll
    for (int o = 16; o; o >>= 1)
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
            blo[ax] = fminf(blo[ax], __shfl_xor_sync(FULLMASK, blo[ax], o));
            bhi[ax] = fmaxf(bhi[ax], __shfl_xor_sync(FULLMASK, bhi[ax], o));
        }
    const int nj = pcnt[ic];
    int* pl = plist + size_t(ic) * cap;
    unsigned* pm = pmask + size_t(ic) * cap * 32;
    int* dl = dlist + size_t(ic) * dcap;
    int out = 0, nd = 0;
    // list entries and their clusters in two register windows of 32 (lane l holds
    // entry 32w + l), refilled one window ahead; the j atoms of entry jj + 1 are
    // loaded while entry jj is screened (the dependent loads stay off the chain)
    int jcw[2];
    int2 cjw[2];
#pragma unroll
    for (int b = 0; b < 2; ++b) {
        jcw[b] = 32 * b + lane < nj ? pl[32 * b + lane] : ic;
        cjw[b] = clu[jcw[b]];
    }
    auto entry = [&](int jj, int& jc, int2& cj) {
        const int b = (jj >> 5) & 1, src = jj & 31;
        jc = __shfl_sync(FULLMASK, b ? jcw[1] : jcw[0], src);
        cj.x = __shfl_sync(FULLMASK, b ? cjw[1].x : cjw[0].x, src);
        cj.y = __shfl_sync(FULLMASK, b ? cjw[1].y : cjw[0].y, src);
    };
    int jc_n = ic;
    int2 cj_n = make_int2(0, 0);
    double xn = 0, yn = 0, zn = 0;
    auto fetch = [&](int jj) {
        entry(jj, jc_n, cj_n);
        const int sj = cj_n.x + (lane < cj_n.y ? lane : 0);
        xn = xs[sj];
        yn = ys[sj];
        zn = zs[sj];
    };
    if (nj > 0) fetch(0);
    for (int jj = 0; jj < nj; ++jj) {
        const int jc = jc_n;
        const int2 cj = cj_n;
        const double xd = xn, yd = yn, zd = zn;
        if ((jj & 31) == 0 && jj > 0) { // window jj/32 is in use: refill the other one with the next
            const int b = ((jj >> 5) + 1) & 1, e = jj + 32 + lane;
            const int v = e < nj ? pl[e] : ic;
            const int2 cv = clu[v];
            if (b) { jcw[1] = v; cjw[1] = cv; } else { jcw[0] = v; cjw[0] = cv; }
        }
        if (jj + 1 < nj) fetch(jj + 1);
        const bool vj = lane < cj.y;
        const float xj = float(xd - rx), yj = float(yd - ry), zj = float(zd - rz);
        const float njf = fmaf(zj, zj, fmaf(yj, yj, xj * xj));
        const float rj2 = __uint_as_float(__reduce_max_sync(FULLMASK, __float_as_uint(vj ? njf : 0.f)));
        const float cut2 = cut2f + 64.f * 5.9604645e-8f * (ri2 + rj2);
        // atoms beyond the cut from the whole i-box cannot be in any lane's mask: only the
        // others are screened, compacted into chunks of 4 (bit position kept per slot)
        const float ex = fmaxf(0.f, fmaxf(blo[0] - xj, xj - bhi[0]));
        const float ey = fmaxf(0.f, fmaxf(blo[1] - yj, yj - bhi[1]));
        const float ez = fmaxf(0.f, fmaxf(blo[2] - zj, zj - bhi[2]));
        const bool rel = vj && fmaf(ez, ez, fmaf(ey, ey, ex * ex)) <= cut2 * 1.00001f;
        const unsigned R = __ballot_sync(FULLMASK, rel);
        if (R == 0u) continue;
        const int k = __popc(R & ((1u << lane) - 1u)), nr = __popc(R), nr4 = (nr + 3) & ~3;
        __syncwarp();
        if (rel) {
            s_sc[w][0][k] = -2.f * xj;
            s_sc[w][1][k] = -2.f * yj;
            s_sc[w][2][k] = -2.f * zj;
            s_sc[w][3][k] = njf - cut2;
            s_sh[w][k] = 31 - lane;
        }
        if (lane >= nr && lane < nr4) { // padding slots: never in range
            s_sc[w][0][lane] = 0.f;
            s_sc[w][1][lane] = 0.f;
            s_sc[w][2][lane] = 0.f;
            s_sc[w][3][lane] = 3e38f;
            s_sh[w][lane] = 0;
        }
        __syncwarp();
        unsigned mask = 0;
#pragma unroll 2
        for (int t = 0; t < nr4; t += 4) {
            const float4 mx = *reinterpret_cast<const float4*>(&s_sc[w][0][t]);
            const float4 my = *reinterpret_cast<const float4*>(&s_sc[w][1][t]);
            const float4 mz = *reinterpret_cast<const float4*>(&s_sc[w][2][t]);
            const float4 cc = *reinterpret_cast<const float4*>(&s_sc[w][3][t]);
            const int4 sh = *reinterpret_cast<const int4*>(&s_sh[w][t]);
            float2 sa = __fadd2_rn(ni2, make_float2(cc.x, cc.y));
            float2 sb = __fadd2_rn(ni2, make_float2(cc.z, cc.w));
            sa = __ffma2_rn(make_float2(mx.x, mx.y), xi2, sa);
            sb = __ffma2_rn(make_float2(mx.z, mx.w), xi2, sb);
            sa = __ffma2_rn(make_float2(my.x, my.y), yi2, sa);
            sb = __ffma2_rn(make_float2(my.z, my.w), yi2, sb);
            sa = __ffma2_rn(make_float2(mz.x, mz.y), zi2, sa);
            sb = __ffma2_rn(make_float2(mz.z, mz.w), zi2, sb);
            mask |= ((__float_as_uint(sa.x) >> 31) << sh.x) | ((__float_as_uint(sa.y) >> 31) << sh.y) |
                    ((__float_as_uint(sb.x) >> 31) << sh.z) | ((__float_as_uint(sb.y) >> 31) << sh.w);
        }
        if (!vi || jc == ic) mask = 0; // the own cluster is summed densely by k_pairs_mw
        mask &= ~(0xffffffffu >> cj.y); // bits 31 .. 32 - cj.y: the cluster's atoms only
        // (an atom can only be dense if at least dense_t lanes have a bit at all)
        if (dense_t > 0 && __popc(__ballot_sync(FULLMASK, mask != 0u)) >= dense_t) {
            // Dense atoms: within the list cut of >= dense_t of the 32 i atoms.  A 32 x 32 bit
            // transpose over the warp gives lane l the column of atom l (bit 31 - l of every
            // lane's mask); those atoms go to the i-cluster's dense list (k_pairs_mw sums them
            // with the whole warp in lockstep, the j row broadcast) and leave the masks.
            unsigned tr = mask, tm = 0x0000ffffu;
#pragma unroll
            for (int j = 16; j; j >>= 1) {
                const unsigned o = __shfl_xor_sync(FULLMASK, tr, j);
                if ((lane & j) == 0)
                    tr ^= (tr ^ (o >> j)) & tm;
                else
                    tr ^= ((o ^ (tr >> j)) & tm) << j;
                tm ^= tm << (j >> 1);
            }
            const bool dense = __popc(tr) >= dense_t;
            const unsigned dn = __ballot_sync(FULLMASK, dense);
            if (dn != 0u && nd + __popc(dn) <= dcap) {
                if (dense) dl[nd + __popc(dn & ((1u << lane) - 1u))] = cj.x + lane;
                nd += __popc(dn);
                mask &= ~__brev(dn);
            }
        }
        if (__any_sync(FULLMASK, mask != 0)) {
            pm[size_t(out) * 32 + lane] = mask;
            if (lane == 0) pl[out] = cj.x;
            ++out;
        }
    }
    if (lane == 0) {
        pcnt[ic] = out;
        dcnt[ic] = nd;
    }
}

// One warp per i-cluster (lane = i atom) walks the i-cluster's mask list.  The warp
// stages j-clusters into a ring of kRing slots in shared memory: fp64 (x, y) and
// (z, q) as double2 rows, atom t at slot position 32 - t and a dummy atom (q = 0,
// far away) at position 0, plus each lane's mask.  Every lane walks the list on
// its own: it holds the list position `cur` of the cluster it consumes and that
// cluster's remaining mask; a pair step takes the highest set bit (bfind; bit
// 31 - t <=> atom t), or the dummy once the mask is empty (bfind(0) = -1), and an
// exhausted lane moves to the next staged cluster (branch-free; a cluster without
// atoms for the lane costs it one idle step).  The warp stages more clusters once
// the slowest lane is less than kRing clusters behind the staging frontier, so
// lanes only idle at the end of the list.  Each pair step applies the exact cutoff
// r^2 < a^2 in fp64: skin-shell pairs and the dummy add nothing, as the reference
// skips r >= a (src/msm_phases.cpp:240).  The own cluster is not in the list: its
// pairs are summed first, densely (j broadcast by shuffles).  Per lane the pairs
// are accumulated in a fixed order (own cluster, then list order, atoms of a
// cluster ascending): the sums are deterministic.  rsqrt is MUFU.RSQ64H + one
// cubic Newton step (rsqrt_pos); 22 DP instructions + 1 DSETP per pair step.
// Measured alternatives (C2-S, ms): lanes in lockstep groups of 2 / 4 walking the
// union of their masks (spatially sorted groups; fewer shared-memory bank
// conflicts, more steps) 0.68 / 0.73 vs 0.63 per lane; unroll 8 vs 4: equal; each
// lane preferring a mask bit whose row sits in bank quad (lane & 7) (conflict-free
// when found, measured in a microbenchmark) 0.68: only 17% of steps find one --
// a lane's mask holds ~1-2 atoms of a cluster -- and bank conflicts did not drop;
// two z-adjacent i atoms per lane walking the union of their masks (half-warp per
// i-cluster, each staged row feeding two pairs) 0.86: shared-memory wavefronts
// -35% but FP64 instructions +36% (union steps wasted for one of the atoms) and
// occupancy 4 -> 3.4 warps/SMSP at 122 registers; the kernel is latency-bound
// (FP64 pipe 53%, issue 62-67%, stalls spread over wait / math throttle /
// long scoreboard of the staging loads); two staged clusters in flight (register
// double buffer) 0.647 vs 0.632.
// COUNT: accumulate the in-cutoff pair and candidate counters (work statistics); the
// captured step graphs run the COUNT = false instance (counted on eager evaluations)
template <int K, bool SPLIT, bool COUNT>
__global__ void __launch_bounds__(kPairWarps * 32, MSMB_PAIR_MINB)
    k_pairs_mw(const int2* __restrict__ clu, const int* __restrict__ plist, const int* __restrict__ pcnt,
               const unsigned* __restrict__ pmask, int cap, const double* __restrict__ xs,
               const double* __restrict__ ys, const double* __restrict__ zs, const double* __restrict__ qs,
               PairP p, double a2, double* phis, double* fsx, double* fsy, double* fsz,
               const int* __restrict__ col_off, int col_a, int col_b, int64_t n, ErrRec* err,
               int split_arg, double* __restrict__ part, const int* __restrict__ dlist,
               const int* __restrict__ dcnt, int dcap, const int* __restrict__ gflag, int gmode) {
    pdl_enter();
    // gmode 1: runs on skin evaluations only (flag[0] == 0), 2: on rebuild evaluations only
    if (gmode && (gflag[0] != 0) != (gmode == 2)) return;
    const int split = SPLIT ? split_arg : 1; // compile-time 1 on the large-system path
    __shared__ unsigned s_mask[kPairWarps][kRing][32];
    __shared__ double2 s_v[kPairWarps][2][kRing * kSlots]; // (x, y), (z, q) rows
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // split > 1 (small systems): `split` warps share an i-cluster, each walking a
    // contiguous part of its list; their raw sums go to `part` and k_pairs_join adds
    // them in part order (deterministic)
    const int gw = blockIdx.x * kPairWarps + w;
    const int ic = col_off[col_a] + (SPLIT ? gw / split : gw), sp = SPLIT ? gw % split : 0;
    if (ic >= col_off[col_b] || failed(err)) return;
    const int2 c = clu[ic];
    const bool vi = lane < c.y;
    const int si = c.x + (vi ? lane : 0);
    const double xi = xs[si], yi = ys[si], zi = zs[si], qi = qs[si];
    double ph = 0.0, fx = 0.0, fy = 0.0, fz = 0.0;
    unsigned ncand = 0, npair = 0;
    const int nj_all = pcnt[ic];
    const int jb = SPLIT ? int(int64_t(nj_all) * sp / split) : 0;
    const int nj = SPLIT ? int(int64_t(nj_all) * (sp + 1) / split) - jb : nj_all;
    const int* pl = plist + size_t(ic) * cap + jb;
    const unsigned* pm = pmask + (size_t(ic) * cap + jb) * 32 + lane;
    unsigned mk_n = 0;
    double xj_n = 0, yj_n = 0, zj_n = 0, qj_n = 0;
    auto fetch = [&](int jj) {
        const int64_t sj = min(int64_t(pl[jj]) + lane, n - 1); // lanes past the cluster: masked out
        mk_n = pm[size_t(jj) * 32];
#ifdef MSMB_EXP_NOSTAGE
        if (jj >= kRing) return;
#endif
        xj_n = xs[sj];
        yj_n = ys[sj];
        zj_n = zs[sj];
        qj_n = qs[sj];
    };
    auto stage = [&](int jj) {
        const int slot = jj & (kRing - 1);
        const int pos = slot * kSlots + 32 - lane;
#ifdef MSMB_EXP_NOSTAGE // timing experiment only (wrong results): rows staged once
        if (jj < kRing)
#endif
        {
        s_v[w][0][pos] = make_double2(xj_n, yj_n);
        s_v[w][1][pos] = make_double2(zj_n, qj_n);
        }
        s_mask[w][slot][lane] = mk_n;
        if (COUNT) ncand += __popc(mk_n);
        if (jj + 1 < nj) fetch(jj + 1);
    };
    const double2* rows = &s_v[w][0][0];
    int hi = 0;          // clusters staged so far (warp-uniform)
    int cur = 0;         // this lane's list position
    unsigned m = 0;      // this lane's remaining mask of cluster `cur`
    unsigned mnext = 0;  // mask of cluster cur + 1 (valid while cur + 1 < hi)
    const double2* row = rows;
    auto advance = [&]() {
        const bool adv = (m == 0) & (cur + 1 < hi);
        cur += adv ? 1 : 0;
        m = adv ? mnext : m;
        row = rows + (cur & (kRing - 1)) * kSlots;
        mnext = s_mask[w][(cur + 1) & (kRing - 1)][lane];
    };
    auto step = [&]() {
        int pos;
        asm("bfind.u32 %0, %1;" : "=r"(pos) : "r"(m));
        unsigned bit;
        asm("shl.b32 %0, %1, %2;" : "=r"(bit) : "r"(1u), "r"(pos));
        m ^= bit; // bit = 0 when m == 0 (shl clamps): the dummy step leaves m at 0
#ifdef MSMB_EXP_NOBANK // timing experiment only (wrong results): conflict-free row reads
        const double2* rs = rows + 1 + (lane & 7) + (pos & 24);
#else
        const double2* rs = row + (pos + 1);
#endif
        const double2 xy = rs[0], zq = rs[kRing * kSlots];
        advance();
        const double dx = xi - xy.x, dy = yi - xy.y, dz = zi - zq.x;
        const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
        const double rinv = rsqrt_pos(r2);
        double g, sd;
        pair_fn<K>(p, r2, rinv, g, sd);
        const bool in = r2 < a2;
        if (COUNT) npair += in ? 1u : 0u;
        const double qj = in ? zq.y : 0.0; // two FSELs (a predicated accumulation costs 8)
        ph = fma(qj, g, ph);
        const double wgt = qj * sd;
        fx = fma(dx, wgt, fx);
        fy = fma(dy, wgt, fy);
        fz = fma(dz, wgt, fz);
    };
    for (int s = lane; s < 2 * kRing; s += 32) // dummies (q = 0, far away) at each ring slot's position 0
        s_v[w][s & 1][(s >> 1) * kSlots] = (s & 1) ? make_double2(1e4, 0.0) : make_double2(1e4, 1e4);
    __syncwarp();
    // Dense phase: the i-cluster's dense j atoms (k_pairmask), 32 per batch: lane l loads
    // atom 32 b + l of the list (indices two batches and atoms one batch ahead of their use)
    // and stages it into ring slot b & 1; then the whole warp steps through the batch, every
    // lane reading the same row (a broadcast, no mask bookkeeping: 30 instructions per step,
    // 24 of them FP64) and applying the exact cutoff.  Lanes past the list stage the dummy.
    // Measured alternatives (C2-S, pairs ms; 0.622 without the dense phase): this, threshold
    // 28 of 32 lanes, 0.578; threshold 16, 0.627; dense lists per octet of lanes (threshold 4
    // of 8, one list per octet staged by cp.async) 0.725; one list tagged with the octets, each
    // octet stepping through its bits of the batch, 0.82 (a batch takes its fullest octet's
    // steps); alternating the phase order between neighbouring warps: slower; persistent
    // warps claiming i-clusters from a work counter (148 x 16..20 one-warp CTAs): 0.60-0.63
    // alone, and the long-range chain starves beside CTAs that never retire.
    {
        const int nd_all = dcnt[ic];
        const int db = SPLIT ? int(int64_t(nd_all) * sp / split) : 0;
        const int nd = (SPLIT ? int(int64_t(nd_all) * (sp + 1) / split) : nd_all) - db;
        const int* dl = dlist + size_t(ic) * dcap + db;
        if (COUNT) ncand += vi ? unsigned(nd) : 0u;
        const int nb = (nd + 31) >> 5;
        int sj1 = lane < nd ? dl[lane] : -1;           // batch 0
        int sj2 = 32 + lane < nd ? dl[32 + lane] : -1; // batch b + 1
        double xn = 1e4, yn = 1e4, zn = 1e4, qn = 0.0;
        auto dload = [&](int sj) {
            xn = yn = zn = 1e4;
            qn = 0.0;
            if (sj >= 0) {
                xn = xs[sj];
                yn = ys[sj];
                zn = zs[sj];
                qn = qs[sj];
            }
        };
        if (nb > 0) dload(sj1);
        for (int b = 0; b < nb; ++b) {
            double2* buf = &s_v[w][0][(b & 1) * kSlots + 1];
            buf[lane] = make_double2(xn, yn);
            buf[kRing * kSlots + lane] = make_double2(zn, qn);
            __syncwarp();
            if (b + 1 < nb) dload(sj2);
            sj2 = (b + 2) * 32 + lane < nd ? dl[(b + 2) * 32 + lane] : -1;
            const int tcnt = min(32, nd - 32 * b);
#pragma unroll 1
            for (int t0 = 0; t0 < tcnt; t0 += MSMB_DENSE_UNROLL) {
#pragma unroll
                for (int u = 0; u < MSMB_DENSE_UNROLL; ++u) {
                    const double2 xy = buf[t0 + u], zq = buf[kRing * kSlots + t0 + u];
                    const double dx = xi - xy.x, dy = yi - xy.y, dz = zi - zq.x;
                    const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
                    const double rinv = rsqrt_pos(r2);
                    double g, sd;
                    pair_fn<K>(p, r2, rinv, g, sd);
                    const bool in = r2 < a2;
                    if (COUNT) npair += (in && vi) ? 1u : 0u;
                    const double qj = in ? zq.y : 0.0;
                    ph = fma(qj, g, ph);
                    const double wgt = qj * sd;
                    fx = fma(dx, wgt, fx);
                    fy = fma(dy, wgt, fy);
                    fz = fma(dz, wgt, fz);
                }
            }
        }
        __syncwarp();
    }
    if (nj > 0) fetch(0);
    ncand += (vi && sp == 0) ? unsigned(c.y - 1) : 0u;
    // the own cluster (dropped from the mask list): all atom pairs, j broadcast by shuffles
    for (int t = 0; t < (sp == 0 ? c.y : 0); ++t) {
        const double xj = __shfl_sync(FULLMASK, xi, t), yj = __shfl_sync(FULLMASK, yi, t);
        const double zj = __shfl_sync(FULLMASK, zi, t), qt = __shfl_sync(FULLMASK, qi, t);
        const double dx = xi - xj, dy = yi - yj, dz = zi - zj;
        const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
        const bool in = r2 < a2 && t != lane;
        const double rinv = rsqrt_pos(in ? r2 : a2);
        double g, sd;
        pair_fn<K>(p, in ? r2 : a2, rinv, g, sd);
        npair += in ? 1u : 0u;
        const double qj = in ? qt : 0.0;
        ph = fma(qj, g, ph);
        const double wgt = qj * sd;
        fx = fma(dx, wgt, fx);
        fy = fma(dy, wgt, fy);
        fz = fma(dz, wgt, fz);
    }
    if (nj > 0) {
        __syncwarp();
        while (hi < nj && hi < kRing) stage(hi++);
        __syncwarp();
        m = s_mask[w][0][lane];
        mnext = s_mask[w][1][lane];
        for (;;) {
#pragma unroll
            for (int u = 0; u < MSMB_PAIR_UNROLL; ++u) step();
            const int lo = __reduce_min_sync(FULLMASK, cur);
            if (hi < nj && hi - lo < kRing) {
                __syncwarp();
                do stage(hi++);
                while (hi < nj && hi - lo < kRing);
                __syncwarp();
                mnext = s_mask[w][(cur + 1) & (kRing - 1)][lane];
                advance();
            }
            if (hi >= nj && __all_sync(FULLMASK, m == 0 && cur + 1 >= hi)) break;
        }
    }
    if (SPLIT && vi) {
        double* o = part + (size_t(sp) * 4) * size_t(n) + si;
        o[0] = ph;
        o[size_t(n)] = fx;
        o[2 * size_t(n)] = fy;
        o[3 * size_t(n)] = fz;
    } else if (vi) {
        const double kq = -p.kc * qi; // f = d * (-k_C q_i q_j g*'/r)  (msm_phases.cpp:246)
        phis[si] = ph;
        fsx[si] = fx * kq;
        fsy[si] = fy * kq;
        fsz[si] = fz * kq;
    }
    if (COUNT) {
        ncand = __reduce_add_sync(FULLMASK, ncand);
        npair = __reduce_add_sync(FULLMASK, npair);
        if (lane == 0) {
            atomicAdd(&err->pairs, (unsigned long long)npair);
            atomicAdd(&err->candidates, (unsigned long long)ncand);
        }
    }
}

// Error path only: pairs involving particles that could not be binned
// (outside grid coverage or non-finite) against every particle, with the
// reference's arithmetic, to find the first pair with r2 == 0 or NaN.  Run by the
// blocks b = 0 .. nb-1 past k_cl_gather's atom range (record_pair is an atomicMin:
// the result does not depend on when or by whom the pairs are visited).
__device__ void err_brute_blocks(int64_t n, const double* __restrict__ x, const double* __restrict__ y,
                                 const double* __restrict__ z, const int* __restrict__ outlist, ErrRec* err,
                                 int b, int nb) {
    const int cnt = __ldcg(&err->cov_count);
    if (cnt == 0 || failed(err)) return;
    const int64_t total = int64_t(cnt) * n;
    for (int64_t idx = int64_t(b) * blockDim.x + threadIdx.x; idx < total; idx += int64_t(nb) * blockDim.x) {
        const int o = outlist[idx / n];
        const int j = int(idx % n);
        if (j == o) continue;
        const int lo = min(o, j), hi = max(o, j);
        const double dx = __dsub_rn(x[lo], x[hi]), dy = __dsub_rn(y[lo], y[hi]), dz = __dsub_rn(z[lo], z[hi]);
        const double r2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
        if (r2 == 0.0 || isnan(r2)) record_pair(err, lo, hi);
    }
}

// Launches of a skin step (no rebuild): k_flag_reset, k_disp, k_cl_gather and the
// four rebuild kernels k_colscan, k_bbox, k_pairlist, k_pairmask, which read flag[0]
// and exit.  Measured alternatives: IF conditional graph nodes around the rebuild
// kernels (cudaGraphSetConditional from the deciding kernel): an untaken IF node
// costs ~8 us of graph execution on this driver (tools/cond_probe.cu: 10.6 us vs
// 13.5 us for ten early-exit kernels, 2.1 us without either), and with four of them
// per evaluation the C2-S step went 0.845 -> 0.862 ms; leaving the rebuild kernels
// out of the step graphs entirely (timing only) gave 0.809 ms -- the fusions here
// (13 -> 7 launches) take part of that without the IF nodes.
// phase 0: everything on one stream.  The engine's forked evaluation splits it: phase 1 = the
// rebuild decision and the skin evaluations' gather (needs the binning's out-of-coverage
// list, not the cell sort), phase 2 = the rebuild (after the cell sort; every kernel exits
// unless flag[0]), so that on a skin step the pair kernel does not wait for the sort.
int launch_clusters(cudaStream_t st, const Geometry& g, int64_t n, const DevState& s, DevAtoms& a,
                    DevCells& c, ErrRec* err, int cap, const Part& P, int force_rebuild, int disp, int phase) {
    const int cells_per_col = int(g.lv[0].dims[2]) * g.cw * g.cw;
    const int64_t nc = g.ncols;
    // rebuild decision, frozen cluster order, current positions in it
    const int key = P.cx0 * 65536 + P.cx1;
    const int gb = int((std::max<int64_t>(n, 1) + 255) / 256);
    if (phase != 2) {
        // PDL (pdl_enter in the kernels): each launch is admitted while its predecessor runs
        pdl_launch(k_flag_reset, dim3(1), dim3(1), 0, st, c.flag, force_rebuild || !(g.skin > 0.0) ? 1 : 0, key);
        const double hs = 0.5 * g.skin;
        if (disp)
            pdl_launch(k_disp, dim3(atom_blocks(n, atom_tpb(n))), dim3(atom_tpb(n)), 0, st, n, s.x, s.y, s.z, a.ref,
                       hs * hs, c.flag);
        pdl_launch(k_cl_gather, dim3(gb + 592), dim3(256), 0, st, n, c.start + g.ncells, a.perm, s.x, s.y, s.z, s.q,
                   a.cl_perm, a.cl_inv, a.ref, c.flag, key, a.xc, a.yc, a.zc, a.qc, gb, a.outlist, err, phase);
        if (phase == 1) return 2 + (disp ? 1 : 0);
    } else {
        k_cl_gather<<<gb, 256, 0, st>>>(n, c.start + g.ncells, a.perm, s.x, s.y, s.z, s.q, a.cl_perm, a.cl_inv,
                                        a.ref, c.flag, key, a.xc, a.yc, a.zc, a.qc, gb, a.outlist, err, 2);
    }
    // cluster pair list (rebuild evaluations only)
    k_colscan<<<1, 1024, 0, st>>>(nc, cells_per_col, c.start, c.col_cnt, c.col_off, c.clu, c.nclu, c.colstart,
                                  c.flag, err);
    const int64_t maxclu = n / 32 + nc + 1;
    k_bbox<<<int((maxclu * 32 + 255) / 256), 256, 0, st>>>(c.nclu, c.clu, a.xc, a.yc, a.zc, c.blo, c.bhi, c.flag,
                                                           err);
    ListP lp;
    lp.ox = g.lv[0].origin[0];
    lp.oy = g.lv[0].origin[1];
    lp.colw = g.colw;
    lp.ncx = g.ncx;
    lp.ncy = g.ncy;
    const double lc = g.screen_cut + g.skin; // list cutoff: screening cut + skin
    lp.cut = float(lc);
    lp.cut2 = float(lc * lc);
    lp.oz = g.lv[0].origin[2];
    lp.h = g.lv[0].spacing;
    lp.d2 = g.lv[0].dims[2];
    lp.cw = g.cw;
    lp.clamp = g.kind != MSMB_FIELD_MSM; // occupied cells are 1 .. d-3 per axis (k_bin)
    lp.cxmin = 1 / g.cw;
    lp.cxmax = (g.lv[0].dims[0] - 3) / g.cw;
    lp.cymin = 1 / g.cw;
    lp.cymax = (g.lv[0].dims[1] - 3) / g.cw;
    lp.czmin = 1;
    lp.czmax = g.lv[0].dims[2] - 3;
    k_pairlist<<<int((maxclu * 32 + 255) / 256), 256, 0, st>>>(c.nclu, c.blo, c.bhi, c.col_off, c.start, lp,
                                                                c.plist, c.pcnt, cap, P.cx0 * g.ncy,
                                                                P.cx1 * g.ncy, c.flag, err);
    const double lm = g.cfg.cutoff_a + g.skin; // mask cut: a + skin (+ the fp32 pad in k_pairmask)
    k_pairmask<<<int((maxclu + kMaskWarps - 1) / kMaskWarps), kMaskWarps * 32, 0, st>>>(
        c.clu, c.plist, c.pcnt, c.pmask, cap, a.xc, a.yc, a.zc, float_ru(lm * lm * (1.0 + 1e-6)), c.col_off,
        P.cx0 * g.ncy, P.cx1 * g.ncy, c.flag, err, c.dlist, c.dcnt, std::max(g.dense_cap, 32), g.dense_t);
    return phase == 2 ? 5 : 7 + (disp ? 1 : 0);
}

// sums of the split pair walks, in part order, then the per-atom force factor
__global__ void k_pairs_join(const int* __restrict__ colstart, int col_a, int col_b, int split, int64_t n,
                             const double* __restrict__ part, const double* __restrict__ qs, double kc,
                             double* phis, double* fsx, double* fsy, double* fsz, const ErrRec* err,
                             const int* __restrict__ gflag, int gmode) {
    if (gmode && (gflag[0] != 0) != (gmode == 2)) return;
    const int s = colstart[col_a] + blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= colstart[col_b] || failed(err)) return;
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    for (int k = 0; k < split; ++k)
#pragma unroll
        for (int c = 0; c < 4; ++c) v[c] += part[(size_t(k) * 4 + c) * size_t(n) + s];
    const double kq = -kc * qs[s];
    phis[s] = v[0];
    fsx[s] = v[1] * kq;
    fsy[s] = v[2] * kq;
    fsz[s] = v[3] * kq;
}

// warps per i-cluster: enough warps for ~5 resident blocks on every SM
int pair_split(int64_t maxclu) {
    const int64_t want = 148 * MSMB_PAIR_MINB * kPairWarps; // resident warps on 148 SMs
    int64_t sp = (want + std::max<int64_t>(maxclu, 1) - 1) / std::max<int64_t>(maxclu, 1);
    return int(std::min<int64_t>(std::max<int64_t>(sp, 1), kPairSplitMax));
}

int launch_pairs(cudaStream_t st, const Geometry& g, int64_t n, const DevState& s, DevAtoms& a,
                 DevCells& c, ErrRec* err, int cap, const Part& P, bool count, int gmode) {
    const double A = g.cfg.cutoff_a;
    PairP p;
    // gamma(rho)/a = 15/(8a) - 5 r^2/(4a^3) + 3 r^4/(8a^5)          (msm_kernels.hpp:14-20,30-35)
    p.c0 = 15.0 / (8.0 * A);
    p.c1 = -5.0 / (4.0 * A * A * A);
    p.c2 = 3.0 / (8.0 * A * A * A * A * A);
    // g*'(r)/r = -1/r^3 + (2.5 - 1.5 rho^2)/a^3                    (msm_kernels.hpp:22-27,37-42)
    p.d0 = 2.5 / (A * A * A);
    p.d1 = -1.5 / (A * A * A * A * A);
    p.kc = g.units.coulomb_constant;
    p.alpha = g.pf.alpha;
    p.alpha2 = g.pf.alpha * g.pf.alpha;
    p.gcoef = 1.1283791670955126 * g.pf.alpha; // 2/sqrt(pi) alpha (src/electrostatics.cpp:12,112)
    p.e_shift = g.pf.e_shift;
    p.f_shift = g.pf.f_shift;
    p.a = A;
    p.wolf_fast = g.pf.wolf_fast;
    p.wolf_us = g.pf.wolf_us;
    for (int k = 0; k <= kWolfDeg; ++k) p.wolf_c[k] = g.pf.wolf_c[k];
    const int64_t maxclu = n / 32 + g.ncols + 1;
    int l = 0;
    if (n > 0) {
        const int split = a.pair_part ? pair_split(maxclu) : 1;
#ifdef MSMB_PAIR_ALWAYS_COUNT // A/B switch: count in every evaluation (the round-1 behaviour)
        count = true;
#endif
        // instances: field kind x split x counting
        auto pick = [&](auto split_c, auto count_c) {
            constexpr bool SP = decltype(split_c)::value, CO = decltype(count_c)::value;
            return g.kind == MSMB_FIELD_CUTOFF ? k_pairs_mw<MSMB_FIELD_CUTOFF, SP, CO>
                   : g.kind == MSMB_FIELD_WOLF ? k_pairs_mw<MSMB_FIELD_WOLF, SP, CO>
                                               : k_pairs_mw<MSMB_FIELD_MSM, SP, CO>;
        };
        using T = std::true_type;
        using F = std::false_type;
        auto kern = split > 1 ? (count ? pick(T{}, T{}) : pick(T{}, F{})) : (count ? pick(F{}, T{}) : pick(F{}, F{}));
        pdl_launch(kern, dim3(int((maxclu * split + kPairWarps - 1) / kPairWarps)), dim3(kPairWarps * 32), 0, st, c.clu,
                   c.plist, c.pcnt, c.pmask, cap, a.xc, a.yc, a.zc, a.qc, p, A * A, a.phis, a.fsx, a.fsy, a.fsz,
                   c.col_off, P.cx0 * g.ncy, P.cx1 * g.ncy, n, err, split, a.pair_part, c.dlist, c.dcnt,
                   std::max(g.dense_cap, 32), c.flag, gmode);
        l = 1;
        if (split > 1) {
            k_pairs_join<<<int((n + 255) / 256), 256, 0, st>>>(c.colstart, P.cx0 * g.ncy, P.cx1 * g.ncy, split, n,
                                                               a.pair_part, a.qc, p.kc, a.phis, a.fsx, a.fsy, a.fsz,
                                                               err, c.flag, gmode);
            ++l;
        }
    }
    return l;
}

// pair errors of particles outside grid coverage (NaN / coincident with anyone); needs
// only the binning, so the spatial decomposition checks it before the pair sum

// ============================================================================
// K3: anterpolation as an owner-computes gather (no atomics).  16 lanes own a quad
// of 4 consecutive level-0 points along z; lane (ox, oy) sums the contributions
// of the particles in its cell column (cells along z in order, particles in
// sorted order), using the per-particle weights of k_gather:
// q_mu += ((q*wx[dx]) * wy[dy]) * wz[dz]  (the reference's qa/qab products,
// src/msm_phases.cpp:52-57), and a fixed xor-shuffle tree adds the 16 lanes.
// One weight fetch serves up to 4 points; the 7 cell ranges are fetched up front.
// ============================================================================
constexpr int kAQ = 4; // points per thread along z
#ifndef MSMB_ANTERP_STREAM_MIN
#define MSMB_ANTERP_STREAM_MIN 4000000
#endif
constexpr int64_t kAnterpStreamMin = MSMB_ANTERP_STREAM_MIN; // level-0 points above which k_anterp_stream runs

#ifndef MSMB_ANTERP_TPB
#define MSMB_ANTERP_TPB 64 // C2-S: 64 0.095, 128 0.096, 256 0.109 ms
#endif
constexpr int kAnterpTpb = MSMB_ANTERP_TPB;
__global__ void __launch_bounds__(kAnterpTpb)
    k_anterp(BinP p, const int2* __restrict__ nat, const double* __restrict__ aw, double* q0,
             int x_begin, int x_end, const ErrRec* err) {
    if (failed(err)) return;
    const int d0 = p.d[0], d1 = p.d[1], d2 = p.d[2];
    const int nzq = (d2 + kAQ - 1) / kAQ;
    // 16 lanes per quad of points, one cell column (ox, oy) each; the partial sums
    // are combined by a fixed xor-shuffle tree over the 16 lanes
    const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int ox = int(tid & 3), oy = int((tid >> 2) & 3);
    const int64_t idx = tid >> 4;
    const bool live = idx < int64_t(x_end - x_begin) * d1 * nzq;
    const int zq = live ? int(idx % nzq) : 0;
    const int y = live ? int((idx / nzq) % d1) : 0;
    const int x = live ? x_begin + int(idx / (int64_t(nzq) * d1)) : 0;
    const int z0 = zq * kAQ;
    double acc[kAQ];
#pragma unroll
    for (int k = 0; k < kAQ; ++k) acc[k] = 0.0;
    const int cx = x - 2 + ox, cy = y - 2 + oy;
    if (live && cx >= 1 && cx <= d0 - 3 && cy >= 1 && cy <= d1 - 3) {
        const int dxw = 3 - ox;     // weight index x - base = x - (cx - 1)
        const int dyw = 4 + 3 - oy;
        const int2* row = nat + (size_t(cx) * d1 + cy) * d2;
        // cells cz = z0 - 2 + u, u = 0 .. kAQ + 2, reach points z0 + k with dz = k - u + 3;
        // all ranges fetched up front (independent loads)
        int2 rg[kAQ + 3];
#pragma unroll
        for (int u = 0; u < kAQ + 3; ++u) {
            const int cz = z0 - 2 + u;
            rg[u] = (cz >= 1 && cz <= d2 - 3) ? __ldg(row + cz) : make_int2(0, 0);
        }
        // the first atom of every cell is fetched up front (one batch of independent
        // loads: ~1.2 atoms per cell, so most atoms), the rest as the cells are summed
        double fx_[kAQ + 3], fy_[kAQ + 3];
        double2 f01[kAQ + 3], f23[kAQ + 3];
#pragma unroll
        for (int u = 0; u < kAQ + 3; ++u) {
            const double* w = aw + size_t(rg[u].x < rg[u].y ? rg[u].x : 0) * 12;
            fx_[u] = __ldg(w + dxw);
            fy_[u] = __ldg(w + dyw);
            f01[u] = __ldg(reinterpret_cast<const double2*>(w + 8));
            f23[u] = __ldg(reinterpret_cast<const double2*>(w + 10));
        }
#pragma unroll
        for (int u = 0; u < kAQ + 3; ++u) {
            if (rg[u].x >= rg[u].y) continue;
            double wxv = fx_[u], wyv = fy_[u];
            double2 wz01 = f01[u], wz23 = f23[u];
            for (int s = rg[u].x;;) {
                const double cxy = __dmul_rn(wxv, wyv);
                const double wzv[4] = {wz01.x, wz01.y, wz23.x, wz23.y};
#pragma unroll
                for (int k = 0; k < kAQ; ++k) {
                    const int dz = k - u + 3;
                    if (dz >= 0 && dz <= 3) acc[k] = fma(cxy, wzv[dz], acc[k]);
                }
                if (++s >= rg[u].y) break;
                const double* w = aw + size_t(s) * 12;
                wxv = __ldg(w + dxw);
                wyv = __ldg(w + dyw);
                wz01 = __ldg(reinterpret_cast<const double2*>(w + 8));
                wz23 = __ldg(reinterpret_cast<const double2*>(w + 10));
            }
        }
    }
#pragma unroll
    for (int k = 0; k < kAQ; ++k) {
        acc[k] += __shfl_xor_sync(FULLMASK, acc[k], 1);
        acc[k] += __shfl_xor_sync(FULLMASK, acc[k], 2);
        acc[k] += __shfl_xor_sync(FULLMASK, acc[k], 4);
        acc[k] += __shfl_xor_sync(FULLMASK, acc[k], 8);
    }
    if (!live || (tid & 15) != 0) return;
    double* out = q0 + (size_t(x) * d1 + y) * d2;
#pragma unroll
    for (int k = 0; k < kAQ; ++k)
        if (z0 + k < d2) out[z0 + k] = acc[k];
}

// Layer-streaming anterpolation (same contributions, coalesced weight traffic):
// a block owns kSX x kSY rows (x, y) of level-0 points over a z-chunk of kSZ
// points.  For every cell layer cz whose stencils reach the chunk, it stages the
// anterpolation weights of the atoms in the footprint cells (x0-2 .. x0+kSX,
// y0-2 .. y0+kSY) in shared memory (each cell's atoms are contiguous in sorted
// order: coalesced copies), then every thread adds them to the 4 points of its
// row that the layer reaches (cz-1 .. cz+2) and retires point cz-1.  Order per
// point: layers ascending, cell offsets (ox, oy), atoms in sorted order --
// deterministic.  A layer with more atoms than the staging buffer reads its
// weights from global memory instead.
#ifndef MSMB_AS_Y
#define MSMB_AS_Y 16
#endif
#ifndef MSMB_AS_Z
#define MSMB_AS_Z 16
#endif
constexpr int kSX = 8, kSY = MSMB_AS_Y, kSZ = MSMB_AS_Z;
constexpr int kSCX = kSX + 3, kSCY = kSY + 3, kSCells = kSCX * kSCY;
constexpr int kSMaxAtoms = kSY == 16 ? 464 : 320; // weights + slot sources: static shared memory under 48 KB

__global__ void __launch_bounds__(kSX * kSY)
    k_anterp_stream(BinP p, const int2* __restrict__ nat, const double* __restrict__ aw, double* q0,
                    int x_begin, int x_end, const ErrRec* err) {
    __shared__ int s_off[kSCells + 1];
    __shared__ int s_beg[kSCells];
    __shared__ double s_w[kSMaxAtoms * 12];
    __shared__ int s_src[kSMaxAtoms];
    __shared__ int s_wsum[kSX * kSY / 32];
    if (failed(err)) return;
    const int d0 = p.d[0], d1 = p.d[1], d2 = p.d[2];
    const int nty = (d1 + kSY - 1) / kSY, ntz = (d2 + kSZ - 1) / kSZ;
    const int bz = blockIdx.x % ntz, by = (blockIdx.x / ntz) % nty, bx = blockIdx.x / (ntz * nty);
    const int x0 = x_begin + bx * kSX, y0 = by * kSY, z0 = bz * kSZ;
    const int z1 = min(z0 + kSZ, d2);
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    const int tx = t / kSY, ty = t % kSY;
    const int x = x0 + tx, y = y0 + ty;
    const bool row_ok = x < x_end && y < d1;
    const int czs = max(1, z0 - 2), cze = min(d2 - 3, z1);
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0; // points pb .. pb + 3, pb = cz - 1
    int pb = czs - 1;
    double* out = q0 + (size_t(x) * d1 + y) * d2;
    for (int cz = czs; cz <= cze; ++cz) {
        // ---- stage the layer: cell ranges, offsets (block scan), weights
        int cnt[2], beg[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int c = t + h * (kSX * kSY);
            cnt[h] = 0;
            beg[h] = 0;
            if (c < kSCells) {
                const int cx = x0 - 2 + c / kSCY, cy = y0 - 2 + c % kSCY;
                if (cx >= 1 && cx <= d0 - 3 && cy >= 1 && cy <= d1 - 3) {
                    const int2 r = __ldg(nat + (size_t(cx) * d1 + cy) * d2 + cz);
                    cnt[h] = r.y - r.x;
                    beg[h] = r.x;
                }
            }
        }
        // exclusive scan over cells t and t + 128 (two passes of a 128-wide block scan)
        int base = 0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            int v = cnt[h], inc = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int u = __shfl_up_sync(FULLMASK, inc, o);
                if (lane >= o) inc += u;
            }
            if (lane == 31) s_wsum[wid] = inc;
            __syncthreads();
            int wpre = 0, tot = 0;
#pragma unroll
            for (int k = 0; k < kSX * kSY / 32; ++k) {
                const int sk = s_wsum[k];
                wpre += k < wid ? sk : 0;
                tot += sk;
            }
            const int c = t + h * (kSX * kSY);
            if (c < kSCells) {
                s_off[c] = base + wpre + inc - v;
                s_beg[c] = beg[h];
            }
            base += tot;
            __syncthreads();
        }
        const int total = base;
        if (t == 0) s_off[kSCells] = total;
        const bool staged = total <= kSMaxAtoms;
        if (staged) {
            // source atom of every staged slot (this thread's two cells), then one flat
            // copy with independent loads (8 in flight per thread)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int c = t + h * (kSX * kSY);
                if (c < kSCells) {
                    const int o = s_off[c];
                    for (int k = 0; k < cnt[h]; ++k) s_src[o + k] = beg[h] + k;
                }
            }
            __syncthreads();
            const int n = 12 * total;
            for (int e0 = t; e0 < n; e0 += 8 * kSX * kSY) {
                double v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int e = e0 + u * kSX * kSY;
                    v[u] = e < n ? __ldg(aw + size_t(s_src[e / 12]) * 12 + e % 12) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (e0 + u * kSX * kSY < n) s_w[e0 + u * kSX * kSY] = v[u];
            }
        }
        __syncthreads();
        // ---- accumulate: this row's 16 footprint cells of the layer
        if (row_ok) {
#pragma unroll
            for (int ox = 0; ox < 4; ++ox) {
#pragma unroll
                for (int oy = 0; oy < 4; ++oy) {
                    const int c = (tx + ox) * kSCY + (ty + oy);
                    const int o = s_off[c];
                    const int n = s_off[c + 1] - o;
                    const double* wp = staged ? s_w + size_t(o) * 12 : aw + size_t(s_beg[c]) * 12;
                    for (int a = 0; a < n; ++a, wp += 12) {
                        const double cxy = __dmul_rn(wp[3 - ox], wp[7 - oy]);
                        acc0 = fma(cxy, wp[8], acc0);
                        acc1 = fma(cxy, wp[9], acc1);
                        acc2 = fma(cxy, wp[10], acc2);
                        acc3 = fma(cxy, wp[11], acc3);
                    }
                }
            }
            if (pb >= z0 && pb < z1) out[pb] = acc0;
        }
        acc0 = acc1;
        acc1 = acc2;
        acc2 = acc3;
        acc3 = 0.0;
        ++pb;
        __syncthreads();
    }
    if (row_ok) { // points the last layers left in the ring
        if (pb >= z0 && pb < z1) out[pb] = acc0;
        if (pb + 1 >= z0 && pb + 1 < z1) out[pb + 1] = acc1;
        if (pb + 2 >= z0 && pb + 2 < z1) out[pb + 2] = acc2;
        if (pb + 3 >= z0 && pb + 3 < z1) out[pb + 3] = acc3;
    }
}

// Tiled scatter anterpolation (MSMB_ANTERP_TILE, the default): one warp per block of
// kTX x kTY x kTZ level-0 cells scatters the atoms of its cells -- cells in
// (x, y, z) order, atoms in sorted order -- into a private shared-memory tile of the
// (kTX+3) x (kTY+3) x (kTZ+3) points they reach, lane (dx, dy, cz) adding the
// products ((q wx[dx]) wy[dy]) wz[cz] and wz[cz + 2] (the reference's qa / qab
// products, src/msm_phases.cpp:52-57) for one atom at a time (__syncwarp between
// atoms orders the read-modify-writes of overlapping stencils).  The tiles are then
// combined per point in block order (k_anterp_combine: at most 2 blocks per axis
// reach a point).  Fixed orders throughout: deterministic, no atomics.  Each atom is
// read once, with the next atom's weights prefetched while the current one is added.
constexpr int kTX = 4, kTY = 4, kTZ = 4;
constexpr int kTPX = kTX + 3, kTPY = kTY + 3, kTPZ = kTZ + 3, kTPts = kTPX * kTPY * kTPZ;

constexpr int kTStage = 32; // atoms staged in shared memory per batch (one per lane)

__global__ void __launch_bounds__(32)
    k_anterp_tile(BinP p, const int2* __restrict__ nat, const int* __restrict__ perm, const double* __restrict__ xs,
                  const double* __restrict__ ys, const double* __restrict__ zs, const double* __restrict__ qs,
                  double* part, int bx0, int nbx, const ErrRec* err) {
    __shared__ double acc[kTPts];
    __shared__ double sw[kTStage * 12]; // the staged atoms' weights (k_gather layout)
    __shared__ int sidx[kTStage];       // their sorted slots
    __shared__ int scl[kTStage];        // their cells (block-local index)
    pdl_enter();
    if (failed(err)) return;
    const int d0 = p.d[0], d1 = p.d[1], d2 = p.d[2];
    const int nby = (d1 + kTY - 1) / kTY, nbz = (d2 + kTZ - 1) / kTZ;
    const int bz = blockIdx.x % nbz, by = (blockIdx.x / nbz) % nby, bx = bx0 + blockIdx.x / (nbz * nby);
    const int X0 = bx * kTX, Y0 = by * kTY, Z0 = bz * kTZ;
    const int lane = threadIdx.x;
    for (int e = lane; e < kTPts; e += 32) acc[e] = 0.0;
    const int dx = lane >> 3, dy = (lane >> 1) & 3, cz = lane & 1;
    constexpr int kCells = kTX * kTY * kTZ;
    for (int cb = 0; cb < kCells; cb += 32) {
        // lane j: cell cb + j of the block, in (x, y, z) order
        int2 rg = make_int2(0, 0);
        {
            const int k = cb + lane;
            const int cx = X0 + k / (kTY * kTZ), cy = Y0 + (k / kTZ) % kTY, czz = Z0 + k % kTZ;
            if (cx >= 1 && cx <= d0 - 3 && cy >= 1 && cy <= d1 - 3 && czz >= 1 && czz <= d2 - 3)
                rg = __ldg(nat + (size_t(cx) * d1 + cy) * d2 + czz);
        }
        const int cnt = max(0, rg.y - rg.x);
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(FULLMASK, incl, o);
            if (lane >= o) incl += v;
        }
        const int excl = incl - cnt, total = __shfl_sync(FULLMASK, incl, 31);
        for (int base = 0; base < total; base += kTStage) {
            const int nst = min(kTStage, total - base);
            __syncwarp();
            for (int k = max(0, base - excl); k < cnt && excl + k < base + kTStage; ++k) {
                sidx[excl + k - base] = rg.x + k;
                scl[excl + k - base] = cb + lane;
            }
            __syncwarp();
            if (lane < nst) { // one staged atom per lane: its weights from its position
                const int i = perm[sidx[lane]];
                anterp_weights(p, xs[i], ys[i], zs[i], qs[i], sw + lane * 12);
            }
            __syncwarp();
            for (int t = 0; t < nst; ++t) {
                const int k = scl[t];
                const int lx = k / (kTY * kTZ), ly = (k / kTZ) % kTY, lz = k % kTZ;
                const double* w = sw + t * 12;
                // the cell's stencil base (cell - 1) in tile coordinates: points lx .. lx + 3
                const int o1 = ((lx + dx) * kTPY + (ly + dy)) * kTPZ + lz + cz;
                const double cxy = __dmul_rn(w[dx], w[4 + dy]);
                const double a1 = __dmul_rn(cxy, w[8 + cz]), a2 = __dmul_rn(cxy, w[10 + cz]);
                acc[o1] += a1;
                acc[o1 + 2] += a2;
                __syncwarp();
            }
        }
    }
    __syncwarp();
    double* out = part + size_t(blockIdx.x) * kTPts;
    for (int e = lane; e < kTPts; e += 32) out[e] = acc[e];
}

// point (x, y, z) of the owned planes = the sum of the tiles of the <= 2 x 2 x 2 blocks
// reaching it, in block order
__global__ void k_anterp_combine(int d0, int d1, int d2, const double* __restrict__ part, int bx0, int nbx,
                                 double* q0, int x_begin, int x_end, const ErrRec* err) {
    pdl_enter();
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t npl = int64_t(d1) * d2;
    if (t >= int64_t(x_end - x_begin) * npl || failed(err)) return;
    const int z = int(t % d2), y = int((t / d2) % d1), x = x_begin + int(t / npl);
    const int nby = (d1 + kTY - 1) / kTY, nbz = (d2 + kTZ - 1) / kTZ;
    // block b reaches points [b*T - 1, b*T + T + 2): b in [floor((x-2)/T), floor((x+1)/T)]
    const int bxb = min(bx0 + nbx - 1, (x + 1) / kTX);
    double s = 0.0;
    for (int bx = max(bx0, (x - 2 + kTX) / kTX - 1); bx <= bxb; ++bx) {
        const int lx = x - (bx * kTX - 1);
        if (lx < 0 || lx >= kTPX) continue;
        for (int by = max(0, (y - 2 + kTY) / kTY - 1); by <= min(nby - 1, (y + 1) / kTY); ++by) {
            const int ly = y - (by * kTY - 1);
            if (ly < 0 || ly >= kTPY) continue;
            for (int bz = max(0, (z - 2 + kTZ) / kTZ - 1); bz <= min(nbz - 1, (z + 1) / kTZ); ++bz) {
                const int lz = z - (bz * kTZ - 1);
                if (lz < 0 || lz >= kTPZ) continue;
                const size_t blk = (size_t(bx - bx0) * nby + by) * nbz + bz;
                s += part[blk * kTPts + (lx * kTPY + ly) * kTPZ + lz];
            }
        }
    }
    q0[(size_t(x) * d1 + y) * d2 + z] = s;
}

size_t anterp_tile_part_doubles(const Geometry& g) {
    const int* d = g.lv[0].dims;
    return size_t((d[0] + kTX - 1) / kTX) * ((d[1] + kTY - 1) / kTY) * ((d[2] + kTZ - 1) / kTZ) * kTPts;
}

int launch_anterp(cudaStream_t st, const Geometry& g, const DevState& sv, DevAtoms& a, DevCells& c, DevLevels& L,
                  ErrRec* err, const Part& P) {
    const BinP p = make_binp(g);
    if (MSMB_ANTERP_TILE && L.anterp_part) {
        // the cell blocks whose atoms reach the owned planes [pl0, pl1): cells pl0 - 2 .. pl1
        const int x0 = P.pl0[0], x1 = P.pl1[0];
        if (x1 <= x0) return 0;
        const int bxa = std::max(0, (x0 - 2) / kTX), bxb = std::min((p.d[0] - 1) / kTX, (x1 + 1) / kTX);
        const int nbx = bxb - bxa + 1;
        const int nby = (p.d[1] + kTY - 1) / kTY, nbz = (p.d[2] + kTZ - 1) / kTZ;
        pdl_launch(k_anterp_tile, dim3(nbx * nby * nbz), dim3(32), 0, st, p, c.nat, a.perm, sv.x, sv.y, sv.z, sv.q,
                   L.anterp_part, bxa, nbx, err);
        const int64_t m = int64_t(x1 - x0) * p.d[1] * p.d[2];
        pdl_launch(k_anterp_combine, dim3(int((m + 255) / 256)), dim3(256), 0, st, p.d[0], p.d[1], p.d[2],
                   L.anterp_part, bxa, nbx, L.charge + g.lv[0].offset, x0, x1, err);
        return 2;
    }
    // large lattices (C3, C4): the layer-streaming kernel (measured 3.2 vs 5.0 ms at C3);
    // small ones (C2): the 16-lane gather has more parallelism (0.099 vs 0.206 ms)
    if (int64_t(g.lv[0].size) > kAnterpStreamMin) {
        const int nx = P.pl1[0] - P.pl0[0];
        if (nx <= 0) return 0;
        const int blocks = ((nx + kSX - 1) / kSX) * ((p.d[1] + kSY - 1) / kSY) * ((p.d[2] + kSZ - 1) / kSZ);
        k_anterp_stream<<<blocks, kSX * kSY, 0, st>>>(p, c.nat, a.aw, L.charge + g.lv[0].offset, P.pl0[0],
                                                       P.pl1[0], err);
        return 1;
    }
    const int64_t m = 16 * int64_t(P.pl1[0] - P.pl0[0]) * p.d[1] * ((p.d[2] + kAQ - 1) / kAQ);
    if (m == 0) return 0;
    k_anterp<<<int((m + kAnterpTpb - 1) / kAnterpTpb), kAnterpTpb, 0, st>>>(p, c.nat, a.aw, L.charge + g.lv[0].offset, P.pl0[0],
                                                   P.pl1[0], err);
    return 1;
}

// ============================================================================
// K4 / K7: restriction and prolongation, reference order (bitwise)
// ============================================================================
struct XferP {
    int fd[3], cd[3];
    const int* base[3];
    const double* w[3];
    const int* rcnt[3];
    const int* ridx[3];
    const double* rw[3];
};

static XferP make_xfer(const Geometry& g, int k, DevLevels& L) {
    XferP p;
    for (int ax = 0; ax < 3; ++ax) {
        p.fd[ax] = g.lv[k].dims[ax];
        p.cd[ax] = g.lv[k + 1].dims[ax];
        p.base[ax] = L.tr_base[k][ax];
        p.w[ax] = L.tr_w[k][ax];
        p.rcnt[ax] = L.tr_rcnt[k][ax];
        p.ridx[ax] = L.tr_ridx[k][ax];
        p.rw[ax] = L.tr_rw[k][ax];
    }
    return p;
}

// Per-point restriction: coarse(I,J,K) = sum over the fine points feeding it in
// row-major order of ((q*wx)*wy)*wz, skipping zero charges -- the order and
// arithmetic of the reference's scatter (src/msm_phases.cpp:67-89), hence bit
// for bit.  `fine_at(i, j, k)` abstracts where the fine values live (global
// memory or a shared-memory tile).
template <class FineAt>
__device__ __forceinline__ double restrict_point(const XferP& p, int I, int J, int K, FineAt fine_at) {
    const int ni = p.rcnt[0][I], nj = p.rcnt[1][J], nk = p.rcnt[2][K];
    int iy[kRestrictMax], iz[kRestrictMax];
    double wy[kRestrictMax], wz[kRestrictMax];
#pragma unroll
    for (int a = 0; a < kRestrictMax; ++a) {
        iy[a] = a < nj ? p.ridx[1][J * kRestrictMax + a] : 0;
        wy[a] = a < nj ? p.rw[1][J * kRestrictMax + a] : 0.0;
        iz[a] = a < nk ? p.ridx[2][K * kRestrictMax + a] : 0;
        wz[a] = a < nk ? p.rw[2][K * kRestrictMax + a] : 0.0;
    }
    double acc = 0.0;
#pragma unroll 1
    for (int a = 0; a < ni; ++a) {
        const int ix = p.ridx[0][I * kRestrictMax + a];
        const double wx = p.rw[0][I * kRestrictMax + a];
#pragma unroll
        for (int b = 0; b < kRestrictMax; ++b) {
            if (b >= nj) break;
            double q[kRestrictMax];
#pragma unroll
            for (int c = 0; c < kRestrictMax; ++c) q[c] = c < nk ? fine_at(ix, iy[b], iz[c]) : 0.0;
#pragma unroll
            for (int c = 0; c < kRestrictMax; ++c) {
                if (c < nk && q[c] != 0.0) {
                    const double qab = __dmul_rn(__dmul_rn(q[c], wx), wy[b]);
                    acc = __dadd_rn(acc, __dmul_rn(qab, wz[c]));
                }
            }
        }
    }
    return acc;
}

// Large levels: a CTA computes a 4x4x8 block of coarse points from a zero-padded
// shared-memory tile of the fine lattice (fine i in [2I0-5, 2(I0+3)+1], etc.).
// Chain kernels in one-warp CTAs (MSMB_CHAIN_SMALL, default off): a CTA of the small
// variants needs <= 4096 registers and <= 16 KB of shared memory, so it fits beside
// the pair kernel's one-warp CTAs.  Measured on C2-S: 0.864 ms/step against 0.849
// with the large CTAs -- the chain does not start earlier (it waits on the
// anterpolation, which follows the sort, not the pair sum) and the small CTAs
// re-read their halos more often.
#ifndef MSMB_CHAIN_SMALL
#define MSMB_CHAIN_SMALL 0
#endif

// xlo/xhi: the coarse x-planes to compute (a spatial-decomposition part's own)
template <bool BITWISE, int kRTx, int kRTy, int kRTz>
__global__ void __launch_bounds__(kRTx * kRTy * kRTz)
    k_restrict_tile(XferP p, const double* __restrict__ fine, double* coarse, const ErrRec* err, int xlo, int xhi,
                    int early) {
    constexpr int kRFx = 2 * kRTx + 6, kRFy = 2 * kRTy + 6, kRFz = 2 * kRTz + 6;
    __shared__ double tile[kRFx * kRFy * kRFz];
    pdl_enter(early);
    if (failed(err)) return;
    const int tz_n = (p.cd[2] + kRTz - 1) / kRTz, ty_n = (p.cd[1] + kRTy - 1) / kRTy;
    const int bz = blockIdx.x % tz_n, by = (blockIdx.x / tz_n) % ty_n, bx = blockIdx.x / (tz_n * ty_n);
    const int I0 = xlo + bx * kRTx, J0 = by * kRTy, K0 = bz * kRTz;
    const int fi0 = 2 * I0 - 5, fj0 = 2 * J0 - 5, fk0 = 2 * K0 - 5;
    constexpr int kTile = kRFx * kRFy * kRFz;
    // the whole tile in one batch of asynchronous 8-byte copies (zero-filled outside
    // the lattice): one memory latency instead of one per round of register loads
    for (int e = threadIdx.x; e < kTile; e += blockDim.x) {
        const int kk = e % kRFz, jj = (e / kRFz) % kRFy, ii = e / (kRFz * kRFy);
        const int i = fi0 + ii, j = fj0 + jj, k = fk0 + kk;
        const bool in = i >= 0 && i < p.fd[0] && j >= 0 && j < p.fd[1] && k >= 0 && k < p.fd[2];
        const double* src = in ? fine + (size_t(i) * p.fd[1] + j) * p.fd[2] + k : fine;
        const unsigned dst = unsigned(__cvta_generic_to_shared(tile + e));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src), "r"(in ? 8 : 0));
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    const int tz = threadIdx.x % kRTz, ty = (threadIdx.x / kRTz) % kRTy, tx = threadIdx.x / (kRTz * kRTy);
    const int I = I0 + tx, J = J0 + ty, K = K0 + tz;
    if (I >= xhi || J >= p.cd[1] || K >= p.cd[2]) return;
    double v;
    if (BITWISE) {
        v = restrict_point(p, I, J, K, [&](int i, int j, int k) {
            return tile[((i - fi0) * kRFy + (j - fj0)) * kRFz + (k - fk0)];
        });
    } else {
        // production: sum_a wx[a] (sum_b wy[b] (sum_c wz[c] q)) with FMA -- exact in exact
        // arithmetic, ~1e-16 relative from the reference's scatter order (tolerance-tested)
        const int ni = p.rcnt[0][I], nj = p.rcnt[1][J], nk = p.rcnt[2][K];
        int lz[kRestrictMax];
        double wz[kRestrictMax];
#pragma unroll
        for (int c = 0; c < kRestrictMax; ++c) {
            lz[c] = c < nk ? p.ridx[2][K * kRestrictMax + c] - fk0 : 0;
            wz[c] = c < nk ? p.rw[2][K * kRestrictMax + c] : 0.0;
        }
        // all table entries up front (independent loads), zero weights pad to kRestrictMax
        int lx[kRestrictMax], ly[kRestrictMax];
        double wx[kRestrictMax], wy[kRestrictMax];
#pragma unroll
        for (int c = 0; c < kRestrictMax; ++c) {
            lx[c] = c < ni ? p.ridx[0][I * kRestrictMax + c] - fi0 : 0;
            wx[c] = c < ni ? p.rw[0][I * kRestrictMax + c] : 0.0;
            ly[c] = c < nj ? p.ridx[1][J * kRestrictMax + c] - fj0 : 0;
            wy[c] = c < nj ? p.rw[1][J * kRestrictMax + c] : 0.0;
        }
        double acc = 0.0;
#pragma unroll 1
        for (int a = 0; a < ni; ++a) {
            double accb = 0.0;
#pragma unroll
            for (int b = 0; b < kRestrictMax; ++b) {
                if (b < nj) {
                    const double* row = tile + (lx[a] * kRFy + ly[b]) * kRFz;
                    double accc = 0.0;
#pragma unroll
                    for (int c = 0; c < kRestrictMax; ++c) accc = fma(wz[c], row[lz[c]], accc); // wz = 0 pads
                    accb = fma(wy[b], accc, accb);
                }
            }
            acc = fma(wx[a], accb, acc);
        }
        v = acc;
    }
    coarse[(size_t(I) * p.cd[1] + J) * p.cd[2] + K] = v;
}

// fine(i,j,k) += sum_a wx[a] (sum_b wy[b] (sum_c wz[c] u_coarse)) (src/msm_phases.cpp:177-189)
__device__ __forceinline__ void prolong_point(const XferP& p, const double* __restrict__ coarse,
                                              double* fine, int64_t idx) {
    const int k = int(idx % p.fd[2]);
    const int j = int((idx / p.fd[2]) % p.fd[1]);
    const int i = int(idx / (int64_t(p.fd[2]) * p.fd[1]));
    const int bx = p.base[0][i], by = p.base[1][j], bz = p.base[2][k];
    const double* wx = p.w[0] + 4 * i;
    const double* wy = p.w[1] + 4 * j;
    const double* wz = p.w[2] + 4 * k;
    double acc = 0.0;
    for (int a = 0; a < 4; ++a) {
        double accb = 0.0;
        for (int b = 0; b < 4; ++b) {
            const double* row = coarse + (size_t(bx + a) * p.cd[1] + (by + b)) * p.cd[2] + bz;
            double accc = 0.0;
            for (int c = 0; c < 4; ++c) accc = __dadd_rn(accc, __dmul_rn(wz[c], row[c]));
            accb = __dadd_rn(accb, __dmul_rn(wy[b], accc));
        }
        acc = __dadd_rn(acc, __dmul_rn(wx[a], accb));
    }
    fine[idx] = __dadd_rn(fine[idx], acc);
}

__global__ void k_prolong(XferP p, const double* __restrict__ coarse, double* fine,
                          const ErrRec* err) {
    const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t m = int64_t(p.fd[0]) * p.fd[1] * p.fd[2];
    if (idx >= m || failed(err)) return;
    prolong_point(p, coarse, fine, idx);
}

template <int TX, int TY, int TZ>
static int restrict_blocks(const XferP& p, int nx) {
    return ((nx + TX - 1) / TX) * ((p.cd[1] + TY - 1) / TY) * ((p.cd[2] + TZ - 1) / TZ);
}

int launch_restrict_all(cudaStream_t st, const Geometry& g, DevLevels& L, ErrRec* err) {
    int l = 0;
    for (int k = 0; k + 1 < g.levels; ++k) {
        // the next level's restriction is a few CTAs: let them be admitted while this one runs
        int early = 0;
        if (k + 2 < g.levels && !MSMB_CHAIN_SMALL) {
            const XferP pn = make_xfer(g, k + 1, L);
            early = restrict_blocks<4, 4, 8>(pn, g.lv[k + 2].dims[0]) <= kPdlEarlyMaxBlocks;
        }
        l += launch_restrict_planes(st, g, k, L, err, 0, g.lv[k + 1].dims[0], early);
    }
    return l;
}

// production restriction k -> k+1 of the coarse x-planes [xlo, xhi)
int launch_restrict_planes(cudaStream_t st, const Geometry& g, int k, DevLevels& L, ErrRec* err, int xlo, int xhi,
                           int early) {
    const XferP p = make_xfer(g, k, L);
    if (xhi <= xlo) return 0;
    if (MSMB_CHAIN_SMALL)
        pdl_launch(k_restrict_tile<false, 2, 4, 4>, dim3(restrict_blocks<2, 4, 4>(p, xhi - xlo)), dim3(32), 0, st, p,
                   L.charge + g.lv[k].offset, L.charge + g.lv[k + 1].offset, err, xlo, xhi, early);
    else
        pdl_launch(k_restrict_tile<false, 4, 4, 8>, dim3(restrict_blocks<4, 4, 8>(p, xhi - xlo)), dim3(128), 0, st, p,
                   L.charge + g.lv[k].offset, L.charge + g.lv[k + 1].offset, err, xlo, xhi, early);
    return 1;
}

// bit-exact restriction of one level (msmb_debug_stage; tests/test_gpu_stages.py)
int launch_restrict(cudaStream_t st, const Geometry& g, int k, DevLevels& L, ErrRec* err) {
    const XferP p = make_xfer(g, k, L);
    k_restrict_tile<true, 4, 4, 8><<<restrict_blocks<4, 4, 8>(p, p.cd[0]), 128, 0, st>>>(
        p, L.charge + g.lv[k].offset, L.charge + g.lv[k + 1].offset, err, 0, p.cd[0], 0);
    return 1;
}

// Prolongation by fine tiles of 4 x 8 x 8 points: the coarse window they read
// (base .. base + 3 per axis, monotone in the fine index) is staged in shared
// memory, then each point forms the reference's nested sums (prolong_point order).

// xlo/xhi: the fine x-planes to update (a spatial-decomposition part's own)
template <int kPx, int kPy, int kPz>
__global__ void __launch_bounds__(kPx * kPy * kPz)
    k_prolong_tile(XferP p, const double* __restrict__ coarse, double* fine, const ErrRec* err, int xlo, int xhi,
                   int early) {
    constexpr int kPCx = kPx / 2 + 5, kPCy = kPy / 2 + 5, kPCz = kPz / 2 + 5;
    __shared__ double ct[kPCx * kPCy * kPCz];
    pdl_enter(early);
    if (failed(err)) return;
    const int tz_n = (p.fd[2] + kPz - 1) / kPz, ty_n = (p.fd[1] + kPy - 1) / kPy;
    const int bz = blockIdx.x % tz_n, by = (blockIdx.x / tz_n) % ty_n, bx = blockIdx.x / (tz_n * ty_n);
    const int I0 = xlo + bx * kPx, J0 = by * kPy, K0 = bz * kPz;
    const int I1 = min(I0 + kPx, xhi) - 1, J1 = min(J0 + kPy, p.fd[1]) - 1, K1 = min(K0 + kPz, p.fd[2]) - 1;
    const int cx0 = p.base[0][I0], cy0 = p.base[1][J0], cz0 = p.base[2][K0];
    const int nx = p.base[0][I1] + 4 - cx0, ny = p.base[1][J1] + 4 - cy0, nz = p.base[2][K1] + 4 - cz0;
    if (nx > kPCx || ny > kPCy || nz > kPCz) { // not expected (base ~ i/2); stay exact without staging
        const int tz = threadIdx.x % kPz, ty = (threadIdx.x / kPz) % kPy, tx = threadIdx.x / (kPz * kPy);
        if (I0 + tx <= I1 && J0 + ty <= J1 && K0 + tz <= K1)
            prolong_point(p, coarse, fine, (int64_t(I0 + tx) * p.fd[1] + (J0 + ty)) * p.fd[2] + (K0 + tz));
        return;
    }
    for (int e = threadIdx.x; e < nx * ny * nz; e += blockDim.x) {
        const int c = e % nz, b = (e / nz) % ny, a = e / (nz * ny);
        ct[e] = coarse[(size_t(cx0 + a) * p.cd[1] + (cy0 + b)) * p.cd[2] + (cz0 + c)];
    }
    __syncthreads();
    const int tz = threadIdx.x % kPz, ty = (threadIdx.x / kPz) % kPy, tx = threadIdx.x / (kPz * kPy);
    const int i = I0 + tx, j = J0 + ty, k = K0 + tz;
    if (i > I1 || j > J1 || k > K1) return;
    const int ox = p.base[0][i] - cx0, oy = p.base[1][j] - cy0, oz = p.base[2][k] - cz0;
    const double* wx = p.w[0] + 4 * i;
    const double* wy = p.w[1] + 4 * j;
    const double* wz = p.w[2] + 4 * k;
    double x4[4], y4[4], z4[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) x4[t] = wx[t], y4[t] = wy[t], z4[t] = wz[t];
    double acc = 0.0;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        double accb = 0.0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const double* row = ct + ((ox + a) * ny + (oy + b)) * nz + oz;
            double accc = 0.0;
#pragma unroll
            for (int c = 0; c < 4; ++c) accc = __dadd_rn(accc, __dmul_rn(z4[c], row[c]));
            accb = __dadd_rn(accb, __dmul_rn(y4[b], accc));
        }
        acc = __dadd_rn(acc, __dmul_rn(x4[a], accb));
    }
    const size_t idx = (size_t(i) * p.fd[1] + j) * p.fd[2] + k;
    fine[idx] = __dadd_rn(fine[idx], acc);
}

static int prolong_blocks(const Geometry& g, int k) {
    const int* d = g.lv[k].dims;
    return MSMB_CHAIN_SMALL ? d[0] * ((d[1] + 3) / 4) * ((d[2] + 7) / 8)
                            : ((d[0] + 3) / 4) * ((d[1] + 7) / 8) * ((d[2] + 7) / 8);
}

int launch_prolong(cudaStream_t st, const Geometry& g, int k, DevLevels& L, ErrRec* err) {
    // the next prolongation (k - 1) is a few CTAs: let them be admitted while this one runs
    const int early = k > 0 && prolong_blocks(g, k - 1) <= kPdlEarlyMaxBlocks;
    return launch_prolong_planes(st, g, k, L, err, 0, g.lv[k].dims[0], early);
}

// prolongation k+1 -> k into the fine x-planes [xlo, xhi)
int launch_prolong_planes(cudaStream_t st, const Geometry& g, int k, DevLevels& L, ErrRec* err, int xlo, int xhi,
                          int early) {
    const XferP p = make_xfer(g, k, L);
    if (xhi <= xlo) return 0;
    auto go = [&](auto kern, int px, int py, int pz) {
        const int blocks = ((xhi - xlo + px - 1) / px) * ((p.fd[1] + py - 1) / py) * ((p.fd[2] + pz - 1) / pz);
        pdl_launch(kern, dim3(blocks), dim3(px * py * pz), 0, st, p, L.pot + g.lv[k + 1].offset, L.pot + g.lv[k].offset,
                   err, xlo, xhi, early);
    };
    if (MSMB_CHAIN_SMALL)
        go(k_prolong_tile<1, 4, 8>, 1, 4, 8);
    else
        go(k_prolong_tile<4, 8, 8>, 4, 8, 8);
    return 1;
}

// (The small levels chained in one single-block launch measured slower: C2-S prolong
// 0.037 -> 0.078 ms, one SM cannot hide the per-point load latency.)
int launch_prolong_all(cudaStream_t st, const Geometry& g, DevLevels& L, ErrRec* err) {
    int l = 0;
    for (int k = g.levels - 2; k >= 0; --k) l += launch_prolong(st, g, k, L, err);
    return l;
}

// ============================================================================
// K5 / K6: 3-D stencil convolution u(t) = sum_d K(d) q(t - d), clipped at the
// lattice edges (no wrap, src/msm_phases.cpp:119-121).  CTA = 32 y-rows (one
// per lane) x (kConvNWZ warps x kConvB consecutive z) at one x-plane.  For each
// source plane the CTA stages a zero-padded (y, z) slab in shared memory; the
// odd row pitch makes the lane-per-row loads conflict-free.  Each thread keeps
// kConvB accumulators and a rolling register window along z, so one shared
// load feeds up to kConvL FMAs.
// ============================================================================
struct ConvJob {
    const double* q;
    double* u;
    const int4* rows;
    const int* dxb;
    const double* taps;
    int d0, d1, d2;
    int Rx, Ry, Rz;
    int ty, tz;
    int blk0;
    int P, SY, SZ;
};

struct ConvJobs {
    ConvJob j[kMaxLevels];
    int njobs;
};

template <int B, int L, int NWZ>
__global__ void __launch_bounds__(32 * NWZ) k_conv(ConvJobs J, const ErrRec* err) {
    extern __shared__ double slab[];
    if (failed(err)) return;
    int b = blockIdx.x;
    int jj = 0;
    while (jj + 1 < J.njobs && b >= J.j[jj + 1].blk0) ++jj;
    const ConvJob jb = J.j[jj];
    b -= jb.blk0;
    const int tzi = b % jb.tz;
    const int rest = b / jb.tz;
    const int tyi = rest % jb.ty;
    const int x = rest / jb.ty;
    const int y0 = tyi * 32, z0 = tzi * (B * NWZ);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int zw = z0 + w * B; // first output z of this warp
    double acc[B];
#pragma unroll
    for (int i = 0; i < B; ++i) acc[i] = 0.0;
    const int ylo = y0, yhi = min(y0 + 31, jb.d1 - 1);
    for (int dx = -jb.Rx; dx <= jb.Rx; ++dx) {
        const int xs = x - dx;
        if (xs < 0 || xs >= jb.d0) continue;
        const int r0 = jb.dxb[dx + jb.Rx], r1 = jb.dxb[dx + jb.Rx + 1];
        if (r0 == r1) continue;
        __syncthreads();
        const double* plane = jb.q + size_t(xs) * jb.d1 * jb.d2;
        for (int r = w; r < jb.SY; r += NWZ) { // warp per slab row, lanes along z (coalesced)
            const int ys = y0 - jb.Ry + r;
            const bool yok = ys >= 0 && ys < jb.d1;
            const double* src = plane + size_t(yok ? ys : 0) * jb.d2;
            for (int cc = lane; cc < jb.SZ; cc += 32) {
                const int zs = z0 - jb.Rz + cc;
                slab[r * jb.P + cc] = (yok && zs >= 0 && zs < jb.d2) ? src[zs] : 0.0;
            }
        }
        __syncthreads();
        for (int r = r0; r < r1; ++r) {
            const int4 row = jb.rows[r]; // dx, dy, m, tap_off
            const int dy = row.y, m = row.z;
            if (ylo - dy > jb.d1 - 1 || yhi - dy < 0) continue; // no source row in range
            // chunks whose sources z - dz (dz = -m + t) intersect [0, d2)
            const int nch = (2 * m + L) / L;
            // output z uses source z + j - m for tap j; keep the chunks whose
            // sources reach [0, d2) for some z in [zw, zw + B)
            const int jlo = max(0, m - zw - B + 1);
            const int jhi = min(nch * L - 1, jb.d2 - 1 + m - zw);
            if (jlo > jhi) continue;
            const int c_lo = jlo / L, c_hi = jhi / L;
            const double* srow = slab + (lane - dy + jb.Ry) * jb.P + (w * B + jb.Rz - m);
            const double* tp = jb.taps + row.w;
            double win[B + L - 1];
#pragma unroll
            for (int i = 0; i < B + L - 1; ++i) win[i] = srow[c_lo * L + i];
            for (int c = c_lo; c <= c_hi; ++c) {
                double t[L];
#pragma unroll
                for (int j = 0; j < L; ++j) t[j] = __ldg(tp + c * L + j);
#pragma unroll
                for (int j = 0; j < L; ++j)
#pragma unroll
                    for (int bb = 0; bb < B; ++bb) acc[bb] = fma(t[j], win[j + bb], acc[bb]);
                if (c < c_hi) {
#pragma unroll
                    for (int i = 0; i < B - 1; ++i) win[i] = win[i + L];
#pragma unroll
                    for (int i = B - 1; i < B + L - 1; ++i) win[i] = srow[(c + 1) * L + i];
                }
            }
        }
    }
    const int y = y0 + lane;
    if (y < jb.d1) {
        double* out = jb.u + (size_t(x) * jb.d1 + y) * jb.d2;
#pragma unroll
        for (int bb = 0; bb < B; ++bb) {
            const int z = zw + bb;
            if (z < jb.d2) out[z] = acc[bb];
        }
    }
}

static ConvJob make_job(const ConvTable& t, const LevelGeom& lv, const double* q, double* u,
                        const int4* rows, const int* dxb, const double* taps, int blk0, int Z) {
    ConvJob j;
    j.q = q;
    j.u = u;
    j.rows = rows;
    j.dxb = dxb;
    j.taps = taps;
    j.d0 = lv.dims[0];
    j.d1 = lv.dims[1];
    j.d2 = lv.dims[2];
    j.Rx = t.Rx;
    j.Ry = t.Ry;
    j.Rz = t.Rz;
    j.ty = (j.d1 + 31) / 32;
    j.tz = (j.d2 + Z - 1) / Z;
    j.blk0 = blk0;
    j.SY = 32 + 2 * t.Ry;
    j.SZ = Z + 2 * t.Rz + kConvL;
    j.P = j.SZ | 1;
    return j;
}

// Two stencil variants: 16 outputs per thread (large lattices: fewest loads per
// FMA) and 8 outputs per thread (small lattices: twice the CTAs).
constexpr int kConvBSmall = 8;

size_t conv_smem_bytes(const ConvTable& t) {
    const int SY = 32 + 2 * t.Ry;
    const int SZ = kConvZ + 2 * t.Rz + kConvL;
    return size_t(SY) * size_t(SZ | 1) * sizeof(double);
}

cudaError_t conv_prepare(size_t bytes) {
    const int b = int(std::max<size_t>(bytes, 48 * 1024));
    cudaError_t e = smem_grow(reinterpret_cast<const void*>(k_conv<kConvB, kConvL, kConvNWZ>), size_t(b));
    if (e != cudaSuccess) return e;
    return smem_grow(reinterpret_cast<const void*>(k_conv<kConvBSmall, kConvL, kConvNWZ>), size_t(b));
}

static int launch_conv_jobs(cudaStream_t st, ConvJobs& J, int blocks, bool big, const ErrRec* err) {
    size_t smem = 0;
    for (int i = 0; i < J.njobs; ++i) smem = std::max(smem, size_t(J.j[i].SY) * J.j[i].P * sizeof(double));
    if (big)
        k_conv<kConvB, kConvL, kConvNWZ><<<blocks, 32 * kConvNWZ, smem, st>>>(J, err);
    else
        k_conv<kConvBSmall, kConvL, kConvNWZ><<<blocks, 32 * kConvNWZ, smem, st>>>(J, err);
    return 1;
}

// ----------------------------------------------------------------------------
// K5 (lattice cutoff, levels 0..l-2): one warp per tile of 4 x-planes x 32 y-rows
// (a lane each) x 8 consecutive z.  For every source x-plane the warp stages a
// zero-padded (y, z) slab in shared memory (odd pitch: the lane-per-row loads are
// conflict-free) and, for every dy, slides a register window along z in 4-tap
// chunks; each window chunk feeds all 4 output planes (their own dx rows of the
// stencil), so one shared-memory load serves up to 4 x 8 x 4 = 128 FMAs.  Chunks
// where no plane has a nonzero tap are skipped.  The stencil is the level-0 table
// in absolute-dz layout; level k is scaled by 2^-k, which is exact (see
// msmb_geometry.cpp).  Large grids run one warp per tile; small ones split the
// source planes over S warps and a second kernel adds the S partial lattices in
// fixed order (deterministic).
// ----------------------------------------------------------------------------
constexpr int kLB = 8, kLP = 4, kLC = 4;
constexpr int kLatConstRows = 320, kLatConstTW = 24; // constant-memory capacity (R <= 10)
__constant__ double c_lat_taps[kLatConstRows * kLatConstTW];
__constant__ int2 c_lat_chunks[kLatConstRows];

struct LatJob {
    const double* q;
    double* out;
    int d0, d1, d2;
    int tzn, tyn;
    int blk0;      // first tile index of this job
    int x0;        // first owned output plane (multiple of 4)
    double scale;  // 2^-k
    size_t off;    // lattice offset (partials)
};

struct LatJobs {
    LatJob j[kMaxLevels];
    int n, S, R, TW, SZ, P;
    const int* rowidx;
    const int2* rowchunks;
    const double* taps;
    double* partial;     // S * lattice_total (S > 1)
    size_t pstride;      // lattice_total
};

template <bool CONST_TABLE>
__global__ void __launch_bounds__(32) k_lattice(LatJobs J, const ErrRec* err) {
    extern __shared__ double slab[];
    if (failed(err)) return;
    const int lane = threadIdx.x;
    const int split = blockIdx.x % J.S;
    int t = blockIdx.x / J.S;
    int jj = 0;
    while (jj + 1 < J.n && t >= J.j[jj + 1].blk0) ++jj;
    const LatJob jb = J.j[jj];
    t -= jb.blk0;
    const int tz = t % jb.tzn, rest = t / jb.tzn;
    const int ty = rest % jb.tyn, tx = rest / jb.tyn;
    const int x0 = jb.x0 + tx * kLP, y0 = ty * 32, z0 = tz * kLB;
    const int R = J.R, W = 2 * J.R + 1, SY = 32 + 2 * J.R;
    int xs_lo = max(0, x0 - R), xs_hi = min(jb.d0 - 1, x0 + kLP - 1 + R);
    {
        const int cnt = xs_hi - xs_lo + 1, per = (cnt + J.S - 1) / J.S;
        xs_lo += split * per;
        xs_hi = min(xs_hi, xs_lo + per - 1);
    }
    double acc[kLP][kLB];
#pragma unroll
    for (int p = 0; p < kLP; ++p)
#pragma unroll
        for (int b = 0; b < kLB; ++b) acc[p][b] = 0.0;
    for (int xs = xs_lo; xs <= xs_hi; ++xs) {
        // row ids of the 4 planes for every dy: lane (dy + R) fetches, shuffles broadcast
        int rid[kLP], rlo[kLP], rhi[kLP];
#pragma unroll
        for (int p = 0; p < kLP; ++p) {
            const int dxp = x0 + p - xs;
            int r = -1;
            if (lane < W && dxp >= -R && dxp <= R) r = __ldg(J.rowidx + (dxp + R) * W + lane);
            int2 ch = make_int2(1 << 30, -1);
            if (r >= 0) ch = CONST_TABLE ? c_lat_chunks[r] : __ldg(J.rowchunks + r);
            rid[p] = r;
            rlo[p] = ch.x;
            rhi[p] = ch.y;
        }
        __syncwarp();
        const double* plane = jb.q + size_t(xs) * jb.d1 * jb.d2;
        for (int r = 0; r < SY; ++r) {
            const int ys = y0 - R + r;
            const bool yok = ys >= 0 && ys < jb.d1;
            for (int cc = lane; cc < J.SZ; cc += 32) {
                const int zs = z0 - R + cc;
                slab[r * J.P + cc] = (yok && zs >= 0 && zs < jb.d2) ? plane[size_t(ys) * jb.d2 + zs] : 0.0;
            }
        }
        __syncwarp();
        for (int dy = -R; dy <= R; ++dy) {
            int rp[kLP], cl[kLP], ch[kLP];
            int cmin = 1 << 30, cmax = -1;
#pragma unroll
            for (int p = 0; p < kLP; ++p) {
                rp[p] = __shfl_sync(FULLMASK, rid[p], dy + R);
                cl[p] = __shfl_sync(FULLMASK, rlo[p], dy + R);
                ch[p] = __shfl_sync(FULLMASK, rhi[p], dy + R);
                cmin = min(cmin, cl[p]);
                cmax = max(cmax, ch[p]);
            }
            if (cmax < 0) continue;
            // lane's source row y - dy sits at slab row lane - dy + R; sources z0 + b + dz
            // (dz = -R + 4c + j) at slab column b + 4c + j
            const double* srow = slab + (lane - dy + R) * J.P;
            double win[kLB + kLC - 1];
#pragma unroll
            for (int i = 0; i < kLB + kLC - 1; ++i) win[i] = srow[kLC * cmin + i];
            for (int c = cmin; c <= cmax; ++c) {
#pragma unroll
                for (int p = 0; p < kLP; ++p) {
                    if (c < cl[p] || c > ch[p]) continue;
                    double tv[kLC];
                    if (CONST_TABLE) {
#pragma unroll
                        for (int j = 0; j < kLC; ++j) tv[j] = c_lat_taps[rp[p] * kLatConstTW + kLC * c + j];
                    } else {
                        const double2 t01 = __ldg(reinterpret_cast<const double2*>(J.taps + size_t(rp[p]) * J.TW + kLC * c));
                        const double2 t23 = __ldg(reinterpret_cast<const double2*>(J.taps + size_t(rp[p]) * J.TW + kLC * c + 2));
                        tv[0] = t01.x;
                        tv[1] = t01.y;
                        tv[2] = t23.x;
                        tv[3] = t23.y;
                    }
#pragma unroll
                    for (int j = 0; j < kLC; ++j)
#pragma unroll
                        for (int b = 0; b < kLB; ++b) acc[p][b] = fma(tv[j], win[j + b], acc[p][b]);
                }
                if (c < cmax) {
#pragma unroll
                    for (int i = 0; i < kLB - 1; ++i) win[i] = win[i + kLC];
#pragma unroll
                    for (int i = kLB - 1; i < kLB + kLC - 1; ++i) win[i] = srow[kLC * (c + 1) + i];
                }
            }
        }
    }
    const int y = y0 + lane;
    if (y >= jb.d1) return;
#pragma unroll
    for (int p = 0; p < kLP; ++p) {
        const int x = x0 + p;
        if (x >= jb.d0) break;
        const size_t rowoff = (size_t(x) * jb.d1 + y) * jb.d2;
#pragma unroll
        for (int b = 0; b < kLB; ++b) {
            const int z = z0 + b;
            if (z >= jb.d2) break;
            if (J.S == 1)
                jb.out[rowoff + z] = acc[p][b] * jb.scale;
            else
                J.partial[split * J.pstride + jb.off + rowoff + z] = acc[p][b];
        }
    }
}

// u = 2^-k * (((p_0 + p_1) + p_2) + ...) over the S partial lattices (fixed order)
__global__ void k_lattice_reduce(LatJobs J, int64_t total, const ErrRec* err) {
    if (failed(err)) return;
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= total) return;
    int jj = 0;
    while (jj + 1 < J.n && size_t(i) >= J.j[jj + 1].off) ++jj;
    const LatJob& jb = J.j[jj];
    const size_t local = size_t(i) - jb.off;
    double s = J.partial[jb.off + local];
    for (int k = 1; k < J.S; ++k) s += J.partial[k * J.pstride + jb.off + local];
    jb.out[local] = s * jb.scale;
}

size_t lattice_smem_bytes(const Geometry& g) {
    if (g.levels < 2) return 0;
    const int SY = 32 + 2 * g.lat.R, SZ = g.lat.TW + kLB - 1;
    return size_t(SY) * size_t(SZ | 1) * sizeof(double);
}

cudaError_t lattice_prepare(size_t bytes) {
    cudaError_t e = smem_grow(reinterpret_cast<const void*>(k_lattice<true>), bytes);
    if (e != cudaSuccess) return e;
    return smem_grow(reinterpret_cast<const void*>(k_lattice<false>), bytes);
}

bool lattice_const_fits(const Geometry& g) {
    return g.levels >= 2 && g.lat.nrows <= kLatConstRows && g.lat.TW <= kLatConstTW;
}

// Copies the level-0 stencil into constant memory (the constant bank is global to
// the module: the last field that uploads wins; engine.cu re-uploads per evaluation
// when fields with different stencils share a process -- see Workspace::lat_key).
cudaError_t lattice_upload_const(const Geometry& g, cudaStream_t st) {
    if (!lattice_const_fits(g)) return cudaSuccess;
    std::vector<double> taps(size_t(kLatConstRows) * kLatConstTW, 0.0);
    for (int r = 0; r < g.lat.nrows; ++r)
        for (int i = 0; i < g.lat.TW; ++i) taps[size_t(r) * kLatConstTW + i] = g.lat.taps[size_t(r) * g.lat.TW + i];
    std::vector<int2> ch(kLatConstRows, make_int2(0, -1));
    for (int r = 0; r < g.lat.nrows; ++r) ch[r] = make_int2(g.lat.rowchunks[r].x, g.lat.rowchunks[r].y);
    cudaError_t e = cudaMemcpyToSymbolAsync(c_lat_taps, taps.data(), taps.size() * sizeof(double), 0,
                                            cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return e;
    e = cudaMemcpyToSymbolAsync(c_lat_chunks, ch.data(), ch.size() * sizeof(int2), 0, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return e;
    return cudaStreamSynchronize(st);
}

int lattice_splits(const Geometry& g) {
    if (g.levels < 2) return 1;
    int64_t tiles = 0;
    for (int k = 0; k + 1 < g.levels; ++k) {
        const LevelGeom& lv = g.lv[k];
        tiles += int64_t((lv.dims[0] + kLP - 1) / kLP) * ((lv.dims[1] + 31) / 32) * ((lv.dims[2] + kLB - 1) / kLB);
    }
    const int64_t target = 148 * 16; // ~16 warps per SM
    return int(std::max<int64_t>(1, std::min<int64_t>(8, (target + tiles - 1) / tiles)));
}

int launch_lattice(cudaStream_t st, const Geometry& g, DevLevels& L, ErrRec* err, const Part& P) {
    if (g.levels < 2) return 0;
    LatJobs J;
    J.n = 0;
    J.S = L.lat_S;
    J.R = g.lat.R;
    J.TW = g.lat.TW;
    J.SZ = g.lat.TW + kLB - 1;
    J.P = J.SZ | 1;
    J.rowidx = L.lat_rowidx;
    J.rowchunks = L.lat_rowchunks;
    J.taps = L.lat_taps;
    J.partial = L.lat_partial;
    J.pstride = g.lattice_total;
    int tiles = 0;
    int64_t total = 0;
    for (int k = 0; k + 1 < g.levels; ++k) {
        const LevelGeom& lv = g.lv[k];
        LatJob j;
        j.q = L.charge + lv.offset;
        j.out = L.pot + lv.offset;
        j.d0 = lv.dims[0];
        j.d1 = lv.dims[1];
        j.d2 = lv.dims[2];
        j.tzn = (j.d2 + kLB - 1) / kLB;
        j.tyn = (j.d1 + 31) / 32;
        j.blk0 = tiles;
        j.x0 = P.pl0[k];
        j.scale = std::ldexp(1.0, -k);
        j.off = lv.offset;
        tiles += ((P.pl1[k] - P.pl0[k] + kLP - 1) / kLP) * j.tyn * j.tzn;
        total = int64_t(lv.offset + lv.size);
        J.j[J.n++] = j;
    }
    if (tiles == 0) return 0;
    const size_t smem = lattice_smem_bytes(g);
    if (L.lat_const)
        k_lattice<true><<<tiles * J.S, 32, smem, st>>>(J, err);
    else
        k_lattice<false><<<tiles * J.S, 32, smem, st>>>(J, err);
    if (J.S == 1) return 1;
    k_lattice_reduce<<<int((total + 255) / 256), 256, 0, st>>>(J, total, err);
    return 2;
}

// Small top levels: one thread per target point, a dense sum over every source
// point in ascending row-major order with the reference's mul-then-add
// (src/msm_phases.cpp:153-160); kernel values come from the offset table, which
// equals the reference's per-pair g(norm(coords[mu]-coords[nu])) whenever the
// grid coordinates are exact (msmb_geometry.cpp build_top_table).
__global__ void __launch_bounds__(128)
    k_top_direct(const double* __restrict__ q, double* u, int d0, int d1, int d2,
                 const double* __restrict__ taps, int rowlen, const ErrRec* err) {
    if (failed(err)) return;
    const int64_t m = int64_t(d0) * d1 * d2;
    const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= m) return;
    const int z = int(idx % d2);
    const int y = int((idx / d2) % d1);
    const int x = int(idx / (int64_t(d2) * d1));
    const int Rx = d0 - 1, Ry = d1 - 1, Rz = d2 - 1;
    double acc = 0.0;
    for (int xs = 0; xs < d0; ++xs)
        for (int ys = 0; ys < d1; ++ys) {
            const double* trow = taps + size_t((x - xs + Rx) * (2 * Ry + 1) + (y - ys + Ry)) * rowlen + (z + Rz);
            const double* qrow = q + (size_t(xs) * d1 + ys) * d2;
            for (int zs = 0; zs < d2; ++zs) acc = __dadd_rn(acc, __dmul_rn(__ldg(trow - zs), __ldg(qrow + zs)));
        }
    u[idx] = acc;
}

constexpr int64_t kTopDirectMax = 8192; // top levels up to this many points use k_top_direct

// k_top_direct with the offset table and the charges staged in shared memory (when
// they fit): the same sequential sum per point, without global-load latency in its
// dependent chain.
__global__ void __launch_bounds__(128)
    k_top_direct_smem(const double* __restrict__ q, double* u, int d0, int d1, int d2,
                      const double* __restrict__ taps, int rowlen, const ErrRec* err) {
    extern __shared__ double sh[];
    if (failed(err)) return;
    const int m = d0 * d1 * d2;
    const int ntab = (2 * d0 - 1) * (2 * d1 - 1) * rowlen;
    double* st = sh;
    double* sq = sh + ntab;
    for (int i0 = threadIdx.x; i0 < ntab + m; i0 += 8 * blockDim.x) { // 8 independent loads in flight
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = i0 + u * blockDim.x;
            v[u] = i < ntab ? taps[i] : (i < ntab + m ? q[i - ntab] : 0.0);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (i0 + u * blockDim.x < ntab + m) sh[i0 + u * blockDim.x] = v[u];
    }
    __syncthreads();
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= m) return;
    const int z = idx % d2, y = (idx / d2) % d1, x = idx / (d2 * d1);
    const int Rx = d0 - 1, Ry = d1 - 1, Rz = d2 - 1;
    double acc = 0.0;
    for (int xs = 0; xs < d0; ++xs)
        for (int ys = 0; ys < d1; ++ys) {
            const double* trow = st + ((x - xs + Rx) * (2 * Ry + 1) + (y - ys + Ry)) * rowlen + (z + Rz);
            const double* qrow = sq + (xs * d1 + ys) * d2;
#pragma unroll 8
            for (int zs = 0; zs < d2; ++zs) acc = __dadd_rn(acc, __dmul_rn(trow[-zs], qrow[zs]));
        }
    u[idx] = acc;
}

size_t top_smem_bytes(const Geometry& g) {
    const LevelGeom& lv = g.lv[g.levels - 1];
    const int rowlen = (2 * g.top.Rz + 1 + kConvL - 1) / kConvL * kConvL;
    return sizeof(double) * (size_t(2 * lv.dims[0] - 1) * (2 * lv.dims[1] - 1) * rowlen + lv.size);
}

cudaError_t top_prepare(const Geometry& g) {
    const size_t b = top_smem_bytes(g);
    if (b > 220 * 1024) return cudaSuccess;
    return smem_grow(reinterpret_cast<const void*>(k_top_direct_smem), b);
}

// Production top level (small tops): one warp per point, the lanes take every 32nd
// source in row-major order, FMA, and a fixed xor-shuffle tree adds the lanes --
// deterministic, equal to the reference's sequential sum to rounding (the bit-exact
// k_top_direct_smem above serves the stage tests).  The sources of a point are
// independent, so the sum is ~m/32 FMAs deep instead of m dependent adds: the
// top level of C1 (14^3) 87 -> a few us.
__global__ void __launch_bounds__(256)
    k_top_warp(const double* __restrict__ q, double* u, int d0, int d1, int d2,
               const double* __restrict__ taps, int rowlen, const ErrRec* err, int early) {
    pdl_enter(early);
    if (failed(err)) return;
    const int m = d0 * d1 * d2;
    const int idx = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (idx >= m) return;
    const int z = idx % d2, y = (idx / d2) % d1, x = idx / (d2 * d1);
    const int Rx = d0 - 1, Ry = d1 - 1, Rz = d2 - 1;
    // source s = (xs, ys, zs) row-major; lane starts at s = lane and steps by 32; the
    // table offset of (xs, ys, zs) is base - zs - rowlen * (ys + (2 Ry + 1) xs)
    const int base = ((x + Rx) * (2 * Ry + 1) + (y + Ry)) * rowlen + (z + Rz);
    int zs = lane % d2, ys = (lane / d2) % d1, xs = lane / (d2 * d1);
    const int dz = 32 % d2, dy = (32 / d2) % d1, dx = 32 / (d2 * d1);
    constexpr int U = 8;  // independent loads in flight per lane
    double acc[U];
#pragma unroll
    for (int k = 0; k < U; ++k) acc[k] = 0.0;
    for (int s0 = lane; s0 < m; s0 += 32 * U) {
        int off[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            off[k] = base - zs - rowlen * (ys + (2 * Ry + 1) * xs);
            zs += dz;
            ys += dy;
            xs += dx;
            if (zs >= d2) { zs -= d2; ++ys; }
            if (ys >= d1) { ys -= d1; ++xs; }
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const int s = s0 + 32 * k;
            if (s < m) acc[k] = fma(__ldg(taps + off[k]), __ldg(q + s), acc[k]);
        }
    }
    double a = 0.0;
#pragma unroll
    for (int k = 0; k < U; ++k) a += acc[k];
#pragma unroll
    for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(FULLMASK, a, o);
    if (lane == 0) u[idx] = a;
}

int launch_top(cudaStream_t st, const Geometry& g, DevLevels& L, ErrRec* err, bool exact) {
    const int k = g.levels - 1;
    const LevelGeom& lv = g.lv[k];
    if (!exact && int64_t(lv.size) <= kTopDirectMax) {
        const int rowlen = (2 * g.top.Rz + 1 + kConvL - 1) / kConvL * kConvL;
        const int wpb = MSMB_CHAIN_SMALL ? 1 : 8; // warps (points) per CTA
        pdl_launch(k_top_warp, dim3(int((lv.size + wpb - 1) / wpb)), dim3(32 * wpb), 0, st, L.charge + lv.offset,
                   L.pot + lv.offset, lv.dims[0], lv.dims[1], lv.dims[2], L.taps[k], rowlen, err,
                   g.levels >= 2 && prolong_blocks(g, g.levels - 2) <= kPdlEarlyMaxBlocks ? 1 : 0);
        return 1;
    }
    if (int64_t(lv.size) <= kTopDirectMax) {
        const int rowlen = (2 * g.top.Rz + 1 + kConvL - 1) / kConvL * kConvL;
        const size_t sb = top_smem_bytes(g);
        if (sb <= 220 * 1024) {
            k_top_direct_smem<<<int((lv.size + 127) / 128), 128, sb, st>>>(L.charge + lv.offset, L.pot + lv.offset,
                                                                           lv.dims[0], lv.dims[1], lv.dims[2],
                                                                           L.taps[k], rowlen, err);
            return 1;
        }
        k_top_direct<<<int((lv.size + 127) / 128), 128, 0, st>>>(L.charge + lv.offset, L.pot + lv.offset,
                                                                 lv.dims[0], lv.dims[1], lv.dims[2],
                                                                 L.taps[k], rowlen, err);
        return 1;
    }
    ConvJobs J;
    J.njobs = 1;
    J.j[0] = make_job(g.top, lv, L.charge + lv.offset, L.pot + lv.offset, L.rows[k], L.dxb[k],
                      L.taps[k], 0, kConvZ);
    const int blocks = J.j[0].d0 * J.j[0].ty * J.j[0].tz;
    return launch_conv_jobs(st, J, blocks, true, err);
}

// ============================================================================
// K8: interpolation + long-range forces + assembly (src/msm_phases.cpp:195-222,
// src/msm.cpp:16-48, 69-86), reference arithmetic order.
// ============================================================================
struct InterpP {
    double o[3];
    double inv_h;
    int d[3];
    double self_term; // smoothing_gamma(0)/a
    double kc;
};

__device__ __forceinline__ void interp_atom(const InterpP& p, const double* __restrict__ pot,
                                            double px, double py, double pz, double& u,
                                            double& gx, double& gy, double& gz) {
    const double pp[3] = {px, py, pz};
    double w[3][4], dw[3][4];
    int base[3];
    for (int ax = 0; ax < 3; ++ax) {
        const double t = __dmul_rn(__dsub_rn(pp[ax], p.o[ax]), p.inv_h);
        base[ax] = int(floor(t)) - 1;
        for (int d = 0; d < 4; ++d) {
            const double xi = __dsub_rn(t, double(base[ax] + d));
            w[ax][d] = phi_rn(xi);
            dw[ax][d] = __dmul_rn(dphi_rn(xi), p.inv_h);
        }
    }
    double acc = 0.0;
    gx = gy = gz = 0.0;
    for (int a = 0; a < 4; ++a) {
        double accb = 0.0;
        for (int b = 0; b < 4; ++b) {
            const double* row = pot + (size_t(base[0] + a) * p.d[1] + (base[1] + b)) * p.d[2] + base[2];
            double accc = 0.0;
            for (int c = 0; c < 4; ++c) {
                const double uu = __ldg(row + c);
                accc = __dadd_rn(accc, __dmul_rn(w[2][c], uu));
                gx = __dadd_rn(gx, __dmul_rn(__dmul_rn(__dmul_rn(dw[0][a], w[1][b]), w[2][c]), uu));
                gy = __dadd_rn(gy, __dmul_rn(__dmul_rn(__dmul_rn(w[0][a], dw[1][b]), w[2][c]), uu));
                gz = __dadd_rn(gz, __dmul_rn(__dmul_rn(__dmul_rn(w[0][a], w[1][b]), dw[2][c]), uu));
            }
            accb = __dadd_rn(accb, __dmul_rn(w[1][b], accc));
        }
        acc = __dadd_rn(acc, __dmul_rn(w[0][a], accb));
    }
    u = acc;
}

// Production interpolation: the same tensor-product sums factored separably with
// FMAs -- per (a, b) row S = sum_c wz[c] u, Sd = sum_c dwz[c] u, then the y and x
// sums -- 192 DP ops per atom instead of ~750 for the reference's per-point
// products (interp_atom, kept bit-exact for the stage tests: msmb_debug_stage 4).
// Reassociation moves phi_long and the long-range force by ~1e-16 relative.
__device__ __forceinline__ void interp_atom_fast(const InterpP& p, const double* __restrict__ pot,
                                                 double px, double py, double pz, double& u,
                                                 double& gx, double& gy, double& gz) {
    const double pp[3] = {px, py, pz};
    double w[3][4], dw[3][4];
    int base[3];
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
        const double t = __dmul_rn(__dsub_rn(pp[ax], p.o[ax]), p.inv_h);
        base[ax] = int(floor(t)) - 1;
#pragma unroll
        for (int d = 0; d < 4; ++d) {
            const double xi = __dsub_rn(t, double(base[ax] + d));
            w[ax][d] = phi_rn(xi);
            dw[ax][d] = __dmul_rn(dphi_rn(xi), p.inv_h);
        }
    }
    const double* r0 = pot + (size_t(base[0]) * p.d[1] + base[1]) * p.d[2] + base[2];
    double uu = 0.0, ax_ = 0.0, ay_ = 0.0, az_ = 0.0;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        double T = 0.0, Td = 0.0, Tz = 0.0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const double* row = r0 + (size_t(a) * p.d[1] + b) * p.d[2];
            const double u0 = __ldg(row), u1 = __ldg(row + 1), u2 = __ldg(row + 2), u3 = __ldg(row + 3);
            const double S = fma(w[2][3], u3, fma(w[2][2], u2, fma(w[2][1], u1, w[2][0] * u0)));
            const double Sd = fma(dw[2][3], u3, fma(dw[2][2], u2, fma(dw[2][1], u1, dw[2][0] * u0)));
            T = fma(w[1][b], S, T);
            Td = fma(dw[1][b], S, Td);
            Tz = fma(w[1][b], Sd, Tz);
        }
        uu = fma(w[0][a], T, uu);
        ax_ = fma(dw[0][a], T, ax_);
        ay_ = fma(w[0][a], Td, ay_);
        az_ = fma(w[0][a], Tz, az_);
    }
    u = uu;
    gx = ax_;
    gy = ay_;
    gz = az_;
}

static InterpP make_interp(const Geometry& g) {
    InterpP p;
    for (int ax = 0; ax < 3; ++ax) {
        p.o[ax] = g.lv[0].origin[ax];
        p.d[ax] = g.lv[0].dims[ax];
    }
    p.inv_h = g.inv_h0;
    p.self_term = g.self_term;
    p.kc = g.units.coulomb_constant;
    return p;
}

#ifndef MSMB_INTERP_TPB
#define MSMB_INTERP_TPB 32 // C2-S: 32 0.0313, 64 0.0325, 128 0.0332 ms
#endif
// one thread per atom in cluster order (the short-range results are in that order);
// four lanes per atom (one x-offset each, xor-tree combine) measured slower on C2-S
// (0.045 vs 0.033 ms: the weights are recomputed by every lane)
#ifndef MSMB_INTERP_MINB
#define MSMB_INTERP_MINB 5
#endif
__global__ void __launch_bounds__(128, MSMB_INTERP_MINB)
    k_interp(InterpP p, const int* __restrict__ colstart, int col_a, int col_b,
                         const int* __restrict__ perm,
                         const double* __restrict__ xs, const double* __restrict__ ys,
                         const double* __restrict__ zs, const double* __restrict__ qs,
                         const double* __restrict__ pot, const double* __restrict__ phis,
                         const double* __restrict__ fsx, const double* __restrict__ fsy,
                         const double* __restrict__ fsz, DevOut o, const ErrRec* err) {
    pdl_enter(1); // k_finalize (one thread) may be admitted
    const int s = colstart[col_a] + blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= colstart[col_b] || failed(err)) return;
    double u, gx, gy, gz;
    const double q = qs[s];
    interp_atom_fast(p, pot, xs[s], ys[s], zs[s], u, gx, gy, gz);
    const double ul = __dsub_rn(u, __dmul_rn(q, p.self_term));  // msm.cpp:73
    const double kq = __dmul_rn(p.kc, q);                          // msm.cpp:47
    const int i = perm[s];
    o.fx[i] = __dsub_rn(fsx[s], __dmul_rn(gx, kq));
    o.fy[i] = __dsub_rn(fsy[s], __dmul_rn(gy, kq));
    o.fz[i] = __dsub_rn(fsz[s], __dmul_rn(gz, kq));
    const double ph = __dadd_rn(phis[s], ul);                       // msm.cpp:80
    if (o.phi) o.phi[i] = ph;
    if (o.phis) o.phis[i] = phis[s];
    if (o.phil) o.phil[i] = ul;
    if (o.e) o.e[i] = __dmul_rn(__dmul_rn(0.5, q), ph);             // msm.cpp:83
}

// energy: deterministic two-level tree over e[] in original index order
__global__ void __launch_bounds__(256) k_energy1(int64_t n, const double* __restrict__ e,
                                                 double* partial, const ErrRec* err) {
    __shared__ double sh[256];
    if (failed(err)) return;
    const int64_t base = int64_t(blockIdx.x) * 4096 + threadIdx.x * 16;
    double s = 0.0;
    for (int k = 0; k < 16; ++k)
        if (base + k < n) s += e[base + k];
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int o = 128; o; o >>= 1) {
        if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
}

__global__ void __launch_bounds__(256) k_energy2(int nb, const double* __restrict__ partial,
                                                 double kc, double* out, const ErrRec* err, int accumulate = 0) {
    __shared__ double sh[256];
    if (failed(err)) return;
    double s = 0.0;
    for (int i = threadIdx.x; i < nb; i += 256) s += partial[i];
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int o = 128; o; o >>= 1) {
        if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = accumulate ? *out + sh[0] * kc : sh[0] * kc;
}

int launch_energy_sum(cudaStream_t st, int64_t n, const double* e, double* partial, double scale, double* out,
                      int accumulate, ErrRec* err) {
    const int nb = reduce_blocks(n);
    k_energy1<<<nb, 256, 0, st>>>(n, e, partial, err);
    k_energy2<<<1, 256, 0, st>>>(nb, partial, scale, out, err, accumulate);
    return 2;
}

// kinetic_energy (src/system.cpp:51-55): e_i = (0.5 m_i) |v_i|^2 with norm2's
// operation order, summed by the fixed-order energy tree
__global__ void k_kinetic(int64_t n, const double* __restrict__ vx, const double* __restrict__ vy,
                          const double* __restrict__ vz, const double* __restrict__ m, double* e) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double v2 = __dadd_rn(__dadd_rn(__dmul_rn(vx[i], vx[i]), __dmul_rn(vy[i], vy[i])), __dmul_rn(vz[i], vz[i]));
    e[i] = __dmul_rn(__dmul_rn(0.5, m[i]), v2);
}

int launch_kinetic(cudaStream_t st, const DevState& s, double* e, double* partial, double scale, double* out,
                   ErrRec* err) {
    if (s.n <= 0) return 0;
    k_kinetic<<<atom_blocks(s.n, 256), 256, 0, st>>>(s.n, s.vx, s.vy, s.vz, s.m, e);
    return 1 + launch_energy_sum(st, s.n, e, partial, scale, out, 0, err);
}

int reduce_blocks(int64_t n) { return int((n + 4095) / 4096) > 0 ? int((n + 4095) / 4096) : 1; }

int launch_interp(cudaStream_t st, const Geometry& g, int64_t n, DevAtoms& a, DevCells& c,
                  DevLevels& L, DevOut& o, ErrRec* err, int want_energy, const Part& P) {
    if (n == 0) return 0;
    const int itpb = n < 148 * 512 ? 64 : MSMB_INTERP_TPB;
    k_interp<<<atom_blocks(n, itpb), itpb, 0, st>>>(make_interp(g), c.colstart, P.cx0 * g.ncy, P.cx1 * g.ncy,
                                                   a.cl_perm, a.xc, a.yc, a.zc, a.qc, L.pot + g.lv[0].offset, a.phis,
                                                   a.fsx, a.fsy, a.fsz, o, err);
    if (!want_energy) return 1;
    const int nb = reduce_blocks(n);
    k_energy1<<<nb, 256, 0, st>>>(n, o.e, o.partial, err);
    k_energy2<<<1, 256, 0, st>>>(nb, o.partial, g.units.coulomb_constant, o.energy, err);
    return 3;
}

// Pair-only fields (simple_cutoff / wolf_summation, src/electrostatics.cpp:66-132):
// per-atom outputs in original order from the pair sums; the Wolf self term
// q_i * self_per_charge is added after the pair sum (electrostatics.cpp:123-124);
// e_i = 0.5 q_i phi_i for the index-order energy (finish_total, :27-33).  A NaN
// coordinate (nan_count > 0, n >= 2) makes every pair of that particle NaN in the
// reference, hence every output NaN.
__global__ void k_pair_out(const int* __restrict__ colstart, int col_a, int col_b, const int* __restrict__ perm,
                           const double* __restrict__ qs, const double* __restrict__ phis,
                           const double* __restrict__ fsx, const double* __restrict__ fsy,
                           const double* __restrict__ fsz, double self_per_charge, int wolf, int64_t n,
                           DevOut o, const ErrRec* err) {
    const int s = colstart[col_a] + blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= colstart[col_b] || failed(err)) return;
    const int i = perm[s];
    const bool poison = n >= 2 && __ldcg(&err->nan_count) > 0;
    const double nanv = __longlong_as_double(0x7ff8000000000000ll);
    const double q = qs[s];
    double ph = phis[s];
    if (wolf) ph = __dadd_rn(ph, __dmul_rn(q, self_per_charge));
    if (poison) ph = nanv;
    o.fx[i] = poison ? nanv : fsx[s];
    o.fy[i] = poison ? nanv : fsy[s];
    o.fz[i] = poison ? nanv : fsz[s];
    if (o.phi) o.phi[i] = ph;
    if (o.phis) o.phis[i] = ph;
    if (o.phil) o.phil[i] = 0.0;
    if (o.e) o.e[i] = __dmul_rn(__dmul_rn(0.5, q), ph);
}

int launch_pair_out(cudaStream_t st, const Geometry& g, int64_t n, DevAtoms& a, DevCells& c, DevOut& o,
                    ErrRec* err, int want_energy, const Part& P) {
    if (n == 0) return 0;
    k_pair_out<<<int((n + 127) / 128), 128, 0, st>>>(c.colstart, P.cx0 * g.ncy, P.cx1 * g.ncy, a.cl_perm, a.qc,
                                                     a.phis, a.fsx, a.fsy, a.fsz, g.pf.self_per_charge,
                                                     g.kind == MSMB_FIELD_WOLF ? 1 : 0, n, o, err);
    if (!want_energy) return 1;
    const int nb = reduce_blocks(n);
    k_energy1<<<nb, 256, 0, st>>>(n, o.e, o.partial, err);
    k_energy2<<<1, 256, 0, st>>>(nb, o.partial, g.units.coulomb_constant, o.energy, err);
    return 3;
}

// Decide the evaluation's outcome with the reference's precedence:
// short_range errors (first pair in i<j order) > coverage (min particle).
__global__ void k_finalize(const double* __restrict__ x, const double* __restrict__ y,
                           const double* __restrict__ z, int pair_field, ErrRec* err) {
    pdl_enter();
    if (err->kind) return;
    if (err->overflow) {
        err->kind = kOverflowKind;
        err->step = err->cur_step;
        return;
    }
    if (err->pair_key != ~0ull) {
        const int i = int(err->pair_key >> 32), j = int(err->pair_key & 0xffffffffu);
        const double dx = __dsub_rn(x[i], x[j]), dy = __dsub_rn(y[i], y[j]), dz = __dsub_rn(z[i], z[j]);
        const double r2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
        err->kind = r2 == 0.0 ? MSMB_ERR_COINCIDENT : MSMB_ERR_DOMAIN;
        err->err_i = i;
        err->err_j = j;
        err->step = err->cur_step;
        return;
    }
    if (err->cov_count > 0) { // pair-only fields: infinite coordinates (msmb.h)
        err->kind = pair_field ? MSMB_ERR_DOMAIN : MSMB_ERR_COVERAGE;
        err->err_i = err->cov_min;
        err->err_j = -1;
        err->step = err->cur_step;
    }
}

int launch_finalize(cudaStream_t st, const DevState& s, ErrRec* err, int pair_field) {
    pdl_launch(k_finalize, dim3(1), dim3(1), 0, st, s.x, s.y, s.z, pair_field, err);
    return 1;
}

__global__ void k_reset_err(ErrRec* err, int step) {
    err->kind = 0;
    err->step = -1;
    err->overflow = 0;
    err->cov_count = 0;
    err->pair_key = ~0ull;
    err->cov_min = LLONG_MAX;
    err->err_i = -1;
    err->err_j = -1;
    err->cur_step = step;
    err->nan_count = 0;
    err->pairs = 0;
    err->candidates = 0;
}

int launch_reset_err(cudaStream_t st, ErrRec* err, int step) {
    k_reset_err<<<1, 1, 0, st>>>(err, step);
    return 1;
}

// ============================================================================
// K9: velocity Verlet (src/integrate.cpp:24-33), reference arithmetic:
// c = ((0.5*dt)*conv)/m;  v += F*c;  [v += F*c];  r += v*dt
// `kicks` = 2 fuses the closing half-kick of step s-1 with the opening one of s.
// ============================================================================
__global__ void k_kick_drift(int64_t n, double* x, double* y, double* z, double* vx, double* vy,
                             double* vz, const double* __restrict__ m, const double* __restrict__ fx,
                             const double* __restrict__ fy, const double* __restrict__ fz,
                             double dt, double hdc, int kicks, ErrRec* err) {
    if (failed(err)) return;
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i == 0) err->pairs = 0, err->candidates = 0, err->cur_step += 1;
    if (i >= n) return;
    const double c = __ddiv_rn(hdc, m[i]);
    double a = vx[i], b = vy[i], d = vz[i];
    const double Fx = fx[i], Fy = fy[i], Fz = fz[i];
    for (int k = 0; k < kicks; ++k) {
        a = __dadd_rn(a, __dmul_rn(Fx, c));
        b = __dadd_rn(b, __dmul_rn(Fy, c));
        d = __dadd_rn(d, __dmul_rn(Fz, c));
    }
    vx[i] = a;
    vy[i] = b;
    vz[i] = d;
    x[i] = __dadd_rn(x[i], __dmul_rn(a, dt));
    y[i] = __dadd_rn(y[i], __dmul_rn(b, dt));
    z[i] = __dadd_rn(z[i], __dmul_rn(d, dt));
}

__global__ void k_kick(int64_t n, double* vx, double* vy, double* vz, const double* __restrict__ m,
                       const double* __restrict__ fx, const double* __restrict__ fy,
                       const double* __restrict__ fz, double hdc, const ErrRec* err) {
    if (failed(err)) return;
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double c = __ddiv_rn(hdc, m[i]);
    vx[i] = __dadd_rn(vx[i], __dmul_rn(fx[i], c));
    vy[i] = __dadd_rn(vy[i], __dmul_rn(fy[i], c));
    vz[i] = __dadd_rn(vz[i], __dmul_rn(fz[i], c));
}

int launch_kick_drift(cudaStream_t st, DevState& s, const DevOut& o, double dt, double conv,
                      int kicks, ErrRec* err) {
    const double hdc = 0.5 * dt * conv; // (0.5*dt)*conv, host IEEE, same as the reference
    k_kick_drift<<<atom_blocks(s.n, atom_tpb(s.n)), atom_tpb(s.n), 0, st>>>(
        s.n, s.x, s.y, s.z, s.vx, s.vy, s.vz, s.m, o.fx, o.fy, o.fz, dt, hdc, kicks, err);
    return 1;
}

int launch_kick(cudaStream_t st, DevState& s, const DevOut& o, double dt, double conv,
                ErrRec* err) {
    if (s.n == 0) return 0;
    const double hdc = 0.5 * dt * conv;
    k_kick<<<atom_blocks(s.n, atom_tpb(s.n)), atom_tpb(s.n), 0, st>>>(s.n, s.vx, s.vy, s.vz, s.m, o.fx, o.fy, o.fz, hdc,
                                                   err);
    return 1;
}

// ============================================================================
// K10: parareal state algebra (src/parareal.cpp:58-90)
// ============================================================================
__global__ void __launch_bounds__(256) k_state_sub(int64_t n, DevState a, DevState b, double* dpos,
                                                   double* dvel, double* partial) {
    __shared__ double sh[256];
    const int64_t base = int64_t(blockIdx.x) * 4096 + threadIdx.x * 16;
    double s = 0.0;
    for (int k = 0; k < 16; ++k) {
        const int64_t i = base + k;
        if (i >= n) break;
        const double dx = __dsub_rn(a.x[i], b.x[i]), dy = __dsub_rn(a.y[i], b.y[i]),
                     dz = __dsub_rn(a.z[i], b.z[i]);
        dpos[3 * i] = dx;
        dpos[3 * i + 1] = dy;
        dpos[3 * i + 2] = dz;
        dvel[3 * i] = __dsub_rn(a.vx[i], b.vx[i]);
        dvel[3 * i + 1] = __dsub_rn(a.vy[i], b.vy[i]);
        dvel[3 * i + 2] = __dsub_rn(a.vz[i], b.vz[i]);
        s = __dadd_rn(s, __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
    }
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int o = 128; o; o >>= 1) {
        if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
}

__global__ void k_state_add(int64_t n, DevState base, const double* __restrict__ dpos,
                            const double* __restrict__ dvel, DevState out) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    out.x[i] = __dadd_rn(base.x[i], dpos[3 * i]);
    out.y[i] = __dadd_rn(base.y[i], dpos[3 * i + 1]);
    out.z[i] = __dadd_rn(base.z[i], dpos[3 * i + 2]);
    out.vx[i] = __dadd_rn(base.vx[i], dvel[3 * i]);
    out.vy[i] = __dadd_rn(base.vy[i], dvel[3 * i + 1]);
    out.vz[i] = __dadd_rn(base.vz[i], dvel[3 * i + 2]);
}

__global__ void __launch_bounds__(256) k_rms(int64_t n, DevState a, DevState b, double* partial) {
    __shared__ double sh[256];
    const int64_t base = int64_t(blockIdx.x) * 4096 + threadIdx.x * 16;
    double s = 0.0;
    for (int k = 0; k < 16; ++k) {
        const int64_t i = base + k;
        if (i >= n) break;
        const double dx = __dsub_rn(a.x[i], b.x[i]), dy = __dsub_rn(a.y[i], b.y[i]),
                     dz = __dsub_rn(a.z[i], b.z[i]);
        s = __dadd_rn(s, __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
    }
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int o = 128; o; o >>= 1) {
        if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
}

int launch_state_sub(cudaStream_t st, int64_t n, const DevState& a, const DevState& b,
                     double* dpos, double* dvel, double* partial, int nblk) {
    k_state_sub<<<nblk, 256, 0, st>>>(n, a, b, dpos, dvel, partial);
    return 1;
}

int launch_state_add(cudaStream_t st, int64_t n, const DevState& base, const double* dpos,
                     const double* dvel, DevState& out) {
    k_state_add<<<int((n + 255) / 256), 256, 0, st>>>(n, base, dpos, dvel, out);
    return 1;
}

int launch_rms_change(cudaStream_t st, int64_t n, const DevState& a, const DevState& b,
                      double* partial, int nblk) {
    k_rms<<<nblk, 256, 0, st>>>(n, a, b, partial);
    return 1;
}

__global__ void k_aos_to_soa(int64_t n, const double* __restrict__ aos, double* x, double* y, double* z) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    x[i] = aos[3 * i];
    y[i] = aos[3 * i + 1];
    z[i] = aos[3 * i + 2];
}

__global__ void k_soa_to_aos(int64_t n, const double* __restrict__ x, const double* __restrict__ y,
                             const double* __restrict__ z, double* aos) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    aos[3 * i] = x[i];
    aos[3 * i + 1] = y[i];
    aos[3 * i + 2] = z[i];
}

int launch_aos_to_soa(cudaStream_t st, int64_t n, const double* aos, double* x, double* y, double* z) {
    if (n == 0) return 0;
    k_aos_to_soa<<<int((n + 255) / 256), 256, 0, st>>>(n, aos, x, y, z);
    return 1;
}

int launch_soa_to_aos(cudaStream_t st, int64_t n, const double* x, const double* y, const double* z,
                      double* aos) {
    if (n == 0) return 0;
    k_soa_to_aos<<<int((n + 255) / 256), 256, 0, st>>>(n, x, y, z, aos);
    return 1;
}

__global__ void k_debug_cells(int64_t n, BinP p, const double* x, const double* y, const double* z,
                              int* cells, int* covered) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double pp[3] = {x[i], y[i], z[i]};
    int ok = 1;
    for (int ax = 0; ax < 3; ++ax) {
        const double t = __dmul_rn(__dsub_rn(pp[ax], p.o[ax]), p.inv_h);
        const double f = floor(t);
        const bool c = (f >= 1.0) && (f <= double(p.d[ax]) - 3.0);
        ok &= c ? 1 : 0;
        cells[3 * i + ax] = (f > -2147483648.0 && f < 2147483647.0) ? int(f) : INT_MIN;
    }
    covered[i] = ok;
}

int launch_debug_cells(cudaStream_t st, const Geometry& g, const DevState& s, int* cells, int* covered) {
    if (s.n == 0) return 0;
    k_debug_cells<<<int((s.n + 255) / 256), 256, 0, st>>>(s.n, make_binp(g), s.x, s.y, s.z, cells, covered);
    return 1;
}

__global__ void k_debug_interp(int64_t n, InterpP p, const double* x, const double* y,
                               const double* z, const double* pot, double* u) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double gx, gy, gz;
    interp_atom(p, pot, x[i], y[i], z[i], u[i], gx, gy, gz);
}

int launch_debug_interp(cudaStream_t st, const Geometry& g, const DevState& s, const double* pot0,
                        double* u) {
    if (s.n == 0) return 0;
    k_debug_interp<<<int((s.n + 127) / 128), 128, 0, st>>>(s.n, make_interp(g), s.x, s.y, s.z, pot0, u);
    return 1;
}

} // namespace msmb

// ---- diagnostic: globaltimer stamps for a step timeline (MSMB_TIMELINE, msmb_engine.cu) ----
namespace msmb {
__device__ unsigned long long g_stamps[16];
__global__ void k_stamp(int idx) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_stamps[idx] = t;
}
bool pdl_enabled() {
    static const bool on = !(std::getenv("MSMB_PDL") && std::atoi(std::getenv("MSMB_PDL")) == 0);
    return on;
}
void launch_stamp(cudaStream_t st, int idx) { k_stamp<<<1, 1, 0, st>>>(idx); }
void read_stamps(unsigned long long* h) { cudaMemcpyFromSymbol(h, g_stamps, sizeof(unsigned long long) * 16); }
} // namespace msmb
