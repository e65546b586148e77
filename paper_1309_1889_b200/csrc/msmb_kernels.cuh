// Device-side declarations: argument bundles and launch wrappers for the
// sm_100a kernels in msmb_kernels.cu.
#pragma once
#include <cuda_runtime.h>

#include "msmb_internal.h"

namespace msmb {

// Per-workspace device pointers (all device memory).
struct DevAtoms {       // sorted-order working set, capacity n
    int* key;           // [n] sorted-cell index of atom i (original order), -1 = not binned
    int* rank;          // [n]
    int* perm;          // [n] sorted slot -> original index
    int* outlist;       // [n] out-of-coverage atoms
    double* aw;         // [n*12] anterpolation weights: q*wx[4], wy[4], wz[4]
    double* phis;       // [n] short-range potential (per unit charge), cluster order
    double* fsx; double* fsy; double* fsz; // short-range forces (with k_C), cluster order
    // pair-list (Verlet skin) state: the cluster order is the sorted order of the
    // last list rebuild; positions are gathered into it every evaluation
    int* cl_perm;       // [n] cluster slot -> original index
    int* cl_inv;        // [n] original index -> cluster slot (ownership tests in original order)
    double* xc; double* yc; double* zc; double* qc; // [n] positions / charges, cluster order
    double* ref;        // [3n] positions (original order) at the last rebuild
    double* pair_part;  // [kPairSplitMax * 4 * n] split pair-walk partial sums (small systems), or null
};
constexpr int kPairSplitMax = 8;
int pair_split(int64_t maxclu); // warps per i-cluster in the pair kernel

struct DevCells {
    int* count;         // [ncells+1]
    int* start;         // [ncells+1]
    int2* nat;          // [d0*d1*d2] level-0 cell (x,y,z row-major) -> sorted range [start, end)
    int* col_cnt;       // [ncols+1] clusters per column
    int* col_off;       // [ncols+1] first cluster of each column
    int2* clu;          // [max_clusters] (first sorted slot, count)
    float4* blo; float4* bhi; // cluster bounding boxes
    int* nclu;          // [1]
    int* plist;         // [max_clusters * cap]
    int* pcnt;          // [max_clusters]
    unsigned* pmask;    // [max_clusters * cap * 32] per-lane j-atom masks (k_pairmask)
    int* dlist;         // [max_clusters * dense_cap] dense j atoms (sorted slots) of each i-cluster
    int* dcnt;          // [max_clusters]
    int* scan_tmp;      // scratch for the multi-block scan
    int* colstart;      // [ncols+1] first cluster slot of each pair column (frozen at rebuild)
    int* flag;          // [10] [0] rebuild the pair list this evaluation, [1] clustered atoms,
                        //     [2] rebuild count (diagnostics), [3] list valid, [4] list's part key,
                        //     [5] some atom changed cell (k_bin), [6] cell sort valid, [7] sort now,
                        //     [8], [9] spare
};

// Programmatic dependent launch (PDL) for the long-range chain's small kernels.  A kernel
// launched with pdl_launch may be admitted to the SMs as soon as every CTA of the previous
// kernel in its stream has started (pdl_enter's launch_dependents), and waits in pdl_enter
// (griddepcontrol.wait) until that kernel has completed and its writes are visible.  Beside
// the pair kernel, which holds nearly all registers of every SM, a chain launch otherwise
// costs ~25-60 us of admission latency after its predecessor ends, whatever its size.
// Every kernel launched this way must call pdl_enter() before its first global access;
// without the launch attribute the two instructions are no-ops.  MSMB_PDL=0 turns it off.
#ifdef __CUDACC__
// early: let the next kernel's CTAs be admitted (they block in their pdl_enter) while this one
// runs -- only worth it when that kernel is a handful of CTAs: blocked CTAs hold SM resources
// the pair kernel would use (early for every chain kernel: C2-S 0.751 -> 0.864 ms/step)
constexpr int kPdlEarlyMaxBlocks = 128;
__device__ __forceinline__ void pdl_enter(int early = 0) {
    if (early) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
}
bool pdl_enabled();
template <class... KArgs, class... Args>
inline void pdl_launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    cudaLaunchKernelEx(&cfg, kern, KArgs(args)...);
}
#endif

struct DevLevels {      // concatenated lattices + tables
    double* charge;     // [lattice_total]
    double* pot;        // [lattice_total]
    // transfer tables per transition k and axis
    int* tr_base[kMaxLevels][3];
    double* tr_w[kMaxLevels][3];
    int* tr_rcnt[kMaxLevels][3];
    int* tr_ridx[kMaxLevels][3];
    double* tr_rw[kMaxLevels][3];
    // k_lattice: shared level-0 stencil + split partial lattices
    int* lat_rowidx;
    int2* lat_rowchunks;
    double* lat_taps;
    double* lat_partial;
    double* anterp_part; // tiled anterpolation: one (kTX+3)(kTY+3)(kTZ+3) tile per cell block
    int lat_S;
    int lat_const;      // stencil lives in constant memory (k_lattice<true>)
    // stencil tables: lattice levels then top (index levels-1)
    int4* rows[kMaxLevels];
    int* dxb[kMaxLevels];
    double* taps[kMaxLevels];
};

// FFT lattice cutoff (msmb_fft.cu): per level and axis a padded length M = 2^a 3^b
// >= d + R, its radix list and the offset of its twiddle table exp(-2 pi i m / M)
constexpr int kFftMaxF = 20;
struct FftAxis {
    int M, nf, tw;
    int fac[kFftMaxF];
};
struct FftLevel {
    int d[3];
    FftAxis ax[3];
    size_t boff, soff;  // complex work buffer / spectrum offsets
    const double* q;    // level charges
    double* u;          // level potentials
    int blk0;           // first block of this level in the current pass
};
struct FftJobs {
    FftLevel lv[kMaxLevels];
    int n, L, maxM;     // levels, lines per tile, max M
    double2* buf;
    double* spec;
    const double2* tw;
};
struct FftKernel {       // where the spectrum precompute reads a job's kernel
    int dense;          // 0: cutoff stencil (rowidx/taps rows), 1: dense top table
    const int* rowidx;
    const double* taps;
    int R[3];           // half-widths of the table
    int rowlen;         // taps per (dx, dy) row
    double scale;       // 2^-k for cutoff levels, 1 for the top
};
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is process-wide per device:
// fields with different geometries share the kernels, so the limit only ever grows
// (a smaller workspace must not lower what a larger one's launches need).
cudaError_t smem_grow(const void* func, size_t bytes);
int fft_len(int need);
FftAxis fft_axis(int M, int tw_off);
cudaError_t fft_prepare(size_t smem);
int launch_fft_spectrum(cudaStream_t st, FftJobs J, const FftKernel* K);
int launch_lattice_fft(cudaStream_t st, FftJobs J, const ErrRec* err);

struct DevState {       // a device-resident ParticleSystem (SoA)
    int64_t n;
    double* x; double* y; double* z;
    double* vx; double* vy; double* vz;
    double* q; double* m;
};

struct DevOut {         // per-atom outputs in original order (optional)
    double* fx; double* fy; double* fz;
    double* phi; double* phis; double* phil;
    double* e;          // [n] 0.5 q phi
    double* partial;    // [nblocks] energy partial sums
    double* energy;     // [1]
};

// Launch wrappers (all asynchronous on `st`).  Each returns the number of kernel
// launches issued so the engine can count them.
// exclusive scan of int[m] (tmp: >= (m + 4095) / 4096 + 8 ints)
int launch_scan_exclusive(cudaStream_t st, const int* in, int* out, int* tmp, int64_t m);
// list != nullptr: only the atoms list[0..nlist) (a spatial-decomposition part's local atoms)
int launch_bin(cudaStream_t st, const Geometry& g, const DevState& s, DevAtoms& a, DevCells& c,
               ErrRec* err, const int* list = nullptr, int64_t nlist = 0);
int launch_sort(cudaStream_t st, const Geometry& g, const DevState& s, DevAtoms& a, DevCells& c,
                ErrRec* err, const int* list = nullptr, int64_t nlist = 0);
// disp = 0: no skin/2 displacement test (the caller decided the rebuild: force_rebuild)
int launch_clusters(cudaStream_t st, const Geometry& g, int64_t n, const DevState& s, DevAtoms& a,
                    DevCells& c, ErrRec* err, int cap, const Part& P, int force_rebuild, int disp = 1,
                    int phase = 0);
// count: accumulate the pair / candidate statistics (eager evaluations; graphs skip it)
int launch_pairs(cudaStream_t st, const Geometry& g, int64_t n, const DevState& s, DevAtoms& a,
                 DevCells& c, ErrRec* err, int cap, const Part& P, bool count = true, int gmode = 0);
int launch_anterp(cudaStream_t st, const Geometry& g, const DevState& s, DevAtoms& a, DevCells& c, DevLevels& L,
                  ErrRec* err, const Part& P);
size_t anterp_tile_part_doubles(const Geometry& g);
int launch_restrict(cudaStream_t st, const Geometry& g, int k, DevLevels& L, ErrRec* err);
int launch_restrict_all(cudaStream_t st, const Geometry& g, DevLevels& L, ErrRec* err);
int launch_restrict_planes(cudaStream_t st, const Geometry& g, int k, DevLevels& L, ErrRec* err, int xlo, int xhi,
                           int early = 0);
int launch_prolong_planes(cudaStream_t st, const Geometry& g, int k, DevLevels& L, ErrRec* err, int xlo, int xhi,
                          int early = 0);
int launch_prolong_all(cudaStream_t st, const Geometry& g, DevLevels& L, ErrRec* err);
int launch_lattice(cudaStream_t st, const Geometry& g, DevLevels& L, ErrRec* err, const Part& P);
size_t lattice_smem_bytes(const Geometry& g);
cudaError_t lattice_prepare(size_t bytes);
int lattice_splits(const Geometry& g);
bool lattice_const_fits(const Geometry& g);
cudaError_t lattice_upload_const(const Geometry& g, cudaStream_t st);
// exact: the reference's sequential per-point sum, bit for bit (stage tests);
// otherwise the warp-parallel production kernel (equal to rounding)
int launch_top(cudaStream_t st, const Geometry& g, DevLevels& L, ErrRec* err, bool exact = false);
cudaError_t top_prepare(const Geometry& g); // dynamic smem of the staged direct top kernel
constexpr int64_t kTopFftMin = 4096; // FFT lattice mode: top levels above this many points use an FFT job
int launch_prolong(cudaStream_t st, const Geometry& g, int k, DevLevels& L, ErrRec* err);
int launch_interp(cudaStream_t st, const Geometry& g, int64_t n, DevAtoms& a, DevCells& c,
                  DevLevels& L, DevOut& o, ErrRec* err, int want_energy, const Part& P);

int launch_finalize(cudaStream_t st, const DevState& s, ErrRec* err, int pair_field = 0);
// pair-only fields: per-atom outputs and energy from the pair sums (no grid)
int launch_pair_out(cudaStream_t st, const Geometry& g, int64_t n, DevAtoms& a, DevCells& c, DevOut& o,
                    ErrRec* err, int want_energy, const Part& P);
// fixed-order energy tree: *out = scale * sum(e[0..n)) (accumulate: *out += ...)
// kinetic_energy (src/system.cpp:51-55) of s into *out (times scale), e = n scratch doubles
int launch_kinetic(cudaStream_t st, const DevState& s, double* e, double* partial, double scale, double* out,
                   ErrRec* err);
int launch_energy_sum(cudaStream_t st, int64_t n, const double* e, double* partial, double scale, double* out,
                      int accumulate, ErrRec* err);
// all-pairs kernels (msmb_direct.cu): direct Coulomb (coul) and/or the
// PairRepulsionOverlay term (rep) over all pairs of the state in original order.  coul writes
// phi/F/e of `o`; rep adds its forces to F and its per-atom energy to e_rep.
struct AllPairsBuf {
    double* part;       // [S * 5 * n] per-split partial sums (S > 1)
    double* e_rep;      // [n] 0.5 * sum_j eps (sigma/r)^12
    int S;              // j splits
};
int allpairs_splits(int64_t n);
int launch_allpairs(cudaStream_t st, const DevState& s, double kc, int coul, int rep, double eps,
                    double sigma, const AllPairsBuf& B, DevOut& o, ErrRec* err);
int launch_kick_drift(cudaStream_t st, DevState& s, const DevOut& o, double dt, double conv,
                      int kicks, ErrRec* err);
int launch_kick(cudaStream_t st, DevState& s, const DevOut& o, double dt, double conv,
                ErrRec* err);
int launch_reset_err(cudaStream_t st, ErrRec* err, int step);
// parareal state algebra (src/parareal.cpp:58-90)
int launch_state_sub(cudaStream_t st, int64_t n, const DevState& a, const DevState& b,
                     double* dpos, double* dvel, double* partial, int nblk);
int launch_state_add(cudaStream_t st, int64_t n, const DevState& base, const double* dpos,
                     const double* dvel, DevState& out);
int launch_rms_change(cudaStream_t st, int64_t n, const DevState& a, const DevState& b,
                      double* partial, int nblk);
int reduce_blocks(int64_t n);
// AoS <-> SoA
int launch_aos_to_soa(cudaStream_t st, int64_t n, const double* aos, double* x, double* y, double* z);
int launch_soa_to_aos(cudaStream_t st, int64_t n, const double* x, const double* y, const double* z,
                      double* aos);
// debug: level-0 cell triples
int launch_debug_cells(cudaStream_t st, const Geometry& g, const DevState& s, int* cells, int* covered);
// debug: stand-alone interpolation of a level-0 potential at atoms (no sort)
int launch_debug_interp(cudaStream_t st, const Geometry& g, const DevState& s, const double* pot0,
                        double* u);

} // namespace msmb
