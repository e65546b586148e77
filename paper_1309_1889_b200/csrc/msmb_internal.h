// Internal declarations shared by the host engine (msmb_engine.cu), the host
// geometry/table builder (msmb_geometry.cpp) and the kernels (msmb_kernels.cu).
#pragma once
#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/msmb.h"

namespace msmb {

constexpr int kMaxLevels = 16;
// pair kernel CTA shape: one warp per CTA, up to 20 CTAs per SM (C2-S: 0.922 vs 0.929
// ms/step with 4 warps x 5 CTAs; 2 x 10 equal) -- finer-grained scheduling of the
// uneven per-cluster walks
#ifndef MSMB_PAIR_WARPS
#define MSMB_PAIR_WARPS 1
#endif
constexpr int kPairWarps = MSMB_PAIR_WARPS; // warps per CTA in the pair kernels
constexpr int kConvB = 16;         // outputs per thread along z in the stencil kernel
constexpr int kConvL = 8;          // taps per chunk in the stencil kernel
constexpr int kConvNWZ = 2;        // warps along z per stencil CTA
constexpr int kConvZ = kConvB * kConvNWZ;
constexpr int kRestrictMax = 8;    // fine indices feeding one coarse index per axis
constexpr int kOverflowKind = 100; // internal: pair-list capacity exceeded, retry

// ---- host-side error ----------------------------------------------------------
struct Error {
    int kind = MSMB_OK;
    int64_t i = -1, j = -1;
    int step = -1;
    std::string msg;
};

// ---- device error record (one per workspace) ------------------------------------
struct ErrRec {
    int kind;                    // 0 while healthy; msmb_status once an evaluation failed
    int step;                    // Verlet step of the failing evaluation
    int overflow;                // max pair-list entries requested by any cluster (if > cap)
    int cov_count;               // out-of-coverage particles in the current evaluation
    unsigned long long pair_key; // min (i << 32 | j), i < j, with r2 == 0 or NaN
    long long cov_min;           // min out-of-coverage particle index
    long long err_i, err_j;      // indices reported with `kind`
    int cur_step;                // step counter, advanced by the Verlet kernels
    int nan_count;               // cutoff/Wolf fields: particles with a NaN coordinate
    unsigned long long pairs;     // in-cutoff ordered pairs (stats, current evaluation)
    unsigned long long candidates;// screened candidate pairs (stats)
};

// ---- level geometry (src/msm_grid.cpp:24-54) -----------------------------------
struct LevelGeom {
    int k = 0;
    double spacing = 0;
    double origin[3] = {0, 0, 0};
    int dims[3] = {0, 0, 0};
    size_t size = 0;
    size_t offset = 0; // into the concatenated lattice buffers
};

// Grid-to-grid transfer stencil for fine level k -> coarse level k+1, per axis:
// fine index i -> coarse base + 4 weights (stencil_at, src/msm_phases.cpp:21-29),
// and the inverse lists used by the restriction gather.
struct TransferAxis {
    std::vector<int> base;     // [d_fine]
    std::vector<double> w;     // [d_fine * 4]
    std::vector<int> rcnt;     // [d_coarse]
    std::vector<int> ridx;     // [d_coarse * kRestrictMax], ascending fine index
    std::vector<double> rw;    // [d_coarse * kRestrictMax]
};

struct int2_ {
    int x, y;
};

struct ConvRow { // one (dx, dy) row of a 3-D stencil: taps for dz = -m..m
    int dx, dy, m, tap_off;
};

struct ConvTable {
    int Rx = 0, Ry = 0, Rz = 0;       // stencil half-extents (grid units)
    std::vector<ConvRow> rows;        // sorted by dx, then dy
    std::vector<int> dx_begin;        // [2*Rx + 2]: rows of dx are [dx_begin[dx+Rx], dx_begin[dx+Rx+1])
    std::vector<double> taps;         // each row padded to a multiple of kConvL
    int64_t nonzero_taps = 0;         // nonzero taps in the stencil
};

// Level-0 lattice-cutoff stencil in the layout of k_lattice: for every (dx, dy)
// row with a nonzero tap, the taps for dz = -R..R at index dz + R, zero padded to
// a multiple of 4; level k uses 2^-k times these values (bit-identical to the
// reference's per-level table, see msmb_geometry.cpp).
struct LatticeTable {
    int R = 0, TW = 0, nrows = 0;
    std::vector<int> rowidx;   // [(2R+1)^2]: row id of (dx, dy) or -1
    std::vector<int2_> rowchunks; // [nrows]: first / last 4-tap chunk holding nonzero taps
    std::vector<double> taps;  // [nrows * TW]
};

// Pair-only fields (paramd::SimpleCutoffField / WolfField, force_field.hpp:34-60):
// the MSM engine's binning, cluster pair list and pair kernel with another pair
// function and no grid hierarchy.
struct PairFieldP {
    int kind = MSMB_FIELD_MSM;   // msmb_field_kind
    double alpha = 0;            // Wolf damping
    double e_shift = 0, f_shift = 0, self_per_charge = 0; // src/electrostatics.cpp:96-102
    // erfc(x) = exp(-x^2) erfcx(x) with erfcx as a degree-kWolfDeg polynomial in
    // u = 2x/X - 1 on [0, X = alpha a] (Chebyshev interpolation; |rel err| <= 2e-14
    // for X <= 4.5); wolf_fast = 0 falls back to libdevice erfc
    int wolf_fast = 0;
    double wolf_us = 0;          // 2 alpha / X: u = wolf_us r - 1
    double wolf_c[29] = {};      // monomial coefficients in u, degree kWolfDeg
};
constexpr int kWolfDeg = 28;

struct Geometry {
    int kind = MSMB_FIELD_MSM;           // MSM, or a pair-only field (no hierarchy; binning clamps)
    PairFieldP pf{};
    msmb_msm_config cfg{};
    msmb_units units{};
    double box[3] = {0, 0, 0};
    int levels = 0;
    LevelGeom lv[kMaxLevels];
    size_t lattice_total = 0;
    TransferAxis tr[kMaxLevels][3];      // tr[k][axis], k = 0..levels-2
    ConvTable lattice[kMaxLevels];       // k = 0..levels-2
    ConvTable top;
    LatticeTable lat;                    // shared level-0 stencil for k_lattice
    double inv_h0 = 0;                   // 1.0 / spacing of level 0
    double self_term = 0;                // smoothing_gamma(0)/a (src/msm.cpp:72)
    // pair-cell (column) decomposition over level-0 cells
    int cw = 1;                          // column width in level-0 cells
    int ncx = 0, ncy = 0;                // columns
    int64_t ncells = 0;                  // sorted-cell index space
    int64_t ncols = 0;
    double colw = 0;                     // column width in Angstrom
    double screen_cut = 0;               // fp32 bounding-box cutoff (a + margin); the per-atom
                                         // screen in k_pairs pads its own rounding bound
    double skin = 0;                     // pair-list skin (A): rebuilt once an atom moved > skin/2
    int pair_cap = 0;                    // initial pair-list capacity per cluster
    int dense_t = 0;                     // dense threshold: a j atom within the list cut of >= dense_t of an
                                         // i-cluster's 32 atoms is summed by the whole warp in lockstep (0 = off)
    int dense_cap = 0;                   // dense j atoms kept per i-cluster (multiple of 32)
    int64_t lattice_taps_clipped = 0;    // sum over levels 0..l-2 of clipped nonzero taps
    int64_t top_taps = 0;                // M_top^2
};

// Work owned by one part of a spatial decomposition (one part
// per GPU): the pair sum for i-clusters in pair columns [cx0, cx1) along x (all
// y), anterpolation of level-0 planes [pl0[0], pl1[0]), the lattice cutoff of
// level-k output planes [pl0[k], pl1[k]) (starts multiples of 4, the k_lattice
// tile height), and interpolation + Verlet for the atoms binned into the owned
// pair columns.  nparts == 1 is the whole system.
struct Part {
    int nparts = 1, part = 0;
    int cx0 = 0, cx1 = 0;
    int pl0[kMaxLevels] = {}, pl1[kMaxLevels] = {};
};
Part make_part(const Geometry& g, int nparts, int part);

// Validation with the reference's messages.  Returns MSMB_OK or an error.
Error validate_config(const msmb_msm_config& c);
Error validate_units(const msmb_units& u);
// Builds the level hierarchy + all tables.  `n` sizes the pair-list estimate.
Error build_geometry(const msmb_msm_config& c, const msmb_units& u, const double box[3],
                     int64_t n, Geometry& g);
// Pair-only fields: CutoffParams::validate (src/electrostatics.cpp:38-42) and the
// binning geometry (cells of the level-0 layout over the box; atoms outside clamp).
Error validate_cutoff(int kind, const msmb_cutoff_params& p);
Error build_pair_geometry(int kind, const msmb_cutoff_params& p, const msmb_units& u,
                          const double box[3], int64_t n, Geometry& g);
// Reference kernel math on the host (bitwise the reference's, non-FMA).
double host_gamma(double rho);
double host_g_level(double r, double a, int k, int l);
double host_flops_simplified(double a, double h, double n);

} // namespace msmb
