// Host-side geometry and stencil tables (compiled with -ffp-contract=off so the
// arithmetic is the reference's non-FMA arithmetic, bit for bit).
//
//  * level hierarchy: build_grid_hierarchy, src/msm_grid.cpp:24-54
//  * validation:      MsmConfig::validate src/msm_grid.cpp:11-22,
//                     UnitsConfig::validate include/paramd/units.hpp:23-26
//  * transfer stencils (restriction/prolongation): stencil_at
//                     src/msm_phases.cpp:21-29 evaluated at fine grid points as in
//                     restrict_charges / prolongate (src/msm_phases.cpp:63-91,164-193)
//  * lattice-cutoff stencil: src/msm_phases.cpp:98-111 (same r and kernel call)
//  * top-level kernel table: src/msm_phases.cpp:136-162
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <string>

#include "msmb_internal.h"

namespace msmb {

double host_gamma(double rho) { // include/paramd/msm_kernels.hpp:14-20 (m = 2)
    if (rho >= 1.0) return 1.0 / rho;
    const double r2 = rho * rho;
    return 1.875 + r2 * (-1.25 + 0.375 * r2);
}

double host_g_level(double r, double a, int k, int l) { // msm_kernels.hpp:50-61
    const double ak = std::ldexp(a, k);
    if (k == l - 1) return host_gamma(r / ak) / ak;
    const double ak1 = 2.0 * ak;
    if (r >= ak1) return 0.0;
    return host_gamma(r / ak) / ak - host_gamma(r / ak1) / ak1;
}

static double host_phi(double xi) { // msm_kernels.hpp:71-78
    const double t = std::fabs(xi);
    if (t >= 2.0) return 0.0;
    if (t <= 1.0) return 1.0 + t * t * (-2.5 + 1.5 * t);
    const double u = 2.0 - t;
    return -0.5 * (t - 1.0) * u * u;
}

double host_flops_simplified(double a, double h, double n) { // src/cost_model.cpp:37-43
    const double a3 = a * a * a;
    const double h3 = h * h * h;
    return 77.7 * a3 * n + 566.0 * n + 73.0 * a3 / (h3 * h3) * n + 80.0 / h3 * n;
}

static Error err(int kind, const std::string& m) {
    Error e;
    e.kind = kind;
    e.msg = m;
    return e;
}

Error validate_config(const msmb_msm_config& c) {
    if (!(c.cutoff_a > 0.0)) return err(MSMB_ERR_CONFIG, "msm: cutoff_a must be > 0");
    if (!(c.spacing_h > 0.0)) return err(MSMB_ERR_CONFIG, "msm: spacing_h must be > 0");
    if (c.levels_l < 1) return err(MSMB_ERR_CONFIG, "msm: levels_l must be >= 1");
    if (c.interp_order_p != 3)
        return err(MSMB_ERR_CONFIG,
                   "msm: unsupported interpolation order p=" + std::to_string(c.interp_order_p));
    if (c.smoothing_m != 2)
        return err(MSMB_ERR_CONFIG,
                   "msm: unsupported smoothing order m=" + std::to_string(c.smoothing_m));
    if (c.cutoff_a / c.spacing_h < 1.0)
        return err(MSMB_ERR_CONFIG, "msm: cutoff_a / spacing_h must be >= 1");
    if (c.levels_l > kMaxLevels)
        return err(MSMB_ERR_CONFIG, "msm: levels_l > " + std::to_string(kMaxLevels) +
                                        " is not supported by this build");
    return Error{};
}

Error validate_units(const msmb_units& u) {
    if (!(u.coulomb_constant > 0.0)) return err(MSMB_ERR_CONFIG, "coulomb_constant must be > 0");
    if (!(u.energy_to_native > 0.0)) return err(MSMB_ERR_CONFIG, "energy_to_native must be > 0");
    return Error{};
}

// stencil_at (src/msm_phases.cpp:21-29); false when the stencil leaves the lattice
static bool stencil_at(double t, int dims, int& base, double w[4]) {
    const double f = std::floor(t);
    if (!(f >= 1.0) || !(f <= double(dims) - 3.0)) return false;
    base = int(f) - 1;
    for (int d = 0; d < 4; ++d) w[d] = host_phi(t - (base + d));
    return true;
}

static void finish_rows(ConvTable& t) {
    std::stable_sort(t.rows.begin(), t.rows.end(), [](const ConvRow& a, const ConvRow& b) {
        return a.dx != b.dx ? a.dx < b.dx : a.dy < b.dy;
    });
    t.dx_begin.assign(2 * t.Rx + 2, 0);
    for (const auto& r : t.rows) t.dx_begin[r.dx + t.Rx + 1]++;
    for (size_t i = 1; i < t.dx_begin.size(); ++i) t.dx_begin[i] += t.dx_begin[i - 1];
}

static void push_row(ConvTable& t, int dx, int dy, int m, const double* taps /* 2m+1 */) {
    ConvRow r{dx, dy, m, int(t.taps.size())};
    const int T = 2 * m + 1;
    const int padded = (T + kConvL - 1) / kConvL * kConvL;
    for (int i = 0; i < padded; ++i) t.taps.push_back(i < T ? taps[i] : 0.0);
    t.rows.push_back(r);
}

static void build_lattice_table(const Geometry& g, int k, ConvTable& t) {
    const double a = g.cfg.cutoff_a, h = g.cfg.spacing_h;
    const int R = int(std::ceil(2.0 * a / h)); // src/msm_phases.cpp:99-100
    t.Rx = t.Ry = t.Rz = R;
    const int w = 2 * R + 1;
    std::vector<double> st(size_t(w) * w * w);
    const LevelGeom& L = g.lv[k];
    for (int di = -R; di <= R; ++di)
        for (int dj = -R; dj <= R; ++dj)
            for (int dk = -R; dk <= R; ++dk) {
                const double r =
                    L.spacing * std::sqrt(double(di) * di + double(dj) * dj + double(dk) * dk);
                st[(size_t(di + R) * w + (dj + R)) * w + (dk + R)] =
                    host_g_level(r, a, L.k, g.levels);
            }
    t.nonzero_taps = 0;
    std::vector<double> row(w);
    for (int di = -R; di <= R; ++di)
        for (int dj = -R; dj <= R; ++dj) {
            int m = -1;
            for (int dk = -R; dk <= R; ++dk) {
                const double v = st[(size_t(di + R) * w + (dj + R)) * w + (dk + R)];
                if (v != 0.0) {
                    m = std::max(m, std::abs(dk));
                    ++t.nonzero_taps;
                }
            }
            if (m < 0) continue;
            for (int dk = -m; dk <= m; ++dk) row[dk + m] = st[(size_t(di + R) * w + (dj + R)) * w + (dk + R)];
            push_row(t, di, dj, m, row.data());
        }
    finish_rows(t);
}

static void build_top_table(const Geometry& g, ConvTable& t) {
    const LevelGeom& T = g.lv[g.levels - 1];
    t.Rx = T.dims[0] - 1;
    t.Ry = T.dims[1] - 1;
    t.Rz = T.dims[2] - 1;
    const double s = T.spacing;
    std::vector<double> row(2 * t.Rz + 1);
    for (int di = -t.Rx; di <= t.Rx; ++di)
        for (int dj = -t.Ry; dj <= t.Ry; ++dj) {
            for (int dk = -t.Rz; dk <= t.Rz; ++dk) {
                // r = norm(coords[lo] - coords[hi]) with coords = origin + i*spacing
                // (src/msm_phases.cpp:145-156); exact whenever the coordinates are.
                const double ax = T.origin[0] + 0 * s, bx = T.origin[0] + std::abs(di) * s;
                const double ay = T.origin[1] + 0 * s, by = T.origin[1] + std::abs(dj) * s;
                const double az = T.origin[2] + 0 * s, bz = T.origin[2] + std::abs(dk) * s;
                const double dx = ax - bx, dy = ay - by, dz = az - bz;
                const double r = std::sqrt(dx * dx + dy * dy + dz * dz);
                row[dk + t.Rz] = host_g_level(r, g.cfg.cutoff_a, T.k, g.levels);
            }
            push_row(t, di, dj, t.Rz, row.data());
        }
    t.nonzero_taps = int64_t(2 * t.Rx + 1) * (2 * t.Ry + 1) * (2 * t.Rz + 1);
    finish_rows(t);
}

static void set_pair_layout(Geometry& g, const msmb_msm_config& c, const double box[3], int64_t n);

Error build_geometry(const msmb_msm_config& c, const msmb_units& u, const double box[3],
                     int64_t n, Geometry& g) {
    Error e = validate_config(c);
    if (e.kind) return e;
    e = validate_units(u);
    if (e.kind) return e;
    if (!(box[0] > 0.0 && box[1] > 0.0 && box[2] > 0.0))
        return err(MSMB_ERR_CONFIG, "msm: box extents must be positive");
    g = Geometry{};
    g.cfg = c;
    g.units = u;
    for (int ax = 0; ax < 3; ++ax) g.box[ax] = box[ax];
    g.levels = c.levels_l;
    size_t off = 0;
    for (int k = 0; k < g.levels; ++k) { // src/msm_grid.cpp:31-52
        LevelGeom& L = g.lv[k];
        L.k = k;
        L.spacing = std::ldexp(c.spacing_h, k);
        for (int ax = 0; ax < 3; ++ax) {
            L.origin[ax] = -2.0 * L.spacing;
            int d = int(std::ceil(box[ax] / L.spacing)) + 5;
            if (k > 0) d = std::max(d, (g.lv[k - 1].dims[ax] + 1) / 2 + 3);
            if (d < 2)
                return err(MSMB_ERR_CONFIG, "msm: level " + std::to_string(k) +
                                                " would have fewer than 2 points per axis");
            L.dims[ax] = d;
        }
        L.size = size_t(L.dims[0]) * L.dims[1] * L.dims[2];
        L.offset = off;
        off += L.size;
    }
    g.lattice_total = off;
    g.inv_h0 = 1.0 / g.lv[0].spacing;
    g.self_term = host_gamma(0.0) / c.cutoff_a; // src/msm.cpp:72

    // transfer stencils, level k -> k+1
    for (int k = 0; k + 1 < g.levels; ++k) {
        const LevelGeom& F = g.lv[k];
        const LevelGeom& C = g.lv[k + 1];
        const double inv_s = 1.0 / C.spacing;
        for (int ax = 0; ax < 3; ++ax) {
            TransferAxis& T = g.tr[k][ax];
            T.base.assign(F.dims[ax], 0);
            T.w.assign(size_t(F.dims[ax]) * 4, 0.0);
            for (int i = 0; i < F.dims[ax]; ++i) {
                const double t = (F.origin[ax] + i * F.spacing - C.origin[ax]) * inv_s;
                int b;
                double w[4];
                if (!stencil_at(t, C.dims[ax], b, w))
                    return err(MSMB_ERR_COVERAGE,
                               "fine grid point " + std::to_string(i) + " outside grid coverage");
                T.base[i] = b;
                for (int d = 0; d < 4; ++d) T.w[size_t(i) * 4 + d] = w[d];
            }
            T.rcnt.assign(C.dims[ax], 0);
            T.ridx.assign(size_t(C.dims[ax]) * kRestrictMax, 0);
            T.rw.assign(size_t(C.dims[ax]) * kRestrictMax, 0.0);
            for (int i = 0; i < F.dims[ax]; ++i) // ascending fine index
                for (int d = 0; d < 4; ++d) {
                    const int I = T.base[i] + d;
                    const double w = T.w[size_t(i) * 4 + d];
                    if (w == 0.0) continue; // adds +-0: bitwise neutral
                    int& cnt = T.rcnt[I];
                    if (cnt >= kRestrictMax) return err(MSMB_ERR_INTERNAL, "restriction list overflow");
                    T.ridx[size_t(I) * kRestrictMax + cnt] = i;
                    T.rw[size_t(I) * kRestrictMax + cnt] = w;
                    ++cnt;
                }
        }
    }
    // stencils
    g.lattice_taps_clipped = 0;
    for (int k = 0; k + 1 < g.levels; ++k) {
        build_lattice_table(g, k, g.lattice[k]);
        // clipped nonzero FMAs: sum over nonzero offsets of prod(d - |off|)
        const ConvTable& t = g.lattice[k];
        const LevelGeom& L = g.lv[k];
        for (const auto& r : t.rows)
            for (int dz = -r.m; dz <= r.m; ++dz) {
                if (t.taps[r.tap_off + dz + r.m] == 0.0) continue;
                const int64_t ex = std::max(0, L.dims[0] - std::abs(r.dx));
                const int64_t ey = std::max(0, L.dims[1] - std::abs(r.dy));
                const int64_t ez = std::max(0, L.dims[2] - std::abs(dz));
                g.lattice_taps_clipped += ex * ey * ez;
            }
    }
    // k_lattice table: level-0 stencil, absolute dz layout (levels k > 0 scale by 2^-k)
    if (g.levels >= 2) {
        const ConvTable& t0 = g.lattice[0];
        LatticeTable& L = g.lat;
        L.R = t0.Rx;
        L.TW = (2 * L.R + 1 + 3) / 4 * 4;
        const int W = 2 * L.R + 1;
        L.rowidx.assign(size_t(W) * W, -1);
        for (const auto& r : t0.rows) {
            const int id = L.nrows++;
            L.rowidx[size_t(r.dx + L.R) * W + (r.dy + L.R)] = id;
            L.rowchunks.push_back(int2_{(L.R - r.m) / 4, (L.R + r.m) / 4});
            for (int i = 0; i < L.TW; ++i) {
                const int dz = i - L.R;
                L.taps.push_back((dz >= -r.m && dz <= r.m) ? t0.taps[r.tap_off + dz + r.m] : 0.0);
            }
        }
    }
    build_top_table(g, g.top);
    g.top_taps = int64_t(g.lv[g.levels - 1].size) * int64_t(g.lv[g.levels - 1].size);

    set_pair_layout(g, c, box, n);
    return Error{};
}

// Pair-search columns over level-0 cells, screening margin,
// pair-list skin and the initial list capacity.
static void set_pair_layout(Geometry& g, const msmb_msm_config& c, const double box[3], int64_t n) {
    const LevelGeom& L0 = g.lv[0];
    const double vol = box[0] * box[1] * box[2];
    const double rho = std::max(1e-6, double(std::max<int64_t>(n, 1)) / vol);
    const double edge = std::cbrt(32.0 / rho);
    g.cw = std::max(1, int(std::lround(edge / c.spacing_h)));
    g.cw = std::min(g.cw, std::max(1, std::min(L0.dims[0], L0.dims[1])));
    g.ncx = (L0.dims[0] + g.cw - 1) / g.cw;
    g.ncy = (L0.dims[1] + g.cw - 1) / g.cw;
    g.ncols = int64_t(g.ncx) * g.ncy;
    g.ncells = g.ncols * L0.dims[2] * int64_t(g.cw) * g.cw;
    g.colw = g.cw * L0.spacing;
    double maxabs = 0;
    for (int ax = 0; ax < 3; ++ax)
        maxabs = std::max(maxabs, std::fabs(L0.origin[ax]) + L0.dims[ax] * L0.spacing);
    const double margin = 8.0 * std::ldexp(1.0, -24) * (2.0 * maxabs + c.cutoff_a) + 1e-6 * c.cutoff_a;
    g.screen_cut = c.cutoff_a + margin;
    // pair-list skin: the cluster pair list is rebuilt only once some atom moved more
    // than skin/2 since the last build (MSMB_SKIN overrides, 0 = rebuild every evaluation)
    g.skin = 0.2;
    if (const char* e = std::getenv("MSMB_SKIN")) g.skin = std::max(0.0, std::atof(e));
    {
        const double zext = 32.0 / (rho * g.colw * g.colw);
        const double lc = c.cutoff_a + g.skin;
        const double ext_xy = 2.0 * (g.colw + lc);
        const double ext_z = 2.0 * (std::min(zext, box[2] + 4 * L0.spacing) + lc);
        const double ncand = 1.5 * rho * ext_xy * ext_xy * ext_z / 32.0;
        const double ncol_range = (ext_xy / g.colw + 1) * (ext_xy / g.colw + 1);
        double cap = ncand + 2.0 * ncol_range + 32.0;
        cap = std::min(cap, 1.0e6);
        g.pair_cap = std::max(64, int(cap));
        // dense j atoms of an i-cluster lie within the list cut of most of its atoms: at most
        // about a sphere of that radius (k_pairmask leaves the excess to the per-lane masks)
        g.dense_t = 28;
        if (const char* e = std::getenv("MSMB_DENSE_T")) g.dense_t = std::max(0, std::min(33, std::atoi(e)));
        if (g.dense_t > 32) g.dense_t = 0;
        const double sphere = 4.18879 * lc * lc * lc * rho;
        g.dense_cap = int(std::min(4096.0, std::max(64.0, 1.4 * sphere + 64.0)));
        if (const char* e = std::getenv("MSMB_DENSE_CAP")) g.dense_cap = std::max(32, std::atoi(e)); // tests: overflow path
        g.dense_cap = (g.dense_cap + 31) & ~31;
    }
}

Error validate_cutoff(int kind, const msmb_cutoff_params& p) { // src/electrostatics.cpp:38-42
    if (kind != MSMB_FIELD_CUTOFF && kind != MSMB_FIELD_WOLF)
        return err(MSMB_ERR_CONFIG, "unknown pair field kind " + std::to_string(kind));
    if (!(p.cutoff > 0.0)) return err(MSMB_ERR_CONFIG, "cutoff must be > 0");
    if (kind == MSMB_FIELD_WOLF && !p.has_wolf_alpha) return err(MSMB_ERR_CONFIG, "wolf_alpha is required");
    if (p.has_wolf_alpha && !(p.wolf_alpha >= 0.0)) return err(MSMB_ERR_CONFIG, "wolf_alpha must be >= 0");
    return Error{};
}

// Pair-only fields: one "level" that only lays out the binning cells (the MSM
// level-0 layout: origin -2s, dims ceil(L/s) + 5, cells 1 .. dims-3 used), with the
// cell size s = max(a/4, (V/n)^(1/3)) so the cell count stays O(n); no hierarchy.
Error build_pair_geometry(int kind, const msmb_cutoff_params& p, const msmb_units& u,
                          const double box[3], int64_t n, Geometry& g) {
    Error e = validate_cutoff(kind, p);
    if (e.kind) return e;
    e = validate_units(u);
    if (e.kind) return e;
    if (!(box[0] > 0.0 && box[1] > 0.0 && box[2] > 0.0) || !std::isfinite(box[0] * box[1] * box[2]))
        return err(MSMB_ERR_CONFIG, "pair field: box extents must be positive and finite (binning extent)");
    const double vol = box[0] * box[1] * box[2];
    const double s = std::max(p.cutoff / 4.0, std::cbrt(vol / double(std::max<int64_t>(n, 1))));
    msmb_msm_config c{p.cutoff, s, 1, 3, 2};
    g = Geometry{};
    g.kind = kind;
    g.cfg = c;
    g.units = u;
    for (int ax = 0; ax < 3; ++ax) g.box[ax] = box[ax];
    g.levels = 1;
    LevelGeom& L0 = g.lv[0];
    L0.spacing = s;
    for (int ax = 0; ax < 3; ++ax) {
        L0.origin[ax] = -2.0 * s;
        L0.dims[ax] = int(std::ceil(box[ax] / s)) + 5;
    }
    L0.size = size_t(L0.dims[0]) * L0.dims[1] * L0.dims[2];
    g.lattice_total = L0.size;
    g.inv_h0 = 1.0 / s;
    PairFieldP& pf = g.pf;
    pf.kind = kind;
    if (kind == MSMB_FIELD_WOLF) { // src/electrostatics.cpp:91-102, same operations
        const double a = p.cutoff, alpha = p.wolf_alpha;
        const double two_over_sqrt_pi = 1.1283791670955126;
        const double erfc_aa = std::erfc(alpha * a);
        pf.alpha = alpha;
        pf.e_shift = erfc_aa / a;
        pf.f_shift = erfc_aa / (a * a) + two_over_sqrt_pi * alpha * std::exp(-alpha * alpha * a * a) / a;
        pf.self_per_charge = -(pf.e_shift + two_over_sqrt_pi * alpha);
        // erfcx(x) on [0, X] (only pairs with r < a, i.e. x < X, are accumulated):
        // interpolation at the D+1 Chebyshev points in long double, then the monomial
        // coefficients in u (sum |a_k| ~ 1 on [-1, 1], so Horner loses nothing)
        const double X = alpha * a * (1.0 + 1e-9);
        if (X >= 1e-3 && X <= 4.5) {
            const int D = kWolfDeg;
            const long double PI = 3.141592653589793238462643383279502884L;
            long double f[kWolfDeg + 1], c[kWolfDeg + 1];
            for (int j = 0; j <= D; ++j) {
                const long double u = cosl(PI * (j + 0.5L) / (D + 1));
                const long double x = (u + 1.0L) * 0.5L * X;
                f[j] = expl(x * x) * erfcl(x);
            }
            for (int k = 0; k <= D; ++k) {
                long double acc = 0;
                for (int j = 0; j <= D; ++j) acc += f[j] * cosl(PI * k * (j + 0.5L) / (D + 1));
                c[k] = acc * 2.0L / (D + 1);
            }
            c[0] *= 0.5L;
            // Chebyshev -> monomial: T_{k+1} = 2u T_k - T_{k-1}
            long double T0[kWolfDeg + 1] = {}, T1[kWolfDeg + 1] = {}, T2[kWolfDeg + 1], mono[kWolfDeg + 1] = {};
            T0[0] = 1;
            T1[1] = 1;
            for (int i = 0; i <= D; ++i) mono[i] += c[0] * T0[i];
            for (int i = 0; i <= D; ++i) mono[i] += c[1] * T1[i];
            for (int k = 2; k <= D; ++k) {
                for (int i = 0; i <= D; ++i) T2[i] = (i > 0 ? 2.0L * T1[i - 1] : 0.0L) - T0[i];
                for (int i = 0; i <= D; ++i) mono[i] += c[k] * T2[i];
                for (int i = 0; i <= D; ++i) {
                    T0[i] = T1[i];
                    T1[i] = T2[i];
                }
            }
            for (int i = 0; i <= D; ++i) pf.wolf_c[i] = double(mono[i]);
            pf.wolf_us = 2.0 * alpha / X;
            pf.wolf_fast = std::getenv("MSMB_WOLF_LIBDEVICE") ? 0 : 1;
        }
    }
    set_pair_layout(g, c, box, n);
    return Error{};
}

// Even split of [0, n) into `parts` ranges, range `part`, boundaries rounded down
// to multiples of `align` (the last range ends at n).
static void split_range(int n, int parts, int part, int align, int& b, int& e) {
    auto cut = [&](int k) {
        if (k >= parts) return n;
        const int64_t c = int64_t(n) * k / parts;
        return int(c - c % align);
    };
    b = cut(part);
    e = cut(part + 1);
    if (e < b) e = b;
}

Part make_part(const Geometry& g, int nparts, int part) {
    Part P;
    P.nparts = nparts < 1 ? 1 : nparts;
    P.part = (part < 0 || part >= P.nparts) ? 0 : part;
    split_range(g.ncx, P.nparts, P.part, 1, P.cx0, P.cx1);
    for (int k = 0; k < g.levels; ++k) split_range(g.lv[k].dims[0], P.nparts, P.part, 4, P.pl0[k], P.pl1[k]);
    return P;
}

} // namespace msmb

