/*
 * oracle/msm_oracle.c -- TEST INFRASTRUCTURE ONLY.  Never linked into, loaded by,
 * or called from the product path (paper_1309_1889_b200/).  Only tests/,
 * bench.py's cpu_baseline / --impl reference legs and __graft_entry__.smoke()
 * may load it, and only as the checker.
 *
 * A plain-C restatement of the reference (`paramd`, /root/reference/proj) hot
 * path: MSM energy/forces, velocity Verlet and parareal.  It is written to be
 * BITWISE identical to the reference on the same inputs:
 *   - compiled with -ffp-contract=off (the reference is built without -march,
 *     so x86-64 never contracts mul+add into FMA), same operation order;
 *   - the O(N^2) short-range loop of src/msm_phases.cpp:233-250 is restated as
 *     an O(N) cell search that visits each atom's in-cutoff partners in
 *     ascending index order, which is exactly the order in which the
 *     reference's i<j loop adds contributions to that atom (partners j<i arrive
 *     while the outer loop is at j, partners j>i while it is at i);
 *   - lattice_cutoff / top_level scatter loops are restated as per-target
 *     gathers over sources in ascending row-major order, which is the order in
 *     which the reference's scatter reaches each target.
 * Pinned against oracle/_ref (the compiled reference) and tests/golden by
 * tests/test_oracle.py.  Errors use the integer codes of include/msmb.h and the
 * reference's message texts.
 */
#include <math.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum {
    OK = 0,
    E_CONFIG = 1,
    E_DOMAIN = 2,
    E_COVERAGE = 3,
    E_COINCIDENT = 4,
    E_HIERARCHY = 5,
    E_RUNTIME = 6,
    E_NONCONV = 7,
    E_OTHER = 9
};

static int fail(char* msg, int cap, int code, const char* fmt, ...) {
    if (msg && cap > 0) {
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(msg, (size_t)cap, fmt, ap);
        va_end(ap);
    }
    return code;
}

static int ok(char* msg, int cap) {
    if (msg && cap > 0) msg[0] = 0;
    return OK;
}

/* ---- kernel math: include/paramd/msm_kernels.hpp:14-92 ---------------------- */
static double smoothing_gamma(double rho) { /* msm_kernels.hpp:14-20 */
    if (rho >= 1.0) return 1.0 / rho;
    const double r2 = rho * rho;
    return 1.875 + r2 * (-1.25 + 0.375 * r2);
}
static double smoothing_gamma_deriv(double rho) { /* msm_kernels.hpp:22-27 */
    if (rho >= 1.0) return -1.0 / (rho * rho);
    return rho * (-2.5 + 1.5 * rho * rho);
}
static double kernel_g_star(double r, double a) { /* msm_kernels.hpp:30-35 */
    if (r >= a) return 0.0;
    return 1.0 / r - smoothing_gamma(r / a) / a;
}
static double kernel_g_star_deriv(double r, double a) { /* msm_kernels.hpp:37-42 */
    if (r >= a) return 0.0;
    return -1.0 / (r * r) - smoothing_gamma_deriv(r / a) / (a * a);
}
static double kernel_g_level(double r, double a, int k, int l) { /* msm_kernels.hpp:50-61 */
    const double ak = ldexp(a, k);
    if (k == l - 1) return smoothing_gamma(r / ak) / ak;
    const double ak1 = 2.0 * ak;
    if (r >= ak1) return 0.0;
    return smoothing_gamma(r / ak) / ak - smoothing_gamma(r / ak1) / ak1;
}
static double basis_phi(double xi) { /* msm_kernels.hpp:71-78 */
    const double t = fabs(xi);
    if (t >= 2.0) return 0.0;
    if (t <= 1.0) return 1.0 + t * t * (-2.5 + 1.5 * t);
    const double u = 2.0 - t;
    return -0.5 * (t - 1.0) * u * u;
}
static double basis_phi_deriv(double xi) { /* msm_kernels.hpp:80-92 */
    const double t = fabs(xi);
    double d;
    if (t >= 2.0)
        d = 0.0;
    else if (t <= 1.0)
        d = t * (-5.0 + 4.5 * t);
    else
        d = -0.5 * (2.0 - t) * (4.0 - 3.0 * t);
    return xi < 0.0 ? -d : d;
}

double orc_kernel(int which, double x, double a, int k, int l) {
    switch (which) {
        case 0: return smoothing_gamma(x);
        case 1: return smoothing_gamma_deriv(x);
        case 2: return kernel_g_star(x, a);
        case 3: return kernel_g_star_deriv(x, a);
        case 4: return kernel_g_level(x, a, k, l);
        case 5: return basis_phi(x);
        case 6: return basis_phi_deriv(x);
    }
    return NAN;
}

/* ---- configuration: MsmConfig::validate src/msm_grid.cpp:11-22,
 *      UnitsConfig::validate include/paramd/units.hpp:23-26 --------------------- */
typedef struct {
    double a, h;
    int l, p, m;
} cfg_t;

static int validate_cfg(const cfg_t* c, char* msg, int cap) {
    if (!(c->a > 0.0)) return fail(msg, cap, E_CONFIG, "msm: cutoff_a must be > 0");
    if (!(c->h > 0.0)) return fail(msg, cap, E_CONFIG, "msm: spacing_h must be > 0");
    if (c->l < 1) return fail(msg, cap, E_CONFIG, "msm: levels_l must be >= 1");
    if (c->p != 3)
        return fail(msg, cap, E_CONFIG, "msm: unsupported interpolation order p=%d", c->p);
    if (c->m != 2)
        return fail(msg, cap, E_CONFIG, "msm: unsupported smoothing order m=%d", c->m);
    if (c->a / c->h < 1.0) return fail(msg, cap, E_CONFIG, "msm: cutoff_a / spacing_h must be >= 1");
    return OK;
}

static int validate_units(double kc, double conv, char* msg, int cap) {
    if (!(kc > 0.0)) return fail(msg, cap, E_CONFIG, "coulomb_constant must be > 0");
    if (!(conv > 0.0)) return fail(msg, cap, E_CONFIG, "energy_to_native must be > 0");
    return OK;
}

/* ---- grid hierarchy: src/msm_grid.cpp:24-54 --------------------------------- */
typedef struct {
    int level;
    double spacing;
    double origin[3];
    int dims[3];
    size_t size;
    double* charge;
    double* potential;
} level_t;

static int build_levels(const double* box, const cfg_t* c, level_t* lv, int alloc, char* msg,
                        int cap) {
    int rc = validate_cfg(c, msg, cap);
    if (rc) return rc;
    if (!(box[0] > 0.0 && box[1] > 0.0 && box[2] > 0.0))
        return fail(msg, cap, E_CONFIG, "msm: box extents must be positive");
    for (int k = 0; k < c->l; ++k) {
        level_t* L = &lv[k];
        L->level = k;
        L->spacing = ldexp(c->h, k);
        for (int ax = 0; ax < 3; ++ax) {
            L->origin[ax] = -2.0 * L->spacing;
            int d = (int)ceil(box[ax] / L->spacing) + 5;
            if (k > 0) {
                const int fine_d = lv[k - 1].dims[ax];
                const int dd = (fine_d + 1) / 2 + 3;
                if (dd > d) d = dd;
            }
            if (d < 2)
                return fail(msg, cap, E_CONFIG,
                            "msm: level %d would have fewer than 2 points per axis", k);
            L->dims[ax] = d;
        }
        L->size = (size_t)L->dims[0] * L->dims[1] * L->dims[2];
        L->charge = L->potential = NULL;
        if (alloc) {
            L->charge = (double*)calloc(L->size, sizeof(double));
            L->potential = (double*)calloc(L->size, sizeof(double));
        }
    }
    return OK;
}

static void free_levels(level_t* lv, int l) {
    for (int k = 0; k < l; ++k) {
        free(lv[k].charge);
        free(lv[k].potential);
    }
}

#define IDX(L, i, j, k) (((size_t)(i) * (L)->dims[1] + (j)) * (L)->dims[2] + (k))

int orc_grid_geometry(const double* box, double a, double h, int levels, int p, int m,
                      int* dims_out, double* spacing_out, double* origin_out, char* msg,
                      int cap) {
    cfg_t c = {a, h, levels, p, m};
    if (levels < 1 || levels > 64) return validate_cfg(&c, msg, cap) ? E_CONFIG : E_CONFIG;
    level_t lv[64];
    int rc = build_levels(box, &c, lv, 0, msg, cap);
    if (rc) return rc;
    for (int k = 0; k < levels; ++k) {
        for (int ax = 0; ax < 3; ++ax) {
            dims_out[3 * k + ax] = lv[k].dims[ax];
            origin_out[3 * k + ax] = lv[k].origin[ax];
        }
        spacing_out[k] = lv[k].spacing;
    }
    return ok(msg, cap);
}

/* ---- stencil_at: src/msm_phases.cpp:21-29 ------------------------------------ */
typedef struct {
    int base;
    double w[4];
} st1d;

/* returns 0 if covered; the reference casts floor(t) to int, a non-finite or
 * out-of-int t can never be covered, so the range test is done in double. */
static int stencil_at(double t, int dims, st1d* st) {
    const double f = floor(t);
    if (!(f >= 1.0) || !(f <= (double)dims - 3.0)) return 1;
    st->base = (int)f - 1;
    for (int d = 0; d < 4; ++d) st->w[d] = basis_phi(t - (st->base + d));
    return 0;
}

/* ---- anterpolate: src/msm_phases.cpp:39-61 ----------------------------------
 * The reference scatters particle by particle (index order).  Here each thread
 * owns a range of x-planes and runs the same index-order loop, adding only into its
 * planes: every grid point still receives its contributions in particle order, so
 * the lattice is bitwise the reference's.  The coverage error is the first failing
 * particle in index order (checked before any scatter). */
static int anterpolate(int64_t n, const double* pos, const double* q, level_t* L0, char* msg,
                       int cap) {
    memset(L0->charge, 0, L0->size * sizeof(double));
    const double inv_h = 1.0 / L0->spacing;
    for (int64_t p = 0; p < n; ++p) {
        st1d sx, sy, sz;
        if (stencil_at((pos[3 * p] - L0->origin[0]) * inv_h, L0->dims[0], &sx) ||
            stencil_at((pos[3 * p + 1] - L0->origin[1]) * inv_h, L0->dims[1], &sy) ||
            stencil_at((pos[3 * p + 2] - L0->origin[2]) * inv_h, L0->dims[2], &sz))
            return fail(msg, cap, E_COVERAGE, "particle %lld outside grid coverage",
                        (long long)p);
    }
#pragma omp parallel
    {
        int nt = 1, me = 0;
#ifdef _OPENMP
        nt = omp_get_num_threads();
        me = omp_get_thread_num();
#endif
        const int x0 = (int)((int64_t)L0->dims[0] * me / nt), x1 = (int)((int64_t)L0->dims[0] * (me + 1) / nt);
        for (int64_t p = 0; p < n; ++p) {
            st1d sx, sy, sz;
            stencil_at((pos[3 * p] - L0->origin[0]) * inv_h, L0->dims[0], &sx);
            if (sx.base + 3 < x0 || sx.base >= x1) continue;
            stencil_at((pos[3 * p + 1] - L0->origin[1]) * inv_h, L0->dims[1], &sy);
            stencil_at((pos[3 * p + 2] - L0->origin[2]) * inv_h, L0->dims[2], &sz);
            const double qq = q[p];
            for (int a = 0; a < 4; ++a) {
                const int xi = sx.base + a;
                if (xi < x0 || xi >= x1) continue;
                const double qa = qq * sx.w[a];
                for (int b = 0; b < 4; ++b) {
                    const double qab = qa * sy.w[b];
                    for (int c = 0; c < 4; ++c)
                        L0->charge[IDX(L0, xi, sy.base + b, sz.base + c)] += qab * sz.w[c];
                }
            }
        }
    }
    return OK;
}

/* ---- restrict_charges: src/msm_phases.cpp:63-91 ----------------------------- */
static int restrict_charges(const level_t* F, level_t* C, char* msg, int cap) {
    memset(C->charge, 0, C->size * sizeof(double));
    const double inv_s = 1.0 / C->spacing;
    for (int i = 0; i < F->dims[0]; ++i) {
        const double tx = (F->origin[0] + i * F->spacing - C->origin[0]) * inv_s;
        for (int j = 0; j < F->dims[1]; ++j) {
            const double ty = (F->origin[1] + j * F->spacing - C->origin[1]) * inv_s;
            for (int k = 0; k < F->dims[2]; ++k) {
                const double q = F->charge[IDX(F, i, j, k)];
                if (q == 0.0) continue;
                const double tz = (F->origin[2] + k * F->spacing - C->origin[2]) * inv_s;
                st1d sx, sy, sz;
                if (stencil_at(tx, C->dims[0], &sx))
                    return fail(msg, cap, E_COVERAGE, "fine grid point %d outside grid coverage", i);
                if (stencil_at(ty, C->dims[1], &sy))
                    return fail(msg, cap, E_COVERAGE, "fine grid point %d outside grid coverage", j);
                if (stencil_at(tz, C->dims[2], &sz))
                    return fail(msg, cap, E_COVERAGE, "fine grid point %d outside grid coverage", k);
                for (int a = 0; a < 4; ++a) {
                    const double qa = q * sx.w[a];
                    for (int b = 0; b < 4; ++b) {
                        const double qab = qa * sy.w[b];
                        for (int c = 0; c < 4; ++c)
                            C->charge[IDX(C, sx.base + a, sy.base + b, sz.base + c)] += qab * sz.w[c];
                    }
                }
            }
        }
    }
    return OK;
}

/* ---- lattice_cutoff: src/msm_phases.cpp:93-134 ------------------------------
 * Restated as a gather: target t sums q_s * sten[t-s+R] over sources s with
 * q_s != 0 in ascending row-major order of s = the order of the reference's
 * scatter loop (each source adds at most once to each target). */
static void lattice_cutoff(level_t* L, const cfg_t* c) {
    const int radius = (int)ceil(2.0 * c->a / c->h);
    const int w = 2 * radius + 1;
    double* stencil = (double*)malloc((size_t)w * w * w * sizeof(double));
    for (int di = -radius; di <= radius; ++di)
        for (int dj = -radius; dj <= radius; ++dj)
            for (int dk = -radius; dk <= radius; ++dk) {
                const double r = L->spacing * sqrt((double)di * di + (double)dj * dj + (double)dk * dk);
                stencil[((size_t)(di + radius) * w + (dj + radius)) * w + (dk + radius)] =
                    kernel_g_level(r, c->a, L->level, c->l);
            }
    const int* dims = L->dims;
#pragma omp parallel for schedule(dynamic, 1) collapse(2)
    for (int ti = 0; ti < dims[0]; ++ti)
        for (int tj = 0; tj < dims[1]; ++tj)
            for (int tk = 0; tk < dims[2]; ++tk) {
                double acc = 0.0;
                const int ilo = ti - radius < 0 ? 0 : ti - radius;
                const int ihi = ti + radius > dims[0] - 1 ? dims[0] - 1 : ti + radius;
                const int jlo = tj - radius < 0 ? 0 : tj - radius;
                const int jhi = tj + radius > dims[1] - 1 ? dims[1] - 1 : tj + radius;
                const int klo = tk - radius < 0 ? 0 : tk - radius;
                const int khi = tk + radius > dims[2] - 1 ? dims[2] - 1 : tk + radius;
                for (int i = ilo; i <= ihi; ++i)
                    for (int j = jlo; j <= jhi; ++j)
                        for (int k = klo; k <= khi; ++k) {
                            const double q = L->charge[IDX(L, i, j, k)];
                            if (q == 0.0) continue;
                            acc += q * stencil[((size_t)(ti - i + radius) * w + (tj - j + radius)) * w +
                                               (tk - k + radius)];
                        }
                L->potential[IDX(L, ti, tj, tk)] = acc;
            }
    free(stencil);
}

/* ---- top_level: src/msm_phases.cpp:136-162 ----------------------------------
 * Gather restatement: point p receives g(mu,p) q_mu for mu<p in ascending mu,
 * then self*q_p, then g(p,nu) q_nu for nu>p -- the reference's order.  r is
 * norm(coords[min]-coords[max]) as in the reference (norm is sign-symmetric). */
static void top_level(level_t* T, const cfg_t* c) {
    const size_t m = T->size;
    const double self = kernel_g_level(0.0, c->a, T->level, c->l);
    double* cx = (double*)malloc(m * 3 * sizeof(double));
    size_t idx = 0;
    for (int i = 0; i < T->dims[0]; ++i)
        for (int j = 0; j < T->dims[1]; ++j)
            for (int k = 0; k < T->dims[2]; ++k) {
                cx[3 * idx] = T->origin[0] + i * T->spacing;
                cx[3 * idx + 1] = T->origin[1] + j * T->spacing;
                cx[3 * idx + 2] = T->origin[2] + k * T->spacing;
                ++idx;
            }
#pragma omp parallel for schedule(dynamic, 16)
    for (size_t p = 0; p < m; ++p) {
        double acc = 0.0;
        for (size_t s = 0; s < m; ++s) {
            if (s == p) {
                acc += self * T->charge[p];
                continue;
            }
            const size_t lo = s < p ? s : p, hi = s < p ? p : s;
            const double dx = cx[3 * lo] - cx[3 * hi];
            const double dy = cx[3 * lo + 1] - cx[3 * hi + 1];
            const double dz = cx[3 * lo + 2] - cx[3 * hi + 2];
            const double r = sqrt(dx * dx + dy * dy + dz * dz);
            const double g = kernel_g_level(r, c->a, T->level, c->l);
            acc += g * T->charge[s];
        }
        T->potential[p] = acc;
    }
    free(cx);
}

/* ---- prolongate: src/msm_phases.cpp:164-193 --------------------------------- */
static int prolongate(const level_t* C, level_t* F, char* msg, int cap) {
    const double inv_s = 1.0 / C->spacing;
    int bad = -1;
#pragma omp parallel for schedule(static)
    for (int i = 0; i < F->dims[0]; ++i) {
        const double tx = (F->origin[0] + i * F->spacing - C->origin[0]) * inv_s;
        st1d sx;
        if (stencil_at(tx, C->dims[0], &sx)) {
            bad = i;
            continue;
        }
        for (int j = 0; j < F->dims[1]; ++j) {
            const double ty = (F->origin[1] + j * F->spacing - C->origin[1]) * inv_s;
            st1d sy;
            if (stencil_at(ty, C->dims[1], &sy)) {
                bad = j;
                continue;
            }
            for (int k = 0; k < F->dims[2]; ++k) {
                const double tz = (F->origin[2] + k * F->spacing - C->origin[2]) * inv_s;
                st1d sz;
                if (stencil_at(tz, C->dims[2], &sz)) {
                    bad = k;
                    continue;
                }
                double acc = 0.0;
                for (int a = 0; a < 4; ++a) {
                    double accb = 0.0;
                    for (int b = 0; b < 4; ++b) {
                        double accc = 0.0;
                        for (int cc = 0; cc < 4; ++cc)
                            accc += sz.w[cc] * C->potential[IDX(C, sx.base + a, sy.base + b, sz.base + cc)];
                        accb += sy.w[b] * accc;
                    }
                    acc += sx.w[a] * accb;
                }
                F->potential[IDX(F, i, j, k)] += acc;
            }
        }
    }
    if (bad >= 0) return fail(msg, cap, E_COVERAGE, "fine grid point %d outside grid coverage", bad);
    return OK;
}

/* ---- interpolate_to_atoms: src/msm_phases.cpp:195-222 ----------------------- */
static int interpolate(int64_t n, const double* pos, const level_t* L0, double* u, char* msg,
                       int cap) {
    const double inv_h = 1.0 / L0->spacing;
    int64_t bad = -1;
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < n; ++p) {
        st1d sx, sy, sz;
        if (stencil_at((pos[3 * p] - L0->origin[0]) * inv_h, L0->dims[0], &sx) ||
            stencil_at((pos[3 * p + 1] - L0->origin[1]) * inv_h, L0->dims[1], &sy) ||
            stencil_at((pos[3 * p + 2] - L0->origin[2]) * inv_h, L0->dims[2], &sz)) {
#pragma omp critical
            if (bad < 0 || p < bad) bad = p;
            continue;
        }
        double acc = 0.0;
        for (int a = 0; a < 4; ++a) {
            double accb = 0.0;
            for (int b = 0; b < 4; ++b) {
                double accc = 0.0;
                for (int c = 0; c < 4; ++c)
                    accc += sz.w[c] * L0->potential[IDX(L0, sx.base + a, sy.base + b, sz.base + c)];
                accb += sy.w[b] * accc;
            }
            acc += sx.w[a] * accb;
        }
        u[p] = acc;
    }
    if (bad >= 0) return fail(msg, cap, E_COVERAGE, "particle %lld outside grid coverage", (long long)bad);
    return OK;
}

/* ---- short_range: src/msm_phases.cpp:224-252 --------------------------------
 * O(N) restatement with cells of edge >= a; see the file header for why the
 * per-atom results are bitwise those of the reference's i<j loop.  Error
 * precedence is the reference's: the lexicographically first pair (i<j) whose
 * r2 is 0 (CoincidentParticlesError) or NaN (DomainError from kernel_g_star). */
static int isfin3(const double* p) { return isfinite(p[0]) && isfinite(p[1]) && isfinite(p[2]); }

static double pair_r2(const double* pos, int64_t i, int64_t j) { /* i < j, as the reference */
    const double dx = pos[3 * i] - pos[3 * j];
    const double dy = pos[3 * i + 1] - pos[3 * j + 1];
    const double dz = pos[3 * i + 2] - pos[3 * j + 2];
    return dx * dx + dy * dy + dz * dz;
}

typedef struct {
    int64_t* j;
    size_t cap;
    int64_t* t; /* radix-sort scratch */
} jbuf_t;

/* ascending sort of indices < n (LSD radix, 8-bit digits): the reference's j order */
static void radix_sort(int64_t* a, int64_t* tmp, size_t cnt, int64_t n) {
    int64_t* src = a;
    int64_t* dst = tmp;
    for (int shift = 0; ((int64_t)1 << shift) < n && shift < 64; shift += 8) {
        size_t hist[257] = {0};
        for (size_t k = 0; k < cnt; ++k) hist[((src[k] >> shift) & 255) + 1]++;
        for (int b = 0; b < 256; ++b) hist[b + 1] += hist[b];
        for (size_t k = 0; k < cnt; ++k) dst[hist[(src[k] >> shift) & 255]++] = src[k];
        int64_t* t = src;
        src = dst;
        dst = t;
    }
    if (src != a) memcpy(a, src, cnt * sizeof(int64_t));
}

static int cmp_i64(const void* a, const void* b) {
    const int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return x < y ? -1 : x > y;
}

/* scan_only: run the error scan and skip the pair sum (phi/force untouched) */
static int short_range_impl(int64_t n, const double* pos, const double* q, double a, double kc,
                            double* phi, double* force, char* msg, int cap, int scan_only) {
    if (!scan_only)
        for (int64_t i = 0; i < n; ++i) {
            phi[i] = 0.0;
            force[3 * i] = force[3 * i + 1] = force[3 * i + 2] = 0.0;
        }
    if (n < 2) return ok(msg, cap);
    const double a2 = a * a;
    /* cell grid over the finite atoms */
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    int64_t nfin = 0;
    int64_t* nonfin = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    int64_t nnf = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (!isfin3(pos + 3 * i)) {
            nonfin[nnf++] = i;
            continue;
        }
        ++nfin;
        for (int ax = 0; ax < 3; ++ax) {
            if (pos[3 * i + ax] < lo[ax]) lo[ax] = pos[3 * i + ax];
            if (pos[3 * i + ax] > hi[ax]) hi[ax] = pos[3 * i + ax];
        }
    }
    int nc[3] = {1, 1, 1};
    double cs[3] = {1, 1, 1};
    if (nfin > 0)
        for (int ax = 0; ax < 3; ++ax) {
            const double ext = hi[ax] - lo[ax];
            double c = 0.5 * a; /* pair sum: cells of a/2, neighbours within 2 cells */
            if (ext / c > 1024.0) c = ext / 1024.0;
            cs[ax] = c;
            nc[ax] = (int)(ext / c) + 1;
            if (nc[ax] < 1) nc[ax] = 1;
        }
    const size_t ncell = (size_t)nc[0] * nc[1] * nc[2];
    int RX[3]; /* cells to search per axis for the pair sum */
    for (int ax = 0; ax < 3; ++ax) RX[ax] = (int)ceil(a / cs[ax]);
    int64_t* head = (int64_t*)malloc(sizeof(int64_t) * (ncell + 1));
    int64_t* cell_of = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    memset(head, 0, sizeof(int64_t) * (ncell + 1));
    for (int64_t i = 0; i < n; ++i) {
        cell_of[i] = -1;
        if (!isfin3(pos + 3 * i)) continue;
        int c3[3];
        for (int ax = 0; ax < 3; ++ax) {
            int c = (int)((pos[3 * i + ax] - lo[ax]) / cs[ax]);
            if (c >= nc[ax]) c = nc[ax] - 1;
            if (c < 0) c = 0;
            c3[ax] = c;
        }
        cell_of[i] = ((int64_t)c3[0] * nc[1] + c3[1]) * nc[2] + c3[2];
        head[cell_of[i] + 1]++;
    }
    for (size_t c = 0; c < ncell; ++c) head[c + 1] += head[c];
    {
        int64_t* fillp = (int64_t*)malloc(sizeof(int64_t) * ncell);
        memcpy(fillp, head, sizeof(int64_t) * ncell);
        for (int64_t i = 0; i < n; ++i)
            if (cell_of[i] >= 0) order[fillp[cell_of[i]]++] = i; /* ascending index per cell */
        free(fillp);
    }
    const double a2m = a2 * (1.0 + 1e-9) + 1e-300;
    double* spos = (double*)malloc(sizeof(double) * 3 * (size_t)(n > 0 ? n : 1));
    {
        const int64_t nb = head[ncell];
        for (int64_t s = 0; s < nb; ++s)
            for (int ax = 0; ax < 3; ++ax) spos[3 * s + ax] = pos[3 * order[s] + ax];
    }

    /* error scan: lexicographically first pair with r2 == 0 or r2 NaN */
    int64_t ei = -1, ej = -1;
#define CONSIDER(I, J)                                                  \
    do {                                                                \
        int64_t _i = (I), _j = (J);                                     \
        if (_i > _j) { int64_t _t = _i; _i = _j; _j = _t; }             \
        const double _r2 = pair_r2(pos, _i, _j);                        \
        if (_r2 == 0.0 || isnan(_r2)) {                                 \
            if (ei < 0 || _i < ei || (_i == ei && _j < ej)) { ei = _i; ej = _j; } \
        }                                                               \
    } while (0)
    for (int64_t t = 0; t < nnf; ++t)
        for (int64_t j = 0; j < n; ++j)
            if (j != nonfin[t]) CONSIDER(nonfin[t], j);
    /* coincident pairs among finite atoms (r2 == 0: equal coordinates, or differences
     * whose squares underflow) are in the same or adjacent cells; per-thread minima,
     * combined in a fixed order (the result is the global minimum either way) */
#pragma omp parallel
    {
        int64_t ti = -1, tj = -1;
#pragma omp for schedule(dynamic, 1024)
        for (int64_t i = 0; i < n; ++i) {
            if (cell_of[i] < 0) continue;
            const int64_t ci = cell_of[i];
            const int cz = (int)(ci % nc[2]), cy = (int)((ci / nc[2]) % nc[1]), cxx = (int)(ci / ((int64_t)nc[1] * nc[2]));
            for (int dx = -1; dx <= 1; ++dx)
                for (int dy = -1; dy <= 1; ++dy)
                    for (int dz = -1; dz <= 1; ++dz) {
                        const int x = cxx + dx, y = cy + dy, z = cz + dz;
                        if (x < 0 || y < 0 || z < 0 || x >= nc[0] || y >= nc[1] || z >= nc[2]) continue;
                        const int64_t c = ((int64_t)x * nc[1] + y) * nc[2] + z;
                        for (int64_t s = head[c]; s < head[c + 1]; ++s) {
                            const int64_t j = order[s];
                            if (j <= i) continue;
                            if (fabs(pos[3 * i] - pos[3 * j]) > 1e-100) continue; /* r2 > 0 for sure */
                            const double r2 = pair_r2(pos, i, j);
                            if (r2 == 0.0) {
                                if (ti < 0 || i < ti || (i == ti && j < tj)) { ti = i; tj = j; }
                            }
                        }
                    }
        }
#pragma omp critical
        {
            if (ti >= 0 && (ei < 0 || ti < ei || (ti == ei && tj < ej))) { ei = ti; ej = tj; }
        }
    }
#undef CONSIDER
    int rc = OK;
    if (ei >= 0) {
        const double r2 = pair_r2(pos, ei, ej);
        if (r2 == 0.0)
            rc = fail(msg, cap, E_COINCIDENT, "particles %lld and %lld coincide", (long long)ei,
                      (long long)ej);
        else
            rc = fail(msg, cap, E_DOMAIN, "kernel_g_star: r must be > 0");
    }

    if (rc == OK && !scan_only) {
#pragma omp parallel
        {
            jbuf_t jb = {NULL, 0, NULL};
#pragma omp for schedule(dynamic, 64)
            for (int64_t i = 0; i < n; ++i) {
                if (cell_of[i] < 0) continue;
                size_t cnt = 0;
                const int64_t ci = cell_of[i];
                const int cz = (int)(ci % nc[2]), cy = (int)((ci / nc[2]) % nc[1]),
                          cxx = (int)(ci / ((int64_t)nc[1] * nc[2]));
                const int cc3[3] = {cxx, cy, cz};
                const double xi0 = pos[3 * i], yi0 = pos[3 * i + 1], zi0 = pos[3 * i + 2];
                for (int dx = -RX[0]; dx <= RX[0]; ++dx)
                    for (int dy = -RX[1]; dy <= RX[1]; ++dy)
                        for (int dz = -RX[2]; dz <= RX[2]; ++dz) {
                            const int x = cxx + dx, y = cy + dy, z = cz + dz;
                            if (x < 0 || y < 0 || z < 0 || x >= nc[0] || y >= nc[1] || z >= nc[2]) continue;
                            /* skip cells entirely beyond the cutoff (gap between the cell boxes) */
                            const int dd[3] = {dx, dy, dz};
                            double gap2 = 0.0;
                            for (int ax = 0; ax < 3; ++ax) {
                                const int g = dd[ax] > 0 ? dd[ax] - 1 : (dd[ax] < 0 ? -dd[ax] - 1 : 0);
                                gap2 += (g * cs[ax]) * (g * cs[ax]);
                            }
                            (void)cc3;
                            if (gap2 > a2 * 1.000001) continue;
                            const int64_t c = ((int64_t)x * nc[1] + y) * nc[2] + z;
                            for (int64_t s = head[c]; s < head[c + 1]; ++s) {
                                /* cheap prefilter on the cell-ordered copy (a margin covers rounding);
                                 * the reference's r2 decides */
                                const double ex = spos[3 * s] - xi0, ey = spos[3 * s + 1] - yi0, ez = spos[3 * s + 2] - zi0;
                                if (ex * ex + ey * ey + ez * ez > a2m) continue;
                                const int64_t j = order[s];
                                if (j == i) continue;
                                const double r2 = i < j ? pair_r2(pos, i, j) : pair_r2(pos, j, i);
                                if (r2 >= a2) continue;
                                if (cnt == jb.cap) {
                                    jb.cap = jb.cap ? 2 * jb.cap : 1024;
                                    jb.j = (int64_t*)realloc(jb.j, jb.cap * sizeof(int64_t));
                                    jb.t = (int64_t*)realloc(jb.t, jb.cap * sizeof(int64_t));
                                }
                                jb.j[cnt++] = j;
                            }
                        }
                radix_sort(jb.j, jb.t, cnt, n);
                double ph = 0.0, fx = 0.0, fy = 0.0, fz = 0.0;
                const double qi = q[i];
                for (size_t t = 0; t < cnt; ++t) {
                    const int64_t j = jb.j[t];
                    const double qj = q[j];
                    if (j > i) { /* reference pair (i, j): F_i += f */
                        const double dx = pos[3 * i] - pos[3 * j];
                        const double dy = pos[3 * i + 1] - pos[3 * j + 1];
                        const double dz = pos[3 * i + 2] - pos[3 * j + 2];
                        const double r = sqrt(dx * dx + dy * dy + dz * dz);
                        const double g = kernel_g_star(r, a);
                        ph += qj * g;
                        const double dg = kernel_g_star_deriv(r, a);
                        const double s = -kc * qi * qj * dg / r;
                        fx += dx * s;
                        fy += dy * s;
                        fz += dz * s;
                    } else { /* reference pair (j, i): F_i -= f */
                        const double dx = pos[3 * j] - pos[3 * i];
                        const double dy = pos[3 * j + 1] - pos[3 * i + 1];
                        const double dz = pos[3 * j + 2] - pos[3 * i + 2];
                        const double r = sqrt(dx * dx + dy * dy + dz * dz);
                        const double g = kernel_g_star(r, a);
                        ph += qj * g;
                        const double dg = kernel_g_star_deriv(r, a);
                        const double s = -kc * qj * qi * dg / r;
                        fx -= dx * s;
                        fy -= dy * s;
                        fz -= dz * s;
                    }
                }
                phi[i] = ph;
                force[3 * i] = fx;
                force[3 * i + 1] = fy;
                force[3 * i + 2] = fz;
            }
            free(jb.j);
            free(jb.t);
        }
    }
    free(nonfin);
    free(head);
    free(cell_of);
    free(order);
    free(spos);
    return rc == OK ? ok(msg, cap) : rc;
}

int orc_short_range(int64_t n, const double* pos, const double* q, double a, double kc,
                    double* phi, double* force, char* msg, int cap) {
    return short_range_impl(n, pos, q, a, kc, phi, force, msg, cap, 0);
}

/* The particle anterpolate would report first (src/msm_phases.cpp:42-50: index
 * order, x then y then z), checked before the pair sum so that an aborting
 * evaluation does not pay for it; the outputs are those of the reference's order. */
static int coverage_scan(int64_t n, const double* pos, const level_t* L0, char* msg, int cap) {
    const double inv_h = 1.0 / L0->spacing;
    for (int64_t p = 0; p < n; ++p) {
        st1d sx, sy, sz;
        if (stencil_at((pos[3 * p] - L0->origin[0]) * inv_h, L0->dims[0], &sx) ||
            stencil_at((pos[3 * p + 1] - L0->origin[1]) * inv_h, L0->dims[1], &sy) ||
            stencil_at((pos[3 * p + 2] - L0->origin[2]) * inv_h, L0->dims[2], &sz))
            return fail(msg, cap, E_COVERAGE, "particle %lld outside grid coverage", (long long)p);
    }
    return OK;
}

/* ---- add_long_range_forces: src/msm.cpp:16-48 (file-local there) ----------- */
static void add_long_range_forces(int64_t n, const double* pos, const double* q, const level_t* L0, double kc,
                                  double* sf) {
    const double inv_h = 1.0 / L0->spacing;
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < n; ++p) {
        const double tx = (pos[3 * p] - L0->origin[0]) * inv_h;
        const double ty = (pos[3 * p + 1] - L0->origin[1]) * inv_h;
        const double tz = (pos[3 * p + 2] - L0->origin[2]) * inv_h;
        const int bx = (int)floor(tx) - 1, by = (int)floor(ty) - 1, bz = (int)floor(tz) - 1;
        double wx[4], wy[4], wz[4], dwx[4], dwy[4], dwz[4];
        for (int d = 0; d < 4; ++d) {
            wx[d] = basis_phi(tx - (bx + d));
            wy[d] = basis_phi(ty - (by + d));
            wz[d] = basis_phi(tz - (bz + d));
            dwx[d] = basis_phi_deriv(tx - (bx + d)) * inv_h;
            dwy[d] = basis_phi_deriv(ty - (by + d)) * inv_h;
            dwz[d] = basis_phi_deriv(tz - (bz + d)) * inv_h;
        }
        double gx = 0.0, gy = 0.0, gz = 0.0;
        for (int a = 0; a < 4; ++a)
            for (int b = 0; b < 4; ++b)
                for (int cc = 0; cc < 4; ++cc) {
                    const double u = L0->potential[IDX(L0, bx + a, by + b, bz + cc)];
                    gx += dwx[a] * wy[b] * wz[cc] * u;
                    gy += wx[a] * dwy[b] * wz[cc] * u;
                    gz += wx[a] * wy[b] * dwz[cc] * u;
                }
        const double s = kc * q[p];
        sf[3 * p] -= gx * s;
        sf[3 * p + 1] -= gy * s;
        sf[3 * p + 2] -= gz * s;
    }
}

/* ---- msm_potential: src/msm.cpp:52-90 (+ add_long_range_forces 16-48) -------- */
static int msm_eval(int64_t n, const double* pos, const double* q, const double* box,
                    const cfg_t* c, double kc, double conv, double* phi, double* phi_short,
                    double* phi_long, double* force, double* energy, double* level_charge,
                    double* level_potential, char* msg, int cap) {
    int rc = validate_cfg(c, msg, cap);
    if (rc) return rc;
    rc = validate_units(kc, conv, msg, cap);
    if (rc) return rc;
    double* sphi = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    double* sf = (double*)malloc(sizeof(double) * 3 * (size_t)(n > 0 ? n : 1));
    double* ul = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    level_t lv[64];
    int built = 0;
    /* msm.cpp:58-61: short_range (its pair errors first), the hierarchy (box errors),
     * then anterpolation (coverage); the pair sum itself runs once no error is left */
    rc = short_range_impl(n, pos, q, c->a, kc, sphi, sf, msg, cap, 1);
    if (rc) goto done;
    if (c->l > 64) { rc = fail(msg, cap, E_CONFIG, "levels_l too large for the oracle"); goto done; }
    rc = build_levels(box, c, lv, 1, msg, cap);
    if (rc) goto done;
    built = 1;
    rc = coverage_scan(n, pos, &lv[0], msg, cap);
    if (rc) goto done;
    rc = orc_short_range(n, pos, q, c->a, kc, sphi, sf, msg, cap);
    if (rc) goto done;
    rc = anterpolate(n, pos, q, &lv[0], msg, cap);
    if (rc) goto done;
    for (int k = 0; k + 1 < c->l; ++k) {
        rc = restrict_charges(&lv[k], &lv[k + 1], msg, cap);
        if (rc) goto done;
        lattice_cutoff(&lv[k], c);
    }
    top_level(&lv[c->l - 1], c);
    for (int k = c->l - 2; k >= 0; --k) {
        rc = prolongate(&lv[k + 1], &lv[k], msg, cap);
        if (rc) goto done;
    }
    rc = interpolate(n, pos, &lv[0], ul, msg, cap);
    if (rc) goto done;
    {
        const double self = smoothing_gamma(0.0) / c->a; /* msm.cpp:72-73 */
        for (int64_t i = 0; i < n; ++i) ul[i] -= q[i] * self;
        add_long_range_forces(n, pos, q, &lv[0], kc, sf);
        double e = 0.0;
        for (int64_t i = 0; i < n; ++i) {
            const double ph = sphi[i] + ul[i];
            if (phi) phi[i] = ph;
            e += 0.5 * q[i] * ph;
        }
        if (energy) *energy = e * kc;
        if (phi_short) memcpy(phi_short, sphi, sizeof(double) * (size_t)n);
        if (phi_long) memcpy(phi_long, ul, sizeof(double) * (size_t)n);
        if (force) memcpy(force, sf, sizeof(double) * 3 * (size_t)n);
        if (level_charge || level_potential) {
            size_t off = 0;
            for (int k = 0; k < c->l; ++k) {
                if (level_charge) memcpy(level_charge + off, lv[k].charge, lv[k].size * 8);
                if (level_potential) memcpy(level_potential + off, lv[k].potential, lv[k].size * 8);
                off += lv[k].size;
            }
        }
    }
    rc = ok(msg, cap);
done:
    if (built) free_levels(lv, c->l);
    free(sphi);
    free(sf);
    free(ul);
    return rc;
}

int orc_msm_potential(int64_t n, const double* pos, const double* q, const double* box,
                      double a, double h, int levels, int p, int m, double kc, double conv,
                      double* phi, double* phi_short, double* phi_long, double* force,
                      double* energy, double* level_charge, double* level_potential,
                      char* msg, int cap) {
    cfg_t c = {a, h, levels, p, m};
    return msm_eval(n, pos, q, box, &c, kc, conv, phi, phi_short, phi_long, force, energy,
                    level_charge, level_potential, msg, cap);
}

/* individual phases on caller lattices (mirror of oracle/ref_shim.cpp) */
#define WITH_LEVELS(BOX, A, H, L)                     \
    cfg_t c = {A, H, L, 3, 2};                        \
    if (L < 1 || L > 64) return fail(msg, cap, E_CONFIG, "bad levels"); \
    level_t lv[64];                                   \
    int rc = build_levels(BOX, &c, lv, 1, msg, cap);  \
    if (rc) return rc;

int orc_anterpolate(int64_t n, const double* pos, const double* q, const double* box, double a,
                    double h, int levels, double* q0_out, char* msg, int cap) {
    WITH_LEVELS(box, a, h, levels)
    rc = anterpolate(n, pos, q, &lv[0], msg, cap);
    if (!rc) memcpy(q0_out, lv[0].charge, lv[0].size * 8);
    free_levels(lv, levels);
    return rc ? rc : ok(msg, cap);
}

int orc_restrict(const double* box, double a, double h, int levels, int k,
                 const double* fine_charge, double* coarse_out, char* msg, int cap) {
    WITH_LEVELS(box, a, h, levels)
    memcpy(lv[k].charge, fine_charge, lv[k].size * 8);
    rc = restrict_charges(&lv[k], &lv[k + 1], msg, cap);
    if (!rc) memcpy(coarse_out, lv[k + 1].charge, lv[k + 1].size * 8);
    free_levels(lv, levels);
    return rc ? rc : ok(msg, cap);
}

int orc_lattice_cutoff(const double* box, double a, double h, int levels, int k,
                       const double* charge, double* pot_out, char* msg, int cap) {
    WITH_LEVELS(box, a, h, levels)
    memcpy(lv[k].charge, charge, lv[k].size * 8);
    lattice_cutoff(&lv[k], &c);
    memcpy(pot_out, lv[k].potential, lv[k].size * 8);
    free_levels(lv, levels);
    return ok(msg, cap);
}

int orc_top_level(const double* box, double a, double h, int levels, const double* charge,
                  double* pot_out, char* msg, int cap) {
    WITH_LEVELS(box, a, h, levels)
    level_t* T = &lv[levels - 1];
    memcpy(T->charge, charge, T->size * 8);
    top_level(T, &c);
    memcpy(pot_out, T->potential, T->size * 8);
    free_levels(lv, levels);
    return ok(msg, cap);
}

int orc_prolongate(const double* box, double a, double h, int levels, int k,
                   const double* coarse_pot, double* fine_pot, char* msg, int cap) {
    WITH_LEVELS(box, a, h, levels)
    memcpy(lv[k + 1].potential, coarse_pot, lv[k + 1].size * 8);
    memcpy(lv[k].potential, fine_pot, lv[k].size * 8);
    rc = prolongate(&lv[k + 1], &lv[k], msg, cap);
    if (!rc) memcpy(fine_pot, lv[k].potential, lv[k].size * 8);
    free_levels(lv, levels);
    return rc ? rc : ok(msg, cap);
}

int orc_interpolate(int64_t n, const double* pos, const double* box, double a, double h,
                    int levels, const double* pot0, double* u_out, char* msg, int cap) {
    WITH_LEVELS(box, a, h, levels)
    memcpy(lv[0].potential, pot0, lv[0].size * 8);
    rc = interpolate(n, pos, &lv[0], u_out, msg, cap);
    free_levels(lv, levels);
    return rc ? rc : ok(msg, cap);
}

/* The long-range half of msm_potential (src/msm.cpp:69-78) from a given level-0
 * potential: u_long = interpolate(pot0) - q gamma(0)/a (msm.cpp:72-73) and the
 * long-range forces F = -k_C q grad (add_long_range_forces, msm.cpp:16-48, applied
 * to zero forces).  Lets a test check the GPU's production interpolation/force
 * kernel on the GPU's own level-0 potential. */
int orc_long_range(int64_t n, const double* pos, const double* q, const double* box, double a, double h,
                   int levels, double kc, const double* pot0, double* u_out, double* f_out, char* msg, int cap) {
    WITH_LEVELS(box, a, h, levels)
    memcpy(lv[0].potential, pot0, lv[0].size * 8);
    rc = interpolate(n, pos, &lv[0], u_out, msg, cap);
    if (!rc) {
        const double self = smoothing_gamma(0.0) / a;
        for (int64_t i = 0; i < n; ++i) u_out[i] -= q[i] * self;
        memset(f_out, 0, sizeof(double) * 3 * (size_t)n);
        add_long_range_forces(n, pos, q, &lv[0], kc, f_out);
    }
    free_levels(lv, levels);
    return rc ? rc : ok(msg, cap);
}

/* ---- propagate: src/integrate.cpp:7-36 --------------------------------------- */
/* ---- pair-only fields: src/electrostatics.cpp:10-132, src/force_field.cpp:45-68 ----
 * direct_coulomb, simple_cutoff, wolf_summation and PairRepulsionOverlay, restated
 * with the reference's own i<j double loops (same operation order, so bitwise equal;
 * O(N^2): these are the checkers for the GPU fields at test sizes).
 * kind: 1 cutoff, 2 wolf, 3 direct. */
enum { FK_MSM = 0, FK_CUTOFF = 1, FK_WOLF = 2, FK_DIRECT = 3 };

typedef struct {
    int kind;            /* FK_* */
    cfg_t msm;           /* FK_MSM */
    double cutoff;       /* CutoffParams::cutoff */
    int has_alpha;       /* CutoffParams::wolf_alpha engaged */
    double alpha;
    double rep_eps, rep_sigma; /* PairRepulsionOverlay (rep_eps > 0 = on) */
} field_t;

static int pair_field_eval(const field_t* F, int64_t n, const double* pos, const double* q, double kc,
                           double conv, double* phi, double* force, double* energy, char* msg, int cap) {
    int rc = validate_units(kc, conv, msg, cap); /* units.validate(), electrostatics.cpp:44,68,93 */
    if (rc) return rc;
    if (F->kind != FK_DIRECT) { /* CutoffParams::validate, electrostatics.cpp:38-42 */
        if (!(F->cutoff > 0.0)) return fail(msg, cap, E_CONFIG, "cutoff must be > 0");
        if (F->kind == FK_WOLF && !F->has_alpha) return fail(msg, cap, E_CONFIG, "wolf_alpha is required");
        if (F->has_alpha && !(F->alpha >= 0.0)) return fail(msg, cap, E_CONFIG, "wolf_alpha must be >= 0");
    }
    const size_t N = (size_t)(n > 0 ? n : 1);
    double* ph = (double*)calloc(N, sizeof(double));
    double* fo = (double*)calloc(3 * N, sizeof(double));
    const double a = F->cutoff, a2 = a * a;
    const double k2sp = 1.1283791670955126; /* 2/sqrt(pi), electrostatics.cpp:12 */
    double e_shift = 0, f_shift = 0, self_pc = 0, alpha = F->alpha;
    if (F->kind == FK_WOLF) { /* electrostatics.cpp:96-102 */
        const double erfc_aa = erfc(alpha * a);
        e_shift = erfc_aa / a;
        f_shift = erfc_aa / (a * a) + k2sp * alpha * exp(-alpha * alpha * a * a) / a;
        self_pc = -(e_shift + k2sp * alpha);
    }
    for (int64_t i = 0; i < n && rc == OK; ++i)
        for (int64_t j = i + 1; j < n; ++j) {
            const double dx = pos[3 * i] - pos[3 * j], dy = pos[3 * i + 1] - pos[3 * j + 1],
                         dz = pos[3 * i + 2] - pos[3 * j + 2];
            const double r2 = dx * dx + dy * dy + dz * dz;
            if (r2 == 0.0) { /* check_distinct, electrostatics.cpp:14-18 */
                rc = fail(msg, cap, E_COINCIDENT, "particles %lld and %lld coincide", (long long)i, (long long)j);
                break;
            }
            double pair, s;
            if (F->kind == FK_DIRECT || F->kind == FK_CUTOFF) { /* :52-61, :76-86 */
                if (F->kind == FK_CUTOFF && r2 >= a2) continue;
                const double r = sqrt(r2);
                const double inv_r = 1.0 / r;
                pair = inv_r;
                s = kc * q[i] * q[j] * inv_r * inv_r * inv_r;
            } else { /* :108-118 */
                if (r2 >= a2) continue;
                const double r = sqrt(r2);
                const double erfc_ar = erfc(alpha * r);
                const double gauss = k2sp * alpha * exp(-alpha * alpha * r2);
                pair = erfc_ar / r - e_shift + f_shift * (r - a);
                const double fmag = erfc_ar / r2 + gauss / r - f_shift;
                s = kc * q[i] * q[j] * fmag / r;
            }
            ph[i] += q[j] * pair;
            ph[j] += q[i] * pair;
            const double fx = dx * s, fy = dy * s, fz = dz * s;
            fo[3 * i] += fx;
            fo[3 * i + 1] += fy;
            fo[3 * i + 2] += fz;
            fo[3 * j] -= fx;
            fo[3 * j + 1] -= fy;
            fo[3 * j + 2] -= fz;
        }
    if (rc == OK && F->kind == FK_WOLF) /* :123-124 */
        for (int64_t i = 0; i < n; ++i) ph[i] += q[i] * self_pc;
    double e = 0.0; /* finish_total, :27-33 */
    for (int64_t i = 0; i < n; ++i) e += 0.5 * q[i] * ph[i];
    e = e * kc;
    if (rc == OK && F->rep_eps > 0.0) { /* PairRepulsionOverlay::evaluate, force_field.cpp:45-68 */
        const double s6 = pow(F->rep_sigma, 6.0);
        const double s12 = s6 * s6;
        double er = 0.0;
        for (int64_t i = 0; i < n && rc == OK; ++i)
            for (int64_t j = i + 1; j < n; ++j) {
                const double dx = pos[3 * i] - pos[3 * j], dy = pos[3 * i + 1] - pos[3 * j + 1],
                             dz = pos[3 * i + 2] - pos[3 * j + 2];
                const double r2 = dx * dx + dy * dy + dz * dz;
                if (r2 == 0.0) {
                    rc = fail(msg, cap, E_COINCIDENT, "particles %lld and %lld coincide", (long long)i, (long long)j);
                    break;
                }
                const double inv_r2 = 1.0 / r2;
                const double inv_r12 = inv_r2 * inv_r2 * inv_r2 * inv_r2 * inv_r2 * inv_r2;
                er += F->rep_eps * s12 * inv_r12;
                const double sc = 12.0 * F->rep_eps * s12 * inv_r12 * inv_r2;
                const double fx = dx * sc, fy = dy * sc, fz = dz * sc;
                fo[3 * i] += fx;
                fo[3 * i + 1] += fy;
                fo[3 * i + 2] += fz;
                fo[3 * j] -= fx;
                fo[3 * j + 1] -= fy;
                fo[3 * j + 2] -= fz;
            }
        e += er;
    }
    if (rc == OK) {
        if (phi) memcpy(phi, ph, sizeof(double) * (size_t)n);
        if (force) memcpy(force, fo, sizeof(double) * 3 * (size_t)n);
        if (energy) *energy = e;
    }
    free(ph);
    free(fo);
    return rc == OK ? ok(msg, cap) : rc;
}

/* fspec = {kind, a, h, levels, has_alpha, alpha, rep_eps, rep_sigma}: a = MSM cutoff_a or
 * CutoffParams::cutoff; h/levels for MSM only. */
static field_t field_of(const double* fs) {
    field_t F;
    memset(&F, 0, sizeof F);
    F.kind = (int)fs[0];
    F.msm = (cfg_t){fs[1], fs[2], (int)fs[3], 3, 2};
    F.cutoff = fs[1];
    F.has_alpha = fs[4] != 0.0;
    F.alpha = fs[5];
    F.rep_eps = fs[6];
    F.rep_sigma = fs[7];
    return F;
}

static int msm_eval(int64_t n, const double* pos, const double* q, const double* box,
                    const cfg_t* c, double kc, double conv, double* phi, double* phi_short,
                    double* phi_long, double* force, double* energy, double* level_charge,
                    double* level_potential, char* msg, int cap);

static int field_eval(const field_t* F, int64_t n, const double* pos, const double* q, const double* box,
                      double kc, double conv, double* phi, double* force, double* energy, char* msg, int cap) {
    if (F->kind == FK_MSM && !(F->rep_eps > 0.0))
        return msm_eval(n, pos, q, box, &F->msm, kc, conv, phi, NULL, NULL, force, energy, NULL, NULL, msg, cap);
    if (F->kind == FK_MSM) return fail(msg, cap, E_OTHER, "oracle: repulsion overlay on MSM not restated");
    return pair_field_eval(F, n, pos, q, kc, conv, phi, force, energy, msg, cap);
}

int orc_field_evaluate(const double* fspec, int64_t n, const double* pos, const double* q, const double* box,
                       double kc, double conv, double* phi, double* force, double* energy, char* msg, int cap) {
    const field_t F = field_of(fspec);
    return field_eval(&F, n, pos, q, box, kc, conv, phi, force, energy, msg, cap);
}

typedef struct {
    field_t field;
    double dt;
    int steps;
} spec_t;

static int propagate(int64_t n, double* pos, double* vel, const double* q, const double* mass,
                     const double* box, const spec_t* sp, double kc, double conv,
                     int* steps_done, char* msg, int cap) {
    if (steps_done) *steps_done = 0;
    if (!(sp->dt > 0.0)) return fail(msg, cap, E_CONFIG, "dt must be > 0");
    if (sp->steps < 1) return fail(msg, cap, E_CONFIG, "steps_per_slice must be >= 1");
    int rc = validate_units(kc, conv, msg, cap);
    if (rc) return rc;
    double* f = (double*)malloc(sizeof(double) * 3 * (size_t)(n > 0 ? n : 1));
    const double dt = sp->dt;
    rc = field_eval(&sp->field, n, pos, q, box, kc, conv, NULL, f, NULL, msg, cap);
    for (int step = 0; rc == OK && step < sp->steps; ++step) {
        for (int64_t i = 0; i < n; ++i) {
            const double cc = 0.5 * dt * conv / mass[i];
            for (int ax = 0; ax < 3; ++ax) vel[3 * i + ax] += f[3 * i + ax] * cc;
            for (int ax = 0; ax < 3; ++ax) pos[3 * i + ax] += vel[3 * i + ax] * dt;
        }
        rc = field_eval(&sp->field, n, pos, q, box, kc, conv, NULL, f, NULL, msg, cap);
        if (rc) break;
        for (int64_t i = 0; i < n; ++i) {
            const double cc = 0.5 * dt * conv / mass[i];
            for (int ax = 0; ax < 3; ++ax) vel[3 * i + ax] += f[3 * i + ax] * cc;
        }
        if (steps_done) *steps_done = step + 1;
    }
    free(f);
    return rc;
}

int orc_propagate(int64_t n, double* pos, double* vel, const double* q, const double* mass,
                  const double* box, double a, double h, int levels, double kc, double conv,
                  double dt, int steps, int* steps_done, char* msg, int cap) {
    spec_t sp;
    memset(&sp, 0, sizeof sp);
    sp.field.msm = (cfg_t){a, h, levels, 3, 2};
    sp.dt = dt;
    sp.steps = steps;
    /* propagate works on a copy: on error the caller's state is untouched */
    double* p2 = (double*)malloc(sizeof(double) * 3 * (size_t)(n > 0 ? n : 1));
    double* v2 = (double*)malloc(sizeof(double) * 3 * (size_t)(n > 0 ? n : 1));
    memcpy(p2, pos, sizeof(double) * 3 * (size_t)n);
    memcpy(v2, vel, sizeof(double) * 3 * (size_t)n);
    int rc = propagate(n, p2, v2, q, mass, box, &sp, kc, conv, steps_done, msg, cap);
    if (rc == OK) {
        memcpy(pos, p2, sizeof(double) * 3 * (size_t)n);
        memcpy(vel, v2, sizeof(double) * 3 * (size_t)n);
        ok(msg, cap);
    }
    free(p2);
    free(v2);
    return rc;
}

/* propagate with any field (fspec as orc_field_evaluate) */
int orc_field_propagate(const double* fspec, int64_t n, double* pos, double* vel, const double* q,
                        const double* mass, const double* box, double kc, double conv, double dt, int steps,
                        int* steps_done, char* msg, int cap) {
    spec_t sp;
    memset(&sp, 0, sizeof sp);
    sp.field = field_of(fspec);
    sp.dt = dt;
    sp.steps = steps;
    double* p2 = (double*)malloc(sizeof(double) * 3 * (size_t)(n > 0 ? n : 1));
    double* v2 = (double*)malloc(sizeof(double) * 3 * (size_t)(n > 0 ? n : 1));
    memcpy(p2, pos, sizeof(double) * 3 * (size_t)n);
    memcpy(v2, vel, sizeof(double) * 3 * (size_t)n);
    int rc = propagate(n, p2, v2, q, mass, box, &sp, kc, conv, steps_done, msg, cap);
    if (rc == OK) {
        memcpy(pos, p2, sizeof(double) * 3 * (size_t)n);
        memcpy(vel, v2, sizeof(double) * 3 * (size_t)n);
        ok(msg, cap);
    }
    free(p2);
    free(v2);
    return rc;
}

/* ---- parareal: src/parareal.cpp:43-239 --------------------------------------- */
typedef struct {
    double* pos;
    double* vel;
} state_t; /* charges, masses and box never change along a trajectory */

typedef struct {
    double* dpos;
    double* dvel;
    double rms_pos;
    double max_pos;
} delta_t;

typedef struct {
    int64_t n;
    const double *q, *mass, *box;
    spec_t fine, coarse;
    double kc, conv;
    int window, max_iter;
    double tol;
    int has_skip;
    double skip;
    int short_circuit;
    int64_t g_evals, f_evals, f_skipped;
} pr_t;

static state_t st_new(int64_t n) {
    state_t s = {(double*)calloc(3 * (size_t)n, 8), (double*)calloc(3 * (size_t)n, 8)};
    return s;
}
static state_t st_copy(int64_t n, state_t a) {
    state_t s = st_new(n);
    memcpy(s.pos, a.pos, 24 * (size_t)n);
    memcpy(s.vel, a.vel, 24 * (size_t)n);
    return s;
}
static void st_free(state_t s) {
    free(s.pos);
    free(s.vel);
}
static delta_t dl_zero(int64_t n) {
    delta_t d = {(double*)calloc(3 * (size_t)n, 8), (double*)calloc(3 * (size_t)n, 8), 0.0, 0.0};
    return d;
}
static delta_t dl_copy(int64_t n, delta_t a) {
    delta_t d = dl_zero(n);
    memcpy(d.dpos, a.dpos, 24 * (size_t)n);
    memcpy(d.dvel, a.dvel, 24 * (size_t)n);
    d.rms_pos = a.rms_pos;
    d.max_pos = a.max_pos;
    return d;
}
static void dl_free(delta_t d) {
    free(d.dpos);
    free(d.dvel);
}

static delta_t state_sub(int64_t n, state_t a, state_t b) { /* parareal.cpp:58-73 */
    delta_t d = dl_zero(n);
    double sum2 = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        for (int ax = 0; ax < 3; ++ax) {
            d.dpos[3 * i + ax] = a.pos[3 * i + ax] - b.pos[3 * i + ax];
            d.dvel[3 * i + ax] = a.vel[3 * i + ax] - b.vel[3 * i + ax];
        }
        const double p2 = d.dpos[3 * i] * d.dpos[3 * i] + d.dpos[3 * i + 1] * d.dpos[3 * i + 1] +
                          d.dpos[3 * i + 2] * d.dpos[3 * i + 2];
        sum2 += p2;
        const double s = sqrt(p2);
        if (d.max_pos < s) d.max_pos = s; /* std::max(max_pos, sqrt) */
    }
    d.rms_pos = sqrt(sum2 / (3.0 * (double)n));
    return d;
}

static state_t state_add(int64_t n, state_t base, delta_t d) { /* parareal.cpp:75-82 */
    state_t o = st_copy(n, base);
    for (int64_t i = 0; i < 3 * n; ++i) {
        o.pos[i] += d.dpos[i];
        o.vel[i] += d.dvel[i];
    }
    return o;
}

static double rms_pos_change(int64_t n, state_t a, state_t b) { /* parareal.cpp:86-90 */
    double sum2 = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        const double dx = a.pos[3 * i] - b.pos[3 * i];
        const double dy = a.pos[3 * i + 1] - b.pos[3 * i + 1];
        const double dz = a.pos[3 * i + 2] - b.pos[3 * i + 2];
        sum2 += dx * dx + dy * dy + dz * dz;
    }
    return sqrt(sum2 / (3.0 * (double)n));
}

static int prop_state(pr_t* P, const spec_t* sp, state_t in, state_t* out, char* msg, int cap) {
    *out = st_copy(P->n, in);
    int rc = propagate(P->n, out->pos, out->vel, P->q, P->mass, P->box, sp, P->kc, P->conv, NULL,
                       msg, cap);
    if (rc) {
        st_free(*out);
        out->pos = out->vel = NULL;
    }
    return rc;
}

typedef struct {
    int points, rows;
    state_t** lambda; /* [rows][points+1] */
    state_t** g;      /* [rows][points+1], slot 0 unused */
    delta_t** delta;  /* [rows][points+1], slot 0 unused */
} window_t;

static void win_free(int64_t n, window_t* w) {
    (void)n;
    for (int r = 0; r < w->rows; ++r) {
        for (int i = 0; i <= w->points; ++i) {
            if (w->lambda[r][i].pos) st_free(w->lambda[r][i]);
            if (w->g[r][i].pos) st_free(w->g[r][i]);
            if (w->delta[r][i].dpos) dl_free(w->delta[r][i]);
        }
        free(w->lambda[r]);
        free(w->g[r]);
        free(w->delta[r]);
    }
    free(w->lambda);
    free(w->g);
    free(w->delta);
}

static void win_add_row(window_t* w) {
    w->lambda = (state_t**)realloc(w->lambda, sizeof(void*) * (size_t)(w->rows + 1));
    w->g = (state_t**)realloc(w->g, sizeof(void*) * (size_t)(w->rows + 1));
    w->delta = (delta_t**)realloc(w->delta, sizeof(void*) * (size_t)(w->rows + 1));
    w->lambda[w->rows] = (state_t*)calloc((size_t)w->points + 1, sizeof(state_t));
    w->g[w->rows] = (state_t*)calloc((size_t)w->points + 1, sizeof(state_t));
    w->delta[w->rows] = (delta_t*)calloc((size_t)w->points + 1, sizeof(delta_t));
    w->rows++;
}

static int validate_pr(const pr_t* P, char* msg, int cap) { /* parareal.cpp:43-56 */
    if (P->window < 1) return fail(msg, cap, E_CONFIG, "window_points must be >= 1");
    if (P->max_iter < 1) return fail(msg, cap, E_CONFIG, "max_iter must be >= 1");
    if (!(P->tol > 0.0)) return fail(msg, cap, E_CONFIG, "tol must be > 0");
    const spec_t* sp[2] = {&P->fine, &P->coarse}; /* PropagatorSpec::validate integrate.cpp:7-11 */
    for (int s = 0; s < 2; ++s) {
        if (!(sp[s]->dt > 0.0)) return fail(msg, cap, E_CONFIG, "dt must be > 0");
        if (sp[s]->steps < 1) return fail(msg, cap, E_CONFIG, "steps_per_slice must be >= 1");
    }
    int rc = validate_units(P->kc, P->conv, msg, cap);
    if (rc) return rc;
    const double sf = P->fine.dt * P->fine.steps, sg = P->coarse.dt * P->coarse.steps;
    const double mx = fabs(sf) > fabs(sg) ? fabs(sf) : fabs(sg);
    if (fabs(sf - sg) > 1e-12 * mx)
        return fail(msg, cap, E_CONFIG, "fine and coarse propagators span different slice lengths");
    if (P->has_skip && !(P->skip >= 0.0)) return fail(msg, cap, E_CONFIG, "skip threshold must be >= 0");
    return OK;
}

static int pr_init(pr_t* P, state_t v, int t, window_t* w, char* msg, int cap) { /* :94-115 */
    memset(w, 0, sizeof(*w));
    w->points = t;
    win_add_row(w);
    w->lambda[0][0] = st_copy(P->n, v);
    for (int n = 1; n <= t; ++n) {
        int rc = prop_state(P, &P->coarse, w->lambda[0][n - 1], &w->lambda[0][n], msg, cap);
        if (rc) return rc;
        P->g_evals++;
        w->g[0][n] = st_copy(P->n, w->lambda[0][n]);
    }
    return OK;
}

static int pr_iterate(pr_t* P, window_t* w, char* msg, int cap) { /* :117-180 */
    const int t = w->points;
    const int prev = w->rows - 1;
    int* skip = (int*)calloc((size_t)t + 1, sizeof(int));
    if (P->has_skip && w->rows >= 2) { /* metastable_skip_indices :117-127 */
        for (int n = 1; n <= t; ++n)
            if (rms_pos_change(P->n, w->lambda[w->rows - 1][n - 1], w->lambda[w->rows - 2][n - 1]) < P->skip)
                skip[n] = 1;
    }
    delta_t* deltas = (delta_t*)calloc((size_t)t + 1, sizeof(delta_t));
    int rc = OK;
    for (int n = 1; n <= t; ++n)
        if (skip[n]) {
            deltas[n] = dl_copy(P->n, w->delta[prev][n]);
            P->f_skipped++;
        }
    for (int n = 1; n <= t && rc == OK; ++n) { /* the executor's work list, sequentially */
        if (skip[n]) continue;
        state_t f;
        rc = prop_state(P, &P->fine, w->lambda[prev][n - 1], &f, msg, cap);
        if (rc) break;
        deltas[n] = state_sub(P->n, f, w->g[prev][n]);
        st_free(f);
        P->f_evals++;
    }
    if (rc == OK) {
        win_add_row(w);
        const int r = w->rows - 1;
        w->lambda[r][0] = st_copy(P->n, w->lambda[0][0]);
        for (int n = 1; n <= t && rc == OK; ++n) {
            state_t g;
            if (prev == 0 && n == 1) {
                g = st_copy(P->n, w->g[prev][1]);
            } else {
                rc = prop_state(P, &P->coarse, w->lambda[r][n - 1], &g, msg, cap);
                if (rc) break;
                P->g_evals++;
            }
            w->lambda[r][n] = state_add(P->n, g, deltas[n]);
            w->g[r][n] = g;
        }
        for (int n = 1; n <= t; ++n) w->delta[r][n] = deltas[n];
    } else {
        for (int n = 1; n <= t; ++n)
            if (deltas[n].dpos) dl_free(deltas[n]);
    }
    free(deltas);
    free(skip);
    return rc;
}

static void pr_setup(pr_t* P, int64_t n, const double* q, const double* mass, const double* box,
                     double fa, double fh, int fl, double fdt, int fsteps, double ga, double gh,
                     int gl, double gdt, int gsteps, double kc, double conv) {
    memset(P, 0, sizeof(*P));
    P->n = n;
    P->q = q;
    P->mass = mass;
    P->box = box;
    memset(&P->fine, 0, sizeof P->fine);
    memset(&P->coarse, 0, sizeof P->coarse);
    P->fine.field.msm = (cfg_t){fa, fh, fl, 3, 2};
    P->fine.dt = fdt;
    P->fine.steps = fsteps;
    P->coarse.field.msm = (cfg_t){ga, gh, gl, 3, 2};
    P->coarse.dt = gdt;
    P->coarse.steps = gsteps;
    P->kc = kc;
    P->conv = conv;
}

int orc_parareal_window(int64_t n, const double* pos, const double* vel, const double* q,
                        const double* mass, const double* box, double fa, double fh, int fl,
                        double fdt, int fsteps, double ga, double gh, int gl, double gdt,
                        int gsteps, double kc, double conv, int t_points, int k_iters,
                        int threads, double* row_pos, double* row_vel, double* delta_rms,
                        int64_t* counts, char* msg, int cap) {
    (void)threads;
    pr_t P;
    pr_setup(&P, n, q, mass, box, fa, fh, fl, fdt, fsteps, ga, gh, gl, gdt, gsteps, kc, conv);
    P.window = t_points;
    P.max_iter = k_iters;
    P.tol = 1e300;
    int rc = validate_pr(&P, msg, cap);
    if (rc) return rc;
    state_t v = {(double*)pos, (double*)vel};
    window_t w;
    rc = pr_init(&P, v, t_points, &w, msg, cap);
    for (int k = 0; rc == OK && k < k_iters; ++k) rc = pr_iterate(&P, &w, msg, cap);
    if (rc == OK) {
        const int r = w.rows - 1;
        for (int i = 0; i <= t_points; ++i) {
            if (row_pos) memcpy(row_pos + 3 * n * i, w.lambda[r][i].pos, 24 * (size_t)n);
            if (row_vel) memcpy(row_vel + 3 * n * i, w.lambda[r][i].vel, 24 * (size_t)n);
        }
        if (delta_rms)
            for (int i = 1; i <= t_points; ++i) delta_rms[i] = w.delta[r][i].rms_pos;
        if (counts) {
            counts[0] = P.g_evals;
            counts[1] = P.f_evals;
            counts[2] = P.f_skipped;
        }
        ok(msg, cap);
    }
    win_free(n, &w);
    return rc;
}

/* parareal window with any fine/coarse fields (fspec as orc_field_evaluate) */
int orc_field_parareal_window(int64_t n, const double* pos, const double* vel, const double* q,
                              const double* mass, const double* box, const double* fine_spec, double fdt,
                              int fsteps, const double* coarse_spec, double gdt, int gsteps, double kc,
                              double conv, int t_points, int k_iters, double* row_pos, double* row_vel,
                              double* delta_rms, int64_t* counts, char* msg, int cap) {
    pr_t P;
    pr_setup(&P, n, q, mass, box, 0, 0, 0, fdt, fsteps, 0, 0, 0, gdt, gsteps, kc, conv);
    P.fine.field = field_of(fine_spec);
    P.coarse.field = field_of(coarse_spec);
    P.window = t_points;
    P.max_iter = k_iters;
    P.tol = 1e300;
    int rc = validate_pr(&P, msg, cap);
    if (rc) return rc;
    state_t v = {(double*)pos, (double*)vel};
    window_t w;
    rc = pr_init(&P, v, t_points, &w, msg, cap);
    for (int k = 0; rc == OK && k < k_iters; ++k) rc = pr_iterate(&P, &w, msg, cap);
    if (rc == OK) {
        const int r = w.rows - 1;
        for (int i = 0; i <= t_points; ++i) {
            if (row_pos) memcpy(row_pos + 3 * n * i, w.lambda[r][i].pos, 24 * (size_t)n);
            if (row_vel) memcpy(row_vel + 3 * n * i, w.lambda[r][i].vel, 24 * (size_t)n);
        }
        if (delta_rms)
            for (int i = 1; i <= t_points; ++i) delta_rms[i] = w.delta[r][i].rms_pos;
        if (counts) {
            counts[0] = P.g_evals;
            counts[1] = P.f_evals;
            counts[2] = P.f_skipped;
        }
        ok(msg, cap);
    }
    win_free(n, &w);
    return rc;
}

int orc_parareal_run(int64_t n, const double* pos, const double* vel, const double* q,
                     const double* mass, const double* box, double fa, double fh, int fl,
                     double fdt, int fsteps, double ga, double gh, int gl, double gdt,
                     int gsteps, double kc, double conv, int window, int max_iter, double tol,
                     int short_circuit, double skip_threshold, int total_points, int threads,
                     double* traj_pos, double* traj_vel, int64_t* counts, char* msg, int cap) {
    (void)threads;
    pr_t P;
    pr_setup(&P, n, q, mass, box, fa, fh, fl, fdt, fsteps, ga, gh, gl, gdt, gsteps, kc, conv);
    P.window = window;
    P.max_iter = max_iter;
    P.tol = tol;
    P.short_circuit = short_circuit;
    P.has_skip = skip_threshold >= 0.0;
    P.skip = skip_threshold;
    int rc = validate_pr(&P, msg, cap);
    if (rc) return rc;
    if (total_points < 1) return fail(msg, cap, E_CONFIG, "total_points must be >= 1");
    state_t current = st_copy(n, (state_t){(double*)pos, (double*)vel});
    int remaining = total_points, window_idx = 0, out_idx = 0;
    while (remaining > 0 && rc == OK) { /* parareal.cpp:193-235 */
        ++window_idx;
        const int t = window < remaining ? window : remaining;
        window_t w;
        rc = pr_init(&P, current, t, &w, msg, cap);
        int prefix = 0;
        for (int k = 0; rc == OK && k < max_iter; ++k) {
            rc = pr_iterate(&P, &w, msg, cap);
            if (rc) break;
            prefix = 0;
            int unbroken = 1;
            for (int m = 1; m <= t; ++m) {
                const double change = rms_pos_change(n, w.lambda[w.rows - 1][m], w.lambda[w.rows - 2][m]);
                const int okc = change <= tol;
                if (unbroken && okc)
                    prefix = m;
                else
                    unbroken = 0;
            }
            if (short_circuit && prefix == t) break;
        }
        if (rc == OK && prefix == 0) {
            rc = fail(msg, cap, E_NONCONV, "window %d did not converge within max_iter=%d",
                      window_idx, max_iter);
        }
        if (rc == OK) {
            const int r = w.rows - 1;
            for (int m = 1; m <= prefix; ++m, ++out_idx) {
                if (traj_pos) memcpy(traj_pos + 3 * n * out_idx, w.lambda[r][m].pos, 24 * (size_t)n);
                if (traj_vel) memcpy(traj_vel + 3 * n * out_idx, w.lambda[r][m].vel, 24 * (size_t)n);
            }
            st_free(current);
            current = st_copy(n, w.lambda[r][prefix]);
            remaining -= prefix;
        }
        win_free(n, &w);
    }
    if (counts) {
        counts[0] = P.g_evals;
        counts[1] = P.f_evals;
        counts[2] = P.f_skipped;
        counts[3] = window_idx;
        counts[4] = rc == OK ? 1 : 0;
    }
    st_free(current);
    return rc == OK ? ok(msg, cap) : rc;
}

int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
