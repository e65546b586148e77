/*
 * Seeded synthetic inputs for the BASELINE.json configurations (SURVEY.md
 * Appendix B).  Not on the hot path: bench.py and tests/ use it to build
 * ParticleSystems in-process (16.7M atoms do not fit through XYZ files, and
 * water H atoms may sit outside the box, which the reference loader rejects,
 * src/system.cpp:26-31).
 *
 * fx_uniform() is the reference's generate_random_system (src/generate.cpp:
 * 13-93): mt19937_64(seed), next_u01 = (rng() >> 11) * 2^-53, rejection of
 * candidates closer than min_separation to any accepted point, and the three
 * charge schemes.  The min-separation test runs on a cell grid but accepts or
 * rejects exactly the same candidates as the reference's O(N^2) scan, so the
 * output is identical (checked against oracle/_ref in tests/test_fixtures.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- mt19937_64 (the standard 64-bit Mersenne twister) ---------------------- */
typedef struct {
    uint64_t mt[312];
    int idx;
} mt64;

static void mt_seed(mt64* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->idx = 312;
}

static uint64_t mt_next(mt64* r) {
    if (r->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            const uint64_t x = (r->mt[i] & 0xFFFFFFFF80000000ULL) | (r->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
        }
        r->idx = 0;
    }
    uint64_t y = r->mt[r->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

static double next_u01(mt64* r) { return (double)(mt_next(r) >> 11) * 0x1.0p-53; }

static size_t next_below(mt64* r, size_t bound) {
    size_t v = (size_t)(next_u01(r) * (double)bound);
    return v >= bound ? bound - 1 : v;
}

/* ---- cell grid for min-separation rejection --------------------------------- */
typedef struct {
    int nc[3];
    double inv[3];
    int64_t* head; /* per cell, -1 terminated linked list through next[] */
    int64_t* next;
} rgrid;

static int rgrid_init(rgrid* g, const double* box, double sep, int64_t n) {
    for (int ax = 0; ax < 3; ++ax) {
        double edge = sep;
        if (box[ax] / edge > 256.0) edge = box[ax] / 256.0;
        g->nc[ax] = (int)(box[ax] / edge);
        if (g->nc[ax] < 1) g->nc[ax] = 1;
        g->inv[ax] = g->nc[ax] / box[ax];
    }
    const size_t nc = (size_t)g->nc[0] * g->nc[1] * g->nc[2];
    g->head = (int64_t*)malloc(nc * sizeof(int64_t));
    g->next = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    if (!g->head || !g->next) return 1;
    for (size_t i = 0; i < nc; ++i) g->head[i] = -1;
    return 0;
}

static void rgrid_cell(const rgrid* g, const double* p, int* c) {
    for (int ax = 0; ax < 3; ++ax) {
        int v = (int)(p[ax] * g->inv[ax]);
        if (v < 0) v = 0;
        if (v >= g->nc[ax]) v = g->nc[ax] - 1;
        c[ax] = v;
    }
}

/* 1 if p is closer than sep (norm2 < sep2, the reference's test) to an accepted point */
static int rgrid_clash(const rgrid* g, const double* pos, const double* p, double sep2) {
    int c[3];
    rgrid_cell(g, p, c);
    for (int dx = -1; dx <= 1; ++dx)
        for (int dy = -1; dy <= 1; ++dy)
            for (int dz = -1; dz <= 1; ++dz) {
                const int x = c[0] + dx, y = c[1] + dy, z = c[2] + dz;
                if (x < 0 || y < 0 || z < 0 || x >= g->nc[0] || y >= g->nc[1] || z >= g->nc[2]) continue;
                for (int64_t j = g->head[((size_t)x * g->nc[1] + y) * g->nc[2] + z]; j >= 0; j = g->next[j]) {
                    const double ddx = p[0] - pos[3 * j], ddy = p[1] - pos[3 * j + 1], ddz = p[2] - pos[3 * j + 2];
                    if (ddx * ddx + ddy * ddy + ddz * ddz < sep2) return 1;
                }
            }
    return 0;
}

static void rgrid_add(rgrid* g, const double* pos, int64_t j) {
    int c[3];
    rgrid_cell(g, pos + 3 * j, c);
    const size_t cell = ((size_t)c[0] * g->nc[1] + c[1]) * g->nc[2] + c[2];
    g->next[j] = g->head[cell];
    g->head[cell] = j;
}

static void rgrid_free(rgrid* g) {
    free(g->head);
    free(g->next);
}

/* ---- generate_random_system (src/generate.cpp:40-93) -------------------------
 * scheme: 0 AllPlusOne, 1 Alternating, 2 RandomNeutral.  Returns 0, or 1 when the
 * attempt budget (10000*n, generate.cpp:52) is exhausted, 2 on bad arguments. */
int fx_uniform(int64_t n, const double* box, int scheme, double min_sep, uint64_t seed,
               double* pos, double* q) {
    if (n < 1 || min_sep < 0.0 || !(box[0] > 0 && box[1] > 0 && box[2] > 0)) return 2;
    mt64* rng = (mt64*)malloc(sizeof(mt64));
    mt_seed(rng, seed);
    const double sep2 = min_sep * min_sep;
    rgrid g;
    const int use_grid = min_sep > 0.0;
    if (use_grid && rgrid_init(&g, box, min_sep, n)) return 2;
    const unsigned long long budget = 10000ULL * (unsigned long long)n;
    unsigned long long attempts = 0;
    int64_t placed = 0;
    while (placed < n) {
        if (attempts >= budget) {
            if (use_grid) rgrid_free(&g);
            free(rng);
            return 1;
        }
        ++attempts;
        double p[3];
        p[0] = next_u01(rng) * box[0];
        p[1] = next_u01(rng) * box[1];
        p[2] = next_u01(rng) * box[2];
        if (use_grid && rgrid_clash(&g, pos, p, sep2)) continue;
        memcpy(pos + 3 * placed, p, sizeof p);
        if (use_grid) rgrid_add(&g, pos, placed);
        ++placed;
    }
    for (int64_t i = 0; i < n; ++i) q[i] = 1.0;
    if (scheme == 1) {
        for (int64_t i = 0; i < n; ++i) q[i] = (i % 2 == 0) ? 1.0 : -1.0;
    } else if (scheme == 2) {
        const int64_t plus = (n + 1) / 2;
        for (int64_t i = 0; i < n; ++i) q[i] = i < plus ? 1.0 : -1.0;
        for (int64_t i = n - 1; i > 0; --i) {
            const size_t j = next_below(rng, (size_t)i + 1);
            const double t = q[i];
            q[i] = q[j];
            q[j] = t;
        }
    }
    if (use_grid) rgrid_free(&g);
    free(rng);
    return 0;
}

/* ---- charges drawn uniformly from {-1,+1}, then rebalanced to net zero by
 * flipping surplus-sign charges in a seeded random order (config 3). -------- */
int fx_rebalanced_charges(int64_t n, uint64_t seed, double* q) {
    mt64* rng = (mt64*)malloc(sizeof(mt64));
    mt_seed(rng, seed);
    int64_t sum = 0;
    for (int64_t i = 0; i < n; ++i) {
        q[i] = next_u01(rng) < 0.5 ? -1.0 : 1.0;
        sum += q[i] > 0 ? 1 : -1;
    }
    if (sum != 0) {
        int64_t* perm = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
        for (int64_t i = 0; i < n; ++i) perm[i] = i;
        for (int64_t i = n - 1; i > 0; --i) {
            const size_t j = next_below(rng, (size_t)i + 1);
            const int64_t t = perm[i];
            perm[i] = perm[j];
            perm[j] = t;
        }
        const double surplus = sum > 0 ? 1.0 : -1.0;
        for (int64_t k = 0; k < n && sum != 0 && (sum > 1 || sum < -1); ++k) {
            const int64_t i = perm[k];
            if (q[i] == surplus) {
                q[i] = -surplus;
                sum -= 2 * (int64_t)surplus;
            }
        }
        free(perm);
    }
    free(rng);
    return (int)(sum != 0);
}

/* ---- Maxwell-Boltzmann velocities (Box-Muller), centre-of-mass removed ----- */
/* kT in the integrator's native units amu*A^2/fs^2:
 * k_B = 0.0019872041 kcal/(mol K), 1 kcal/mol = energy_to_native (4.184e-4). */
int fx_maxwell_boltzmann(int64_t n, const double* mass, double temperature_k,
                         double energy_to_native, uint64_t seed, double* vel) {
    mt64* rng = (mt64*)malloc(sizeof(mt64));
    mt_seed(rng, seed);
    const double kt = 0.0019872041 * temperature_k * energy_to_native;
    const double two_pi = 6.283185307179586476925286766559;
    double spare = 0.0;
    int have_spare = 0;
    for (int64_t i = 0; i < 3 * n; ++i) {
        double z;
        if (have_spare) {
            z = spare;
            have_spare = 0;
        } else {
            const double u1 = 1.0 - next_u01(rng); /* (0, 1] */
            const double u2 = next_u01(rng);
            const double r = sqrt(-2.0 * log(u1));
            z = r * cos(two_pi * u2);
            spare = r * sin(two_pi * u2);
            have_spare = 1;
        }
        vel[i] = z * sqrt(kt / mass[i / 3]);
    }
    double pm[3] = {0, 0, 0}, mt = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        for (int ax = 0; ax < 3; ++ax) pm[ax] += mass[i] * vel[3 * i + ax];
        mt += mass[i];
    }
    for (int64_t i = 0; i < n; ++i)
        for (int ax = 0; ax < 3; ++ax) vel[3 * i + ax] -= pm[ax] / mt;
    free(rng);
    return 0;
}

/* ---- rigid 3-site water-like molecules (configs 2 and 4) ----------------------
 * Atom order O,H,H per molecule; O uniform in the box (optionally with an O-O
 * minimum separation by the same rejection rule), random orientation; charges
 * O -0.834 / H +0.417, masses 16 / 1 amu, O-H 0.9572 A, H-O-H 104.52 deg. */
static void unit_normal3(mt64* r, double* v) {
    const double two_pi = 6.283185307179586476925286766559;
    for (;;) {
        double z[4];
        for (int k = 0; k < 4; k += 2) {
            const double u1 = 1.0 - next_u01(r), u2 = next_u01(r);
            const double rr = sqrt(-2.0 * log(u1));
            z[k] = rr * cos(two_pi * u2);
            z[k + 1] = rr * sin(two_pi * u2);
        }
        const double nn = sqrt(z[0] * z[0] + z[1] * z[1] + z[2] * z[2]);
        if (nn > 1e-6) {
            v[0] = z[0] / nn;
            v[1] = z[1] / nn;
            v[2] = z[2] / nn;
            return;
        }
    }
}

int fx_water(int64_t n_mol, const double* box, double min_oo, uint64_t seed, double* pos,
             double* q, double* mass) {
    if (n_mol < 1 || !(box[0] > 0 && box[1] > 0 && box[2] > 0)) return 2;
    double* opos = (double*)malloc(sizeof(double) * 3 * (size_t)n_mol);
    double* dummy = (double*)malloc(sizeof(double) * (size_t)n_mol);
    const int rc = fx_uniform(n_mol, box, 0, min_oo, seed, opos, dummy);
    free(dummy);
    if (rc) {
        free(opos);
        return rc;
    }
    mt64* rng = (mt64*)malloc(sizeof(mt64));
    mt_seed(rng, seed ^ 0x9E3779B97F4A7C15ULL);
    const double d_oh = 0.9572;
    const double theta = 104.52 * 3.14159265358979323846 / 180.0;
    const double ct = cos(theta), st = sin(theta);
    for (int64_t m = 0; m < n_mol; ++m) {
        double u1[3], w[3];
        unit_normal3(rng, u1);
        for (;;) {
            unit_normal3(rng, w);
            const double d = w[0] * u1[0] + w[1] * u1[1] + w[2] * u1[2];
            for (int ax = 0; ax < 3; ++ax) w[ax] -= d * u1[ax];
            const double nn = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
            if (nn > 1e-3) {
                for (int ax = 0; ax < 3; ++ax) w[ax] /= nn;
                break;
            }
        }
        double* o = pos + 9 * m;
        for (int ax = 0; ax < 3; ++ax) {
            o[ax] = opos[3 * m + ax];
            o[3 + ax] = o[ax] + d_oh * u1[ax];
            o[6 + ax] = o[ax] + d_oh * (ct * u1[ax] + st * w[ax]);
        }
        q[3 * m] = -0.834;
        q[3 * m + 1] = 0.417;
        q[3 * m + 2] = 0.417;
        mass[3 * m] = 16.0;
        mass[3 * m + 1] = 1.0;
        mass[3 * m + 2] = 1.0;
    }
    free(rng);
    free(opos);
    return 0;
}
