// All-pairs kernels:
//   F3  direct_coulomb             src/electrostatics.cpp:43-64  (DirectCoulombField)
//   F2  PairRepulsionOverlay       src/force_field.cpp:45-68     (U = sum eps (sigma/r)^12)
// Both are O(N^2) over every pair in the reference.  Here one thread owns atom i
// (original order) and walks all j, staged 128 at a time into shared memory as
// (x, y, z, q) rows that every lane reads at the same address (broadcast: no bank
// conflicts), so the loop is bound by the FP64 pipe.  For small N the j range is
// split over S blocks per i-block (grid >= ~4 waves on 148 SMs) and the S partial
// sums are added in split order by k_allpairs_reduce: deterministic, no atomics
// on values.  Each pair is evaluated from both sides (no Newton-3 scatter), so a
// pair costs ~20 DP instructions per side.
//
// Reference semantics kept: a coincident pair (r2 == 0, i != j) is reported as the
// lexicographically first (i, j) (check_distinct, electrostatics.cpp:14-18,
// force_field.cpp:54-56); phi_i += q_j / r; F_i += d k_C q_i q_j / r^3; the overlay
// adds F_i += d 12 eps sigma^12 / r^14 and eps sigma^12 / r^12 per pair to the total
// energy, and leaves the per-particle potential alone.  The reference's i<j loop
// accumulates in a different order: results agree to rounding (tests: 1e-10 E,
// 1e-8 RMS F).
#include <cuda_runtime.h>

#include <algorithm>

#include "msmb_kernels.cuh"

namespace msmb {

namespace {

constexpr int kAP = 128; // threads per block = j rows per shared-memory tile

__device__ __forceinline__ bool ap_failed(const ErrRec* e) { return __ldcg(&e->kind) != 0; }

// 1/sqrt(x), 0 < x < inf: MUFU.RSQ64H seed + one cubic Newton step (full precision;
// same as the pair kernel's rsqrt_pos in msmb_kernels.cu)
__device__ __forceinline__ double ap_rsqrt(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double e = fma(-(x * y), y, 1.0);
    return fma(y * e, fma(e, 0.375, 0.5), y);
}

// partial sums: [s][k][n], k = 0 phi, 1..3 F (without the k_C q_i factor for coul),
// 4 e_rep; S == 1 writes the final values directly
template <int COUL, int REP>
__global__ void __launch_bounds__(kAP)
    k_allpairs(int64_t n, const double* __restrict__ x, const double* __restrict__ y,
               const double* __restrict__ z, const double* __restrict__ q, double kc, double rep_a,
               double rep_f, int64_t chunk, int S, double* __restrict__ part, DevOut o,
               double* __restrict__ e_rep, ErrRec* err) {
    __shared__ double4 s_j[kAP];
    if (ap_failed(err)) return;
    const int64_t i = int64_t(blockIdx.x) * kAP + threadIdx.x;
    const int s = blockIdx.y;
    const int64_t j0 = int64_t(s) * chunk, j1 = min(n, j0 + chunk);
    const bool vi = i < n;
    const double xi = vi ? x[i] : 0.0, yi = vi ? y[i] : 0.0, zi = vi ? z[i] : 0.0;
    double ph = 0.0, fx = 0.0, fy = 0.0, fz = 0.0, er = 0.0, rx = 0.0, ry = 0.0, rz = 0.0;
    unsigned long long bad = ~0ull;
    for (int64_t t0 = j0; t0 < j1; t0 += kAP) {
        __syncthreads();
        const int64_t jt = t0 + threadIdx.x;
        s_j[threadIdx.x] = jt < j1 ? make_double4(x[jt], y[jt], z[jt], q[jt]) : make_double4(0, 0, 0, 0);
        __syncthreads();
        const int m = int(j1 - t0 < kAP ? j1 - t0 : kAP);
#pragma unroll 4
        for (int t = 0; t < m; ++t) {
            const double4 J = s_j[t];
            const int64_t j = t0 + t;
            const double dx = xi - J.x, dy = yi - J.y, dz = zi - J.z;
            const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
            const bool self = j == i;
            if (r2 == 0.0 && !self && vi) // coincident (never on the hot path)
                bad = min(bad, (static_cast<unsigned long long>(min(i, j)) << 32) |
                                   static_cast<unsigned long long>(max(i, j)));
            const double rinv = ap_rsqrt(self ? 1.0 : r2);
            const double rinv2 = rinv * rinv;
            if (COUL) {
                const double qj = self ? 0.0 : J.w;
                ph = fma(qj, rinv, ph);
                const double w = qj * rinv * rinv2;
                fx = fma(dx, w, fx);
                fy = fma(dy, w, fy);
                fz = fma(dz, w, fz);
            }
            if (REP) {
                const double i4 = rinv2 * rinv2;
                const double i12 = self ? 0.0 : i4 * i4 * i4;
                er = fma(rep_a, i12, er);              // eps sigma^12 / r^12
                const double w = rep_f * i12 * rinv2;  // 12 eps sigma^12 / r^14
                rx = fma(dx, w, rx);
                ry = fma(dy, w, ry);
                rz = fma(dz, w, rz);
            }
        }
    }
    if (bad != ~0ull) atomicMin(&err->pair_key, bad);
    if (!vi) return;
    // F_i = sum d k_C q_i q_j / r^3 (electrostatics.cpp:57-61) + sum d 12 eps sigma^12 / r^14
    const double kq = kc * q[i];
    const double Fx = (COUL ? fx * kq : 0.0) + (REP ? rx : 0.0);
    const double Fy = (COUL ? fy * kq : 0.0) + (REP ? ry : 0.0);
    const double Fz = (COUL ? fz * kq : 0.0) + (REP ? rz : 0.0);
    if (S == 1) {
        if (COUL) {
            o.fx[i] = Fx;
            o.fy[i] = Fy;
            o.fz[i] = Fz;
            if (o.phi) o.phi[i] = ph;
            if (o.phis) o.phis[i] = ph;
            if (o.phil) o.phil[i] = 0.0;
            if (o.e) o.e[i] = 0.5 * q[i] * ph;
        } else {
            o.fx[i] += Fx;
            o.fy[i] += Fy;
            o.fz[i] += Fz;
        }
        if (REP) e_rep[i] = 0.5 * er;
        return;
    }
    double* P = part + size_t(s) * 5 * size_t(n);
    P[i] = ph;
    P[size_t(n) + i] = Fx;
    P[2 * size_t(n) + i] = Fy;
    P[3 * size_t(n) + i] = Fz;
    P[4 * size_t(n) + i] = er;
}

template <int COUL, int REP>
__global__ void k_allpairs_reduce(int64_t n, int S, const double* __restrict__ part, const double* __restrict__ q,
                                  DevOut o, double* __restrict__ e_rep, const ErrRec* err) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n || ap_failed(err)) return;
    double v[5] = {0, 0, 0, 0, 0};
    for (int s = 0; s < S; ++s) // split order: deterministic
        for (int k = 0; k < 5; ++k) v[k] += part[(size_t(s) * 5 + k) * size_t(n) + i];
    if (COUL) {
        o.fx[i] = v[1];
        o.fy[i] = v[2];
        o.fz[i] = v[3];
        if (o.phi) o.phi[i] = v[0];
        if (o.phis) o.phis[i] = v[0];
        if (o.phil) o.phil[i] = 0.0;
        if (o.e) o.e[i] = 0.5 * q[i] * v[0];
    } else {
        o.fx[i] += v[1];
        o.fy[i] += v[2];
        o.fz[i] += v[3];
    }
    if (REP) e_rep[i] = 0.5 * v[4];
}

template <int COUL, int REP>
int launch_t(cudaStream_t st, const DevState& s, double kc, double eps, double sigma, const AllPairsBuf& B,
             DevOut& o, ErrRec* err) {
    const int64_t n = s.n;
    const int ib = int((n + kAP - 1) / kAP);
    const int S = B.S;
    const int64_t chunk = ((n + S - 1) / S + kAP - 1) / kAP * kAP;
    const double s6 = pow(sigma, 6.0), s12 = s6 * s6; // force_field.cpp:47-48
    k_allpairs<COUL, REP><<<dim3(ib, S), kAP, 0, st>>>(n, s.x, s.y, s.z, s.q, kc, eps * s12, 12.0 * eps * s12,
                                                       chunk, S, B.part, o, B.e_rep, err);
    if (S == 1) return 1;
    k_allpairs_reduce<COUL, REP><<<int((n + 255) / 256), 256, 0, st>>>(n, S, B.part, s.q, o, B.e_rep, err);
    return 2;
}

} // namespace

int allpairs_splits(int64_t n) {
    const int64_t ib = (n + kAP - 1) / kAP;
    const int64_t want = 148 * 16; // ~4 waves of 4 resident 128-thread blocks per SM
    int64_t S = (want + std::max<int64_t>(ib, 1) - 1) / std::max<int64_t>(ib, 1);
    S = std::min<int64_t>(S, std::max<int64_t>(1, n / kAP)); // at least one tile per split
    return int(std::max<int64_t>(1, std::min<int64_t>(S, 64)));
}

int launch_allpairs(cudaStream_t st, const DevState& s, double kc, int coul, int rep, double eps, double sigma,
                    const AllPairsBuf& B, DevOut& o, ErrRec* err) {
    if (s.n <= 0) return 0;
    if (coul && rep) return launch_t<1, 1>(st, s, kc, eps, sigma, B, o, err);
    if (coul) return launch_t<1, 0>(st, s, kc, eps, sigma, B, o, err);
    if (rep) return launch_t<0, 1>(st, s, kc, eps, sigma, B, o, err);
    return 0;
}

} // namespace msmb
