// K5 (lattice cutoff, levels 0..l-2) as a zero-padded FFT convolution.
//
// The reference sums the (2R+1)^3 stencil directly, R = ceil(2a/h), clipped at the
// lattice edges (src/msm_phases.cpp:93-134).  That is a linear convolution of the
// level-k charges with a real, even kernel K_k = 2^-k K_0.  Take per axis a padded
// length M >= d + R with M = 2^a 3^b.  A circular convolution of length M then
// equals the clipped linear one at every output 0 <= x < d: sources at x - dx < 0
// wrap to indices >= M - R >= d, where the padded charges are zero.  So
//     u_k = IFFT( FFT(q_k padded) * Khat_k ) restricted to [0, d),
// with Khat_k = FFT(K_k wrapped) real (K is even), precomputed once per geometry
// and pre-divided by M0*M1*M2.  Cost per level: O(M^3 log M) instead of
// (d^3 * nonzero taps) DFMAs.  For C2 that is 9.2e8 FMAs into a few MB of
// L2-resident passes; for C3 (L0 226^3) it is 4.7e10 FMAs into ~2 GB of passes.
// Results differ from the direct sum only by rounding: ~1e-15 of the lattice
// scale (tests/test_gpu_stages.py holds it to 1e-13).
//
// Layout: per level a complex buffer B[x][y][z] (z fastest) of M0 x M1 x M2.
// Every 1-D transform runs on tiles of L lines staged in shared memory, with a
// mixed-radix (4, 2, 3) Stockham autosort and ping-pong buffers.  Passes
// (lines/outputs pruned to what is nonzero or needed):
//   X fwd  lines (y < d1, z < d2)  in: q (x < d0, real)   out: B, all x
//   Y fwd  lines (x < M0, z < d2)  in: B (y < d1)         out: B, all y
//   Z      lines (x < M0, y < M1)  in: B (z < d2)         fwd, * Khat, inv; out z < d2
//   Y inv  lines (x < M0, z < d2)  in: B (all y)          out: B, y < d1
//   X inv  lines (y < d1, z < d2)  in: B (all x)          out: u = Re, x < d0
// All levels of one pass are one launch.  There are no atomics and the order is
// fixed, so results are deterministic.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "msmb_kernels.cuh"

namespace msmb {

namespace {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }

// In-place (ping-pong) Stockham over L lines of length M at a[l * M + i].
// Returns the buffer that holds the result.
__device__ double2* fft_lines(double2* a, double2* b, int L, const FftAxis& ax, const double2* __restrict__ tw,
                              bool inv) {
    const int M = ax.M;
    int Ns = 1;
    for (int s = 0; s < ax.nf; ++s) {
        const int R = ax.fac[s];
        const int NR = M / R;
        const int stride = M / (Ns * R);
        for (int t = threadIdx.x; t < L * NR; t += blockDim.x) {
            const int l = t / NR, j = t - l * NR;
            const int jm = j % Ns;
            const double2* src = a + l * M;
            double2* dst = b + l * M;
            double2 v[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                if (r < R) {
                    v[r] = src[j + r * NR];
                    if (r > 0 && jm > 0) {
                        double2 w = __ldg(tw + ax.tw + jm * r * stride);
                        if (inv) w.y = -w.y;
                        v[r] = cmul(v[r], w);
                    }
                }
            }
            const int d0 = (j / Ns) * Ns * R + jm;
            if (R == 4) {
                const double2 t0 = cadd(v[0], v[2]), t1 = csub(v[0], v[2]);
                const double2 t2 = cadd(v[1], v[3]), t3 = csub(v[1], v[3]);
                dst[d0] = cadd(t0, t2);
                dst[d0 + 2 * Ns] = csub(t0, t2);
                if (!inv) {
                    dst[d0 + Ns] = make_double2(t1.x + t3.y, t1.y - t3.x);
                    dst[d0 + 3 * Ns] = make_double2(t1.x - t3.y, t1.y + t3.x);
                } else {
                    dst[d0 + Ns] = make_double2(t1.x - t3.y, t1.y + t3.x);
                    dst[d0 + 3 * Ns] = make_double2(t1.x + t3.y, t1.y - t3.x);
                }
            } else if (R == 2) {
                dst[d0] = cadd(v[0], v[1]);
                dst[d0 + Ns] = csub(v[0], v[1]);
            } else { // R == 3
                const double c = 0.86602540378443864676; // sqrt(3)/2
                const double2 sm = cadd(v[1], v[2]), df = csub(v[1], v[2]);
                const double2 m = make_double2(v[0].x - 0.5 * sm.x, v[0].y - 0.5 * sm.y);
                dst[d0] = cadd(v[0], sm);
                const double sx = inv ? -c : c;
                dst[d0 + Ns] = make_double2(m.x + sx * df.y, m.y - sx * df.x);
                dst[d0 + 2 * Ns] = make_double2(m.x - sx * df.y, m.y + sx * df.x);
            }
        }
        __syncthreads();
        double2* tmp = a;
        a = b;
        b = tmp;
        Ns *= R;
    }
    return a;
}

__device__ __forceinline__ int find_level(const FftJobs& J, int blk) {
    int k = 0;
    while (k + 1 < J.n && blk >= J.lv[k + 1].blk0) ++k;
    return k;
}

// X pass: lines along x at (y, z0 + l).  mode 2: forward from B over every line
// (spectrum precompute, complex).  Modes 0 / 1 use that the charges and potentials are
// real: two lines (z0 + 2p, z0 + 2p + 1) travel as one complex line c = e + i o, and
// only the x-frequencies 0 .. M0/2 are kept (the rest is the complex conjugate), so the
// Y and Z passes run on M0/2 + 1 planes instead of M0 (half the work and traffic):
//   mode 0: q -> c -> FFT -> E[k] = (C[k] + conj C[M0-k]) / 2, O[k] = (C[k] - conj C[M0-k]) / 2i
//   mode 1: E, O (k <= M0/2, conjugate-extended) -> C = E + i O -> IFFT -> u_e = Re, u_o = Im
__global__ void __launch_bounds__(256) k_fft_x(FftJobs J, int mode, const ErrRec* err) {
    extern __shared__ double2 sm[];
    pdl_enter();
    if (err && __ldcg(&err->kind)) return;
    const int k = find_level(J, blockIdx.x);
    const FftLevel& lv = J.lv[k];
    const int M0 = lv.ax[0].M, M1 = lv.ax[1].M, M2 = lv.ax[2].M;
    const int zlim = mode == 2 ? M2 : lv.d[2];
    const int b = blockIdx.x - lv.blk0;
    const int nzt = (zlim + J.L - 1) / J.L;
    const int y = b / nzt, z0 = (b % nzt) * J.L;
    const int L = min(J.L, zlim - z0);
    double2* A = sm;
    double2* Bf = sm + J.L * J.maxM;
    double2* buf = J.buf + lv.boff;
    if (mode == 2) {
        for (int t = threadIdx.x; t < L * M0; t += blockDim.x) {
            const int x = t / L, l = t - x * L, z = z0 + l;
            A[l * M0 + x] = buf[(size_t(x) * M1 + y) * M2 + z];
        }
        __syncthreads();
        const double2* R = fft_lines(A, Bf, L, lv.ax[0], J.tw, false);
        for (int t = threadIdx.x; t < L * M0; t += blockDim.x) {
            const int x = t / L, l = t - x * L, z = z0 + l;
            buf[(size_t(x) * M1 + y) * M2 + z] = R[l * M0 + x];
        }
        return;
    }
    const int H0 = M0 / 2 + 1;
    const int Lp = (L + 1) / 2; // line pairs in this tile
    if (mode == 0) {
        for (int t = threadIdx.x; t < Lp * M0; t += blockDim.x) {
            const int x = t / Lp, p = t - x * Lp, ze = z0 + 2 * p, zo = ze + 1;
            double2 v = make_double2(0.0, 0.0);
            if (x < lv.d[0]) {
                const double* qr = lv.q + (size_t(x) * lv.d[1] + y) * lv.d[2];
                v.x = qr[ze];
                if (zo < z0 + L) v.y = qr[zo];
            }
            A[p * M0 + x] = v;
        }
        __syncthreads();
        const double2* R = fft_lines(A, Bf, Lp, lv.ax[0], J.tw, false);
        for (int t = threadIdx.x; t < Lp * H0; t += blockDim.x) {
            const int kx = t / Lp, p = t - kx * Lp, ze = z0 + 2 * p, zo = ze + 1;
            const double2 c = R[p * M0 + kx], cm = R[p * M0 + (M0 - kx) % M0];
            buf[(size_t(kx) * M1 + y) * M2 + ze] = make_double2(0.5 * (c.x + cm.x), 0.5 * (c.y - cm.y));
            if (zo < z0 + L) buf[(size_t(kx) * M1 + y) * M2 + zo] = make_double2(0.5 * (c.y + cm.y), 0.5 * (cm.x - c.x));
        }
        return;
    }
    // mode 1: inverse to u
    for (int t = threadIdx.x; t < Lp * M0; t += blockDim.x) {
        const int kx = t / Lp, p = t - kx * Lp, ze = z0 + 2 * p, zo = ze + 1;
        const bool lo = kx < H0;
        const int ks = lo ? kx : M0 - kx;
        double2 e = buf[(size_t(ks) * M1 + y) * M2 + ze];
        double2 o = zo < z0 + L ? buf[(size_t(ks) * M1 + y) * M2 + zo] : make_double2(0.0, 0.0);
        if (!lo) { // conjugate symmetry of the spectra of real lines
            e.y = -e.y;
            o.y = -o.y;
        }
        A[p * M0 + kx] = make_double2(e.x - o.y, e.y + o.x); // E + i O
    }
    __syncthreads();
    const double2* R = fft_lines(A, Bf, Lp, lv.ax[0], J.tw, true);
    for (int t = threadIdx.x; t < Lp * M0; t += blockDim.x) {
        const int x = t / Lp, p = t - x * Lp, ze = z0 + 2 * p, zo = ze + 1;
        if (x >= lv.d[0]) continue;
        double* ur = lv.u + (size_t(x) * lv.d[1] + y) * lv.d[2];
        const double2 c = R[p * M0 + x];
        ur[ze] = c.x;
        if (zo < z0 + L) ur[zo] = c.y;
    }
}

// Y pass: lines along y at (x, z0 + l).  mode 0: forward (input y < d1);
// 1: inverse (output y < d1); 2: forward over every line.
__global__ void __launch_bounds__(256) k_fft_y(FftJobs J, int mode, const ErrRec* err) {
    extern __shared__ double2 sm[];
    pdl_enter();
    if (err && __ldcg(&err->kind)) return;
    const int k = find_level(J, blockIdx.x);
    const FftLevel& lv = J.lv[k];
    const int M1 = lv.ax[1].M, M2 = lv.ax[2].M;
    const int zlim = mode == 2 ? M2 : lv.d[2];
    const int b = blockIdx.x - lv.blk0;
    const int nzt = (zlim + J.L - 1) / J.L;
    const int x = b / nzt, z0 = (b % nzt) * J.L;
    const int L = min(J.L, zlim - z0);
    double2* A = sm;
    double2* Bf = sm + J.L * J.maxM;
    double2* buf = J.buf + lv.boff + size_t(x) * M1 * M2;
    const int inlen = mode == 0 ? lv.d[1] : M1;
    for (int t = threadIdx.x; t < L * M1; t += blockDim.x) {
        const int y = t / L, l = t - y * L;
        A[l * M1 + y] = y < inlen ? buf[size_t(y) * M2 + z0 + l] : make_double2(0.0, 0.0);
    }
    __syncthreads();
    const double2* R = fft_lines(A, Bf, L, lv.ax[1], J.tw, mode == 1);
    const int outlen = mode == 1 ? lv.d[1] : M1;
    for (int t = threadIdx.x; t < L * M1; t += blockDim.x) {
        const int y = t / L, l = t - y * L;
        if (y < outlen) buf[size_t(y) * M2 + z0 + l] = R[l * M1 + y];
    }
}

// Z pass: lines along z at (x, y0 + l).  mode 0: forward (input z < d2), * Khat,
// inverse, output z < d2; 2: forward over every line, Khat = Re / (M0 M1 M2).
__global__ void __launch_bounds__(256) k_fft_z(FftJobs J, int mode, const ErrRec* err) {
    extern __shared__ double2 sm[];
    pdl_enter();
    if (err && __ldcg(&err->kind)) return;
    const int k = find_level(J, blockIdx.x);
    const FftLevel& lv = J.lv[k];
    const int M0 = lv.ax[0].M, M1 = lv.ax[1].M, M2 = lv.ax[2].M;
    const int b = blockIdx.x - lv.blk0;
    const int nyt = (M1 + J.L - 1) / J.L;
    const int x = b / nyt, y0 = (b % nyt) * J.L;
    const int L = min(J.L, M1 - y0);
    double2* A = sm;
    double2* Bf = sm + J.L * J.maxM;
    const size_t base = (size_t(x) * M1 + y0) * M2;
    double2* buf = J.buf + lv.boff + base;
    const int inlen = mode == 0 ? lv.d[2] : M2;
    for (int t = threadIdx.x; t < L * M2; t += blockDim.x) {
        const int l = t / M2, z = t - l * M2;
        A[t] = z < inlen ? buf[size_t(l) * M2 + z] : make_double2(0.0, 0.0);
    }
    __syncthreads();
    double2* R = fft_lines(A, Bf, L, lv.ax[2], J.tw, false);
    double2* O = R == A ? Bf : A;
    if (mode == 2) {
        const double inv = 1.0 / (double(M0) * M1 * M2);
        double* spec = J.spec + lv.soff + base;
        for (int t = threadIdx.x; t < L * M2; t += blockDim.x) spec[t] = R[t].x * inv;
        return;
    }
    const double* spec = J.spec + lv.soff + base;
    for (int t = threadIdx.x; t < L * M2; t += blockDim.x) {
        const double s = __ldg(spec + t);
        R[t] = make_double2(R[t].x * s, R[t].y * s);
    }
    __syncthreads();
    R = fft_lines(R, O, L, lv.ax[2], J.tw, true);
    for (int t = threadIdx.x; t < L * M2; t += blockDim.x) {
        const int l = t / M2, z = t - l * M2;
        if (z < lv.d[2]) buf[size_t(l) * M2 + z] = R[t];
    }
}

// The kernel of job k wrapped into B (spectrum precompute):
// B[dx mod M0][dy mod M1][dz mod M2] = K(dx, dy, dz) for the offsets a pair of
// lattice points can have (|d| < dims).  Those wrap to distinct slots: M >= d + R
// for the cutoff levels, M >= 2d - 1 for the dense top level.  The other offsets
// would alias (M < 2R + 1 on small levels) and only feed discarded outputs.
//   cutoff levels: K = 2^-k * level-0 stencil (rowidx / taps, half-width R)
//   top level:     dense offset table [2d0-1][2d1-1][rowlen] of k_top_direct
__global__ void k_fft_stencil(FftJobs J, int k, FftKernel K) {
    const FftLevel& lv = J.lv[k];
    const int W0 = 2 * K.R[0] + 1, W1 = 2 * K.R[1] + 1, W2 = 2 * K.R[2] + 1;
    const int64_t tot = int64_t(W0) * W1 * W2;
    const int M0 = lv.ax[0].M, M1 = lv.ax[1].M, M2 = lv.ax[2].M;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < tot; i += int64_t(gridDim.x) * blockDim.x) {
        const int dz = int(i % W2) - K.R[2], dy = int((i / W2) % W1) - K.R[1], dx = int(i / (int64_t(W2) * W1)) - K.R[0];
        if (abs(dx) >= lv.d[0] || abs(dy) >= lv.d[1] || abs(dz) >= lv.d[2]) continue;
        double v;
        if (K.dense) {
            v = K.taps[(size_t(dx + K.R[0]) * W1 + (dy + K.R[1])) * K.rowlen + (dz + K.R[2])];
        } else {
            const int r = K.rowidx[(dx + K.R[0]) * W1 + (dy + K.R[1])];
            v = r >= 0 ? K.taps[size_t(r) * K.rowlen + dz + K.R[2]] : 0.0;
        }
        const int x = (dx + M0) % M0, y = (dy + M1) % M1, z = (dz + M2) % M2;
        J.buf[lv.boff + (size_t(x) * M1 + y) * M2 + z] = make_double2(v * K.scale, 0.0);
    }
}

int blocks_x(FftJobs& J, bool all) {
    int tot = 0;
    for (int k = 0; k < J.n; ++k) {
        FftLevel& lv = J.lv[k];
        lv.blk0 = tot;
        const int zl = all ? lv.ax[2].M : lv.d[2], yl = all ? lv.ax[1].M : lv.d[1];
        tot += yl * ((zl + J.L - 1) / J.L);
    }
    return tot;
}
// the Y and Z passes of the convolution (modes 0 / 1) cover the x-frequencies
// 0 .. M0/2 only (real data, see k_fft_x); the spectrum precompute covers all
int blocks_y(FftJobs& J, bool all) {
    int tot = 0;
    for (int k = 0; k < J.n; ++k) {
        FftLevel& lv = J.lv[k];
        lv.blk0 = tot;
        const int zl = all ? lv.ax[2].M : lv.d[2];
        const int planes = all ? lv.ax[0].M : lv.ax[0].M / 2 + 1;
        tot += planes * ((zl + J.L - 1) / J.L);
    }
    return tot;
}
int blocks_z(FftJobs& J, bool all) {
    int tot = 0;
    for (int k = 0; k < J.n; ++k) {
        FftLevel& lv = J.lv[k];
        lv.blk0 = tot;
        const int planes = all ? lv.ax[0].M : lv.ax[0].M / 2 + 1;
        tot += planes * ((lv.ax[1].M + J.L - 1) / J.L);
    }
    return tot;
}

size_t fft_smem(const FftJobs& J) { return size_t(2) * J.L * J.maxM * sizeof(double2); }
// threads per tile: 256 for the default 16-line tiles, one warp for tiles of <= 2 lines
int fft_threads(const FftJobs& J) { return J.L >= 16 ? 256 : std::max(32, ((J.L * 16 + 31) / 32) * 32); }

} // namespace

int fft_len(int need) { // smallest 2^a 3^b >= need
    int best = 1 << 30;
    for (int64_t p2 = 1; p2 < (1 << 30); p2 *= 2)
        for (int64_t p = p2; p < (1 << 30); p *= 3)
            if (p >= need) {
                best = std::min<int64_t>(best, p);
                break;
            }
    return best;
}

FftAxis fft_axis(int M, int tw_off) {
    FftAxis a{};
    a.M = M;
    a.tw = tw_off;
    int n = M;
    while (n % 4 == 0) a.fac[a.nf++] = 4, n /= 4;
    while (n % 2 == 0) a.fac[a.nf++] = 2, n /= 2;
    while (n % 3 == 0) a.fac[a.nf++] = 3, n /= 3;
    return a;
}

cudaError_t fft_prepare(size_t smem) {
    cudaError_t e = smem_grow(reinterpret_cast<const void*>(k_fft_x), smem);
    if (e == cudaSuccess) e = smem_grow(reinterpret_cast<const void*>(k_fft_y), smem);
    if (e == cudaSuccess) e = smem_grow(reinterpret_cast<const void*>(k_fft_z), smem);
    return e;
}

int launch_fft_spectrum(cudaStream_t st, FftJobs J, const FftKernel* K) {
    int nl = 0;
    for (int k = 0; k < J.n; ++k) {
        const FftLevel& lv = J.lv[k];
        cudaMemsetAsync(J.buf + lv.boff, 0, sizeof(double2) * size_t(lv.ax[0].M) * lv.ax[1].M * lv.ax[2].M, st);
        k_fft_stencil<<<148, 256, 0, st>>>(J, k, K[k]);
        ++nl;
    }
    const size_t sm = fft_smem(J);
    int nb = blocks_x(J, true);
    k_fft_x<<<nb, fft_threads(J), sm, st>>>(J, 2, nullptr);
    nb = blocks_y(J, true);
    k_fft_y<<<nb, fft_threads(J), sm, st>>>(J, 2, nullptr);
    nb = blocks_z(J, true);
    k_fft_z<<<nb, fft_threads(J), sm, st>>>(J, 2, nullptr);
    return nl + 3;
}

int launch_lattice_fft(cudaStream_t st, FftJobs J, const ErrRec* err) {
    if (J.n == 0) return 0;
    const size_t sm = fft_smem(J);
    const dim3 tb(fft_threads(J));
    pdl_launch(k_fft_x, dim3(blocks_x(J, false)), tb, sm, st, J, 0, err);
    pdl_launch(k_fft_y, dim3(blocks_y(J, false)), tb, sm, st, J, 0, err);
    pdl_launch(k_fft_z, dim3(blocks_z(J, false)), tb, sm, st, J, 0, err);
    pdl_launch(k_fft_y, dim3(blocks_y(J, false)), tb, sm, st, J, 1, err);
    pdl_launch(k_fft_x, dim3(blocks_x(J, false)), tb, sm, st, J, 1, err);
    return 5;
}

} // namespace msmb
