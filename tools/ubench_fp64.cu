// Microbenchmark (design input for the pair kernel's dense phase): what the FP64 pipe of
// one B200 sustains on instruction mixes, 20 one-warp CTAs per SM like k_pairs_mw.
//   dfma  : 8 independent DFMA chains (the bench's peak definition)
//   dadd / dmul : the same with DADD / DMUL only
//   mix3  : DADD, DMUL, DFMA round-robin on independent chains
//   pair  : the MSM pair step on register-resident j data (no memory), unrolled 4
//   pairs : the same with the j rows read from shared memory at a warp-uniform address
//   oct32 / oct33 : one row per octet of lanes, the four rows in the same / in different bank quads
//   half33 : one row per half-warp
// Prints DP instructions per clock per SM (peak = 2 warp instructions = 64 lanes).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_fp64 ubench_fp64.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITER = 2048;

__device__ __forceinline__ double rsqrt_pos(double x) {
    double y0;
    asm("{.reg .b32 lo, hi; mov.b64 {lo, hi}, %1; rsqrt.approx.ftz.f64 %0, %1;}" : "=d"(y0) : "d"(x));
    const double t = x * y0, e = fma(-t, y0, 1.0);
    return fma(y0 * e, fma(e, 0.375, 0.5), y0);
}

template <int MODE>
__global__ void __launch_bounds__(32, 20) k(double* out, double seed, double a2) {
    __shared__ double2 rows[2][192];
    const int lane = threadIdx.x;
    for (int i = lane; i < 192; i += 32) {
        rows[0][i] = make_double2(i * 1.0 + seed, i * 2.0);
        rows[1][i] = make_double2(i * 3.0, i * 0.01);
    }
    __syncwarp();
    double x = lane * 0.5 + seed, y = lane * 0.25 + 1.0, z = lane * 0.125 + 2.0;
    double a[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) a[c] = seed * c;
    const double c0 = 0.15 * seed, c1 = -7e-4 * seed, c2 = 1.5e-6 * seed, d0 = 1.4e-3 * seed, d1 = -6e-6 * seed;
    double ph = 0, fx = 0, fy = 0, fz = 0;
    for (int it = 0; it < ITER; ++it) {
        if (MODE == 0) {
#pragma unroll
            for (int u = 0; u < 3; ++u)
#pragma unroll
                for (int c = 0; c < 8; ++c) a[c] = fma(a[c], x, y);
        } else if (MODE == 1) {
#pragma unroll
            for (int u = 0; u < 3; ++u)
#pragma unroll
                for (int c = 0; c < 8; ++c) a[c] = a[c] + x;
        } else if (MODE == 2) {
#pragma unroll
            for (int u = 0; u < 3; ++u)
#pragma unroll
                for (int c = 0; c < 8; ++c) a[c] = a[c] * x;
        } else if (MODE == 3) {
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                a[c] = a[c] + x;
                a[c] = a[c] * y;
                a[c] = fma(a[c], z, x);
            }
        } else {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                double xj, yj, zj, qj0;
                if (MODE == 4) {
                    xj = a[u] + it;
                    yj = a[u + 4];
                    zj = z * 0.5;
                    qj0 = y;
                } else {
                    const int o = lane >> 3;
                    const int r = MODE == 5 ? ((it * 4 + u) & 31) : MODE == 6 ? o * 32 + ((it * 4 + u) & 31)
                                : MODE == 7 ? o * 33 + ((it * 4 + u) & 31) : (lane >> 4) * 33 + ((it * 4 + u) & 31);
                    const double2 xy = rows[0][r], zq = rows[1][r];
                    xj = xy.x; yj = xy.y; zj = zq.x; qj0 = zq.y;
                }
                const double dx = x - xj, dy = y - yj, dz = z - zj;
                const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
                const double rinv = rsqrt_pos(r2);
                const double g = rinv - fma(r2, fma(r2, c2, c1), c0);
                const double sd = fma(-rinv, rinv * rinv, fma(r2, d1, d0));
                const bool in = r2 < a2;
                const double qj = in ? qj0 : 0.0;
                ph = fma(qj, g, ph);
                const double wgt = qj * sd;
                fx = fma(dx, wgt, fx);
                fy = fma(dy, wgt, fy);
                fz = fma(dz, wgt, fz);
            }
        }
    }
    double s = ph + fx + fy + fz;
#pragma unroll
    for (int c = 0; c < 8; ++c) s += a[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE>
void run(const char* name, double* out, double dp_per_iter) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int blocks = 148 * 20 * 4;
    k<MODE><<<blocks, 32>>>(out, 1.0, 144.0);
    cudaEventRecord(a);
    k<MODE><<<blocks, 32>>>(out, 1.0, 144.0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    int khz = 0;
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    const double warp_instr = double(blocks) * ITER * dp_per_iter;
    const double clk = ms * 1e-3 * 1.965e9 * 148;
    printf("%-6s %.3f ms  %.3f DP warp-instr/clk/SM (peak 2)  %.2f TFLOP/s-equivalent as DFMA\n", name, ms,
           warp_instr / clk, warp_instr * 64 / (ms * 1e-3) / 1e12);
}

int main() {
    double* out;
    cudaMalloc(&out, sizeof(double) * 148 * 20 * 4 * 32);
    run<0>("dfma", out, 24);
    run<1>("dadd", out, 24);
    run<2>("dmul", out, 24);
    run<3>("mix3", out, 24);
    run<4>("pair", out, 4 * 24);
    run<5>("pairs", out, 4 * 24);
    run<6>("oct32", out, 4 * 24);
    run<7>("oct33", out, 4 * 24);
    run<8>("half33", out, 4 * 24);
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
