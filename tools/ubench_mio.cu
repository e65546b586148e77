// Microbenchmark (design input for the pair kernel): throughput of the MIO-side
// operations a pair step can use to move j-atom data, measured on one B200.
//   shfl  : 8 x SHFL.IDX (four doubles) with a per-lane permutation source
//   ldsp  : 2 x LDS.128 with a permutation of rows (conflict-free)
//   ldsr  : 2 x LDS.128 with pseudo-random rows (bank conflicts as in k_pairs_mw)
//   mix   : shfl + ldsp in the same loop (do they share a pipe?)
//   dfma  : 24 independent DFMA (FP64 pipe reference)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_mio ubench_mio.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITER = 4096;

template <int MODE>
__global__ void __launch_bounds__(128) k(double* out, int seed) {
    __shared__ double2 rows[4][2][64];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int i = lane; i < 64; i += 32) {
        rows[w][0][i] = make_double2(i * 1.0, i * 2.0);
        rows[w][1][i] = make_double2(i * 3.0, i * 4.0);
    }
    __syncwarp();
    double x = lane * 0.5 + seed, y = lane * 0.25, z = lane * 0.125, q = 1.0;
    double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    unsigned r = lane * 2654435761u + seed;
    int perm = lane;
    for (int it = 0; it < ITER; ++it) {
        perm = (perm * 5 + 7 + it) & 31; // x -> 5x + c mod 32 is a permutation of lanes
        if (MODE == 0 || MODE == 3) {
            const double xs = __shfl_sync(0xffffffffu, x, perm), ys = __shfl_sync(0xffffffffu, y, perm);
            const double zs = __shfl_sync(0xffffffffu, z, perm), qs = __shfl_sync(0xffffffffu, q, perm);
            a0 += xs; a1 += ys; a2 += zs; a3 += qs;
        }
        if (MODE == 1 || MODE == 3) {
            const double2 u = rows[w][0][perm + 1], v = rows[w][1][perm + 1];
            a0 += u.x; a1 += u.y; a2 += v.x; a3 += v.y;
        }
        if (MODE == 2) {
            r = r * 1664525u + 1013904223u;
            const int row = (r >> 20) & 31;
            const double2 u = rows[w][0][row + 1], v = rows[w][1][row + 1];
            a0 += u.x; a1 += u.y; a2 += v.x; a3 += v.y;
        }
        if (MODE == 4) {
#pragma unroll
            for (int u = 0; u < 6; ++u) {
                a0 = fma(a0, x, y); a1 = fma(a1, x, z); a2 = fma(a2, y, z); a3 = fma(a3, z, x);
            }
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3;
}

template <int MODE>
float run(double* out, int blocks) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k<MODE><<<blocks, 128>>>(out, 1);
    cudaEventRecord(a);
    for (int rep = 0; rep < 5; ++rep) k<MODE><<<blocks, 128>>>(out, rep);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / 5;
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int blocks = sms * 5; // 20 warps per SM
    double* out;
    cudaMalloc(&out, sizeof(double) * blocks * 128);
    const char* names[] = {"shfl(8xSHFL)", "lds_perm(2xLDS.128)", "lds_rand(2xLDS.128)", "mix(8SHFL+2LDS)", "dfma(24)"};
    float t[5] = {run<0>(out, blocks), run<1>(out, blocks), run<2>(out, blocks), run<3>(out, blocks),
                  run<4>(out, blocks)};
    const double warp_iters_per_sm = double(blocks) * 4 * ITER / sms;
    for (int m = 0; m < 5; ++m) {
        const double cyc = t[m] * 1e-3 * clk * 1e3 / warp_iters_per_sm;
        printf("%-22s %.3f ms  %.2f SM-cycles per warp-iteration\n", names[m], t[m], cyc);
    }
    printf("sm clock %d kHz, %d SMs, err=%s\n", clk, sms, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
