// Probe: cost of early-exit kernels between kernels with different shared-memory
// needs, with and without a common preferred carveout (max shared) for all.
// nvcc -gencode arch=compute_100a,code=sm_100a -o tools/carveout_probe tools/carveout_probe.cu && tools/carveout_probe
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(32) k_big(float* out) { // 9.5 KB of static shared memory per 1-warp CTA
    __shared__ float s[2432];
    for (int i = threadIdx.x; i < 2432; i += 32) s[i] = float(i);
    __syncwarp();
    if (threadIdx.x == 0 && s[blockIdx.x % 2432] < 0.f) out[0] = 1.f;
}
__global__ void k_exit(const int* flag, float* out) {
    if (!flag[0]) return;
    out[1] = 1.f;
}
__global__ void __launch_bounds__(256) k_exit_smem(const int* flag, float* out) {
    __shared__ float s[1024];
    if (!flag[0]) return;
    s[threadIdx.x] = 1.f;
    __syncthreads();
    out[2] = s[(threadIdx.x + 1) & 255];
}

int main() {
    int* flag;
    float* out;
    cudaMalloc(&flag, 4);
    cudaMalloc(&out, 64);
    cudaMemset(flag, 0, 4);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int mode = 0; mode < 4; ++mode) {
        if (mode == 2) {
            cudaFuncSetAttribute(k_big, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
            cudaFuncSetAttribute(k_exit, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
            cudaFuncSetAttribute(k_exit_smem, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 cudaSharedmemCarveoutMaxShared);
        }
        const bool withbig = mode != 1;
        cudaGraph_t g;
        cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
        for (int rep = 0; rep < 50; ++rep) {
            if (withbig) k_big<<<2960, 32, 0, st>>>(out);
            for (int i = 0; i < 2; ++i) k_exit<<<1172, 256, 0, st>>>(flag, out);
            for (int i = 0; i < 2; ++i) k_exit_smem<<<1200, 256, 0, st>>>(flag, out);
        }
        cudaStreamEndCapture(st, &g);
        cudaGraphExec_t ex;
        cudaGraphInstantiate(&ex, g, 0);
        cudaGraphLaunch(ex, st);
        cudaStreamSynchronize(st);
        cudaEventRecord(a, st);
        for (int i = 0; i < 4; ++i) cudaGraphLaunch(ex, st);
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("mode %d (%s): %.2f us per repetition (big kernel + 4 early-exit kernels)\n", mode,
               mode == 0 ? "default carveouts" : mode == 1 ? "no big kernel" : mode == 2 ? "all max-shared" : "again",
               ms * 1000.f / 200);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
