// Probe: cost of IF conditional graph nodes (built during stream capture) against
// kernels that read a device flag and exit, the two ways of skipping the pair-list
// rebuild kernels on skin steps.
// nvcc -gencode arch=compute_100a,code=sm_100a -o tools/cond_probe tools/cond_probe.cu && tools/cond_probe
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess) {                                                                \
            printf("%s:%d %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_));        \
            return 1;                                                                           \
        }                                                                                       \
    } while (0)

__global__ void k_set(cudaGraphConditionalHandle h, const int* flag) { cudaGraphSetConditional(h, flag[0] ? 1u : 0u); }
__global__ void k_exit(const int* flag, int* out) { // early exit on flag 0 (1172 blocks, like k_cl_perm)
    if (!flag[0]) return;
    atomicAdd(out, 1);
}
__global__ void k_work(int* out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) atomicAdd(out, 1);
}

static cudaStream_t st, st2;
static int *flag, *out;

// mode 0: 1 work kernel + 10 early-exit kernels + 1 work kernel
// mode 1: 1 work kernel + set + IF{10 kernels} + 1 work kernel
// mode 2: 2 work kernels only
static int build(int mode, cudaGraphExec_t* ex) {
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    for (int rep = 0; rep < 50; ++rep) { // 50 repetitions per graph: GPU time, not host launch rate
    k_work<<<148, 256, 0, st>>>(out);
    if (mode == 0)
        for (int i = 0; i < 10; ++i) k_exit<<<1172, 256, 0, st>>>(flag, out);
    if (mode == 1) {
        cudaStreamCaptureStatus cs;
        cudaGraph_t g;
        const cudaGraphNode_t* deps;
        size_t nd;
        CK(cudaStreamGetCaptureInfo(st, &cs, nullptr, &g, &deps, &nd));
        cudaGraphConditionalHandle h;
        CK(cudaGraphConditionalHandleCreate(&h, g, 0, cudaGraphCondAssignDefault));
        k_set<<<1, 1, 0, st>>>(h, flag);
        CK(cudaStreamGetCaptureInfo(st, &cs, nullptr, &g, &deps, &nd));
        cudaGraphNodeParams p = {};
        p.type = cudaGraphNodeTypeConditional;
        p.conditional.handle = h;
        p.conditional.type = cudaGraphCondTypeIf;
        p.conditional.size = 1;
        cudaGraphNode_t node;
        CK(cudaGraphAddNode(&node, g, deps, nd, &p));
        CK(cudaStreamUpdateCaptureDependencies(st, &node, 1, cudaStreamSetCaptureDependencies));
        cudaGraph_t body = p.conditional.phGraph_out[0];
        CK(cudaStreamBeginCaptureToGraph(st2, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
        for (int i = 0; i < 10; ++i) k_exit<<<1172, 256, 0, st2>>>(flag, out);
        CK(cudaStreamEndCapture(st2, &body));
    }
    k_work<<<148, 256, 0, st>>>(out);
    }
    cudaGraph_t whole;
    CK(cudaStreamEndCapture(st, &whole));
    CK(cudaGraphInstantiateWithFlags(ex, whole, cudaGraphInstantiateFlagUseNodePriority));
    return 0;
}

int main() {
    CK(cudaMalloc(&flag, 4));
    CK(cudaMalloc(&out, 4));
    CK(cudaMemset(out, 0, 4));
    CK(cudaMemset(flag, 0, 4));
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&st2, cudaStreamNonBlocking));
    cudaGraphExec_t ex[3];
    for (int m = 0; m < 3; ++m)
        if (build(m, &ex[m])) return 1;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const char* names[3] = {"10 early-exit kernels", "IF node (untaken) over them", "neither"};
    for (int rep = 0; rep < 2; ++rep)
        for (int m = 0; m < 3; ++m) {
            // a long kernel first so the launches queue up: GPU time only
            for (int i = 0; i < 2; ++i) CK(cudaGraphLaunch(ex[m], st));
            CK(cudaStreamSynchronize(st));
            cudaEventRecord(a, st);
            for (int i = 0; i < 4; ++i) cudaGraphLaunch(ex[m], st);
            cudaEventRecord(b, st);
            CK(cudaEventSynchronize(b));
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("%-30s %.2f us per repetition\n", names[m], ms * 1000.f / 200);
        }
    printf("OK\n");
    return 0;
}
