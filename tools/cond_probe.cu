// Overhead of CUDA graph conditional nodes on this GPU (diagnostic tool):
// a WHILE node whose body is 1 or 3 small kernels, iterated N times, vs the
// same kernels as plain graph nodes.
#include <cuda_runtime.h>
#include <cstdio>

__global__ void k_body(int* ctr, int n, cudaGraphConditionalHandle h, int set) {
    if (set && threadIdx.x == 0 && blockIdx.x == 0) {
        const int c = ++*ctr;
        cudaGraphSetConditional(h, c < n ? 1u : 0u);
    }
}
__global__ void k_plain(int* ctr) {
    if (threadIdx.x == 0 && blockIdx.x == 0) ++*ctr;
}
__global__ void k_reset(int* ctr) { *ctr = 0; }

int main() {
    int* ctr;
    cudaMalloc(&ctr, 4);
    cudaStream_t st, cap;
    cudaStreamCreate(&st);
    cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking);
    const int N = 100;
    for (int nk = 1; nk <= 3; nk += 2) {
        for (int grid : {1, 400}) {
            // WHILE graph
            cudaGraph_t g;
            cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
            k_reset<<<1, 1, 0, st>>>(ctr);
            cudaStreamCaptureStatus cs;
            cudaGraph_t cg;
            const cudaGraphNode_t* deps;
            size_t nd;
            cudaStreamGetCaptureInfo(st, &cs, nullptr, &cg, &deps, &nd);
            cudaGraphConditionalHandle h;
            cudaGraphConditionalHandleCreate(&h, cg, 1, cudaGraphCondAssignDefault);
            cudaGraphNodeParams prm = {};
            prm.type = cudaGraphNodeTypeConditional;
            prm.conditional.handle = h;
            prm.conditional.type = cudaGraphCondTypeWhile;
            prm.conditional.size = 1;
            cudaGraphNode_t cn;
            cudaGraphAddNode(&cn, cg, deps, nd, &prm);
            cudaStreamUpdateCaptureDependencies(st, &cn, 1, cudaStreamSetCaptureDependencies);
            cudaGraph_t body = prm.conditional.phGraph_out[0];
            cudaStreamBeginCaptureToGraph(cap, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
            for (int i = 0; i < nk; ++i) k_body<<<grid, 128, 0, cap>>>(ctr, N, h, i == nk - 1);
            cudaStreamEndCapture(cap, &body);
            cudaStreamEndCapture(st, &g);
            cudaGraphExec_t ge;
            cudaGraphInstantiate(&ge, g, 0);
            // plain graph with N*nk kernels
            cudaGraph_t g2;
            cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
            for (int i = 0; i < N * nk; ++i) k_plain<<<grid, 128, 0, st>>>(ctr);
            cudaStreamEndCapture(st, &g2);
            cudaGraphExec_t ge2;
            cudaGraphInstantiate(&ge2, g2, 0);
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            for (int w = 0; w < 3; ++w) cudaGraphLaunch(ge, st);
            cudaEventRecord(a, st);
            for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge, st);
            cudaEventRecord(b, st);
            cudaEventSynchronize(b);
            float ms1;
            cudaEventElapsedTime(&ms1, a, b);
            for (int w = 0; w < 3; ++w) cudaGraphLaunch(ge2, st);
            cudaEventRecord(a, st);
            for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge2, st);
            cudaEventRecord(b, st);
            cudaEventSynchronize(b);
            float ms2;
            cudaEventElapsedTime(&ms2, a, b);
            printf("kernels/iter %d grid %4d: WHILE %.2f us/iter (%.2f us/kernel) | plain graph %.2f us/kernel\n", nk,
                   grid, 1e3 * ms1 / (10 * N), 1e3 * ms1 / (10 * N * nk), 1e3 * ms2 / (10 * N * nk));
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
