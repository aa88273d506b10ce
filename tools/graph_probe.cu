// Probe: cost of a graph launch with 3 full-GPU kernel nodes (391 CTAs each,
// trivial bodies), launched back to back, against the same kernels launched
// directly.  nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/graph_probe.cu -o tools/graph_probe
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_noop(int* p, int v) {
    if (threadIdx.x == 0 && blockIdx.x == 0 && v < 0) *p = v;
}
struct Big { char pad[900]; };  // kernel parameters of the size the Lloyd kernels pass
__global__ void k_noop_big(int* p, const __grid_constant__ Big b) {
    if (threadIdx.x == 0 && blockIdx.x == 0 && b.pad[0] == 42) *p = 1;
}
int main() {
    int* d;
    cudaMalloc(&d, 4);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    Big big{};
    for (int variant = 0; variant < 2; ++variant) {
        cudaGraph_t g;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
        for (int i = 0; i < 3; ++i) {
            if (variant == 0) k_noop<<<391, 256, 0, s>>>(d, i);
            else k_noop_big<<<391, 256, 0, s>>>(d, big);
        }
        cudaStreamEndCapture(s, &g);
        cudaGraphExec_t e;
        cudaGraphInstantiate(&e, g, 0);
        for (int w = 0; w < 20; ++w) cudaGraphLaunch(e, s);
        cudaStreamSynchronize(s);
        const int N = 400;
        cudaEventRecord(a, s);
        for (int r = 0; r < N; ++r) cudaGraphLaunch(e, s);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("graph of 3 kernels (%s params): %.2f us per graph launch\n", variant ? "900-byte" : "small",
               1e3 * ms / N);
        cudaEventRecord(a, s);
        for (int r = 0; r < N; ++r)
            for (int i = 0; i < 3; ++i) {
                if (variant == 0) k_noop<<<391, 256, 0, s>>>(d, i);
                else k_noop_big<<<391, 256, 0, s>>>(d, big);
            }
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("3 direct launches (%s params): %.2f us per group\n", variant ? "900-byte" : "small", 1e3 * ms / N);
    }
    return 0;
}
