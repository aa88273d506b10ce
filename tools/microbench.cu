// Micro-benchmarks of the pipes the Big-means kernels lean on (sm_100a).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dadd_chain(double* out, double a, int iters, long long* cyc) {
    double s = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) s = __dadd_rn(s, a);
    long long t1 = clock64();
    if (threadIdx.x == 0) { *cyc = t1 - t0; }
    out[threadIdx.x] = s;
}
__global__ void ffma_chain(float* out, float a, int iters, long long* cyc) {
    float s = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) s = __fmaf_rn(s, a, a);
    long long t1 = clock64();
    if (threadIdx.x == 0) { *cyc = t1 - t0; }
    out[threadIdx.x] = s;
}
template <int CH>
__global__ void dfp_tput(double* out, double a, int iters) {
    double s[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) s[c] = threadIdx.x + c;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int c = 0; c < CH; ++c) { double d = __dsub_rn(s[c], a); s[c] = __dadd_rn(s[c], __dmul_rn(d, d)); }
    double t = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) t += s[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
template <int CH>
__global__ void ffp_tput(float* out, float a, int iters) {
    float s[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) s[c] = threadIdx.x + c;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int c = 0; c < CH; ++c) { float d = __fsub_rn(s[c], a); s[c] = __fmaf_rn(d, d, s[c]); }
    float t = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) t += s[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
__global__ void cvt_tput(float* out, const double* in, int iters) {
    double v = in[threadIdx.x];
    float acc = 0;
    for (int i = 0; i < iters; ++i) { acc += __double2float_rn(v); v += 1.0; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
    double* d; float* f; long long* c; double* in;
    cudaMalloc(&d, 1 << 26); cudaMalloc(&f, 1 << 26); cudaMalloc(&c, 8); cudaMalloc(&in, 1 << 20);
    cudaMemset(in, 0, 1 << 20);
    long long cyc;
    int iters = 4096;
    dadd_chain<<<1, 32>>>(d, 1.0, iters, c); cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
    printf("DADD dependent latency: %.2f cycles\n", (double)cyc / iters);
    ffma_chain<<<1, 32>>>(f, 1.0f, iters, c); cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
    printf("FFMA dependent latency: %.2f cycles\n", (double)cyc / iters);
    int dev; cudaGetDevice(&dev); int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
    dfp_tput<16><<<sms * 4, 256>>>(d, 1.5, 10);
    cudaEventRecord(a); dfp_tput<16><<<sms * 4, 256>>>(d, 1.5, 2000); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    double ops = 3.0 * 16 * 2000 * (double)sms * 4 * 256;
    printf("fp64 sub/mul/add: %.2f Tops/s  (%.1f ops/clk/SM at %d MHz)\n", ops / ms / 1e9, ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
    ffp_tput<16><<<sms * 4, 256>>>(f, 1.5f, 10);
    cudaEventRecord(a); ffp_tput<16><<<sms * 4, 256>>>(f, 1.5f, 2000); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    ops = 2.0 * 16 * 2000 * (double)sms * 4 * 256;
    printf("fp32 sub+fma: %.2f Tinstr/s  (%.1f instr/clk/SM)\n", ops / ms / 1e9, ops / (ms * 1e-3) / sms / (clk * 1e3));
    cudaEventRecord(a); cvt_tput<<<sms * 4, 256>>>(f, in, 2000); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    ops = 2000.0 * sms * 4 * 256;
    printf("f64->f32 cvt (+dadd+fadd): %.2f Gcvt/s  (%.1f /clk/SM)\n", ops / ms / 1e6, ops / (ms * 1e-3) / sms / (clk * 1e3));
    printf("SMs %d clock %d MHz\n", sms, clk / 1000);
    return 0;
}
