// fp64_peak.cu — measured FP64 roof of this B200 (BASELINE.md §2's secondary
// roof for the FV1 kernel): DFMA, DADD and DMUL issue rates of a kernel made
// of long runs of independent FP64 operations (8 chains per thread, every SM
// full), timed with CUDA events, best of 5. Prints one JSON line.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu && ./fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void __launch_bounds__(256) k_fp64(double* out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                if (OP == 0) x[k] = __fma_rn(x[k], a, b);
                else if (OP == 1) x[k] = __dadd_rn(x[k], b);
                else x[k] = __dmul_rn(x[k], a);
            }
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 12345.678) out[0] = s;  // keep the chains alive
}

template <int OP>
double rate(int sms) {  // operations (thread instructions) per second
    double* d;
    cudaMalloc(&d, 8);
    const int blocks = sms * 8, iters = 2048;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_fp64<OP><<<blocks, 256>>>(d, 16, 1.0000001, 1e-9);
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        k_fp64<OP><<<blocks, 256>>>(d, iters, 1.0000001, 1e-9);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaFree(d);
    return double(blocks) * 256 * iters * 16 * 8 / (best * 1e-3);
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    const double fma = rate<0>(p.multiProcessorCount), add = rate<1>(p.multiProcessorCount),
                 mul = rate<2>(p.multiProcessorCount);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("{\"gpu\": \"%s\", \"sms\": %d, \"dfma_per_s\": %.4e, \"dadd_per_s\": %.4e, \"dmul_per_s\": %.4e, "
           "\"fp64_tflops_fma\": %.3f, \"dfma_per_clk_per_sm_at_max\": %.2f}\n",
           p.name, p.multiProcessorCount, fma, add, mul, 2.0 * fma * 1e-12,
           fma / (p.multiProcessorCount * clk * 1e3));
    return 0;
}
