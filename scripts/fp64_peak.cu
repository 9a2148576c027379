// Measured fp64 FMA throughput of this B200 (the roofline denominator of the fp64-bound geometric
// sweeps): 8 independent DFMA chains per thread, 148 x 8 blocks of 256 threads, CUDA events.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/fp64_peak.cu -o /tmp/fp64 && /tmp/fp64
#include <cstdio>

__global__ void k_dfma(double* out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-3 + j;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = fma(x[j], a, b);
    double s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += x[j];
    if (s == 12345.678) out[0] = s;
}

int main() {
    double* out;
    cudaMalloc(&out, 8);
    const int blocks = 148 * 8, threads = 256, iters = 1 << 14;
    k_dfma<<<blocks, threads>>>(out, 16, 0.999, 1e-3);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        k_dfma<<<blocks, threads>>>(out, iters, 0.999, 1e-3);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    const double fma = static_cast<double>(blocks) * threads * iters * 8;
    printf("{\"fp64_fma_per_s\": %.4e, \"fp64_tflops\": %.2f, \"dp_instr_per_s\": %.4e}\n", fma / (best / 1e3),
           2 * fma / (best / 1e3) / 1e12, fma / (best / 1e3));
    return 0;
}
