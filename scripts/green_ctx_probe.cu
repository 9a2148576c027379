// Probe: can runtime-API kernels run in a green-context stream (SM partition) on buffers
// allocated in the primary context, and do they stay on the partition's SMs?
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>

__global__ void k_probe(const float* a, float* b, int n, unsigned* smids) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) b[i] = a[i] * 2.0f;
    if (threadIdx.x == 0) {
        unsigned s;
        asm("mov.u32 %0, %%smid;" : "=r"(s));
        atomicOr(&smids[s / 32], 1u << (s % 32));
    }
}

#define CKD(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* m; cuGetErrorString(r, &m); printf("%s -> %s\n", #x, m); return 1; } } while (0)
#define CKR(x) do { cudaError_t r = (x); if (r != cudaSuccess) { printf("%s -> %s\n", #x, cudaGetErrorString(r)); return 1; } } while (0)

int main() {
    CKR(cudaSetDevice(0));
    CKR(cudaFree(0));
    const int n = 1 << 24;
    float *a, *b;
    unsigned* sm;
    CKR(cudaMalloc(&a, n * 4));
    CKR(cudaMalloc(&b, n * 4));
    CKR(cudaMallocManaged(&sm, 64));
    CKR(cudaMemset(a, 0, n * 4));
    CUdevice dev;
    CKD(cuDeviceGet(&dev, 0));
    CUdevResource all;
    CKD(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
    printf("SMs in device resource: %u\n", all.sm.smCount);
    CUdevResource groups[2], rest;
    unsigned ng = 1;
    CKD(cuDevSmResourceSplitByCount(groups, &ng, &all, &rest, 0, 96));
    printf("group0 %u SMs, remaining %u SMs\n", groups[0].sm.smCount, rest.sm.smCount);
    CUdevResourceDesc d0, d1;
    CKD(cuDevResourceGenerateDesc(&d0, &groups[0], 1));
    CKD(cuDevResourceGenerateDesc(&d1, &rest, 1));
    CUgreenCtx g0, g1;
    CKD(cuGreenCtxCreate(&g0, d0, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CKD(cuGreenCtxCreate(&g1, d1, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CUstream s0, s1;
    CKD(cuGreenCtxStreamCreate(&s0, g0, CU_STREAM_NON_BLOCKING, 0));
    CKD(cuGreenCtxStreamCreate(&s1, g1, CU_STREAM_NON_BLOCKING, 0));
    for (int part = 0; part < 2; ++part) {
        for (int i = 0; i < 16; ++i) sm[i] = 0;
        k_probe<<<(n + 255) / 256, 256, 0, part ? (cudaStream_t)s1 : (cudaStream_t)s0>>>(a, b, n, sm);
        cudaError_t e = cudaGetLastError();
        printf("launch in partition %d: %s\n", part, cudaGetErrorString(e));
        e = cudaStreamSynchronize(part ? (cudaStream_t)s1 : (cudaStream_t)s0);
        printf("sync: %s\n", cudaGetErrorString(e));
        int cnt = 0;
        for (int i = 0; i < 8; ++i) cnt += __builtin_popcount(sm[i]);
        printf("partition %d kernel ran on %d distinct SMs\n", part, cnt);
    }
    return 0;
}
