// membw.cu — HBM write / read / copy ceilings on this B200 for the store flavours the
// feature kernels use (measurement aid; not part of the product library).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_write(float4* out, size_t n4, int mode) {
    const float4 v = make_float4(1.f, 2.f, 3.f, 4.f);
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
        if (mode == 0) out[i] = v;
        else if (mode == 1) __stcs(out + i, v);
        else __stwt(out + i, v);
    }
}

__global__ void k_read(const float4* in, size_t n4, float* sink) {
    float4 a = make_float4(0, 0, 0, 0);
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
        const float4 v = __ldg(in + i);
        a.x += v.x; a.y += v.y; a.z += v.z; a.w += v.w;
    }
    if (a.x + a.y + a.z + a.w == 12345.f) *sink = a.x;
}

__global__ void k_copy(const float4* in, float4* out, size_t n4) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
        __stcs(out + i, __ldg(in + i));
}

int main() {
    const size_t bytes = 1632000000ull;  // = config-3 F map (816000 x 512 x 4)
    const size_t n4 = bytes / 16;
    float4 *a, *b;
    float* sink;
    cudaMalloc(&a, bytes);
    cudaMalloc(&b, bytes);
    cudaMalloc(&sink, 4);
    cudaMemset(a, 0, bytes);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char* names[] = {"write st.global", "write st.cs", "write st.wt"};
    for (int grid : {148 * 8, 148 * 32}) {
        for (int mode = 0; mode < 3; ++mode) {
            float best = 1e9f;
            for (int r = 0; r < 5; ++r) {
                cudaEventRecord(e0);
                k_write<<<grid, 256>>>(b, n4, mode);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                best = ms < best ? ms : best;
            }
            printf("grid %5d %-16s %8.1f GB/s\n", grid, names[mode], bytes / best / 1e6);
        }
        float best = 1e9f;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0);
            k_read<<<grid, 256>>>(a, n4, sink);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = ms < best ? ms : best;
        }
        printf("grid %5d %-16s %8.1f GB/s\n", grid, "read ld.nc", bytes / best / 1e6);
        best = 1e9f;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0);
            k_copy<<<grid, 256>>>(a, b, n4);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = ms < best ? ms : best;
        }
        printf("grid %5d %-16s %8.1f GB/s (read+write)\n", grid, "copy", 2 * bytes / best / 1e6);
    }
    float best = 1e9f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        cudaMemsetAsync(b, 0, bytes);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    printf("cudaMemset %8.1f GB/s\n", bytes / best / 1e6);
    return 0;
}
