// sort.cuh — hand-written device primitives: exclusive scan and stable LSD radix sort.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace tk {

size_t align_bytes(size_t b);  // round up to 256 B

// measured fp64 FMA instructions per second of the device (throughput probe, ~30 ms)
double measure_fp64_fma_rate(cudaStream_t st);

// words x 8 bytes from device memory into host-mapped (cudaHostAllocMapped) memory, by a kernel
void copy_words_to_mapped(void* dst_mapped, const void* src, int words, cudaStream_t st);

// Scratch bytes needed by scan_exclusive for n elements.
size_t scan_scratch_bytes(int64_t n);
// out[i] = sum(in[0..i)), out may alias nothing; *total (device, int64) = sum(in).
// Launches 3 kernels.  in/out int32 (callers check *total against INT32_MAX).
void scan_exclusive(const int32_t* in, int32_t* out, int64_t n, int64_t* total, void* scratch,
                    cudaStream_t st);

// Stable LSD radix sort of (key, value) pairs over key bits [begin_bit, end_bit), 8 bits per
// pass.  Results end in keys_out/vals_out (buffers are ping-ponged internally; the *_alt
// buffers are scratch of the same size).  Onesweep: one all-pass digit histogram, then one
// scatter per pass whose blocks find their digit offsets by decoupled look-back (n < 2^30;
// TK_RADIX_LEGACY=1 or larger n: per-pass histogram + scan + scatter).
size_t radix_scratch_bytes(int64_t n);
void radix_sort_pairs_u64(uint64_t* keys, uint32_t* vals, uint64_t* keys_alt, uint32_t* vals_alt,
                          int64_t n, int begin_bit, int end_bit, void* scratch, cudaStream_t st,
                          bool* result_in_alt);
void radix_sort_pairs_u32(uint32_t* keys, uint32_t* vals, uint32_t* keys_alt, uint32_t* vals_alt,
                          int64_t n, int begin_bit, int end_bit, void* scratch, cudaStream_t st,
                          bool* result_in_alt);

// After sorting bits >= lo_bit only: order runs of equal high bits by (key, value).  Sets
// *overflow (device int) when a run exceeds 64 keys; the caller then sorts all bits.
void fixup_runs_u64(uint64_t* keys, uint32_t* vals, int64_t n, int lo_bit, int32_t* overflow, cudaStream_t st);

// offsets[g] = first index i with keys[i] >= g, for g in [0, n_segments]; keys sorted ascending.
void segment_offsets_u32(const uint32_t* keys, int64_t n, int32_t* offsets, int64_t n_segments,
                         cudaStream_t st);

}  // namespace tk
