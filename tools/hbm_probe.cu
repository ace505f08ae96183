// HBM ceilings for the pack / gather access patterns on one B200:
//   copy        1 read : 1 write, sequential 4 KB rows
//   write       write-only, sequential rows
//   bcast8      1 read : 8 writes, each token row to 8 rows spread over the
//               destination buffer (the pack's expert-major pattern)
//   gather8     8 reads : 1 write, the mirror (the combine's gather pattern)
// GB/s = bytes moved / kernel time (best of 5, CUDA events).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/hbm_probe tools/hbm_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

constexpr int kRow = 4096;

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

__global__ void k_copy(const int4* __restrict__ src, int4* __restrict__ dst, int64_t rows) {
  const int lane = threadIdx.x & 31;
  int64_t w = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5), nw = (int64_t)gridDim.x * 8;
  for (int64_t r = w; r < rows; r += nw) {
    int4 v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __ldg(src + r * 256 + i * 32 + lane);
#pragma unroll
    for (int i = 0; i < 8; ++i) dst[r * 256 + i * 32 + lane] = v[i];
  }
}

__global__ void k_write(int4* __restrict__ dst, int64_t rows) {
  const int lane = threadIdx.x & 31;
  int64_t w = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5), nw = (int64_t)gridDim.x * 8;
  const int4 z = make_int4(1, 2, 3, 4);
  for (int64_t r = w; r < rows; r += nw)
#pragma unroll
    for (int i = 0; i < 8; ++i) dst[r * 256 + i * 32 + lane] = z;
}

// token t -> 8 destination rows spread over [0, 8 * tokens)
__device__ __forceinline__ int64_t dest_row(int64_t t, int k, int64_t tokens) {
  return ((int64_t)k * tokens + (int64_t)(hash32((uint32_t)(t * 8 + k)) % (uint32_t)tokens));
}

__global__ void k_bcast8(const int4* __restrict__ src, int4* __restrict__ dst, int64_t tokens) {
  const int lane = threadIdx.x & 31;
  int64_t w = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5), nw = (int64_t)gridDim.x * 8;
  for (int64_t t = w; t < tokens; t += nw) {
    int4 v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __ldg(src + t * 256 + i * 32 + lane);
    for (int k = 0; k < 8; ++k) {
      int4* d = dst + dest_row(t, k, tokens) * 256;
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(d + i * 32 + lane),
                     "r"(v[i].x), "r"(v[i].y), "r"(v[i].z), "r"(v[i].w));
    }
  }
}

__global__ void k_gather8(const int4* __restrict__ src, int4* __restrict__ dst, int64_t tokens) {
  const int lane = threadIdx.x & 31;
  int64_t w = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5), nw = (int64_t)gridDim.x * 8;
  for (int64_t t = w; t < tokens; t += nw) {
    for (int c = 0; c < 8; c += 2) {
      int4 acc[2] = {make_int4(0, 0, 0, 0), make_int4(0, 0, 0, 0)};
      int4 v[8][2];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int4* s = src + dest_row(t, k, tokens) * 256;
#pragma unroll
        for (int u = 0; u < 2; ++u) v[k][u] = __ldg(s + (c + u) * 32 + lane);
      }
#pragma unroll
      for (int k = 0; k < 8; ++k)
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          acc[u].x ^= v[k][u].x;
          acc[u].y ^= v[k][u].y;
          acc[u].z ^= v[k][u].z;
          acc[u].w ^= v[k][u].w;
        }
#pragma unroll
      for (int u = 0; u < 2; ++u) dst[t * 256 + (c + u) * 32 + lane] = acc[u];
    }
  }
}

int main() {
  const int64_t tokens = 32768;               // the Qwen3 N = 1 step
  int4 *x, *big;
  cudaMalloc(&x, tokens * kRow);
  cudaMalloc(&big, 8 * tokens * kRow);
  cudaMemset(x, 1, tokens * kRow);
  cudaMemset(big, 2, 8 * tokens * kRow);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int grids[] = {148 * 4, 148 * 8, 148 * 16};
  printf("{\"rows\": %lld", (long long)tokens);
  for (int kind = 0; kind < 4; ++kind) {
    for (int gi = 0; gi < 3; ++gi) {
      float best = 1e30f;
      for (int rep = 0; rep < 6; ++rep) {
        cudaEventRecord(e0);
        if (kind == 0) k_copy<<<grids[gi], 256>>>(x, big, tokens);
        if (kind == 1) k_write<<<grids[gi], 256>>>(big, 8 * tokens);
        if (kind == 2) k_bcast8<<<grids[gi], 256>>>(x, big, tokens);
        if (kind == 3) k_gather8<<<grids[gi], 256>>>(big, x, tokens);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep && ms < best) best = ms;
      }
      const double bytes = kind == 0 ? 2.0 * tokens * kRow
                           : kind == 1 ? 8.0 * tokens * kRow
                                       : 9.0 * tokens * kRow;
      const char* names[] = {"copy", "write", "bcast8", "gather8"};
      printf(", \"%s_%d\": %.1f", names[kind], grids[gi], bytes / (best * 1e-3) / 1e9);
    }
  }
  printf("}\n");
  return cudaGetLastError() != cudaSuccess;
}
