// NVLink write-path probe: all-to-all pushes of 4 KB rows from every GPU to
// every other GPU of the box, three ways:
//   st    warps copy rows with 16-B loads + 16-B stores to peer memory
//   bulk  warps stage rows in shared memory (16-B loads) and push them with
//         cp.async.bulk shared -> global (TMA bulk store) to peer memory
//   copy  cudaMemcpyPeerAsync, one stream per peer
// Prints GB/s per direction per GPU (bytes leaving one GPU / its kernel time).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/link_probe tools/link_probe.cu
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
#include <vector>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return 1;                                                                \
    }                                                                          \
  } while (0)

constexpr int kRow = 4096;
constexpr int kMaxGpus = 8;
struct Peers {
  uint8_t* dst[kMaxGpus];   // destination buffer on each GPU (this GPU's slice)
};

__global__ void k_st(const uint8_t* __restrict__ src, Peers p, int P, int me, int64_t rows) {
  const int lane = threadIdx.x & 31;
  int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = w; r < rows; r += nw) {
    int peer = (int)(r % (P - 1));
    peer += peer >= me;
    const int4* s = reinterpret_cast<const int4*>(src + r * kRow);
    int4* d = reinterpret_cast<int4*>(p.dst[peer] + r * kRow);
    int4 v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __ldg(s + i * 32 + lane);
#pragma unroll
    for (int i = 0; i < 8; ++i) d[i * 32 + lane] = v[i];
  }
}

__device__ __forceinline__ uint32_t sa(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// one 4 KB smem slot per warp x 2; bulk store from smem to the peer
__global__ void k_bulk(const uint8_t* __restrict__ src, Peers p, int P, int me, int64_t rows) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint8_t* slot0 = sm + (size_t)wid * 2 * kRow;
  int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + wid;
  int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  int it = 0;
  for (int64_t r = w; r < rows; r += nw, ++it) {
    uint8_t* slot = slot0 + (it & 1) * kRow;
    // the bulk store issued from this slot two iterations ago must have read it
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncwarp();
    int peer = (int)(r % (P - 1));
    peer += peer >= me;
    const int4* s = reinterpret_cast<const int4*>(src + r * kRow);
    int4 v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __ldg(s + i * 32 + lane);
#pragma unroll
    for (int i = 0; i < 8; ++i) reinterpret_cast<int4*>(slot)[i * 32 + lane] = v[i];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                       p.dst[peer] + r * kRow),
                   "r"(sa(slot)), "r"(kRow)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
  int P = 0;
  CK(cudaGetDeviceCount(&P));
  if (P < 2) {
    printf("{\"error\": \"needs >= 2 GPUs\"}\n");
    return 0;
  }
  if (P > kMaxGpus) P = kMaxGpus;
  const int64_t rows = (argc > 1) ? atoll(argv[1]) : 65536;   // rows pushed per GPU
  std::vector<uint8_t*> src(P), dst(P);
  std::vector<cudaStream_t> st(P);
  std::vector<cudaEvent_t> e0(P), e1(P);
  for (int g = 0; g < P; ++g) {
    CK(cudaSetDevice(g));
    for (int q = 0; q < P; ++q)
      if (q != g) {
        cudaError_t e = cudaDeviceEnablePeerAccess(q, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
      }
    cudaGetLastError();
    CK(cudaMalloc(&src[g], rows * kRow));
    CK(cudaMalloc(&dst[g], (size_t)P * rows * kRow));
    CK(cudaMemset(src[g], g + 1, rows * kRow));
    CK(cudaStreamCreateWithFlags(&st[g], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[g]));
    CK(cudaEventCreate(&e1[g]));
  }
  auto sync_all = [&]() {
    for (int g = 0; g < P; ++g) {
      cudaSetDevice(g);
      cudaDeviceSynchronize();
    }
  };
  const int smem = 8 * 2 * kRow;
  for (int g = 0; g < P; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  }
  printf("{\"gpus\": %d, \"rows_per_gpu\": %lld, \"row_bytes\": %d", P, (long long)rows, kRow);
  const char* names[] = {"st", "bulk", "copy"};
  const int ctas_opts[] = {148, 296, 592, 1184};
  for (int mode = 0; mode < 3; ++mode) {
    for (int ci = 0; ci < (mode == 2 ? 1 : 4); ++ci) {
      const int ctas = ctas_opts[ci];
      float best = 1e30f;
      for (int rep = 0; rep < 6; ++rep) {
        sync_all();
        for (int g = 0; g < P; ++g) {
          cudaSetDevice(g);
          Peers p;
          for (int q = 0; q < P; ++q) p.dst[q] = dst[q] + (size_t)g * rows * kRow;
          cudaEventRecord(e0[g], st[g]);
          if (mode == 0)
            k_st<<<ctas, 256, 0, st[g]>>>(src[g], p, P, g, rows);
          else if (mode == 1)
            k_bulk<<<ctas, 256, smem, st[g]>>>(src[g], p, P, g, rows);
          else {
            int64_t per = rows / (P - 1);
            for (int q = 0, k = 0; q < P; ++q) {
              if (q == g) continue;
              cudaMemcpyPeerAsync(p.dst[q] + k * per * kRow, q, src[g] + k * per * kRow, g,
                                  per * kRow, st[g]);
              ++k;
            }
          }
          cudaEventRecord(e1[g], st[g]);
        }
        float worst = 0.f;
        for (int g = 0; g < P; ++g) {
          cudaSetDevice(g);
          CK(cudaEventSynchronize(e1[g]));
          float ms = 0.f;
          cudaEventElapsedTime(&ms, e0[g], e1[g]);
          worst = ms > worst ? ms : worst;
        }
        CK(cudaGetLastError());
        if (rep > 0 && worst < best) best = worst;
      }
      printf(", \"%s_%d\": %.1f", names[mode], mode == 2 ? 0 : ctas,
             (double)rows * kRow / (best * 1e-3) / 1e9);
    }
  }
  printf("}\n");
  return 0;
}
