// Expert migration (K11): apply a planned slot swap (apply_swap, swap.py:255-259;
// Placement.swapped, routing.py:129-133) to the physical expert state.
//
// An expert store keeps, per GPU, n_arrays tensors laid out slot-major
// ([slots_per_gpu][slice_bytes[a]]: bf16 weights, fp32 master copy, Adam m/v,
// ...), inside one CUDA-IPC region mapped by every peer.  Swapping global
// slots r and c:
//   same GPU      one kernel swaps the two slices of every array in place;
//   two GPUs      each owner pushes its slot's slices into the partner's
//                 staging area with 16-B peer stores (NVLink), a pair barrier
//                 (release/acquire flags, bounded), then each commits staging
//                 into its own slot.  Other GPUs only advance the epoch.
//                 Every GPU has one staging record PER SOURCE GPU: chained
//                 swaps that share a GPU (0<->1 then 0<->2) can never
//                 overwrite a record before its owner committed it, because a
//                 record is only reused by the same partner, which first has
//                 to pass the previous swap's second pair barrier.
// The reference has no cost model for this step.

#include "hm_common.cuh"

#include <string.h>
#include <vector>

namespace {

using namespace hm;

constexpr int kMaxArrays = 16;
constexpr int kMaxGpus = 64;

struct StoreDev {
  int P, p, S, n;                       // gpus, my index, slots per gpu, arrays
  int64_t slice[kMaxArrays];            // bytes per slot, per array
  int64_t arr_off[kMaxArrays];          // array offsets in a region
  int64_t staging_off, flags_off;       // staging: [P][rec] records, one per source GPU
  int64_t rec;                          // bytes of one slot across all arrays
  uint8_t* base[kMaxGpus];              // region base per GPU (peer-mapped)
};

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// copy slot `slot` (local index) of every array to a contiguous destination
__global__ void k_push(const StoreDev* __restrict__ sp, int slot, uint8_t* __restrict__ dst) {
  const StoreDev& s = *sp;
  const uint8_t* mine = s.base[s.p];
  int64_t doff = 0;
  for (int a = 0; a < s.n; ++a) {
    const int4* src = reinterpret_cast<const int4*>(mine + s.arr_off[a] + (int64_t)slot * s.slice[a]);
    int4* d = reinterpret_cast<int4*>(dst + doff);
    const int64_t nv = s.slice[a] / 16;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv;
         i += (int64_t)gridDim.x * blockDim.x)
      d[i] = src[i];
    doff += s.slice[a];
  }
}

__global__ void k_commit(const StoreDev* __restrict__ sp, int slot, int partner) {
  const StoreDev& s = *sp;
  uint8_t* mine = s.base[s.p];
  const uint8_t* stg = mine + s.staging_off + (int64_t)partner * s.rec;
  int64_t soff = 0;
  for (int a = 0; a < s.n; ++a) {
    int4* d = reinterpret_cast<int4*>(mine + s.arr_off[a] + (int64_t)slot * s.slice[a]);
    const int4* src = reinterpret_cast<const int4*>(stg + soff);
    const int64_t nv = s.slice[a] / 16;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv;
         i += (int64_t)gridDim.x * blockDim.x)
      d[i] = src[i];
    soff += s.slice[a];
  }
}

__global__ void k_swap_local(const StoreDev* __restrict__ sp, int a_slot, int b_slot) {
  const StoreDev& s = *sp;
  uint8_t* mine = s.base[s.p];
  for (int a = 0; a < s.n; ++a) {
    int4* x = reinterpret_cast<int4*>(mine + s.arr_off[a] + (int64_t)a_slot * s.slice[a]);
    int4* y = reinterpret_cast<int4*>(mine + s.arr_off[a] + (int64_t)b_slot * s.slice[a]);
    const int64_t nv = s.slice[a] / 16;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv;
         i += (int64_t)gridDim.x * blockDim.x) {
      int4 t = x[i];
      x[i] = y[i];
      y[i] = t;
    }
  }
}

__global__ void k_pair_barrier(const StoreDev* __restrict__ sp, int partner,
                               unsigned long long epoch, int* status) {
  const StoreDev& s = *sp;
  if (threadIdx.x || blockIdx.x) return;
  __threadfence_system();
  unsigned long long* theirs =
      reinterpret_cast<unsigned long long*>(s.base[partner] + s.flags_off) + s.p;
  st_release_sys(theirs, epoch);
  const unsigned long long* mine =
      reinterpret_cast<const unsigned long long*>(s.base[s.p] + s.flags_off) + partner;
  uint64_t t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (ld_acquire_sys(mine) < epoch) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (t1 - t0 > 20000000000ull) {
      atomicExch(status, 3);
      break;
    }
    __nanosleep(100);
  }
}

}  // namespace

struct hm_store {
  StoreDev h;
  StoreDev* d = nullptr;
  uint8_t* region = nullptr;
  size_t bytes = 0;
  std::vector<void*> opened;
  unsigned long long epoch = 0;
  int* status = nullptr;
};

static size_t al(size_t x) { return (x + 255) / 256 * 256; }

HM_API int hm_store_create(int32_t gpus, int32_t gpu_index, int32_t slots_per_gpu,
                           const int64_t* slice_bytes, int32_t n_arrays, hm_store** out) {
  HM_CHECK_ARG(out && slice_bytes, "hm_store_create: null argument");
  HM_CHECK_ARG(gpus >= 1 && gpus <= kMaxGpus && gpu_index >= 0 && gpu_index < gpus,
               "hm_store_create: bad gpu count/index");
  HM_CHECK_ARG(n_arrays >= 1 && n_arrays <= kMaxArrays, "hm_store_create: 1..%d arrays", kMaxArrays);
  HM_CHECK_ARG(slots_per_gpu >= 1, "hm_store_create: slots_per_gpu >= 1");
  for (int a = 0; a < n_arrays; ++a)
    HM_CHECK_ARG(slice_bytes[a] > 0 && slice_bytes[a] % 16 == 0,
                 "hm_store_create: slice sizes must be positive multiples of 16 bytes");
  hm_store* s = new hm_store();
  memset(&s->h, 0, sizeof(s->h));
  s->h.P = gpus;
  s->h.p = gpu_index;
  s->h.S = slots_per_gpu;
  s->h.n = n_arrays;
  size_t o = 0, rec = 0;
  for (int a = 0; a < n_arrays; ++a) {
    s->h.slice[a] = slice_bytes[a];
    s->h.arr_off[a] = (int64_t)o;
    o = al(o + (size_t)slots_per_gpu * slice_bytes[a]);
    rec += slice_bytes[a];
  }
  s->h.staging_off = (int64_t)o;
  s->h.rec = (int64_t)rec;
  o = al(o + (size_t)gpus * rec);
  s->h.flags_off = (int64_t)o;
  o = al(o + (size_t)gpus * 8);
  s->bytes = o;
  int st = cuda_status(cudaMalloc(&s->region, s->bytes));
  if (!st) st = cuda_status(cudaMemset(s->region + s->h.flags_off, 0, (size_t)gpus * 8));
  if (!st) st = cuda_status(cudaMalloc(&s->status, 16));
  if (!st) st = cuda_status(cudaMemset(s->status, 0, 16));
  if (!st) st = cuda_status(cudaMalloc(&s->d, sizeof(StoreDev)));
  s->h.base[gpu_index] = s->region;
  if (!st && gpus == 1) st = cuda_status(cudaMemcpy(s->d, &s->h, sizeof(StoreDev), cudaMemcpyHostToDevice));
  if (st) {
    cudaFree(s->region);
    delete s;
    return st;
  }
  *out = s;
  return 0;
}

HM_API int hm_store_destroy(hm_store* s) {
  if (!s) return 0;
  for (void* p : s->opened) cudaIpcCloseMemHandle(p);
  cudaFree(s->region);
  cudaFree(s->status);
  cudaFree(s->d);
  delete s;
  return 0;
}

HM_API int hm_store_ipc_handle(hm_store* s, void* out_handle) {
  HM_CHECK_ARG(s && out_handle, "hm_store_ipc_handle: null argument");
  cudaIpcMemHandle_t h;
  HM_CUDA(cudaIpcGetMemHandle(&h, s->region));
  memcpy(out_handle, &h, sizeof(h));
  return 0;
}

HM_API int hm_store_open_peers(hm_store* s, const void* handles) {
  HM_CHECK_ARG(s && handles, "hm_store_open_peers: null argument");
  const cudaIpcMemHandle_t* hs = reinterpret_cast<const cudaIpcMemHandle_t*>(handles);
  for (int q = 0; q < s->h.P; ++q) {
    if (q == s->h.p) continue;
    void* b = nullptr;
    HM_CUDA(cudaIpcOpenMemHandle(&b, hs[q], cudaIpcMemLazyEnablePeerAccess));
    s->opened.push_back(b);
    s->h.base[q] = reinterpret_cast<uint8_t*>(b);
  }
  HM_CUDA(cudaMemcpy(s->d, &s->h, sizeof(StoreDev), cudaMemcpyHostToDevice));
  return 0;
}

// device pointer of array a on this GPU ([slots_per_gpu][slice bytes])
HM_API int hm_store_array(hm_store* s, int32_t a, void** ptr) {
  HM_CHECK_ARG(s && ptr && a >= 0 && a < s->h.n, "hm_store_array: bad argument");
  *ptr = s->region + s->h.arr_off[a];
  return 0;
}

HM_API int hm_store_status(hm_store* s, int32_t* out4) {
  HM_CHECK_ARG(s && out4, "hm_store_status: null argument");
  HM_CUDA(cudaMemcpy(out4, s->status, 16, cudaMemcpyDeviceToHost));
  return 0;
}

// Swap global slots r and c (slot s lives on GPU s / slots_per_gpu).  Every
// GPU calls this with the same pair (SPMD); stream-ordered, no host sync.
HM_API int hm_migrate(hm_store* s, int32_t slot_r, int32_t slot_c, void* stream) {
  HM_RANGE("hm_migrate");
  HM_CHECK_ARG(s, "hm_migrate: null store");
  const int total = s->h.P * s->h.S;
  HM_CHECK_ARG(slot_r >= 0 && slot_c >= 0 && slot_r < total && slot_c < total,
               "hm_migrate: slot out of range");
  cudaStream_t st = (cudaStream_t)stream;
  const int gr = slot_r / s->h.S, gc = slot_c / s->h.S, me = s->h.p;
  const unsigned long long ep = ++s->epoch;
  if (slot_r == slot_c) return 0;
  const int blocks = kSMs * 4;
  if (gr == gc) {
    if (me == gr) {
      k_swap_local<<<blocks, 256, 0, st>>>(s->d, slot_r % s->h.S, slot_c % s->h.S);
      HM_LAUNCHED();
    }
    return 0;
  }
  if (me != gr && me != gc) return 0;
  const int mine = me == gr ? slot_r : slot_c;
  const int partner = me == gr ? gc : gr;
  // my record in the partner's staging area, written through the peer mapping (NVLink)
  uint8_t* dst = s->h.base[partner] + s->h.staging_off + (int64_t)me * s->h.rec;
  k_push<<<blocks, 256, 0, st>>>(s->d, mine % s->h.S, dst);
  HM_LAUNCHED();
  k_pair_barrier<<<1, 32, 0, st>>>(s->d, partner, 2 * ep - 1, s->status);
  HM_LAUNCHED();
  k_commit<<<blocks, 256, 0, st>>>(s->d, mine % s->h.S, partner);
  HM_LAUNCHED();
  // a second pair barrier so the partner may not reuse our staging early
  k_pair_barrier<<<1, 32, 0, st>>>(s->d, partner, 2 * ep, s->status);
  HM_LAUNCHED();
  return 0;
}
