// MoE-layer hot path: top-K gating, dedup dispatch, expert-side re-expansion,
// dedup combine -- over a world of G virtual EP ranks hosted on P physical
// GPUs (L = G/P per GPU), connected by CUDA-IPC peer mappings over NVLink.
//
// Step (all stream-ordered on the caller's stream, no host synchronisation):
//   k_plan     per 256-token chunk of every local source rank: destination
//              mask, stable within-chunk ranks per destination and per slot,
//              chunk histograms (G dest + E slot counters)
//   k_notify   one CTA: chunk prefix sums, this GPU's per-source totals
//              (= h[s,:] dedup rows per destination, c[s,:] selections per
//              slot) stored into every peer's count matrix, barrier, derived
//              offsets (receive offsets, expert-major bases, group sizes)
//   k_pack     warp per token: 16-B vector copy of the row into every hit
//              destination's receive buffer (dedup: one copy per destination;
//              raw: one copy per selection straight into expert-major rows),
//              peer stores over NVLink for remote destinations
//   barrier
//   k_expand   (dedup) destination re-expands each received row into its
//              local experts' expert-major rows
//   ... expert FFN on expert-major rows (grouped GEMM) ...
//   k_reduce   (dedup) destination pre-reduces sum_k w_k y_k over its local
//              experts into one row per (token, destination)
//   barrier
//   k_gather   source sums its (token, destination) rows in ascending
//              destination order (dedup) or sum_k w_k y_k (raw), peer loads
//
// Receive order at destination d is the global (rank-major) token order of
// the tokens hitting d: the row-major copy order of propagate_level
// (routing.py:204-215) restricted to d, with h = group_reduce column sums
// (traffic.py:58-71).

#include "hm_common.cuh"
#include "exch.cuh"

#include <cuda_bf16.h>
#include <string.h>
#include <stdlib.h>
#include <type_traits>
#include <vector>

namespace {

using namespace hm;

constexpr int kMaxRanks = 64;
constexpr int kMaxK = 16;
constexpr int kChunk = 256;      // tokens per plan chunk (8 warps x 32)
constexpr int kPlanWarps = kChunk / 32;

struct RowMeta {
  int32_t epos;  // expert-major row at this destination (relay: slot id), -1 if not here
  float w;
};


// device-resident view of the world (pointers valid on this GPU)
struct WorldDev {
  int G, L, P, p, E, K, M, E_loc, elem;
  int e_shift;   // log2(E_loc) when E_loc is a power of two, else -1
  // relay (phase-1 of a two-level dispatch): U1 > 0 groups of F = G/U1 ranks;
  // pick e of source s goes to rank (e / (E/U1)) * F + s % F (the rank with
  // the source's local index inside the pick's group), carrying slot ids
  int U1, F;
  int64_t T_r, R_cap, N_cap, row_bytes;
  uint8_t* recv_x[kMaxRanks];
  RowMeta* recv_meta[kMaxRanks];
  uint8_t* xmaj[kMaxRanks];
  uint8_t* ymaj[kMaxRanks];
  uint8_t* comb[kMaxRanks];
  uint8_t* ret[kMaxRanks];    // per source rank: [G][T_r][M] pre-reduced rows pushed back
  // mode 3 (dedup per destination GPU): per GPU q a receive buffer + meta
  // (epos = local rank * N_cap + expert-major row), per source rank a return
  // buffer [P][T_r][M]
  uint8_t* recv_g[kMaxRanks];
  RowMeta* meta_g[kMaxRanks];
  uint8_t* ret_g[kMaxRanks];
  int64_t Rg_cap;
  uint8_t* gy[kMaxRanks];     // backward: grad of expert outputs (expert-major), or null
  uint8_t* gx[kMaxRanks];     // backward: grad of expert inputs (expert-major), or null
  float* gw[kMaxRanks];       // backward: gate grads of dedup picks [R_cap][K], or null
  int32_t* counts[kMaxRanks];                 // count matrix [G][G+E] on d's GPU
  unsigned long long* flags[kMaxRanks];       // per GPU q: flags[q][0..P)
  // barrier epoch counter (this GPU, device memory): advanced by the device
  // barriers themselves, so a step is replayable from a CUDA graph
  unsigned long long* epoch_ctr;
};

__device__ __forceinline__ int rank_of_slot(const WorldDev& w, int e) {
  return w.e_shift >= 0 ? e >> w.e_shift : e / w.E_loc;
}
__device__ __forceinline__ int dest_of(const WorldDev& w, int s, int e) {
  return w.U1 ? (e / (w.E / w.U1)) * w.F + s % w.F : rank_of_slot(w, e);
}

// per-step offsets computed by k_notify (local, not symmetric)
struct Offsets {
  int32_t off[kMaxRanks][kMaxRanks];  // [local src][dest]  receive offset
  int32_t offd[kMaxRanks][kMaxRanks + 1];  // [local dest][src] receive offset (+ total)
  int32_t off_g[kMaxRanks][kMaxRanks];  // [local src][dest gpu] mode-3 receive offset
  int32_t offd_g[kMaxRanks + 1];        // [src] mode-3 offset of src's rows on this GPU
  int32_t R_g;                          // mode-3 rows received by this GPU
  int32_t R[kMaxRanks];               // rows received per local dest
  int32_t Nd[kMaxRanks];              // expert-major rows per local dest
};

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Called by one full CTA after its peer stores.  Thread 0 advances this GPU's
// epoch counter, publishes the new epoch to every GPU and waits (bounded,
// 20 s) until every GPU published it.  Every GPU issues the same sequence of
// barriers, so the counters agree; keeping the counter on the device (not a
// host-side argument) lets the whole step be captured in a CUDA graph.
__device__ void cta_barrier(const WorldDev& w, int* status) {
  __syncthreads();
  if (threadIdx.x == 0 && w.P > 1) {   // one GPU: nothing to wait for
    const unsigned long long epoch = ++(*w.epoch_ctr);
    {
      __threadfence_system();
      for (int q = 0; q < w.P; ++q) st_release_sys(w.flags[q * w.L] + w.p, epoch);
      unsigned long long* mine = w.flags[w.p * w.L];
      uint64_t t0 = globaltimer();
      for (int q = 0; q < w.P; ++q) {
        while (ld_acquire_sys(mine + q) < epoch) {
          if (globaltimer() - t0 > 20000000000ull) {
            atomicExch(status, 3);  // barrier timeout
            break;
          }
          __nanosleep(64);
        }
      }
    }
  }
  __syncthreads();
}

__global__ void k_barrier(const WorldDev* __restrict__ wp, int* status) {
  cta_barrier(*wp, status);
}

// ---------------------------------------------------------------------------
// K1 router: fp32 logits -> top-K (value desc, index asc) -> softmax weights
// (renormalised over the picks when renorm) -> slot ids via expert_to_slot.
// One warp per token; lanes hold E/32 logits each.
template <int kPerLane>
__global__ void k_route(const float* __restrict__ logits, int64_t T, int E, int K,
                        const int32_t* __restrict__ e2s, int renorm,
                        int32_t* __restrict__ slot_ids, float* __restrict__ weights,
                        int32_t* __restrict__ expert_ids) {
  const int lane = threadIdx.x & 31;
  int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t t = warp; t < T; t += nw) {
    const float* row = logits + t * E;
    float v[kPerLane];
#pragma unroll
    for (int j = 0; j < kPerLane; ++j) {
      int e = j * 32 + lane;
      v[j] = e < E ? row[e] : -INFINITY;
    }
    unsigned taken = 0;
    float vmax = 0.f, sum_all = 0.f;
    float pick_v[kMaxK];
    int pick_e[kMaxK];
    for (int k = 0; k < K; ++k) {
      float bv = -INFINITY;
      int be = 0x7fffffff;
#pragma unroll
      for (int j = 0; j < kPerLane; ++j) {
        int e = j * 32 + lane;
        if (e < E && !(taken & (1u << j)) && (v[j] > bv || (v[j] == bv && e < be))) {
          bv = v[j];
          be = e;
        }
      }
      for (int o = 16; o; o >>= 1) {
        float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        int oe = __shfl_xor_sync(0xffffffffu, be, o);
        if (ov > bv || (ov == bv && oe < be)) {
          bv = ov;
          be = oe;
        }
      }
      if ((be & 31) == lane) taken |= 1u << (be >> 5);
      pick_v[k] = bv;
      pick_e[k] = be;
    }
    vmax = pick_v[0];
    if (!renorm) {
      float s = 0.f;
#pragma unroll
      for (int j = 0; j < kPerLane; ++j)
        if (j * 32 + lane < E) s += expf(v[j] - vmax);
      for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      sum_all = s;
    } else {
      float s = 0.f;
      for (int k = 0; k < K; ++k) s += expf(pick_v[k] - vmax);
      sum_all = s;
    }
    if (lane < K) {
      int k = lane;
      float pv = 0.f;
      int pe = 0;
      for (int q = 0; q < K; ++q)
        if (q == k) {
          pv = pick_v[q];
          pe = pick_e[q];
        }
      weights[t * K + k] = expf(pv - vmax) / sum_all;
      slot_ids[t * K + k] = e2s ? e2s[pe] : pe;
      if (expert_ids) expert_ids[t * K + k] = pe;
    }
  }
}

// K1 router, four lanes per token (E % 16 == 0, E <= 256): a warp takes 8
// tokens; lane j of a token's quad loads float4 columns j, j+4, ... (all in
// flight at once), keeps its sorted top-K (strict > in ascending expert
// order: ties keep the lower index), then the quad merges its four lists
// by two butterfly steps with the same (value desc, index asc) order.  4x
// the warps of the lane-per-token kernel for the same tokens.
// Threshold pre-pass (the kernel is issue-bound on the insertions): each
// lane's two largest float4-group maxima are logits of the token, so the
// quad holds >= 8 >= K logits at or above theta = the smallest of the four
// lanes' second-largest group maxima, and no logit below theta is among the
// top K.  Only the lane's candidates (>= theta, typically 2-4 of 32) are
// inserted, in ascending expert order, read back from the lane's shared-
// memory row; the merged top K is the one the full insertion builds.
// 4-warp CTAs: the grid of 32-token CTAs spreads the (issue-bound) work over
// the SMs in finer steps than 64-token CTAs (at most 28 instead of 32 warp-
// tasks per SM for the Qwen3 step's 4096).
constexpr int kRouteWarps = 4;
template <int K, int F4, int LPT = 4>   // F4 = float4 columns per lane = E / (4 LPT)
__global__ void __launch_bounds__(32 * kRouteWarps) k_route_quad(const float* __restrict__ logits, int64_t T,
                                                    int E, const int32_t* __restrict__ e2s,
                                                    int renorm, int32_t* __restrict__ slot_ids,
                                                    float* __restrict__ weights,
                                                    int32_t* __restrict__ expert_ids) {
  constexpr int TPW = 32 / LPT;   // tokens per warp
  // the pre-pass keeps the lane's logits in a shared-memory row (E <= 128:
  // up to 32 per lane, one 32-bit candidate mask); wider rows insert all
  constexpr bool kPre = 4 * F4 <= 32;
  constexpr int kRow = kPre ? 4 * F4 + 4 : 4;   // row stride (floats): float4 stores conflict-free
  __shared__ float4 s_rows[32 * kRouteWarps * kRow / 4];
  float* row_s = reinterpret_cast<float*>(s_rows) + threadIdx.x * kRow;
  const int lane = threadIdx.x & 31, j = lane & (LPT - 1);
  int64_t warp = (int64_t)blockIdx.x * kRouteWarps + (threadIdx.x >> 5);
  const int64_t nw = (int64_t)gridDim.x * kRouteWarps;
  for (int64_t base = warp * TPW; base < T; base += nw * TPW) {
    const int64_t t = base + lane / LPT;
    const bool live = t < T;
    float4 v[F4];
    const float4* row = reinterpret_cast<const float4*>(logits + (live ? t : 0) * E);
#pragma unroll
    for (int i = 0; i < F4; ++i)
      v[i] = live ? __ldg(row + j + LPT * i)
                  : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
    float tv[K];
    int ti[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      tv[k] = -INFINITY;
      ti[k] = 0x7fffffff;
    }
    auto insert = [&](float x, int e) {
      if (!(x > tv[K - 1])) return;
#pragma unroll
      for (int k = K - 1; k > 0; --k) {
        if (x > tv[k]) {
          const bool up = x > tv[k - 1];
          tv[k] = up ? tv[k - 1] : x;
          ti[k] = up ? ti[k - 1] : e;
        }
      }
      if (x > tv[0]) {
        tv[0] = x;
        ti[0] = e;
      }
    };
    if constexpr (!kPre) {
#pragma unroll
      for (int i = 0; i < F4; ++i) {
        const int e = 4 * (j + LPT * i);
        insert(v[i].x, e);
        insert(v[i].y, e + 1);
        insert(v[i].z, e + 2);
        insert(v[i].w, e + 3);
      }
    } else {
      float m1 = -INFINITY, m2 = -INFINITY;   // the lane's two largest group maxima
#pragma unroll
      for (int i = 0; i < F4; ++i) {
        const float gm = fmaxf(fmaxf(v[i].x, v[i].y), fmaxf(v[i].z, v[i].w));
        m2 = fmaxf(m2, fminf(m1, gm));
        m1 = fmaxf(m1, gm);
        reinterpret_cast<float4*>(row_s)[i] = v[i];
      }
      float theta = m2;
#pragma unroll
      for (int m = 1; m < LPT; m <<= 1) theta = fminf(theta, __shfl_xor_sync(0xffffffffu, theta, m));
      unsigned cand = 0;
#pragma unroll
      for (int i = 0; i < F4; ++i) {
        cand |= (v[i].x >= theta ? 1u : 0u) << (4 * i);
        cand |= (v[i].y >= theta ? 1u : 0u) << (4 * i + 1);
        cand |= (v[i].z >= theta ? 1u : 0u) << (4 * i + 2);
        cand |= (v[i].w >= theta ? 1u : 0u) << (4 * i + 3);
      }
      while (cand) {   // ascending position = ascending expert index
        const int pos = __ffs(cand) - 1;
        cand &= cand - 1;
        insert(row_s[pos], 4 * (j + LPT * (pos >> 2)) + (pos & 3));
      }
    }
    // butterfly merge inside the token's lane group
#pragma unroll
    for (int m = 1; m < LPT; m <<= 1) {
      float ov[K];
      int oi[K];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        ov[k] = __shfl_xor_sync(0xffffffffu, tv[k], m);
        oi[k] = __shfl_xor_sync(0xffffffffu, ti[k], m);
      }
      if constexpr ((K & (K - 1)) == 0) {
        // bitonic top-K merge: the better of A[k] and B[K-1-k] is a bitonic
        // sequence holding the top K of both lists; log2(K) half-cleaner
        // stages sort it -- 20 compare-exchanges at K = 8 instead of the
        // K^2 selects of the two-pointer merge, same (value desc, index asc)
        // total order, so the same picks in the same order
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const float bv = ov[K - 1 - k];
          const int bi = oi[K - 1 - k];
          if (bv > tv[k] || (bv == tv[k] && bi < ti[k])) {
            tv[k] = bv;
            ti[k] = bi;
          }
        }
#pragma unroll
        for (int st = K / 2; st > 0; st >>= 1) {
#pragma unroll
          for (int k = 0; k < K; ++k) {
            if (k & st) continue;
            const float xv = tv[k], yv = tv[k + st];
            const int xi = ti[k], yi = ti[k + st];
            const bool swap = yv > xv || (yv == xv && yi < xi);
            tv[k] = swap ? yv : xv;
            ti[k] = swap ? yi : xi;
            tv[k + st] = swap ? xv : yv;
            ti[k + st] = swap ? xi : yi;
          }
        }
      } else {
        float nv[K];
        int ni[K];
        int a = 0, b = 0;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          float av = -INFINITY, bv = -INFINITY;
          int ai = 0x7fffffff, bi = 0x7fffffff;
#pragma unroll
          for (int q = 0; q < K; ++q) {
            if (q == a) { av = tv[q]; ai = ti[q]; }
            if (q == b) { bv = ov[q]; bi = oi[q]; }
          }
          const bool takea = av > bv || (av == bv && ai < bi);
          nv[k] = takea ? av : bv;
          ni[k] = takea ? ai : bi;
          a += takea;
          b += !takea;
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
          tv[k] = nv[k];
          ti[k] = ni[k];
        }
      }
    }
    const float vmax = tv[0];
    float denom = 0.f;
    if (renorm) {
#pragma unroll
      for (int k = 0; k < K; ++k) denom += expf(tv[k] - vmax);
    } else {
      float part = 0.f;
#pragma unroll
      for (int i = 0; i < F4; ++i)
        part += expf(v[i].x - vmax) + expf(v[i].y - vmax) + expf(v[i].z - vmax) +
                expf(v[i].w - vmax);
#pragma unroll
      for (int m = 1; m < LPT; m <<= 1) part += __shfl_xor_sync(0xffffffffu, part, m);
      denom = part;
    }
    if (live && j == 0) {
#pragma unroll
      for (int k = 0; k < K; ++k) {
        weights[t * K + k] = expf(tv[k] - vmax) / denom;
        slot_ids[t * K + k] = e2s ? e2s[ti[k]] : ti[k];
        if (expert_ids) expert_ids[t * K + k] = ti[k];
      }
    }
  }
}

// DeepSeek-V3 gate (group-limited, sigmoid + bias correction):
// scores = sigmoid(logit) (fp64, rounded to fp32), choice = scores + bias;
// group score = sum of the two largest choices of each contiguous group of
// E / n_group experts; the topk_group best groups stay; top-K choices inside
// them; weights = picked scores / their sum * scale.  Selections are value
// descending, index ascending.  Warp per token: lanes hold experts j*32+lane,
// the choices are staged in shared memory for the per-group scans.
template <int PER>
__global__ void __launch_bounds__(256) k_route_group(const float* __restrict__ logits, int64_t T,
                                                     int E, int K, int n_group, int topk_group,
                                                     const float* __restrict__ bias, float scale,
                                                     const int32_t* __restrict__ e2s,
                                                     int32_t* __restrict__ slot_ids,
                                                     float* __restrict__ weights,
                                                     int32_t* __restrict__ expert_ids) {
  __shared__ float s_ch[8][PER * 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  float* chs = s_ch[wid];
  const int gs = E / n_group;
  int64_t warp = (int64_t)blockIdx.x * 8 + wid;
  const int64_t nw = (int64_t)gridDim.x * 8;
  for (int64_t t = warp; t < T; t += nw) {
    float sc[PER], ch[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int e = j * 32 + lane;
      if (e < E) {
        const double xv = (double)logits[t * E + e];
        sc[j] = (float)(1.0 / (1.0 + exp(-xv)));
        ch[j] = sc[j] + (bias ? bias[e] : 0.f);
      } else {
        sc[j] = 0.f;
        ch[j] = -INFINITY;
      }
      chs[j * 32 + lane] = ch[j];
    }
    __syncwarp();
    // group scores (lane g scans group g), then the topk_group best groups
    float gsc = -INFINITY;
    if (lane < n_group) {
      float a = -INFINITY, b = -INFINITY;
      for (int i = 0; i < gs; ++i) {
        const float v = chs[lane * gs + i];
        if (v > a) {
          b = a;
          a = v;
        } else if (v > b) {
          b = v;
        }
      }
      gsc = gs > 1 ? a + b : a;
    }
    unsigned gsel = 0;
    bool avail = lane < n_group;
    for (int r = 0; r < topk_group; ++r) {
      float bv = avail ? gsc : -INFINITY;
      int bi = avail ? lane : 0x7fffffff;
      for (int o = 16; o; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) {
          bv = ov;
          bi = oi;
        }
      }
      gsel |= 1u << bi;
      if (lane == bi) avail = false;
    }
    // top-K choices inside the kept groups
    unsigned taken = 0;
    float pick_s[kMaxK];
    int pick_e[kMaxK];
    for (int k = 0; k < K; ++k) {
      float bv = -INFINITY, bs = 0.f;
      int be = 0x7fffffff;
#pragma unroll
      for (int j = 0; j < PER; ++j) {
        const int e = j * 32 + lane;
        if (e < E && !((taken >> j) & 1u) && ((gsel >> (e / gs)) & 1u) &&
            (ch[j] > bv || (ch[j] == bv && e < be))) {
          bv = ch[j];
          be = e;
          bs = sc[j];
        }
      }
      for (int o = 16; o; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oe = __shfl_xor_sync(0xffffffffu, be, o);
        const float os = __shfl_xor_sync(0xffffffffu, bs, o);
        if (ov > bv || (ov == bv && oe < be)) {
          bv = ov;
          be = oe;
          bs = os;
        }
      }
      if ((be & 31) == lane) taken |= 1u << (be >> 5);
      pick_s[k] = bs;
      pick_e[k] = be;
    }
    float sum = 0.f;
    for (int k = 0; k < K; ++k) sum += pick_s[k];
    if (lane < K) {
      float ps = 0.f;
      int pe = 0;
      for (int q = 0; q < K; ++q)
        if (q == lane) {
          ps = pick_s[q];
          pe = pick_e[q];
        }
      weights[t * K + lane] = ps / sum * scale;
      slot_ids[t * K + lane] = e2s ? e2s[pe] : pe;
      if (expert_ids) expert_ids[t * K + lane] = pe;
    }
    __syncwarp();
  }
}

// K1 router, lane-per-token variant for compile-time K: a warp stages 32
// tokens x 32 logits at a time in shared memory (padded rows -> conflict-free
// lane reads), every lane keeps its token's sorted top-K in registers
// (insertion with an early-out against the K-th value; strict > keeps the
// lower index on ties because columns arrive in ascending order).  With
// E % 4 == 0 the tile is fetched as 16-B vectors (8 per lane, all in flight)
// and the next tile's loads are issued before the current one is scanned.
template <int K, bool VEC>
__global__ void __launch_bounds__(256, 3) k_route_lane(const float* __restrict__ logits, int64_t T,
                                                    int E, const int32_t* __restrict__ e2s,
                                                    int renorm, int32_t* __restrict__ slot_ids,
                                                    float* __restrict__ weights,
                                                    int32_t* __restrict__ expert_ids) {
  __shared__ float tile[8][32][33];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  float (*tl)[33] = tile[wid];
  const int64_t nwarps = (int64_t)gridDim.x * 8;
  // vector staging: lane owns rows (lane >> 3) + 4 i, columns 4 (lane & 7) .. +3
  const int vr = lane >> 3, vc = (lane & 7) * 4;
  auto load_tile = [&](int64_t base, int c0, float4* buf) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int64_t tr = base + vr + 4 * i;
      const int col = c0 + vc;
      buf[i] = (tr < T && col < E)
                   ? __ldg(reinterpret_cast<const float4*>(logits + tr * E + col))
                   : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
    }
  };
  auto stage = [&](int64_t base, int c0, const float4* buf) {
    if constexpr (VEC) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float* d = &tl[vr + 4 * i][vc];
        d[0] = buf[i].x;
        d[1] = buf[i].y;
        d[2] = buf[i].z;
        d[3] = buf[i].w;
      }
    } else {
      const int col = c0 + lane;
#pragma unroll 8
      for (int r = 0; r < 32; ++r) {
        int64_t tr = base + r;
        tl[r][lane] = (tr < T && col < E) ? __ldg(logits + tr * E + col) : -INFINITY;
      }
    }
  };
  for (int64_t base = ((int64_t)blockIdx.x * 8 + wid) * 32; base < T; base += nwarps * 32) {
    const int64_t t = base + lane;
    float vals[K];
    int idx[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      vals[k] = -INFINITY;
      idx[k] = 0x7fffffff;
    }
    float4 buf[VEC ? 8 : 1];
    if constexpr (VEC) load_tile(base, 0, buf);
    for (int c0 = 0; c0 < E; c0 += 32) {
      stage(base, c0, buf);
      __syncwarp();
      if constexpr (VEC) {
        if (c0 + 32 < E) load_tile(base, c0 + 32, buf);   // in flight during the scan
      }
      const int ncol = E - c0 < 32 ? E - c0 : 32;
      for (int j = 0; j < ncol; ++j) {
        float v = tl[lane][j];
        if (v > vals[K - 1]) {
          const int e = c0 + j;
#pragma unroll
          for (int k = K - 1; k > 0; --k) {
            if (v > vals[k]) {
              bool up = v > vals[k - 1];
              vals[k] = up ? vals[k - 1] : v;
              idx[k] = up ? idx[k - 1] : e;
            }
          }
          if (v > vals[0]) {
            vals[0] = v;
            idx[0] = e;
          }
        }
      }
      __syncwarp();
    }
    const float vmax = vals[0];
    float denom = 0.f;
    if (renorm) {
#pragma unroll
      for (int k = 0; k < K; ++k) denom += expf(vals[k] - vmax);
    } else {
      for (int c0 = 0; c0 < E; c0 += 32) {   // second pass: full softmax denominator
        const int col = c0 + lane;
        for (int r = 0; r < 32; ++r) {
          int64_t tr = base + r;
          tl[r][lane] = (tr < T && col < E) ? __ldg(logits + tr * E + col) : -INFINITY;
        }
        __syncwarp();
        const int ncol = E - c0 < 32 ? E - c0 : 32;
        for (int j = 0; j < ncol; ++j) denom += expf(tl[lane][j] - vmax);
        __syncwarp();
      }
    }
    if (t < T) {
#pragma unroll
      for (int k = 0; k < K; ++k) {
        weights[t * K + k] = expf(vals[k] - vmax) / denom;
        slot_ids[t * K + k] = e2s ? e2s[idx[k]] : idx[k];
        if (expert_ids) expert_ids[t * K + k] = idx[k];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// plan: grid (chunks, L).  Stable ranks: destination ranks by warp ballot,
// slot ranks by comparing with earlier lanes' picks via shuffles, then a
// prefix over the chunk's warps.
template <int KT>   // KT = K (1..8) or kMaxK (any K, guarded by w.K)
__global__ void __launch_bounds__(kChunk) k_plan(const WorldDev* __restrict__ wp,
                                                 const int32_t* __restrict__ ids, int nchunks,
                                                 int32_t* __restrict__ chunk_cnt,
                                                 int32_t* __restrict__ rank_d,
                                                 int32_t* __restrict__ rank_e,
                                                 unsigned long long* __restrict__ hitmask,
                                                 int32_t* __restrict__ rank_g,
                                                 int* __restrict__ status) {
  const WorldDev& w = *wp;
  // [kPlanWarps][G+E+P] counters (ranks, slots, GPUs), then [kPlanWarps][E] lane masks
  extern __shared__ int32_t s_cnt[];
  const int C = w.G + w.E + w.P;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s_loc = blockIdx.y;
  const int chunk = blockIdx.x;
  for (int i = threadIdx.x; i < kPlanWarps * (C + w.E); i += blockDim.x) s_cnt[i] = 0;
  __syncthreads();
  const int64_t t_in = (int64_t)chunk * kChunk + warp * 32 + lane;  // token within source
  const bool valid = t_in < w.T_r;
  const int64_t t = (int64_t)s_loc * w.T_r + t_in;                   // local token index
  int S[KT];
  unsigned long long hit = 0;
#pragma unroll
  for (int k = 0; k < KT; ++k) {
    S[k] = -1;
    if ((KT != kMaxK || k < w.K) && valid) {
      int e = ids[t * w.K + k];
      if (e < -1 || e >= w.E) {   // -1 = padding (no pick)
        atomicExch(status, 4);
        e = -1;
      }
      S[k] = e;
      if (e >= 0) hit |= 1ull << dest_of(w, w.p * w.L + s_loc, e);
    }
  }
  // per-warp counts per destination rank and per destination GPU (mode 3:
  // a GPU is hit if any of its L ranks is); the within-warp ranks are
  // recomputed from the same ballots after the prefix (no global RMW)
  const unsigned lt = (1u << lane) - 1u;
  for (int d = 0; d < w.G; ++d) {
    unsigned b = __ballot_sync(0xffffffffu, (hit >> d) & 1ull);
    if (lane == 0) s_cnt[warp * C + d] = __popc(b);
  }
  const unsigned long long gmask = w.L >= 64 ? ~0ull : ((1ull << w.L) - 1ull);
  for (int q = 0; q < w.P; ++q) {
    unsigned b = __ballot_sync(0xffffffffu, (hit >> (q * w.L)) & gmask);
    if (lane == 0) s_cnt[warp * C + w.G + w.E + q] = __popc(b);
  }
  // slot ranks within the warp: a lane mask per slot in shared memory; the
  // rank of my pick = earlier lanes in that slot's mask (stable, O(K))
  unsigned* s_lanes = reinterpret_cast<unsigned*>(s_cnt + kPlanWarps * C) + warp * w.E;
#pragma unroll
  for (int k = 0; k < KT; ++k)
    if ((KT != kMaxK || k < w.K) && S[k] >= 0) atomicOr(s_lanes + S[k], 1u << lane);
  __syncwarp();
  int re[KT];
#pragma unroll
  for (int k = 0; k < KT; ++k)
    re[k] = ((KT != kMaxK || k < w.K) && S[k] >= 0) ? __popc(s_lanes[S[k]] & lt) : 0;
  for (int e = lane; e < w.E; e += 32) s_cnt[warp * C + w.G + e] = __popc(s_lanes[e]);
  __syncthreads();
  // exclusive prefix over warps per counter; chunk totals out
  int32_t* out = chunk_cnt + ((int64_t)s_loc * nchunks + chunk) * C;
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    int run = 0;
    for (int wi = 0; wi < kPlanWarps; ++wi) {
      int v = s_cnt[wi * C + c];
      s_cnt[wi * C + c] = run;
      run += v;
    }
    out[c] = run;
  }
  __syncthreads();
  for (int d = 0; d < w.G; ++d) {
    const bool h = (hit >> d) & 1ull;
    const unsigned b = __ballot_sync(0xffffffffu, h);
    if (valid) rank_d[t * w.G + d] = h ? __popc(b & lt) + s_cnt[warp * C + d] : -1;
  }
  for (int q = 0; q < w.P; ++q) {
    const bool h = (hit >> (q * w.L)) & gmask;
    const unsigned b = __ballot_sync(0xffffffffu, h);
    if (valid) rank_g[t * w.P + q] = h ? __popc(b & lt) + s_cnt[warp * C + w.G + w.E + q] : -1;
  }
  if (valid) {
#pragma unroll
    for (int k = 0; k < KT; ++k)
      if (KT != kMaxK || k < w.K) rank_e[t * w.K + k] = S[k] >= 0 ? re[k] + s_cnt[warp * C + w.G + S[k]] : -1;
    hitmask[t] = hit;
  }
}

// ---------------------------------------------------------------------------
// notify: one CTA.  chunk_cnt -> exclusive chunk offsets (in place) + totals;
// totals stored into every GPU's count matrix; barrier; derived offsets.
//   eoff[s_loc][e] = ebase[e] + sum_{s' < s} c[s', e]  (expert-major base of
//   source s's rows for slot e at dest(e)), where ebase[e] = sum of N_e' over
//   earlier local slots of the same destination.
// Latency-bound (one CTA, a few KB of counts): world scalars live in
// registers, the chunk prefix keeps 16 loads in flight per column, and the
// derived offsets are one flat index space over the whole CTA (every output
// is a short sum over the staged count matrix), so no thread walks several
// output families one after another.
__global__ void __launch_bounds__(1024) k_notify(const WorldDev* __restrict__ wp, int nchunks,
                                                 int32_t* __restrict__ chunk_cnt,
                                                 Offsets* __restrict__ offs,
                                                 int32_t* __restrict__ eoff,
                                                 int32_t* __restrict__ n_e, int mode,
                                                 int* __restrict__ status, int stage_cnt) {
  const WorldDev& w = *wp;
  const int G = w.G, E = w.E, L = w.L, P = w.P, gp = w.p, E_loc = w.E_loc;
  const int C = G + E + P, CG = G + E;
  for (int i = threadIdx.x; i < L * C; i += blockDim.x) {
    const int s_loc = i / C, c = i - s_loc * C;
    int32_t* col = chunk_cnt + (int64_t)s_loc * nchunks * C + c;
    int run = 0;
    for (int ch0 = 0; ch0 < nchunks; ch0 += 16) {   // 16 loads in flight, then the stores
      int v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = ch0 + j < nchunks ? col[(int64_t)(ch0 + j) * C] : 0;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        if (ch0 + j < nchunks) col[(int64_t)(ch0 + j) * C] = run;
        run += v[j];
      }
    }
    const int sg = gp * L + s_loc;
    for (int q = 0; q < P; ++q) w.counts[q * L][(int64_t)sg * C + c] = run;
  }
  cta_barrier(w, status);
  // shared memory: s_n[E] per-slot totals, s_eb[E] expert-major bases,
  // s_gpu[G] GPU of each rank, then the [G][C] count matrix when it fits
  extern __shared__ int32_t notify_smem[];
  int32_t* s_n = notify_smem;
  int32_t* s_eb = s_n + E;
  int32_t* s_gpu = s_eb + E;
  const int32_t* cnt = w.counts[gp * L];
  for (int r = threadIdx.x; r < G; r += blockDim.x) s_gpu[r] = r / L;
  if (stage_cnt) {
    int32_t* s_cnt = s_gpu + G;
    for (int i = threadIdx.x; i < G * C; i += blockDim.x) s_cnt[i] = cnt[i];
    __syncthreads();
    cnt = s_cnt;
  }
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int sum = 0;
    for (int src = 0; src < G; ++src) sum += cnt[(int64_t)src * C + G + e];
    s_n[e] = sum;
    n_e[e] = sum;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int base = 0;
    for (int e2 = (e / E_loc) * E_loc; e2 < e; ++e2) base += s_n[e2];
    s_eb[e] = base;
  }
  __syncthreads();
  // mode 2 (dedup across GPUs only): sources on the destination's own GPU
  // write expert-major rows directly and occupy no receive rows
  auto ships = [&](int src, int dst) {
    return mode == 1 || (mode == 2 && s_gpu[src] != s_gpu[dst]);
  };
  // flat index space: [eoff L*E][off L*G][offd L*(G+1)][off_g L*P][offd_g G+1][R/Nd L]
  const int n0 = L * E, n1 = n0 + L * G, n2 = n1 + L * (G + 1), n3 = n2 + L * P,
            n4 = n3 + G + 1, n5 = n4 + L;
  for (int i = threadIdx.x; i < n5; i += blockDim.x) {
    if (i < n0) {
      // expert e's rows at its destination GPU q are source-major starting
      // with q's own ranks (rotation by q * L): the rows already on q form one
      // block in front, so the overlapped forward computes them as whole
      // tiles before the received ones arrive
      const int s_loc = i / E, e = i - s_loc * E;
      const int sg = gp * L + s_loc;
      const int q0 = (e / E_loc) / L * L;
      const int key = sg - q0 < 0 ? sg - q0 + G : sg - q0;   // (sg - q0) mod G
      int base = s_eb[e];
      for (int src = 0; src < G; ++src) {
        const int r = src - q0 < 0 ? src - q0 + G : src - q0;
        if (r < key) base += cnt[(int64_t)src * C + G + e];
      }
      eoff[i] = base;
    } else if (i < n1) {
      const int k = i - n0, s_loc = k / G, d = k - s_loc * G;
      const int sg = gp * L + s_loc;
      int o = 0;
      for (int src = 0; src < sg; ++src)
        if (ships(src, d)) o += cnt[(int64_t)src * C + d];
      offs->off[s_loc][d] = o;
    } else if (i < n2) {
      const int k = i - n1, d_loc = k / (G + 1), src = k - d_loc * (G + 1);
      const int dg = gp * L + d_loc;
      int o = 0;
      for (int s2 = 0; s2 < src; ++s2)
        if (ships(s2, dg)) o += cnt[(int64_t)s2 * C + dg];
      offs->offd[d_loc][src] = o;
    } else if (i < n3) {   // mode 3: GPU-level offsets (only sources on other GPUs ship)
      const int k = i - n2, s_loc = k / P, q = k - s_loc * P;
      const int sg = gp * L + s_loc;
      int o = 0;
      for (int src = 0; src < sg; ++src)
        if (s_gpu[src] != q) o += cnt[(int64_t)src * C + CG + q];
      offs->off_g[s_loc][q] = o;
    } else if (i < n4) {
      const int src = i - n3;
      int o = 0;
      for (int s2 = 0; s2 < src; ++s2)
        if (s_gpu[s2] != gp) o += cnt[(int64_t)s2 * C + CG + gp];
      offs->offd_g[src] = o;
      if (src == G) {
        offs->R_g = o;
        if (mode == 3 && o > w.Rg_cap) atomicExch(status, 2);
      }
    } else {
      const int d_loc = i - n4, dg = gp * L + d_loc;
      int r = 0;
      for (int src = 0; src < G; ++src)
        if (ships(src, dg)) r += cnt[(int64_t)src * C + dg];
      offs->R[d_loc] = r;
      int n = 0;
      for (int e = dg * E_loc; e < (dg + 1) * E_loc; ++e) n += s_n[e];
      offs->Nd[d_loc] = n;
      if (r > w.R_cap || (!w.U1 && n > w.N_cap)) atomicExch(status, 2);  // capacity overflow
    }
  }
}

// ---------------------------------------------------------------------------
// 16-byte vector helpers
__device__ __forceinline__ int4 ld_nc_v4(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ int4 ld_v4(const int4* p) {
  int4 r;
  asm volatile("ld.global.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
// L2-coherent load (no L1 allocation) for rows a peer wrote during this kernel
__device__ __forceinline__ int4 ld_cg_v4(const int4* p) {
  int4 r;
  asm volatile("ld.global.cg.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st_na_v4(int4* p, int4 v) {
  asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w));
}

constexpr int kUnroll = 8;  // 16-B vectors per lane in flight (4 KB per warp)

// pack: warp per token.  dedup: one copy per hit destination + per-row meta;
// raw: one copy per selection into expert-major rows.
// Bijective spread of [0, n) (multiplication by a prime coprime with n): the
// destination-side reducers walk their received rows in this order so that
// at any moment the warps push to every source GPU instead of one source's
// contiguous range at a time (spreads the NVLink traffic over the peers).
__device__ __forceinline__ int64_t spread_index(int64_t i, int64_t n) {
  const int64_t p = (n % 7919) ? 7919 : ((n % 104729) ? 104729 : 1);
  return (i * p) % n;
}

// one token's dispatch (warp): expert-major positions of its picks, then the
// row to every place it goes (direct expert-major rows for picks on this GPU
// in modes 0/2/3, one row per hit remote GPU in mode 3, one row per hit
// destination rank in modes 1/2) with its per-row metadata
__device__ __forceinline__ void pack_token(const WorldDev& w, int64_t t, int lane,
                                           const uint8_t* __restrict__ x,
                                           const int32_t* __restrict__ ids,
                                           const float* __restrict__ wts,
                                           const int32_t* __restrict__ chunk_off,
                                           const int32_t* __restrict__ rank_d,
                                           const int32_t* __restrict__ rank_e,
                                           const unsigned long long* __restrict__ hitmask,
                                           const Offsets* __restrict__ offs,
                                           const int32_t* __restrict__ eoff, int nchunks, int mode,
                                           int32_t* __restrict__ gpos, int32_t* __restrict__ epos_out,
                                           const int32_t* __restrict__ rank_g,
                                           int32_t* __restrict__ gpos_g, int* __restrict__ status,
                                           int32_t* __restrict__ xidx, int copy_rows = 1) {
  const int C = w.G + w.E + w.P;
  const unsigned long long gmask = w.L >= 64 ? ~0ull : ((1ull << w.L) - 1ull);
  const int64_t nvec = w.row_bytes / 16;
  const int s_loc = (int)(t / w.T_r);
  const int64_t t_in = t - (int64_t)s_loc * w.T_r;
  const int32_t* coff = chunk_off + ((int64_t)s_loc * nchunks + t_in / kChunk) * C;
  const int4* src = reinterpret_cast<const int4*>(x + t * w.row_bytes);
  // expert-major positions of my picks (lane k < K computes pick k)
  int my_e = -1, my_ep = -1;
  float my_w = 0.f;
  if (lane < w.K) {
    my_e = ids[t * w.K + lane];
    my_w = wts ? wts[t * w.K + lane] : 0.f;
    if (my_e >= 0 && !w.U1) {   // relay worlds build no expert-major rows
      my_ep = eoff[s_loc * w.E + my_e] + coff[w.G + my_e] + rank_e[t * w.K + lane];
      if (my_ep >= w.N_cap) {
        atomicExch(status, 2);
        my_ep = -1;
      }
    }
    epos_out[t * w.K + lane] = my_ep;
  }
  unsigned long long hit = hitmask[t];
  // destinations (dedup) or picks (raw) this row goes to
  int ndst = 0;
  int64_t dst_row[kMaxRanks > kMaxK ? kMaxRanks : kMaxK];
  uint8_t* dst_base[kMaxRanks > kMaxK ? kMaxRanks : kMaxK];
  // fused dispatch (xidx): picks on this GPU get the token's row index
  // instead of a row copy (the expert GEMM gathers from x)
  if (xidx && lane < w.K && my_e >= 0 && my_ep >= 0) {
    const int d = rank_of_slot(w, my_e);
    if (d / w.L == w.p) xidx[(int64_t)(d - w.p * w.L) * w.N_cap + my_ep] = (int32_t)t;
  }
  // direct expert-major rows: every pick (mode 0) or picks on this GPU (modes 2, 3)
  if (mode != 1 && !xidx) {
    for (int k = 0; k < w.K; ++k) {
      int e = __shfl_sync(0xffffffffu, my_e, k);
      int ep = __shfl_sync(0xffffffffu, my_ep, k);
      if (e < 0 || ep < 0) continue;
      const int d = rank_of_slot(w, e);
      if (mode >= 2 && d / w.L != w.p) continue;
      dst_base[ndst] = w.xmaj[d];
      dst_row[ndst] = ep;
      ++ndst;
    }
  }
  // mode 3: one row per (token, other GPU hit); meta carries, per pick on
  // that GPU, its local rank's expert-major row (l * N_cap + epos)
  if (mode == 3) {
    for (int q = 0; q < w.P; ++q) {
      if (q == w.p) continue;
      if (!((hit >> (q * w.L)) & gmask)) {
        if (lane == 0) gpos_g[t * w.P + q] = -1;
        continue;
      }
      const int64_t g = (int64_t)offs->off_g[s_loc][q] + coff[w.G + w.E + q] + rank_g[t * w.P + q];
      if (lane == 0) gpos_g[t * w.P + q] = (int32_t)g;
      if (g >= w.Rg_cap) {
        if (lane == 0) atomicExch(status, 2);
        continue;
      }
      const int dr = my_e >= 0 ? rank_of_slot(w, my_e) : -1;
      const bool on_q = dr >= 0 && dr / w.L == q && my_ep >= 0;
      if (lane < w.K) {
        RowMeta m;
        m.epos = on_q ? (int32_t)((dr - q * w.L) * w.N_cap + my_ep) : -1;
        m.w = my_w;
        w.meta_g[q][g * w.K + lane] = m;
      }
      // the row lands directly in the expert-major slot of its first pick on
      // GPU q; the destination's expansion copies it to the remaining picks
      // (fused: into q's receive buffer, whose row index the picks then get)
      const unsigned on = __ballot_sync(0xffffffffu, on_q && lane < w.K);
      if (on && xidx) {
        dst_base[ndst] = w.recv_g[q];
        dst_row[ndst] = g;
        ++ndst;
      } else if (on) {
        const int k0 = __ffs(on) - 1;
        const int d0 = __shfl_sync(0xffffffffu, dr, k0);
        const int e0 = __shfl_sync(0xffffffffu, my_ep, k0);
        dst_base[ndst] = w.xmaj[d0];
        dst_row[ndst] = e0;
        ++ndst;
      }
    }
  }
  // dedup rows: every hit destination (mode 1) or destinations on other GPUs (mode 2)
  if (mode == 1 || mode == 2) {
    for (int d = 0; d < w.G; ++d) {
      if (!((hit >> d) & 1ull)) continue;
      if (mode == 2 && d / w.L == w.p) {
        if (lane == 0) gpos[t * w.G + d] = -1;
        continue;
      }
      int64_t g = (int64_t)offs->off[s_loc][d] + coff[d] + rank_d[t * w.G + d];
      if (lane == 0) gpos[t * w.G + d] = (int32_t)g;
      if (g >= w.R_cap) {
        if (lane == 0) atomicExch(status, 2);
        continue;
      }
      // meta: lane k writes pick k's local expert-major row (relay: its slot
      // id, restricted to the destination's group) or -1, plus the gate
      if (lane < w.K) {
        RowMeta m;
        const int sg = w.p * w.L + s_loc;
        const bool here = my_e >= 0 && dest_of(w, sg, my_e) == d;
        m.epos = here ? (w.U1 ? my_e : my_ep) : -1;
        m.w = my_w;
        w.recv_meta[d][g * w.K + lane] = m;
      }
      dst_base[ndst] = w.recv_x[d];
      dst_row[ndst] = g;
      ++ndst;
    }
    if (lane == 0)
      for (int d = 0; d < w.G; ++d)
        if (!((hit >> d) & 1ull)) gpos[t * w.G + d] = -1;
  }
  if (!copy_rows) return;   // metadata only: the rows move with the expert GEMM (exch.cuh)
  for (int64_t v0 = 0; v0 < nvec; v0 += 32 * kUnroll) {
    int4 buf[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      int64_t v = v0 + u * 32 + lane;
      if (v < nvec) buf[u] = ld_nc_v4(src + v);
    }
    for (int j = 0; j < ndst; ++j) {
      int4* dst = reinterpret_cast<int4*>(dst_base[j] + dst_row[j] * w.row_bytes);
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        int64_t v = v0 + u * 32 + lane;
        if (v < nvec) st_na_v4(dst + v, buf[u]);
      }
    }
  }
}

__global__ void __launch_bounds__(256) k_pack(const WorldDev* __restrict__ wp,
                                              const uint8_t* __restrict__ x,
                                              const int32_t* __restrict__ ids,
                                              const float* __restrict__ wts,
                                              const int32_t* __restrict__ chunk_off,
                                              const int32_t* __restrict__ rank_d,
                                              const int32_t* __restrict__ rank_e,
                                              const unsigned long long* __restrict__ hitmask,
                                              const Offsets* __restrict__ offs,
                                              const int32_t* __restrict__ eoff, int nchunks,
                                              int mode, int32_t* __restrict__ gpos,
                                              int32_t* __restrict__ epos_out,
                                              const int32_t* __restrict__ rank_g,
                                              int32_t* __restrict__ gpos_g,
                                              int* __restrict__ status,
                                              int32_t* __restrict__ xidx, int copy_rows) {
  const WorldDev& w = *wp;
  const int lane = threadIdx.x & 31;
  const int64_t T = (int64_t)w.L * w.T_r;
  int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  // across GPUs, tokens are walked in a spread order (like the reducers) so the
  // concurrent warps' NVLink stores land all over the peers' receive buffers
  const bool spread = mode == 3 && w.P > 1;
  for (int64_t i = warp; i < T; i += nw)
    pack_token(w, spread ? spread_index(i, T) : i, lane, x, ids, wts, chunk_off, rank_d,
                   rank_e, hitmask, offs, eoff, nchunks, mode, gpos, epos_out, rank_g, gpos_g,
                   status, xidx, copy_rows);
}

// One-GPU pack (every destination local: modes 0, 2, 3 at P = 1): warp per
// token, the row's first 4 KB loaded before the position bookkeeping, lane k
// holds pick k's destination pointer (no per-token destination arrays), the
// stores broadcast the pointers by shuffle.  Lean registers -> more resident
// warps than the general pack_token.
template <int VPL>
__global__ void __launch_bounds__(256) k_pack_local(const WorldDev* __restrict__ wp,
                                                    const uint8_t* __restrict__ x,
                                                    const int32_t* __restrict__ ids,
                                                    const int32_t* __restrict__ chunk_off,
                                                    const int32_t* __restrict__ rank_e,
                                                    const int32_t* __restrict__ eoff, int nchunks,
                                                    int32_t* __restrict__ epos_out,
                                                    int* __restrict__ status) {
  const WorldDev& w = *wp;
  const int lane = threadIdx.x & 31;
  const int C = w.G + w.E + w.P;
  const int64_t T = (int64_t)w.L * w.T_r;
  int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t t = warp; t < T; t += nw) {
    const int4* src = reinterpret_cast<const int4*>(x + t * w.row_bytes);
    int4 buf[VPL];
#pragma unroll
    for (int u = 0; u < VPL; ++u) buf[u] = ld_nc_v4(src + u * 32 + lane);
    const int s_loc = (int)(t / w.T_r);
    const int64_t t_in = t - (int64_t)s_loc * w.T_r;
    uint8_t* dst = nullptr;
    if (lane < w.K) {
      const int e = ids[t * w.K + lane];
      int ep = -1;
      if (e >= 0) {
        const int32_t* coff = chunk_off + ((int64_t)s_loc * nchunks + t_in / kChunk) * C;
        ep = eoff[s_loc * w.E + e] + coff[w.G + e] + rank_e[t * w.K + lane];
        if (ep >= w.N_cap) {
          atomicExch(status, 2);
          ep = -1;
        }
      }
      epos_out[t * w.K + lane] = ep;
      if (ep >= 0) dst = w.xmaj[rank_of_slot(w, e)] + (int64_t)ep * w.row_bytes;
    }
    for (int k = 0; k < w.K; ++k) {
      int4* d = reinterpret_cast<int4*>(
          __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(dst), k));
      if (!d) continue;
#pragma unroll
      for (int u = 0; u < VPL; ++u) st_na_v4(d + u * 32 + lane, buf[u]);
    }
  }
}

// Fused one-GPU dispatch (hm_world_set_option 10): the expert-major rows are
// not materialised -- each pick's expert-major position gets the token's row
// index (xidx[local rank][epos] = t), and the expert GEMM gathers its A rows
// from x with TMA gather4 (hm_expert_ffn_gather).  Thread per (token, pick):
// T*K*(4 + 4) bytes instead of T*M*v + T*K*M*v.
__global__ void __launch_bounds__(256) k_index_local(const WorldDev* __restrict__ wp,
                                                     const int32_t* __restrict__ ids,
                                                     const int32_t* __restrict__ chunk_off,
                                                     const int32_t* __restrict__ rank_e,
                                                     const int32_t* __restrict__ eoff, int nchunks,
                                                     int32_t* __restrict__ epos_out,
                                                     int32_t* __restrict__ xidx,
                                                     int* __restrict__ status) {
  const WorldDev& w = *wp;
  const int C = w.G + w.E + w.P;
  const int64_t T = (int64_t)w.L * w.T_r;
  const int64_t n = T * w.K;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i / w.K;
    const int e = ids[i];
    int ep = -1;
    if (e >= 0) {
      const int s_loc = (int)(t / w.T_r);
      const int64_t t_in = t - (int64_t)s_loc * w.T_r;
      const int32_t* coff = chunk_off + ((int64_t)s_loc * nchunks + t_in / kChunk) * C;
      ep = eoff[s_loc * w.E + e] + coff[w.G + e] + rank_e[i];
      const int d = rank_of_slot(w, e);
      if (ep >= w.N_cap) {
        atomicExch(status, 2);
        ep = -1;
      } else if (d / w.L == w.p) {   // picks on this GPU (every pick with one GPU)
        xidx[(int64_t)(d - w.p * w.L) * w.N_cap + ep] = (int32_t)t;
      }
    }
    epos_out[i] = ep;
  }
}

// expand (dedup, destination side): warp per received row -> its local
// experts' expert-major rows.
__global__ void __launch_bounds__(256) k_expand(const WorldDev* __restrict__ wp,
                                                const Offsets* __restrict__ offs) {
  const WorldDev& w = *wp;
  const int lane = threadIdx.x & 31;
  const int64_t nvec = w.row_bytes / 16;
  int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  int64_t total = 0;
  for (int d = 0; d < w.L; ++d) total += offs->R[d];
  for (int64_t i = warp; i < total; i += nw) {
    int d_loc = 0;
    int64_t r = i;
    while (r >= offs->R[d_loc]) {
      r -= offs->R[d_loc];
      ++d_loc;
    }
    const int dg = w.p * w.L + d_loc;
    int ep = -1;
    if (lane < w.K) ep = w.recv_meta[dg][r * w.K + lane].epos;
    const int4* src = reinterpret_cast<const int4*>(w.recv_x[dg] + r * w.row_bytes);
    for (int64_t v0 = 0; v0 < nvec; v0 += 32 * kUnroll) {
      int4 buf[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        int64_t v = v0 + u * 32 + lane;
        if (v < nvec) buf[u] = ld_nc_v4(src + v);
      }
      for (int k = 0; k < w.K; ++k) {
        int e = __shfl_sync(0xffffffffu, ep, k);
        if (e < 0) continue;
        int4* dst = reinterpret_cast<int4*>(w.xmaj[dg] + (int64_t)e * w.row_bytes);
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          int64_t v = v0 + u * 32 + lane;
          if (v < nvec) st_na_v4(dst + v, buf[u]);
        }
      }
    }
  }
}

// element conversion helpers for 16-B vectors: 8 bf16 or 4 fp32
template <typename T>
struct Vec;
template <>
struct Vec<__nv_bfloat16> {
  static constexpr int N = 8;
  __device__ static void to_f32(const int4& v, float* f) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 x = __bfloat1622float2(h[i]);
      f[2 * i] = x.x;
      f[2 * i + 1] = x.y;
    }
  }
  __device__ static int4 from_f32(const float* f) {
    int4 v;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
    return v;
  }
};
template <>
struct Vec<float> {
  static constexpr int N = 4;
  __device__ static void to_f32(const int4& v, float* f) {
    f[0] = __int_as_float(v.x);
    f[1] = __int_as_float(v.y);
    f[2] = __int_as_float(v.z);
    f[3] = __int_as_float(v.w);
  }
  __device__ static int4 from_f32(const float* f) {
    return make_int4(__float_as_int(f[0]), __float_as_int(f[1]), __float_as_int(f[2]),
                     __float_as_int(f[3]));
  }
};


// dst row = sum_j ws[j] * row_j (fp32 accumulation in j order), rows in the
// payload dtype.  The source table (srcs/ws) lives in shared memory (one slice
// per warp; broadcast reads) so it costs neither registers nor a local-memory
// stack frame.  Fixed-width rows: each lane owns kCh 16-B vectors per chunk
// and the loads of kSu sources are issued before the first is accumulated
// (kCh * kSu * 16 B in flight per lane; registers stay under the 3-CTA/SM
// budget of __launch_bounds__(256, 3)).
constexpr int kU = 4;
constexpr int kCh = 2, kSu = 4;

// compile-time row width: VPL 16-B vectors per lane (row = 32 * VPL vectors)
template <typename T, int VPL, bool CG = false, int SU = kSu>
__device__ __forceinline__ void weighted_row_sum_fixed(const uint8_t* const* srcs, const float* ws,
                                                       int n, int lane, int4* dst) {
  constexpr int CH = VPL < kCh ? VPL : kCh;
  static_assert(VPL % CH == 0, "row width must be a multiple of the chunk");
#pragma unroll 1
  for (int c = 0; c < VPL; c += CH) {
    float acc[CH][Vec<T>::N];
#pragma unroll
    for (int u = 0; u < CH; ++u)
#pragma unroll
      for (int q = 0; q < Vec<T>::N; ++q) acc[u][q] = 0.f;
    const int off = c * 32 + lane;
#pragma unroll 1
    for (int j0 = 0; j0 < n; j0 += SU) {
      int4 buf[SU][CH];
#pragma unroll
      for (int s = 0; s < SU; ++s) {
        if (j0 + s < n) {
          const int4* src = reinterpret_cast<const int4*>(srcs[j0 + s]) + off;
#pragma unroll
          for (int u = 0; u < CH; ++u) buf[s][u] = CG ? ld_cg_v4(src + u * 32) : ld_v4(src + u * 32);
        }
      }
#pragma unroll
      for (int s = 0; s < SU; ++s) {
        if (j0 + s < n) {
          const float wj = ws[j0 + s];
#pragma unroll
          for (int u = 0; u < CH; ++u) {
            float f[Vec<T>::N];
            Vec<T>::to_f32(buf[s][u], f);
#pragma unroll
            for (int q = 0; q < Vec<T>::N; ++q) acc[u][q] = fmaf(wj, f[q], acc[u][q]);
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < CH; ++u) st_na_v4(dst + off + u * 32, Vec<T>::from_f32(acc[u]));
  }
}

// VPL > 0: compile-time row width (one kernel instantiation per width, so the
// register allocation is not shared with the generic loop); VPL == 0: any width
template <typename T, bool CG = false>
__device__ __forceinline__ void weighted_row_sum_any(const uint8_t* const* srcs, const float* ws,
                                                     int n, int64_t nvec, int lane, int4* dst) {
  for (int64_t v0 = 0; v0 < nvec; v0 += 32 * kU) {
    float acc[kU][Vec<T>::N];
#pragma unroll
    for (int u = 0; u < kU; ++u)
#pragma unroll
      for (int q = 0; q < Vec<T>::N; ++q) acc[u][q] = 0.f;
    for (int j = 0; j < n; ++j) {
      const int4* src = reinterpret_cast<const int4*>(srcs[j]);
      int4 buf[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int64_t v = v0 + u * 32 + lane;
        if (v < nvec) buf[u] = CG ? ld_cg_v4(src + v) : ld_v4(src + v);
      }
      const float wj = ws[j];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        float f[Vec<T>::N];
        Vec<T>::to_f32(buf[u], f);
#pragma unroll
        for (int q = 0; q < Vec<T>::N; ++q) acc[u][q] = fmaf(wj, f[q], acc[u][q]);
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t v = v0 + u * 32 + lane;
      if (v < nvec) st_na_v4(dst + v, Vec<T>::from_f32(acc[u]));
    }
  }
}

template <typename T, int VPL, bool CG = false, int SU = kSu>
__device__ __forceinline__ void weighted_row_sum(const uint8_t* const* srcs, const float* ws,
                                                 int n, int64_t nvec, int lane, int4* dst) {
  if constexpr (VPL > 0)
    weighted_row_sum_fixed<T, VPL, CG, SU>(srcs, ws, n, lane, dst);
  else
    weighted_row_sum_any<T, CG>(srcs, ws, n, nvec, lane, dst);
}


// expert-side source rows of a received row: lane k resolves meta k
__device__ __forceinline__ int meta_sources_warp(const RowMeta* meta, int K, const uint8_t* ybase,
                                                 int64_t row_bytes, int grad, int lane,
                                                 const uint8_t** srcs, float* ws) {
  bool v = false;
  RowMeta m;
  m.epos = -1;
  m.w = 0.f;
  if (lane < K) {
    m = meta[lane];
    v = m.epos >= 0;
  }
  const unsigned b = __ballot_sync(0xffffffffu, v);
  if (v) {
    const int pos = __popc(b & ((1u << lane) - 1u));
    srcs[pos] = ybase + (int64_t)m.epos * row_bytes;
    ws[pos] = grad ? 1.f : m.w;
  }
  return __popc(b);
}

// reduce (dedup, destination side): partial[i] = sum_k w_k * y[epos_k] over the
// row's local picks in k order, fp32 accumulation, stored in payload dtype.
template <typename T, int VPL>
__global__ void __launch_bounds__(256, 3) k_reduce(const WorldDev* __restrict__ wp,
                                                   const Offsets* __restrict__ offs, int grad,
                                                   int push) {
  const WorldDev& w = *wp;
  __shared__ const uint8_t* s_src[8][kMaxK];
  __shared__ float s_w[8][kMaxK];
  const int lane = threadIdx.x & 31;
  const int64_t nvec = w.row_bytes / 16;
  int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  int64_t total = 0;
  for (int d = 0; d < w.L; ++d) total += offs->R[d];
  for (int64_t i = warp; i < total; i += nw) {
    int d_loc = 0;
    int64_t r = spread_index(i, total);
    while (r >= offs->R[d_loc]) {
      r -= offs->R[d_loc];
      ++d_loc;
    }
    const int dg = w.p * w.L + d_loc;
    const uint8_t* ysrc = grad ? w.gx[dg] : w.ymaj[dg];
    __syncwarp();
    const uint8_t** srcs = s_src[threadIdx.x >> 5];
    float* ws = s_w[threadIdx.x >> 5];
    // dispatch backward (grad): unweighted sum of input grads
    const int n = meta_sources_warp(w.recv_meta[dg] + r * w.K, w.K, ysrc, w.row_bytes, grad,
                                    lane, srcs, ws);
    uint8_t* out_row = w.comb[dg] + r * w.row_bytes;
    if (push) {   // store straight into the source rank's return buffer (NVLink if remote)
      int src = 0;
      while (src + 1 < w.G && offs->offd[d_loc][src + 1] <= r) ++src;
      const int64_t pos = r - offs->offd[d_loc][src];
      out_row = w.ret[src] + ((int64_t)dg * w.T_r + pos) * w.row_bytes;
    }
    __syncwarp();
    weighted_row_sum<T, VPL>(srcs, ws, n, nvec, lane, reinterpret_cast<int4*>(out_row));
  }
}

// gather (source side).  dedup: out[t] = sum over hit destinations d
// (ascending) of comb[d][gpos[t,d]]; raw: out[t] = sum_k w_k * ymaj[dest][epos].
// Warp-cooperative gather_sources: lane k resolves pick k, lane q GPU q, lane
// d rank d, in one round of loads; ballots compact them into the warp's
// shared-memory source table in the same (summation) order.  Returns n
// (warp-uniform); the caller __syncwarp()s before reading the table.
__device__ __forceinline__ int gather_sources_warp(const WorldDev& w, int64_t t, int lane,
                                                   const int32_t* ids, const float* wts,
                                                   const unsigned long long* hitmask,
                                                   const int32_t* gpos, const int32_t* epos,
                                                   int mode, int grad, int push,
                                                   const Offsets* offs, const int32_t* gpos_g,
                                                   const uint8_t** srcs, float* ws) {
  const unsigned full = 0xffffffffu, lt = (1u << lane) - 1u;
  int n = 0;
  if (mode != 1) {   // weighted expert rows on this GPU (every pick in mode 0), k order
    bool v = false;
    const uint8_t* ptr = nullptr;
    float wk = 1.f;
    if (lane < w.K) {
      const int e = ids[t * w.K + lane];
      const int ep = epos[t * w.K + lane];
      if (e >= 0 && ep >= 0) {
        const int d = rank_of_slot(w, e);
        if (!(mode >= 2 && d / w.L != w.p)) {
          v = true;
          ptr = (grad ? w.gx[d] : w.ymaj[d]) + (int64_t)ep * w.row_bytes;
          if (!grad) wk = wts[t * w.K + lane];
        }
      }
    }
    const unsigned b = __ballot_sync(full, v);
    if (v) {
      const int pos = __popc(b & lt);
      srcs[pos] = ptr;
      ws[pos] = wk;
    }
    n = __popc(b);
  }
  if (mode == 3) {   // pre-reduced rows returned by the other GPUs hit, ascending GPU
    bool v = false;
    const uint8_t* ptr = nullptr;
    if (lane < w.P && lane != w.p) {
      const unsigned long long gmask = w.L >= 64 ? ~0ull : ((1ull << w.L) - 1ull);
      if ((hitmask[t] >> (lane * w.L)) & gmask) {
        const int g = gpos_g[t * w.P + lane];
        if (g >= 0) {
          const int s_loc = (int)(t / w.T_r);
          const int64_t pos = g - offs->off_g[s_loc][lane];
          ptr = w.ret_g[w.p * w.L + s_loc] + ((int64_t)lane * w.T_r + pos) * w.row_bytes;
          v = true;
        }
      }
    }
    const unsigned b = __ballot_sync(full, v);
    if (v) {
      const int pos = n + __popc(b & lt);
      srcs[pos] = ptr;
      ws[pos] = 1.f;
    }
    n += __popc(b);
  }
  if (mode == 1 || mode == 2) {   // partial rows of dedup destinations, ascending rank
    const unsigned long long hit = hitmask[t];
    for (int d0 = 0; d0 < w.G; d0 += 32) {
      const int d = d0 + lane;
      bool v = false;
      const uint8_t* ptr = nullptr;
      if (d < w.G && ((hit >> d) & 1ull) && !(mode == 2 && d / w.L == w.p)) {
        const int g = gpos[t * w.G + d];
        if (g >= 0 && g < w.R_cap) {
          v = true;
          if (push) {
            const int s_loc = (int)(t / w.T_r);
            const int64_t pos = g - offs->off[s_loc][d];
            ptr = w.ret[w.p * w.L + s_loc] + ((int64_t)d * w.T_r + pos) * w.row_bytes;
          } else {
            ptr = w.comb[d] + (int64_t)g * w.row_bytes;
          }
        }
      }
      const unsigned b = __ballot_sync(full, v);
      if (v) {
        const int pos = n + __popc(b & lt);
        srcs[pos] = ptr;
        ws[pos] = 1.f;
      }
      n += __popc(b);
    }
  }
  return n;
}

constexpr int kMaxSrc = kMaxRanks > kMaxK ? kMaxRanks : kMaxK;

template <typename T, int VPL>
__global__ void __launch_bounds__(256, 3) k_gather(const WorldDev* __restrict__ wp,
                                                const int32_t* __restrict__ ids,
                                                const float* __restrict__ wts,
                                                const unsigned long long* __restrict__ hitmask,
                                                const int32_t* __restrict__ gpos,
                                                const int32_t* __restrict__ epos, int mode,
                                                int grad, int push,
                                                const Offsets* __restrict__ offs,
                                                const int32_t* __restrict__ gpos_g,
                                                uint8_t* __restrict__ out,
                                                const uint8_t* __restrict__ addend) {
  const WorldDev& w = *wp;
  const int lane = threadIdx.x & 31;
  const int64_t nvec = w.row_bytes / 16;
  const int64_t ntok = (int64_t)w.L * w.T_r;
  int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  __shared__ const uint8_t* s_src[8][kMaxSrc];
  __shared__ float s_w[8][kMaxSrc];
  const uint8_t** srcs = s_src[threadIdx.x >> 5];
  float* ws = s_w[threadIdx.x >> 5];
  for (int64_t t = warp; t < ntok; t += nw) {
    __syncwarp();
    int n = gather_sources_warp(w, t, lane, ids, wts, hitmask, gpos, epos, mode, grad, push,
                                offs, gpos_g, srcs, ws);
    if (addend) {   // e.g. the shared expert's output, added last in fp32
      srcs[n] = addend + t * w.row_bytes;
      ws[n] = 1.f;
      ++n;
    }
    __syncwarp();
    weighted_row_sum<T, VPL>(srcs, ws, n, nvec, lane,
                             reinterpret_cast<int4*>(out + t * w.row_bytes));
  }
}

// mode 3 destination side: rows received by this GPU (one per token x GPU)
// re-expanded into the local ranks' expert-major rows (xmaj is [L][N_cap]
// contiguous, meta epos = l * N_cap + row) ...
__global__ void __launch_bounds__(256) k_expand_g(const WorldDev* __restrict__ wp,
                                                  const Offsets* __restrict__ offs) {
  const WorldDev& w = *wp;
  const int lane = threadIdx.x & 31;
  const int64_t nvec = w.row_bytes / 16;
  int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t total = offs->R_g;
  uint8_t* xbase = w.xmaj[w.p * w.L];
  const RowMeta* meta = w.meta_g[w.p];
  for (int64_t r = warp; r < total; r += nw) {
    int ep = -1;
    if (lane < w.K) ep = meta[r * w.K + lane].epos;
    // the sender stored the row in its first pick's slot: copy it to the others
    const unsigned on = __ballot_sync(0xffffffffu, ep >= 0);
    if (__popc(on) < 2) continue;
    const int k0 = __ffs(on) - 1;
    const int e0 = __shfl_sync(0xffffffffu, ep, k0);
    const int4* src = reinterpret_cast<const int4*>(xbase + (int64_t)e0 * w.row_bytes);
    for (int64_t v0 = 0; v0 < nvec; v0 += 32 * kUnroll) {
      int4 buf[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        int64_t v = v0 + u * 32 + lane;
        if (v < nvec) buf[u] = ld_v4(src + v);
      }
      for (int k = k0 + 1; k < w.K; ++k) {
        int e = __shfl_sync(0xffffffffu, ep, k);
        if (e < 0) continue;
        int4* dst = reinterpret_cast<int4*>(xbase + (int64_t)e * w.row_bytes);
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          int64_t v = v0 + u * 32 + lane;
          if (v < nvec) st_na_v4(dst + v, buf[u]);
        }
      }
    }
  }
}

// Fused dispatch at N > 1: the received rows stay in the receive buffers and
// every local pick they carry gets the row's index in the receive space
// (encoded ~r, so xidx >= 0 = local token, < 0 = received row): mode 3 rows
// of recv_g (meta epos = l * N_cap + row), mode 2 rows of recv_x [L][R_cap]
// (meta epos = row of rank l).  Replaces the row copies of k_expand(_g).
__global__ void __launch_bounds__(256) k_index_recv_g(const WorldDev* __restrict__ wp,
                                                      const Offsets* __restrict__ offs,
                                                      int32_t* __restrict__ xidx) {
  const WorldDev& w = *wp;
  const RowMeta* meta = w.meta_g[w.p];
  const int64_t n = (int64_t)offs->R_g * w.K;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int ep = meta[i].epos;
    if (ep >= 0) xidx[ep] = ~(int32_t)(i / w.K);
  }
}

__global__ void __launch_bounds__(256) k_index_recv(const WorldDev* __restrict__ wp,
                                                    const Offsets* __restrict__ offs,
                                                    int32_t* __restrict__ xidx) {
  const WorldDev& w = *wp;
  for (int l = 0; l < w.L; ++l) {
    const RowMeta* meta = w.recv_meta[w.p * w.L + l];
    const int64_t n = (int64_t)offs->R[l] * w.K;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
      const int ep = meta[i].epos;
      if (ep >= 0) xidx[(int64_t)l * w.N_cap + ep] = ~(int32_t)(l * w.R_cap + i / w.K);
    }
  }
}

// ... and pre-reduced (sum_k w_k y_k over this GPU's picks), pushed straight
// into the source rank's return buffer slot [this GPU][position]
template <typename T, int VPL>
__global__ void __launch_bounds__(256, 3) k_reduce_g(const WorldDev* __restrict__ wp,
                                                     const Offsets* __restrict__ offs, int grad) {
  const WorldDev& w = *wp;
  __shared__ const uint8_t* s_src[8][kMaxK];
  __shared__ float s_w[8][kMaxK];
  const uint8_t** srcs = s_src[threadIdx.x >> 5];
  float* ws = s_w[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  const int64_t nvec = w.row_bytes / 16;
  int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t total = offs->R_g;
  const uint8_t* ybase = grad ? w.gx[w.p * w.L] : w.ymaj[w.p * w.L];
  const RowMeta* meta = w.meta_g[w.p];
  for (int64_t i = warp; i < total; i += nw) {
    const int64_t r = spread_index(i, total);
    __syncwarp();
    const int n = meta_sources_warp(meta + r * w.K, w.K, ybase, w.row_bytes, grad, lane, srcs,
                                    ws);
    int src = 0;
    while (src + 1 < w.G && offs->offd_g[src + 1] <= r) ++src;
    const int64_t pos = r - offs->offd_g[src];
    uint8_t* out_row = w.ret_g[src] + ((int64_t)w.p * w.T_r + pos) * w.row_bytes;
    __syncwarp();
    weighted_row_sum<T, VPL>(srcs, ws, n, nvec, lane, reinterpret_cast<int4*>(out_row));
  }
}

// relay -> phase-2 inputs: per local relay rank, received row i carries the
// token's picks inside this rank's group (slot ids, -1 elsewhere) + gates;
// rows past the received count are padding (-1).
__global__ void k_relay_ids(const WorldDev* __restrict__ wp, const Offsets* __restrict__ offs,
                            int32_t* __restrict__ ids2, float* __restrict__ w2) {
  const WorldDev& w = *wp;
  const int64_t n = (int64_t)w.L * w.R_cap * w.K;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / w.K;
    const int k = (int)(i % w.K);
    const int l = (int)(row / w.R_cap);
    const int64_t r = row % w.R_cap;
    int32_t id = -1;
    float wt = 0.f;
    if (r < offs->R[l]) {
      RowMeta m = w.recv_meta[w.p * w.L + l][r * w.K + k];
      id = m.epos;
      wt = m.w;
    }
    ids2[i] = id;
    w2[i] = wt;
  }
}


// ---------------------------------------------------------------------------
// backward (K8).  Combine backward = dedup broadcast of the output gradient g
// replaying the forward plan (same gpos/epos): direct picks get
// gy[epos] = w_k g and their gate grad <g, y_k>; dedup destinations get g once
// and scale per local pick there (k_expand_grad).  Dispatch backward = the
// combine machinery with unit weights over gx (k_reduce/k_gather grad=1).
template <typename T>
__global__ void __launch_bounds__(256) k_pack_grad(const WorldDev* __restrict__ wp,
                                                   const uint8_t* __restrict__ g,
                                                   const int32_t* __restrict__ ids,
                                                   const float* __restrict__ wts,
                                                   const unsigned long long* __restrict__ hitmask,
                                                   const int32_t* __restrict__ gpos,
                                                   const int32_t* __restrict__ epos, int mode,
                                                   const int32_t* __restrict__ gpos_g,
                                                   float* __restrict__ dw) {
  const WorldDev& w = *wp;
  const int lane = threadIdx.x & 31;
  const int64_t nvec = w.row_bytes / 16;
  const int64_t ntok = (int64_t)w.L * w.T_r;
  int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  const bool spread = mode == 3 && w.P > 1;   // NVLink stores all over the peers' buffers
  for (int64_t i = warp; i < ntok; i += nw) {
    const int64_t t = spread ? spread_index(i, ntok) : i;
    // direct picks (scaled rows + dot products) and dedup destinations (raw rows)
    int nd = 0, nr = 0;
    uint8_t* drow[kMaxK];
    const uint8_t* yrow[kMaxK];
    float dwk[kMaxK];
    int dk[kMaxK];
    uint8_t* rrow[kMaxRanks];
    if (mode != 1) {
      for (int k = 0; k < w.K; ++k) {
        int e = ids[t * w.K + k], ep = epos[t * w.K + k];
        if (e < 0 || ep < 0) continue;
        const int d = rank_of_slot(w, e);
        if (mode >= 2 && d / w.L != w.p) continue;
        drow[nd] = w.gy[d] + (int64_t)ep * w.row_bytes;
        yrow[nd] = w.ymaj[d] + (int64_t)ep * w.row_bytes;
        dwk[nd] = wts[t * w.K + k];
        dk[nd] = k;
        ++nd;
      }
    }
    if (mode == 3) {   // one row per other GPU hit, into its GPU-level row space of comb
      for (int q = 0; q < w.P; ++q) {
        if (q == w.p) continue;
        const int gp = gpos_g[t * w.P + q];
        if (gp >= 0 && gp < w.Rg_cap) rrow[nr++] = w.comb[q * w.L] + (int64_t)gp * w.row_bytes;
      }
    } else if (mode != 0) {
      unsigned long long hit = hitmask[t];
      for (int d = 0; d < w.G; ++d) {
        if (!((hit >> d) & 1ull)) continue;
        if (mode == 2 && d / w.L == w.p) continue;
        int gp = gpos[t * w.G + d];
        if (gp < 0) continue;
        // gradient rows go to comb (free in push-combine worlds), not recv_x:
        // the fused dispatch's backward still gathers x rows from recv_x
        rrow[nr++] = w.comb[d] + (int64_t)gp * w.row_bytes;
      }
    }
    float dot[kMaxK];
#pragma unroll
    for (int j = 0; j < kMaxK; ++j) dot[j] = 0.f;
    const int4* src = reinterpret_cast<const int4*>(g + t * w.row_bytes);
    for (int64_t v = lane; v < nvec; v += 32) {
      int4 gv = src[v];
      float gf[Vec<T>::N];
      Vec<T>::to_f32(gv, gf);
      for (int j = 0; j < nr; ++j) st_na_v4(reinterpret_cast<int4*>(rrow[j]) + v, gv);
#pragma unroll
      for (int j = 0; j < kMaxK; ++j) {
        if (j >= nd) break;
        float yf[Vec<T>::N], sf[Vec<T>::N];
        Vec<T>::to_f32(ld_v4(reinterpret_cast<const int4*>(yrow[j]) + v), yf);
#pragma unroll
        for (int q = 0; q < Vec<T>::N; ++q) {
          dot[j] = fmaf(gf[q], yf[q], dot[j]);
          sf[q] = dwk[j] * gf[q];
        }
        st_na_v4(reinterpret_cast<int4*>(drow[j]) + v, Vec<T>::from_f32(sf));
      }
    }
#pragma unroll
    for (int j = 0; j < kMaxK; ++j) {
      if (j >= nd) break;
      float x = dot[j];
      for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      if (lane == 0) dw[t * w.K + dk[j]] = x;
    }
  }
}

// Combine backward when every pick is direct (mode 0, or per-GPU dedup on one
// GPU): warp per token, lane k holds pick k's gy / y row pointers and weight
// (broadcast by shuffle, so no per-thread pointer arrays in local memory), the
// gradient row is staged kGradU 16-B vectors per lane at a time and each
// pick's y vectors are all loaded before its first store.  Same per-lane
// accumulation order as k_pack_grad, so gy and the gate grads are bit-identical.
constexpr int kGradU = 8;
template <typename T>
__global__ void __launch_bounds__(256) k_pack_grad_direct(const WorldDev* __restrict__ wp,
                                                          const uint8_t* __restrict__ g,
                                                          const int32_t* __restrict__ ids,
                                                          const float* __restrict__ wts,
                                                          const int32_t* __restrict__ epos,
                                                          float* __restrict__ dw) {
  const WorldDev& w = *wp;
  const int lane = threadIdx.x & 31;
  const int64_t nvec = w.row_bytes / 16;
  const int64_t ntok = (int64_t)w.L * w.T_r;
  int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t t = warp; t < ntok; t += nw) {
    const int4* yl = nullptr;
    int4* dl = nullptr;
    float wl = 0.f;
    if (lane < w.K) {
      const int e = ids[t * w.K + lane], ep = epos[t * w.K + lane];
      if (e >= 0 && ep >= 0) {
        const int d = rank_of_slot(w, e);
        yl = reinterpret_cast<const int4*>(w.ymaj[d] + (int64_t)ep * w.row_bytes);
        dl = reinterpret_cast<int4*>(w.gy[d] + (int64_t)ep * w.row_bytes);
        wl = wts[t * w.K + lane];
      }
    }
    float dot[kMaxK];
#pragma unroll
    for (int j = 0; j < kMaxK; ++j) dot[j] = 0.f;
    const int4* src = reinterpret_cast<const int4*>(g + t * w.row_bytes);
    for (int64_t base = 0; base < nvec; base += 32 * kGradU) {
      int4 gv[kGradU];
#pragma unroll
      for (int u = 0; u < kGradU; ++u) {
        const int64_t v = base + u * 32 + lane;
        if (v < nvec) gv[u] = ld_nc_v4(src + v);
      }
#pragma unroll
      for (int j = 0; j < kMaxK; ++j) {
        if (j >= w.K) break;
        const int4* yr = reinterpret_cast<const int4*>(
            __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(yl), j));
        int4* dr = reinterpret_cast<int4*>(
            __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(dl), j));
        const float wk = __shfl_sync(0xffffffffu, wl, j);
        if (!yr) continue;
        int4 yv[kGradU];
#pragma unroll
        for (int u = 0; u < kGradU; ++u) {
          const int64_t v = base + u * 32 + lane;
          if (v < nvec) yv[u] = ld_nc_v4(yr + v);
        }
#pragma unroll
        for (int u = 0; u < kGradU; ++u) {
          const int64_t v = base + u * 32 + lane;
          if (v >= nvec) break;
          float gf[Vec<T>::N], yf[Vec<T>::N], sf[Vec<T>::N];
          Vec<T>::to_f32(gv[u], gf);
          Vec<T>::to_f32(yv[u], yf);
#pragma unroll
          for (int q = 0; q < Vec<T>::N; ++q) {
            dot[j] = fmaf(gf[q], yf[q], dot[j]);
            sf[q] = wk * gf[q];
          }
          st_na_v4(dr + v, Vec<T>::from_f32(sf));
        }
      }
    }
#pragma unroll
    for (int j = 0; j < kMaxK; ++j) {
      if (j >= w.K) break;
      float x = dot[j];
      for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      if (lane == j && yl) dw[t * w.K + j] = x;
    }
  }
}

// destination: received gradient row -> scaled rows for each local pick, and
// the pick's gate gradient <g, y_k> into gw[row][k]
template <typename T>
__global__ void __launch_bounds__(256) k_expand_grad(const WorldDev* __restrict__ wp,
                                                     const Offsets* __restrict__ offs) {
  const WorldDev& w = *wp;
  const int lane = threadIdx.x & 31;
  const int64_t nvec = w.row_bytes / 16;
  int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  int64_t total = 0;
  for (int d = 0; d < w.L; ++d) total += offs->R[d];
  for (int64_t i = warp; i < total; i += nw) {
    int d_loc = 0;
    int64_t r = i;
    while (r >= offs->R[d_loc]) {
      r -= offs->R[d_loc];
      ++d_loc;
    }
    const int dg = w.p * w.L + d_loc;
    int nd = 0;
    int eps[kMaxK], ks[kMaxK];
    float wk[kMaxK];
    for (int k = 0; k < w.K; ++k) {
      RowMeta m = w.recv_meta[dg][r * w.K + k];
      if (m.epos < 0) continue;
      eps[nd] = m.epos;
      wk[nd] = m.w;
      ks[nd] = k;
      ++nd;
    }
    float dot[kMaxK];
#pragma unroll
    for (int j = 0; j < kMaxK; ++j) dot[j] = 0.f;
    const int4* src = reinterpret_cast<const int4*>(w.comb[dg] + r * w.row_bytes);
    for (int64_t v = lane; v < nvec; v += 32) {
      float gf[Vec<T>::N];
      Vec<T>::to_f32(ld_nc_v4(src + v), gf);
#pragma unroll
      for (int j = 0; j < kMaxK; ++j) {
        if (j >= nd) break;
        float yf[Vec<T>::N], sf[Vec<T>::N];
        Vec<T>::to_f32(ld_nc_v4(reinterpret_cast<const int4*>(w.ymaj[dg] + (int64_t)eps[j] * w.row_bytes) + v), yf);
#pragma unroll
        for (int q = 0; q < Vec<T>::N; ++q) {
          dot[j] = fmaf(gf[q], yf[q], dot[j]);
          sf[q] = wk[j] * gf[q];
        }
        st_na_v4(reinterpret_cast<int4*>(w.gy[dg] + (int64_t)eps[j] * w.row_bytes) + v,
                 Vec<T>::from_f32(sf));
      }
    }
#pragma unroll
    for (int j = 0; j < kMaxK; ++j) {
      if (j >= nd) break;
      float x = dot[j];
      for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      if (lane == 0) w.gw[dg][r * w.K + ks[j]] = x;
    }
  }
}

// ... per-GPU dedup (mode 3): received gradient row r (the GPU-level row space
// of comb, same positions as the forward's recv_g rows) -> scaled rows for
// each of its picks on this GPU (meta_g epos = l * N_cap + row, flat over the
// local ranks) and their gate gradients into the flat gw rows
template <typename T>
__global__ void __launch_bounds__(256) k_expand_grad_g(const WorldDev* __restrict__ wp,
                                                       const Offsets* __restrict__ offs) {
  const WorldDev& w = *wp;
  const int lane = threadIdx.x & 31;
  const int64_t nvec = w.row_bytes / 16;
  int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t total = offs->R_g;
  const RowMeta* meta = w.meta_g[w.p];
  const uint8_t* ybase = w.ymaj[w.p * w.L];
  uint8_t* gbase = w.gy[w.p * w.L];
  float* gw = w.gw[w.p * w.L];
  for (int64_t r = warp; r < total; r += nw) {
    int nd = 0;
    int eps[kMaxK], ks[kMaxK];
    float wk[kMaxK];
    for (int k = 0; k < w.K; ++k) {
      RowMeta m = meta[r * w.K + k];
      if (m.epos < 0) continue;
      eps[nd] = m.epos;
      wk[nd] = m.w;
      ks[nd] = k;
      ++nd;
    }
    float dot[kMaxK];
#pragma unroll
    for (int j = 0; j < kMaxK; ++j) dot[j] = 0.f;
    const int4* src = reinterpret_cast<const int4*>(w.comb[w.p * w.L] + r * w.row_bytes);
    for (int64_t v = lane; v < nvec; v += 32) {
      float gf[Vec<T>::N];
      Vec<T>::to_f32(ld_nc_v4(src + v), gf);
#pragma unroll
      for (int j = 0; j < kMaxK; ++j) {
        if (j >= nd) break;
        float yf[Vec<T>::N], sf[Vec<T>::N];
        Vec<T>::to_f32(ld_nc_v4(reinterpret_cast<const int4*>(ybase + (int64_t)eps[j] * w.row_bytes) + v), yf);
#pragma unroll
        for (int q = 0; q < Vec<T>::N; ++q) {
          dot[j] = fmaf(gf[q], yf[q], dot[j]);
          sf[q] = wk[j] * gf[q];
        }
        st_na_v4(reinterpret_cast<int4*>(gbase + (int64_t)eps[j] * w.row_bytes) + v,
                 Vec<T>::from_f32(sf));
      }
    }
#pragma unroll
    for (int j = 0; j < kMaxK; ++j) {
      if (j >= nd) break;
      float x = dot[j];
      for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      if (lane == 0) gw[r * w.K + ks[j]] = x;
    }
  }
}

// source: gate grads of dedup picks from the destination's gw rows (peer loads)
__global__ void k_gate_grad(const WorldDev* __restrict__ wp, const int32_t* __restrict__ ids,
                            const int32_t* __restrict__ gpos, int mode,
                            const int32_t* __restrict__ gpos_g, float* __restrict__ dw) {
  const WorldDev& w = *wp;
  const int64_t n = (int64_t)w.L * w.T_r * w.K;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i / w.K;
    const int k = (int)(i % w.K);
    const int e = ids[i];
    if (e < 0 || mode == 0) continue;
    const int d = rank_of_slot(w, e);
    if (mode >= 2 && d / w.L == w.p) continue;   // direct pick: k_pack_grad wrote it
    if (mode == 3) {   // the pick's GPU q wrote it at its GPU-level row of this token
      const int q = d / w.L;
      const int gp = gpos_g[t * w.P + q];
      if (gp >= 0) dw[i] = w.gw[q * w.L][(int64_t)gp * w.K + k];
      continue;
    }
    const int gp = gpos[t * w.G + d];
    if (gp >= 0) dw[i] = w.gw[d][(int64_t)gp * w.K + k];
  }
}

// Row groups of this GPU's expert-major layout split by where the rows come
// from (the overlapped forward, hm_experts_overlap).  An expert's rows start
// with the ones from this GPU's sources (k_notify's rotated order): group
// l*E_loc + j = the whole 256-row tiles of those, group L*E_loc + l*E_loc + j =
// the rest (the partial local tile + the rows that crossed NVLink), so the
// split adds no partial tile.  Row starts in the flat [L][N_cap] space,
// weight index l*E_loc + j.
__global__ void k_ffn_groups(const WorldDev* __restrict__ wp, const int32_t* __restrict__ n_e,
                             int32_t* __restrict__ row0, int32_t* __restrict__ rows,
                             int32_t* __restrict__ wsel) {
  const WorldDev& w = *wp;
  const int L = w.L, El = w.E_loc, C = w.G + w.E + w.P, nl = L * El;
  const int32_t* cnt = w.counts[w.p * L];
  for (int i = threadIdx.x; i < nl; i += blockDim.x) {
    const int l = i / El, j = i - l * El;
    const int e = (w.p * L + l) * El + j;
    int base = 0;
    for (int j2 = 0; j2 < j; ++j2) base += n_e[e - j + j2];
    int local = 0;
    for (int src = w.p * L; src < (w.p + 1) * L; ++src) local += cnt[(int64_t)src * C + w.G + e];
    const int whole = local / 256 * 256;
    const int r0 = l * (int)w.N_cap + base;
    row0[i] = r0;
    rows[i] = whole;
    wsel[i] = i;
    row0[nl + i] = r0 + whole;
    rows[nl + i] = n_e[e] - whole;
    wsel[nl + i] = i;
  }
}

}  // namespace

// ===========================================================================
// world object (host side)
// ===========================================================================

struct hm_world {
  WorldDev h;            // host copy of the device table
  WorldDev* d = nullptr;
  int device = 0;
  uint8_t* sym = nullptr;  // symmetric allocation (this GPU)
  size_t sym_bytes = 0;
  size_t off_recv_x = 0, off_meta = 0, off_xmaj = 0, off_ymaj = 0, off_comb = 0, off_counts = 0,
         off_flags = 0, off_gy = 0, off_gx = 0, off_gw = 0, off_ret = 0, off_recv_g = 0,
         off_meta_g = 0, off_ret_g = 0;
  bool grad = false;
  std::vector<void*> opened;  // peer bases opened via IPC
  // local scratch
  int nchunks = 0;
  int32_t* chunk_cnt = nullptr;
  int32_t* rank_d = nullptr;
  int32_t* rank_e = nullptr;
  unsigned long long* hitmask = nullptr;
  int32_t* gpos = nullptr;
  int32_t* epos = nullptr;
  int32_t* rank_g = nullptr;   // mode 3: within-chunk rank per destination GPU
  int32_t* gpos_g = nullptr;   // mode 3: receive row per (token, destination GPU)
  Offsets* offs = nullptr;
  int32_t* eoff = nullptr;
  int32_t* n_e = nullptr;
  int* status = nullptr;
  int max_blocks = 0;          // hm_world_set_option(w, 4, n): grid cap of the exchange kernels
  // hm_world_set_option(w, 10, 1): fused one-GPU dispatch -- row indices
  // instead of expert-major row copies (the expert GEMM gathers)
  bool fused = false;
  int32_t* xidx = nullptr;     // [L][N_cap] source row of every expert-major row
  // overlapped forward (hm_dispatch_meta + hm_experts_overlap): exchange
  // descriptor (device), row groups [3][2 * L * E_loc], and the step's state
  hm::ExchWork* exch = nullptr;
  int32_t* grp = nullptr;
  bool meta_only = false;      // hm_dispatch_meta ran: rows not yet moved
  unsigned long long* epoch_ctr = nullptr;   // device barrier epoch counter
  bool peers_ready = false;
  int last_mode = 0;
  // optional per-kernel CUDA-event timing (segments recorded on the launch stream)
  bool timing = false;
  cudaEvent_t ev[2 * 16];
  float seg_ms[16] = {0};
  int seg_used[16] = {0};
};

// grid of the grid-stride exchange kernels: 8 CTAs per SM, or the caller's
// cap (leaves SMs to concurrent kernels, e.g. another micro-batch's GEMMs)
static inline int exch_blocks(const hm_world* w) {
  return w->max_blocks > 0 ? w->max_blocks : kSMs * 8;
}

// segment ids for hm_world_timings
enum Seg { kSegPlan, kSegNotify, kSegPack, kSegBarrier1, kSegExpand, kSegReduce, kSegBarrier2,
           kSegGather, kSegFfnLocal, kSegFfnRest, kSegCount };

struct SegScope {
  hm_world* w;
  int id;
  cudaStream_t s;
  SegScope(hm_world* w_, int id_, cudaStream_t s_) : w(w_), id(id_), s(s_) {
    if (w->timing) cudaEventRecord(w->ev[2 * id], s);
  }
  ~SegScope() {
    if (w->timing) {
      cudaEventRecord(w->ev[2 * id + 1], s);
      w->seg_used[id] = 1;
    }
  }
};

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

static void fill_tables(hm_world* w, int q, uint8_t* base) {
  // virtual ranks q*L .. q*L+L-1 live on GPU q at `base`
  WorldDev& h = w->h;
  for (int l = 0; l < h.L; ++l) {
    int d = q * h.L + l;
    h.recv_x[d] = base + w->off_recv_x + (size_t)l * h.R_cap * h.row_bytes;
    h.recv_meta[d] = reinterpret_cast<RowMeta*>(base + w->off_meta) + (size_t)l * h.R_cap * h.K;
    h.xmaj[d] = base + w->off_xmaj + (size_t)l * h.N_cap * h.row_bytes;
    h.ymaj[d] = base + w->off_ymaj + (size_t)l * h.N_cap * h.row_bytes;
    h.comb[d] = base + w->off_comb + (size_t)l * h.R_cap * h.row_bytes;
    h.ret[d] = base + w->off_ret + (size_t)l * h.G * h.T_r * h.row_bytes;
    h.ret_g[d] = base + w->off_ret_g + (size_t)l * h.P * h.T_r * h.row_bytes;
    h.gy[d] = w->grad ? base + w->off_gy + (size_t)l * h.N_cap * h.row_bytes : nullptr;
    h.gx[d] = w->grad ? base + w->off_gx + (size_t)l * h.N_cap * h.row_bytes : nullptr;
    h.gw[d] = w->grad ? reinterpret_cast<float*>(base + w->off_gw) + (size_t)l * h.R_cap * h.K
                      : nullptr;
    h.counts[d] = reinterpret_cast<int32_t*>(base + w->off_counts);
    h.flags[d] = reinterpret_cast<unsigned long long*>(base + w->off_flags);
  }
  h.recv_g[q] = base + w->off_recv_g;
  h.meta_g[q] = reinterpret_cast<RowMeta*>(base + w->off_meta_g);
}

HM_API int hm_world_create(int32_t ranks, int32_t gpus, int32_t gpu_index, int32_t experts,
                           int32_t top_k, int32_t hidden, int32_t elem_bytes,
                           int64_t tokens_per_rank, int64_t n_cap_rows, int32_t relay_groups,
                           int32_t flags, hm_world** out) {
  HM_CHECK_ARG(out, "hm_world_create: null out");
  *out = nullptr;
  HM_CHECK_ARG(ranks >= 1 && ranks <= kMaxRanks, "ranks must be 1..%d", kMaxRanks);
  HM_CHECK_ARG(gpus >= 1 && ranks % gpus == 0, "ranks (%d) must be a multiple of gpus (%d)", ranks, gpus);
  HM_CHECK_ARG(gpu_index >= 0 && gpu_index < gpus, "gpu_index out of range");
  HM_CHECK_ARG(experts >= ranks && experts % ranks == 0,
               "experts (%d) must be a positive multiple of the rank count (%d)", experts, ranks);
  HM_CHECK_ARG(top_k >= 1 && top_k <= kMaxK && top_k <= experts, "top_k must be 1..%d", kMaxK);
  HM_CHECK_ARG(elem_bytes == 2 || elem_bytes == 4, "elem_bytes must be 2 (bf16) or 4 (fp32)");
  HM_CHECK_ARG(((int64_t)hidden * elem_bytes) % 16 == 0 && hidden > 0,
               "hidden * elem_bytes must be a positive multiple of 16");
  HM_CHECK_ARG(tokens_per_rank >= 1, "tokens_per_rank must be >= 1");
  HM_CHECK_ARG(experts + ranks <= 8192, "experts too large");
  hm_world* w = new hm_world();
  WorldDev& h = w->h;
  memset(&h, 0, sizeof(h));
  h.G = ranks;
  h.P = gpus;
  h.p = gpu_index;
  h.L = ranks / gpus;
  h.E = experts;
  h.K = top_k;
  h.M = hidden;
  h.E_loc = experts / ranks;
  h.e_shift = -1;
  for (int b = 0; b < 31; ++b)
    if ((1 << b) == h.E_loc) h.e_shift = b;
  h.elem = elem_bytes;
  h.T_r = tokens_per_rank;
  h.row_bytes = (int64_t)hidden * elem_bytes;
  h.U1 = relay_groups;
  h.F = relay_groups ? ranks / relay_groups : 0;
  // a relay receives from the U1 ranks sharing its local index; it never
  // builds expert-major rows
  h.R_cap = (int64_t)(relay_groups ? relay_groups : ranks) * tokens_per_rank;
  int64_t worst = (int64_t)ranks * tokens_per_rank * (top_k < h.E_loc ? top_k : h.E_loc);
  h.N_cap = relay_groups ? 1 : (n_cap_rows > 0 && n_cap_rows < worst ? n_cap_rows : worst);
  // mode 3 receive capacity: every token of every rank on another GPU
  h.Rg_cap = (int64_t)(ranks - h.L) * tokens_per_rank;
  if (h.Rg_cap < 1 || relay_groups) h.Rg_cap = 1;
  HM_CHECK_ARG(h.R_cap < (1ll << 31) && h.N_cap < (1ll << 31) && h.Rg_cap < (1ll << 31) &&
                   (int64_t)h.L * h.N_cap < (1ll << 31),
               "row capacity exceeds int32");
  cudaGetDevice(&w->device);

  size_t o = 0;
  w->off_recv_x = o; o = align_up(o + (size_t)h.L * h.R_cap * h.row_bytes, 256);
  w->off_meta = o;   o = align_up(o + (size_t)h.L * h.R_cap * h.K * sizeof(RowMeta), 256);
  w->off_xmaj = o;   o = align_up(o + (size_t)h.L * h.N_cap * h.row_bytes, 256);
  w->off_ymaj = o;   o = align_up(o + (size_t)h.L * h.N_cap * h.row_bytes, 256);
  w->off_comb = o;   o = align_up(o + (size_t)h.L * h.R_cap * h.row_bytes, 256);
  w->off_ret = o;    o = align_up(o + (size_t)(h.U1 ? 0 : h.L * h.G * h.T_r) * h.row_bytes, 256);
  w->off_recv_g = o; o = align_up(o + (size_t)h.Rg_cap * h.row_bytes, 256);
  w->off_meta_g = o; o = align_up(o + (size_t)h.Rg_cap * h.K * sizeof(RowMeta), 256);
  w->off_ret_g = o;  o = align_up(o + (size_t)(h.U1 ? 0 : h.L * h.P * h.T_r) * h.row_bytes, 256);
  w->grad = (flags & 1) != 0;   // backward buffers gy, gx, gw
  if (w->grad) {
    w->off_gy = o; o = align_up(o + (size_t)h.L * h.N_cap * h.row_bytes, 256);
    w->off_gx = o; o = align_up(o + (size_t)h.L * h.N_cap * h.row_bytes, 256);
    w->off_gw = o; o = align_up(o + (size_t)h.L * h.R_cap * h.K * 4, 256);
  }
  w->off_counts = o; o = align_up(o + (size_t)h.G * (h.G + h.E + h.P) * 4, 256);
  w->off_flags = o;  o = align_up(o + (size_t)h.P * 8, 256);
  w->sym_bytes = o;
  int st;
#define HM_TRY(call) do { st = hm::cuda_status(call); if (st) { delete w; return st; } } while (0)
  HM_TRY(cudaMalloc(&w->sym, w->sym_bytes));
  HM_TRY(cudaMemset(w->sym + w->off_counts, 0, w->sym_bytes - w->off_counts));
  w->nchunks = (int)((tokens_per_rank + kChunk - 1) / kChunk);
  const int64_t T = (int64_t)h.L * h.T_r;
  HM_TRY(cudaMalloc(&w->chunk_cnt, (size_t)h.L * w->nchunks * (h.G + h.E + h.P) * 4));
  HM_TRY(cudaMalloc(&w->rank_g, (size_t)T * h.P * 4));
  HM_TRY(cudaMalloc(&w->gpos_g, (size_t)T * h.P * 4));
  HM_TRY(cudaMalloc(&w->rank_d, (size_t)T * h.G * 4));
  HM_TRY(cudaMalloc(&w->rank_e, (size_t)T * h.K * 4));
  HM_TRY(cudaMalloc(&w->hitmask, (size_t)T * 8));
  HM_TRY(cudaMalloc(&w->gpos, (size_t)T * h.G * 4));
  HM_TRY(cudaMalloc(&w->epos, (size_t)T * h.K * 4));
  HM_TRY(cudaMalloc(&w->offs, sizeof(Offsets)));
  HM_TRY(cudaMalloc(&w->eoff, (size_t)h.L * h.E * 4));
  HM_TRY(cudaMalloc(&w->n_e, (size_t)h.E * 4));
  HM_TRY(cudaMalloc(&w->status, 16));
  HM_TRY(cudaMemset(w->status, 0, 16));
  HM_TRY(cudaMalloc(&w->epoch_ctr, 8));
  HM_TRY(cudaMemset(w->epoch_ctr, 0, 8));
  h.epoch_ctr = w->epoch_ctr;
  HM_TRY(cudaMalloc(&w->d, sizeof(WorldDev)));
  fill_tables(w, h.p, w->sym);
  if (h.P == 1) {
    HM_TRY(cudaMemcpy(w->d, &h, sizeof(WorldDev), cudaMemcpyHostToDevice));
    w->peers_ready = true;
  }
#undef HM_TRY
  *out = w;
  return 0;
}

HM_API int hm_world_destroy(hm_world* w) {
  if (!w) return 0;
  if (w->timing)
    for (int i = 0; i < 2 * 16; ++i) cudaEventDestroy(w->ev[i]);
  for (void* p : w->opened) cudaIpcCloseMemHandle(p);
  cudaFree(w->sym);
  cudaFree(w->exch);
  cudaFree(w->grp);
  cudaFree(w->chunk_cnt);
  cudaFree(w->rank_d);
  cudaFree(w->rank_e);
  cudaFree(w->hitmask);
  cudaFree(w->gpos);
  cudaFree(w->epos);
  cudaFree(w->rank_g);
  cudaFree(w->gpos_g);
  cudaFree(w->offs);
  cudaFree(w->eoff);
  cudaFree(w->n_e);
  cudaFree(w->status);
  cudaFree(w->xidx);
  cudaFree(w->epoch_ctr);
  cudaFree(w->d);
  delete w;
  return 0;
}

HM_API int64_t hm_world_ipc_handle_size(void) { return (int64_t)sizeof(cudaIpcMemHandle_t); }

HM_API int hm_world_ipc_handle(hm_world* w, void* out_handle) {
  HM_CHECK_ARG(w && out_handle, "hm_world_ipc_handle: null argument");
  cudaIpcMemHandle_t hnd;
  HM_CUDA(cudaIpcGetMemHandle(&hnd, w->sym));
  memcpy(out_handle, &hnd, sizeof(hnd));
  return 0;
}

// handles: P consecutive cudaIpcMemHandle_t, index = GPU index (own entry ignored)
HM_API int hm_world_open_peers(hm_world* w, const void* handles) {
  HM_CHECK_ARG(w && handles, "hm_world_open_peers: null argument");
  const cudaIpcMemHandle_t* hs = reinterpret_cast<const cudaIpcMemHandle_t*>(handles);
  for (int q = 0; q < w->h.P; ++q) {
    if (q == w->h.p) continue;
    void* base = nullptr;
    HM_CUDA(cudaIpcOpenMemHandle(&base, hs[q], cudaIpcMemLazyEnablePeerAccess));
    w->opened.push_back(base);
    fill_tables(w, q, reinterpret_cast<uint8_t*>(base));
  }
  HM_CUDA(cudaMemcpy(w->d, &w->h, sizeof(WorldDev), cudaMemcpyHostToDevice));
  const WorldDev& h = w->h;
  if (h.P > 1 && !h.U1 && h.P <= hm::kExchMaxGpus && !w->exch) {
    // the overlapped forward's exchange descriptor (pointer tables are fixed
    // per world) and row-group arrays, set up here so the step itself makes no
    // allocation or synchronous copy (CUDA-graph capturable)
    hm::ExchWork e;
    memset(&e, 0, sizeof(e));
    e.P = h.P;
    e.p = h.p;
    e.G = h.G;
    e.K = h.K;
    e.T_r = (int)h.T_r;
    e.nvec = h.row_bytes / 16;
    e.ntok = (int64_t)h.L * h.T_r;
    e.rg_cap = h.Rg_cap;
    e.gpos_g = w->gpos_g;
    for (int q = 0; q < h.P; ++q) e.recv_g[q] = reinterpret_cast<int4*>(h.recv_g[q]);
    HM_CUDA(cudaMalloc(&w->exch, sizeof(hm::ExchWork)));
    HM_CUDA(cudaMemcpy(w->exch, &e, sizeof(e), cudaMemcpyHostToDevice));
    HM_CUDA(cudaMalloc(&w->grp, (size_t)3 * 2 * h.L * h.E_loc * 4));
  }
  w->peers_ready = true;
  return 0;
}

// router kernel choice (hm_route_set_option): quad (4 lanes per token) or
// lane-per-token.  The quad is the default where it applies (renormalised
// weights, E in {32, 64, 128, 256}): 14.7 vs 16.3 us device time for the
// Qwen3 step's 32768 x 128 logits (warm, tools/ctrl_time.py); identical bits.
static int w_route_quad = 1;

HM_API int hm_route_set_option(int32_t quad) {
  w_route_quad = quad != 0;
  return 0;
}

HM_API int hm_route_topk(const float* logits, int64_t T, int32_t E, int32_t K,
                         const int32_t* expert_to_slot, int32_t renormalize, int32_t* slot_ids,
                         float* weights, int32_t* expert_ids, void* stream) {
  HM_RANGE("hm_route_topk");
  HM_CHECK_ARG(E >= 1 && E <= 512, "hm_route_topk: E must be 1..512");
  HM_CHECK_ARG(K >= 1 && K <= kMaxK && K <= E, "hm_route_topk: K must be 1..%d and <= E", kMaxK);
  if (T == 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  // (renormalised weights only: the full-softmax denominator is summed in the
  // lane kernel's column order, which the quad's split sum would not reproduce)
  const bool quad_ok = w_route_quad && renormalize && (E == 128 || E == 256 || E == 64 || E == 32) &&
                       ((uintptr_t)logits & 15) == 0 && K <= 8;
  if (quad_ok) {
    constexpr int kL = 4;   // lanes per token (8: 0.2385 vs 0.2343 ms for the N = 1 step)
    const int blocks = grid_for(T, kRouteWarps * (32 / kL), kSMs * 16);
#define HM_RQ(KK, FF) k_route_quad<KK, FF, kL><<<blocks, 32 * kRouteWarps, 0, s>>>(logits, T, E, expert_to_slot, \
                                                               renormalize, slot_ids, weights, expert_ids)
#define HM_RQ_K(KK)                    \
  case KK:                             \
    if (E == 32) HM_RQ(KK, 8 / kL);    \
    else if (E == 64) HM_RQ(KK, 16 / kL);    \
    else if (E == 128) HM_RQ(KK, 32 / kL);   \
    else HM_RQ(KK, 64 / kL);                \
    break;
    switch (K) {
      HM_RQ_K(1) HM_RQ_K(2) HM_RQ_K(3) HM_RQ_K(4) HM_RQ_K(5) HM_RQ_K(6) HM_RQ_K(7) HM_RQ_K(8)
    }
#undef HM_RQ_K
#undef HM_RQ
    HM_LAUNCHED();
    return 0;
  }
  if (K <= 8) {
    int blocks = grid_for(T, 256, kSMs * 8);
#define HM_ROUTE_K(KK)                                                                      \
  case KK:                                                                                  \
    if (E % 4 == 0 && ((uintptr_t)logits & 15) == 0)                                        \
      k_route_lane<KK, true><<<blocks, 256, 0, s>>>(logits, T, E, expert_to_slot, renormalize, \
                                                    slot_ids, weights, expert_ids);         \
    else                                                                                    \
      k_route_lane<KK, false><<<blocks, 256, 0, s>>>(logits, T, E, expert_to_slot,          \
                                                     renormalize, slot_ids, weights,        \
                                                     expert_ids);                           \
    break;
    switch (K) {
      HM_ROUTE_K(1) HM_ROUTE_K(2) HM_ROUTE_K(3) HM_ROUTE_K(4)
      HM_ROUTE_K(5) HM_ROUTE_K(6) HM_ROUTE_K(7) HM_ROUTE_K(8)
    }
#undef HM_ROUTE_K
    HM_LAUNCHED();
    return 0;
  }
  int blocks = grid_for(T, 8, kSMs * 16);
  int per = (E + 31) / 32;
  if (per <= 1)
    k_route<1><<<blocks, 256, 0, s>>>(logits, T, E, K, expert_to_slot, renormalize, slot_ids, weights, expert_ids);
  else if (per <= 2)
    k_route<2><<<blocks, 256, 0, s>>>(logits, T, E, K, expert_to_slot, renormalize, slot_ids, weights, expert_ids);
  else if (per <= 4)
    k_route<4><<<blocks, 256, 0, s>>>(logits, T, E, K, expert_to_slot, renormalize, slot_ids, weights, expert_ids);
  else if (per <= 8)
    k_route<8><<<blocks, 256, 0, s>>>(logits, T, E, K, expert_to_slot, renormalize, slot_ids, weights, expert_ids);
  else
    k_route<16><<<blocks, 256, 0, s>>>(logits, T, E, K, expert_to_slot, renormalize, slot_ids, weights, expert_ids);
  HM_LAUNCHED();
  return 0;
}

HM_API int hm_route_group(const float* logits, int64_t T, int32_t E, int32_t K, int32_t n_group,
                          int32_t topk_group, const float* bias, float route_scale,
                          const int32_t* expert_to_slot, int32_t* slot_ids, float* weights,
                          int32_t* expert_ids, void* stream) {
  HM_RANGE("hm_route_group");
  HM_CHECK_ARG(E >= 1 && E <= 512, "hm_route_group: E must be 1..512");
  HM_CHECK_ARG(n_group >= 1 && n_group <= 32 && E % n_group == 0,
               "hm_route_group: n_group must be 1..32 and divide E");
  HM_CHECK_ARG(topk_group >= 1 && topk_group <= n_group, "hm_route_group: bad topk_group");
  HM_CHECK_ARG(K >= 1 && K <= kMaxK && K <= topk_group * (E / n_group),
               "hm_route_group: K must be 1..%d and fit in the kept groups", kMaxK);
  if (T == 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  const int blocks = grid_for(T, 8, kSMs * 8);
  const int per = (E + 31) / 32;
#define HM_RG(P)                                                                              \
  k_route_group<P><<<blocks, 256, 0, s>>>(logits, T, E, K, n_group, topk_group, bias,        \
                                          route_scale, expert_to_slot, slot_ids, weights,   \
                                          expert_ids)
  if (per <= 4)
    HM_RG(4);
  else if (per <= 8)
    HM_RG(8);
  else
    HM_RG(16);
#undef HM_RG
  HM_LAUNCHED();
  return 0;
}

// dispatch: plan + notify (+barrier) + pack + barrier.  x: [L*T_r, M] payload
// rows of this GPU's local source ranks; ids/wts: [L*T_r, K] slot ids + gates.
// The dispatch in two phases (hm_dispatch = both): plan = per-chunk plan +
// count exchange + offsets (k_plan, k_notify); push = the row movement (pack /
// index kernels + device barrier).  The counts are final after the plan, so a
// caller may read them (e.g. the transport choice) before moving any row.
static int dispatch_push(hm_world* w, const void* x, const int32_t* ids, const float* wts,
                         int32_t mode, cudaStream_t s);

HM_API int hm_dispatch_plan(hm_world* w, const int32_t* ids, const float* wts, int32_t mode,
                            void* stream) {
  HM_RANGE("hm_dispatch_plan");
  HM_CHECK_ARG(w && ids, "hm_dispatch: null argument");
  HM_CHECK_ARG(mode >= 0 && mode <= 3,
               "hm_dispatch: mode must be 0 (raw), 1 (dedup per rank), 2 (dedup per remote rank), "
               "3 (dedup per remote GPU)");
  if (mode) HM_CHECK_ARG(wts, "hm_dispatch: dedup modes need gate weights");
  HM_CHECK_ARG(!w->h.U1 || mode == 1, "hm_dispatch: a relay world ships dedup rows (mode 1)");
  w->last_mode = mode;
  if (!w->peers_ready) {
    hm::set_error("hm_dispatch: peers not opened");
    return hm::kNotReady;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const WorldDev& h = w->h;
  dim3 grid(w->nchunks, h.L);
  size_t smem = (size_t)kPlanWarps * (h.G + 2 * h.E + h.P) * 4;
  {SegScope sc(w, kSegPlan, s);
#define HM_PLAN(KK)                                                                          \
  do {                                                                                       \
    if (smem > 48 * 1024)                                                                    \
      HM_CUDA(cudaFuncSetAttribute(k_plan<KK>, cudaFuncAttributeMaxDynamicSharedMemorySize,  \
                                   (int)smem));                                              \
    k_plan<KK><<<grid, kChunk, smem, s>>>(w->d, ids, w->nchunks, w->chunk_cnt, w->rank_d,    \
                                          w->rank_e, w->hitmask, w->rank_g, w->status);      \
  } while (0)
  switch (h.K) {
    case 1: HM_PLAN(1); break;
    case 2: HM_PLAN(2); break;
    case 4: HM_PLAN(4); break;
    case 6: HM_PLAN(6); break;
    case 8: HM_PLAN(8); break;
    default: HM_PLAN(kMaxK); break;
  }
#undef HM_PLAN
  }
  HM_LAUNCHED();
  {SegScope sc(w, kSegNotify, s);
  const size_t cnt_bytes = (size_t)h.G * (h.G + h.E + h.P) * 4;
  const int stage_cnt = ((2 * h.E + h.G) * 4 + cnt_bytes) <= 160 * 1024 ? 1 : 0;
  const size_t nsmem = (size_t)(2 * h.E + h.G) * 4 + (stage_cnt ? cnt_bytes : 0);
  if (nsmem > 48 * 1024)
    HM_CUDA(cudaFuncSetAttribute(k_notify, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)nsmem));
  k_notify<<<1, 1024, nsmem, s>>>(w->d, w->nchunks, w->chunk_cnt, w->offs, w->eoff, w->n_e, mode,
                                  w->status, stage_cnt);
  }
  HM_LAUNCHED();
  return 0;
}

HM_API int hm_dispatch_push(hm_world* w, const void* x, const int32_t* ids, const float* wts,
                            int32_t mode, void* stream) {
  HM_RANGE("hm_dispatch_push");
  HM_CHECK_ARG(w && x && ids, "hm_dispatch_push: null argument");
  HM_CHECK_ARG(mode == w->last_mode, "hm_dispatch_push: mode differs from the plan's");
  return dispatch_push(w, x, ids, wts, mode, (cudaStream_t)stream);
}

HM_API int hm_dispatch(hm_world* w, const void* x, const int32_t* ids, const float* wts,
                       int32_t mode, void* stream) {
  HM_RANGE("hm_dispatch");
  HM_CHECK_ARG(w && x && ids, "hm_dispatch: null argument");
  int st = hm_dispatch_plan(w, ids, wts, mode, stream);
  if (st) return st;
  return dispatch_push(w, x, ids, wts, mode, (cudaStream_t)stream);
}

static int dispatch_push(hm_world* w, const void* x, const int32_t* ids, const float* wts,
                         int32_t mode, cudaStream_t s) {
  const WorldDev& h = w->h;
  const int64_t T = (int64_t)h.L * h.T_r;
  int blocks = grid_for(T, 8, exch_blocks(w));
  const int64_t nv = h.row_bytes / 16;
  const bool local_only = h.P == 1 && mode != 1 && !h.U1;
  HM_CHECK_ARG(!(w->fused && (mode == 1 || (mode == 0 && h.P > 1))),
               "hm_dispatch: the fused dispatch writes expert-major row indices (modes 2, 3; "
               "mode 0 on one GPU)");
  if (local_only && w->fused) {
    SegScope sc(w, kSegPack, s);
    k_index_local<<<grid_for(T * h.K, 256, kSMs * 8), 256, 0, s>>>(
        w->d, ids, w->chunk_cnt, w->rank_e, w->eoff, w->nchunks, w->epos, w->xidx, w->status);
    HM_LAUNCHED();
    return 0;
  }
  if (local_only && (nv == 32 || nv == 64 || nv == 128 || nv == 256)) {
    // one token per warp up to 32 CTAs per SM: the block scheduler keeps
    // every SM full of fresh warps (233 -> 220 us for the Qwen3 N = 1 step
    // vs the 8-per-SM grid-stride grid, tools/pack_grid.py)
    blocks = grid_for(T, 8, w->max_blocks > 0 ? w->max_blocks : kSMs * 32);
    SegScope sc(w, kSegPack, s);
#define HM_PL(V)                                                                             \
  k_pack_local<V><<<blocks, 256, 0, s>>>(w->d, (const uint8_t*)x, ids, w->chunk_cnt, w->rank_e, \
                                         w->eoff, w->nchunks, w->epos, w->status)
    if (nv == 32)
      HM_PL(1);
    else if (nv == 64)
      HM_PL(2);
    else if (nv == 128)
      HM_PL(4);
    else
      HM_PL(8);
#undef HM_PL
  } else {
    SegScope sc(w, kSegPack, s);
    k_pack<<<blocks, 256, 0, s>>>(w->d, (const uint8_t*)x, ids, wts, w->chunk_cnt, w->rank_d,
                                  w->rank_e, w->hitmask, w->offs, w->eoff, w->nchunks, mode,
                                  w->gpos, w->epos, w->rank_g, w->gpos_g, w->status,
                                  w->fused ? w->xidx : nullptr, 1);
  }
  HM_LAUNCHED();
  if (h.P > 1) {
    SegScope sc(w, kSegBarrier1, s);
    k_barrier<<<1, 32, 0, s>>>(w->d, w->status);
    HM_LAUNCHED();
  }
  return 0;
}

HM_API int hm_expand(hm_world* w, void* stream) {
  HM_RANGE("hm_expand");
  HM_CHECK_ARG(w, "hm_expand: null world");
  if (w->h.P == 1 && w->last_mode == 2) return 0;  // every rank shares this GPU: nothing received
  if (w->h.U1) return 0;                             // relay rows are re-dispatched, not expanded
  if (w->last_mode == 3 && w->h.P == 1) return 0;    // one GPU: every row went direct
  int blocks = exch_blocks(w);
  SegScope sc(w, kSegExpand, (cudaStream_t)stream);
  if (w->fused) {   // row indices into the receive buffers instead of row copies
    if (w->last_mode == 3)
      k_index_recv_g<<<blocks, 256, 0, (cudaStream_t)stream>>>(w->d, w->offs, w->xidx);
    else
      k_index_recv<<<blocks, 256, 0, (cudaStream_t)stream>>>(w->d, w->offs, w->xidx);
    HM_LAUNCHED();
    return 0;
  }
  if (w->last_mode == 3)
    k_expand_g<<<blocks, 256, 0, (cudaStream_t)stream>>>(w->d, w->offs);
  else
    k_expand<<<blocks, 256, 0, (cudaStream_t)stream>>>(w->d, w->offs);
  HM_LAUNCHED();
  return 0;
}

// Overlapped forward, step 1 (per-GPU dedup across GPUs, fused dispatch):
// after hm_dispatch_plan, write every pick's position, the receive rows'
// metadata and the local picks' row indices -- but move no rows: they cross
// NVLink inside hm_experts_overlap's first GEMM.
HM_API int hm_dispatch_meta(hm_world* w, const int32_t* ids, const float* wts, void* stream) {
  HM_RANGE("hm_dispatch_meta");
  HM_CHECK_ARG(w && ids && wts, "hm_dispatch_meta: null argument");
  HM_CHECK_ARG(w->last_mode == 3 && w->h.P > 1 && w->fused && !w->h.U1,
               "hm_dispatch_meta: needs a per-GPU dedup plan (mode 3) across GPUs with the "
               "fused dispatch");
  HM_CHECK_ARG(w->h.P <= hm::kExchMaxGpus, "hm_dispatch_meta: at most %d GPUs",
               hm::kExchMaxGpus);
  cudaStream_t s = (cudaStream_t)stream;
  const WorldDev& h = w->h;
  const int64_t T = (int64_t)h.L * h.T_r;
  SegScope sc(w, kSegPack, s);
  k_pack<<<grid_for(T, 8, exch_blocks(w)), 256, 0, s>>>(
      w->d, nullptr, ids, wts, w->chunk_cnt, w->rank_d, w->rank_e, w->hitmask, w->offs, w->eoff,
      w->nchunks, 3, w->gpos, w->epos, w->rank_g, w->gpos_g, w->status, w->xidx, 0);
  HM_LAUNCHED();
  w->meta_only = true;
  return 0;
}

// Overlapped forward, step 2: the expert FFN of this GPU's ranks with the
// dispatch folded into it --
//   GEMM1 over the whole tiles of rows already here (local tokens), its warp 3
//     pushing every token row to the other GPUs hit (exch.cuh);
//   device barrier; received rows get their row indices;
//   GEMM1 over the remaining rows, GEMM2 over all rows.
// hm_combine follows as usual.  x: this GPU's token
// rows (the fused dispatch's source); w13 / w2: [L * E_loc] experts; h [L*N_cap][I],
// y = the world's ymaj; g13 optional pre-activations.  Same rows, same bits as
// hm_dispatch + hm_expand + hm_expert_ffn_multi + hm_combine.
HM_API int hm_experts_overlap(hm_world* w, const void* x, const void* w13, const void* w2,
                              int32_t hidden, int32_t inter, void* h_buf, void* g13,
                              void* stream) {
  HM_RANGE("hm_experts_overlap");
  HM_CHECK_ARG(w && x && w13 && w2 && h_buf, "hm_experts_overlap: null argument");
  HM_CHECK_ARG(w->meta_only, "hm_experts_overlap: call hm_dispatch_meta first");
  const WorldDev& h = w->h;
  HM_CHECK_ARG((int64_t)hidden * 2 == h.row_bytes && h.elem == 2,
               "hm_experts_overlap: bf16 rows of `hidden` features");
  cudaStream_t s = (cudaStream_t)stream;
  const int nl = h.L * h.E_loc;
  HM_CHECK_ARG(nl <= 256, "hm_experts_overlap: at most 256 experts per GPU");
  HM_CHECK_ARG(w->n_e, "hm_experts_overlap: no plan");
  HM_CHECK_ARG(w->exch && w->grp, "hm_experts_overlap: world has no exchange descriptor");
  int32_t* row0 = w->grp;
  int32_t* rows = row0 + 2 * nl;
  int32_t* wsel = rows + 2 * nl;
  k_ffn_groups<<<1, 256, 0, s>>>(w->d, w->n_e, row0, rows, wsel);
  HM_LAUNCHED();
  const int64_t R = (int64_t)h.L * h.N_cap;
  const void* recv = h.recv_g[h.p];
  __nv_bfloat16* y = reinterpret_cast<__nv_bfloat16*>(h.ymaj[h.p * h.L]);
  const int M = hidden, I = inter;
  int st;
  // local rows: GEMM1, pushing the rows to the other GPUs beside the tiles
  {
    SegScope sc(w, kSegFfnLocal, s);
    if ((st = hm::ffn_gemm_groups(x, R, w13, nl, rows, row0, wsel, nl, 2 * I, M, 1, h_buf, I,
                                  g13, w->xidx, (int64_t)h.L * h.T_r, recv, w->exch, 1, x, s)))
      return st;
  }
  {
    SegScope sc(w, kSegBarrier1, s);
    k_barrier<<<1, 32, 0, s>>>(w->d, w->status);
    HM_LAUNCHED();
  }
  {
    SegScope sc(w, kSegExpand, s);
    k_index_recv_g<<<exch_blocks(w), 256, 0, s>>>(w->d, w->offs, w->xidx);
    HM_LAUNCHED();
  }
  // received rows: GEMM1; then GEMM2 over every row (one launch, the
  // hm_expert_ffn_multi layout: rank l's experts at rows l * N_cap ..)
  {
    SegScope sc(w, kSegFfnRest, s);
    if ((st = hm::ffn_gemm_groups(x, R, w13, nl, rows + nl, row0 + nl, wsel + nl, nl, 2 * I, M,
                                  1, h_buf, I, g13, w->xidx, (int64_t)h.L * h.T_r, recv, nullptr,
                                  0, nullptr, s)))
      return st;
    if ((st = hm::ffn_gemm_segments(h_buf, R, w2, nl, w->n_e + h.p * nl, M, I, y, M, h.E_loc,
                                    h.N_cap, s)))
      return st;
  }
  w->meta_only = false;
  return 0;
}

// combine: dedup -> reduce + barrier + gather; raw -> barrier + gather.
// host dispatch of the row-sum kernels on (payload dtype, row width): common
// widths get their own compile-time instantiation, others the generic loop
template <class T>
struct TypeTag {
  using type = T;
};
template <class F>
static void with_row_type(const WorldDev& h, F&& f) {
  auto width = [&](auto t) {
    switch (h.row_bytes / 16) {
      case 32: return f(t, std::integral_constant<int, 1>{});
      case 64: return f(t, std::integral_constant<int, 2>{});
      case 128: return f(t, std::integral_constant<int, 4>{});
      case 256: return f(t, std::integral_constant<int, 8>{});
      case 512: return f(t, std::integral_constant<int, 16>{});
      case 896: return f(t, std::integral_constant<int, 28>{});
      default: return f(t, std::integral_constant<int, 0>{});
    }
  };
  if (h.elem == 2)
    width(TypeTag<__nv_bfloat16>{});
  else
    width(TypeTag<float>{});
}

// `out`: [L*T_r, M] payload rows.
static int combine_impl(hm_world* w, const float* wts, const int32_t* ids, int32_t mode,
                        const void* addend_v, void* out, void* stream) {
  const uint8_t* addend = (const uint8_t*)addend_v;
  HM_CHECK_ARG(w && out, "hm_combine: null argument");
  HM_CHECK_ARG(mode >= 0 && mode <= 3, "hm_combine: mode must be 0..3");
  const int dedup = mode;
  // non-relay worlds push pre-reduced rows to the source (stores over NVLink);
  // a relay's rows are produced by phase 2 and pulled by the source
  const int push = w->h.U1 ? 0 : 1;
  cudaStream_t s = (cudaStream_t)stream;
  const WorldDev& h = w->h;
  if (mode == 3 && h.P > 1) {
    SegScope sc(w, kSegReduce, s);
    with_row_type(h, [&](auto t, auto v) {
      k_reduce_g<typename decltype(t)::type, decltype(v)::value>
          <<<exch_blocks(w), 256, 0, s>>>(w->d, w->offs, 0);
    });
    HM_LAUNCHED();
  }
  if (dedup && mode != 3 && !(h.P == 1 && mode == 2) && !h.U1) {   // relay: rows arrive pre-reduced
    SegScope sc(w, kSegReduce, s);
    with_row_type(h, [&](auto t, auto v) {
      k_reduce<typename decltype(t)::type, decltype(v)::value>
          <<<exch_blocks(w), 256, 0, s>>>(w->d, w->offs, 0, 1);
    });
    HM_LAUNCHED();
  }
  if (mode != 1) HM_CHECK_ARG(wts && ids, "hm_combine: raw/hybrid combine needs ids and weights");
  if (h.P > 1) {
    SegScope sc(w, kSegBarrier2, s);
    k_barrier<<<1, 32, 0, s>>>(w->d, w->status);
    HM_LAUNCHED();
  }
  const int64_t T = (int64_t)h.L * h.T_r;
  int blocks = grid_for(T, 8, exch_blocks(w));
  SegScope sc(w, kSegGather, s);
  with_row_type(h, [&](auto t, auto v) {
    k_gather<typename decltype(t)::type, decltype(v)::value><<<blocks, 256, 0, s>>>(
        w->d, ids, wts, w->hitmask, w->gpos, w->epos, mode, 0, push, w->offs, w->gpos_g,
        (uint8_t*)out, addend);
  });
  HM_LAUNCHED();
  return 0;
}

HM_API int hm_combine(hm_world* w, const float* wts, const int32_t* ids, int32_t mode, void* out,
                      void* stream) {
  HM_RANGE("hm_combine");
  return combine_impl(w, wts, ids, mode, nullptr, out, stream);
}

// combine + an addend row per token (e.g. the shared expert's output), summed
// in fp32 after the routed rows: out = sum_k w_k y_k + addend
// bf16 -> fp32 widening with 16-byte loads and stores (the router GEMM's
// fp32 operand; torch's casting copy runs at ~2.3 TB/s on B200)
__global__ void __launch_bounds__(256) k_bf16_to_f32(const __nv_bfloat16* __restrict__ src,
                                                     float* __restrict__ dst, int64_t n) {
  const int64_t nv = n / 8;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // four independent 16-byte loads in flight per thread
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < nv; i0 += 4 * stride) {
    int4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (i0 + u * stride < nv) v[u] = ld_nc_v4(reinterpret_cast<const int4*>(src) + i0 + u * stride);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = i0 + u * stride;
      if (i >= nv) break;
      float f[8];
      Vec<__nv_bfloat16>::to_f32(v[u], f);
      float4* d = reinterpret_cast<float4*>(dst) + 2 * i;
      d[0] = make_float4(f[0], f[1], f[2], f[3]);
      d[1] = make_float4(f[4], f[5], f[6], f[7]);
    }
  }
  for (int64_t i = nv * 8 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    dst[i] = __bfloat162float(src[i]);
}

// Gate backward: gradient of the router logits from the gate
// weights' gradient dw [T, K], written as a dense bf16 row (the router GEMMs'
// operand).  mode 0: softmax over the K picks (renormalised; Qwen3):
// dlogit[ex_k] = w_k (dw_k - sum_j w_j dw_j); mode 1: softmax over all E:
// dlogit_e = p_e (dp_e - sum p . dp) with dp = dw scattered to the picks;
// mode 2: DeepSeek-V3 normalised sigmoid (w_k = c s_k / S, s = sigmoid):
// dlogit[ex_k] = (c / S) (dw_k - sum_j dw_j w_j / c) s_k (1 - s_k).  Warp per
// token: the lanes zero the row (16-byte stores), then lane k writes pick k.
__global__ void __launch_bounds__(256) k_gate_backward(const float* __restrict__ logits,
                                                       const int32_t* __restrict__ ex,
                                                       const float* __restrict__ w,
                                                       const float* __restrict__ dw, int64_t T,
                                                       int E, int K, int mode, float scale,
                                                       __nv_bfloat16* __restrict__ dlogits, int ld) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < T; t += nw) {
    const float* lg = logits + t * E;
    __nv_bfloat16* out = dlogits + t * ld;
    int e = -1;
    float wk = 0.f, dk = 0.f;
    if (lane < K) {
      e = ex[t * K + lane];
      wk = w[t * K + lane];
      dk = dw[t * K + lane];
    }
    if (mode == 1) {   // softmax over all experts: every entry is nonzero
      float mx = -INFINITY;
      for (int c = lane; c < E; c += 32) mx = fmaxf(mx, lg[c]);
#pragma unroll
      for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      float den = 0.f;
      for (int c = lane; c < E; c += 32) den += __expf(lg[c] - mx);
#pragma unroll
      for (int o = 16; o; o >>= 1) den += __shfl_xor_sync(0xffffffffu, den, o);
      float pd = lane < K && e >= 0 ? __expf(lg[e] - mx) / den * dk : 0.f;
#pragma unroll
      for (int o = 16; o; o >>= 1) pd += __shfl_xor_sync(0xffffffffu, pd, o);
      for (int c0 = 0; c0 < ld; c0 += 32) {   // warp-uniform trip count (shuffles)
        const int c = c0 + lane;
        float dp = 0.f;
        for (int k = 0; k < K; ++k) {
          const int ek = __shfl_sync(0xffffffffu, e, k);
          const float dwk = __shfl_sync(0xffffffffu, dk, k);
          if (ek == c) dp += dwk;
        }
        if (c < E) out[c] = __float2bfloat16(__expf(lg[c] - mx) / den * (dp - pd));
        else if (c < ld) out[c] = __float2bfloat16(0.f);
      }
      continue;
    }
    // sparse modes: zero the row, then the K picks
    for (int c = lane * 8; c < ld; c += 256)
      *reinterpret_cast<int4*>(out + c) = make_int4(0, 0, 0, 0);
    __syncwarp();
    float g = 0.f;
    if (mode == 0) {
      float sdot = lane < K ? wk * dk : 0.f;
#pragma unroll
      for (int o = 16; o; o >>= 1) sdot += __shfl_xor_sync(0xffffffffu, sdot, o);
      g = wk * (dk - sdot);
    } else {   // mode 2
      const float sk = lane < K && e >= 0 ? 1.f / (1.f + __expf(-lg[e])) : 0.f;
      float ssum = sk, sdw = lane < K ? dk * wk : 0.f;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        ssum += __shfl_xor_sync(0xffffffffu, ssum, o);
        sdw += __shfl_xor_sync(0xffffffffu, sdw, o);
      }
      g = (scale / ssum) * (dk - sdw / scale) * sk * (1.f - sk);
    }
    if (lane < K && e >= 0) out[e] = __float2bfloat16(g);
  }
}

HM_API int hm_gate_backward(const float* logits, const int32_t* expert_ids, const float* weights,
                            const float* dw, int64_t T, int32_t E, int32_t K, int32_t mode,
                            float route_scale, void* dlogits, int32_t ld, void* stream) {
  HM_RANGE("hm_gate_backward");
  HM_CHECK_ARG(logits && expert_ids && weights && dw && dlogits, "hm_gate_backward: null argument");
  HM_CHECK_ARG(ld >= E && ld % 8 == 0 && K >= 1 && K <= 32 && mode >= 0 && mode <= 2,
               "hm_gate_backward: ld >= E, ld %% 8 == 0, 1 <= K <= 32, mode 0..2");
  if (T <= 0) return 0;
  k_gate_backward<<<grid_for(T, 8, kSMs * 8), 256, 0, (cudaStream_t)stream>>>(
      logits, expert_ids, weights, dw, T, E, K, mode, route_scale, (__nv_bfloat16*)dlogits, ld);
  HM_LAUNCHED();
  return 0;
}

HM_API int hm_bf16_to_f32(const void* src, float* dst, int64_t n, void* stream) {
  HM_CHECK_ARG(n >= 0 && (n == 0 || (src && dst)), "hm_bf16_to_f32: null argument");
  HM_CHECK_ARG(((uintptr_t)src & 15) == 0 && ((uintptr_t)dst & 15) == 0,
               "hm_bf16_to_f32: buffers must be 16-byte aligned");
  if (n == 0) return 0;
  const int64_t want = (n / 8 + 255) / 256;
  const int blocks = (int)(want < 1 ? 1 : (want > kSMs * 16 ? kSMs * 16 : want));
  k_bf16_to_f32<<<blocks, 256, 0, (cudaStream_t)stream>>>((const __nv_bfloat16*)src, dst, n);
  HM_LAUNCHED();
  return 0;
}

// out = bf16((a + b) + c) with fp32 sums (c optional): the router backward's
// input gradient (router-GEMM term + routed-path dx + shared-expert dx)
// rounded once, 16-byte accesses
__global__ void __launch_bounds__(256) k_sum_to_bf16(const float* __restrict__ a,
                                                     const __nv_bfloat16* __restrict__ b,
                                                     const __nv_bfloat16* __restrict__ c,
                                                     __nv_bfloat16* __restrict__ out, int64_t n) {
  const int64_t nv = n / 8;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // two elements-of-8 per thread per iteration, all loads issued first
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < nv; i0 += 2 * stride) {
    float4 a0[2], a1[2];
    int4 bv[2], cv[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int64_t i = i0 + u * stride;
      if (i >= nv) break;
      a0[u] = __ldg(reinterpret_cast<const float4*>(a) + 2 * i);
      a1[u] = __ldg(reinterpret_cast<const float4*>(a) + 2 * i + 1);
      bv[u] = ld_nc_v4(reinterpret_cast<const int4*>(b) + i);
      if (c) cv[u] = ld_nc_v4(reinterpret_cast<const int4*>(c) + i);
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int64_t i = i0 + u * stride;
      if (i >= nv) break;
      float f[8] = {a0[u].x, a0[u].y, a0[u].z, a0[u].w, a1[u].x, a1[u].y, a1[u].z, a1[u].w};
      float fb[8];
      Vec<__nv_bfloat16>::to_f32(bv[u], fb);
#pragma unroll
      for (int q = 0; q < 8; ++q) f[q] += fb[q];
      if (c) {
        Vec<__nv_bfloat16>::to_f32(cv[u], fb);
#pragma unroll
        for (int q = 0; q < 8; ++q) f[q] += fb[q];
      }
      reinterpret_cast<int4*>(out)[i] = Vec<__nv_bfloat16>::from_f32(f);
    }
  }
  for (int64_t i = nv * 8 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    float v = a[i] + __bfloat162float(b[i]);
    if (c) v += __bfloat162float(c[i]);
    out[i] = __float2bfloat16(v);
  }
}

HM_API int hm_sum_to_bf16(const float* a, const void* b, const void* c, void* out, int64_t n,
                          void* stream) {
  HM_CHECK_ARG(n >= 0 && (n == 0 || (a && b && out)), "hm_sum_to_bf16: null argument");
  HM_CHECK_ARG((((uintptr_t)a | (uintptr_t)b | (uintptr_t)c | (uintptr_t)out) & 15) == 0,
               "hm_sum_to_bf16: buffers must be 16-byte aligned");
  if (n == 0) return 0;
  const int64_t want = (n / 8 + 255) / 256;
  const int blocks = (int)(want < 1 ? 1 : (want > kSMs * 16 ? kSMs * 16 : want));
  k_sum_to_bf16<<<blocks, 256, 0, (cudaStream_t)stream>>>(
      a, (const __nv_bfloat16*)b, (const __nv_bfloat16*)c, (__nv_bfloat16*)out, n);
  HM_LAUNCHED();
  return 0;
}

HM_API int hm_combine_add(hm_world* w, const float* wts, const int32_t* ids, int32_t mode,
                          const void* addend, void* out, void* stream) {
  HM_CHECK_ARG(addend, "hm_combine_add: null addend");
  return combine_impl(w, wts, ids, mode, addend, out, stream);
}

// explicit barrier (e.g. after an expert FFN when the raw combine follows)
HM_API int hm_world_barrier(hm_world* w, void* stream) {
  HM_RANGE("hm_world_barrier");
  HM_CHECK_ARG(w, "hm_world_barrier: null world");
  if (w->h.P > 1) {
    k_barrier<<<1, 32, 0, (cudaStream_t)stream>>>(w->d, w->status);
    HM_LAUNCHED();
  }
  return 0;
}

// buffer access for tests / the expert FFN.  kinds:
//  0 recv_x  1 recv_meta  2 xmaj  3 ymaj  4 comb  (local rank l in 0..L-1)
//  5 counts [G][G+E]  6 gpos [L*T_r][G]  7 epos [L*T_r][K]  8 hitmask [L*T_r]
//  9 offsets (R[L] then Nd[L], int32)  10 n_e [E]  11 status [4] int32
HM_API int hm_world_buffer(hm_world* w, int32_t kind, int32_t local_rank, void** ptr,
                           int64_t* bytes) {
  HM_CHECK_ARG(w && ptr && bytes, "hm_world_buffer: null argument");
  const WorldDev& h = w->h;
  HM_CHECK_ARG(local_rank >= 0 && local_rank < h.L, "local_rank out of range");
  int d = h.p * h.L + local_rank;
  const int64_t T = (int64_t)h.L * h.T_r;
  switch (kind) {
    case 0: *ptr = h.recv_x[d]; *bytes = h.R_cap * h.row_bytes; break;
    case 1: *ptr = h.recv_meta[d]; *bytes = h.R_cap * h.K * (int64_t)sizeof(RowMeta); break;
    case 2: *ptr = h.xmaj[d]; *bytes = h.N_cap * h.row_bytes; break;
    case 3: *ptr = h.ymaj[d]; *bytes = h.N_cap * h.row_bytes; break;
    case 4: *ptr = h.comb[d]; *bytes = h.R_cap * h.row_bytes; break;
    case 5: *ptr = h.counts[d]; *bytes = (int64_t)h.G * (h.G + h.E + h.P) * 4; break;
    case 6: *ptr = w->gpos; *bytes = T * h.G * 4; break;
    case 7: *ptr = w->epos; *bytes = T * h.K * 4; break;
    case 8: *ptr = w->hitmask; *bytes = T * 8; break;
    case 9: *ptr = reinterpret_cast<uint8_t*>(w->offs) + offsetof(Offsets, R);
            *bytes = sizeof(int32_t) * 2 * kMaxRanks; break;
    case 10: *ptr = w->n_e; *bytes = h.E * 4; break;
    case 11: *ptr = w->status; *bytes = 16; break;
    case 12: *ptr = h.gy[d]; *bytes = w->grad ? h.N_cap * h.row_bytes : 0; break;
    case 13: *ptr = h.gx[d]; *bytes = w->grad ? h.N_cap * h.row_bytes : 0; break;
    case 14: *ptr = h.recv_g[h.p]; *bytes = h.Rg_cap * h.row_bytes; break;
    case 15: *ptr = w->gpos_g; *bytes = T * h.P * 4; break;
    case 16: *ptr = reinterpret_cast<uint8_t*>(w->offs) + offsetof(Offsets, R_g); *bytes = 4; break;
    case 17: *ptr = w->xidx ? w->xidx + (int64_t)local_rank * h.N_cap : nullptr;
             *bytes = w->xidx ? h.N_cap * 4 : 0; break;
    default: hm::set_error("hm_world_buffer: unknown kind %d", kind); return hm::kInvalid;
  }
  return 0;
}

HM_API int hm_world_info(hm_world* w, int64_t* out8) {
  HM_CHECK_ARG(w && out8, "hm_world_info: null argument");
  const WorldDev& h = w->h;
  out8[0] = h.G; out8[1] = h.P; out8[2] = h.p; out8[3] = h.L;
  out8[4] = h.R_cap; out8[5] = h.N_cap; out8[6] = h.row_bytes; out8[7] = (int64_t)w->sym_bytes;
  return 0;
}

// stream-ordered device/host copy (cudaMemcpyDefault), for buffer inspection
HM_API int hm_memcpy(void* dst, const void* src, int64_t bytes, void* stream) {
  HM_CHECK_ARG(bytes >= 0, "hm_memcpy: negative size");
  if (bytes == 0) return 0;
  HM_CUDA(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDefault, (cudaStream_t)stream));
  return 0;
}

// Per-kernel CUDA-event timing of the world's launches (enable=1 creates the
// events; each launch records a start/stop pair on its stream).
HM_API int hm_world_set_timing(hm_world* w, int32_t enable) {
  HM_CHECK_ARG(w, "hm_world_set_timing: null world");
  if (enable && !w->timing) {
    for (int i = 0; i < 2 * 16; ++i) HM_CUDA(cudaEventCreate(&w->ev[i]));
  }
  w->timing = enable != 0 || w->timing;
  if (!enable) w->timing = false;
  for (int i = 0; i < 16; ++i) w->seg_used[i] = 0;
  return 0;
}

// Milliseconds of the most recent launch of each segment (after a stream sync):
// plan, notify, pack, barrier1, expand, reduce, barrier2, gather, and the
// overlapped forward's local-rows GEMM1 (+ row push) and remaining GEMMs;
// -1 if unused.
HM_API int hm_world_timings(hm_world* w, float* ms, int32_t n) {
  HM_CHECK_ARG(w && ms, "hm_world_timings: null argument");
  for (int i = 0; i < n && i < kSegCount; ++i) {
    ms[i] = -1.f;
    if (w->timing && w->seg_used[i]) {
      float v = 0.f;
      if (cudaEventElapsedTime(&v, w->ev[2 * i], w->ev[2 * i + 1]) == cudaSuccess) ms[i] = v;
    }
  }
  return 0;
}

// phase-2 inputs of a two-level dispatch from a relay world's received rows:
// ids2/w2 are [L * R_cap, K] (R_cap = U1 * T_r), the same row layout as the
// relay's receive buffer (which is the phase-2 payload).
HM_API int hm_relay_ids(hm_world* w, int32_t* ids2, float* w2, void* stream) {
  HM_RANGE("hm_relay_ids");
  HM_CHECK_ARG(w && ids2 && w2, "hm_relay_ids: null argument");
  HM_CHECK_ARG(w->h.U1 > 0, "hm_relay_ids: not a relay world");
  int64_t n = (int64_t)w->h.L * w->h.R_cap * w->h.K;
  k_relay_ids<<<grid_for(n, 256, kSMs * 8), 256, 0, (cudaStream_t)stream>>>(w->d, w->offs, ids2, w2);
  HM_LAUNCHED();
  return 0;
}

// Combine backward: grad of the combined output g [L*T_r, M] -> expert-output
// grads gy (expert-major, every local rank) + gate grads of direct picks into
// dw [L*T_r, K]; replays the last forward plan (no re-planning).
HM_API int hm_dispatch_grad(hm_world* w, const void* g, const int32_t* ids, const float* wts,
                            int32_t mode, float* dw, void* stream) {
  HM_RANGE("hm_dispatch_grad");
  HM_CHECK_ARG(w && g && ids && wts && dw, "hm_dispatch_grad: null argument");
  HM_CHECK_ARG(w->grad, "hm_dispatch_grad: world created without backward buffers");
  HM_CHECK_ARG(mode == w->last_mode, "hm_dispatch_grad: mode differs from the forward's");
  HM_CHECK_ARG(mode <= 3, "hm_dispatch_grad: mode must be 0..3");
  HM_CHECK_ARG(!w->h.U1, "hm_dispatch_grad: relay worlds have no backward");
  cudaStream_t s = (cudaStream_t)stream;
  const WorldDev& h = w->h;
  const int64_t T = (int64_t)h.L * h.T_r;
  int blocks = grid_for(T, 8, exch_blocks(w));
  if (mode == 0 || (mode >= 2 && h.P == 1)) {
    // every pick direct: one token per warp, up to 32 CTAs per SM
    blocks = grid_for(T, 8, w->max_blocks > 0 ? w->max_blocks : kSMs * 32);
    if (h.elem == 2)
      k_pack_grad_direct<__nv_bfloat16><<<blocks, 256, 0, s>>>(w->d, (const uint8_t*)g, ids, wts,
                                                               w->epos, dw);
    else
      k_pack_grad_direct<float><<<blocks, 256, 0, s>>>(w->d, (const uint8_t*)g, ids, wts, w->epos,
                                                       dw);
  } else if (h.elem == 2)
    k_pack_grad<__nv_bfloat16><<<blocks, 256, 0, s>>>(w->d, (const uint8_t*)g, ids, wts, w->hitmask,
                                                      w->gpos, w->epos, mode, w->gpos_g, dw);
  else
    k_pack_grad<float><<<blocks, 256, 0, s>>>(w->d, (const uint8_t*)g, ids, wts, w->hitmask,
                                              w->gpos, w->epos, mode, w->gpos_g, dw);
  HM_LAUNCHED();
  if (h.P > 1) {
    k_barrier<<<1, 32, 0, s>>>(w->d, w->status);
    HM_LAUNCHED();
  }
  if (mode == 3 && h.P > 1) {
    if (h.elem == 2)
      k_expand_grad_g<__nv_bfloat16><<<exch_blocks(w), 256, 0, s>>>(w->d, w->offs);
    else
      k_expand_grad_g<float><<<exch_blocks(w), 256, 0, s>>>(w->d, w->offs);
    HM_LAUNCHED();
  } else if (mode != 0 && mode != 3 && !(h.P == 1 && mode == 2)) {
    if (h.elem == 2)
      k_expand_grad<__nv_bfloat16><<<exch_blocks(w), 256, 0, s>>>(w->d, w->offs);
    else
      k_expand_grad<float><<<exch_blocks(w), 256, 0, s>>>(w->d, w->offs);
    HM_LAUNCHED();
  }
  return 0;
}

// Dispatch backward: expert-input grads gx (expert-major) -> token grads
// dx [L*T_r, M] (unweighted dedup reduction), and the dedup picks' gate grads
// into dw.
HM_API int hm_combine_grad(hm_world* w, const int32_t* ids, int32_t mode, float* dw, void* dx,
                           void* stream) {
  HM_RANGE("hm_combine_grad");
  HM_CHECK_ARG(w && ids && dw && dx, "hm_combine_grad: null argument");
  HM_CHECK_ARG(w->grad, "hm_combine_grad: world created without backward buffers");
  HM_CHECK_ARG(mode == w->last_mode, "hm_combine_grad: mode differs from the forward's");
  cudaStream_t s = (cudaStream_t)stream;
  const WorldDev& h = w->h;
  if (mode == 3 && h.P > 1) {   // unweighted sums of this GPU's picks per received row
    with_row_type(h, [&](auto t, auto v) {
      k_reduce_g<typename decltype(t)::type, decltype(v)::value>
          <<<exch_blocks(w), 256, 0, s>>>(w->d, w->offs, 1);
    });
    HM_LAUNCHED();
  } else if (mode != 0 && mode != 3 && !(h.P == 1 && mode == 2)) {
    with_row_type(h, [&](auto t, auto v) {
      k_reduce<typename decltype(t)::type, decltype(v)::value>
          <<<exch_blocks(w), 256, 0, s>>>(w->d, w->offs, 1, 1);
    });
    HM_LAUNCHED();
  }
  if (h.P > 1) {
    k_barrier<<<1, 32, 0, s>>>(w->d, w->status);
    HM_LAUNCHED();
  }
  const int64_t T = (int64_t)h.L * h.T_r;
  int blocks = grid_for(T, 8, exch_blocks(w));
  with_row_type(h, [&](auto t, auto v) {
    k_gather<typename decltype(t)::type, decltype(v)::value><<<blocks, 256, 0, s>>>(
        w->d, ids, nullptr, w->hitmask, w->gpos, w->epos, mode, 1, 1, w->offs, w->gpos_g,
        (uint8_t*)dx, nullptr);
  });
  HM_LAUNCHED();
  k_gate_grad<<<grid_for(T * h.K, 256, kSMs * 8), 256, 0, s>>>(w->d, ids, w->gpos, mode,
                                                                 w->gpos_g, dw);
  HM_LAUNCHED();
  return 0;
}

// runtime options: 4 = grid cap of the exchange kernels (CTAs, 0 = 8 per SM;
// leaves SMs to concurrent kernels); 10 = fused one-GPU dispatch (row indices
// instead of expert-major copies, hm_expert_ffn_gather).  Options 0-3 and 5-9
// selected measured-slower variants (TMA gather, staged pipelined exchange,
// bulk / split / general one-GPU pack, store hints, 8-source gather batches)
// that round 2 removed; they are rejected.
HM_API int hm_world_set_option(hm_world* w, int32_t option, int32_t value) {
  HM_CHECK_ARG(w, "hm_world_set_option: null world");
  HM_CHECK_ARG(option == 4 || option == 10, "hm_world_set_option: unknown option %d", option);
  if (option == 4) w->max_blocks = value > 0 ? value : 0;
  if (option == 10) {
    HM_CHECK_ARG(!value || !w->h.U1, "hm_world_set_option: no fused dispatch on a relay world");
    if (value && !w->xidx) {
      HM_CUDA(cudaMalloc(&w->xidx, (size_t)w->h.L * w->h.N_cap * 4));
      HM_CUDA(cudaMemset(w->xidx, 0, (size_t)w->h.L * w->h.N_cap * 4));
    }
    w->fused = value != 0;
  }
  return 0;
}
