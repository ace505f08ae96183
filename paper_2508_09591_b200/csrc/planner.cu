// Decision-path kernels: routing-mask packing, per-group dedup/raw counts,
// hierarchical propagation (copy lists), swap tensors, smooth-max cost matrix
// and argmin.  Each kernel reproduces one reference hiera2a function bit for
// bit (see include/hiermoe.h for the file:line each entry point replaces).
//
// Compiled with -fmad=false: the cost kernel must round every fp64 + and *
// individually, exactly like numpy.
//
// Mask layout in HBM: packed rows, W = ceil(E/32) uint32 words per token, bit
// e of row t = (bits[t*W + e/32] >> (e%32)) & 1.  Slot s belongs to group
// s / (E/g) of a g-group cut (topology.py:95-97).

#include "hm_common.cuh"
#include "ddmath.cuh"
#include "numpy_pow.cuh"

#include <stdarg.h>
#include <string.h>

namespace hm {

static thread_local char g_err[512];

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

}  // namespace hm

HM_API const char* hm_last_error(void) { return hm::g_err; }
HM_API int hm_version(void) { return 10000; }
HM_API unsigned long long hm_launch_count(void) { return hm::launch_counter().load(); }

namespace {

using namespace hm;

__device__ __forceinline__ int words_of(int E) { return (E + 31) >> 5; }

// ---------------------------------------------------------------------------
// mask packing: one warp per row, ballot over 32 columns at a time.  Optional
// column gather slot_view(bits)[:, s] = bits[:, slot_to_expert[s]]
// (routing.py:98-106).  Row popcounts feed the K-per-row validation
// (routing.py:38-48).
__global__ void k_mask_pack(const uint8_t* __restrict__ mask, int64_t T, int E,
                            const int32_t* __restrict__ s2e, uint32_t* __restrict__ bits,
                            int32_t* __restrict__ popcnt) {
  const int lane = threadIdx.x & 31;
  const int W = words_of(E);
  int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t t = warp; t < T; t += nwarps) {
    const uint8_t* row = mask + t * E;
    int pc = 0;
    for (int w = 0; w < W; ++w) {
      int col = w * 32 + lane;
      bool v = false;
      if (col < E) v = row[s2e ? __ldg(s2e + col) : col] != 0;
      uint32_t word = __ballot_sync(0xffffffffu, v);
      if (lane == 0) bits[t * W + w] = word;
      pc += __popc(word);
    }
    if (popcnt && lane == 0) popcnt[t] = pc;
  }
}

__global__ void k_mask_unpack(const uint32_t* __restrict__ bits, int64_t T, int E,
                              uint8_t* __restrict__ mask) {
  const int W = words_of(E);
  int64_t n = T * E;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = i / E;
    int e = (int)(i - t * E);
    mask[i] = (bits[t * W + (e >> 5)] >> (e & 31)) & 1u;
  }
}

// K-per-row ids (already in slot space or mapped through expert_to_slot)
__global__ void k_ids_to_bits(const int32_t* __restrict__ ids, int64_t T, int K, int E,
                              const int32_t* __restrict__ e2s, uint32_t* __restrict__ bits,
                              int* __restrict__ bad) {
  const int W = words_of(E);
  int64_t n = T * K;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = i / K;
    int e = ids[i];
    if (e < 0 || e >= E) {
      atomicExch(bad, 1);
      continue;
    }
    int s = e2s ? e2s[e] : e;
    uint32_t old = atomicOr(bits + t * W + (s >> 5), 1u << (s & 31));
    if (old & (1u << (s & 31))) atomicExch(bad, 2);  // duplicate id in a row
  }
}

// ---------------------------------------------------------------------------
// per-group counts, several cuts in one pass (traffic.py:58-82).  A row's set
// bits are visited in ascending slot order, so group ids are non-decreasing and
// "group changed" marks each distinct hit exactly once.
constexpr int kMaxCuts = 8;
struct Cuts {
  int n;
  int groups[kMaxCuts];
  int offset[kMaxCuts];  // into the concatenated output / smem histogram
};

__global__ void k_level_counts(const uint32_t* __restrict__ bits, int64_t T, int E, Cuts cuts,
                               unsigned long long* __restrict__ dedup,
                               unsigned long long* __restrict__ raw,
                               uint8_t* __restrict__ hit, int hit_cut) {
  extern __shared__ unsigned int sm[];
  int total = cuts.offset[cuts.n - 1] + cuts.groups[cuts.n - 1];
  unsigned int* s_dedup = sm;
  unsigned int* s_raw = sm + total;
  for (int i = threadIdx.x; i < 2 * total; i += blockDim.x) sm[i] = 0;
  __syncthreads();
  const int W = words_of(E);
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < T;
       t += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t* row = bits + t * W;
    for (int c = 0; c < cuts.n; ++c) {
      const int g = cuts.groups[c];
      const int size = E / g;
      int last = -1;
      for (int w = 0; w < W; ++w) {
        uint32_t word = row[w];
        while (word) {
          int b = __ffs(word) - 1;
          word &= word - 1;
          int grp = (w * 32 + b) / size;
          atomicAdd(s_raw + cuts.offset[c] + grp, 1u);
          if (grp != last) {
            atomicAdd(s_dedup + cuts.offset[c] + grp, 1u);
            if (hit && c == hit_cut) hit[t * g + grp] = 1;
            last = grp;
          }
        }
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < total; i += blockDim.x) {
    if (s_dedup[i]) atomicAdd(dedup + i, (unsigned long long)s_dedup[i]);
    if (s_raw[i]) atomicAdd(raw + i, (unsigned long long)s_raw[i]);
  }
}

// ---------------------------------------------------------------------------
// propagation (routing.py:189-215): copies[t] = #distinct groups hit by row t,
// exclusive scan -> first copy index, then emit copies in row-major
// (row, group) order with selections restricted to the group.
__global__ void k_prop_count(const uint32_t* __restrict__ bits, int64_t T, int E, int g,
                             int64_t* __restrict__ copies) {
  const int W = words_of(E);
  const int size = E / g;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < T;
       t += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t* row = bits + t * W;
    int last = -1, n = 0;
    for (int w = 0; w < W; ++w) {
      uint32_t word = row[w];
      while (word) {
        int b = __ffs(word) - 1;
        word &= word - 1;
        int grp = (w * 32 + b) / size;
        if (grp != last) {
          ++n;
          last = grp;
        }
      }
    }
    copies[t] = n;
  }
}

// block-level exclusive scan of int64 (blockDim = 1024)
__device__ int64_t block_exclusive_scan(int64_t v, int64_t* s_warp, int64_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t x = v;
  for (int o = 1; o < 32; o <<= 1) {
    int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int nw = blockDim.x >> 5;
    int64_t w = lane < nw ? s_warp[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      int64_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < nw) s_warp[lane] = w;
  }
  __syncthreads();
  int64_t incl = x + (warp ? s_warp[warp - 1] : 0);
  if (total) *total = s_warp[(blockDim.x >> 5) - 1];
  __syncthreads();
  return incl - v;
}

constexpr int kScanThreads = 1024;
constexpr int kScanPerThread = 4;
constexpr int kScanChunk = kScanThreads * kScanPerThread;

__global__ void k_scan_partials(const int64_t* __restrict__ in, int64_t n,
                                int64_t* __restrict__ partial) {
  __shared__ int64_t s_warp[32];
  int64_t base = (int64_t)blockIdx.x * kScanChunk;
  int64_t sum = 0;
  for (int i = 0; i < kScanPerThread; ++i) {
    int64_t j = base + (int64_t)threadIdx.x * kScanPerThread + i;
    if (j < n) sum += in[j];
  }
  int64_t tot;
  block_exclusive_scan(sum, s_warp, &tot);
  if (threadIdx.x == 0) partial[blockIdx.x] = tot;
}

__global__ void k_scan_top(int64_t* __restrict__ partial, int64_t nb, int64_t* __restrict__ grand) {
  __shared__ int64_t s_warp[32];
  int64_t carry = 0;
  for (int64_t base = 0; base < nb; base += blockDim.x) {
    int64_t j = base + threadIdx.x;
    int64_t v = j < nb ? partial[j] : 0;
    int64_t tot;
    int64_t ex = block_exclusive_scan(v, s_warp, &tot);
    if (j < nb) partial[j] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) *grand = carry;
}

__global__ void k_scan_apply(const int64_t* __restrict__ in, int64_t n,
                             const int64_t* __restrict__ partial, int64_t* __restrict__ out) {
  __shared__ int64_t s_warp[32];
  int64_t base = (int64_t)blockIdx.x * kScanChunk;
  int64_t v[kScanPerThread];
  int64_t sum = 0;
  for (int i = 0; i < kScanPerThread; ++i) {
    int64_t j = base + (int64_t)threadIdx.x * kScanPerThread + i;
    v[i] = j < n ? in[j] : 0;
    sum += v[i];
  }
  int64_t ex = block_exclusive_scan(sum, s_warp, nullptr) + partial[blockIdx.x];
  for (int i = 0; i < kScanPerThread; ++i) {
    int64_t j = base + (int64_t)threadIdx.x * kScanPerThread + i;
    if (j < n) out[j] = ex;
    ex += v[i];
  }
}

__global__ void k_prop_emit(const uint32_t* __restrict__ bits, int64_t T, int E, int g,
                            const int64_t* __restrict__ first, const int64_t* __restrict__ origin_in,
                            uint32_t* __restrict__ out_bits, int64_t* __restrict__ out_origin,
                            int64_t* __restrict__ out_parent) {
  const int W = words_of(E);
  const int size = E / g;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < T;
       t += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t* row = bits + t * W;
    int64_t c = first[t] - 1;
    int last = -1;
    int64_t org = origin_in ? origin_in[t] : t;
    for (int w = 0; w < W; ++w) {
      uint32_t word = row[w];
      while (word) {
        int b = __ffs(word) - 1;
        word &= word - 1;
        int s = w * 32 + b;
        int grp = s / size;
        if (grp != last) {
          ++c;
          last = grp;
          uint32_t* orow = out_bits + c * W;
          for (int x = 0; x < W; ++x) orow[x] = 0;
          out_origin[c] = org;
          out_parent[c] = grp;
        }
        out_bits[c * W + w] |= 1u << b;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// swap partials (swap.py:81-118, restated with integer counts).  For a cut
// of g groups of `size` slots, per token with selection set S and hit groups H:
//   base[k]      += [k in H]
//   sel[a]       += [a in S]
//   hitsel[a,k]  += [a in S][k in H]                 (raises = sel - hitsel)
//   lone[a]      += [a in S, a alone in its group]
//   lonesel[a,b] += [a lone][b in S][grp(b) != grp(a)]   (drops = lone - lonesel)
// Shared-memory histograms over a tile of `a` rows, flushed with u64 atomics.
constexpr int kMaxSel = 128;  // max selections per row handled in registers/smem

__global__ void k_swap_partials(const uint32_t* __restrict__ bits, int64_t T, int E, int g,
                                int a_lo, int a_hi,
                                unsigned long long* __restrict__ base,
                                unsigned long long* __restrict__ sel,
                                unsigned long long* __restrict__ hitsel,
                                unsigned long long* __restrict__ lone,
                                unsigned long long* __restrict__ lonesel,
                                int* __restrict__ too_dense) {
  extern __shared__ unsigned int sm[];
  const int rows = a_hi - a_lo;
  unsigned int* s_hitsel = sm;                 // rows x g
  unsigned int* s_lonesel = sm + rows * g;     // rows x E
  unsigned int* s_base = s_lonesel + rows * E; // g
  unsigned int* s_sel = s_base + g;            // rows
  unsigned int* s_lone = s_sel + rows;         // rows
  const int total = rows * g + rows * E + g + 2 * rows;
  for (int i = threadIdx.x; i < total; i += blockDim.x) sm[i] = 0;
  __syncthreads();
  const int W = words_of(E);
  const int size = E / g;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < T;
       t += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t* row = bits + t * W;
    short S[kMaxSel];
    int n = 0;
    for (int w = 0; w < W; ++w) {
      uint32_t word = row[w];
      while (word) {
        int b = __ffs(word) - 1;
        word &= word - 1;
        if (n < kMaxSel) S[n] = (short)(w * 32 + b);
        ++n;
      }
    }
    if (n > kMaxSel) {
      atomicExch(too_dense, 1);
      continue;
    }
    // distinct groups (ascending) and per-group multiplicity via run lengths
    for (int i = 0; i < n;) {
      int grp = S[i] / size;
      int j = i;
      while (j < n && S[j] / size == grp) ++j;
      if (a_lo == 0) atomicAdd(s_base + grp, 1u);
      bool is_lone = (j - i) == 1;
      for (int x = i; x < j; ++x) {
        int a = S[x];
        if (a < a_lo || a >= a_hi) continue;
        int ar = a - a_lo;
        atomicAdd(s_sel + ar, 1u);
        // a x every hit group
        int last = -1;
        for (int y = 0; y < n; ++y) {
          int gy = S[y] / size;
          if (gy != last) {
            atomicAdd(s_hitsel + ar * g + gy, 1u);
            last = gy;
          }
        }
        if (is_lone) {
          atomicAdd(s_lone + ar, 1u);
          for (int y = 0; y < n; ++y)
            if (S[y] / size != grp) atomicAdd(s_lonesel + ar * E + S[y], 1u);
        }
      }
      i = j;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < rows * g; i += blockDim.x)
    if (s_hitsel[i]) atomicAdd(hitsel + (int64_t)a_lo * g + i, (unsigned long long)s_hitsel[i]);
  for (int i = threadIdx.x; i < rows * E; i += blockDim.x)
    if (s_lonesel[i]) atomicAdd(lonesel + (int64_t)a_lo * E + i, (unsigned long long)s_lonesel[i]);
  for (int i = threadIdx.x; i < rows; i += blockDim.x) {
    if (s_sel[i]) atomicAdd(sel + a_lo + i, (unsigned long long)s_sel[i]);
    if (s_lone[i]) atomicAdd(lone + a_lo + i, (unsigned long long)s_lone[i]);
  }
  if (a_lo == 0)
    for (int i = threadIdx.x; i < g; i += blockDim.x)
      if (s_base[i]) atomicAdd(base + i, (unsigned long long)s_base[i]);
}

// Z[a,b,k] = base[k] + d[a,b,k] + d[b,a,k],
// d[a,b,k] = raises[a,k][grp(b)=k] - drops[a,b][grp(a)=k][grp(a)!=grp(b)]
__device__ __forceinline__ int64_t swap_delta(int a, int b, int k, int size, int g, int E,
                                              const int64_t* sel, const int64_t* hitsel,
                                              const int64_t* lone, const int64_t* lonesel) {
  int ga = a / size, gb = b / size;
  int64_t d = 0;
  if (gb == k) d += sel[a] - hitsel[(int64_t)a * g + k];
  if (ga == k && ga != gb) d -= lone[a] - lonesel[(int64_t)a * E + b];
  return d;
}

__global__ void k_swap_tensor(const int64_t* __restrict__ base, const int64_t* __restrict__ sel,
                              const int64_t* __restrict__ hitsel, const int64_t* __restrict__ lone,
                              const int64_t* __restrict__ lonesel, int E, int g,
                              int64_t* __restrict__ z) {
  const int size = E / g;
  int64_t n = (int64_t)E * E * g;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int k = (int)(i % g);
    int64_t ab = i / g;
    int b = (int)(ab % E), a = (int)(ab / E);
    z[i] = base[k] + swap_delta(a, b, k, size, g, E, sel, hitsel, lone, lonesel) +
           swap_delta(b, a, k, size, g, E, sel, hitsel, lone, lonesel);
  }
}

// ---------------------------------------------------------------------------
// cost matrix (swap.py:180-206) for dim = *dim_dev (or dim_host if dim_dev is
// null).  q[r,c] accumulates, in level order,
//   ((participants * smax(Z[r,c,:])) * token_bytes) * beta + alpha
// exactly in numpy's operation order; the gamma=inf variant (exact max) is
// written to q_exact.
struct PhaseDesc {
  const int64_t* z;  // E x E x g
  int groups;
  int participants;
  double alpha, beta;
};
constexpr int kMaxPhases = 8;
struct CostArgs {
  PhaseDesc inter[kMaxPhases];  // inter-level-i, i = 1..D-1 (index i-1)
  PhaseDesc intra[kMaxPhases];  // intra per dimension d (index d-1)
  int depth;
  int E;
  double token_bytes;
  double gamma, gamma_inv;
};

__device__ double smax_entry(const int64_t* z, int g, double gamma, double gamma_inv) {
  double v[64];
  double scratch[64];
  for (int k = 0; k < g; ++k) v[k] = (double)z[k];
  return smooth_max_vec_np(v, g, gamma, gamma_inv, scratch);
}

__global__ void k_cost(CostArgs args, const int* __restrict__ dim_dev, int dim_host,
                       double* __restrict__ q, double* __restrict__ q_exact) {
  const int dim = dim_dev ? *dim_dev : dim_host;
  const int64_t n = (int64_t)args.E * args.E;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0, acc_x = 0.0;
    for (int p = 0; p < dim; ++p) {
      const PhaseDesc& ph = (p < dim - 1) ? args.inter[p] : args.intra[dim - 1];
      const int64_t* zp = ph.z + i * ph.groups;
      double sm = smax_entry(zp, ph.groups, args.gamma, args.gamma_inv);
      double mx = smax_entry(zp, ph.groups, INFINITY, 0.0);
      double vol = (double)ph.participants * sm;
      double vx = (double)ph.participants * mx;
      acc = acc + (vol * args.token_bytes * ph.beta + ph.alpha);
      acc_x = acc_x + (vx * args.token_bytes * ph.beta + ph.alpha);
    }
    if (q) q[i] = acc;
    if (q_exact) q_exact[i] = acc_x;
  }
}

// first-occurrence argmin over n doubles (np.argmin, NaN-free input), then the
// select_swap decision (swap.py:240-252):
//   out_i64[0] = flat argmin, out_i64[1] = r, out_i64[2] = c, out_i64[3] = chosen(0/1)
//   out_f64[0] = no_swap = q_exact[0,0], out_f64[1] = saving
__global__ void k_argmin_select(const double* __restrict__ q, const double* __restrict__ q_exact,
                                int E, int64_t* __restrict__ out_i64, double* __restrict__ out_f64) {
  __shared__ double s_v[32];
  __shared__ int64_t s_i[32];
  const int64_t n = (int64_t)E * E;
  double best = INFINITY;
  int64_t bi = n;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    double v = q[i];
    if (v < best) {  // strictly smaller keeps the first occurrence per thread
      best = v;
      bi = i;
    }
  }
  for (int o = 16; o; o >>= 1) {
    double v2 = __shfl_xor_sync(0xffffffffu, best, o);
    int64_t i2 = __shfl_xor_sync(0xffffffffu, bi, o);
    if (v2 < best || (v2 == best && i2 < bi)) {
      best = v2;
      bi = i2;
    }
  }
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    s_v[warp] = best;
    s_i[warp] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      if (s_v[w] < best || (s_v[w] == best && s_i[w] < bi)) {
        best = s_v[w];
        bi = s_i[w];
      }
    if (bi >= n) bi = 0;  // all-NaN guard (cannot happen for valid params)
    int64_t r = bi / E, c = bi % E;
    double no_swap = q_exact[0];
    double saving = 0.0;
    int chosen = 0;
    if (r != c) {
      double sv = no_swap - q_exact[bi];
      if (!(sv < 0.0)) {
        saving = sv;
        chosen = 1;
      }
    }
    out_i64[0] = bi;
    out_i64[1] = r;
    out_i64[2] = c;
    out_i64[3] = chosen;
    out_f64[0] = no_swap;
    out_f64[1] = saving;
  }
}

// ---------------------------------------------------------------------------
// time model + d* (traffic.py:123-221) from per-cut maxima.  One thread.
//   cut_max[i]   = max dedup count at U[i] (i = 1..D-1), cut_max[0] unused
//   gpu_max      = max per-GPU count (invariant under propagation)
// Writes times[D], d_star.
struct TimeArgs {
  int depth;
  int fanout_groups[kMaxPhases];  // U[i]
  int gpus;
  long long token_bytes;
  double a_inter[kMaxPhases], b_inter[kMaxPhases], a_intra[kMaxPhases], b_intra[kMaxPhases];
};

__global__ void k_time_model(TimeArgs a, const unsigned long long* __restrict__ dedup,
                             const int* __restrict__ cut_off, double* __restrict__ times,
                             int* __restrict__ d_star, long long* __restrict__ maxima) {
  if (threadIdx.x || blockIdx.x) return;
  // maxima per cut: cut c covers U[c+1] for c < depth-1, GPU cut last
  long long mx[kMaxPhases + 1];
  for (int c = 0; c < a.depth; ++c) {
    int g = c < a.depth - 1 ? a.fanout_groups[c + 1] : a.gpus;
    long long m = 0;
    for (int k = 0; k < g; ++k) {
      long long v = (long long)dedup[cut_off[c] + k];
      m = v > m ? v : m;
    }
    mx[c] = m;
    if (maxima) maxima[c] = m;
  }
  long long gpu_max = mx[a.depth - 1];
  for (int d = 1; d <= a.depth; ++d) {
    double total = 0.0;
    for (int level = 1; level < d; ++level) {
      long long part = a.fanout_groups[level] / a.fanout_groups[level - 1];
      // python: int bytes (exact) * beta + alpha
      double vol = (double)(part * mx[level - 1] * a.token_bytes);
      total = total + (vol * a.b_inter[level - 1] + a.a_inter[level - 1]);
    }
    long long part = a.gpus / a.fanout_groups[d - 1];
    double vol = (double)(part * gpu_max * a.token_bytes);
    total = total + (vol * a.b_intra[d - 1] + a.a_intra[d - 1]);
    times[d - 1] = total;
  }
  int best = 1;
  if (a.depth > 1) {
    int deep = 2;
    for (int d = 3; d <= a.depth; ++d)
      if (times[d - 1] < times[deep - 1]) deep = d;
    best = times[0] < times[deep - 1] ? 1 : deep;
  }
  *d_star = best;
}

// generic smooth max of a host-provided vector (swap.py:35-48)
__global__ void k_smooth_max_rows(const double* __restrict__ x, int64_t rows, int n, double gamma,
                                  double gamma_inv, double* __restrict__ out) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    double scratch[256];
    double v[256];
    for (int i = 0; i < n; ++i) v[i] = x[r * n + i];
    out[r] = smooth_max_vec_np(v, n, gamma, gamma_inv, scratch);
  }
}

__global__ void k_np_pow(const double* __restrict__ x, const double* __restrict__ y, int64_t n,
                         double* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = np_pow(x[i], y[i]);
}

}  // namespace

// ===========================================================================
// C-ABI
// ===========================================================================

HM_API int hm_mask_pack(const uint8_t* mask, int64_t T, int32_t E, const int32_t* slot_to_expert,
                        uint32_t* bits, int32_t* row_popcount, void* stream) {
  HM_RANGE("hm_mask_pack");
  HM_CHECK_ARG(T >= 0 && E >= 1 && E <= 4096, "hm_mask_pack: bad shape T=%lld E=%d", (long long)T, E);
  if (T == 0) return 0;
  HM_CHECK_ARG(mask && bits, "hm_mask_pack: null pointer");
  int blocks = grid_for(T, 8, kSMs * 16);
  k_mask_pack<<<blocks, 256, 0, (cudaStream_t)stream>>>(mask, T, E, slot_to_expert, bits, row_popcount);
  HM_LAUNCHED();
  return 0;
}

HM_API int hm_mask_unpack(const uint32_t* bits, int64_t T, int32_t E, uint8_t* mask, void* stream) {
  HM_CHECK_ARG(T >= 0 && E >= 1 && E <= 4096, "hm_mask_unpack: bad shape");
  if (T == 0) return 0;
  int blocks = grid_for(T * E, 256, kSMs * 16);
  k_mask_unpack<<<blocks, 256, 0, (cudaStream_t)stream>>>(bits, T, E, mask);
  HM_LAUNCHED();
  return 0;
}

HM_API int hm_ids_to_bits(const int32_t* ids, int64_t T, int32_t K, int32_t E,
                          const int32_t* expert_to_slot, uint32_t* bits, int32_t* bad_flag,
                          void* stream) {
  HM_CHECK_ARG(T >= 0 && K >= 1 && E >= 1 && E <= 4096 && K <= E, "hm_ids_to_bits: bad shape");
  if (T == 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  HM_CUDA(cudaMemsetAsync(bits, 0, (size_t)T * ((E + 31) / 32) * 4, s));
  int blocks = grid_for(T * K, 256, kSMs * 16);
  k_ids_to_bits<<<blocks, 256, 0, s>>>(ids, T, K, E, expert_to_slot, bits, bad_flag);
  HM_LAUNCHED();
  return 0;
}

HM_API int hm_level_counts(const uint32_t* bits, int64_t T, int32_t E, const int32_t* groups,
                           int32_t n_cuts, int64_t* dedup, int64_t* raw, uint8_t* hit,
                           int32_t hit_cut, void* stream) {
  HM_RANGE("hm_level_counts");
  HM_CHECK_ARG(n_cuts >= 1 && n_cuts <= kMaxCuts, "hm_level_counts: 1..%d cuts", kMaxCuts);
  HM_CHECK_ARG(E >= 1 && E <= 4096, "hm_level_counts: E out of range");
  Cuts cuts;
  cuts.n = n_cuts;
  int off = 0;
  for (int i = 0; i < n_cuts; ++i) {
    HM_CHECK_ARG(groups[i] >= 1 && E % groups[i] == 0,
                 "group count %d does not divide %d experts", groups[i], E);
    cuts.groups[i] = groups[i];
    cuts.offset[i] = off;
    off += groups[i];
  }
  cudaStream_t s = (cudaStream_t)stream;
  HM_CUDA(cudaMemsetAsync(dedup, 0, (size_t)off * 8, s));
  HM_CUDA(cudaMemsetAsync(raw, 0, (size_t)off * 8, s));
  if (hit) {
    HM_CHECK_ARG(hit_cut >= 0 && hit_cut < n_cuts, "hm_level_counts: bad hit_cut");
    HM_CUDA(cudaMemsetAsync(hit, 0, (size_t)T * groups[hit_cut], s));
  }
  if (T == 0) return 0;
  size_t smem = (size_t)2 * off * 4;
  HM_CHECK_ARG(smem <= 200 * 1024, "hm_level_counts: too many groups");
  if (smem > 48 * 1024)
    HM_CUDA(cudaFuncSetAttribute(k_level_counts, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int blocks = grid_for(T, 256, kSMs * 4);
  k_level_counts<<<blocks, 256, smem, s>>>(bits, T, E, cuts, (unsigned long long*)dedup,
                                           (unsigned long long*)raw, hit, hit ? hit_cut : -1);
  HM_LAUNCHED();
  return 0;
}

// exclusive scan of n int64 -> out (n entries) and *grand total.  Workspace:
// ceil(n / 4096) int64.
HM_API size_t hm_scan_workspace(int64_t n) {
  return (size_t)((n + kScanChunk - 1) / kScanChunk + 1) * 8;
}

HM_API int hm_scan_i64(const int64_t* in, int64_t n, int64_t* out, int64_t* grand, void* workspace,
                       void* stream) {
  HM_CHECK_ARG(n >= 0, "hm_scan_i64: n < 0");
  cudaStream_t s = (cudaStream_t)stream;
  if (n == 0) {
    HM_CUDA(cudaMemsetAsync(grand, 0, 8, s));
    return 0;
  }
  int64_t nb = (n + kScanChunk - 1) / kScanChunk;
  int64_t* partial = (int64_t*)workspace;
  k_scan_partials<<<(unsigned)nb, kScanThreads, 0, s>>>(in, n, partial);
  HM_LAUNCHED();
  k_scan_top<<<1, 1024, 0, s>>>(partial, nb, grand);
  HM_LAUNCHED();
  k_scan_apply<<<(unsigned)nb, kScanThreads, 0, s>>>(in, n, partial, out);
  HM_LAUNCHED();
  return 0;
}

HM_API int hm_propagate_count(const uint32_t* bits, int64_t T, int32_t E, int32_t groups,
                              int64_t* copies, void* stream) {
  HM_RANGE("hm_propagate_count");
  HM_CHECK_ARG(groups >= 1 && E % groups == 0, "group count %d does not divide %d experts", groups, E);
  if (T == 0) return 0;
  int blocks = grid_for(T, 256, kSMs * 8);
  k_prop_count<<<blocks, 256, 0, (cudaStream_t)stream>>>(bits, T, E, groups, copies);
  HM_LAUNCHED();
  return 0;
}

HM_API int hm_propagate_emit(const uint32_t* bits, int64_t T, int32_t E, int32_t groups,
                             const int64_t* first_copy, const int64_t* origin_in, uint32_t* out_bits,
                             int64_t* out_origin, int64_t* out_parent, void* stream) {
  HM_RANGE("hm_propagate_emit");
  HM_CHECK_ARG(groups >= 1 && E % groups == 0, "group count %d does not divide %d experts", groups, E);
  if (T == 0) return 0;
  int blocks = grid_for(T, 256, kSMs * 8);
  k_prop_emit<<<blocks, 256, 0, (cudaStream_t)stream>>>(bits, T, E, groups, first_copy, origin_in,
                                                        out_bits, out_origin, out_parent);
  HM_LAUNCHED();
  return 0;
}

HM_API int hm_swap_partials(const uint32_t* bits, int64_t T, int32_t E, int32_t groups, int64_t* base,
                            int64_t* sel, int64_t* hitsel, int64_t* lone, int64_t* lonesel,
                            int32_t* too_dense, void* stream) {
  HM_RANGE("hm_swap_partials");
  HM_CHECK_ARG(groups >= 1 && E % groups == 0, "group count %d does not divide %d experts", groups, E);
  HM_CHECK_ARG(E <= 4096, "hm_swap_partials: E too large");
  cudaStream_t s = (cudaStream_t)stream;
  HM_CUDA(cudaMemsetAsync(base, 0, (size_t)groups * 8, s));
  HM_CUDA(cudaMemsetAsync(sel, 0, (size_t)E * 8, s));
  HM_CUDA(cudaMemsetAsync(hitsel, 0, (size_t)E * groups * 8, s));
  HM_CUDA(cudaMemsetAsync(lone, 0, (size_t)E * 8, s));
  HM_CUDA(cudaMemsetAsync(lonesel, 0, (size_t)E * E * 8, s));
  if (T == 0) return 0;
  // tile the `a` dimension so each block's histograms fit in shared memory
  const size_t budget = 160 * 1024;
  int rows = E;
  auto need = [&](int r) { return (size_t)(r * groups + r * E + groups + 2 * r) * 4; };
  while (rows > 1 && need(rows) > budget) rows = (rows + 1) / 2;
  size_t smem = need(rows);
  HM_CUDA(cudaFuncSetAttribute(k_swap_partials, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int blocks = grid_for(T, 256, 64);
  for (int a_lo = 0; a_lo < E; a_lo += rows) {
    int a_hi = a_lo + rows < E ? a_lo + rows : E;
    k_swap_partials<<<blocks, 256, smem, s>>>(bits, T, E, groups, a_lo, a_hi,
                                              (unsigned long long*)base, (unsigned long long*)sel,
                                              (unsigned long long*)hitsel, (unsigned long long*)lone,
                                              (unsigned long long*)lonesel, too_dense);
    HM_LAUNCHED();
  }
  return 0;
}

HM_API int hm_swap_tensor(const int64_t* base, const int64_t* sel, const int64_t* hitsel,
                          const int64_t* lone, const int64_t* lonesel, int32_t E, int32_t groups,
                          int64_t* z, void* stream) {
  HM_RANGE("hm_swap_tensor");
  HM_CHECK_ARG(groups >= 1 && E % groups == 0, "group count %d does not divide %d experts", groups, E);
  int64_t n = (int64_t)E * E * groups;
  int blocks = grid_for(n, 256, kSMs * 16);
  k_swap_tensor<<<blocks, 256, 0, (cudaStream_t)stream>>>(base, sel, hitsel, lone, lonesel, E, groups, z);
  HM_LAUNCHED();
  return 0;
}

// Phase tables are passed as flat host arrays:
//   inter_z[i], inter_groups[i], inter_part[i], a_inter[i], b_inter[i]  (i < depth-1)
//   intra_z[d], intra_groups[d], intra_part[d], a_intra[d], b_intra[d]  (d < depth)
HM_API int hm_swap_cost(const int64_t* const* inter_z, const int32_t* inter_groups,
                        const int32_t* inter_part, const double* a_inter, const double* b_inter,
                        const int64_t* const* intra_z, const int32_t* intra_groups,
                        const int32_t* intra_part, const double* a_intra, const double* b_intra,
                        int32_t depth, int32_t E, int64_t token_bytes, double gamma,
                        const int32_t* dim_dev, int32_t dim_host, double* q, double* q_exact,
                        void* stream) {
  HM_RANGE("hm_swap_cost");
  HM_CHECK_ARG(depth >= 1 && depth <= kMaxPhases, "hm_swap_cost: depth out of range");
  HM_CHECK_ARG(gamma > 0.0, "gamma must be > 0, got %g", gamma);
  CostArgs a;
  memset(&a, 0, sizeof(a));
  a.depth = depth;
  a.E = E;
  a.token_bytes = (double)token_bytes;
  a.gamma = gamma;
  a.gamma_inv = 1.0 / gamma;
  for (int i = 0; i < depth - 1; ++i) {
    HM_CHECK_ARG(inter_groups[i] <= 64, "hm_swap_cost: > 64 groups per cut");
    a.inter[i] = {inter_z[i], inter_groups[i], inter_part[i], a_inter[i], b_inter[i]};
  }
  for (int d = 0; d < depth; ++d) {
    HM_CHECK_ARG(intra_groups[d] <= 64, "hm_swap_cost: > 64 groups per cut");
    a.intra[d] = {intra_z[d], intra_groups[d], intra_part[d], a_intra[d], b_intra[d]};
  }
  int64_t n = (int64_t)E * E;
  int blocks = grid_for(n, 128, kSMs * 8);
  k_cost<<<blocks, 128, 0, (cudaStream_t)stream>>>(a, (const int*)dim_dev, dim_host, q, q_exact);
  HM_LAUNCHED();
  return 0;
}

HM_API int hm_swap_select(const double* q, const double* q_exact, int32_t E, int64_t* out_i64,
                          double* out_f64, void* stream) {
  HM_RANGE("hm_swap_select");
  HM_CHECK_ARG(E >= 1, "hm_swap_select: E < 1");
  k_argmin_select<<<1, 1024, 0, (cudaStream_t)stream>>>(q, q_exact, E, out_i64, out_f64);
  HM_LAUNCHED();
  return 0;
}

// cut_groups: [U[1], ..., U[D-1], G]; dedup counts concatenated in that order.
HM_API int hm_time_model(const int64_t* dedup_concat, const int32_t* fanout_groups /*U[0..D-1]*/,
                         int32_t depth, int32_t gpus, int64_t token_bytes, const double* a_inter,
                         const double* b_inter, const double* a_intra, const double* b_intra,
                         int32_t* cut_offsets_dev, double* times, int32_t* d_star, int64_t* maxima,
                         void* stream) {
  HM_RANGE("hm_time_model");
  HM_CHECK_ARG(depth >= 1 && depth <= kMaxPhases, "hm_time_model: depth out of range");
  TimeArgs a;
  memset(&a, 0, sizeof(a));
  a.depth = depth;
  a.gpus = gpus;
  a.token_bytes = token_bytes;
  for (int i = 0; i < depth; ++i) a.fanout_groups[i] = fanout_groups[i];
  for (int i = 0; i < depth - 1; ++i) {
    a.a_inter[i] = a_inter[i];
    a.b_inter[i] = b_inter[i];
  }
  for (int i = 0; i < depth; ++i) {
    a.a_intra[i] = a_intra[i];
    a.b_intra[i] = b_intra[i];
  }
  k_time_model<<<1, 32, 0, (cudaStream_t)stream>>>(a, (const unsigned long long*)dedup_concat,
                                                    cut_offsets_dev, times, d_star,
                                                    (long long*)maxima);
  HM_LAUNCHED();
  return 0;
}

HM_API int hm_smooth_max_rows(const double* x, int64_t rows, int32_t n, double gamma, double* out,
                              void* stream) {
  HM_CHECK_ARG(n >= 1 && n <= 256, "hm_smooth_max_rows: 1 <= n <= 256");
  HM_CHECK_ARG(gamma >= 1.0, "gamma must be >= 1, got %g", gamma);
  int blocks = grid_for(rows, 128, kSMs * 4);
  k_smooth_max_rows<<<blocks, 128, 0, (cudaStream_t)stream>>>(x, rows, n, gamma, 1.0 / gamma, out);
  HM_LAUNCHED();
  return 0;
}

// elementwise numpy float64 power (np.power rounding, see numpy_pow.cuh)
HM_API int hm_np_pow(const double* x, const double* y, int64_t n, double* out, void* stream) {
  HM_CHECK_ARG(n >= 0, "hm_np_pow: n < 0");
  if (n == 0) return 0;
  int blocks = grid_for(n, 256, kSMs * 16);
  k_np_pow<<<blocks, 256, 0, (cudaStream_t)stream>>>(x, y, n, out);
  HM_LAUNCHED();
  return 0;
}
