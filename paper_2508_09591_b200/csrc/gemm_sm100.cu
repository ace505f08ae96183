// Grouped expert FFN GEMMs on sm_100a tensor cores (tcgen05 + TMA + TMEM).
//
// Expert-major rows (the dispatch output, one contiguous block of n_g rows
// per local expert g) are multiplied by per-expert weights:
//   GEMM1: H[r, :] = silu(X W1_g^T) * (X W3_g^T)   (SwiGLU fused in the epilogue)
//   GEMM2: Y[r, :] = H W2_g^T
// with X [rows, K] bf16 K-major, W [groups * N, K] bf16 K-major, fp32
// accumulation in TMEM, bf16 output.  For GEMM1 the weight rows are packed in
// blocks of 128: rows [256 b, 256 b + 128) = W1 rows [128 b, 128 b + 128) and
// rows [256 b + 128, 256 b + 256) = W3 rows of the same block, so one
// 128 x 256 accumulator tile holds a gate tile and its matching up tile.
//
// Kernel shape (one CTA per SM, persistent over (group, m-tile, n-tile)):
//   warp 0      TMA producer (one elected lane): A 128x64 + B 256x64 bf16 per
//               stage, 128-byte swizzle, 4-stage smem ring (mbarrier full/empty)
//   warp 1      MMA issuer (one lane): 4 x tcgen05.mma.kind::f16 M128 N256 K16
//               per stage into one of two TMEM accumulators (256 columns each),
//               tcgen05.commit -> empty[stage] / tmem_full[acc]
//   warp 2      TMEM allocator (512 columns)
//   warps 4-7   epilogue: tcgen05.ld 32x32b -> fp32 regs -> (SwiGLU) -> bf16
//               stores, rows >= n_g masked; arrive tmem_empty[acc]
// Group sizes are read on the device (no host sync).

#include "hm_common.cuh"
#include "exch.cuh"

#include <atomic>
#include <cuda.h>
#include <cuda_bf16.h>
#include <string.h>

namespace {

using namespace hm;

constexpr int BM = 128, BN = 256, BK = 64, UK = 16;
constexpr int kStages = 4;
constexpr int kThreads = 256;
constexpr uint32_t kABytes = BM * BK * 2;   // 16 KB
constexpr uint32_t kBBytes = BN * BK * 2;   // 32 KB
constexpr uint32_t kStageBytes = kABytes + kBBytes;
constexpr int kMaxGroups = 256;
constexpr uint32_t kTmemCols = 2 * BN;      // double-buffered accumulator
int g_gemm_ctas = 0;   // hm_ffn_set_option(1, n): cap the persistent GEMM grid (0 = all SMs)
int g_wgrad_pair = 1;  // hm_ffn_set_option(2, 0): single-CTA weight gradients (A/B reference)
// hm_ffn_set_option(5, v): 256 x 512 pair tiles -- 0 never, 1 (default) for
// the long-K data-gradient GEMMs with B read as stored (K >= 4096: measured
// 11-16 % faster there, slower elsewhere), 2 wherever N % 512 == 0
int g_wide_tiles = 1;
int g_tma_store = 1;   // hm_ffn_set_option(6, 0): LSU epilogue stores only
struct GemmArgs {
  const int32_t* n_rows;  // [groups] rows per group (device); wgrad: K extent per group
  int groups;
  int m_out;              // wgrad: output rows per group (A rows)
  int N;                  // output features per group (weight rows per group)
  int K;                  // reduction length
  int swiglu;             // 1: out = silu(gate) * up, out_cols = N / 2
  __nv_bfloat16* out;     // [rows, out_cols]
  int64_t ld_out;         // elements
  __nv_bfloat16* out2;    // SwiGLU mode: optional pre-activations [rows, N] (gate/up blocks)
  int accumulate;         // modes 2/3: out += result (fp32 add of the stored bf16)
  int* status;
  // fused dispatch: gather the A rows (modes 0/1, pair kernel) or the B token
  // rows (mode 3) by row index from a token-major source (16-byte cp.async by
  // four producer warps, straight into the 128-byte-swizzled stage) instead
  // of reading materialised expert-major copies: row r of the group layout
  // is source row idx[r] of src (row pitch ld bytes)
  const int32_t* a_idx;
  const int32_t* b_idx;
  const uint8_t* g_src;
  int64_t g_ld;
  // fused dispatch across GPUs: a negative index ~r names row r of g_src2
  // (the receive buffer of rows that arrived over NVLink); same row pitch
  const uint8_t* g_src2;
  // fp32 output (modes 0 / 3; the router GEMMs): outf [rows, ld_out] floats,
  // only the first n_valid columns stored (a zero-padded expert dimension)
  float* outf;
  int n_valid;
  // several EP ranks' expert groups in one launch: groups [s * seg_groups,
  // (s + 1) * seg_groups) are segment s, whose rows start at s * seg_rows
  // (the [L][N_cap] expert-major buffers); seg_groups = 0: one segment
  int seg_groups;
  int64_t seg_rows;
  // explicit groups (pair kernel, modes 0 / 1): group g = rows
  // [g_row0[g], g_row0[g] + n_rows[g]) of the row space, multiplied by weight
  // g_wsel[g] -- e.g. only the rows of one source range of every expert (the
  // overlapped exchange computes the rows already on this GPU first)
  const int32_t* g_row0;
  const int32_t* g_wsel;
  // exchange work run by warp 3 beside the tiles (exch.cuh): 0 none,
  // 1 dispatch rows of exch_x
  const hm::ExchWork* exch;
  int exch_kind;
  const int4* exch_x;
  // mode 0, bf16 rows of exactly N columns: whole 32-row blocks leave the
  // epilogue through TMA tensor stores (map_c) instead of LSU stores
  int tma_store = 0;
  // mode 0, bf16 out: out = bf16((acc + add1) + add2) with fp32 sums, addend
  // rows [rows][ld_out] bf16 (add2 optional) -- the router's input gradient
  // summed with the routed and shared-expert ones, rounded once
  const __nv_bfloat16* add1 = nullptr;
  const __nv_bfloat16* add2 = nullptr;
};


__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

constexpr int kGatherThreads = 128;   // warps 8-11 of a gathering kernel
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
// arrive on `bar` once this thread's cp.async copies so far have landed
__device__ __forceinline__ void cp_async_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ uint32_t mbar_try(uint32_t addr, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(addr), "r"(phase)
      : "memory");
  return ok;
}
// bounded wait: a pipeline bug must not hang the GPU (trap after ~10 s)
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  const uint32_t addr = smem_u32(bar);
  if (mbar_try(addr, phase)) return;
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (!mbar_try(addr, phase)) {
    uint64_t t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (t1 - t0 > 10000000000ull) __trap();
  }
}

// wait with cluster-scope acquire: the stage's arrivals include a release
// from the peer CTA (the gathered A of a CTA pair)
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t phase) {
  const uint32_t addr = smem_u32(bar);
  uint64_t t0 = 0;
  for (int it = 0;; ++it) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(addr), "r"(phase)
        : "memory");
    if (ok) return;
    uint64_t t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (it == 0) t0 = t1;
    if (t1 - t0 > 10000000000ull) __trap();
  }
}

__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* map, uint64_t* bar,
                                            int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

// UMMA shared-memory descriptor, K-major, 128-byte swizzle: 8-row x 128 B
// atoms stacked at SBO = 1024 B; version 1 (sm_100), layout type 2.
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                  // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;        // SBO
  d |= (uint64_t)1 << 46;                  // version
  d |= (uint64_t)2 << 61;                  // SWIZZLE_128B
  return d;
}

// MN-major (transposed) operand, 128-byte swizzle: each K index is one 128 B
// line of 64 MN-contiguous elements; 8-line atoms at SBO = 1024 B along K,
// 64-element MN chunks (separate TMA boxes of 64 lines) at LBO = 8 KB.
__device__ __forceinline__ uint64_t smem_desc_mn(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)(8192 >> 4) << 16;        // LBO: next 64-element MN chunk
  d |= (uint64_t)(1024 >> 4) << 32;        // SBO: next 8 K-lines
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// kind::f16 instruction descriptor: D f32, A/B bf16, both K-major, M=128, N=256
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                            ((uint32_t)(BM >> 4) << 24);
// ... with A and B MN-major (bits 15 / 16: transpose A / B)
constexpr uint32_t kIdescMN = kIdesc | (1u << 15) | (1u << 16);

template <uint32_t IDESC = kIdesc>
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(IDESC), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

// Two 32-column TMEM loads in flight, one wait: the registers are tied to the
// wait (and to an empty volatile asm after it) so no use moves above it.
#define HM_R32(r)                                                                              \
  "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),          \
      "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),  \
      "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),            \
      "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),            \
      "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
#define HM_T32(r)                                                                              \
  "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]),          \
      "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]),  \
      "+r"(r[14]), "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]),            \
      "+r"(r[20]), "+r"(r[21]), "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]),            \
      "+r"(r[26]), "+r"(r[27]), "+r"(r[28]), "+r"(r[29]), "+r"(r[30]), "+r"(r[31])
#define HM_LD32 \
  "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14," \
  "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"

__device__ __forceinline__ void tmem_ld32x2(uint32_t ta, uint32_t tb, float* va, float* vb) {
  uint32_t a[32], b[32];
  asm volatile(HM_LD32 : HM_R32(a) : "r"(ta));
  asm volatile(HM_LD32 : HM_R32(b) : "r"(tb));
  asm volatile("tcgen05.wait::ld.sync.aligned;" : HM_T32(a)::"memory");
  asm volatile("" : HM_T32(b)::"memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    va[i] = __uint_as_float(a[i]);
    vb[i] = __uint_as_float(b[i]);
  }
}

struct TileMap {
  int ntile_n;
  int total;
  int start[kMaxGroups + 1];    // first tile index of each group
  int row0[kMaxGroups];         // first row of each group in A (wgrad: first K column)
  int rows[kMaxGroups];         // rows of each group (wgrad: padded K extent)
  int wsel[kMaxGroups];         // weight index of each group (pair kernel)
};

// first row of each group: prefix sums of the group sizes, restarting at
// every segment's base row
__device__ __forceinline__ int seg_row0(const GemmArgs& a, int g, int run) {
  return (a.seg_groups > 0 && g % a.seg_groups == 0) ? (int)((g / a.seg_groups) * a.seg_rows)
                                                       : run;
}

__device__ __forceinline__ void tile_coords(const TileMap& tm, int groups, int t, int& g, int& mt,
                                            int& nt) {
  int lo = 0, hi = groups - 1;   // last group with start <= t (binary search)
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (tm.start[mid] <= t) lo = mid; else hi = mid - 1;
  }
  g = lo;
  int local = t - tm.start[g];
  mt = local / tm.ntile_n;
  nt = local % tm.ntile_n;
}

// Coalesced epilogue stores through a 4 KB per-warp shared-memory stage:
// each lane writes its own row's U 16-byte units (swizzled: unit u of row r
// at u ^ key(r), conflict-free), then the warp stores R = 32 / U rows per
// instruction with U lanes per row, so every global store instruction writes
// whole 64 / 128-byte row segments instead of 32 rows x 16 bytes (the
// row-per-lane TMEM layout made the epilogue the GEMM's bottleneck: with the
// stores skipped, GEMM2 ran at 1450 instead of 1077 TFLOP/s).  Rows >= nvalid
// (past the group) are not written.
constexpr int kEpiStageBytes = 4096;   // per epilogue warp
__device__ __forceinline__ void sts128(uint32_t a, int4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}
__device__ __forceinline__ int4 lds128(uint32_t a) {
  int4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(a)
               : "memory");
  return v;
}
template <int U>
__device__ __forceinline__ void stage_store(uint8_t* sw, int lane, const int4* v,
                                            __nv_bfloat16* dst0, int64_t ld, int nvalid,
                                            int umax = U) {
  const uint32_t base = smem_u32(sw);   // explicit shared-window accesses (STS / LDS)
  // swizzle key of row r: rows sharing a 128-byte bank line (8 / U of them)
  // get the same key, consecutive lines different ones, so the 8 lanes of a
  // 16-byte store phase hit 8 distinct 16-byte bank groups
  constexpr int RPL = U >= 8 ? 1 : 8 / U;
#pragma unroll
  for (int u = 0; u < U; ++u)
    sts128(base + lane * (U * 16) + ((u ^ ((lane / RPL) % U)) << 4), v[u]);
  __syncwarp();
  constexpr int R = 32 / U;
  const int ur = lane % U, rr = lane / U;
#pragma unroll
  for (int p = 0; p < U; ++p) {
    const int r = p * R + rr;
    const int4 w = lds128(base + r * (U * 16) + ((ur ^ ((r / RPL) % U)) << 4));
    if (r < nvalid && ur < umax) *reinterpret_cast<int4*>(dst0 + (int64_t)r * ld + ur * 8) = w;
  }
  __syncwarp();
}

// silu(g) = g * rcp(1 + exp(-g)) on the MUFU (the IEEE division's fix-up
// sequence made the SwiGLU epilogue instruction-bound); g << 0: rcp(inf) = 0
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// Epilogue of one accumulator tile for the 32 rows of TMEM lane quarter q:
// TMEM -> fp32 registers -> (SwiGLU / accumulate) -> bf16 rows.  r0 = the
// warp's first row within group g (weight-gradient modes: output row); sw =
// the warp's shared-memory store stage.
// TMA tensor store of one warp's 32 rows x 64 columns (bf16): the stage is
// written in the 128-byte swizzle (unit u of row r at u ^ (r % 8), the same
// layout stage_store<8> uses, stage 1024-byte aligned) and lane 0 issues one
// cp.async.bulk.tensor store -- the row data leave through the async proxy
// instead of 8 LSU store instructions per lane.  The previous store must have
// finished reading the stage first (wait_group.read).
__device__ __forceinline__ void tma_store_wait_read(int lane) {
  if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  __syncwarp();
}
__device__ __forceinline__ void tma_store_chunk(uint8_t* sw, int lane, const int4* v,
                                                const CUtensorMap* map, int col, int row) {
  const uint32_t base = smem_u32(sw);
  tma_store_wait_read(lane);
#pragma unroll
  for (int u = 0; u < 8; ++u) sts128(base + lane * 128 + ((u ^ (lane & 7)) << 4), v[u]);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (lane == 0) {
    asm volatile(
        "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
            reinterpret_cast<uint64_t>(map)),
        "r"(col), "r"(row), "r"(base)
        : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
}

// kHalfStage: 2 KB store stages (the NA = 2 pair kernel's eight epilogue
// warps): bf16 rows go out as 64-byte instead of 128-byte row segments
template <int kMode, bool kHalfStage = false>
__device__ __forceinline__ void store_tile(const GemmArgs& args, const TileMap& tm, int g, int nt,
                                           int r0, int lane, uint32_t tbase, uint8_t* sw,
                                           const CUtensorMap* tmac = nullptr) {
  int nvalid = kMode >= 2 ? 32 : tm.rows[g] - r0;
  nvalid = nvalid < 0 ? 0 : (nvalid > 32 ? 32 : nvalid);
  const bool valid = lane < nvalid;
  const bool zero = kMode >= 2 && tm.rows[g] == 0;    // empty K: nothing accumulated
  const int64_t row_base = kMode >= 2 ? (int64_t)g * args.m_out + r0 : (int64_t)(tm.row0[g] + r0);
  if (kMode != 1 && args.outf) {   // fp32 rows, 32 columns (128 B) per staged store
#pragma unroll 1
    for (int c2 = 0; c2 < BN; c2 += 64) {
      if (nt * BN + c2 >= args.n_valid) break;
      float v2[2][32];
      tmem_ld32x2(tbase + c2, tbase + c2 + 32, v2[0], v2[1]);
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const int col = nt * BN + c2 + 32 * half;
        if (col >= args.n_valid) break;
        float* v = v2[half];
        if (zero) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = 0.f;
        }
        if (kMode >= 2 && args.accumulate && valid) {
          const float4* old = reinterpret_cast<const float4*>(args.outf + (row_base + lane) *
                                                              args.ld_out + col);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float4 o = old[i];
            v[4 * i] += o.x;
            v[4 * i + 1] += o.y;
            v[4 * i + 2] += o.z;
            v[4 * i + 3] += o.w;
          }
        }
        // 32 floats = 8 16-byte units (stage_store moves them as raw bits);
        // a partial last chunk stores only its first (n_valid - col) / 4 units
        const int um = (args.n_valid - col) >= 32 ? 8 : (args.n_valid - col) / 4;
        stage_store<8>(sw, lane, reinterpret_cast<const int4*>(v),
                       reinterpret_cast<__nv_bfloat16*>(args.outf + row_base * args.ld_out + col),
                       args.ld_out * 2, nvalid, um);
      }
    }
    return;
  }
  __nv_bfloat16* orow = args.out + (row_base + lane) * args.ld_out;
  if (kMode == 1) {
#pragma unroll 1
    for (int c = 0; c < BN / 2; c += 32) {
      float gv[32], uv[32];
      tmem_ld32x2(tbase + c, tbase + BN / 2 + c, gv, uv);
      __align__(16) __nv_bfloat162 hv[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        float g0 = gv[2 * i], g1 = gv[2 * i + 1];
        float h0 = g0 * rcp_approx(1.f + __expf(-g0)) * uv[2 * i];
        float h1 = g1 * rcp_approx(1.f + __expf(-g1)) * uv[2 * i + 1];
        hv[i] = __floats2bfloat162_rn(h0, h1);
      }
      stage_store<4>(sw, lane, reinterpret_cast<const int4*>(hv),
                     args.out + row_base * args.ld_out + nt * (BN / 2) + c, args.ld_out, nvalid);
      if (args.out2) {   // keep the pre-activations for the backward
        __nv_bfloat16* p0 = args.out2 + (int64_t)(tm.row0[g] + r0) * args.N + nt * BN + c;
        __align__(16) __nv_bfloat162 gb[16], ub[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          gb[i] = __floats2bfloat162_rn(gv[2 * i], gv[2 * i + 1]);
          ub[i] = __floats2bfloat162_rn(uv[2 * i], uv[2 * i + 1]);
        }
        stage_store<4>(sw, lane, reinterpret_cast<const int4*>(gb), p0, args.N, nvalid);
        stage_store<4>(sw, lane, reinterpret_cast<const int4*>(ub), p0 + BN / 2, args.N, nvalid);
      }
    }
  } else if (kMode >= 2 && args.accumulate) {   // weight grads summed over micro-batches
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      float v[32], unused[32];
      tmem_ld32x2(tbase + c, tbase + c, v, unused);
      if (zero) {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = 0.f;
      }
      int4* dst = reinterpret_cast<int4*>(orow + nt * BN + c);
      __align__(16) __nv_bfloat162 old[16], hv[16];
#pragma unroll
      for (int i = 0; i < 4; ++i) reinterpret_cast<int4*>(old)[i] = dst[i];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float2 o = __bfloat1622float2(old[i]);
        hv[i] = __floats2bfloat162_rn(v[2 * i] + o.x, v[2 * i + 1] + o.y);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) dst[i] = reinterpret_cast<const int4*>(hv)[i];
    }
  } else {
#pragma unroll 1
    for (int c2 = 0; c2 < BN; c2 += 64) {
      float v2[2][32];
      tmem_ld32x2(tbase + c2, tbase + c2 + 32, v2[0], v2[1]);
      if (kMode == 0 && args.add1 && valid) {   // + bf16 addends, this lane's row
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const __nv_bfloat16* ad = t ? args.add2 : args.add1;
          if (!ad) break;
          const int4* ap =
              reinterpret_cast<const int4*>(ad + (row_base + lane) * args.ld_out + nt * BN + c2);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int4 w = __ldg(ap + q);
            const __nv_bfloat162* w2 = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 f = __bfloat1622float2(w2[e]);
              v2[q >> 2][(q & 3) * 8 + 2 * e] += f.x;
              v2[q >> 2][(q & 3) * 8 + 2 * e + 1] += f.y;
            }
          }
        }
      }
      __align__(16) __nv_bfloat162 hv[32];
#pragma unroll
      for (int half = 0; half < 2; ++half)
#pragma unroll
        for (int i = 0; i < 16; ++i)
          hv[16 * half + i] = zero ? __floats2bfloat162_rn(0.f, 0.f)
                                   : __floats2bfloat162_rn(v2[half][2 * i], v2[half][2 * i + 1]);
      __nv_bfloat16* dst = args.out + row_base * args.ld_out + nt * BN + c2;
      if (tmac && nvalid == 32 && !zero) {   // whole 32-row block: TMA tensor store
        tma_store_chunk(sw, lane, reinterpret_cast<const int4*>(hv), tmac, nt * BN + c2,
                        (int)row_base);
        continue;
      }
      if (tmac) tma_store_wait_read(lane);    // the stage may still be read by a TMA store
      if (kHalfStage) {
        stage_store<4>(sw, lane, reinterpret_cast<const int4*>(hv), dst, args.ld_out, nvalid);
        stage_store<4>(sw, lane, reinterpret_cast<const int4*>(hv) + 4, dst + 32, args.ld_out,
                       nvalid);
      } else {
        stage_store<8>(sw, lane, reinterpret_cast<const int4*>(hv), dst, args.ld_out, nvalid);
      }
    }
  }
  (void)valid;
}

// kMode 0: out = A_g B_g^T over row groups; 1: same + SwiGLU epilogue;
// 2: weight-gradient mode -- every group g is a full [m_out x N] output
// (rows g*m_out..), reducing over its own K range [row0_g, row0_g + rows_g)
// of A [m_out x K_total] and B [N x K_total] (K_total = padded token rows).
// 3: weight gradient straight from the token-major activations, no
// transposes: out_g = A_g^T B_g with A [tokens, m_out], B [tokens, N] (the
// group's tokens are its rows), both operands MN-major in shared memory (TMA
// boxes of 64 tokens x 64 features, one 128 B line per token); the tail
// k-block's lines past the group are zeroed before the MMA reads them.
// GB (mode 3 only): B's token rows are gathered by index (args.b_idx) by
// warps 8-11 with cp.async into the swizzled stage instead of TMA boxes
template <int kMode, bool GB = false>
__global__ void __launch_bounds__(GB ? kThreads + kGatherThreads : kThreads, 1)
    k_grouped_gemm(const __grid_constant__ CUtensorMap map_a,
                   const __grid_constant__ CUtensorMap map_b, GemmArgs args) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sa = smem;
  uint8_t* sb = smem + kStages * kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  uint8_t* epi = smem + kStages * kStageBytes + 256;   // epilogue store stages
  __shared__ TileMap tm;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    int acc = 0, row = 0;
    tm.ntile_n = args.N / BN;
    for (int g = 0; g < args.groups; ++g) {
      int n = args.n_rows[g];
      if (kMode == 2) n = (n + BK - 1) / BK * BK;   // K padded to the k-block
      row = seg_row0(args, g, row);
      tm.start[g] = acc;
      tm.row0[g] = row;
      tm.rows[g] = n;
      acc += (kMode >= 2 ? args.m_out / BM : (n + BM - 1) / BM) * tm.ntile_n;
      row += n;
    }
    tm.start[args.groups] = acc;
    tm.total = acc;
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full + s, GB ? 1 + kGatherThreads : 1);
      mbar_init(empty + s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull + a, 1);
      mbar_init(tempty + a, 4);   // one arrive per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int kblocks_fixed = args.K / BK;

  if (warp == 0) {
    // lane 0 drives the ring (with GB only A's boxes; warps 8-11 fill B)
    constexpr bool gather_b = kMode == 3 && GB;
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");

      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < tm.total; t += gridDim.x) {
        int g, mt, nt;
        tile_coords(tm, args.groups, t, g, mt, nt);
        const int arow = kMode >= 2 ? mt * BM : tm.row0[g] + mt * BM;
        const int brow = kMode >= 2 ? nt * BN : g * args.N + nt * BN;
        const int k0 = kMode >= 2 ? tm.row0[g] : 0;
        const int kblocks = kMode == 2   ? tm.rows[g] / BK
                            : kMode == 3 ? (tm.rows[g] + BK - 1) / BK
                                         : kblocks_fixed;
        for (int kb = 0; kb < kblocks; ++kb) {
          {
            mbar_wait(empty + stage, phase ^ 1);
            mbar_expect_tx(full + stage, gather_b ? kABytes : kStageBytes);
            if (kMode == 3) {   // 64-token x 64-feature boxes: 2 for A, 4 for B
#pragma unroll
              for (int j = 0; j < BM / 64; ++j)
                tma_load_2d(sa + stage * kABytes + j * 8192, &map_a, full + stage, arow + 64 * j,
                            k0 + kb * BK);
              if (!gather_b) {
#pragma unroll
                for (int j = 0; j < BN / 64; ++j)
                  tma_load_2d(sb + stage * kBBytes + j * 8192, &map_b, full + stage,
                              brow + 64 * j, k0 + kb * BK);
              }
            } else {
              tma_load_2d(sa + stage * kABytes, &map_a, full + stage, k0 + kb * BK, arow);
              tma_load_2d(sb + stage * kBBytes, &map_b, full + stage, k0 + kb * BK, brow);
            }
          }
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1 && kMode == 3) {
    // whole warp: lanes zero the tail k-block's lines past the group, lane 0
    // issues the MMAs (MN-major operands: a 16-token k-step is 16 lines)
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int t = blockIdx.x; t < tm.total; t += gridDim.x, ++it) {
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      mbar_wait(tempty + acc, acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d = tmem_base + acc * BN;
      int g, mt, nt;
      tile_coords(tm, args.groups, t, g, mt, nt);
      const int kblocks = (tm.rows[g] + BK - 1) / BK;
      for (int kb = 0; kb < kblocks; ++kb) {
        mbar_wait(full + stage, phase);
        const int valid = tm.rows[g] - kb * BK;
        // tail block: MMAs only for the 16-token steps that hold group rows;
        // the lines of the last partial step past the group are zeroed in all
        // 6 boxes (at most 15 lines)
        const int ksteps = valid >= BK ? BK / UK : (valid + UK - 1) / UK;
        const int zend = ksteps * UK;
        if (valid < zend) {
          const int nlines = zend - valid;
          for (int i = lane; i < 6 * nlines * 8; i += 32) {
            const int box = i / (nlines * 8), rem = i % (nlines * 8);
            const int line = valid + rem / 8, chunk = rem % 8;
            uint8_t* base = box < 2 ? sa + stage * kABytes + box * 8192
                                    : sb + stage * kBBytes + (box - 2) * 8192;
            *reinterpret_cast<int4*>(base + line * 128 + chunk * 16) = make_int4(0, 0, 0, 0);
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
        }
        if (lane == 0) {
          tc_fence_after();
          const uint32_t a0 = smem_u32(sa + stage * kABytes);
          const uint32_t b0 = smem_u32(sb + stage * kBBytes);
          for (int k = 0; k < ksteps; ++k)
            umma_bf16<kIdescMN>(d, smem_desc_mn(a0 + k * UK * 128),
                                smem_desc_mn(b0 + k * UK * 128), (kb | k) ? 1u : 0u);
          umma_commit(empty + stage);
        }
        __syncwarp();
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (lane == 0) umma_commit(tfull + acc);
      __syncwarp();
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = blockIdx.x; t < tm.total; t += gridDim.x, ++it) {
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait(tempty + acc, acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + acc * BN;
        int kblocks = kblocks_fixed;
        if (kMode == 2) {
          int g, mt, nt;
          tile_coords(tm, args.groups, t, g, mt, nt);
          kblocks = tm.rows[g] / BK;
        }
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(full + stage, phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sa + stage * kABytes);
          const uint32_t b0 = smem_u32(sb + stage * kBBytes);
#pragma unroll
          for (int k = 0; k < BK / UK; ++k)
            umma_bf16(d, smem_desc(a0 + k * UK * 2), smem_desc(b0 + k * UK * 2),
                      (kb | k) ? 1u : 0u);
          umma_commit(empty + stage);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(tfull + acc);
      }
    }
  } else if (warp >= 4 && warp < 8) {
    const int q = warp - 4;  // TMEM lane quarter
    int it = 0;
    for (int t = blockIdx.x; t < tm.total; t += gridDim.x, ++it) {
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      int g, mt, nt;
      tile_coords(tm, args.groups, t, g, mt, nt);
      mbar_wait(tfull + acc, acc_phase);
      tc_fence_after();
      store_tile<kMode>(args, tm, g, nt, mt * BM + q * 32, lane,
                        tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN,
                        epi + q * kEpiStageBytes);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty + acc);
    }
  } else if (GB && warp >= 8) {
    // B gather (mode 3): 64 token lines x 4 feature boxes x 8 16-byte chunks
    // per stage; thread g owns chunk g % 8 of lines g / 8 + 16 i in every box
    const int g_t = threadIdx.x - kThreads;
    const int c = g_t & 7, l0 = g_t >> 3;
    int stage = 0;
    uint32_t phase = 0;
    for (int t = blockIdx.x; t < tm.total; t += gridDim.x) {
      int g, mt, nt;
      tile_coords(tm, args.groups, t, g, mt, nt);
      const int kblocks = (tm.rows[g] + BK - 1) / BK;
      const int end = tm.row0[g] + tm.rows[g];
      const uint8_t* col = args.g_src + (int64_t)(nt * BN + 8 * c) * 2;
      // the k-block's token indices are loaded one k-block ahead (their load
      // latency would otherwise sit in every stage's critical path)
      auto load_tok = [&](int kb, int* tk) {
        const int r0 = tm.row0[g] + kb * BK + l0;
#pragma unroll
        for (int i = 0; i < 4; ++i) tk[i] = args.b_idx[r0 + 16 * i < end ? r0 + 16 * i : tm.row0[g]];
      };
      int nxt[4];
      load_tok(0, nxt);
      for (int kb = 0; kb < kblocks; ++kb) {
        int tok[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) tok[i] = nxt[i];
        if (kb + 1 < kblocks) load_tok(kb + 1, nxt);
        mbar_wait(empty + stage, phase ^ 1);
        const uint32_t base = smem_u32(sb + stage * kBBytes);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int l = l0 + 16 * i;
          const int v = tok[i];
          const uint8_t* src = v >= 0 ? col + (int64_t)v * args.g_ld
                                      : col + (args.g_src2 - args.g_src) + (int64_t)(~v) * args.g_ld;
          const uint32_t dl = base + l * 128 + ((c ^ (l & 7)) << 4);
#pragma unroll
          for (int j = 0; j < BN / 64; ++j) cp_async16(dl + j * 8192, src + j * 128);
        }
        cp_async_arrive(full + stage);
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(kTmemCols));
  }
}


// ---------------------------------------------------------------------------
// CTA-pair variant (modes 0 / 1): a cluster of 2 CTAs on one TPC computes a
// 256 x 256 tile with tcgen05.mma.cta_group::2 -- each CTA stages 128 rows of
// A and half (128 rows) of B per k-block (32 KB instead of 48 KB, so 6
// stages fit), both CTAs' TMA loads complete on the leader's full barrier,
// the leader's single MMA thread drives both SMs' tensor cores, commits are
// multicast to both CTAs' barriers, and each CTA's epilogue drains the 128
// accumulator rows in its own TMEM (arriving on the leader's tmem-empty
// barrier through the cluster window).
constexpr int BM2 = 256, kStages2 = 6;
constexpr uint32_t kHalfBytes = 128 * BK * 2;                 // 16 KB
constexpr uint32_t kStageBytes2 = 2 * kHalfBytes;             // A half + B half per CTA
constexpr uint32_t kIdesc2 = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)(BM2 >> 4) << 24);

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n"
               "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// TMA load into this CTA's smem, completing on the pair leader's barrier
__device__ __forceinline__ void tma_load_2d_pair(void* smem_dst, const CUtensorMap* map,
                                                 uint64_t* bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar) & 0xFEFFFFFFu)
      : "memory");
}
// tcgen05.mma / commit on a CTA pair, issued by one elected lane of a warp
// that runs the loop in lockstep:
// the operands are warp-uniform, so they stay on the uniform datapath (no
// per-MMA waterfall loop moving a single lane's registers to uniform ones)
// TMA pair load / expect-tx by one elected lane of a lockstep warp
__device__ __forceinline__ void tma_load_2d_pair_elect(void* smem_dst, const CUtensorMap* map,
                                                       uint64_t* bar, int x, int y) {
  asm volatile(
      "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
      " @e cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];\n}\n" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar) & 0xFEFFFFFFu)
      : "memory");
}
__device__ __forceinline__ void mbar_expect_tx_elect(uint64_t* bar, uint32_t bytes) {
  asm volatile(
      "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
      " @e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n}\n" ::"r"(smem_u32(bar)),
      "r"(bytes)
      : "memory");
}
template <uint32_t IDESC = kIdesc2>
__device__ __forceinline__ void umma_bf16_pair_elect(uint32_t tmem_d, uint64_t adesc,
                                                     uint64_t bdesc, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p, e;\n setp.ne.b32 p, %4, 0;\n elect.sync _|e, 0xffffffff;\n"
      " @e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(IDESC), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit_pair_elect(uint64_t* bar) {
  asm volatile(
      "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
      " @e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;\n}\n" ::"r"(smem_u32(bar)),
      "h"((uint16_t)0x3)
      : "memory");
}
// ... with B MN-major (bit 16: transpose B): the weights used as stored
constexpr uint32_t kIdesc2BMN = kIdesc2 | (1u << 16);
// arrive on the barrier at the same offset in CTA `rank` of the cluster.
// Default (.release.cta) semantics: the only user is the epilogue's
// TMEM-empty arrive, ordered after its tcgen05.ld by the before_thread_sync
// fence; a .release.cluster arrive compiled to MEMBAR.ALL.GPU + ERRBAR, i.e.
// waited for the tile's global stores (2-3 % of GEMM time)
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t* bar, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(rank));
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}

// ---------------------------------------------------------------------------
// Exchange executor (exch.cuh), one warp per CTA.  Rows are walked in the
// dispatch kernels' spread order so concurrent warps' NVLink stores land all
// over the peers' buffers.
__device__ __forceinline__ int64_t exch_spread(int64_t i, int64_t n) {
  const int64_t p = (n % 7919) ? 7919 : ((n % 104729) ? 104729 : 1);
  return (i * p) % n;
}
__device__ __forceinline__ int4 exch_ld(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void exch_st(int4* p, int4 v) {
  asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w));
}
constexpr int kExchU = 8;   // 16-byte vectors per lane in flight

// kind 1: token t's row to every other GPU q with a receive row gpos_g[t][q]
__device__ __noinline__ void exch_push(const hm::ExchWork& e, const int4* x, int lane) {
  const int64_t n = e.ntok, nvec = e.nvec;
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
    const int64_t t = exch_spread(i, n);
    int4* mine = nullptr;
    if (lane < e.P && lane != e.p) {
      const int g = e.gpos_g[t * e.P + lane];
      if (g >= 0 && g < e.rg_cap) mine = e.recv_g[lane] + (int64_t)g * nvec;
    }
    const unsigned m = __ballot_sync(0xffffffffu, mine != nullptr);
    if (!m) continue;
    const int4* src = x + t * nvec;
    for (int64_t v0 = 0; v0 < nvec; v0 += 32 * kExchU) {
      int4 buf[kExchU];
#pragma unroll
      for (int u = 0; u < kExchU; ++u) {
        const int64_t v = v0 + u * 32 + lane;
        if (v < nvec) buf[u] = exch_ld(src + v);
      }
      for (unsigned mm = m; mm; mm &= mm - 1) {
        int4* d = reinterpret_cast<int4*>(
            __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(mine), __ffs(mm) - 1));
#pragma unroll
        for (int u = 0; u < kExchU; ++u) {
          const int64_t v = v0 + u * 32 + lane;
          if (v < nvec) exch_st(d + v, buf[u]);
        }
      }
    }
  }
}

// GA (modes 0/1): the A rows are gathered by index (args.a_idx) by warps 8-11
// of each CTA with cp.async into its swizzled stage; they arrive on a local
// gfull barrier, and warp 2's lane 0 forwards each completed stage to the
// leader's full barrier (which then counts the B TMA bytes + 2 forwarders)
// BMN: B read MN-major straight from [groups][K][N] weights (two 64 x 64 TMA
// boxes per CTA and k-block, the tcgen05 transpose-B bit) -- the data-gradient
// GEMMs then need no transposed weight copies
// NA = 2 (r2, "wide" tiles): 256 x 512 output tiles, two N = 256 MMAs per
// k-step sharing the A half (per-CTA operand bytes per flop -25 %: 48 KB per
// 16.8 MFLOP instead of 32 KB per 8.4) -- the TMEM then holds one tile's two
// accumulators (all 512 columns), so the epilogue releases them one at a
// time (tempty[0] / tempty[1]) and the MMA warp runs the next tile's first
// k-blocks on accumulator 0 (holding their stages) until accumulator 1 is
// drained.  4 ring stages of 48 KB.  Same k order per output element as
// NA = 1: bit-identical results.
constexpr int kEpi2Threads = 128;   // NA = 2: a second epilogue warpgroup (accumulator 1)
template <int NA>
struct PairCfg {
  static constexpr int kStages = NA == 1 ? kStages2 : 4;
  static constexpr uint32_t kBBytes = NA * kHalfBytes;        // this CTA's B halves
  static constexpr uint32_t kStage = kHalfBytes + kBBytes;    // A half + B halves
  static constexpr int kEpiStage = kEpiStageBytes / NA;       // per epilogue warp
  static constexpr size_t smem() {
    return (size_t)kStages * kStage + 1024 + 1024 + 4 * NA * kEpiStage;
  }
};
template <int kMode, bool GA = false, bool BMN = false, int NA = 1>
__global__ void __cluster_dims__(2, 1, 1)
    __launch_bounds__(kThreads + (GA ? kGatherThreads : 0) + (NA == 2 ? kEpi2Threads : 0), 1)
    k_grouped_gemm_pair(const __grid_constant__ CUtensorMap map_a,
                        const __grid_constant__ CUtensorMap map_b,
                        const __grid_constant__ CUtensorMap map_c, GemmArgs args) {
  using C = PairCfg<NA>;
  constexpr int ST = C::kStages;
  constexpr int kEpi2Warp = (kThreads + (GA ? kGatherThreads : 0)) / 32;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sa = smem;
  uint8_t* sb = smem + ST * kHalfBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ST * C::kStage);
  uint64_t* empty = full + ST;
  uint64_t* tfull = empty + ST;
  uint64_t* tempty = tfull + 2;
  uint64_t* gfull = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gfull + ST);
  uint8_t* epi = smem + ST * C::kStage + 1024;   // epilogue store stages (1024-B aligned)
  __shared__ TileMap tm;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  if (threadIdx.x == 0) {
    int acc = 0, row = 0;
    tm.ntile_n = args.N / (BN * NA);
    for (int g = 0; g < args.groups; ++g) {
      int n = args.n_rows[g];
      if (kMode == 2) n = (n + BK - 1) / BK * BK;   // K padded to the k-block
      row = args.g_row0 ? args.g_row0[g] : seg_row0(args, g, row);
      tm.start[g] = acc;
      tm.row0[g] = row;
      tm.rows[g] = n;
      tm.wsel[g] = args.g_wsel ? args.g_wsel[g] : g;
      acc += (kMode == 2 ? args.m_out / BM2 : (n + BM2 - 1) / BM2) * tm.ntile_n;
      row += n;
    }
    tm.start[args.groups] = acc;
    tm.total = acc;
    for (int s = 0; s < ST; ++s) {
      mbar_init(full + s, GA ? 3 : 1);
      mbar_init(empty + s, 1);
      mbar_init(gfull + s, kGatherThreads);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull + a, 1);
      mbar_init(tempty + a, 8);   // 4 epilogue warps in each CTA of the pair
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int kblocks_fixed = args.K / BK;

  if (warp == 0) {
    // the warp drives the ring in lockstep, one elected lane issuing (with GA
    // only B's TMA loads; warps 8-11 fill A)
    {
      if (lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
      }
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cid; t < tm.total; t += ncl) {
        int g, mt, nt;
        tile_coords(tm, args.groups, t, g, mt, nt);
        // mode 2 (weight gradient from transposed operands): A [m_out][K_all],
        // B [N][K_all], group g's reduction range = its padded token columns
        const int arow = (kMode == 2 ? 0 : tm.row0[g]) + mt * BM2 + (int)rank * 128;
        const int brow = (kMode == 2 ? 0 : tm.wsel[g] * args.N) + nt * BN * NA + (int)rank * 128;
        const int k0 = kMode == 2 ? tm.row0[g] : 0;
        const int kblocks = kMode == 2 ? tm.rows[g] / BK : kblocks_fixed;
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(empty + stage, phase ^ 1);
          if (leader) mbar_expect_tx_elect(full + stage, GA ? 2 * C::kBBytes : 2 * C::kStage);
          if (!GA)
            tma_load_2d_pair_elect(sa + stage * kHalfBytes, &map_a, full + stage, k0 + kb * BK, arow);
#pragma unroll
          for (int a = 0; a < NA; ++a) {
            uint8_t* sbs = sb + stage * C::kBBytes + a * kHalfBytes;
            if (BMN) {   // B [g][K][N]: rows g * K + k, 64-column chunks of this CTA's 128
              const int bcol = nt * BN * NA + a * BN + (int)rank * 128;
#pragma unroll
              for (int j = 0; j < 2; ++j)
                tma_load_2d_pair_elect(sbs + j * 8192, &map_b, full + stage, bcol + 64 * j,
                                 tm.wsel[g] * args.K + kb * BK);
            } else {
              tma_load_2d_pair_elect(sbs, &map_b, full + stage, k0 + kb * BK, brow + a * BN);
            }
          }
          if (++stage == ST) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {   // the whole warp runs the loop; one elected lane issues
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      // one k-block's MMAs into accumulator a (TMEM columns a * 256)
      // descriptors built once per k-block; the k-steps advance the 14-bit
      // start-address field (16-byte units, no carry below 256 KB): +2 per
      // 32-byte K step (K-major), +128 per 16 K lines (MN-major B)
      auto mma_kb = [&](uint32_t d, int st, int kb, int a) {
        const uint64_t da = smem_desc(smem_u32(sa + st * kHalfBytes));
        const uint32_t b0 = smem_u32(sb + st * C::kBBytes + a * kHalfBytes);
        const uint64_t db = BMN ? smem_desc_mn(b0) : smem_desc(b0);
#pragma unroll
        for (int k = 0; k < BK / UK; ++k) {
          if (BMN)
            umma_bf16_pair_elect<kIdesc2BMN>(d, da + 2 * k, db + 128 * k, (kb | k) ? 1u : 0u);
          else
            umma_bf16_pair_elect(d, da + 2 * k, db + 2 * k, (kb | k) ? 1u : 0u);
        }
      };
      auto wait_full = [&](int st, uint32_t ph) {
        if (GA)
          mbar_wait_cluster(full + st, ph);
        else
          mbar_wait(full + st, ph);
        tc_fence_after();
      };
      for (int t = cid; t < tm.total; t += ncl, ++it) {
        int kblocks = kblocks_fixed;
        if (kMode == 2) {
          int g, mt, nt;
          tile_coords(tm, args.groups, t, g, mt, nt);
          kblocks = tm.rows[g] / BK;
        }
        if (NA == 1) {
          const int acc = it & 1;
          const uint32_t acc_phase = (it >> 1) & 1;
          mbar_wait(tempty + acc, acc_phase ^ 1);
          tc_fence_after();
          const uint32_t d = tmem_base + acc * BN;
          for (int kb = 0; kb < kblocks; ++kb) {
            wait_full(stage, phase);
            mma_kb(d, stage, kb, 0);
            umma_commit_pair_elect(empty + stage);
            if (++stage == ST) {
              stage = 0;
              phase ^= 1;
            }
          }
          umma_commit_pair_elect(tfull + acc);
        } else {
          // single TMEM buffer: accumulator 0 as soon as the epilogue released
          // it; accumulator 1's MMAs of the held stages once it is released too
          const uint32_t tph = (it & 1) ^ 1;
          mbar_wait(tempty + 0, tph);
          tc_fence_after();
          bool free1 = false;
          int held = 0, hstage = stage, hkb = 0;
          for (int kb = 0; kb < kblocks; ++kb) {
            wait_full(stage, phase);
            mma_kb(tmem_base, stage, kb, 0);
            if (!free1) {
              if (held + 1 >= ST) {
                mbar_wait(tempty + 1, tph);
                free1 = true;
              } else {
                free1 = __shfl_sync(0xffffffffu, mbar_try(smem_u32(tempty + 1), tph), 0) != 0;
              }
              if (free1) tc_fence_after();
            }
            if (free1) {
              for (; held > 0; --held) {   // catch up on the held stages
                mma_kb(tmem_base + BN, hstage, hkb, 1);
                umma_commit_pair_elect(empty + hstage);
                if (++hstage == ST) hstage = 0;
                ++hkb;
              }
              mma_kb(tmem_base + BN, stage, kb, 1);
              umma_commit_pair_elect(empty + stage);
            } else {
              if (held++ == 0) {
                hstage = stage;
                hkb = kb;
              }
            }
            if (++stage == ST) {
              stage = 0;
              phase ^= 1;
            }
          }
          if (!free1) {   // fewer k-blocks than the epilogue took to drain
            mbar_wait(tempty + 1, tph);
            tc_fence_after();
            for (; held > 0; --held) {
              mma_kb(tmem_base + BN, hstage, hkb, 1);
              umma_commit_pair_elect(empty + hstage);
              if (++hstage == ST) hstage = 0;
              ++hkb;
            }
          }
          umma_commit_pair_elect(tfull + 0);
        }
      }
    }
  } else if ((warp >= 4 && warp < 8) || (NA == 2 && warp >= kEpi2Warp)) {
    // NA = 2: warps 4-7 drain accumulator 0, the second warpgroup accumulator 1
    const int q = warp & 3;
    const int a = (NA == 2 && warp >= kEpi2Warp) ? 1 : 0;
    int it = 0;
    for (int t = cid; t < tm.total; t += ncl, ++it) {
      const int acc = NA == 1 ? it & 1 : 0;
      const uint32_t acc_phase = NA == 1 ? (it >> 1) & 1 : it & 1;
      int g, mt, nt;
      tile_coords(tm, args.groups, t, g, mt, nt);
      mbar_wait(tfull + acc, acc_phase);
      tc_fence_after();
      store_tile<kMode, NA == 2>(args, tm, g, nt * NA + a, mt * BM2 + (int)rank * 128 + q * 32,
                                 lane, tmem_base + ((uint32_t)(q * 32) << 16) + (acc + a) * BN,
                                 epi + (a * 4 + q) * C::kEpiStage,
                                 (kMode == 0 && NA == 1 && args.tma_store) ? &map_c : nullptr);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty + acc + a, 0);
    }
    // the TMA stores must be complete (and done reading the stages) before exit
    if (kMode == 0 && NA == 1 && args.tma_store && lane == 0)
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  } else if (warp == 3 && args.exch_kind == 1) {   // dispatch rows beside the tiles
    exch_push(*args.exch, args.exch_x, lane);
  } else if (GA && warp == 2) {
    if (lane == 0) {   // forwarder: this CTA's gathered stage -> the leader's full barrier
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cid; t < tm.total; t += ncl) {
        for (int kb = 0; kb < kblocks_fixed; ++kb) {
          mbar_wait(gfull + stage, phase);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          if (leader) {
            mbar_arrive(full + stage);
          } else {
            // relaxed: the stage's bytes live in THIS CTA's shared memory (the
            // cp.async completion observed above + the proxy fence make them
            // visible to this SM's tensor core); no cluster-wide release
            uint32_t remote;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                         : "=r"(remote) : "r"(smem_u32(full + stage)), "r"(0));
            asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];"
                         ::"r"(remote) : "memory");
          }
          if (++stage == ST) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (GA && warp >= 8 && warp < 12) {
    // A gather: this CTA's 128 rows x 8 16-byte chunks per stage; thread g owns
    // chunk g % 8 of rows g / 8 + 16 i (row pointers loaded once per tile)
    const int g_t = threadIdx.x - kThreads;
    const int c = g_t & 7, r0 = g_t >> 3;
    int stage = 0;
    uint32_t phase = 0;
    for (int t = cid; t < tm.total; t += ncl) {
      int g, mt, nt;
      tile_coords(tm, args.groups, t, g, mt, nt);
      const uint8_t* src[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = mt * BM2 + (int)rank * 128 + r0 + 16 * i;   // row within the group
        const int row = tm.row0[g] + (r < tm.rows[g] ? r : 0);
        const int v = args.a_idx[row];
        src[i] = (v >= 0 ? args.g_src + (int64_t)v * args.g_ld
                         : args.g_src2 + (int64_t)(~v) * args.g_ld) + c * 16;
      }
      for (int kb = 0; kb < kblocks_fixed; ++kb) {
        mbar_wait(empty + stage, phase ^ 1);
        const uint32_t base = smem_u32(sa + stage * kHalfBytes);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int r = r0 + 16 * i;
          cp_async16(base + r * 128 + ((c ^ (r & 7)) << 4), src[i] + kb * (BK * 2));
        }
        cp_async_arrive(gfull + stage);
        if (++stage == ST) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  }
  __syncthreads();
  cluster_sync_all();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(kTmemCols));
  }
}

// ---------------------------------------------------------------------------
// Weight gradients on CTA pairs (r2): out_g [m_out x N] = A_g^T B_g over group
// g's token rows, A [tokens, m_out] and B [tokens, N] token-major -- both
// MN-major tcgen05 operands (transpose bits), 256 x 256 output tiles, 64-token
// k-blocks.  CTA rank r stages output rows [r*128, +128) of A's tile and
// columns [r*128, +128) of B's (2 + 2 TMA boxes of 64 tokens x 64 features:
// 32 KB, the forward's per-CTA operand bytes per 8.4 MFLOP instead of the
// single-CTA kernel's 48 KB).  Whole k-blocks load straight onto the
// leader's full barrier (cta_group::2 TMA, as the forward); a group's last,
// partial k-block reaches into the next group's rows, so its loads land on
// each CTA's own gfull barrier and warp 2 zeroes those lines, fences and
// forwards the stage to the leader (relaxed cluster arrive).  Either way the
// leader's full barrier sees two arrivals per stage.
// GB: B's token rows are gathered by index (warps 8-11, cp.async) -- dW13 under
// the fused dispatch.
constexpr uint32_t kIdesc2MN = kIdesc2 | (1u << 15) | (1u << 16);
template <bool GB>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(GB ? kThreads + kGatherThreads : kThreads, 1)
    k_wgrad_pair(const __grid_constant__ CUtensorMap map_a,
                 const __grid_constant__ CUtensorMap map_b, GemmArgs args) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sa = smem;
  uint8_t* sb = smem + kStages2 * kHalfBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages2 * kStageBytes2);
  uint64_t* empty = full + kStages2;
  uint64_t* tfull = empty + kStages2;
  uint64_t* tempty = tfull + 2;
  uint64_t* gfull = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gfull + kStages2);
  uint8_t* epi = smem + kStages2 * kStageBytes2 + 256;
  __shared__ TileMap tm;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  if (threadIdx.x == 0) {
    int acc = 0, row = 0;
    tm.ntile_n = args.N / BN;
    for (int g = 0; g < args.groups; ++g) {
      const int n = args.n_rows[g];
      row = seg_row0(args, g, row);
      tm.start[g] = acc;
      tm.row0[g] = row;
      tm.rows[g] = n;
      tm.wsel[g] = g;
      acc += args.m_out / BM2 * tm.ntile_n;
      row += n;
    }
    tm.start[args.groups] = acc;
    tm.total = acc;
    for (int st = 0; st < kStages2; ++st) {
      mbar_init(full + st, 2);                            // one forwarder per CTA
      mbar_init(empty + st, 1);
      mbar_init(gfull + st, 1 + (GB ? kGatherThreads : 0));
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull + a, 1);
      mbar_init(tempty + a, 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {   // this CTA's boxes (A; B unless gathered) -> its own gfull
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cid; t < tm.total; t += ncl) {
        int g, mt, nt;
        tile_coords(tm, args.groups, t, g, mt, nt);
        const int arow = mt * BM2 + (int)rank * 128, bcol = nt * BN + (int)rank * 128;
        const int kblocks = (tm.rows[g] + BK - 1) / BK;
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(empty + stage, phase ^ 1);
          const int tok = tm.row0[g] + kb * BK;
          if (!GB && tm.rows[g] - kb * BK >= BK) {
            // a whole k-block: both CTAs' boxes complete on the leader's full
            // barrier (its expect_tx is one arrival, the peer's arrive the other)
            if (leader) {
              mbar_expect_tx(full + stage, 2 * kStageBytes2);
            } else {
              uint32_t remote;
              asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                           : "=r"(remote) : "r"(smem_u32(full + stage)), "r"(0));
              asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];"
                           ::"r"(remote) : "memory");
            }
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              tma_load_2d_pair(sa + stage * kHalfBytes + j * 8192, &map_a, full + stage,
                               arow + 64 * j, tok);
              tma_load_2d_pair(sb + stage * kHalfBytes + j * 8192, &map_b, full + stage,
                               bcol + 64 * j, tok);
            }
          } else {   // the tail block (or gathered B): own gfull, then the forwarder
            mbar_expect_tx(gfull + stage, GB ? kHalfBytes : 2 * kHalfBytes);
#pragma unroll
            for (int j = 0; j < 2; ++j)
              tma_load_2d(sa + stage * kHalfBytes + j * 8192, &map_a, gfull + stage,
                          arow + 64 * j, tok);
            if (!GB) {
#pragma unroll
              for (int j = 0; j < 2; ++j)
                tma_load_2d(sb + stage * kHalfBytes + j * 8192, &map_b, gfull + stage,
                            bcol + 64 * j, tok);
            }
          }
          if (++stage == kStages2) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 2) {
    // forwarder: tail lines zeroed, then the stage -> the leader's full barrier.
    // gfull[s] completes only when stage s carries a forwarded block, so its
    // parity is tracked per stage (bit s of gph), not by ring laps
    int stage = 0;
    uint32_t gph = 0;
    for (int t = cid; t < tm.total; t += ncl) {
      int g, mt, nt;
      tile_coords(tm, args.groups, t, g, mt, nt);
      const int kblocks = (tm.rows[g] + BK - 1) / BK;
      for (int kb = 0; kb < kblocks; ++kb) {
        const int valid = tm.rows[g] - kb * BK;
        if (!GB && valid >= BK) {   // went straight to the leader's barrier
          if (++stage == kStages2) stage = 0;
          continue;
        }
        mbar_wait(gfull + stage, (gph >> stage) & 1u);
        gph ^= 1u << stage;
        const int zend = valid >= BK ? BK : (valid + UK - 1) / UK * UK;
        if (valid < zend) {
          const int nlines = zend - valid;
          for (int i = lane; i < 4 * nlines * 8; i += 32) {
            const int box = i / (nlines * 8), rem = i % (nlines * 8);
            const int line = valid + rem / 8, chunk = rem % 8;
            uint8_t* base = box < 2 ? sa + stage * kHalfBytes + box * 8192
                                    : sb + stage * kHalfBytes + (box - 2) * 8192;
            *reinterpret_cast<int4*>(base + line * 128 + chunk * 16) = make_int4(0, 0, 0, 0);
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          if (leader) {
            mbar_arrive(full + stage);
          } else {
            uint32_t remote;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                         : "=r"(remote) : "r"(smem_u32(full + stage)), "r"(0));
            asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];"
                         ::"r"(remote) : "memory");
          }
        }
        __syncwarp();
        if (++stage == kStages2) stage = 0;
      }
    }
  } else if (warp == 1) {
    if (leader) {   // the whole warp runs the loop; one elected lane issues
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = cid; t < tm.total; t += ncl, ++it) {
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait(tempty + acc, acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + acc * BN;
        int g, mt, nt;
        tile_coords(tm, args.groups, t, g, mt, nt);
        const int rows = tm.rows[g];
        const int whole = rows / BK, kblocks = (rows + BK - 1) / BK;
        for (int kb = 0; kb < kblocks; ++kb) {
          // descriptors once per k-block, +128 (16 K lines) per k-step
          const uint64_t da = smem_desc_mn(smem_u32(sa + stage * kHalfBytes));
          const uint64_t db = smem_desc_mn(smem_u32(sb + stage * kHalfBytes));
          if (kb < whole) {   // TMA-only stage: the 4 k-steps unrolled
            mbar_wait(full + stage, phase);
            tc_fence_after();
#pragma unroll
            for (int k = 0; k < BK / UK; ++k)
              umma_bf16_pair_elect<kIdesc2MN>(d, da + 128 * k, db + 128 * k,
                                              (kb | k) ? 1u : 0u);
          } else {   // the forwarded tail block (zeroed lines: cluster acquire)
            mbar_wait_cluster(full + stage, phase);
            tc_fence_after();
            const int ksteps = (rows - kb * BK + UK - 1) / UK;
            for (int k = 0; k < ksteps; ++k)
              umma_bf16_pair_elect<kIdesc2MN>(d, da + 128 * k, db + 128 * k,
                                              (kb | k) ? 1u : 0u);
          }
          umma_commit_pair_elect(empty + stage);
          if (++stage == kStages2) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_pair_elect(tfull + acc);
      }
    }
  } else if (warp >= 4 && warp < 8) {
    const int q = warp - 4;
    int it = 0;
    for (int t = cid; t < tm.total; t += ncl, ++it) {
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      int g, mt, nt;
      tile_coords(tm, args.groups, t, g, mt, nt);
      mbar_wait(tfull + acc, acc_phase);
      tc_fence_after();
      store_tile<3>(args, tm, g, nt, mt * BM2 + (int)rank * 128 + q * 32, lane,
                    tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN, epi + q * kEpiStageBytes);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty + acc, 0);
    }
  } else if (GB && warp >= 8) {
    // B gather: 64 token lines x 2 feature boxes (this CTA's 128 columns) x 8
    // 16-byte chunks per stage; thread g owns chunk g % 8 of lines g / 8 + 16 i
    const int g_t = threadIdx.x - kThreads;
    const int c = g_t & 7, l0 = g_t >> 3;
    int stage = 0;
    uint32_t phase = 0;
    for (int t = cid; t < tm.total; t += ncl) {
      int g, mt, nt;
      tile_coords(tm, args.groups, t, g, mt, nt);
      const int kblocks = (tm.rows[g] + BK - 1) / BK;
      const int end = tm.row0[g] + tm.rows[g];
      const uint8_t* col = args.g_src + (int64_t)(nt * BN + (int)rank * 128 + 8 * c) * 2;
      auto load_tok = [&](int kb, int* tk) {
        const int r0 = tm.row0[g] + kb * BK + l0;
#pragma unroll
        for (int i = 0; i < 4; ++i) tk[i] = args.b_idx[r0 + 16 * i < end ? r0 + 16 * i : tm.row0[g]];
      };
      int nxt[4];
      if (kblocks > 0) load_tok(0, nxt);
      for (int kb = 0; kb < kblocks; ++kb) {
        int tok[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) tok[i] = nxt[i];
        if (kb + 1 < kblocks) load_tok(kb + 1, nxt);
        mbar_wait(empty + stage, phase ^ 1);
        const uint32_t base = smem_u32(sb + stage * kHalfBytes);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int l = l0 + 16 * i;
          const int v = tok[i];
          const uint8_t* src = v >= 0 ? col + (int64_t)v * args.g_ld
                                      : col + (args.g_src2 - args.g_src) + (int64_t)(~v) * args.g_ld;
          const uint32_t dl = base + l * 128 + ((c ^ (l & 7)) << 4);
#pragma unroll
          for (int j = 0; j < 2; ++j) cp_async16(dl + j * 8192, src + j * 128);
        }
        cp_async_arrive(gfull + stage);
        if (++stage == kStages2) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  }
  __syncthreads();
  cluster_sync_all();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(kTmemCols));
  }
}

// ---------------------------------------------------------------------------
// expert FFN backward helpers
// group layout for the weight-gradient GEMMs: token rows of group g are
// [row0_g, row0_g + n_g); as K columns they start at col0_g, padded to 64
// used rows per segment (segments of seg_groups groups; rows of segment s
// start at s * seg_rows): pre[0..segs] = prefix sums, the SwiGLU backward's
// flat row space
__global__ void k_group_layout(const int32_t* __restrict__ n_rows, int groups, int seg_groups,
                               int32_t* __restrict__ pre) {
  if (threadIdx.x || blockIdx.x) return;
  const int per = seg_groups > 0 ? seg_groups : groups;
  int run = 0;
  for (int g = 0; g < groups; ++g) {
    if (g % per == 0) pre[g / per] = run;
    run += n_rows[g];
  }
  pre[(groups + per - 1) / per] = run;
}

// SwiGLU backward on 128-column gate/up interleaved pre-activations:
// h = silu(a) u;  da = dh u silu'(a);  du = dh silu(a).
__global__ void __launch_bounds__(256) k_swiglu_bwd_v8(const __nv_bfloat16* __restrict__ g13,
                                                       const __nv_bfloat16* __restrict__ dh,
                                                       const int32_t* __restrict__ pre, int segs,
                                                       int64_t seg_rows, int inter,
                                                       __nv_bfloat16* __restrict__ dg13,
                                                       __nv_bfloat16* __restrict__ h) {
  const int rows = pre[segs];
  const int per_row = inter / 8;
  const int64_t n = (int64_t)rows * per_row;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int f = (int)(i / per_row);          // flat used row -> (segment, row)
    int sg = 0;
    while (sg + 1 < segs && pre[sg + 1] <= f) ++sg;
    const int64_t r = sg * seg_rows + (f - pre[sg]);
    const int j = 8 * (int)(i - (int64_t)f * per_row);
    const int b = j >> 7, c = j & 127;
    const int64_t ga = (int64_t)r * 2 * inter + 256 * b + c, gu = ga + 128;
    const int4 av = __ldg(reinterpret_cast<const int4*>(g13 + ga));
    const int4 uv = __ldg(reinterpret_cast<const int4*>(g13 + gu));
    const int4 dv = __ldg(reinterpret_cast<const int4*>(dh + (int64_t)r * inter + j));
    const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&av);
    const __nv_bfloat162* u2 = reinterpret_cast<const __nv_bfloat162*>(&uv);
    const __nv_bfloat162* d2 = reinterpret_cast<const __nv_bfloat162*>(&dv);
    int4 hv, dav, duv;
    __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&hv);
    __nv_bfloat162* da2 = reinterpret_cast<__nv_bfloat162*>(&dav);
    __nv_bfloat162* du2 = reinterpret_cast<__nv_bfloat162*>(&duv);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float2 a = __bfloat1622float2(a2[q]);
      const float2 u = __bfloat1622float2(u2[q]);
      const float2 d = __bfloat1622float2(d2[q]);
      const float s0 = 1.f / (1.f + __expf(-a.x)), s1 = 1.f / (1.f + __expf(-a.y));
      const float si0 = a.x * s0, si1 = a.y * s1;
      h2[q] = __floats2bfloat162_rn(si0 * u.x, si1 * u.y);
      du2[q] = __floats2bfloat162_rn(d.x * si0, d.y * si1);
      da2[q] = __floats2bfloat162_rn(d.x * u.x * s0 * (1.f + a.x * (1.f - s0)),
                                     d.y * u.y * s1 * (1.f + a.y * (1.f - s1)));
    }
    if (h) *reinterpret_cast<int4*>(h + (int64_t)r * inter + j) = hv;   // null: H kept
    *reinterpret_cast<int4*>(dg13 + gu) = duv;
    *reinterpret_cast<int4*>(dg13 + ga) = dav;
  }
}

// ---------------------------------------------------------------------------
// host: tensor maps through the driver entry point (no -lcuda link needed)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

int make_map(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return kInvalid;
  }
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {(cuuint32_t)BK, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
    return kInvalid;
  }
  return 0;
}

// token-major [rows][cols] bf16 activations as 64 x 64 boxes (64 features =
// one 128 B swizzled line per token) for the MN-major weight-gradient mode
int make_map_mn(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return kInvalid;
  }
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)BK};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
    return kInvalid;
  }
  return 0;
}

// out[g] ([m_out][N], ld_out) = A_g^T B_g over group g's token rows of
// A [a_rows][m_out] and B [a_rows][N] (kMode 3, MN-major operands straight
// from the token-major activations).  b_idx: B's token rows are gathered
// from b [b_src_rows][N] (fused dispatch)
int launch_gemm_wgrad(const void* a, const void* b, int64_t a_rows, int groups,
                      const int32_t* n_rows, int m_out, int N, void* out, int64_t ld_out,
                      cudaStream_t s, int accumulate = 0, const int32_t* b_idx = nullptr,
                      int64_t b_src_rows = 0, float* out_f32 = nullptr, int seg_groups = 0,
                      int64_t seg_rows = 0, const void* b_src2 = nullptr) {
  HM_CHECK_ARG(groups >= 1 && groups <= kMaxGroups, "wgrad gemm: 1..%d groups", kMaxGroups);
  HM_CHECK_ARG(m_out % BM == 0 && N % BN == 0, "wgrad gemm: m_out %% 128 == 0 and N %% 256 == 0");
  HM_CHECK_ARG(a_rows >= 1, "wgrad gemm: empty operands");
  HM_CHECK_ARG(!b_idx || b_src_rows >= 1, "wgrad gemm: gathered B needs its source rows");
  CUtensorMap ma, mb;
  int st = make_map_mn(&ma, a, (uint64_t)a_rows, (uint64_t)m_out);
  if (st) return st;
  st = make_map_mn(&mb, b, (uint64_t)(b_idx ? b_src_rows : a_rows), (uint64_t)N);
  if (st) return st;
  GemmArgs args;
  args.m_out = m_out;
  args.n_rows = n_rows;
  args.groups = groups;
  args.N = N;
  args.K = BK;
  args.swiglu = 0;
  args.out = reinterpret_cast<__nv_bfloat16*>(out);
  args.ld_out = ld_out;
  args.out2 = nullptr;
  args.accumulate = accumulate;
  args.status = nullptr;
  args.a_idx = nullptr;
  args.b_idx = b_idx;
  args.g_src = reinterpret_cast<const uint8_t*>(b);
  args.g_ld = (int64_t)N * 2;
  args.g_src2 = reinterpret_cast<const uint8_t*>(b_src2 ? b_src2 : b);
  args.outf = out_f32;
  args.n_valid = N;
  args.seg_groups = seg_groups;
  args.seg_rows = seg_rows;
  args.g_row0 = nullptr;
  args.g_wsel = nullptr;
  args.exch = nullptr;
  args.exch_kind = 0;
  args.exch_x = nullptr;
  const size_t smem = kStages * kStageBytes + 1024 + 256 + 4 * kEpiStageBytes;
  int dev = 0;
  HM_CUDA(cudaGetDevice(&dev));
  int sms = kSMs;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (g_gemm_ctas > 0 && g_gemm_ctas < sms) sms = g_gemm_ctas;
  if (g_wgrad_pair && m_out % BM2 == 0 && !out_f32 && sms >= 2) {
    // CTA pairs, 256 x 256 tiles (the expert weight gradients)
    const size_t smem2 = (size_t)kStages2 * kStageBytes2 + 1024 + 256 + 4 * kEpiStageBytes;
    if (b_idx) {
      HM_CUDA(cudaFuncSetAttribute(k_wgrad_pair<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem2));
      k_wgrad_pair<true><<<sms & ~1, kThreads + kGatherThreads, smem2, s>>>(ma, mb, args);
    } else {
      HM_CUDA(cudaFuncSetAttribute(k_wgrad_pair<false>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
      k_wgrad_pair<false><<<sms & ~1, kThreads, smem2, s>>>(ma, mb, args);
    }
    HM_LAUNCHED();
    return 0;
  }
  if (b_idx) {
    HM_CUDA(cudaFuncSetAttribute(k_grouped_gemm<3, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_grouped_gemm<3, true><<<sms, kThreads + kGatherThreads, smem, s>>>(ma, mb, args);
  } else {
    HM_CUDA(cudaFuncSetAttribute(k_grouped_gemm<3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    k_grouped_gemm<3><<<sms, kThreads, smem, s>>>(ma, mb, args);
  }
  HM_LAUNCHED();
  return 0;
}

// out[rows of group g] = A[rows of g] . B_g^T on CTA pairs (256 x 256 tiles).
// a_idx: the A rows are gathered from a [a_src_rows][K] by row index (fused
// dispatch); a_rows is then the layout's capacity
int launch_gemm(const void* a, int64_t a_rows, const void* b, int groups, const int32_t* n_rows,
                int N, int K, int swiglu, void* out, int64_t ld_out, int* status,
                cudaStream_t s, void* out2 = nullptr, const int32_t* a_idx = nullptr,
                int64_t a_src_rows = 0, float* out_f32 = nullptr, int n_valid = 0,
                int seg_groups = 0, int64_t seg_rows = 0, const void* a_src2 = nullptr,
                bool b_mn = false, const int32_t* g_row0 = nullptr,
                const int32_t* g_wsel = nullptr, int nweights = 0, int ctas = 0,
                const hm::ExchWork* exch = nullptr, int exch_kind = 0,
                const void* exch_x = nullptr, const void* add1 = nullptr,
                const void* add2 = nullptr) {
  HM_CHECK_ARG(groups >= 1 && groups <= kMaxGroups, "grouped gemm: 1..%d groups", kMaxGroups);
  HM_CHECK_ARG(N % BN == 0 && K % BK == 0, "grouped gemm: N %% 256 == 0 and K %% 64 == 0 required");
  HM_CHECK_ARG(a_rows >= 1, "grouped gemm: empty A");
  HM_CHECK_ARG(!a_idx || a_src_rows >= 1, "grouped gemm: gathered A needs its source rows");
  HM_CHECK_ARG(!out_f32 || (!swiglu && n_valid % 4 == 0 && ld_out % 4 == 0),
               "grouped gemm: fp32 output needs mode 0 and 16-byte rows / widths");
  CUtensorMap ma, mb;
  int st = make_map(&ma, a, (uint64_t)(a_idx ? a_src_rows : a_rows), (uint64_t)K, 128);
  if (st) return st;
  HM_CHECK_ARG(!g_row0 == !g_wsel && (!g_row0 || nweights >= 1),
               "grouped gemm: explicit groups need row starts, weight indices and the weight count");
  const uint64_t nw = g_wsel ? (uint64_t)nweights : (uint64_t)groups;
  st = b_mn ? make_map_mn(&mb, b, nw * K, (uint64_t)N) : make_map(&mb, b, nw * N, (uint64_t)K, 128);
  if (st) return st;
  HM_CHECK_ARG(!b_mn || (!a_idx && !swiglu), "grouped gemm: MN-major B only for mode 0");
  GemmArgs args;
  args.m_out = 0;
  args.n_rows = n_rows;
  args.groups = groups;
  args.N = N;
  args.K = K;
  args.swiglu = swiglu;
  args.out = reinterpret_cast<__nv_bfloat16*>(out);
  args.ld_out = ld_out;
  args.out2 = reinterpret_cast<__nv_bfloat16*>(out2);
  args.accumulate = 0;
  args.status = status;
  args.a_idx = a_idx;
  args.b_idx = nullptr;
  args.g_src = reinterpret_cast<const uint8_t*>(a);
  args.g_ld = (int64_t)K * 2;
  args.g_src2 = reinterpret_cast<const uint8_t*>(a_src2 ? a_src2 : a);
  args.outf = out_f32;
  args.n_valid = n_valid > 0 ? n_valid : N;
  args.seg_groups = seg_groups;
  args.seg_rows = seg_rows;
  args.g_row0 = g_row0;
  args.g_wsel = g_wsel;
  HM_CHECK_ARG(!exch_kind || (exch_kind == 1 && exch && exch_x),
               "grouped gemm: exchange work needs its descriptor and rows");
  args.exch = exch;
  args.exch_kind = exch_kind;
  args.exch_x = reinterpret_cast<const int4*>(exch_x);
  HM_CHECK_ARG(!add1 || (!swiglu && !out_f32 && out), "grouped gemm: addends need bf16 mode 0");
  HM_CHECK_ARG(!add2 || add1, "grouped gemm: the second addend needs the first");
  args.add1 = reinterpret_cast<const __nv_bfloat16*>(add1);
  args.add2 = reinterpret_cast<const __nv_bfloat16*>(add2);
  int dev = 0;
  HM_CUDA(cudaGetDevice(&dev));
  int sms = kSMs;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (g_gemm_ctas > 0 && g_gemm_ctas < sms) sms = g_gemm_ctas;
  if (ctas > 0 && ctas < sms) sms = ctas;
  HM_CHECK_ARG(sms >= 2, "grouped gemm: at least one CTA pair");
  const int grid = sms & ~1;
  // TMA tensor stores of the output (mode 0, bf16 rows of exactly N columns)
  CUtensorMap mc = ma;
  if (g_tma_store && !swiglu && !out_f32 && out && ld_out == N && N % 64 == 0) {
    if (make_map(&mc, out, (uint64_t)a_rows, (uint64_t)N, 32) == 0) args.tma_store = 1;
  }
  auto run = [&](auto kern, int threads, size_t smem2) -> int {
    HM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
    kern<<<grid, threads, smem2, s>>>(ma, mb, mc, args);
    return launch_status();
  };
  const int thr_g = kThreads + kGatherThreads;   // + the A-gather warps
  // 256 x 512 tiles (hm_ffn_set_option(5, .)): the data-gradient GEMMs over a
  // long K (DeepSeek-V3's dH / gX: -11..-16 %); the forward GEMMs and short-K
  // ones measured faster on double-buffered 256 x 256 tiles, whose epilogue
  // hides entirely behind the next tile's k-loop
  const bool wide = g_wide_tiles == 2 || (g_wide_tiles == 1 && b_mn && K >= 4096);
  if (wide && N % (2 * BN) == 0 && !out_f32) {
    const size_t sm = PairCfg<2>::smem();
    const int e2 = kEpi2Threads;   // + the accumulator-1 epilogue warpgroup
    if (b_mn) return run(k_grouped_gemm_pair<0, false, true, 2>, kThreads + e2, sm);
    if (a_idx) return swiglu ? run(k_grouped_gemm_pair<1, true, false, 2>, thr_g + e2, sm)
                             : run(k_grouped_gemm_pair<0, true, false, 2>, thr_g + e2, sm);
    return swiglu ? run(k_grouped_gemm_pair<1, false, false, 2>, kThreads + e2, sm)
                  : run(k_grouped_gemm_pair<0, false, false, 2>, kThreads + e2, sm);
  }
  const size_t sm = PairCfg<1>::smem();
  if (b_mn) return run(k_grouped_gemm_pair<0, false, true>, kThreads, sm);
  if (a_idx) return swiglu ? run(k_grouped_gemm_pair<1, true>, thr_g, sm)
                           : run(k_grouped_gemm_pair<0, true>, thr_g, sm);
  return swiglu ? run(k_grouped_gemm_pair<1>, kThreads, sm)
                : run(k_grouped_gemm_pair<0>, kThreads, sm);
}

}  // namespace

// FFN options (no reference counterpart): 1 = cap on the persistent GEMM grid
// (CTAs; 0 = one per SM, default) so concurrent exchange kernels keep SMs of
// their own; 2 = CTA-pair weight gradients (default 1; 0 = the single-CTA
// kernel, kept as the bit-exactness reference of the pair kernel's tests);
// 5 = 256 x 512 pair tiles: 0 never (the wide kernel's bit-exactness
// reference), 1 (default) for the long-K MN-major data gradients, 2 wherever
// N % 512 == 0.
// Options 0, 3 and 4 selected measured-slower variants (transposed K-major
// weight gradients, single-CTA forward GEMMs, 4-byte SwiGLU backward) that
// round 2 removed; they are rejected.
HM_API int hm_ffn_set_option(int32_t option, int32_t value) {
  HM_CHECK_ARG(option == 1 || option == 2 || option == 5 || option == 6,
               "hm_ffn_set_option: unknown option %d", option);
  if (option == 6) g_tma_store = value != 0;
  if (option == 1) g_gemm_ctas = value > 0 ? value : 0;
  if (option == 2) g_wgrad_pair = value != 0;
  if (option == 5) g_wide_tiles = value < 0 ? 0 : (value > 2 ? 2 : value);
  return 0;
}

// Grouped GEMM: out[rows of group g] = A[rows of g] . B_g^T (bf16 in, fp32
// accumulate, bf16 out); groups are consecutive row blocks of A with sizes
// n_rows[g] (device).  swiglu=1 applies silu(gate)*up to 128-column gate/up
// block pairs (out has N/2 columns).
HM_API int hm_grouped_gemm(const void* a, int64_t a_rows, const void* b, int32_t groups,
                           const int32_t* n_rows, int32_t N, int32_t K, int32_t swiglu, void* out,
                           int64_t ld_out, void* stream) {
  HM_RANGE("hm_grouped_gemm");
  return launch_gemm(a, a_rows, b, groups, n_rows, N, K, swiglu, out, ld_out, nullptr,
                     (cudaStream_t)stream);
}

// ... with B given as stored [groups][K][N] (N contiguous): out = A . B_g,
// read MN-major by the tensor cores (no transposed copy of B)
HM_API int hm_grouped_gemm_kn(const void* a, int64_t a_rows, const void* b, int32_t groups,
                              const int32_t* n_rows, int32_t N, int32_t K, void* out,
                              int64_t ld_out, void* stream) {
  HM_RANGE("hm_grouped_gemm_kn");
  return launch_gemm(a, a_rows, b, groups, n_rows, N, K, 0, out, ld_out, nullptr,
                     (cudaStream_t)stream, nullptr, nullptr, 0, nullptr, 0, 0, 0, nullptr, true);
}

// Router GEMMs on the same tcgen05 kernels, fp32 results:
//   hm_gemm_f32: out[rows, ld] (fp32, first n_valid columns) = A[rows, K] . B^T,
//     B [N][K] bf16 K-major (N a multiple of 256: pad the expert dimension with
//     zero rows); rows_dev = device int32 {rows}.  Router logits = x . Wr^T
//     (bf16 operands, fp32 accumulation; no fp32 copy of x), and the router
//     data gradient dX = dlogits . Wr (B = Wr^T [M][E]).
//   hm_wgrad_f32: out[m_out][N] (fp32, += if accumulate) = A^T . B over rows
//     A [rows, m_out], B [rows, N] token-major (MN-major tcgen05 operands):
//     the router weight gradient dWr = dlogits^T . x.
HM_API int hm_gemm_f32(const void* a, int64_t rows, const int32_t* rows_dev, const void* b,
                       int32_t N, int32_t K, int32_t n_valid, float* out, int64_t ld_out,
                       void* stream) {
  HM_RANGE("hm_gemm_f32");
  HM_CHECK_ARG(a && b && out && rows_dev, "hm_gemm_f32: null argument");
  HM_CHECK_ARG(n_valid > 0 && n_valid <= N, "hm_gemm_f32: 0 < n_valid <= N");
  return launch_gemm(a, rows > 0 ? rows : 1, b, 1, rows_dev, N, K, 0, nullptr, ld_out, nullptr,
                     (cudaStream_t)stream, nullptr, nullptr, 0, out, n_valid);
}

// Split-K for the router weight gradient: its output is only m_out x N (8
// tiles of 128 x 256 for 128 experts x hidden 2048), so one group would keep
// 8 of 148 SMs busy over all T tokens.  The token range is cut into S chunks
// (device-side sizes from the device row count), each chunk a mode-3 group
// with its own fp32 partial [m_out][N] in the caller's scratch, and the
// partials are summed (+ the accumulated gradient) by k_sum_splits.
namespace {
__global__ void k_split_rows(const int32_t* __restrict__ total, int S, int chunk,
                             int32_t* __restrict__ n_rows) {
  const int s = threadIdx.x;
  if (s < S) {
    const int r = *total - s * chunk;
    n_rows[s] = r < 0 ? 0 : (r > chunk ? chunk : r);
  }
}
__global__ void __launch_bounds__(256) k_sum_splits(const float4* __restrict__ part, int S,
                                                    int m_out, int N, float* __restrict__ out,
                                                    int64_t ld_out, int accumulate) {
  const int n4 = N / 4;
  const int64_t total = (int64_t)m_out * n4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / n4, c = (i % n4) * 4;
    float4* o = reinterpret_cast<float4*>(out + r * ld_out + c);
    float4 acc = accumulate ? *o : make_float4(0.f, 0.f, 0.f, 0.f);
    for (int sp = 0; sp < S; ++sp) {
      const float4 v = part[sp * total + i];
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    *o = acc;
  }
}
// chunks of the split: ~one per 8-tile output per SM, >= 4 k-blocks each
int wgrad_splits(int64_t rows, int m_out, int N) {
  int dev = 0, sms = kSMs;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int tiles = (m_out / BM) * (N / BN);
  int S = tiles > 0 ? sms / tiles : 1;
  S = S > 64 ? 64 : S;
  if ((int64_t)S * 4 * BK > rows) S = (int)(rows / (4 * BK));
  return S < 1 ? 1 : S;
}
}  // namespace

// out[rows][ld] bf16 = bf16((A . B^T + add1) + add2), fp32 sums, add2 optional:
// the router's input gradient dlogits . Wr fused with the routed / shared-expert
// input gradients (replaces hm_gemm_f32 + hm_sum_to_bf16, bit-identical)
HM_API int hm_gemm_add_bf16(const void* a, int64_t rows, const int32_t* rows_dev, const void* b,
                            int32_t N, int32_t K, const void* add1, const void* add2, void* out,
                            int64_t ld_out, void* stream) {
  HM_RANGE("hm_gemm_add_bf16");
  HM_CHECK_ARG(a && b && out && rows_dev && add1, "hm_gemm_add_bf16: null argument");
  return launch_gemm(a, rows > 0 ? rows : 1, b, 1, rows_dev, N, K, 0, out, ld_out, nullptr,
                     (cudaStream_t)stream, nullptr, nullptr, 0, nullptr, 0, 0, 0, nullptr, false,
                     nullptr, nullptr, 0, 0, nullptr, 0, nullptr, add1, add2);
}

HM_API int64_t hm_wgrad_f32_scratch_bytes(int64_t rows, int32_t m_out, int32_t N) {
  const int S = wgrad_splits(rows > 0 ? rows : 1, m_out, N);
  return S < 2 ? 0 : 256 + (int64_t)S * m_out * N * 4;
}

HM_API int hm_wgrad_f32(const void* a, const void* b, int64_t rows, const int32_t* rows_dev,
                        int32_t m_out, int32_t N, float* out, int64_t ld_out, int32_t accumulate,
                        void* stream) {
  HM_RANGE("hm_wgrad_f32");
  HM_CHECK_ARG(a && b && out && rows_dev, "hm_wgrad_f32: null argument");
  return launch_gemm_wgrad(a, b, rows > 0 ? rows : 1, 1, rows_dev, m_out, N, nullptr, ld_out,
                           (cudaStream_t)stream, accumulate, nullptr, 0, out);
}

HM_API int hm_wgrad_f32_split(const void* a, const void* b, int64_t rows,
                              const int32_t* rows_dev, int32_t m_out, int32_t N, float* out,
                              int64_t ld_out, int32_t accumulate, void* scratch,
                              int64_t scratch_bytes, void* stream) {
  HM_RANGE("hm_wgrad_f32_split");
  HM_CHECK_ARG(a && b && out && rows_dev, "hm_wgrad_f32_split: null argument");
  HM_CHECK_ARG(m_out % BM == 0 && N % BN == 0 && ld_out % 4 == 0,
               "hm_wgrad_f32_split: m_out %% 128 == 0, N %% 256 == 0, 16-byte output rows");
  cudaStream_t s = (cudaStream_t)stream;
  rows = rows > 0 ? rows : 1;
  const int S = wgrad_splits(rows, m_out, N);
  const int64_t need = S < 2 ? 0 : 256 + (int64_t)S * m_out * N * 4;
  if (S < 2)
    return launch_gemm_wgrad(a, b, rows, 1, rows_dev, m_out, N, nullptr, ld_out, s, accumulate,
                             nullptr, 0, out);
  HM_CHECK_ARG(scratch && scratch_bytes >= need,
               "hm_wgrad_f32_split: scratch of hm_wgrad_f32_scratch_bytes() bytes required");
  int32_t* n_rows = reinterpret_cast<int32_t*>(scratch);   // 64 counts in the first 256 B
  float* part = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(scratch) + 256);
  const int chunk = (int)((rows + S - 1) / S + BK - 1) / BK * BK;
  k_split_rows<<<1, 64, 0, s>>>(rows_dev, S, chunk, n_rows);
  HM_LAUNCHED();
  int st = launch_gemm_wgrad(a, b, rows, S, n_rows, m_out, N, nullptr, N, s, 0, nullptr, 0, part);
  if (st) return st;
  int dev = 0, sms = kSMs;
  HM_CUDA(cudaGetDevice(&dev));
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t n4 = (int64_t)m_out * N / 4;
  const int grid = (int)((n4 + 255) / 256 < 4 * sms ? (n4 + 255) / 256 : 4 * sms);
  k_sum_splits<<<grid, 256, 0, s>>>(reinterpret_cast<const float4*>(part), S, m_out, N, out,
                                    ld_out, accumulate);
  HM_LAUNCHED();
  return 0;
}

// Expert SwiGLU FFN on expert-major rows: H = silu(X W1^T) * (X W3^T),
// Y = H W2^T.  w13: [groups][2I][M] (128-row gate/up blocks interleaved),
// w2: [groups][M][I], h: [a_rows][I], y: [a_rows][M].
HM_API int hm_expert_ffn(const void* x, int64_t a_rows, const int32_t* n_rows, int32_t groups,
                         const void* w13, const void* w2, int32_t hidden, int32_t inter, void* h,
                         void* y, void* stream) {
  HM_RANGE("hm_expert_ffn");
  int st = launch_gemm(x, a_rows, w13, groups, n_rows, 2 * inter, hidden, 1, h, inter, nullptr,
                       (cudaStream_t)stream);
  if (st) return st;
  return launch_gemm(h, a_rows, w2, groups, n_rows, hidden, inter, 0, y, hidden, nullptr,
                     (cudaStream_t)stream);
}

// ... training forward: GEMM1's epilogue also stores the gate/up
// pre-activations g13 [a_rows][2I] so the backward needs no recompute
HM_API int hm_expert_ffn_save(const void* x, int64_t a_rows, const int32_t* n_rows,
                              int32_t groups, const void* w13, const void* w2, int32_t hidden,
                              int32_t inter, void* h, void* y, void* g13, void* stream) {
  HM_RANGE("hm_expert_ffn_save");
  HM_CHECK_ARG(g13, "hm_expert_ffn_save: null g13");
  int st = launch_gemm(x, a_rows, w13, groups, n_rows, 2 * inter, hidden, 1, h, inter, nullptr,
                       (cudaStream_t)stream, g13);
  if (st) return st;
  return launch_gemm(h, a_rows, w2, groups, n_rows, hidden, inter, 0, y, hidden, nullptr,
                     (cudaStream_t)stream);
}

// Expert SwiGLU FFN backward (tcgen05 GEMMs + SwiGLU backward):
//   G13 = X W13^T (recomputed pre-activations unless saved), dH = gY W2,
//   dG13 = swiglu'(G13, dH), H = swiglu(G13), gX = dG13 W13 (both data-gradient
//   GEMMs read the weights as stored, MN-major: no transposed copies),
//   dW2 = gY^T H, dW13 = dG13^T X (weight-gradient GEMMs over each expert's own
//   token rows, MN-major operands; x_idx: X's rows gathered).
// Buffers (rows = a_rows capacity): g13, dg13 [rows, 2I]; dh, h [rows, I];
// layout: 2*(groups+1) int32 scratch.  Outputs: gx [rows, M],
// dw13 [groups][2I][M], dw2 [groups][M][I] (accumulate: added to).
static int ffn_backward(const void* x, int64_t a_rows, const int32_t* n_rows, int32_t groups,
                        const void* w13, const void* w2, const void* gy,
                        int32_t hidden, int32_t inter, void* g13, int g13_saved, void* dh,
                        void* dg13, void* h, int32_t* layout, void* gx, void* dw13, void* dw2,
                        void* stream, int accumulate = 0, const int32_t* x_idx = nullptr,
                        int64_t x_rows = 0, int seg_groups = 0, int64_t seg_rows = 0,
                        const void* x_recv = nullptr, int parts = 3) {
  cudaStream_t s = (cudaStream_t)stream;
  HM_CHECK_ARG(!x_idx || g13_saved,
               "ffn backward: gathered activations need the saved pre-activations");
  // parts bit 4: h already holds the forward's H (GEMM1's epilogue output),
  // so the SwiGLU backward does not rewrite it and dW2 uses the very H that
  // produced the forward's Y
  const bool h_fwd = (parts & 4) != 0;
  parts &= 3;
  HM_CHECK_ARG(parts >= 1 && parts <= 3, "ffn backward: parts must be 1, 2 or 3 (+4)");
  const int M = hidden, I = inter;
  int st;
  const int sg = seg_groups, segs = sg > 0 ? (groups + sg - 1) / sg : 1;
  if (parts & 1) {
  // gate/up pre-activations (recomputed unless the forward saved them), then dH
  if (!g13_saved && (st = launch_gemm(x, a_rows, w13, groups, n_rows, 2 * I, M, 0, g13, 2 * I,
                                      nullptr, s, nullptr, nullptr, 0, nullptr, 0, sg, seg_rows)))
    return st;
  // dH = gY W2: W2 [g][M][I] as stored = B [K = M][N = I], read MN-major
  // (the SwiGLU backward stays a separate HBM-rate kernel: folded into this
  // GEMM's epilogue it made the epilogue the bottleneck, Qwen3 rank backward
  // 0.543 -> 0.590 ms; profiles/r02/negative/swiglu_bwd_in_dh_epilogue_ab.jsonl)
  if ((st = launch_gemm(gy, a_rows, w2, groups, n_rows, I, M, 0, dh, I, nullptr, s, nullptr,
                        nullptr, 0, nullptr, 0, sg, seg_rows, nullptr, true)))
    return st;
  k_group_layout<<<1, 32, 0, s>>>(n_rows, groups, sg, layout);
  HM_LAUNCHED();
  HM_CHECK_ARG(I % 128 == 0, "ffn backward: inter must be a multiple of 128");
  k_swiglu_bwd_v8<<<kSMs * 8, 256, 0, s>>>((const __nv_bfloat16*)g13, (const __nv_bfloat16*)dh,
                                            layout, segs, sg > 0 ? seg_rows : 0, I,
                                            (__nv_bfloat16*)dg13, h_fwd ? nullptr : (__nv_bfloat16*)h);
  HM_LAUNCHED();
  // data gradient gX = dG13 W13: W13 [g][2I][M] as stored = B [K = 2I][N = M]
  if ((st = launch_gemm(dg13, a_rows, w13, groups, n_rows, M, 2 * I, 0, gx, M, nullptr, s,
                        nullptr, nullptr, 0, nullptr, 0, sg, seg_rows, nullptr, true)))
    return st;
  }
  if (!(parts & 2)) return 0;
  // weight gradients straight from the token-major activations (MN-major
  // tcgen05 operands), reduction over each expert's own rows (dg13 and h from
  // part 1, kept in the scratch buffers)
  if ((st = launch_gemm_wgrad(gy, h, a_rows, groups, n_rows, M, I, dw2, I, s, accumulate, nullptr,
                              0, nullptr, sg, seg_rows)))
    return st;
  return launch_gemm_wgrad(dg13, x, a_rows, groups, n_rows, 2 * I, M, dw13, M, s, accumulate,
                           x_idx, x_rows, nullptr, sg, seg_rows, x_recv);
}

HM_API int hm_expert_ffn_backward(const void* x, int64_t a_rows, const int32_t* n_rows,
                                  int32_t groups, const void* w13, const void* w2, const void* gy,
                                  int32_t hidden, int32_t inter, void* g13, void* dh, void* dg13,
                                  void* h, int32_t* layout, void* gx, void* dw13, void* dw2,
                                  void* stream) {
  HM_RANGE("hm_expert_ffn_backward");
  return ffn_backward(x, a_rows, n_rows, groups, w13, w2, gy, hidden, inter, g13, 0, dh, dg13, h,
                      layout, gx, dw13, dw2, stream);
}

// ... with g13 holding the forward's pre-activations (hm_expert_ffn_save): no
// GEMM1 recompute; accumulate != 0 adds the weight grads to dw13 / dw2
// (micro-batched layers: one call per micro-batch)
HM_API int hm_expert_ffn_backward_saved(const void* x, int64_t a_rows, const int32_t* n_rows,
                                        int32_t groups, const void* w13, const void* w2,
                                        const void* gy, int32_t hidden, int32_t inter,
                                        const void* g13, void* dh, void* dg13, void* h,
                                        int32_t* layout, void* gx, void* dw13, void* dw2,
                                        int32_t accumulate, void* stream) {
  HM_RANGE("hm_expert_ffn_backward_saved");
  return ffn_backward(x, a_rows, n_rows, groups, w13, w2, gy, hidden, inter,
                      const_cast<void*>(g13), 1, dh, dg13, h, layout, gx, dw13, dw2, stream,
                      accumulate);
}

// Fused dispatch: the expert-major rows are never materialised -- row r of
// the expert-major layout (capacity a_rows, groups of n_rows[g]) is source
// row idx[r] of x [x_rows][hidden] (the tokens themselves), loaded by GEMM1's
// A-gather warps.  g13 (optional) keeps the pre-activations for the backward.
HM_API int hm_expert_ffn_gather(const void* x, int64_t x_rows, const int32_t* idx, int64_t a_rows,
                                const int32_t* n_rows, int32_t groups, const void* w13,
                                const void* w2, int32_t hidden, int32_t inter, void* h, void* y,
                                void* g13, void* stream) {
  HM_RANGE("hm_expert_ffn_gather");
  HM_CHECK_ARG(x && idx, "hm_expert_ffn_gather: null argument");
  int st = launch_gemm(x, a_rows, w13, groups, n_rows, 2 * inter, hidden, 1, h, inter, nullptr,
                       (cudaStream_t)stream, g13, idx, x_rows);
  if (st) return st;
  return launch_gemm(h, a_rows, w2, groups, n_rows, hidden, inter, 0, y, hidden, nullptr,
                     (cudaStream_t)stream);
}

// ... its backward (saved pre-activations): dW13's token operand is gathered
// from x by the same row indices; accumulate adds the weight grads
HM_API int hm_expert_ffn_backward_gather(const void* x, int64_t x_rows, const int32_t* idx,
                                         int64_t a_rows, const int32_t* n_rows, int32_t groups,
                                         const void* w13, const void* w2, const void* gy,
                                         int32_t hidden, int32_t inter, const void* g13, void* dh,
                                         void* dg13, void* h, int32_t* layout, void* gx,
                                         void* dw13, void* dw2, int32_t accumulate, void* stream) {
  HM_RANGE("hm_expert_ffn_backward_gather");
  HM_CHECK_ARG(x && idx, "hm_expert_ffn_backward_gather: null argument");
  return ffn_backward(x, a_rows, n_rows, groups, w13, w2, gy, hidden, inter,
                      const_cast<void*>(g13), 1, dh, dg13, h, layout, gx, dw13, dw2, stream,
                      accumulate, idx, x_rows);
}

// Several EP ranks' expert FFNs in ONE launch per GEMM (a GPU hosting L ranks):
// segment s = rank s's groups [s * groups_per_seg, (s + 1) * groups_per_seg)
// with its expert-major rows at [s * seg_rows, ...) of every row buffer
// (x / idx / h / y / g13 / gy / gx / dh / dg13: [segs][seg_rows][...]),
// weights [segs * groups_per_seg][...] contiguous.  One grid over all tiles
// instead of L launches: no per-rank fill / drain and one wave tail.  idx
// null: x holds the materialised expert-major rows; otherwise row r of the
// layout is x row idx[r] (fused dispatch), or -- idx < 0 -- row ~idx[r] of
// x_recv (the rows received over NVLink; fused dispatch at N > 1).
HM_API int hm_expert_ffn_multi(const void* x, int64_t x_rows, const int32_t* idx,
                               const void* x_recv, int64_t seg_rows, int32_t segs,
                               const int32_t* n_rows,
                               int32_t groups_per_seg, const void* w13, const void* w2,
                               int32_t hidden, int32_t inter, void* h, void* y, void* g13,
                               void* stream) {
  HM_RANGE("hm_expert_ffn_multi");
  HM_CHECK_ARG(x && segs >= 1 && groups_per_seg >= 1 && seg_rows >= 1,
               "hm_expert_ffn_multi: bad argument");
  const int groups = segs * groups_per_seg;
  const int64_t rows = (int64_t)segs * seg_rows;
  int st = launch_gemm(x, rows, w13, groups, n_rows, 2 * inter, hidden, 1, h, inter, nullptr,
                       (cudaStream_t)stream, g13, idx, idx ? x_rows : 0, nullptr, 0,
                       groups_per_seg, seg_rows, x_recv);
  if (st) return st;
  return launch_gemm(h, rows, w2, groups, n_rows, hidden, inter, 0, y, hidden, nullptr,
                     (cudaStream_t)stream, nullptr, nullptr, 0, nullptr, 0, groups_per_seg,
                     seg_rows);
}

// ... over explicit row groups: group g = rows [g_row0[g], g_row0[g] + g_rows[g])
// of the [rows] row space (x / idx / h / y / g13 as in hm_expert_ffn_multi),
// multiplied by expert weight g_wsel[g] of w13 / w2 ([nweights][...]); ctas > 0
// caps the grid (an exchange kernel running beside it keeps its SMs).  The
// overlapped forward runs the rows already on this GPU while the rest cross
// NVLink, then the received rows; per-row results equal the one-launch FFN's.
HM_API int hm_expert_ffn_groups(const void* x, int64_t x_rows, const int32_t* idx,
                                const void* x_recv, int64_t rows, int32_t groups,
                                const int32_t* g_row0, const int32_t* g_rows,
                                const int32_t* g_wsel, int32_t nweights, const void* w13,
                                const void* w2, int32_t hidden, int32_t inter, void* h, void* y,
                                void* g13, int32_t ctas, void* stream) {
  HM_RANGE("hm_expert_ffn_groups");
  HM_CHECK_ARG(x && g_row0 && g_rows && g_wsel && rows >= 1 && nweights >= 1,
               "hm_expert_ffn_groups: bad argument");
  int st = launch_gemm(x, rows, w13, groups, g_rows, 2 * inter, hidden, 1, h, inter, nullptr,
                       (cudaStream_t)stream, g13, idx, idx ? x_rows : 0, nullptr, 0, 0, 0, x_recv,
                       false, g_row0, g_wsel, nweights, ctas);
  if (st) return st;
  return launch_gemm(h, rows, w2, groups, g_rows, hidden, inter, 0, y, hidden, nullptr,
                     (cudaStream_t)stream, nullptr, nullptr, 0, nullptr, 0, 0, 0, nullptr, false,
                     g_row0, g_wsel, nweights, ctas);
}

int hm::ffn_gemm_groups(const void* a, int64_t rows, const void* b, int groups,
                        const int32_t* g_rows, const int32_t* g_row0, const int32_t* g_wsel,
                        int nweights, int N, int K, int swiglu, void* out, int64_t ld_out,
                        void* out2, const int32_t* a_idx, int64_t a_src_rows, const void* a_src2,
                        const hm::ExchWork* exch, int exch_kind, const void* exch_x,
                        cudaStream_t s) {
  return launch_gemm(a, rows, b, groups, g_rows, N, K, swiglu, out, ld_out, nullptr, s, out2,
                     a_idx, a_src_rows, nullptr, 0, 0, 0, a_src2, false, g_row0, g_wsel,
                     nweights, 0, exch, exch_kind, exch_x);
}

int hm::ffn_gemm_segments(const void* a, int64_t rows, const void* b, int groups,
                          const int32_t* n_rows, int N, int K, void* out, int64_t ld_out,
                          int seg_groups, int64_t seg_rows, cudaStream_t s) {
  return launch_gemm(a, rows, b, groups, n_rows, N, K, 0, out, ld_out, nullptr, s, nullptr,
                     nullptr, 0, nullptr, 0, seg_groups, seg_rows);
}

HM_API int hm_expert_ffn_backward_multi(const void* x, int64_t x_rows, const int32_t* idx,
                                        const void* x_recv, int64_t seg_rows, int32_t segs,
                                        const int32_t* n_rows,
                                        int32_t groups_per_seg, const void* w13, const void* w2,
                                        const void* gy, int32_t hidden, int32_t inter,
                                        const void* g13, void* dh, void* dg13, void* h,
                                        int32_t* layout, void* gx, void* dw13, void* dw2,
                                        int32_t accumulate, int32_t parts, void* stream) {
  HM_RANGE("hm_expert_ffn_backward_multi");
  HM_CHECK_ARG(x && g13 && segs >= 1 && groups_per_seg >= 1 && seg_rows >= 1,
               "hm_expert_ffn_backward_multi: bad argument");
  return ffn_backward(x, (int64_t)segs * seg_rows, n_rows, segs * groups_per_seg, w13, w2, gy,
                      hidden, inter, const_cast<void*>(g13), 1, dh, dg13, h, layout, gx,
                      dw13, dw2, stream, accumulate, idx, idx ? x_rows : 0, groups_per_seg,
                      seg_rows, x_recv, parts);
}
