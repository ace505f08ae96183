// Exchange work carried by the expert GEMM (fused compute + NVLink transfer).
// A GEMM launch with an ExchWork runs it in warp 3 of every CTA -- a warp the
// warp-specialised tile pipeline leaves idle -- while the tensor cores work on
// the rows already on this GPU: each token row goes once to every other GPU
// its picks hit, straight into that GPU's receive buffer (the per-GPU dedup
// rows of hm_dispatch mode 3; positions and metadata were written
// beforehand by hm_dispatch_meta).  The pointer tables are fixed per EP world,
// so the struct is built once and lives in device memory.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace hm {

constexpr int kExchMaxGpus = 16;

struct ExchWork {
  int P, p, G, K, T_r;
  int64_t nvec;                       // 16-byte vectors per row
  int64_t ntok;                       // tokens on this GPU (L * T_r)
  int64_t rg_cap;                     // receive-buffer rows per GPU
  const int32_t* gpos_g;              // [ntok][P] GPU-level row of (token, GPU) or -1
  int4* recv_g[kExchMaxGpus];         // each GPU's receive buffer (peer mappings)
};

// expert FFN GEMM over explicit row groups (gemm_sm100.cu); exch_kind 1 runs
// exch's dispatch beside the tiles (exch_x: the token rows), 0 none
int ffn_gemm_groups(const void* a, int64_t rows, const void* b, int groups,
                    const int32_t* g_rows, const int32_t* g_row0, const int32_t* g_wsel,
                    int nweights, int N, int K, int swiglu, void* out, int64_t ld_out, void* out2,
                    const int32_t* a_idx, int64_t a_src_rows, const void* a_src2,
                    const ExchWork* exch, int exch_kind, const void* exch_x, cudaStream_t s);
// ... over the [segs][seg_rows] segment layout (hm_expert_ffn_multi), mode 0
int ffn_gemm_segments(const void* a, int64_t rows, const void* b, int groups,
                      const int32_t* n_rows, int N, int K, void* out, int64_t ld_out,
                      int seg_groups, int64_t seg_rows, cudaStream_t s);

}  // namespace hm
