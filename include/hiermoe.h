/*
 * libhiermoe -- C-ABI of the B200 (sm_100a) HierMoE dedup dispatch/combine +
 * expert-swap hot path.  Plain pointers and sizes only; every device pointer
 * is caller-owned (torch allocations) unless it comes from an hm_world.
 * Every call is stream-ordered on `stream` (a cudaStream_t) and returns
 *   0  ok,  < 0  invalid argument (message: hm_last_error()),  > 0  CUDA error.
 * Reentrant; the only state lives in hm_world objects created explicitly.
 *
 * Each entry point names the reference interface it replaces
 * (/root/reference/pkg/src/hiera2a/<file>:<line>).
 */
#ifndef HIERMOE_H
#define HIERMOE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* hm_last_error(void);
int hm_version(void);
/* Number of kernels this library has launched since it was loaded (for the
 * bench's gpu_launches count; no reference counterpart). */
unsigned long long hm_launch_count(void);

/* ---------------- decision path (planner) ---------------------------------
 * Mask layout: packed rows, W = ceil(E/32) uint32 words per row; bit e of row
 * t = (bits[t*W + e/32] >> (e%32)) & 1.                                      */

/* bool T x E mask -> packed bits, optional column gather (slot view).
 * Replaces RoutingMask (routing.py:31-56: row popcounts for the K check),
 * mask_bits (routing.py:84-90) and slot_view/apply_placement
 * (routing.py:98-106, 177-186). */
int hm_mask_pack(const uint8_t* mask, int64_t T, int32_t E, const int32_t* slot_to_expert,
                 uint32_t* bits, int32_t* row_popcount, void* stream);
int hm_mask_unpack(const uint32_t* bits, int64_t T, int32_t E, uint8_t* mask, void* stream);
/* K-per-row id lists -> packed slot-space bits (RoutingMask.bits from top-K ids) */
int hm_ids_to_bits(const int32_t* ids, int64_t T, int32_t K, int32_t E,
                   const int32_t* expert_to_slot, uint32_t* bits, int32_t* bad_flag,
                   void* stream);

/* Dedup and raw per-group counts for n_cuts group cuts in one pass, plus the
 * optional T x g dedup mask of cut `hit_cut`.  Replaces group_reduce
 * (traffic.py:58-64), dedup_counts (traffic.py:67-71), raw_counts
 * (traffic.py:74-82); duplication_rate (traffic.py:85-90) derives from them. */
int hm_level_counts(const uint32_t* bits, int64_t T, int32_t E, const int32_t* groups,
                    int32_t n_cuts, int64_t* dedup, int64_t* raw, uint8_t* hit,
                    int32_t hit_cut, void* stream);

/* Device-wide exclusive scan of int64 (workspace: hm_scan_workspace(n) bytes). */
size_t hm_scan_workspace(int64_t n);
int hm_scan_i64(const int64_t* in, int64_t n, int64_t* out, int64_t* grand, void* workspace,
                void* stream);

/* Hierarchical propagation: copies per row, then emit one copy per
 * (row, level group hit) in row-major order with restricted selections,
 * origin token and parent group.  Replaces propagate_level
 * (routing.py:189-215) and PropagatedMask (routing.py:59-78). */
int hm_propagate_count(const uint32_t* bits, int64_t T, int32_t E, int32_t groups,
                       int64_t* copies, void* stream);
int hm_propagate_emit(const uint32_t* bits, int64_t T, int32_t E, int32_t groups,
                      const int64_t* first_copy, const int64_t* origin_in, uint32_t* out_bits,
                      int64_t* out_origin, int64_t* out_parent, void* stream);

/* Swap partials of one group cut (base[g], sel[E], hitsel[E*g], lone[E],
 * lonesel[E*E]) and the E x E x g swap tensor.  Replaces
 * _swap_tensor_incremental / swap_tensors_incremental (swap.py:81-138). */
int hm_swap_partials(const uint32_t* bits, int64_t T, int32_t E, int32_t groups, int64_t* base,
                     int64_t* sel, int64_t* hitsel, int64_t* lone, int64_t* lonesel,
                     int32_t* too_dense, void* stream);
int hm_swap_tensor(const int64_t* base, const int64_t* sel, const int64_t* hitsel,
                   const int64_t* lone, const int64_t* lonesel, int32_t E, int32_t groups,
                   int64_t* z, void* stream);

/* Smooth-max cost matrix (gamma and exact max) for dimension *dim_dev (or
 * dim_host when dim_dev is NULL), numpy rounding order.  Replaces
 * smooth_max/_smooth_max_lastaxis (swap.py:35-57) and cost_matrix
 * (swap.py:180-206).  The inter_* arrays hold depth - 1 entries and the
 * intra_* arrays depth entries; cuts past the dimension evaluated are not
 * read by the kernel and may be passed as a null tensor with 0 groups. */
int hm_swap_cost(const int64_t* const* inter_z, const int32_t* inter_groups,
                 const int32_t* inter_part, const double* a_inter, const double* b_inter,
                 const int64_t* const* intra_z, const int32_t* intra_groups,
                 const int32_t* intra_part, const double* a_intra, const double* b_intra,
                 int32_t depth, int32_t E, int64_t token_bytes, double gamma,
                 const int32_t* dim_dev, int32_t dim_host, double* q, double* q_exact,
                 void* stream);
/* First-occurrence argmin + exact-max gate.  out_i64 = {flat, r, c, chosen},
 * out_f64 = {no_swap_time, saving}.  Replaces select_swap's decision
 * (swap.py:240-252). */
int hm_swap_select(const double* q, const double* q_exact, int32_t E, int64_t* out_i64,
                   double* out_f64, void* stream);

/* Phase time model and d* from dedup counts of cuts [U[1..D-1], G].
 * Replaces _time_for_dim/all_times/pick_dimension/optimal_dimension
 * (traffic.py:144-221); per-level counts are invariant under propagation
 * (swap.py:172-175), so no copy mask is materialised. */
int hm_time_model(const int64_t* dedup_concat, const int32_t* fanout_groups, int32_t depth,
                  int32_t gpus, int64_t token_bytes, const double* a_inter, const double* b_inter,
                  const double* a_intra, const double* b_intra, int32_t* cut_offsets_dev,
                  double* times, int32_t* d_star, int64_t* maxima, void* stream);
/* elementwise float64 x^y with numpy's rounding (np.power, used by
 * swap.py:56-57; numpy_pow.cuh restates numpy's SVML pow). */
int hm_np_pow(const double* x, const double* y, int64_t n, double* out, void* stream);
/* smooth_max over `rows` vectors of length n (swap.py:35-48). */
int hm_smooth_max_rows(const double* x, int64_t rows, int32_t n, double gamma, double* out,
                       void* stream);

/* ---------------- layer path (dispatch / combine) -------------------------
 * A world = G virtual EP ranks on P GPUs (L = G/P per GPU); slot s lives on
 * rank s / (E/G) (topology.py:99-100), tokens are rank-major.
 * The reference only models this exchange (traffic.py:93-170: AlltoAll with
 * and without dedup); these calls execute it. */
typedef struct hm_world hm_world;
/* relay_groups = U[1] > 0 makes a phase-1 (inter-level-1) world of a two-level
 * dispatch: one row per (token, level-1 group) to the rank with the source's
 * local index in that group, carrying the restricted slot ids:
 * the copy list of propagate_level (routing.py:189-215). */
int hm_world_create(int32_t ranks, int32_t gpus, int32_t gpu_index, int32_t experts,
                    int32_t top_k, int32_t hidden, int32_t elem_bytes, int64_t tokens_per_rank,
                    int64_t n_cap_rows, int32_t relay_groups, int32_t flags, hm_world** out);
/* phase-2 ids/gates from a relay world's received copies (HD2 relay, K5) */
int hm_relay_ids(hm_world* w, int32_t* ids2, float* w2, void* stream);
int hm_world_destroy(hm_world* w);
int64_t hm_world_ipc_handle_size(void);
int hm_world_ipc_handle(hm_world* w, void* out_handle);
int hm_world_open_peers(hm_world* w, const void* handles);
int hm_world_buffer(hm_world* w, int32_t kind, int32_t local_rank, void** ptr, int64_t* bytes);
int hm_world_info(hm_world* w, int64_t* out8);
int hm_world_barrier(hm_world* w, void* stream);
/* World options: 4 = grid cap of the exchange kernels (CTAs, 0 = 8 per SM);
 * 10 = fused one-GPU dispatch (expert-major row indices, buffer kind 17,
 * instead of row copies; the expert GEMM gathers the rows). */
int hm_world_set_option(hm_world* w, int32_t option, int32_t value);
/* per-kernel CUDA-event timing of a world's launches: segments plan, notify,
 * pack, barrier1, expand, reduce, barrier2, gather (ms of the last launch) */
int hm_world_set_timing(hm_world* w, int32_t enable);
int hm_world_timings(hm_world* w, float* ms, int32_t n);
/* stream-ordered copy between any two addresses (buffer inspection) */
int hm_memcpy(void* dst, const void* src, int64_t bytes, void* stream);

/* Softmax top-K gating -> slot ids (RoutingMask rows, K per
 * row, routing.py:31-56) and gate weights. */
int hm_route_topk(const float* logits, int64_t T, int32_t E, int32_t K,
                  const int32_t* expert_to_slot, int32_t renormalize, int32_t* slot_ids,
                  float* weights, int32_t* expert_ids, void* stream);
/* Router kernel choice: 1 = four lanes per token where it applies (default;
 * E in {32, 64, 128, 256}, renormalised weights), 0 = lane per token always.
 * Identical results. */
int hm_route_set_option(int32_t quad);
/* DeepSeek-V3 group-limited gate (the reference specifies only
 * softmax top-K): sigmoid scores + bias choice, the topk_group
 * best of n_group contiguous expert groups (group score = sum of its two
 * largest choices), top-K inside them, weights = picked scores / sum *
 * route_scale.  bias may be NULL.  Value-descending, index-ascending order. */
int hm_route_group(const float* logits, int64_t T, int32_t E, int32_t K, int32_t n_group,
                   int32_t topk_group, const float* bias, float route_scale,
                   const int32_t* expert_to_slot, int32_t* slot_ids, float* weights,
                   int32_t* expert_ids, void* stream);
/* Dedup (one row per token x destination rank) or raw (one per selection)
 * dispatch; the per-destination histogram equals dedup_counts / raw_counts
 * at G (traffic.py:67-82). */
int hm_dispatch(hm_world* w, const void* x, const int32_t* ids, const float* wts, int32_t dedup,
                void* stream);
/* hm_dispatch in two phases: the plan (per-chunk ranks, count exchange,
 * offsets) and the push (row movement + device barrier); hm_dispatch = both. */
int hm_dispatch_plan(hm_world* w, const int32_t* ids, const float* wts, int32_t mode,
                     void* stream);
int hm_dispatch_push(hm_world* w, const void* x, const int32_t* ids, const float* wts,
                     int32_t mode, void* stream);
/* Destination-side re-expansion of dedup rows into expert-major rows. */
int hm_expand(hm_world* w, void* stream);
/* Exchange overlapped with the expert FFN (per-GPU dedup, mode 3, fused
 * dispatch, N > 1; no reference counterpart -- the reference only models the
 * AlltoAll, traffic.py:93-170): after hm_dispatch_plan, hm_dispatch_meta writes
 * positions and receive metadata without moving rows; hm_experts_overlap runs
 * the local rows' GEMM1 with the token rows crossing NVLink beside its tiles
 * (warp 3 of every CTA), the device barrier, the received rows' GEMM1 and
 * GEMM2 over all rows; hm_combine follows.  Same results as hm_dispatch +
 * hm_expand + hm_expert_ffn_multi. */
int hm_dispatch_meta(hm_world* w, const int32_t* ids, const float* wts, void* stream);
int hm_experts_overlap(hm_world* w, const void* x, const void* w13, const void* w2,
                       int32_t hidden, int32_t inter, void* h, void* g13, void* stream);
/* Gate-weighted combine (pre-reduce per destination + source sum for dedup). */
int hm_combine(hm_world* w, const float* wts, const int32_t* ids, int32_t dedup, void* out,
               void* stream);
/* hm_combine plus one addend row per token (payload dtype, [L*T_r][M]),
 * accumulated in fp32 after the routed rows: out = sum_k w_k y_k + addend.
 * Used for DeepSeek-V3's shared expert; no reference
 * counterpart. */
int hm_combine_add(hm_world* w, const float* wts, const int32_t* ids, int32_t mode,
                   const void* addend, void* out, void* stream);
/* bf16 -> fp32 widening of n elements (16-byte aligned buffers): the fp32
 * operand of the router logits GEMM (the step before the
 * path); no reference counterpart. */
int hm_bf16_to_f32(const void* src, float* dst, int64_t n, void* stream);
/* Router GEMMs on the tcgen05 kernels (gating PAPER.md:112):
 * hm_gemm_f32: out[rows][ld] fp32 (first n_valid columns) = A[rows][K] . B^T,
 * B [N][K] bf16, N % 256 == 0 (zero-padded expert rows), rows_dev = device
 * {rows}: the router logits x . Wr^T and the router data gradient dlogits . Wr.
 * hm_wgrad_f32: out[m_out][N] fp32 (+= if accumulate) = A^T . B over the
 * token rows of A [rows][m_out], B [rows][N]: the router weight gradient. */
int hm_gemm_f32(const void* a, int64_t rows, const int32_t* rows_dev, const void* b, int32_t N,
                int32_t K, int32_t n_valid, float* out, int64_t ld_out, void* stream);
int hm_wgrad_f32(const void* a, const void* b, int64_t rows, const int32_t* rows_dev,
                 int32_t m_out, int32_t N, float* out, int64_t ld_out, int32_t accumulate,
                 void* stream);
/* out[rows][ld] bf16 = bf16((A . B^T + add1) + add2) (fp32 sums, add2 may be
 * NULL): the router input gradient fused with the routed / shared-expert
 * input gradients -- hm_gemm_f32 + hm_sum_to_bf16 in one launch. */
int hm_gemm_add_bf16(const void* a, int64_t rows, const int32_t* rows_dev, const void* b,
                     int32_t N, int32_t K, const void* add1, const void* add2, void* out,
                     int64_t ld_out, void* stream);
/* ... the same with the token reduction split into chunks (sized on the device
 * from rows_dev) over the SMs, fp32 partials in the caller's scratch
 * (hm_wgrad_f32_scratch_bytes(rows, m_out, N) bytes; 0 = no split needed)
 * summed into out: a 128 x 2048 router gradient is only 8 output tiles. */
int64_t hm_wgrad_f32_scratch_bytes(int64_t rows, int32_t m_out, int32_t N);
int hm_wgrad_f32_split(const void* a, const void* b, int64_t rows, const int32_t* rows_dev,
                       int32_t m_out, int32_t N, float* out, int64_t ld_out, int32_t accumulate,
                       void* scratch, int64_t scratch_bytes, void* stream);
/* Gate backward: dense bf16 dlogits [T][ld] (zero past E) from the gate
 * weights' gradient dw [T][K]; mode 0 softmax over the picks (renormalised),
 * 1 softmax over all experts, 2 DeepSeek-V3 normalised sigmoid (route_scale). */
int hm_gate_backward(const float* logits, const int32_t* expert_ids, const float* weights,
                     const float* dw, int64_t T, int32_t E, int32_t K, int32_t mode,
                     float route_scale, void* dlogits, int32_t ld, void* stream);
/* out = bf16((a + b) + c), fp32 sums, c may be NULL (b, c, out bf16; 16-byte
 * aligned): the layer's input gradient, router-GEMM term + routed dx (+ the
 * shared expert's dx), rounded once; no reference counterpart. */
int hm_sum_to_bf16(const float* a, const void* b, const void* c, void* out, int64_t n,
                   void* stream);
/* Backward (world created with flags & 1).  hm_dispatch_grad = combine
 * backward: output grads -> expert-output grads (dedup broadcast, replaying the
 * forward plan) + direct picks' gate grads; hm_combine_grad = dispatch
 * backward: expert-input grads -> token grads (dedup reduction) + remaining
 * gate grads.  Every transport mode 0..3 (mode 3: one gradient row per
 * (token, other GPU hit), pre-reduced input grads per (token, GPU)). */
int hm_dispatch_grad(hm_world* w, const void* g, const int32_t* ids, const float* wts,
                     int32_t mode, float* dw, void* stream);
int hm_combine_grad(hm_world* w, const int32_t* ids, int32_t mode, float* dw, void* dx,
                    void* stream);

/* ---------------- expert FFN (tcgen05 + TMA + TMEM, sm_100a) -------------
 * The only dense contraction of the layer (E expert FFNs); no
 * reference implementation.  Groups are consecutive row blocks of A with
 * device-side sizes n_rows[g] (the dispatch's expert-major layout). */
/* hm_grouped_gemm with B as stored, [groups][K][N] (read MN-major by the
 * tensor cores): the data-gradient GEMMs on the expert weights themselves. */
int hm_grouped_gemm_kn(const void* a, int64_t a_rows, const void* b, int32_t groups,
                       const int32_t* n_rows, int32_t N, int32_t K, void* out, int64_t ld_out,
                       void* stream);
int hm_grouped_gemm(const void* a, int64_t a_rows, const void* b, int32_t groups,
                    const int32_t* n_rows, int32_t N, int32_t K, int32_t swiglu, void* out,
                    int64_t ld_out, void* stream);
int hm_expert_ffn(const void* x, int64_t a_rows, const int32_t* n_rows, int32_t groups,
                  const void* w13, const void* w2, int32_t hidden, int32_t inter, void* h,
                  void* y, void* stream);
/* Training forward: as hm_expert_ffn, and GEMM1's epilogue also stores the
 * gate/up pre-activations g13 [a_rows][2I] (bf16, 128-column gate/up blocks)
 * for hm_expert_ffn_backward_saved. */
int hm_expert_ffn_save(const void* x, int64_t a_rows, const int32_t* n_rows, int32_t groups,
                       const void* w13, const void* w2, int32_t hidden, int32_t inter, void* h,
                       void* y, void* g13, void* stream);
/* Fused dispatch (one GPU): the expert-major rows are not materialised;
 * layout row r (capacity a_rows, groups of n_rows[g]) is source row idx[r]
 * of x [x_rows][hidden], loaded by GEMM1's A-gather warps (cp.async into the
 * swizzled stage).  g13 optional (the pre-activations for the backward).
 * Replaces the copy half of the dispatch the reference models as one
 * AlltoAll row per selection (traffic.py:164-170) with row indices
 * (hm_world_set_option 10 makes hm_dispatch emit them). */
int hm_expert_ffn_gather(const void* x, int64_t x_rows, const int32_t* idx, int64_t a_rows,
                         const int32_t* n_rows, int32_t groups, const void* w13, const void* w2,
                         int32_t hidden, int32_t inter, void* h, void* y, void* g13,
                         void* stream);
/* Its backward (saved pre-activations, MN-major weight gradients; dW13's
 * token operand gathered from x by idx).  accumulate != 0 adds the weight
 * grads to dw13 / dw2. */
int hm_expert_ffn_backward_gather(const void* x, int64_t x_rows, const int32_t* idx,
                                  int64_t a_rows, const int32_t* n_rows, int32_t groups,
                                  const void* w13, const void* w2, const void* gy,
                                  int32_t hidden, int32_t inter, const void* g13, void* dh,
                                  void* dg13, void* h, int32_t* layout, void* gx, void* dw13,
                                  void* dw2, int32_t accumulate, void* stream);
/* Expert FFN backward: pre-activations recomputed (GEMM1), data-gradient
 * GEMMs on the weights as stored (w13 [g][2I][M], w2 [g][M][I], read MN-major
 * by the tensor cores -- no transposed copies), SwiGLU backward, and
 * weight-gradient GEMMs over each expert's own token rows. */
int hm_expert_ffn_backward(const void* x, int64_t a_rows, const int32_t* n_rows, int32_t groups,
                           const void* w13, const void* w2, const void* gy, int32_t hidden,
                           int32_t inter, void* g13, void* dh, void* dg13, void* h,
                           int32_t* layout, void* gx, void* dw13, void* dw2, void* stream);
/* hm_expert_ffn_backward with g13 holding the forward's pre-activations
 * (hm_expert_ffn_save): skips the GEMM1 recompute.  accumulate != 0 adds the
 * weight grads to dw13 / dw2 (fp32 add of the stored bf16): one call per
 * micro-batch of a layer. */
int hm_expert_ffn_backward_saved(const void* x, int64_t a_rows, const int32_t* n_rows,
                                 int32_t groups, const void* w13, const void* w2,
                                 const void* gy, int32_t hidden, int32_t inter, const void* g13,
                                 void* dh, void* dg13, void* h, int32_t* layout, void* gx,
                                 void* dw13, void* dw2, int32_t accumulate, void* stream);
/* Several EP ranks' expert FFNs in one launch per GEMM (a GPU hosting L
 * ranks): segment s = groups [s * groups_per_seg, (s + 1) * groups_per_seg)
 * with its rows at [s * seg_rows, ...) of every row buffer ([segs][seg_rows]);
 * idx null -> x holds the expert-major rows, else layout row r = x row idx[r]
 * (idx >= 0) or x_recv row ~idx[r] (idx < 0: rows received over NVLink). */
int hm_expert_ffn_multi(const void* x, int64_t x_rows, const int32_t* idx, const void* x_recv,
                        int64_t seg_rows, int32_t segs, const int32_t* n_rows,
                        int32_t groups_per_seg,
                        const void* w13, const void* w2, int32_t hidden, int32_t inter, void* h,
                        void* y, void* g13, void* stream);
/* ... over explicit row groups: group g = rows [g_row0[g], g_row0[g] +
 * g_rows[g]) of the [rows] row space times expert weight g_wsel[g] of
 * [nweights] experts; ctas > 0 caps the grid. */
int hm_expert_ffn_groups(const void* x, int64_t x_rows, const int32_t* idx, const void* x_recv,
                         int64_t rows, int32_t groups, const int32_t* g_row0,
                         const int32_t* g_rows, const int32_t* g_wsel, int32_t nweights,
                         const void* w13, const void* w2, int32_t hidden, int32_t inter, void* h,
                         void* y, void* g13, int32_t ctas, void* stream);
int hm_expert_ffn_backward_multi(const void* x, int64_t x_rows, const int32_t* idx,
                                 const void* x_recv, int64_t seg_rows, int32_t segs,
                                 const int32_t* n_rows,
                                 int32_t groups_per_seg, const void* w13, const void* w2,
                                 const void* gy, int32_t hidden, int32_t inter, const void* g13,
                                 void* dh, void* dg13, void* h, int32_t* layout, void* gx,
                                 void* dw13, void* dw2, int32_t accumulate, int32_t parts,
                                 void* stream);
/* parts: 1 = data gradients (dH, SwiGLU backward, gX), 2 = weight gradients
 * (dW2, dW13 from part 1's scratch), 3 = both -- a caller can run the
 * dispatch backward of gX beside the weight-gradient GEMMs; + 4: h holds the
 * forward's H (not rewritten by the SwiGLU backward; dW2 uses it). */
/* FFN options (no reference counterpart): 1 = cap on the persistent GEMM grid
 * in CTAs (0 = one per SM), so a concurrent exchange keeps SMs of its own;
 * 2 = CTA-pair weight gradients (default 1; 0 = single-CTA kernel);
 * 5 = 256 x 512 pair tiles: 0 never, 1 (default) for the long-K (>= 4096)
 * data-gradient GEMMs on the weights as stored, 2 wherever N % 512 == 0;
 * 6 = TMA tensor stores for whole 32-row output blocks of the bf16 GEMMs
 * (default 1; 0 = LSU stores only). */
int hm_ffn_set_option(int32_t option, int32_t value);

/* ---------------- expert migration (K11) ------------------------------------
 * Apply a planned swap (apply_swap, swap.py:255-259) to the physical expert
 * state: per-GPU symmetric store of n_arrays slot-major tensors (weights,
 * master copy, optimizer moments), peer-to-peer over CUDA IPC / NVLink. */
typedef struct hm_store hm_store;
int hm_store_create(int32_t gpus, int32_t gpu_index, int32_t slots_per_gpu,
                    const int64_t* slice_bytes, int32_t n_arrays, hm_store** out);
int hm_store_destroy(hm_store* s);
int hm_store_ipc_handle(hm_store* s, void* out_handle);
int hm_store_open_peers(hm_store* s, const void* handles);
int hm_store_array(hm_store* s, int32_t a, void** ptr);
int hm_store_status(hm_store* s, int32_t* out4);
int hm_migrate(hm_store* s, int32_t slot_r, int32_t slot_c, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HIERMOE_H */
