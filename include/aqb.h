/*
 * aqb.h — C-ABI of the B200-native DiT denoise hot path (libaqb.so).
 *
 * The reference (ditplan, arXiv 2505.10584) has no FFI for this path: it is a
 * pure-Python planner whose only executable piece of the path is the cache
 * schedule (pkg/src/ditplan/inference.py:48-86).  The denoise step itself is
 * described only in prose.  Each entry
 * point below therefore cites the paper op it implements (Table 2 rows,
 * PAPER.md:246-256, mirrored as BUILTIN_CHUNKS in pkg/src/ditplan/memory.py:92-107)
 * — that is the interface a maintainer would bind.
 *
 * Conventions:
 *  - plain pointers and sizes only; all buffers (including workspace) are
 *    allocated by the caller; element strides are in elements;
 *  - `stream` is a cudaStream_t passed as void*; every call is stream-ordered,
 *    never synchronises the host and is safe to capture in a CUDA graph;
 *  - return 0 (AQB_OK) or a negative status; aqb_last_error() describes it
 *    (thread-local);
 *  - `run_flag`/`run_if`: when run_flag != NULL the kernel does its work only
 *    if *run_flag == run_if (device-side cache decision, no host round-trip).
 *  - bf16 = IEEE bfloat16 stored as uint16; f32 = float.
 */
#ifndef AQB_H_
#define AQB_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AQB_ABI_VERSION 2

#define AQB_OK 0
#define AQB_EINVAL (-1)
#define AQB_ECUDA (-2)
#define AQB_EUNSUPPORTED (-3)

int aqb_abi_version(void);
/* sha256 (hex) of this header as compiled into the library — the Python binding
 * refuses a libaqb.so built from a different header (stale build). */
const char* aqb_build_id(void);
const char* aqb_last_error(void);
int aqb_sm_count(void);
/* Programmatic dependent launch for subsequent launches of this process: 1 = on (the
 * default unless AQB_PDL=0), 0 = off.  Returns the previous setting.  Off makes every
 * kernel's measured duration its own execution (a PDL kernel's span includes its wait on
 * the predecessor); the bench's per-kernel trace pass uses it. */
int aqb_set_pdl(int on);

/* ---------------------------------------------------------------------------
 * "LayerNorm + Scale/Shift" (memory.py:104):
 *   y[i,:] = bf16( norm(x[i,:]) * (1 + scale) + shift )
 * norm_kind 0 = LayerNorm (no affine), 1 = RMSNorm (no affine), 2 = none (cast).
 * x f32 [rows, hidden] (stride ldx); y bf16 (stride ldy); shift/scale f32
 * [hidden] or NULL.  hidden % 128 == 0, hidden <= 4096.
 * Optional rel-L1 probe (diffusion cache, north_star): when probe_prev != NULL
 * (f32 [rows, hidden], dense) the kernel also writes, per row,
 * probe_partials[row] = sum|m - prev| and probe_partials[rows + row] =
 * sum|prev| (f32, m = the un-rounded modulated value), then overwrites prev with m.
 */
int aqb_norm_modulate(const float* x, int64_t ldx, const float* shift, const float* scale, void* y, int64_t ldy,
                      int64_t rows, int32_t hidden, float eps, int32_t norm_kind, float* probe_prev,
                      float* probe_partials, const int32_t* run_flag, int32_t run_if, void* stream);
/* TP-SP "AllGather + ..." (sequence-parallel LayerNorm feeding a
 * column-parallel projection): as aqb_norm_modulate, but row i is stored into each
 * of the ny (1..8) outputs y[d] + i*ldy — every rank's gathered buffer, at this
 * rank's row offset (peer memory over NVLink), so the all-gather is the kernel's
 * own stores.  16-byte aligned outputs. */
/* TP-SP "Out_Linear / FFN_Linear2 + ReduceScatter" fused: this
 * rank's partial of a row-parallel projection, gate[n] * (acc + bias) (bias NULL on all
 * but one rank), is reduce-added (f32, at the destination) into the residual of the
 * rank owning each row: row i -> peer_out[i / rows_per_rank] + (i % rows_per_rank)*ldo.
 * m == nranks * rows_per_rank.  Summation order across ranks is not fixed (f32
 * reductions race at the owner), so results are not bitwise reproducible run to run. */
int aqb_gemm_gate_add_scatter(const void* a, int64_t lda, const void* w, int64_t ldw, float* const* peer_out,
                              int32_t nranks, int64_t ldo, int64_t rows_per_rank, int64_t m, int64_t n, int64_t k,
                              const float* bias, const float* gate, const int32_t* run_flag, int32_t run_if,
                              void* stream);
/* TP-SP all-reduce of replicated rows (MM-DiT text rows), deterministic:
 * aqb_gate_bcast writes gate[c] * src[r, c] (gate NULL: 1) into each of the ndst
 * (1..8) buffers dst[d] + r*ldd (this rank's slot in every rank's slot buffer, over
 * NVLink); after a barrier aqb_sum_slots adds the nslots slots (slot k at
 * slots + k*slot_stride, row stride lds) into x in slot order.  f32, cols % 4 == 0. */
int aqb_gate_bcast(const float* src, int64_t lds, const float* gate, float* const* dst, int32_t ndst, int64_t ldd,
                   int64_t rows, int64_t cols, const int32_t* run_flag, int32_t run_if, void* stream);
int aqb_sum_slots(float* x, int64_t ldx, const float* slots, int32_t nslots, int64_t slot_stride, int64_t lds,
                  int64_t rows, int64_t cols, const int32_t* run_flag, int32_t run_if, void* stream);
int aqb_norm_modulate_gather(const float* x, int64_t ldx, const float* shift, const float* scale, void* const* y,
                             int32_t ny, int64_t ldy, int64_t rows, int32_t hidden, float eps, int32_t norm_kind,
                             float* probe_prev, float* probe_partials, const int32_t* run_flag, int32_t run_if,
                             void* stream);

/* ---------------------------------------------------------------------------
 * Projection GEMMs (AllGather+QKV_Linear, Out_Linear, FFN_Linear1/2, GeLU and
 * Gate fused as epilogues — PAPER.md:249-252,254,256):
 *   acc[m,n] = sum_k A[m,k] * W[n,k]       (A, W bf16, K contiguous; tcgen05)
 * epilogue:
 *   AQB_EPI_BF16       out bf16 = acc + bias
 *   AQB_EPI_GELU_BF16  out bf16 = gelu_tanh(acc + bias)
 *   AQB_EPI_GATE_RES   out f32 (in/out residual) += gate[n] * (acc + bias); if aux != NULL
 *                      also aux bf16 (stride ld_aux) = bf16(new out) — the next projection's A
 *                      operand, so no separate cast pass
 *   AQB_EPI_F32        out f32 = acc + bias
 *   AQB_EPI_EULER      out f32 (latent, in/out) += (*alpha) * (acc + bias);
 *                      aux bf16 (stride ld_aux) = bf16(new out)   [flow-matching Euler step]
 * bias/gate f32 [n] or NULL; alpha: device f32 scalar (EULER only).
 * Requirements: k % 8 == 0, n % 16 == 0, 16-byte aligned rows.
 */
#define AQB_EPI_BF16 0
#define AQB_EPI_GELU_BF16 1
#define AQB_EPI_GATE_RES 2
#define AQB_EPI_F32 3
#define AQB_EPI_EULER 4
#define AQB_EPI_QKNORM_ROPE 5 /* internal: selected by aqb_gemm_qknorm_rope */
int aqb_gemm_bf16(const void* a, int64_t lda, const void* w, int64_t ldw, void* out, int64_t ldo, int64_t m,
                  int64_t n, int64_t k, const float* bias, const float* gate, int32_t epilogue, const float* alpha,
                  void* aux, int64_t ld_aux, const int32_t* run_flag, int32_t run_if, void* stream);

/* ---------------------------------------------------------------------------
 * AllGather+QKV_Linear + Fused QKNorm + 3D RoPE in one kernel (PAPER.md:252-253,
 * 114-115; memory.py:101,103): tcgen05 GEMM whose epilogue RMS-normalises each
 * 128-wide head of the first norm_parts column parts (q_w, k_w), applies the 3D
 * RoPE to rows with (rope_row0 + row) < rope_rows, and TMA-stores bf16 into
 *   out[(h / hpg - g_base) * group_stride + row * out_row_stride
 *       + part * hpg * 128 + (h % hpg) * 128 + d]
 * (groups = Ulysses ranks; columns of heads whose group is outside
 * [0, groups) are dropped).  head_dim must be 128; n = parts * part_width.
 */
int aqb_gemm_qknorm_rope(const void* a, int64_t lda, const void* w, int64_t ldw, int64_t m, int64_t n, int64_t k,
                         const float* bias, int32_t part_width, int32_t norm_parts, const float* q_w,
                         const float* k_w, float eps, const float* rope_cos, const float* rope_sin,
                         int64_t rope_row0, int64_t rope_rows, void* out, int64_t out_row_stride, int32_t groups,
                         int64_t group_stride, int32_t hpg, int32_t g_base, const int32_t* run_flag,
                         int32_t run_if, void* stream);

/* Ulysses "AllGather+QKV_Linear" + "AlltoAll" fused: as
 * aqb_gemm_qknorm_rope, but head group g (heads [g*hpg, (g+1)*hpg)) is
 * TMA-stored straight into rank g's attention-input buffer: element
 * (row, part, h, d) -> peer_out[g] + row*out_row_stride + part*hpg*128
 * + (h % hpg)*128 + d.  peer_out: HOST array of nranks device pointers
 * (peer memory), each already offset to this rank's row block. */
int aqb_gemm_qknorm_rope_scatter(const void* a, int64_t lda, const void* w, int64_t ldw, int64_t m, int64_t n,
                                 int64_t k, const float* bias, int32_t part_width, int32_t norm_parts,
                                 const float* q_w, const float* k_w, float eps, const float* rope_cos,
                                 const float* rope_sin, int64_t rope_row0, int64_t rope_rows, void* const* peer_out,
                                 int32_t nranks, int64_t out_row_stride, int32_t hpg, const int32_t* run_flag,
                                 int32_t run_if, void* stream);

/* ---------------------------------------------------------------------------
 * "Fused QKNorm" (memory.py:103) + 3D RoPE
 * + Ulysses pack.  src bf16 [rows, parts, heads, D] (row stride ld_src), parts
 * in {1,2,3} (q | k,v | q,k,v).  For each row r and head h in
 * [head_begin, head_begin + head_count): part p < norm_parts is RMS-normed
 * with weight (p == 0 ? q_w : k_w) [D] and, if (rope_row0 + r) < rope_rows,
 * its interleaved pairs are rotated by rope_cos/sin[rope_row0 + r, :]
 * (f32 [rope_rows, D/2]); parts >= norm_parts are copied.
 * dst element (r, part, h, d) lives at
 *   dst + (j / hpg) * dst_group_stride + r * dst_row_stride + part * dst_which_stride
 *       + (j % hpg) * D + d,   j = h - head_begin, hpg = heads per group.
 * In place (dst == src, natural strides) is allowed.  D in {32, 64, 128, 256}.
 */
int aqb_qk_norm_rope(const void* src, int64_t ld_src, int64_t rows, int32_t heads, int32_t head_begin,
                     int32_t head_count, int32_t head_dim, const float* q_w, const float* k_w, float eps,
                     const float* rope_cos, const float* rope_sin, int64_t rope_row0, int64_t rope_rows, void* dst,
                     int64_t dst_group_stride, int64_t dst_row_stride, int64_t dst_which_stride, int32_t hpg,
                     int32_t parts, int32_t norm_parts, const int32_t* run_flag, int32_t run_if, void* stream);

/* ---------------------------------------------------------------------------
 * "Flash Attention" (memory.py:97): non-causal softmax(QK^T*scale)V
 * per head, tcgen05/TMEM, TMA-fed.  Rows of head h of Q start at
 * q + h*q_head_stride with row stride ldq (likewise K, V, O).  bf16 in/out;
 * f32 softmax statistics.  head_dim in {32, 64, 128}.  seq_kv >= 1.
 * Split-KV (few heads x queries vs. 148 SMs, e.g. Ulysses' A/P heads):
 * kv_splits = 0 picks a plan (the wave-quantisation tail, or every tile when
 * few, split aqb_attention_splits ways — possibly unevenly: a long first part
 * and short tails), 1 disables it, s > 1 splits all tiles evenly; the partials
 * (f32 O/l + log2-sum-exp2 per row) go to `workspace`
 * (aqb_attention_workspace_bytes) and a combine pass writes O (in split
 * order: deterministic).  Automatic splitting silently stays at 1 split without
 * enough workspace.  seq_kv <= 256 with head_dim 128 and a local output takes
 * the short-KV kernel (kv_splits = 0 only).
 */
int aqb_attention_fwd(const void* q, int64_t ldq, int64_t q_head_stride, const void* k, int64_t ldk,
                      int64_t k_head_stride, const void* v, int64_t ldv, int64_t v_head_stride, void* o,
                      int64_t ldo, int64_t o_head_stride, int64_t seq_q, int64_t seq_kv, int32_t heads,
                      int32_t head_dim, float softmax_scale, int32_t kv_splits, void* workspace,
                      int64_t workspace_bytes, const int32_t* run_flag, int32_t run_if, void* stream);
int aqb_attention_splits(int64_t seq_q, int64_t seq_kv, int32_t heads, int32_t head_dim);
/* tiles (head x 256 queries) the automatic plan runs in one pass; the rest split
 * aqb_attention_splits ways (wave-quantisation tail, or all tiles when few) */
/* Profiling hook: device buffer (>= 64 * CTAs uint64) into which the short-KV attention kernel
 * writes clock64 stamps of its pipeline events; NULL (default) disables.  Not thread-safe
 * against concurrent launches; a measurement aid, off the product path. */
int aqb_attention_trace(void* buffer);
/* Profiling hook: device buffer (>= 128 * CTAs uint64) into which the GEMM kernels write
 * clock64 stamps (entry, after the PDL wait, each k-block the MMA warp consumes, each tile's
 * epilogue start / end); NULL (default) disables.  A measurement aid, off the product path:
 * compiled in only by a build with AQB_BUILD_DEFINES=-DAQB_GEMM_TRACE, otherwise a non-NULL
 * buffer returns AQB_EINVAL. */
int aqb_gemm_trace(void* buffer);
/* The automatic split-KV plan: out[5] = {whole tiles, splits, KV blocks of split 0, KV blocks of
 * each later split, split-major launch order (0/1)}. */
int aqb_attention_plan(int64_t seq_q, int64_t seq_kv, int32_t heads, int32_t head_dim, int32_t* out);
int aqb_attention_whole_tiles(int64_t seq_q, int64_t seq_kv, int32_t heads, int32_t head_dim);
/* 256-query blocks of one head each CTA of a one-pass launch runs with K/V loaded
 * once (short KV: 2 x KV blocks fit the K/V ring, e.g. cross-attention to 256 text
 * tokens); 1 = one block per CTA.  AQB_ATTN_PAIRS=g in the environment forces g. */
int aqb_attention_pairs_per_cta(int64_t seq_q, int64_t seq_kv, int32_t heads, int32_t head_dim);
/* workspace for any plan of <= kv_splits splits, and for the automatic plan */
int64_t aqb_attention_workspace_bytes(int64_t seq_q, int32_t heads, int32_t head_dim, int32_t kv_splits);
int64_t aqb_attention_auto_workspace_bytes(int64_t seq_q, int64_t seq_kv, int32_t heads, int32_t head_dim);

/* Ulysses "AlltoAll after attention" fused into the attention epilogue
 * (comm.py:65-96 costs it): output row r < text_row0 of head h
 * is stored into rank (r / rows_per_rank)'s O buffer, row r % rows_per_rank:
 *   peer_o[r / rows_per_rank] + h*o_head_stride + (r % rows_per_rank)*ldo + d;
 * rows r >= text_row0 (replicated text tokens) go to every rank at row
 * rows_per_rank + (r - text_row0).  peer_o is a HOST array of nranks device
 * pointers (peer memory, see aqb_peer_open), each already offset to this
 * rank's head columns.  text_row0 == rows_per_rank * nranks. */
int aqb_attention_fwd_scatter(const void* q, int64_t ldq, int64_t q_head_stride, const void* k, int64_t ldk,
                              int64_t k_head_stride, const void* v, int64_t ldv, int64_t v_head_stride,
                              void* const* peer_o, int32_t nranks, int64_t ldo, int64_t o_head_stride,
                              int64_t rows_per_rank, int64_t text_row0, int64_t seq_q, int64_t seq_kv, int32_t heads,
                              int32_t head_dim, float softmax_scale, int32_t kv_splits, void* workspace,
                              int64_t workspace_bytes, const int32_t* run_flag, int32_t run_if, void* stream);

/* ---------------------------------------------------------------------------
 * AdaLN / timestep GEMV (tiny, per step):  y[n] = act(sum_k W[n,k] * in(x[k]) + b[n]) + add[n]
 * W bf16 [n, k]; x/b/add/y f32.  in_silu: apply SiLU to x first.  x may be
 * replaced by sinusoidal timestep features of *t (x == NULL, k even):
 * feat = [cos(1000 t f_i), sin(1000 t f_i)], f_i = 10000^(-i/(k/2)).
 */
int aqb_gemv(const void* w, const float* x, const float* t, const float* b, const float* add, float* y, int64_t n,
             int64_t k, int32_t in_silu, void* stream);

/* out[i] = a[i % period] + b[i]  (f32) — per-block modulation tables. */
int aqb_add_bcast(float* out, const float* a, int64_t period, const float* b, int64_t n, void* stream);

/* ---------------------------------------------------------------------------
 * Diffusion cache (north_star).
 * aqb_rel_l1_reduce: sums[0] = sum partials[0:rows], sums[1] = sum partials[rows:2rows]
 *   (single CTA, fixed order — deterministic).
 * aqb_cache_decide: state (int32[4]: step, flag_full, _, _; f32 view at state+2: acc)
 *   advances one step and decides full/cached with the RelL1 rule
 *   (schedule.RelL1Policy.decide); writes flags_out[step] and rel_out[step].
 * aqb_cache_offset: mode 0: off = x (save rear input);  mode 1: off = x - off
 *   (rear output - input);  mode 2: x = x + off (cached step).  f32 [rows, hidden].
 * aqb_step_scalars: cur[0] = ts[*idx], cur[1] = dts[*idx]; mode 1: (*idx)++.
 */
int aqb_rel_l1_reduce(const float* partials, int64_t rows, float* sums, void* stream);
int aqb_cache_decide(const float* sums, int32_t* state, float threshold, int32_t warmup, int32_t total_steps,
                     int32_t force_last, int32_t* flags_out, float* rel_out, void* stream);
int aqb_cache_offset(float* x, int64_t ldx, float* off, int64_t rows, int32_t hidden, int32_t mode,
                     const int32_t* run_flag, int32_t run_if, void* stream);
int aqb_step_scalars(const float* ts, const float* dts, int32_t* idx, float* cur, int32_t mode, void* stream);

/* ---------------------------------------------------------------------------
 * Latent layout: lat f32 [C, lat_frames, H*ph, W*pw] whose frames
 * [frame_offset, frame_offset + T*pt)  <->  tokens [T*H*W, pt*ph*pw*C]
 * (token-major, features ordered (pt, ph, pw, c)).  patchify writes f32 tokens
 * and a bf16 copy (tok_bf16 may be NULL); unpatchify reads f32 tokens.  The
 * frame window serves temporal MultiDiffusion clips of a longer latent
 * (PAPER.md:411); lat_frames = T*pt, frame_offset = 0 for a whole latent.
 */
int aqb_patchify(const float* lat, float* tok, void* tok_bf16, int32_t C, int32_t T, int32_t H, int32_t W,
                 int32_t pt, int32_t ph, int32_t pw, int32_t lat_frames, int32_t frame_offset, void* stream);
int aqb_unpatchify(const float* tok, float* lat, int32_t C, int32_t T, int32_t H, int32_t W, int32_t pt,
                   int32_t ph, int32_t pw, int32_t lat_frames, int32_t frame_offset, void* stream);

/* Ulysses head->sequence repack: src bf16 [P, rows, hpg*D] -> dst [rows, P*hpg*D] (row stride ld_dst). */
int aqb_heads_to_seq(const void* src, int64_t rows, int32_t P, int32_t width, void* dst, int64_t ld_dst,
                     const int32_t* run_flag, int32_t run_if, void* stream);

/* ---------------------------------------------------------------------------
 * Either side of the denoise loop.
 * aqb_tile_blend — VAE tile blend (plan: inference.py:89-226):
 *   out[c, p] = sum_k prof_k(p) * tile_k[c, p - start_k] / sum_k prof_k(p), p = (t, h, w)
 *   over the tiles covering p, where prof_k is the product of per-axis ramps
 *   (rise (j+1)/(e+1) over the first e = min(overlap, size) entries, fall over the
 *   last e).  Tiles form the plan's grid: axis_starts = [t-starts (nt) | h-starts (nh)
 *   | w-starts (nw)] (device int32, ascending), tile_ptrs[(it*nh+ih)*nw+iw] = device
 *   address (int64, device array) of tile f32 [C, tile_t, tile_h, tile_w] (may be peer
 *   memory).  out f32 [C, T, H, W].  fp64 accumulation in plan order.
 * aqb_window_average — temporal MultiDiffusion Eq. 3 (inference.py:229-279):
 *   out[c, i, :] = (sum_{k: s_k <= i < s_k + n} clip_k[c, i - s_k, :]) / |S(i)|,
 *   clip_ptrs (device int64) -> f32 [C, n, hw]; clip_starts device int32; out f32
 *   [C, n_prime, hw]; sum in clip order.
 */
int aqb_tile_blend(const int64_t* tile_ptrs, const int32_t* axis_starts, int32_t nt, int32_t nh, int32_t nw,
                   int32_t tile_t, int32_t tile_h, int32_t tile_w, int32_t ov_t, int32_t ov_h, int32_t ov_w, int32_t T,
                   int32_t H, int32_t W, int32_t C, float* out, void* stream);
int aqb_window_average(const int64_t* clip_ptrs, const int32_t* clip_starts, int32_t nclips, int32_t n,
                       int32_t n_prime, int32_t C, int64_t hw, float* out, void* stream);

/* ---------------------------------------------------------------------------
 * fp32 validation mode (north_star: <= 1e-4 latent rel-L2 vs the CPU
 * reference).  Same semantics as the bf16 entries above with every activation
 * in f32: aqb_norm_modulate_f32 writes f32 y; aqb_qk_norm_rope_f32 reads and
 * writes f32; aqb_gemm_f32 takes f32 A, the bf16 weight W, and always writes
 * f32 (AQB_EPI_BF16 / AQB_EPI_GELU_BF16 produce f32 here; aux of EULER is f32);
 * aqb_attention_f32 is f32 in/out with exact expf.  SIMT kernels for the
 * validation geometries, not the production path.
 */
int aqb_norm_modulate_f32(const float* x, int64_t ldx, const float* shift, const float* scale, float* y, int64_t ldy,
                          int64_t rows, int32_t hidden, float eps, int32_t norm_kind, float* probe_prev,
                          float* probe_partials, const int32_t* run_flag, int32_t run_if, void* stream);
int aqb_qk_norm_rope_f32(const float* src, int64_t ld_src, int64_t rows, int32_t heads, int32_t head_begin,
                         int32_t head_count, int32_t head_dim, const float* q_w, const float* k_w, float eps,
                         const float* rope_cos, const float* rope_sin, int64_t rope_row0, int64_t rope_rows, float* dst,
                         int64_t dst_group_stride, int64_t dst_row_stride, int64_t dst_which_stride, int32_t hpg,
                         int32_t parts, int32_t norm_parts, const int32_t* run_flag, int32_t run_if, void* stream);
int aqb_gemm_f32(const float* a, int64_t lda, const void* w, int64_t ldw, float* out, int64_t ldo, int64_t m,
                 int64_t n, int64_t k, const float* bias, const float* gate, int32_t epilogue, const float* alpha,
                 float* aux, int64_t ld_aux, const int32_t* run_flag, int32_t run_if, void* stream);
int aqb_attention_f32(const float* q, int64_t ldq, int64_t q_head_stride, const float* k, int64_t ldk,
                      int64_t k_head_stride, const float* v, int64_t ldv, int64_t v_head_stride, float* o, int64_t ldo,
                      int64_t o_head_stride, int64_t seq_q, int64_t seq_kv, int32_t heads, int32_t head_dim,
                      float softmax_scale, const int32_t* run_flag, int32_t run_if, void* stream);

/* ---------------------------------------------------------------------------
 * Peer memory over NVLink/NVSwitch (one process per GPU; the Ulysses exchange).
 * aqb_peer_alloc: zeroed device allocation + its CUDA IPC handle
 *   (AQB_IPC_HANDLE_BYTES bytes, exchanged by the caller, e.g. torch.distributed).
 * aqb_peer_open / aqb_peer_close: map / unmap another rank's allocation.
 * aqb_peer_barrier: stream-ordered barrier of nranks ranks.  peer_signal is a
 *   HOST array of nranks device pointers to each rank's AQB_PEER_SIGNAL_BYTES
 *   signal region (peer memory, zeroed); epoch is this rank's device counter
 *   (uint32, starts at 0, advanced by every barrier).  All prior writes of this
 *   rank (incl. stores into peer memory by earlier kernels) are visible to every
 *   rank after the barrier.  With npay > 0 (<= 4) each rank contributes
 *   payload[0:npay] and pay_out receives the sum over ranks in rank order
 *   (bit-identical on every rank).  A peer missing for ~10 s sets *status = 1
 *   and the kernel returns (no hang).  Gated by run_flag like the compute kernels
 *   (every rank must take the same gate decisions).
 */
#define AQB_IPC_HANDLE_BYTES 64
#define AQB_PEER_SIGNAL_BYTES 512
int aqb_peer_alloc(int64_t bytes, void** ptr, void* ipc_handle);
int aqb_peer_open(const void* ipc_handle, void** ptr);
int aqb_peer_close(void* ptr);
int aqb_peer_free(void* ptr);
int aqb_peer_can_access(int32_t device, int32_t peer_device);
int aqb_peer_barrier(void* const* peer_signal, int32_t rank, int32_t nranks, uint32_t* epoch, const float* payload,
                     int32_t npay, float* pay_out, int32_t* status, const int32_t* run_flag, int32_t run_if,
                     void* stream);

#ifdef __cplusplus
}
#endif

#endif /* AQB_H_ */
