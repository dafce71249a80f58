/*
 * star_attn.h — C ABI of the B200 (sm_100a) Star Attention hot path.
 *
 * Drop-in boundary for the two-phase attention path of the reference
 * (`starsim` 0.1.0, /root/reference/pkg/src/starsim, abbreviated ss/).  The
 * reference has no native code; these entry points replace the numpy compute
 * sites its Python API funnels into.  Each declaration cites the reference
 * interface it replaces.
 *
 * Conventions
 *  - Plain pointers and sizes only; no framework types cross the ABI.
 *  - Device pointers are caller-owned CUDA global memory; the library never
 *    allocates device memory.  `stream` is a cudaStream_t passed as void*.
 *  - Every call is stream-ordered and returns STAR_OK or a negative status.
 *    Status classes mirror the reference's error taxonomy (ss/errors.py:4-17):
 *      STAR_ESHAPE  -> ShapeError,  STAR_EDOMAIN -> DomainError,
 *      STAR_ECONFIG -> ConfigError, STAR_ECUDA / STAR_ENOTSUP -> runtime faults.
 *    star_last_error() returns the message of the last failure on the calling
 *    thread.
 *  - Row-major tensors with an explicit row stride (elements) so callers can
 *    pass slices of fused QKV projections.
 *  - Log-sum-exp values are natural logs (ln Σ exp), as PartialAttention.lse
 *    (ss/attention.py:46-64).
 */
#ifndef STAR_ATTN_H_
#define STAR_ATTN_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum star_status {
  STAR_OK = 0,
  STAR_ESHAPE = -1,
  STAR_EDOMAIN = -2,
  STAR_ECONFIG = -3,
  STAR_ECUDA = -4,
  STAR_ENOTSUP = -5
};

enum star_dtype { STAR_F32 = 0, STAR_BF16 = 1 };

/* Library identity and the last error message on this thread. */
int star_version(void);
const char* star_last_error(void);

/*
 * Counter-based splitmix64 fill: out[i] = dtype((2u-1)*scale) with
 * u = (mix64(seed + (first+i)*0x9E3779B97F4A7C15) >> 11) * 2^-53.
 * Replaces Prng._block_u64 + prng_fill (ss/numerics.py:217-263); random access,
 * so the GPU regenerates bit-identical synthetic inputs (first = 1 for a fresh
 * Prng).
 */
int star_prng_fill(void* out, int dtype, int64_t n, uint64_t seed, uint64_t first,
                   double scale, void* stream);

/*
 * Rotary embedding on adjacent pairs (2i, 2i+1) at explicit int64 positions:
 * angle = pos * theta^(-2i/d) reduced in fp64.  x, y: [rows, heads, d] with
 * row strides; y may alias x.  Replaces rope_apply (ss/numerics.py:161-180) as
 * called per head by layer_step (ss/toy_model.py:161-162).
 */
int star_rope(const void* x, void* y, int dtype, int64_t rows, int heads, int d,
              int64_t x_row_stride, int64_t y_row_stride, const int64_t* positions,
              double theta, void* stream);

/*
 * Fused phase-1 prologue: RoPE of q [rows, hq, d] and k [rows, hkv, d]
 * at int64 positions into q_out / k_out, and for every row with cache_rows[r] >= 0
 * (device int64, nullable = no cache writes) the rotated k and the raw v
 * [rows, hkv, d] (row stride kv_in_stride, shared with k) written to logical cache
 * row cache_rows[r] of the paged pool.  Replaces rope_apply on q and k
 * (ss/toy_model.py:161-162) and the own-row retention (ss/sim.py:117-118) in one pass.
 */
int star_rope_qkv(const void* q_in, const void* k_in, const void* v_in, int dtype, int64_t rows,
                  int hq, int hkv, int d, int64_t q_in_stride, int64_t kv_in_stride, void* q_out,
                  void* k_out, int64_t q_out_stride, int64_t k_out_stride,
                  const int64_t* positions, double theta, const int64_t* cache_rows,
                  void* k_pages, void* v_pages, const int32_t* page_table, int page_size,
                  void* stream);

/*
 * Decode append (replaces the per-token KVCache.append of the query host,
 * ss/blocking.py:161-170 via ss/sim.py:275-277, plus rope_apply of the new
 * rows' q and k, ss/numerics.py:161-180) for `batch` sequences of `rows` new
 * rows each: RoPE of q [batch*rows, hq, d] and k [batch*rows, hkv, d] at
 * `positions` (device int64 [batch*rows]); rotated q -> q_out; rotated k and
 * raw v written at the logical cache rows kv_len[b] + r of sequence b's pages
 * (page_table [batch, pages_per_seq]), then kv_len[b] += rows.  kv_len is a
 * DEVICE int32 [batch] counter, so a decode step that calls this is
 * graph-capturable; the caller keeps kv_len[b] + rows <= pages_per_seq *
 * page_size (the rows it reserved).
 */
int star_kv_append(const void* q_in, const void* k_in, const void* v_in, int dtype, int batch,
                   int rows, int hq, int hkv, int d, int64_t q_in_stride, int64_t kv_in_stride,
                   void* q_out, int64_t q_out_stride, const int64_t* positions, double theta,
                   int32_t* kv_len, void* k_pages, void* v_pages, const int32_t* page_table,
                   int pages_per_seq, int page_size, const double* rope_table_cs,
                   int64_t table_pos0, int64_t table_positions, void* stream);

/*
 * Fused decode step of one layer (BF16, one new token per sequence, paged cache as
 * star_phase2_partial): q_raw [batch][hq][d] / k_new, v_new [batch][hkv][d] are the token's
 * PRE-RoPE projections (row strides q_stride / kv_stride elements), positions[batch] its
 * device positions.  Every K2 CTA rotates its q heads itself (RoPE through rope_table_cs when
 * the position is inside it, else the fp64 angle, as star_rope); with append != 0 the CTA
 * whose key range holds row kv_len[b] writes the rotated k and raw v there and K2 attends over
 * kv_len[b] + 1 rows — the append-then-attend of ss/sim.py:275-277 in ONE launch instead of
 * star_kv_append + star_phase2_partial.  kv_len is NOT advanced (call star_decode_advance
 * once per token); append == 0 rotates q only (a rank that is not the query host).
 * rope_cur_cs (nullable): double [batch][d/2][2] cos/sin at positions[b], as
 * star_decode_advance maintains it — read directly, so no load waits on the position.
 * Results are bit-identical to star_kv_append followed by star_phase2_partial.
 */
int star_phase2_decode(const void* q_raw, const void* k_new, const void* v_new, int append,
                       int64_t q_stride, int64_t kv_stride, const int64_t* positions, double theta,
                       const double* rope_table_cs, int64_t table_pos0, int64_t table_positions,
                       const double* rope_cur_cs, int batch, int hq, int hkv, int d, const void* k_pages, const void* v_pages,
                       int64_t num_pages, const int32_t* page_table, int pages_per_seq,
                       int page_size, const int32_t* kv_len, int64_t max_kv_len, float* out,
                       float* lse, int n_splits, void* workspace, void* stream);

/* star_phase2_decode with the fused peer exchange of star_phase2_exchange (C1 fused). */
int star_phase2_decode_exchange(const void* q_raw, const void* k_new, const void* v_new,
                                int append, int64_t q_stride, int64_t kv_stride,
                                const int64_t* positions, double theta,
                                const double* rope_table_cs, int64_t table_pos0,
                                int64_t table_positions, const double* rope_cur_cs, int batch,
                                int hq, int hkv, int d,
                                const void* k_pages, const void* v_pages, int64_t num_pages,
                                const int32_t* page_table, int pages_per_seq, int page_size,
                                const int32_t* kv_len, int64_t max_kv_len, float* out, float* lse,
                                int n_splits, void* workspace, void* const* boxes, int world,
                                int64_t cap_rows, int cap_groups, int rank, void* stream);

/*
 * End of a fused decode token: kv_len[0..n_counters) += add, positions[0..n_positions) += inc,
 * then (cur_cs != NULL) cur_cs[b] = cos/sin of the new positions[b] (d/2 pairs; from the
 * table when inside it, else the fp64 angle) for the next token's star_phase2_decode.
 * inc = add = 0 only fills cur_cs (before the first token).
 */
int star_decode_advance(int32_t* kv_len, int n_counters, int add, int64_t* positions,
                        int n_positions, int inc, double* cur_cs, const double* rope_table_cs,
                        int64_t table_pos0, int64_t table_positions, int d, double theta,
                        void* stream);

/*
 * RoPE cos/sin table for positions [pos0, pos0 + n_positions): cs[(p*d/2 + i)*2 + {0,1}] =
 * {cos, sin} of (pos0 + p) * theta^(-2i/d), fp64, the same expression star_rope evaluates
 * (ss/numerics.py:173-176), so star_kv_append through the table (rope_table_cs != NULL and
 * the position inside [table_pos0, table_pos0 + table_positions)) is bit-identical to
 * forming the angle in place.  A decoder builds it once for its token budget.
 */
int star_rope_table(double* cs, int64_t pos0, int64_t n_positions, int d, double theta,
                    void* stream);

/*
 * Phase 1 (K1): causal self-attention over one or more anchor-augmented
 * blocks concatenated along rows.  Segment s covers rows
 * [seg_start[s], seg_start[s+1]) of q/k/v/out (seg_start: HOST array of
 * n_seg+1 offsets); row i of a segment sees keys j <= i of the same segment.
 * GQA: q head h reads kv head h / (hq/hkv).  q [rows, hq, d], k/v [rows, hkv, d],
 * out [rows, hq, d] in out_dtype (bf16 or f32), lse fp32 [hq, rows] (nullable).
 * bf16 uses the tcgen05/TMEM/TMA kernel (d in {64,128}); f32 uses the fp32
 * check-mode kernel.  Replaces causal_attention (ss/attention.py:109-122) as
 * driven per (block, layer, head) by _encode_block_channels (ss/sim.py:108-123).
 * dedup_anchor_rows (anchor dedup): when > 0 the caller guarantees
 * that rows [0, n) of every segment s >= 1 equal rows [0, n) of segment 0 (q, k
 * and v — first-block anchor content AND positions); the tensor-core path then
 * computes those rows once, in segment 0, and writes them to every segment
 * (bit-identical outputs, ~a(a+1)/2 fewer score pairs per block).  0 = off.
 */
int star_phase1_fwd(const void* q, const void* k, const void* v, int dtype, int n_seg,
                    const int64_t* seg_start, int hq, int hkv, int d, int64_t q_row_stride,
                    int64_t kv_row_stride, void* out, int out_dtype, int64_t out_row_stride,
                    float* lse, int64_t dedup_anchor_rows, void* stream);

/*
 * Check mode of star_phase1_fwd (same arguments, no dedup): every dtype runs the CUDA-core
 * kernel with fp32 scores, softmax and accumulation (ss/attention.py:109-122 at the
 * reference's default fp32 precision) — the yardstick the bf16 tensor-core K1 is compared
 * against, row for row, at full size (tests/test_fullsize_gpu.py).
 */
int star_phase1_fwd_check(const void* q, const void* k, const void* v, int dtype, int n_seg,
                          const int64_t* seg_start, int hq, int hkv, int d,
                          int64_t q_row_stride, int64_t kv_row_stride, void* out, int out_dtype,
                          int64_t out_row_stride, float* lse, void* stream);

/* Phase 1 over a query-row range of ONE segment: causal attention of query rows
 * [q_begin, q_end) against keys [0, q_end) of the segment whose row 0 is at q/k/v/out.
 * Equals causal_attention(q[q_begin:q_end], k[:q_end], v[:q_end], q_offset=q_begin)
 * (ss/attention.py:109-122, the q_offset form); out rows [q_begin, q_end) and lse
 * columns [q_begin, q_end) of [hq, lse_stride] are written, nothing else.  The bf16
 * tensor-core path needs q_begin % 128 == 0 (whole q tiles).  Lets a host pipeline
 * start a block's encode before all of it has arrived and ship its first rows while
 * the rest computes. */
int star_phase1_fwd_range(const void* q, const void* k, const void* v, int dtype, int64_t q_begin,
                          int64_t q_end, int hq, int hkv, int d, int64_t q_row_stride,
                          int64_t kv_row_stride, void* out, int out_dtype, int64_t out_row_stride,
                          float* lse, int64_t lse_stride, void* stream);

/*
 * Dense masked attention, one segment: q rows [lq] at absolute offset
 * q_offset against k/v rows [lk].  mask: 0 = "full", 1 = "causal"
 * (row i sees keys j <= q_offset + i).  out [lq, hq, d] (dtype of q),
 * lse fp32 [hq, lq] (nullable).  Rows with no visible key -> STAR_EDOMAIN
 * (checked on host from the shapes).  Replaces causal_attention /
 * partial_attention(mask="full"|"causal") (ss/attention.py:109-151).
 */
int star_attention_dense(const void* q, const void* k, const void* v, int dtype, int64_t lq,
                         int64_t lk, int64_t q_offset, int mask, int hq, int hkv, int d,
                         int64_t q_row_stride, int64_t kv_row_stride, void* out,
                         int64_t out_row_stride, float* lse, void* stream);

/*
 * Paged KV cache write: rows [0, n_rows) of k_src/v_src ([n_rows, hkv, d],
 * row stride src_row_stride) land at logical cache rows
 * [dst_row0, dst_row0 + n_rows) of one sequence.  Pool layout:
 * k_pages/v_pages [num_pages, hkv, page_size, d]; logical row r lives in
 * physical page page_table[r / page_size], slot r % page_size.
 * Replaces the own-row retention kh[lo:], vh[lo:] (ss/sim.py:117-118,
 * ss/blocking.py:262-265) and KVCache.append (ss/blocking.py:161-170).
 */
int star_kv_write(const void* k_src, const void* v_src, int dtype, int64_t n_rows, int hkv,
                  int d, int64_t src_row_stride, void* k_pages, void* v_pages,
                  const int32_t* page_table, int page_size, int64_t dst_row0, void* stream);

/* Inverse of star_kv_write (materialise a sequence's rows densely; for checks). */
int star_kv_read(const void* k_pages, const void* v_pages, int dtype, const int32_t* page_table,
                 int page_size, int64_t row0, int64_t n_rows, int hkv, int d, void* k_dst,
                 void* v_dst, void* stream);

/*
 * Phase 2 (K2 + intra-GPU split reduction): partial attention of q rows
 * against each sequence's local paged cache, emitting fp32 (out, lse).
 * q [batch, lq, hq, d] (dtype q_dtype, contiguous); caches in kv_dtype, pools of
 * num_pages pages; page_table [batch, pages_per_seq] int32; kv_len int32[batch] (device).
 * own_tail in {0, lq}: when lq, the last lq cache rows are the query's own rows
 * and q row i sees tail row c only if c <= i (the query host's keep mask,
 * ss/sim.py:195-200); otherwise every cached row is visible ("full").
 * out fp32 [batch, lq, hq, d], lse fp32 [batch, lq, hq]; a sequence with
 * kv_len == 0 yields lse = -inf and out = 0 (the caller skips it, as
 * _gather_merge skips empty hosts, ss/sim.py:193-194).
 * bf16 with d in {64,128} runs the TMA + tensor-core (mma.sync) kernel; f32 runs the
 * fp32 check-mode kernel.
 * n_splits: key-range splits per (sequence, kv head) (0 = auto); the split
 * partials are merged on device in ascending order (bf16: inside the kernel, by the
 * last CTA of each (sequence, kv head) to finish).  workspace must hold
 * star_phase2_workspace_bytes(...) bytes (may be NULL when it returns 0) and be
 * zero-initialised before its first use; calls leave it re-armed for reuse.
 * Replaces partial_attention(q, K_h, V_h, "full"|keep) (ss/attention.py:125-151)
 * inside _gather_merge (ss/sim.py:178-213).
 */
int64_t star_phase2_workspace_bytes(int batch, int lq, int hq, int d, int n_splits);
int star_phase2_auto_splits(int batch, int hkv, int64_t max_kv_len, int page_size);
int star_phase2_partial(const void* q, int q_dtype, int batch, int lq, int hq, int hkv, int d,
                        const void* k_pages, const void* v_pages, int kv_dtype, int64_t num_pages,
                        const int32_t* page_table, int pages_per_seq, int page_size,
                        const int32_t* kv_len, int64_t max_kv_len, int own_tail, float* out,
                        float* lse, int n_splits, void* workspace, void* stream);

/*
 * K3: log-domain merge of n_parts partials in ascending part order:
 * s = logaddexp-reduce(lse_p), out = Σ_p exp(lse_p - s) out_p.  outs fp32
 * [n_parts, rows, d], lses fp32 [n_parts, rows]; parts with lse = -inf are
 * skipped.  out may be f32 or bf16 (out_dtype).  Replaces merge_partials
 * (ss/attention.py:154-173).
 */
int star_merge(const float* outs, const float* lses, int n_parts, int64_t rows, int d,
               void* out, int out_dtype, float* lse, void* stream);

/* K3 over strided parts: part p's out rows start at outs + p * out_part_stride and its lse
 * at lses + p * lse_part_stride (elements).  Used on the all-gathered packed partials
 * [out rows*d | lse rows] of every rank, so one collective carries both (see dist.py).
 * Replaces merge_partials (ss/attention.py:154-173) as _gather_merge calls it over the
 * hosts in ascending order (ss/sim.py:190-213). */
int star_merge_strided(const float* outs, int64_t out_part_stride, const float* lses,
                       int64_t lse_part_stride, int n_parts, int64_t rows, int d, void* out,
                       int out_dtype, float* lse, void* stream);

/*
 * Peer exchange of phase-2 partials (C1 fused over NVLink / NVSwitch peer memory).
 * Replaces the gather of every host's (out, lse) to the query host and its ordered merge
 * (_gather_merge, ss/sim.py:178-213; merge_partials, ss/attention.py:154-173).  Every rank
 * owns one "box" of star_exchange_box_bytes(world, cap_rows, cap_groups, d) bytes of device
 * memory, zeroed once, and maps every other rank's box with star_ipc_open_handle (all ranks
 * on one node).  cap_rows >= batch * lq * hq and cap_groups >= batch * hkv of every call;
 * every call passes the same (world, cap_rows, cap_groups).  One exchange (one layer of one
 * phase-2 forward), issued by every rank in the same order:
 *   1. every rank delivers its partial to slot `rank` of every box: star_phase2_partial_push
 *      (the K2 epilogue stores the final partial of each (sequence, kv head) straight into
 *      the boxes and releases a flag per group at system scope), or star_exchange_push for a
 *      partial already in device memory (e.g. an empty cache: out = 0, lse = -inf);
 *   2. star_exchange_merge waits for the flags of all ranks in the rank's own box
 *      (system-scope acquire; a rank that never delivers traps the kernel after
 *      STAR_EXCHANGE_TIMEOUT_S, default 30 s) and merges the slots in ascending rank order
 *      into out (f32 or bf16) / lse (nullable).
 * Exchanges are numbered on the device (a counter in the box header, advanced by step 2),
 * so a stream-captured CUDA graph of a decode step replays correctly; consecutive
 * exchanges alternate between two halves of the box, so a rank may run one ahead.
 * boxes: HOST array of `world` device pointers (boxes[rank] = this rank's own box);
 * world <= 8.  Shapes as star_phase2_partial.  The IPC calls wrap cudaIpcGetMemHandle /
 * cudaIpcOpenMemHandle for a pointer anywhere inside an allocation (offset = its distance
 * from the allocation base).
 */
#define STAR_IPC_HANDLE_BYTES 64
int64_t star_exchange_box_bytes(int world, int64_t cap_rows, int cap_groups, int d);
int star_ipc_get_handle(const void* dev_ptr, void* handle, int64_t* offset);
int star_ipc_open_handle(const void* handle, int64_t offset, void** dev_ptr);
int star_ipc_close_handle(void* dev_ptr, int64_t offset);
int star_phase2_partial_push(const void* q, int q_dtype, int batch, int lq, int hq, int hkv, int d,
                             const void* k_pages, const void* v_pages, int kv_dtype,
                             int64_t num_pages, const int32_t* page_table, int pages_per_seq,
                             int page_size, const int32_t* kv_len, int64_t max_kv_len,
                             int own_tail, float* out, float* lse, int n_splits, void* workspace,
                             void* const* boxes, int world, int64_t cap_rows, int cap_groups,
                             int rank, void* stream);
/* The whole exchange of one layer in one call: partial attention of q over this rank's
 * cache, delivered to every box, merged over all ranks into out fp32 [batch, lq, hq, d] /
 * lse [batch, lq, hq].  When the K2 grid is co-resident (word-mode split fix-up) ONE kernel
 * does all of it — each CTA pushes its slice of the partial and folds the peers' words of
 * the same slice; otherwise K2 pushes and K3x merges (two launches). */
int star_phase2_exchange(const void* q, int q_dtype, int batch, int lq, int hq, int hkv, int d,
                         const void* k_pages, const void* v_pages, int kv_dtype, int64_t num_pages,
                         const int32_t* page_table, int pages_per_seq, int page_size,
                         const int32_t* kv_len, int64_t max_kv_len, int own_tail, float* out,
                         float* lse, int n_splits, void* workspace, void* const* boxes, int world,
                         int64_t cap_rows, int cap_groups, int rank, void* stream);
int star_exchange_push(const float* out, const float* lse, int batch, int lq, int hq, int hkv,
                       int d, void* const* boxes, int world, int64_t cap_rows, int cap_groups,
                       int rank, void* stream);
int star_exchange_merge(void* box, int world, int64_t cap_rows, int cap_groups, int batch, int lq,
                        int hq, int hkv, int d, void* out, int out_dtype, float* lse,
                        void* stream);

/* Debug/validation: C[128x128] fp32 = A[128xK] * B^T via one tcgen05 CTA.
 * mode bit 0: B given MN-major as [K x 128]; bit 1: A staged through TMEM.
 * K multiple of 64. */
int star_debug_umma_gemm(const void* a, const void* b, float* c, int K, int mode, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* STAR_ATTN_H_ */
