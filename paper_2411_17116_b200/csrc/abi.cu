// extern "C" entry points declared in include/star_attn.h: argument checks that
// mirror the reference's ShapeError / DomainError / ConfigError conditions,
// then dispatch to the sm_100a kernels.
#include <stdarg.h>
#include <algorithm>
#include <stdio.h>
#include <stdlib.h>

#include "common.cuh"
#include "exchange.cuh"

namespace star {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
  }
  return n;
}

// kernels (defined in the other translation units)
int prng_fill(void*, int, int64_t, uint64_t, uint64_t, double, cudaStream_t);
int rope(const void*, void*, int, int64_t, int, int, int64_t, int64_t, const int64_t*, double,
         cudaStream_t);
int kv_write(const void*, const void*, int, int64_t, int, int, int64_t, void*, void*,
             const int32_t*, int, int64_t, cudaStream_t);
int rope_qkv(const void*, const void*, const void*, int, int64_t, int, int, int, int64_t, int64_t,
             void*, void*, int64_t, int64_t, const int64_t*, double, const int64_t*, void*, void*,
             const int32_t*, int, cudaStream_t);
int kv_append(const void*, const void*, const void*, int, int, int, int, int, int, int64_t,
              int64_t, void*, int64_t, const int64_t*, double, int32_t*, void*, void*,
              const int32_t*, int, int, const void*, int64_t, int64_t, cudaStream_t);
int rope_table(void*, int64_t, int64_t, int, double, cudaStream_t);
int kv_read(const void*, const void*, int, const int32_t*, int, int64_t, int64_t, int, int, void*,
            void*, cudaStream_t);
int attention_simt(const void*, const void*, const void*, int, SegTable&, int, int, int, int64_t,
                   int64_t, int, void*, int, int64_t, float*, int64_t, cudaStream_t);
int phase1_tc(const void*, const void*, const void*, SegTable&, int, int, int, int64_t, int64_t,
              int64_t, void*, int, int64_t, float*, int64_t, cudaStream_t);
int64_t phase2_workspace_bytes(int, int, int, int, int);
int phase2_auto_splits(int, int, int64_t, int);
int phase2_partial(const void*, int, int, int, int, int, int, const void*, const void*, int,
                   int64_t, const int32_t*, int, int, const int32_t*, int64_t, int, float*, float*,
                   int, void*, const PeerPush*, int*, cudaStream_t,
                   const DecodeAppend* dap = nullptr);
int decode_advance(int32_t*, int, int, int64_t*, int, int, void*, const void*, int64_t, int64_t,
                   int, double, cudaStream_t);
int check_exchange(const ExchangeLayout&, void* const*, int, int64_t, int);
PeerPush make_push(const ExchangeLayout&, void* const*, int);
int exchange_push(const float*, const float*, int, int, int, int, int, void* const*,
                  const ExchangeLayout&, int, cudaStream_t);
int exchange_merge(void*, const ExchangeLayout&, int, int, int, int, int, void*, int, float*,
                   cudaStream_t);
int ipc_get_handle(const void*, void*, int64_t*);
int ipc_open_handle(const void*, int64_t, void**);
int ipc_close_handle(void*, int64_t);
int merge(const float*, const float*, int, int64_t, int, void*, int, float*, cudaStream_t);
int merge_strided(const float*, int64_t, const float*, int64_t, int, int64_t, int, void*, int, float*,
                  cudaStream_t);
int debug_umma_gemm(const void*, const void*, float*, int, int, cudaStream_t);

static int check_heads(int hq, int hkv, int d) {
  if (hq < 1 || hkv < 1) return fail(STAR_ESHAPE, "head counts must be >= 1 (hq=%d hkv=%d)", hq, hkv);
  if (hq % hkv) return fail(STAR_ESHAPE, "hq (%d) must be a multiple of hkv (%d)", hq, hkv);
  if (d < 1) return fail(STAR_ECONFIG, "head_dim must be >= 1, got %d", d);
  return STAR_OK;
}

}  // namespace star

using namespace star;

extern "C" {

int star_version(void) { return 1; }

const char* star_last_error(void) { return g_err; }

int star_prng_fill(void* out, int dtype, int64_t n, uint64_t seed, uint64_t first, double scale,
                   void* stream) {
  return prng_fill(out, dtype, n, seed, first, scale, (cudaStream_t)stream);
}

int star_rope(const void* x, void* y, int dtype, int64_t rows, int heads, int d,
              int64_t x_row_stride, int64_t y_row_stride, const int64_t* positions, double theta,
              void* stream) {
  return rope(x, y, dtype, rows, heads, d, x_row_stride, y_row_stride, positions, theta,
              (cudaStream_t)stream);
}

int star_rope_qkv(const void* q_in, const void* k_in, const void* v_in, int dtype, int64_t rows,
                  int hq, int hkv, int d, int64_t q_in_stride, int64_t kv_in_stride, void* q_out,
                  void* k_out, int64_t q_out_stride, int64_t k_out_stride,
                  const int64_t* positions, double theta, const int64_t* cache_rows,
                  void* k_pages, void* v_pages, const int32_t* page_table, int page_size,
                  void* stream) {
  return rope_qkv(q_in, k_in, v_in, dtype, rows, hq, hkv, d, q_in_stride, kv_in_stride, q_out,
                  k_out, q_out_stride, k_out_stride, positions, theta, cache_rows, k_pages,
                  v_pages, page_table, page_size, (cudaStream_t)stream);
}

int star_kv_append(const void* q_in, const void* k_in, const void* v_in, int dtype, int batch,
                   int rows, int hq, int hkv, int d, int64_t q_in_stride, int64_t kv_in_stride,
                   void* q_out, int64_t q_out_stride, const int64_t* positions, double theta,
                   int32_t* kv_len, void* k_pages, void* v_pages, const int32_t* page_table,
                   int pages_per_seq, int page_size, const double* rope_table_cs,
                   int64_t table_pos0, int64_t table_positions, void* stream) {
  int rc = check_heads(hq, hkv, d);
  if (rc) return rc;
  return kv_append(q_in, k_in, v_in, dtype, batch, rows, hq, hkv, d, q_in_stride, kv_in_stride,
                   q_out, q_out_stride, positions, theta, kv_len, k_pages, v_pages, page_table,
                   pages_per_seq, page_size, rope_table_cs, table_pos0, table_positions,
                   (cudaStream_t)stream);
}

int star_rope_table(double* cs, int64_t pos0, int64_t n_positions, int d, double theta,
                    void* stream) {
  if (cs == nullptr && n_positions > 0) return fail(STAR_ESHAPE, "rope_table: out is NULL");
  return rope_table(cs, pos0, n_positions, d, theta, (cudaStream_t)stream);
}

static int phase1_impl(const void* q, const void* k, const void* v, int dtype, int n_seg,
                       const int64_t* seg_start, int hq, int hkv, int d, int64_t q_row_stride,
                       int64_t kv_row_stride, void* out, int out_dtype, int64_t out_row_stride,
                       float* lse, int64_t dedup_anchor_rows, bool check_mode, void* stream) {
  int rc = check_heads(hq, hkv, d);
  if (out_dtype != STAR_F32 && out_dtype != STAR_BF16)
    return fail(STAR_ECONFIG, "phase1: unknown out dtype %d", out_dtype);
  if (rc) return rc;
  if (n_seg < 0) return fail(STAR_ECONFIG, "phase1: %d segments", n_seg);
  if (n_seg == 0) return STAR_OK;
  if (seg_start == nullptr) return fail(STAR_ESHAPE, "phase1: seg_start is NULL");
  if (out == nullptr) return fail(STAR_ESHAPE, "phase1: out is NULL");
  if (q_row_stride < (int64_t)hq * d || kv_row_stride < (int64_t)hkv * d ||
      out_row_stride < (int64_t)hq * d)
    return fail(STAR_ESHAPE, "phase1: row stride smaller than heads*d");
  if (dedup_anchor_rows < 0) return fail(STAR_ECONFIG, "phase1: negative dedup_anchor_rows");
  for (int i = 0; i < n_seg; ++i) {
    int64_t a = seg_start[i], b = seg_start[i + 1];
    if (a < 0 || b < a) return fail(STAR_ESHAPE, "phase1: segment %d has bounds [%lld, %lld)", i,
                                    (long long)a, (long long)b);
    if (b - a > (1ll << 30)) return fail(STAR_ENOTSUP, "phase1: segment longer than 2^30 rows");
    if (dedup_anchor_rows > 0 && b - a < dedup_anchor_rows)
      return fail(STAR_ESHAPE, "phase1: segment %d shorter than the %lld deduplicated anchor rows",
                  i, (long long)dedup_anchor_rows);
  }
  const int64_t total = seg_start[n_seg];
  const int64_t lse_stride = total;
  cudaStream_t s = (cudaStream_t)stream;
  const bool tc = !check_mode && dtype == STAR_BF16 && (d == 64 || d == 128);
  if (tc && total >= (1ll << 31)) return fail(STAR_ENOTSUP, "phase1: more than 2^31 rows per call");
  // The segment table travels in the kernel parameter block (kMaxSegments entries), so a
  // context with more blocks runs as several stream-ordered launches of up to kMaxSegments
  // segments each.  Rows stay absolute (same tensors, same tensor maps).  Anchor dedup fans
  // segment 0's rows out inside its own launch; later launches encode their anchor rows
  // (identical values, DESIGN §3 f3).
  for (int c0 = 0; c0 < n_seg; c0 += kMaxSegments) {
    const int cn = std::min(kMaxSegments, n_seg - c0);
    SegTable segs;
    segs.n = cn;
    for (int i = 0; i < cn; ++i) {
      const int64_t a = seg_start[c0 + i], b = seg_start[c0 + i + 1];
      segs.q_row0[i] = a;
      segs.k_row0[i] = a;
      segs.lq[i] = (int32_t)(b - a);
      segs.lk[i] = (int32_t)(b - a);
      segs.q_offset[i] = 0;
    }
    if (tc) {
      // only whole 128-row tiles are deduplicated (the tensor-core kernel's q tile)
      segs.dedup_tiles = c0 == 0 ? (int32_t)(dedup_anchor_rows / 128) : 0;
      rc = phase1_tc(q, k, v, segs, hq, hkv, d, total, q_row_stride, kv_row_stride, out,
                     out_dtype == STAR_F32, out_row_stride, lse, lse_stride, s);
    } else {
      rc = attention_simt(q, k, v, dtype, segs, hq, hkv, d, q_row_stride, kv_row_stride, 1, out,
                          out_dtype, out_row_stride, lse, lse_stride, s);
    }
    if (rc) return rc;
  }
  return STAR_OK;
}

int star_phase1_fwd(const void* q, const void* k, const void* v, int dtype, int n_seg,
                    const int64_t* seg_start, int hq, int hkv, int d, int64_t q_row_stride,
                    int64_t kv_row_stride, void* out, int out_dtype, int64_t out_row_stride,
                    float* lse, int64_t dedup_anchor_rows, void* stream) {
  return phase1_impl(q, k, v, dtype, n_seg, seg_start, hq, hkv, d, q_row_stride, kv_row_stride,
                     out, out_dtype, out_row_stride, lse, dedup_anchor_rows, false, stream);
}

int star_phase1_fwd_check(const void* q, const void* k, const void* v, int dtype, int n_seg,
                          const int64_t* seg_start, int hq, int hkv, int d,
                          int64_t q_row_stride, int64_t kv_row_stride, void* out, int out_dtype,
                          int64_t out_row_stride, float* lse, void* stream) {
  return phase1_impl(q, k, v, dtype, n_seg, seg_start, hq, hkv, d, q_row_stride, kv_row_stride,
                     out, out_dtype, out_row_stride, lse, 0, true, stream);
}

int star_phase1_fwd_range(const void* q, const void* k, const void* v, int dtype, int64_t q_begin,
                          int64_t q_end, int hq, int hkv, int d, int64_t q_row_stride,
                          int64_t kv_row_stride, void* out, int out_dtype, int64_t out_row_stride,
                          float* lse, int64_t lse_stride, void* stream) {
  int rc = check_heads(hq, hkv, d);
  if (rc) return rc;
  if (out_dtype != STAR_F32 && out_dtype != STAR_BF16)
    return fail(STAR_ECONFIG, "phase1: unknown out dtype %d", out_dtype);
  if (q_begin < 0 || q_end < q_begin)
    return fail(STAR_ESHAPE, "phase1 range: bad query rows [%lld, %lld)", (long long)q_begin,
                (long long)q_end);
  if (q_end > (1ll << 30)) return fail(STAR_ENOTSUP, "phase1 range: more than 2^30 rows");
  if (out == nullptr) return fail(STAR_ESHAPE, "phase1: out is NULL");
  if (q_row_stride < (int64_t)hq * d || kv_row_stride < (int64_t)hkv * d ||
      out_row_stride < (int64_t)hq * d)
    return fail(STAR_ESHAPE, "phase1: row stride smaller than heads*d");
  if (lse != nullptr && lse_stride < q_end) return fail(STAR_ESHAPE, "phase1: lse stride < rows");
  if (q_end == q_begin) return STAR_OK;
  SegTable segs;
  segs.n = 1;
  segs.q_row0[0] = 0;
  segs.k_row0[0] = 0;
  segs.lq[0] = (int32_t)q_end;
  segs.lk[0] = (int32_t)q_end;
  segs.q_offset[0] = 0;
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == STAR_BF16 && (d == 64 || d == 128)) {
    // the tensor-core kernel launches whole 128-row q tiles
    if (q_begin % 128)
      return fail(STAR_ECONFIG, "phase1 range: q_begin %lld is not a multiple of 128",
                  (long long)q_begin);
    segs.tile_lo[0] = (int32_t)(q_begin / 128);
    return phase1_tc(q, k, v, segs, hq, hkv, d, q_end, q_row_stride, kv_row_stride, out,
                     out_dtype == STAR_F32, out_row_stride, lse, lse_stride, s);
  }
  // CUDA-core path: rows [q_begin, q_end) as queries at offset q_begin
  const size_t esz = dtype == STAR_BF16 ? 2 : 4, osz = out_dtype == STAR_BF16 ? 2 : 4;
  segs.lq[0] = (int32_t)(q_end - q_begin);
  segs.q_offset[0] = (int32_t)q_begin;
  return attention_simt(static_cast<const char*>(q) + q_begin * q_row_stride * esz, k, v, dtype, segs,
                        hq, hkv, d, q_row_stride, kv_row_stride, 1,
                        static_cast<char*>(out) + q_begin * out_row_stride * osz, out_dtype,
                        out_row_stride, lse == nullptr ? nullptr : lse + q_begin, lse_stride, s);
}

int star_attention_dense(const void* q, const void* k, const void* v, int dtype, int64_t lq,
                         int64_t lk, int64_t q_offset, int mask, int hq, int hkv, int d,
                         int64_t q_row_stride, int64_t kv_row_stride, void* out,
                         int64_t out_row_stride, float* lse, void* stream) {
  int rc = check_heads(hq, hkv, d);
  if (rc) return rc;
  if (mask != 0 && mask != 1) return fail(STAR_ECONFIG, "unknown mask kind %d", mask);
  if (lq < 0 || lk < 0) return fail(STAR_ESHAPE, "negative row counts");
  if (lq >= (1ll << 31) || lk >= (1ll << 31))
    return fail(STAR_ENOTSUP, "dense attention: more than 2^31 rows");
  if (mask == 1 && q_offset + lq > lk)
    return fail(STAR_ESHAPE, "q rows [%lld, %lld) extend past %lld keys", (long long)q_offset,
                (long long)(q_offset + lq), (long long)lk);
  if (lk == 0 && lq > 0) return fail(STAR_EDOMAIN, "partial attention over an empty key set");
  if (mask == 1 && q_offset < 0) return fail(STAR_EDOMAIN, "q_offset %lld leaves a query row with no keys",
                                             (long long)q_offset);
  if (lq == 0) return STAR_OK;
  SegTable segs;
  segs.n = 1;
  segs.q_row0[0] = 0;
  segs.k_row0[0] = 0;
  segs.lq[0] = (int32_t)lq;
  segs.lk[0] = (int32_t)lk;
  segs.q_offset[0] = (int32_t)q_offset;
  return attention_simt(q, k, v, dtype, segs, hq, hkv, d, q_row_stride, kv_row_stride, mask, out,
                        dtype, out_row_stride, lse, lq, (cudaStream_t)stream);
}

int star_kv_write(const void* k_src, const void* v_src, int dtype, int64_t n_rows, int hkv, int d,
                  int64_t src_row_stride, void* k_pages, void* v_pages, const int32_t* page_table,
                  int page_size, int64_t dst_row0, void* stream) {
  return kv_write(k_src, v_src, dtype, n_rows, hkv, d, src_row_stride, k_pages, v_pages,
                  page_table, page_size, dst_row0, (cudaStream_t)stream);
}

int star_kv_read(const void* k_pages, const void* v_pages, int dtype, const int32_t* page_table,
                 int page_size, int64_t row0, int64_t n_rows, int hkv, int d, void* k_dst,
                 void* v_dst, void* stream) {
  return kv_read(k_pages, v_pages, dtype, page_table, page_size, row0, n_rows, hkv, d, k_dst, v_dst,
                 (cudaStream_t)stream);
}

int64_t star_phase2_workspace_bytes(int batch, int lq, int hq, int d, int n_splits) {
  return phase2_workspace_bytes(batch, lq, hq, d, n_splits);
}

int star_phase2_auto_splits(int batch, int hkv, int64_t max_kv_len, int page_size) {
  return phase2_auto_splits(batch, hkv, max_kv_len, page_size);
}

int star_phase2_partial(const void* q, int q_dtype, int batch, int lq, int hq, int hkv, int d,
                        const void* k_pages, const void* v_pages, int kv_dtype, int64_t num_pages,
                        const int32_t* page_table, int pages_per_seq, int page_size,
                        const int32_t* kv_len, int64_t max_kv_len, int own_tail, float* out,
                        float* lse, int n_splits, void* workspace, void* stream) {
  int rc = check_heads(hq, hkv, d);
  if (rc) return rc;
  return phase2_partial(q, q_dtype, batch, lq, hq, hkv, d, k_pages, v_pages, kv_dtype, num_pages,
                        page_table,
                        pages_per_seq, page_size, kv_len, max_kv_len, own_tail, out, lse, n_splits,
                        workspace, nullptr, nullptr, (cudaStream_t)stream);
}

static DecodeAppend make_decode_append(const void* q_raw, const void* k_new, const void* v_new,
                                       int64_t q_stride, int64_t kv_stride, const int64_t* positions,
                                       const double* rope_table_cs, int64_t table_pos0,
                                       int64_t table_positions, double theta, int append,
                                       const double* cur_cs) {
  DecodeAppend ap{};
  ap.cur_cs = cur_cs;
  ap.q_raw = q_raw;
  ap.k_new = k_new;
  ap.v_new = v_new;
  ap.q_rs = q_stride;
  ap.kv_rs = kv_stride;
  ap.pos = positions;
  ap.rtab = rope_table_cs;
  ap.rtab_pos0 = table_pos0;
  ap.rtab_n = rope_table_cs != nullptr ? table_positions : 0;
  ap.theta = theta;
  ap.on = 1;
  ap.add = append ? 1 : 0;
  return ap;
}

static int check_decode_args(const void* q_raw, const void* k_new, const void* v_new, int append,
                             const int64_t* positions, int hq, int hkv, int d, int64_t q_stride,
                             int64_t kv_stride, double theta) {
  if (q_raw == nullptr || positions == nullptr) return fail(STAR_ESHAPE, "phase2 decode: NULL q / positions");
  if (append && (k_new == nullptr || v_new == nullptr))
    return fail(STAR_ESHAPE, "phase2 decode: append needs the new k / v rows");
  if (q_stride < (int64_t)hq * d || (append && kv_stride < (int64_t)hkv * d))
    return fail(STAR_ESHAPE, "phase2 decode: row stride smaller than heads*d");
  if ((q_stride | kv_stride) & 1) return fail(STAR_ECONFIG, "phase2 decode: odd row strides");
  if (!(theta > 0)) return fail(STAR_ECONFIG, "rope theta must be positive, got %g", theta);
  return STAR_OK;
}

int star_phase2_decode(const void* q_raw, const void* k_new, const void* v_new, int append,
                       int64_t q_stride, int64_t kv_stride, const int64_t* positions, double theta,
                       const double* rope_table_cs, int64_t table_pos0, int64_t table_positions,
                       const double* rope_cur_cs, int batch, int hq, int hkv, int d, const void* k_pages, const void* v_pages,
                       int64_t num_pages, const int32_t* page_table, int pages_per_seq,
                       int page_size, const int32_t* kv_len, int64_t max_kv_len, float* out,
                       float* lse, int n_splits, void* workspace, void* stream) {
  int rc = check_heads(hq, hkv, d);
  if (rc) return rc;
  if ((rc = check_decode_args(q_raw, k_new, v_new, append, positions, hq, hkv, d, q_stride,
                              kv_stride, theta)))
    return rc;
  const DecodeAppend ap = make_decode_append(q_raw, k_new, v_new, q_stride, kv_stride, positions,
                                             rope_table_cs, table_pos0, table_positions, theta,
                                             append, rope_cur_cs);
  return phase2_partial(q_raw, STAR_BF16, batch, 1, hq, hkv, d, k_pages, v_pages, STAR_BF16,
                        num_pages, page_table, pages_per_seq, page_size, kv_len, max_kv_len, 0, out,
                        lse, n_splits, workspace, nullptr, nullptr, (cudaStream_t)stream, &ap);
}

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
                                int64_t cap_rows, int cap_groups, int rank, void* stream) {
  int rc = check_heads(hq, hkv, d);
  if (rc) return rc;
  if (batch < 1) return fail(STAR_ESHAPE, "phase2: bad batch");
  if (out == nullptr || lse == nullptr) return fail(STAR_ESHAPE, "phase2 exchange: NULL out/lse");
  if ((rc = check_decode_args(q_raw, k_new, v_new, append, positions, hq, hkv, d, q_stride,
                              kv_stride, theta)))
    return rc;
  const ExchangeLayout L{world, cap_rows, d, cap_groups};
  rc = check_exchange(L, boxes, rank, (int64_t)batch * hq, batch * hkv);
  if (rc) return rc;
  PeerPush pp = make_push(L, boxes, rank);
  pp.merge = 1;
  int merged = 0;
  const DecodeAppend ap = make_decode_append(q_raw, k_new, v_new, q_stride, kv_stride, positions,
                                             rope_table_cs, table_pos0, table_positions, theta,
                                             append, rope_cur_cs);
  rc = phase2_partial(q_raw, STAR_BF16, batch, 1, hq, hkv, d, k_pages, v_pages, STAR_BF16,
                      num_pages, page_table, pages_per_seq, page_size, kv_len, max_kv_len, 0, out,
                      lse, n_splits, workspace, &pp, &merged, (cudaStream_t)stream, &ap);
  if (rc || merged) return rc;
  return exchange_merge(boxes[rank], L, batch, 1, hq, hkv, d, out, STAR_F32, lse,
                        (cudaStream_t)stream);
}

int star_decode_advance(int32_t* kv_len, int n_counters, int add, int64_t* positions,
                        int n_positions, int inc, double* cur_cs, const double* rope_table_cs,
                        int64_t table_pos0, int64_t table_positions, int d, double theta,
                        void* stream) {
  if (n_counters < 0 || n_positions < 0) return fail(STAR_ESHAPE, "decode_advance: negative count");
  if ((n_counters > 0 && kv_len == nullptr) || (n_positions > 0 && positions == nullptr))
    return fail(STAR_ESHAPE, "decode_advance: NULL counters / positions");
  return decode_advance(kv_len, n_counters, add, positions, n_positions, inc, cur_cs,
                        rope_table_cs, table_pos0, rope_table_cs ? table_positions : 0, d, theta,
                        (cudaStream_t)stream);
}

int64_t star_exchange_box_bytes(int world, int64_t cap_rows, int cap_groups, int d) {
  if (world < 1 || world > kMaxPeers || cap_rows < 1 || cap_groups < 1 || d < 1)
    return fail(STAR_ESHAPE, "exchange box: bad geometry");
  return ExchangeLayout{world, cap_rows, d, cap_groups}.bytes();
}

int star_ipc_get_handle(const void* dev_ptr, void* handle, int64_t* offset) {
  return ipc_get_handle(dev_ptr, handle, offset);
}

int star_ipc_open_handle(const void* handle, int64_t offset, void** dev_ptr) {
  return ipc_open_handle(handle, offset, dev_ptr);
}

int star_ipc_close_handle(void* dev_ptr, int64_t offset) { return ipc_close_handle(dev_ptr, offset); }

int star_phase2_partial_push(const void* q, int q_dtype, int batch, int lq, int hq, int hkv, int d,
                             const void* k_pages, const void* v_pages, int kv_dtype,
                             int64_t num_pages, const int32_t* page_table, int pages_per_seq,
                             int page_size, const int32_t* kv_len, int64_t max_kv_len,
                             int own_tail, float* out, float* lse, int n_splits, void* workspace,
                             void* const* boxes, int world, int64_t cap_rows, int cap_groups,
                             int rank, void* stream) {
  int rc = check_heads(hq, hkv, d);
  if (rc) return rc;
  if (batch < 1 || lq < 1) return fail(STAR_ESHAPE, "phase2: bad batch/lq");
  const ExchangeLayout L{world, cap_rows, d, cap_groups};
  rc = check_exchange(L, boxes, rank, (int64_t)batch * lq * hq, batch * hkv);
  if (rc) return rc;
  const PeerPush pp = make_push(L, boxes, rank);
  return phase2_partial(q, q_dtype, batch, lq, hq, hkv, d, k_pages, v_pages, kv_dtype, num_pages,
                        page_table, pages_per_seq, page_size, kv_len, max_kv_len, own_tail, out,
                        lse, n_splits, workspace, &pp, nullptr, (cudaStream_t)stream);
}

int star_phase2_exchange(const void* q, int q_dtype, int batch, int lq, int hq, int hkv, int d,
                         const void* k_pages, const void* v_pages, int kv_dtype, int64_t num_pages,
                         const int32_t* page_table, int pages_per_seq, int page_size,
                         const int32_t* kv_len, int64_t max_kv_len, int own_tail, float* out,
                         float* lse, int n_splits, void* workspace, void* const* boxes, int world,
                         int64_t cap_rows, int cap_groups, int rank, void* stream) {
  int rc = check_heads(hq, hkv, d);
  if (rc) return rc;
  if (batch < 1 || lq < 1) return fail(STAR_ESHAPE, "phase2: bad batch/lq");
  if (out == nullptr || lse == nullptr) return fail(STAR_ESHAPE, "phase2 exchange: NULL out/lse");
  const ExchangeLayout L{world, cap_rows, d, cap_groups};
  rc = check_exchange(L, boxes, rank, (int64_t)batch * lq * hq, batch * hkv);
  if (rc) return rc;
  PeerPush pp = make_push(L, boxes, rank);
  pp.merge = 1;
  int merged = 0;
  // the partial goes to the boxes; out / lse receive the merged result (from K2 itself when
  // its grid is co-resident, else from K3x)
  rc = phase2_partial(q, q_dtype, batch, lq, hq, hkv, d, k_pages, v_pages, kv_dtype, num_pages,
                      page_table, pages_per_seq, page_size, kv_len, max_kv_len, own_tail, out, lse,
                      n_splits, workspace, &pp, &merged, (cudaStream_t)stream);
  if (rc || merged) return rc;
  return exchange_merge(boxes[rank], L, batch, lq, hq, hkv, d, out, STAR_F32, lse,
                        (cudaStream_t)stream);
}

int star_exchange_push(const float* out, const float* lse, int batch, int lq, int hq, int hkv,
                       int d, void* const* boxes, int world, int64_t cap_rows, int cap_groups,
                       int rank, void* stream) {
  return exchange_push(out, lse, batch, lq, hq, hkv, d, boxes,
                       ExchangeLayout{world, cap_rows, d, cap_groups}, rank, (cudaStream_t)stream);
}

int star_exchange_merge(void* box, int world, int64_t cap_rows, int cap_groups, int batch, int lq,
                        int hq, int hkv, int d, void* out, int out_dtype, float* lse,
                        void* stream) {
  return exchange_merge(box, ExchangeLayout{world, cap_rows, d, cap_groups}, batch, lq, hq, hkv, d,
                        out, out_dtype, lse, (cudaStream_t)stream);
}

int star_merge(const float* outs, const float* lses, int n_parts, int64_t rows, int d, void* out,
               int out_dtype, float* lse, void* stream) {
  return merge(outs, lses, n_parts, rows, d, out, out_dtype, lse, (cudaStream_t)stream);
}

int star_merge_strided(const float* outs, int64_t out_part_stride, const float* lses,
                       int64_t lse_part_stride, int n_parts, int64_t rows, int d, void* out,
                       int out_dtype, float* lse, void* stream) {
  return merge_strided(outs, out_part_stride, lses, lse_part_stride, n_parts, rows, d, out,
                       out_dtype, lse, (cudaStream_t)stream);
}

int star_debug_umma_gemm(const void* a, const void* b, float* c, int K, int mode, void* stream) {
  return debug_umma_gemm(a, b, c, K, mode, (cudaStream_t)stream);
}

}  // extern "C"
