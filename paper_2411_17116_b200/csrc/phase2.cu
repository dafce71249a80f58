// Phase 2 (K2): GQA-aware split-KV partial attention over a paged KV cache,
// emitting fp32 (out, lse); and K3: the log-domain merge of partials.
//
// Reference semantics: partial_attention(q, K_h, V_h, "full" | keep)
// (ss/attention.py:125-151) as called by _gather_merge (ss/sim.py:178-213),
// including the query host's own-tail causal keep mask (ss/sim.py:195-200);
// merge_partials (ss/attention.py:154-173) in fixed ascending order.
//
// Layout: k/v pool [num_pages, hkv, page_size, d]; a sequence's logical row r
// is page_table[b, r / page_size], slot r % page_size.  One CTA streams one
// contiguous key range ("split") of one (sequence, kv head) and serves all
// G = hq/hkv query heads x lq query rows of that group from each K/V tile load.
#include "common.cuh"
#include "exchange.cuh"

namespace star {

constexpr int kP2Threads = 128;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <typename T> struct VecOf;  // 16-byte vector helpers
template <> struct VecOf<float> {
  static constexpr int kPer16 = 4;
  static __device__ __forceinline__ void unpack(const uint4& w, float* f) {
    f[0] = __uint_as_float(w.x); f[1] = __uint_as_float(w.y);
    f[2] = __uint_as_float(w.z); f[3] = __uint_as_float(w.w);
  }
};
template <> struct VecOf<__nv_bfloat16> {
  static constexpr int kPer16 = 8;
  static __device__ __forceinline__ void unpack(const uint4& w, float* f) {
    f[0] = bf16lo(w.x); f[1] = bf16hi(w.x); f[2] = bf16lo(w.y); f[3] = bf16hi(w.y);
    f[4] = bf16lo(w.z); f[5] = bf16hi(w.z); f[6] = bf16lo(w.w); f[7] = bf16hi(w.w);
  }
};

// QRB: q rows (head-in-group x query row) handled per pass; TN: keys per smem tile.
template <typename TQ, typename TKV, int D, int TN, int QRB>
struct P2Smem {
  static constexpr int kRowBytes = D * (int)sizeof(TKV);
  static constexpr int kTileBytes = TN * kRowBytes;
  static constexpr int kBytes = 4 * kTileBytes   // K,V x double buffer
                                + QRB * D * 4    // q (fp32)
                                + QRB * TN * 4   // scores / probabilities
                                + QRB * 4 * 4;   // alpha, row max, tile sum, running l
};

template <typename TKV> struct Vec4;  // 4 consecutive head-dim elements
template <> struct Vec4<float> {
  static __device__ __forceinline__ float4 load(const float* p) {
    return *reinterpret_cast<const float4*>(p);
  }
};
template <> struct Vec4<__nv_bfloat16> {
  static __device__ __forceinline__ float4 load(const __nv_bfloat16* p) {
    uint2 w = *reinterpret_cast<const uint2*>(p);
    return make_float4(bf16lo(w.x), bf16hi(w.x), bf16lo(w.y), bf16hi(w.y));
  }
};

template <typename TQ, typename TKV, int D, int TN, int QRB>
__global__ void __launch_bounds__(kP2Threads, 4) phase2_partial_kernel(
    const TQ* __restrict__ q, int lq, int hq, int hkv, const TKV* __restrict__ kpool,
    const TKV* __restrict__ vpool, const int32_t* __restrict__ page_table, int pages_per_seq,
    int page_size, const int32_t* __restrict__ kv_len, int own_tail, int64_t chunk,
    float* __restrict__ out, float* __restrict__ lse, int64_t part_stride_rows, float scale) {
  using SM = P2Smem<TQ, TKV, D, TN, QRB>;
  constexpr int kChunks = SM::kRowBytes / 16;  // 16-byte chunks per key row
  constexpr int kPer16 = VecOf<TKV>::kPer16;
  constexpr int kGroups = QRB * D / 4;         // (q row, 4 head-dim lanes) output groups
  constexpr int kGPT = (kGroups + kP2Threads - 1) / kP2Threads;
  constexpr int kSub = kP2Threads / TN;        // threads per key row in the score phase
  // XOR swizzle of the 16-byte chunks of a key row, confined to the row (rows of < 8 chunks)
  constexpr int kSw = kChunks < 8 ? kChunks - 1 : 7;
  static_assert(QRB % kSub == 0, "tile shape");
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* kbuf = smem;                       // [2][TN][row] swizzled 16B chunks
  unsigned char* vbuf = smem + 2 * SM::kTileBytes;  // [2][TN][row] plain
  float* qs = reinterpret_cast<float*>(smem + 4 * SM::kTileBytes);  // [QRB][D]
  float* ps = qs + QRB * D;                                           // [QRB][TN]
  float* alpha_s = ps + QRB * TN;                                     // [QRB]
  float* mrow_s = alpha_s + QRB;                                      // [QRB]
  float* tsum_s = mrow_s + QRB;                                       // [QRB]
  float* lrun_s = tsum_s + QRB;                                       // [QRB]

  const int split = blockIdx.x, kvh = blockIdx.y, b = blockIdx.z;
  const int G = hq / hkv;
  const int QR = G * lq;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t len = kv_len[b];
  const int64_t r0 = (int64_t)split * chunk;
  const int64_t r1 = min(len, r0 + chunk);
  const int64_t tail0 = len - own_tail;  // first own-tail row (own_tail > 0 only)
  const int32_t* table = page_table + (int64_t)b * pages_per_seq;
  float* out_part = out + (int64_t)split * part_stride_rows * D;
  float* lse_part = lse + (int64_t)split * part_stride_rows;

  for (int qr0 = 0; qr0 < QR; qr0 += QRB) {
    const int nq = min(QRB, QR - qr0);
    __syncthreads();
    for (int e = tid; e < QRB * D; e += kP2Threads) {
      int rr = e / D, c = e % D;
      float val = 0.f;
      if (rr < nq) {
        int qr = qr0 + rr, i = qr / G, g = qr % G;
        val = Elem<TQ>::to_f(q[(((int64_t)b * lq + i) * hq + kvh * G + g) * D + c]);
      }
      qs[e] = val;
    }
    if (tid < QRB) {
      mrow_s[tid] = -INFINITY;
      lrun_s[tid] = 0.f;
    }
    float acc[kGPT][4];
#pragma unroll
    for (int o = 0; o < kGPT; ++o) acc[o][0] = acc[o][1] = acc[o][2] = acc[o][3] = 0.f;

    auto load_tile = [&](int buf, int64_t t0) {
      unsigned char* kb = kbuf + buf * SM::kTileBytes;
      unsigned char* vb = vbuf + buf * SM::kTileBytes;
      for (int e = tid; e < TN * kChunks; e += kP2Threads) {
        int n = e / kChunks, c = e % kChunks;
        int64_t row = t0 + n;
        if (row < r1) {
          int64_t page = table[row / page_size];
          int slot = (int)(row % page_size);
          size_t off = (((size_t)page * hkv + kvh) * page_size + slot) * SM::kRowBytes + c * 16;
          int pc = (c & ~kSw) | ((c ^ n) & kSw);
          cp_async16(kb + n * SM::kRowBytes + pc * 16, reinterpret_cast<const char*>(kpool) + off);
          cp_async16(vb + n * SM::kRowBytes + c * 16, reinterpret_cast<const char*>(vpool) + off);
        } else {
          // keep stale smem finite: zero the V row (K is masked by the score phase)
          *reinterpret_cast<uint4*>(vb + n * SM::kRowBytes + c * 16) = make_uint4(0, 0, 0, 0);
        }
      }
      cp_async_commit();
    };

    const int ntiles = r1 > r0 ? (int)((r1 - r0 + TN - 1) / TN) : 0;
    if (ntiles > 0) load_tile(0, r0);
    for (int t = 0; t < ntiles; ++t) {
      const int64_t t0 = r0 + (int64_t)t * TN;
      if (t + 1 < ntiles) {
        load_tile((t + 1) & 1, t0 + TN);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
      // ---- scores: thread -> key row n and q rows {sub, sub+kSub, ...} ----
      {
        const unsigned char* kb = kbuf + (t & 1) * SM::kTileBytes;
        const int n = tid % TN, sub = tid / TN;
        const int64_t row = t0 + n;
        const bool live_row = row < r1;
        float sc[QRB / kSub];
#pragma unroll
        for (int j = 0; j < QRB / kSub; ++j) sc[j] = 0.f;
#pragma unroll 2
        for (int c = 0; c < kChunks; ++c) {
          const int pc = (c & ~kSw) | ((c ^ n) & kSw);
          uint4 w = *reinterpret_cast<const uint4*>(kb + n * SM::kRowBytes + pc * 16);
          float kf[kPer16];
          VecOf<TKV>::unpack(w, kf);
#pragma unroll
          for (int j = 0; j < QRB / kSub; ++j) {
            const float* qr = qs + (sub + j * kSub) * D + c * kPer16;
#pragma unroll
            for (int e = 0; e < kPer16; e += 4) {
              float4 qv = *reinterpret_cast<const float4*>(qr + e);
              sc[j] = fmaf(qv.x, kf[e], sc[j]);
              sc[j] = fmaf(qv.y, kf[e + 1], sc[j]);
              sc[j] = fmaf(qv.z, kf[e + 2], sc[j]);
              sc[j] = fmaf(qv.w, kf[e + 3], sc[j]);
            }
          }
        }
#pragma unroll
        for (int j = 0; j < QRB / kSub; ++j) {
          const int rr = sub + j * kSub;
          bool vis = live_row && rr < nq;
          if (vis && own_tail > 0 && row >= tail0) vis = (row - tail0) <= (qr0 + rr) / G;
          ps[rr * TN + n] = vis ? sc[j] * scale : -INFINITY;
        }
      }
      __syncthreads();
      // ---- online softmax: warp w owns q rows w, w+4, ... ----
      for (int rr = warp; rr < QRB; rr += kP2Threads / 32) {
        float mx = -INFINITY;
        for (int n = lane; n < TN; n += 32) mx = fmaxf(mx, ps[rr * TN + n]);
#pragma unroll
        for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        const float m_prev = mrow_s[rr];
        const float m_new = fmaxf(m_prev, mx);
        float sum = 0.f;
        for (int n = lane; n < TN; n += 32) {
          const float s = ps[rr * TN + n];
          const float p = (s == -INFINITY) ? 0.f : expf(s - m_new);
          ps[rr * TN + n] = p;
          sum += p;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        __syncwarp();  // every lane has read mrow_s[rr] before lane 0 rewrites it
        if (lane == 0) {
          const float a = (m_prev == -INFINITY) ? 0.f : expf(m_prev - m_new);
          alpha_s[rr] = a;
          mrow_s[rr] = m_new;
          lrun_s[rr] = lrun_s[rr] * a + sum;
        }
      }
      __syncthreads();
      // ---- P.V: thread -> (q row, 4 consecutive head-dim lanes) groups ----
      {
        const TKV* vbt = reinterpret_cast<const TKV*>(vbuf + (t & 1) * SM::kTileBytes);
#pragma unroll
        for (int o = 0; o < kGPT; ++o) {
          const int gidx = o * kP2Threads + tid;
          if (gidx < kGroups) {
            const int rr = gidx / (D / 4), c = (gidx % (D / 4)) * 4;
            const float a = alpha_s[rr];
            float s0 = acc[o][0] * a, s1 = acc[o][1] * a, s2 = acc[o][2] * a, s3 = acc[o][3] * a;
            const float* prow = ps + rr * TN;
#pragma unroll 4
            for (int n = 0; n < TN; n += 4) {
              const float4 p4 = *reinterpret_cast<const float4*>(prow + n);
              const float pv[4] = {p4.x, p4.y, p4.z, p4.w};
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const float4 v4 = Vec4<TKV>::load(vbt + (n + u) * D + c);
                s0 = fmaf(pv[u], v4.x, s0);
                s1 = fmaf(pv[u], v4.y, s1);
                s2 = fmaf(pv[u], v4.z, s2);
                s3 = fmaf(pv[u], v4.w, s3);
              }
            }
            acc[o][0] = s0; acc[o][1] = s1; acc[o][2] = s2; acc[o][3] = s3;
          }
        }
      }
      __syncthreads();
    }
    // ---- write this split's partial, normalised locally ----
#pragma unroll
    for (int o = 0; o < kGPT; ++o) {
      const int gidx = o * kP2Threads + tid;
      if (gidx < kGroups) {
        const int rr = gidx / (D / 4), c = (gidx % (D / 4)) * 4;
        if (rr < nq) {
          const int qr = qr0 + rr, i = qr / G, g = qr % G;
          const int64_t orow = ((int64_t)b * lq + i) * hq + kvh * G + g;
          const float l = lrun_s[rr];
          const float inv = l > 0.f ? 1.f / l : 0.f;
          *reinterpret_cast<float4*>(out_part + orow * D + c) =
              make_float4(acc[o][0] * inv, acc[o][1] * inv, acc[o][2] * inv, acc[o][3] * inv);
        }
      }
    }
    if (tid < nq) {
      const int qr = qr0 + tid, i = qr / G, g = qr % G;
      const int64_t orow = ((int64_t)b * lq + i) * hq + kvh * G + g;
      const float l = lrun_s[tid];
      lse_part[orow] = l > 0.f ? mrow_s[tid] + logf(l) : -INFINITY;
    }
  }
}

// ------------------------------------------------------------------ K3 merge
// One warp per output row: the part weights exp(lse_p - s) are formed once per (row, part)
// (lanes over parts, fp64 like merge_partials, ss/attention.py:170-173) and staged in
// shared memory; lanes then sweep the head dim, coalesced.
constexpr int kMergeWarps = 8;
constexpr int kMergeMaxParts = 512;

template <typename TO>
__global__ void __launch_bounds__(kMergeWarps * 32) merge_kernel(
    const float* __restrict__ outs, int64_t out_pstride, const float* __restrict__ lses,
    int64_t lse_pstride, int n_parts, int64_t rows, int d, TO* __restrict__ out,
    float* __restrict__ lse) {
  __shared__ float wsm[kMergeWarps][kMergeMaxParts];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = blockIdx.x * (int64_t)kMergeWarps + warp;
  if (row >= rows) return;
  float* w = wsm[warp];
  double mx = -INFINITY;
  for (int p = lane; p < n_parts; p += 32) mx = fmax(mx, (double)lses[(int64_t)p * lse_pstride + row]);
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  double acc = 0.0;
  for (int p = lane; p < n_parts; p += 32) {
    const double l = lses[(int64_t)p * lse_pstride + row];
    const double e = (l == -INFINITY) ? 0.0 : exp(l - mx);
    w[p] = (float)e;
    acc += e;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  const double s = acc > 0.0 ? mx + log(acc) : -INFINITY;
  const float inv = acc > 0.0 ? (float)(1.0 / acc) : 0.f;
  __syncwarp();
  for (int c = lane; c < d; c += 32) {
    float o = 0.f;
    for (int p = 0; p < n_parts; ++p) o = fmaf(w[p], outs[(int64_t)p * out_pstride + row * d + c], o);
    out[row * d + c] = Elem<TO>::from_f(o * inv);
  }
  if (lse != nullptr && lane == 0) lse[row] = (float)s;
}

int merge_strided(const float* outs, int64_t out_pstride, const float* lses, int64_t lse_pstride,
                  int n_parts, int64_t rows, int d, void* out, int out_dtype, float* lse,
                  cudaStream_t s) {
  if (n_parts < 1) return fail(STAR_EDOMAIN, "merge of zero partials");
  if (n_parts > kMergeMaxParts) return fail(STAR_ENOTSUP, "merge of more than %d partials", kMergeMaxParts);
  if (rows < 0 || d < 1) return fail(STAR_ESHAPE, "merge: bad shape");
  if (out_pstride < rows * d || lse_pstride < rows)
    return fail(STAR_ESHAPE, "merge: part strides smaller than a part");
  if (rows == 0) return STAR_OK;
  int grid = (int)((rows + kMergeWarps - 1) / kMergeWarps);
  if (out_dtype == STAR_F32)
    merge_kernel<float><<<grid, kMergeWarps * 32, 0, s>>>(outs, out_pstride, lses, lse_pstride,
                                                          n_parts, rows, d, (float*)out, lse);
  else if (out_dtype == STAR_BF16)
    merge_kernel<__nv_bfloat16><<<grid, kMergeWarps * 32, 0, s>>>(
        outs, out_pstride, lses, lse_pstride, n_parts, rows, d, (__nv_bfloat16*)out, lse);
  else
    return fail(STAR_ECONFIG, "merge: unknown dtype %d", out_dtype);
  STAR_LAUNCH_CHECK("merge");
  return STAR_OK;
}

int merge(const float* outs, const float* lses, int n_parts, int64_t rows, int d, void* out,
          int out_dtype, float* lse, cudaStream_t s) {
  return merge_strided(outs, rows * d, lses, rows, n_parts, rows, d, out, out_dtype, lse, s);
}

// ------------------------------------------------------------------ host side
constexpr int64_t kCounterBytes = 16384;  // header: 2048 arrival counters | 2048 epochs

int64_t phase2_workspace_bytes(int batch, int lq, int hq, int d, int n_splits) {
  if (n_splits <= 1) return 0;
  int64_t rows = (int64_t)batch * lq * hq;
  // fixed header (per (sequence, kv head): int32 arrival counters of the atomic fix-up, then
  // uint32 epochs of the word fix-up), then the split partials — fp32 (atomic mode) or
  // 8-byte {value, epoch} words (word mode); the header sits at the same offset whatever
  // the split count, so a reused workspace always finds its counters re-armed
  return kCounterBytes + (int64_t)n_splits * rows * (d + 1) * 8;
}

int phase2_auto_splits(int batch, int hkv, int64_t max_kv_len, int page_size) {
  // one wave: about one CTA per SM (the bf16 path keeps 128 KB of TMA stages per CTA);
  // at least 256 keys per split
  int64_t want = (int64_t)num_sms() / std::max(1, batch * hkv);
  // 16 splits (one DSMEM-merged cluster per sequence x kv head) when that still covers
  // most SMs: measured faster than a full 18-split wave with the global fix-up
  if (want > 16 && (int64_t)batch * hkv * 16 * 5 >= (int64_t)num_sms() * 4) want = 16;
  int64_t max_by_len = std::max<int64_t>(1, max_kv_len / 256);
  int64_t s = std::max<int64_t>(1, std::min(want, max_by_len));
  return (int)std::min<int64_t>(s, 256);
}

template <typename TQ, typename TKV, int D, int TN, int QRB>
static int launch_p2(const void* q, int batch, int lq, int hq, int hkv, const void* kp,
                     const void* vp, const int32_t* table, int pps, int page_size,
                     const int32_t* kv_len, int own_tail, int64_t chunk, int n_splits, float* out,
                     float* lse, cudaStream_t s) {
  using SM = P2Smem<TQ, TKV, D, TN, QRB>;
  auto kern = phase2_partial_kernel<TQ, TKV, D, TN, QRB>;
  int bytes = SM::kBytes;
  static bool configured = false;  // per instantiation
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) return fail(STAR_ECUDA, "phase2 smem attr: %s", cudaGetErrorString(e));
    configured = true;
  }
  dim3 grid(n_splits, hkv, batch);
  float scale = 1.0f / sqrtf((float)D);
  int64_t part_rows = (int64_t)batch * lq * hq;
  kern<<<grid, kP2Threads, bytes, s>>>((const TQ*)q, lq, hq, hkv, (const TKV*)kp, (const TKV*)vp,
                                       table, pps, page_size, kv_len, own_tail, chunk, out, lse,
                                       part_rows, scale);
  STAR_LAUNCH_CHECK("phase2_partial");
  return STAR_OK;
}

template <typename TQ, typename TKV, int D>
static int dispatch_qrb(int QR, const void* q, int batch, int lq, int hq, int hkv, const void* kp,
                        const void* vp, const int32_t* table, int pps, int page_size,
                        const int32_t* kv_len, int own_tail, int64_t chunk, int n_splits,
                        float* out, float* lse, cudaStream_t s) {
  constexpr int TN = sizeof(TKV) == 2 ? 64 : 32;
  if (QR <= 4)
    return launch_p2<TQ, TKV, D, TN, 4>(q, batch, lq, hq, hkv, kp, vp, table, pps, page_size,
                                        kv_len, own_tail, chunk, n_splits, out, lse, s);
  if (QR <= 8)
    return launch_p2<TQ, TKV, D, TN, 8>(q, batch, lq, hq, hkv, kp, vp, table, pps, page_size,
                                        kv_len, own_tail, chunk, n_splits, out, lse, s);
  return launch_p2<TQ, TKV, D, TN, 16>(q, batch, lq, hq, hkv, kp, vp, table, pps, page_size,
                                       kv_len, own_tail, chunk, n_splits, out, lse, s);
}

int phase2_mma(const void* q, int batch, int lq, int hq, int hkv, int d, const void* kp,
               const void* vp, int64_t num_pages, const int32_t* table, int pps, int page_size,
               const int32_t* kv_len, int own_tail, int64_t chunk, int n_splits, float* out,
               float* lse, float* final_out, float* final_lse, int* counters, PeerPush pp,
               int* merged, cudaStream_t s, const DecodeAppend* dap);
int push_partial(const float* out, const float* lse, int batch, int lq, int hq, int hkv, int d,
                 const PeerPush& pp, cudaStream_t s);
bool phase2_qe_eligible(int qrows, int d, int page_size);

int phase2_partial(const void* q, int q_dtype, int batch, int lq, int hq, int hkv, int d,
                   const void* kp, const void* vp, int kv_dtype, int64_t num_pages,
                   const int32_t* table, int pps, int page_size, const int32_t* kv_len,
                   int64_t max_kv_len, int own_tail, float* out, float* lse, int n_splits,
                   void* workspace, const PeerPush* push, int* merged, cudaStream_t s,
                   const DecodeAppend* dap) {
  const PeerPush none{};
  if (merged != nullptr) *merged = 0;
  if (batch < 1 || lq < 1 || hq < 1 || hkv < 1 || hq % hkv)
    return fail(STAR_ESHAPE, "phase2: bad heads/batch (batch=%d lq=%d hq=%d hkv=%d)", batch, lq,
                hq, hkv);
  if (own_tail != 0 && own_tail != lq)
    return fail(STAR_ESHAPE, "own_tail must be 0 or the query length, got %d", own_tail);
  if (max_kv_len < 0) return fail(STAR_ESHAPE, "phase2: negative kv length");
  if (page_size < 1 || pps < 1) return fail(STAR_ESHAPE, "phase2: bad page geometry");
  if (q_dtype != kv_dtype) return fail(STAR_ENOTSUP, "phase2: q and kv dtypes must match");
  if (d != 64 && d != 128 && d != 32 && d != 16)
    return fail(STAR_ENOTSUP, "phase2: head_dim %d not in {16,32,64,128}", d);
  // the tensor-core path runs G*lq > 16 query rows as 64-row blocks along grid.y: one wave
  // counts every row block as a group
  const int qrows = (hq / hkv) * lq;
  // (one packed 128-row tile in the tcgen05 query-encode kernel: no row blocks)
  const int n_rb = (qrows <= 16 || (kv_dtype == STAR_BF16 && phase2_qe_eligible(qrows, d, page_size)))
                       ? 1 : (qrows + 63) / 64;
  if (n_splits <= 0) n_splits = phase2_auto_splits(batch, hkv * n_rb, max_kv_len, page_size);
  int64_t chunk = std::max<int64_t>(1, (max_kv_len + n_splits - 1) / n_splits);
  const int TN = kv_dtype == STAR_BF16 ? 64 : 32;
  chunk = (chunk + TN - 1) / TN * TN;
  n_splits = (int)std::max<int64_t>(1, (max_kv_len + chunk - 1) / chunk);
  if (kv_dtype == STAR_BF16 && n_splits > 1) {
    // the in-kernel split fix-up stages n_splits x QR weights in the idle TMA ring
    const int64_t qr = (int64_t)(hq / hkv) * lq;
    // (and the fix-up folds at most 256 splits)
    const int64_t cap = std::min<int64_t>(256, ((d == 128 ? 6 * 32768 : 6 * 16384) - 64) / (4 * qr) - 1);
    if (n_splits > cap) {
      n_splits = (int)std::max<int64_t>(1, cap);
      chunk = (max_kv_len + n_splits - 1) / n_splits;
      chunk = (chunk + TN - 1) / TN * TN;
      n_splits = (int)std::max<int64_t>(1, (max_kv_len + chunk - 1) / chunk);
    }
  }
  float* po = out;
  float* pl = lse;
  int64_t rows = (int64_t)batch * lq * hq;
  if (n_splits > 1) {
    if (workspace == nullptr) return fail(STAR_ECONFIG, "phase2: workspace required for splits");
    if ((int64_t)batch * hkv * n_rb > kEpochOffsetWords)
      return fail(STAR_ENOTSUP, "phase2: batch x kv heads x row blocks > %d", kEpochOffsetWords);
    po = reinterpret_cast<float*>(reinterpret_cast<char*>(workspace) + kCounterBytes);
    pl = po + (int64_t)n_splits * rows * d;
  }
  const int QR = (hq / hkv) * lq;
  int rc;
  const bool tc_path = kv_dtype == STAR_BF16 && (d == 64 || d == 128) && page_size % 64 == 0 &&
                       num_pages > 0;
  if (tc_path) {
    // split partials are folded inside the kernel by the last CTA of each (sequence, kv
    // head); the arrival counters live after the partials in the (zero-initialised) workspace
    int* counters = n_splits > 1 ? reinterpret_cast<int*>(workspace) : nullptr;
    // with an exchange, the final partial of each group goes from the K2 epilogue straight
    // into every rank's box (out / lse are then only the split workspace's neighbours)
    return phase2_mma(q, batch, lq, hq, hkv, d, kp, vp, num_pages, table, pps, page_size, kv_len,
                      own_tail, chunk, n_splits, po, pl, out, lse, counters,
                      push ? *push : none, merged, s, dap);
  }
  if (dap != nullptr && dap->on)
    return fail(STAR_ENOTSUP, "fused decode append needs the bf16 tensor-core path (page_size %% 64 == 0)");
#define STAR_P2_D(TQ, TKV)                                                                    \
  switch (d) {                                                                                \
    case 128: rc = dispatch_qrb<TQ, TKV, 128>(QR, q, batch, lq, hq, hkv, kp, vp, table, pps,   \
                                              page_size, kv_len, own_tail, chunk, n_splits,    \
                                              po, pl, s); break;                               \
    case 64: rc = dispatch_qrb<TQ, TKV, 64>(QR, q, batch, lq, hq, hkv, kp, vp, table, pps,     \
                                            page_size, kv_len, own_tail, chunk, n_splits, po,  \
                                            pl, s); break;                                     \
    case 32: rc = dispatch_qrb<TQ, TKV, 32>(QR, q, batch, lq, hq, hkv, kp, vp, table, pps,     \
                                            page_size, kv_len, own_tail, chunk, n_splits, po,  \
                                            pl, s); break;                                     \
    default: rc = dispatch_qrb<TQ, TKV, 16>(QR, q, batch, lq, hq, hkv, kp, vp, table, pps,     \
                                            page_size, kv_len, own_tail, chunk, n_splits, po,  \
                                            pl, s); break;                                     \
  }
  if (kv_dtype == STAR_BF16) {
    STAR_P2_D(__nv_bfloat16, __nv_bfloat16)
  } else if (kv_dtype == STAR_F32) {
    STAR_P2_D(float, float)
  } else {
    return fail(STAR_ECONFIG, "phase2: unknown dtype %d", kv_dtype);
  }
#undef STAR_P2_D
  if (rc != STAR_OK) return rc;
  if (n_splits > 1) {
    rc = merge(po, pl, n_splits, rows, d, out, STAR_F32, lse, s);
    if (rc != STAR_OK) return rc;
  }
  return push ? push_partial(out, lse, batch, lq, hq, hkv, d, *push, s) : STAR_OK;
}

}  // namespace star
