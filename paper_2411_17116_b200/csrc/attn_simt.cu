// fp32 check-mode attention (and the generic-shape path): segment-batched
// causal / full softmax attention on CUDA cores with fp32 accumulation.
//
// Semantics follow _attend / causal_attention / partial_attention
// (ss/attention.py:79-151): scores = (q.k) / sqrt(d); masked cells are
// skipped; out is locally normalised; lse = max + ln(sum) (natural log).
// The online (tile-folded) softmax is the merge rule of
// streaming_causal_attention (ss/attention.py:176-210).
#include "common.cuh"

namespace star {

constexpr int kSimtBM = 64;   // q rows per CTA
constexpr int kSimtBN = 32;   // kv rows per smem tile
constexpr int kSimtThreads = kSimtBM * 4;

// Thread t owns q row (t / 4) and the head-dim lanes {t%4, t%4+4, ...}.
template <typename T, typename TO, int D>
__global__ void __launch_bounds__(kSimtThreads) attn_simt_kernel(
    const T* __restrict__ q, const T* __restrict__ k, const T* __restrict__ v, SegTable segs,
    int hq, int hkv, int d, int64_t qs, int64_t kvs, int causal, TO* __restrict__ out, int64_t os,
    float* __restrict__ lse, int64_t lse_stride, float scale) {
  constexpr int DPT = D / 4;
  __shared__ float Ks[kSimtBN][D];
  __shared__ float Vs[kSimtBN][D];

  // locate segment / q tile
  const int tile = blockIdx.x;
  int s = 0;
  while (s + 1 < segs.n && segs.tile_start[s + 1] <= tile) ++s;
  const int qt = tile - segs.tile_start[s];
  const int h = blockIdx.y;
  const int kvh = h / (hq / hkv);
  const int tid = threadIdx.x;
  const int r = tid >> 2, qd = tid & 3;
  const int lq = segs.lq[s], lk = segs.lk[s], qoff = segs.q_offset[s];
  const int qrow = qt * kSimtBM + r;
  const bool row_ok = qrow < lq;

  float qv[DPT], acc[DPT];
#pragma unroll
  for (int i = 0; i < DPT; ++i) {
    int c = qd + 4 * i;
    qv[i] = (row_ok && c < d) ? Elem<T>::to_f(q[(segs.q_row0[s] + qrow) * qs + (int64_t)h * d + c])
                              : 0.f;
    acc[i] = 0.f;
  }
  float m = -INFINITY, l = 0.f;

  // keys visible to the last row of this tile
  int kend = lk;
  if (causal) kend = min(lk, qoff + min(lq, (qt + 1) * kSimtBM));
  const T* kb = k + segs.k_row0[s] * kvs + (int64_t)kvh * d;
  const T* vb = v + segs.k_row0[s] * kvs + (int64_t)kvh * d;
  const int my_limit = causal ? qoff + qrow : lk - 1;  // last visible key of my row

  for (int k0 = 0; k0 < kend; k0 += kSimtBN) {
    __syncthreads();
    for (int e = tid; e < kSimtBN * D; e += kSimtThreads) {
      int j = e / D, c = e % D;
      bool ok = (k0 + j < lk) && c < d;
      Ks[j][c] = ok ? Elem<T>::to_f(kb[(int64_t)(k0 + j) * kvs + c]) : 0.f;
      Vs[j][c] = ok ? Elem<T>::to_f(vb[(int64_t)(k0 + j) * kvs + c]) : 0.f;
    }
    __syncthreads();
    float sc[kSimtBN];
    float tmax = -INFINITY;
#pragma unroll
    for (int j = 0; j < kSimtBN; ++j) {
      float p = 0.f;
#pragma unroll
      for (int i = 0; i < DPT; ++i) p = fmaf(qv[i], Ks[j][qd + 4 * i], p);
      p += __shfl_xor_sync(0xffffffffu, p, 1);
      p += __shfl_xor_sync(0xffffffffu, p, 2);
      const int kj = k0 + j;
      const bool vis = kj < lk && kj <= my_limit;
      sc[j] = vis ? p * scale : -INFINITY;
      tmax = fmaxf(tmax, sc[j]);
    }
    if (tmax == -INFINITY) continue;  // nothing visible for this row in this tile
    const float mn = fmaxf(m, tmax);
    const float alpha = (m == -INFINITY) ? 0.f : expf(m - mn);
    float lsum = 0.f;
#pragma unroll
    for (int i = 0; i < DPT; ++i) acc[i] *= alpha;
#pragma unroll
    for (int j = 0; j < kSimtBN; ++j) {
      const float p = (sc[j] == -INFINITY) ? 0.f : expf(sc[j] - mn);
      lsum += p;
#pragma unroll
      for (int i = 0; i < DPT; ++i) acc[i] = fmaf(p, Vs[j][qd + 4 * i], acc[i]);
    }
    l = l * alpha + lsum;
    m = mn;
  }
  if (!row_ok) return;
  const float inv = (l > 0.f) ? 1.f / l : 0.f;
  TO* orow = out + (segs.q_row0[s] + qrow) * os + (int64_t)h * d;
#pragma unroll
  for (int i = 0; i < DPT; ++i) {
    int c = qd + 4 * i;
    if (c < d) orow[c] = Elem<TO>::from_f(acc[i] * inv);
  }
  if (lse != nullptr && qd == 0)
    lse[(int64_t)h * lse_stride + segs.q_row0[s] + qrow] = (l > 0.f) ? m + logf(l) : -INFINITY;
}

template <typename T, typename TO>
static int launch_simt(const void* q, const void* k, const void* v, SegTable& segs, int hq, int hkv,
                       int d, int64_t qs, int64_t kvs, int causal, void* out, int64_t os,
                       float* lse, int64_t lse_stride, cudaStream_t s) {
  segs.tile_start[0] = 0;
  for (int i = 0; i < segs.n; ++i)
    segs.tile_start[i + 1] = segs.tile_start[i] + (segs.lq[i] + kSimtBM - 1) / kSimtBM;
  int tiles = segs.tile_start[segs.n];
  if (tiles == 0) return STAR_OK;
  dim3 grid(tiles, hq);
  float scale = 1.0f / sqrtf((float)d);
#define STAR_SIMT_LAUNCH(DD)                                                                  \
  attn_simt_kernel<T, TO, DD><<<grid, kSimtThreads, 0, s>>>(                                  \
      (const T*)q, (const T*)k, (const T*)v, segs, hq, hkv, d, qs, kvs, causal, (TO*)out, os,  \
      lse, lse_stride, scale)
  if (d <= 32)
    STAR_SIMT_LAUNCH(32);
  else if (d <= 64)
    STAR_SIMT_LAUNCH(64);
  else if (d <= 128)
    STAR_SIMT_LAUNCH(128);
  else
    return fail(STAR_ENOTSUP, "attention: head_dim %d > 128 not supported", d);
#undef STAR_SIMT_LAUNCH
  STAR_LAUNCH_CHECK("attn_simt");
  return STAR_OK;
}

int attention_simt(const void* q, const void* k, const void* v, int dtype, SegTable& segs, int hq,
                   int hkv, int d, int64_t qs, int64_t kvs, int causal, void* out, int out_dtype,
                   int64_t os, float* lse, int64_t lse_stride, cudaStream_t s) {
  if (dtype == STAR_F32 && out_dtype == STAR_F32)
    return launch_simt<float, float>(q, k, v, segs, hq, hkv, d, qs, kvs, causal, out, os, lse,
                                     lse_stride, s);
  if (dtype == STAR_BF16 && out_dtype == STAR_BF16)
    return launch_simt<__nv_bfloat16, __nv_bfloat16>(q, k, v, segs, hq, hkv, d, qs, kvs, causal,
                                                     out, os, lse, lse_stride, s);
  if (dtype == STAR_BF16 && out_dtype == STAR_F32)
    return launch_simt<__nv_bfloat16, float>(q, k, v, segs, hq, hkv, d, qs, kvs, causal, out, os,
                                             lse, lse_stride, s);
  return fail(STAR_ECONFIG, "attention: unsupported dtype pair (%d -> %d)", dtype, out_dtype);
}

}  // namespace star
