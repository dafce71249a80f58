// Elementwise sm_100a kernels of the star-attention path:
//   * counter-based splitmix64 fill  (ss/numerics.py:183-263)
//   * adjacent-pair RoPE at explicit positions, fp64 angles (ss/numerics.py:161-180)
//   * paged KV-cache write / read (own-row retention ss/sim.py:117-118, append
//     ss/blocking.py:161-170)
#include <stdlib.h>

#include "common.cuh"

namespace star {

// ------------------------------------------------------------------ PRNG
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

template <typename T>
__global__ void prng_fill_kernel(T* __restrict__ out, int64_t n, uint64_t seed, uint64_t first,
                                 double scale) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = mix64(seed + (first + (uint64_t)i) * 0x9E3779B97F4A7C15ull);
    double u = (double)(z >> 11) * 0x1.0p-53;
    // the reference draws at fp32 build precision (prng_fill -> astype(float32));
    // bf16 inputs are those fp32 values rounded once more to bf16.
    float f = __double2float_rn((2.0 * u - 1.0) * scale);
    out[i] = Elem<T>::from_f(f);
  }
}

int prng_fill(void* out, int dtype, int64_t n, uint64_t seed, uint64_t first, double scale,
              cudaStream_t s) {
  if (n < 0) return fail(STAR_ESHAPE, "prng_fill: negative size %lld", (long long)n);
  if (!(scale > 0)) return fail(STAR_EDOMAIN, "prng_fill scale must be positive, got %g", scale);
  if (n == 0) return STAR_OK;
  int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 16);
  if (dtype == STAR_F32)
    prng_fill_kernel<float><<<grid, 256, 0, s>>>((float*)out, n, seed, first, scale);
  else if (dtype == STAR_BF16)
    prng_fill_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>((__nv_bfloat16*)out, n, seed, first,
                                                        scale);
  else
    return fail(STAR_ECONFIG, "prng_fill: unknown dtype %d", dtype);
  STAR_LAUNCH_CHECK("prng_fill");
  return STAR_OK;
}

// ------------------------------------------------------------------ RoPE
// One thread per (row, pair i): the angle pos * theta^(-2i/d) is formed and
// reduced in fp64 once, then applied to that pair of every head of the row.
template <typename T>
__global__ void rope_kernel(const T* __restrict__ x, T* __restrict__ y, int64_t rows, int heads,
                            int d, int64_t xs, int64_t ys, const int64_t* __restrict__ pos,
                            double theta) {
  const int half = d >> 1;
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= rows * half) return;
  int64_t r = idx / half;
  int i = (int)(idx - r * half);
  double inv_freq = pow(theta, -2.0 * (double)i / (double)d);
  double ang = (double)pos[r] * inv_freq;
  double sn, cs;
  sincos(ang, &sn, &cs);
  const T* xr = x + r * xs + 2 * i;
  T* yr = y + r * ys + 2 * i;
  for (int h = 0; h < heads; ++h) {
    double x0 = (double)Elem<T>::to_f(xr[h * d]);
    double x1 = (double)Elem<T>::to_f(xr[h * d + 1]);
    double o0 = x0 * cs - x1 * sn;
    double o1 = x0 * sn + x1 * cs;
    yr[h * d] = Elem<T>::from_f(__double2float_rn(o0));
    yr[h * d + 1] = Elem<T>::from_f(__double2float_rn(o1));
  }
}

int rope(const void* x, void* y, int dtype, int64_t rows, int heads, int d, int64_t xs,
         int64_t ys, const int64_t* pos, double theta, cudaStream_t s) {
  if (d < 2 || (d & 1)) return fail(STAR_ECONFIG, "rope head_dim must be even and >= 2, got %d", d);
  if (!(theta > 0)) return fail(STAR_ECONFIG, "rope theta must be positive, got %g", theta);
  if (rows < 0 || heads < 1) return fail(STAR_ESHAPE, "rope: bad shape rows=%lld heads=%d",
                                        (long long)rows, heads);
  if (xs < (int64_t)heads * d || ys < (int64_t)heads * d)
    return fail(STAR_ESHAPE, "rope: row stride smaller than heads*d");
  if (rows == 0) return STAR_OK;
  int64_t n = rows * (d / 2);
  int grid = (int)((n + 255) / 256);
  if (dtype == STAR_F32)
    rope_kernel<float><<<grid, 256, 0, s>>>((const float*)x, (float*)y, rows, heads, d, xs, ys, pos,
                                            theta);
  else if (dtype == STAR_BF16)
    rope_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>((const __nv_bfloat16*)x, (__nv_bfloat16*)y,
                                                    rows, heads, d, xs, ys, pos, theta);
  else
    return fail(STAR_ECONFIG, "rope: unknown dtype %d", dtype);
  STAR_LAUNCH_CHECK("rope");
  return STAR_OK;
}

// ------------------------------------------------------------------ fused prologue
// one pass over the projection outputs of a layer's augmented blocks —
// RoPE of every q and k head at the row's position (angle formed once per (row, pair)),
// rotated q/k written for K1, and for own (cached) rows the rotated k and raw v written
// straight into the paged cache.  Replaces rope(q) + rope(k) + kv_write.
template <typename T>
__global__ void rope_qkv_kernel(const T* __restrict__ qi, const T* __restrict__ ki,
                                const T* __restrict__ vi, T* __restrict__ qo, T* __restrict__ ko,
                                int64_t rows, int hq, int hkv, int d, int64_t qis, int64_t kis,
                                int64_t qos, int64_t kos, const int64_t* __restrict__ pos,
                                double theta, const int64_t* __restrict__ cache_rows,
                                T* __restrict__ kp, T* __restrict__ vp,
                                const int32_t* __restrict__ table, int page_size) {
  const int half = d >> 1;
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= rows * half) return;
  int64_t r = idx / half;
  int i = (int)(idx - r * half);
  double sn, cs;
  sincos((double)pos[r] * pow(theta, -2.0 * (double)i / (double)d), &sn, &cs);
  const T* q = qi + r * qis + 2 * i;
  T* qw = qo + r * qos + 2 * i;
  for (int h = 0; h < hq; ++h) {
    const double x0 = Elem<T>::to_f(q[h * d]), x1 = Elem<T>::to_f(q[h * d + 1]);
    qw[h * d] = Elem<T>::from_f(__double2float_rn(x0 * cs - x1 * sn));
    qw[h * d + 1] = Elem<T>::from_f(__double2float_rn(x0 * sn + x1 * cs));
  }
  const int64_t cr = cache_rows != nullptr ? cache_rows[r] : -1;
  T* kpr = nullptr;
  T* vpr = nullptr;
  if (cr >= 0) {
    const int64_t page = table[cr / page_size];
    const int64_t slot = cr % page_size;
    kpr = kp + (page * hkv * page_size + slot) * d + 2 * i;
    vpr = vp + (page * hkv * page_size + slot) * d + 2 * i;
  }
  const T* k = ki + r * kis + 2 * i;
  const T* v = vi + r * kis + 2 * i;
  T* kw = ko + r * kos + 2 * i;
  for (int h = 0; h < hkv; ++h) {
    const double x0 = Elem<T>::to_f(k[h * d]), x1 = Elem<T>::to_f(k[h * d + 1]);
    const T y0 = Elem<T>::from_f(__double2float_rn(x0 * cs - x1 * sn));
    const T y1 = Elem<T>::from_f(__double2float_rn(x0 * sn + x1 * cs));
    kw[h * d] = y0;
    kw[h * d + 1] = y1;
    if (kpr != nullptr) {
      const int64_t po = (int64_t)h * page_size * d;
      kpr[po] = y0;
      kpr[po + 1] = y1;
      vpr[po] = v[h * d];
      vpr[po + 1] = v[h * d + 1];
    }
  }
}

// bf16 form of rope_qkv_kernel with 16-byte accesses: a thread rotates 4 adjacent pairs
// (8 elements) of one row in every head, so each load / store moves 16 bytes instead of 2.
// The arithmetic per pair (fp64 angle and rotation, one rounding to fp32 then to bf16) is
// rope_qkv_kernel's, so the results are bit-identical.  Needs d % 8 == 0 and 16-byte aligned
// rows (the host checks, else the scalar kernel runs).
__device__ __forceinline__ void rope4_bf16(uint4& w, const double (&cs)[4], const double (&sn)[4]) {
  uint32_t* u = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const __nv_bfloat162 x = *reinterpret_cast<const __nv_bfloat162*>(&u[k]);
    const double x0 = (double)__bfloat162float(x.x), x1 = (double)__bfloat162float(x.y);
    __nv_bfloat162 y;
    y.x = __float2bfloat16_rn(__double2float_rn(x0 * cs[k] - x1 * sn[k]));
    y.y = __float2bfloat16_rn(__double2float_rn(x0 * sn[k] + x1 * cs[k]));
    u[k] = *reinterpret_cast<const uint32_t*>(&y);
  }
}

__global__ void rope_qkv_vec_kernel(const __nv_bfloat16* __restrict__ qi,
                                    const __nv_bfloat16* __restrict__ ki,
                                    const __nv_bfloat16* __restrict__ vi, __nv_bfloat16* __restrict__ qo,
                                    __nv_bfloat16* __restrict__ ko, int64_t rows, int hq, int hkv, int d,
                                    int64_t qis, int64_t kis, int64_t qos, int64_t kos,
                                    const int64_t* __restrict__ pos, double theta,
                                    const int64_t* __restrict__ cache_rows,
                                    __nv_bfloat16* __restrict__ kp, __nv_bfloat16* __restrict__ vp,
                                    const int32_t* __restrict__ table, int page_size) {
  const int groups = d >> 3;  // 8-element groups per head row
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= rows * groups) return;
  const int64_t r = idx / groups;
  const int g = (int)(idx - r * groups);
  double cs[4], sn[4];
  const double p = (double)pos[r];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int i = 4 * g + k;
    sincos(p * pow(theta, -2.0 * (double)i / (double)d), &sn[k], &cs[k]);
  }
  const int64_t col = 8 * (int64_t)g;
  for (int h = 0; h < hq; ++h) {
    uint4 w = *reinterpret_cast<const uint4*>(qi + r * qis + h * d + col);
    rope4_bf16(w, cs, sn);
    *reinterpret_cast<uint4*>(qo + r * qos + h * d + col) = w;
  }
  const int64_t cr = cache_rows != nullptr ? cache_rows[r] : -1;
  int64_t pbase = -1;
  if (cr >= 0) pbase = ((int64_t)table[cr / page_size] * hkv * page_size + cr % page_size) * d + col;
  for (int h = 0; h < hkv; ++h) {
    uint4 w = *reinterpret_cast<const uint4*>(ki + r * kis + h * d + col);
    rope4_bf16(w, cs, sn);
    *reinterpret_cast<uint4*>(ko + r * kos + h * d + col) = w;
    if (pbase >= 0) {
      const int64_t po = pbase + (int64_t)h * page_size * d;
      *reinterpret_cast<uint4*>(kp + po) = w;
      *reinterpret_cast<uint4*>(vp + po) = *reinterpret_cast<const uint4*>(vi + r * kis + h * d + col);
    }
  }
}

int rope_qkv(const void* qi, const void* ki, const void* vi, int dtype, int64_t rows, int hq,
             int hkv, int d, int64_t qis, int64_t kis, void* qo, void* ko, int64_t qos,
             int64_t kos, const int64_t* pos, double theta, const int64_t* cache_rows, void* kp,
             void* vp, const int32_t* table, int page_size, cudaStream_t s) {
  if (d < 2 || (d & 1)) return fail(STAR_ECONFIG, "rope head_dim must be even and >= 2, got %d", d);
  if (!(theta > 0)) return fail(STAR_ECONFIG, "rope theta must be positive, got %g", theta);
  if (rows < 0 || hq < 1 || hkv < 1) return fail(STAR_ESHAPE, "rope_qkv: bad shape");
  if (qis < (int64_t)hq * d || qos < (int64_t)hq * d || kis < (int64_t)hkv * d ||
      kos < (int64_t)hkv * d)
    return fail(STAR_ESHAPE, "rope_qkv: row stride smaller than heads*d");
  if (cache_rows != nullptr && (kp == nullptr || vp == nullptr || table == nullptr || page_size < 1))
    return fail(STAR_ESHAPE, "rope_qkv: cache rows given without a paged cache");
  if (rows == 0) return STAR_OK;
  const bool vec = dtype == STAR_BF16 && d % 8 == 0 && qis % 8 == 0 && kis % 8 == 0 &&
                   qos % 8 == 0 && kos % 8 == 0 &&
                   (((uintptr_t)qi | (uintptr_t)ki | (uintptr_t)vi | (uintptr_t)qo | (uintptr_t)ko |
                     (uintptr_t)kp | (uintptr_t)vp) & 15) == 0;
  if (vec) {
    const int64_t nv = rows * (d / 8);
    rope_qkv_vec_kernel<<<(int)((nv + 255) / 256), 256, 0, s>>>(
        (const __nv_bfloat16*)qi, (const __nv_bfloat16*)ki, (const __nv_bfloat16*)vi,
        (__nv_bfloat16*)qo, (__nv_bfloat16*)ko, rows, hq, hkv, d, qis, kis, qos, kos, pos, theta,
        cache_rows, (__nv_bfloat16*)kp, (__nv_bfloat16*)vp, table, page_size);
    STAR_LAUNCH_CHECK("rope_qkv");
    return STAR_OK;
  }
  const int64_t n = rows * (d / 2);
  const int grid = (int)((n + 255) / 256);
#define STAR_RQKV(T)                                                                              rope_qkv_kernel<T><<<grid, 256, 0, s>>>((const T*)qi, (const T*)ki, (const T*)vi, (T*)qo,                                               (T*)ko, rows, hq, hkv, d, qis, kis, qos, kos, pos,                                              theta, cache_rows, (T*)kp, (T*)vp, table, page_size)
  if (dtype == STAR_F32)
    STAR_RQKV(float);
  else if (dtype == STAR_BF16)
    STAR_RQKV(__nv_bfloat16);
  else
    return fail(STAR_ECONFIG, "rope_qkv: unknown dtype %d", dtype);
#undef STAR_RQKV
  STAR_LAUNCH_CHECK("rope_qkv");
  return STAR_OK;
}

// ------------------------------------------------------------------ decode append
// The per-token append of phase 2 (ss/sim.py:275-277, append-then-attend) with every piece of
// state on the device, so a decode step is graph-capturable: for each of `batch` sequences,
// RoPE of its `rows` new rows' q and k at their device positions (the same fp64 angle as
// rope_kernel), rotated k and raw v written at the cache rows the sequence's device counter
// kv_len[b] names, counter advanced by `rows`.  One CTA per sequence (its counter is read
// before and bumped after a CTA barrier).  It triggers its programmatic dependents at entry:
// the K2 launch that follows (PDL) sets up beside it and waits in griddepcontrol.wait for
// this kernel's stores.
// cos / sin table of the decode positions [pos0, pos0 + n): entry (p, i) = {cos, sin} of
// (pos0 + p) * theta^(-2i/d), the same fp64 expression as rope_kernel / rope_qkv_kernel, so a
// rotation through the table is bit-identical to one that forms the angle in place.  Built
// once per decoder (outside the per-token graph); the per-token append then spends no fp64
// pow / sincos latency.
__global__ void rope_table_kernel(double2* __restrict__ cs, int64_t pos0, int64_t n, int d,
                                  double theta) {
  const int half = d >> 1;
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= n * half) return;
  const int64_t p = idx / half;
  const int i = (int)(idx - p * half);
  double sn, c;
  sincos((double)(pos0 + p) * pow(theta, -2.0 * (double)i / (double)d), &sn, &c);
  cs[idx] = make_double2(c, sn);
}

int rope_table(void* cs, int64_t pos0, int64_t n, int d, double theta, cudaStream_t s) {
  if (d < 2 || (d & 1)) return fail(STAR_ECONFIG, "rope head_dim must be even and >= 2, got %d", d);
  if (!(theta > 0)) return fail(STAR_ECONFIG, "rope theta must be positive, got %g", theta);
  if (n < 0 || pos0 < 0) return fail(STAR_ESHAPE, "rope_table: bad position range");
  if (n == 0) return STAR_OK;
  const int64_t m = n * (d / 2);
  rope_table_kernel<<<(int)((m + 255) / 256), 256, 0, s>>>((double2*)cs, pos0, n, d, theta);
  STAR_LAUNCH_CHECK("rope_table");
  return STAR_OK;
}

template <typename T>
struct Pair;  // two adjacent elements moved as one load / store
template <>
struct Pair<float> {
  using V = float2;
  static __device__ __forceinline__ void get(V v, double& a, double& b) { a = v.x; b = v.y; }
  static __device__ __forceinline__ V make(double a, double b) {
    return make_float2(__double2float_rn(a), __double2float_rn(b));
  }
};
template <>
struct Pair<__nv_bfloat16> {
  using V = __nv_bfloat162;
  static __device__ __forceinline__ void get(V v, double& a, double& b) {
    a = __bfloat162float(v.x);
    b = __bfloat162float(v.y);
  }
  static __device__ __forceinline__ V make(double a, double b) {
    V r;
    r.x = __float2bfloat16_rn(__double2float_rn(a));
    r.y = __float2bfloat16_rn(__double2float_rn(b));
    return r;
  }
};

constexpr int kAppendThreads = 512;
constexpr int kAppendUnroll = 4;

// One CTA per sequence.  Phase A: the (row, pair) cos/sin of the new rows into shared memory
// (from the decode-position table, else formed in place).  Phase B: every (row, head, pair)
// of q and k rotated and every (row, head, pair) of v copied — one independent 2-element item
// per thread, kAppendUnroll items in flight per thread (all loads issued before any store),
// so the kernel costs about one memory round trip instead of one per head.
template <typename T>
__global__ void __launch_bounds__(kAppendThreads) kv_append_kernel(
    const T* __restrict__ qi, const T* __restrict__ ki, const T* __restrict__ vi,
    T* __restrict__ qo, int rows, int hq, int hkv, int d, int64_t qis, int64_t kis, int64_t qos,
    const int64_t* __restrict__ pos, double theta, int32_t* __restrict__ kv_len,
    T* __restrict__ kp, T* __restrict__ vp, const int32_t* __restrict__ page_table, int pps,
    int page_size, const double2* __restrict__ rtab, int64_t rtab_pos0, int64_t rtab_n) {
  using P = Pair<T>;
  using V = typename P::V;
  extern __shared__ double2 cs_s[];  // [rows][half]
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");  // no-op unless launched as a dependent
  const int b = blockIdx.x;
  const int half = d >> 1;
  const int64_t base = kv_len[b];
  const int32_t* table = page_table + (int64_t)b * pps;
  for (int idx = threadIdx.x; idx < rows * half; idx += blockDim.x) {
    const int rl = idx / half, i = idx - rl * half;
    const int64_t p = pos[(int64_t)b * rows + rl];
    const int64_t tp = p - rtab_pos0;
    if (rtab != nullptr && tp >= 0 && tp < rtab_n) {
      cs_s[idx] = rtab[tp * half + i];
    } else {
      double sn, c;
      sincos((double)p * pow(theta, -2.0 * (double)i / (double)d), &sn, &c);
      cs_s[idx] = make_double2(c, sn);
    }
  }
  __syncthreads();
  const int nq = rows * hq * half, nk = rows * hkv * half;
  const int total = nq + 2 * nk;
  for (int i0 = threadIdx.x; i0 < total; i0 += kAppendUnroll * kAppendThreads) {
    V val[kAppendUnroll];
#pragma unroll
    for (int u = 0; u < kAppendUnroll; ++u) {
      const int idx = i0 + u * kAppendThreads;
      if (idx >= total) break;
      const T* src;
      if (idx < nq) {
        const int rl = idx / (hq * half), rem = idx - rl * hq * half;
        src = qi + ((int64_t)b * rows + rl) * qis + 2 * rem;
      } else {
        const int j = idx < nq + nk ? idx - nq : idx - nq - nk;
        const int rl = j / (hkv * half), rem = j - rl * hkv * half;
        src = (idx < nq + nk ? ki : vi) + ((int64_t)b * rows + rl) * kis + 2 * rem;
      }
      val[u] = *reinterpret_cast<const V*>(src);
    }
#pragma unroll
    for (int u = 0; u < kAppendUnroll; ++u) {
      const int idx = i0 + u * kAppendThreads;
      if (idx >= total) break;
      if (idx < nq) {
        const int rl = idx / (hq * half), rem = idx - rl * hq * half;
        const double2 e = cs_s[rl * half + rem % half];
        double x0, x1;
        P::get(val[u], x0, x1);
        *reinterpret_cast<V*>(qo + ((int64_t)b * rows + rl) * qos + 2 * rem) =
            P::make(x0 * e.x - x1 * e.y, x0 * e.y + x1 * e.x);
      } else {
        const bool is_k = idx < nq + nk;
        const int j = is_k ? idx - nq : idx - nq - nk;
        const int rl = j / (hkv * half), rem = j - rl * hkv * half;
        const int h = rem / half, i = rem - h * half;
        const int64_t cr = base + rl;
        const int64_t page = table[cr / page_size];
        const int64_t off = ((page * hkv + h) * page_size + cr % page_size) * d + 2 * i;
        V outv = val[u];
        if (is_k) {
          const double2 e = cs_s[rl * half + i];
          double x0, x1;
          P::get(val[u], x0, x1);
          outv = P::make(x0 * e.x - x1 * e.y, x0 * e.y + x1 * e.x);
        }
        *reinterpret_cast<V*>((is_k ? kp : vp) + off) = outv;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) kv_len[b] = (int32_t)(base + rows);
}

int kv_append(const void* qi, const void* ki, const void* vi, int dtype, int batch, int rows,
              int hq, int hkv, int d, int64_t qis, int64_t kis, void* qo, int64_t qos,
              const int64_t* pos, double theta, int32_t* kv_len, void* kp, void* vp,
              const int32_t* table, int pps, int page_size, const void* rtab, int64_t rtab_pos0,
              int64_t rtab_n, cudaStream_t s) {
  if (d < 2 || (d & 1)) return fail(STAR_ECONFIG, "rope head_dim must be even and >= 2, got %d", d);
  if (!(theta > 0)) return fail(STAR_ECONFIG, "rope theta must be positive, got %g", theta);
  if (batch < 0 || rows < 0 || hq < 1 || hkv < 1 || page_size < 1 || pps < 1)
    return fail(STAR_ESHAPE, "kv_append: bad shape");
  if (qis < (int64_t)hq * d || qos < (int64_t)hq * d || kis < (int64_t)hkv * d)
    return fail(STAR_ESHAPE, "kv_append: row stride smaller than heads*d");
  if (kv_len == nullptr || kp == nullptr || vp == nullptr || table == nullptr || pos == nullptr)
    return fail(STAR_ESHAPE, "kv_append: NULL counter / pool / table / positions");
  if ((int64_t)rows > (int64_t)pps * page_size)
    return fail(STAR_ESHAPE, "kv_append: %d rows exceed the %lld rows a page table maps", rows,
                (long long)pps * page_size);
  if (batch == 0 || rows == 0) return STAR_OK;
  // (the counters live on the device: the caller reserves pps * page_size rows per sequence
  // for the whole decode, DeviceDecoder / PagedKVPool.reserve)
  // launched as a programmatic dependent of the kernel before it (typically the previous
  // layer's K2): its CTA becomes resident while that kernel drains and waits in
  // griddepcontrol.wait (STAR_K2_PDL=0: plain launch)
  static int pdl = -1;
  if (pdl < 0) {
    const char* e = getenv("STAR_K2_PDL");
    pdl = (e != nullptr && e[0] == '0') ? 0 : 1;
  }
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  if ((int64_t)rows * (d / 2) * 16 > 48 * 1024)
    return fail(STAR_ENOTSUP, "kv_append: %d rows per sequence exceed the cos/sin staging", rows);
  if ((qis | kis | qos) & 1) return fail(STAR_ECONFIG, "kv_append: odd row strides");
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(batch);
  cfg.blockDim = dim3(kAppendThreads);
  cfg.dynamicSmemBytes = (size_t)rows * (d / 2) * sizeof(double2);
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = pdl;
  cudaError_t e;
  if (dtype == STAR_F32)
    e = cudaLaunchKernelEx(&cfg, kv_append_kernel<float>, (const float*)qi, (const float*)ki,
                           (const float*)vi, (float*)qo, rows, hq, hkv, d, qis, kis, qos, pos,
                           theta, kv_len, (float*)kp, (float*)vp, table, pps, page_size,
                           (const double2*)rtab, rtab_pos0, rtab_n);
  else if (dtype == STAR_BF16)
    e = cudaLaunchKernelEx(&cfg, kv_append_kernel<__nv_bfloat16>, (const __nv_bfloat16*)qi,
                           (const __nv_bfloat16*)ki, (const __nv_bfloat16*)vi, (__nv_bfloat16*)qo,
                           rows, hq, hkv, d, qis, kis, qos, pos, theta, kv_len, (__nv_bfloat16*)kp,
                           (__nv_bfloat16*)vp, table, pps, page_size, (const double2*)rtab,
                           rtab_pos0, rtab_n);
  else
    return fail(STAR_ECONFIG, "kv_append: unknown dtype %d", dtype);
  if (e != cudaSuccess) return fail(STAR_ECUDA, "kv_append launch: %s", cudaGetErrorString(e));
  return STAR_OK;
}

// ------------------------------------------------------------------ decode advance
// End of a fused decode step (star_phase2_decode appends without moving the counters, which
// every K2 CTA reads): every layer's row counter += add and every position += inc, then the
// cos/sin of the (new) positions into cur_cs [np][d/2] (from the decode-position table, else
// the fp64 angle), so the next token's K2 reads them without a dependent position load.
// One launch per token (inc = 0, add = 0: just fill cur_cs).
__global__ void decode_advance_kernel(int32_t* __restrict__ kv_len, int n, int add,
                                      int64_t* __restrict__ pos, int np, int inc,
                                      double2* __restrict__ cur_cs, const double2* __restrict__ rtab,
                                      int64_t pos0, int64_t ntab, int d, double theta) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  for (int i = threadIdx.x; i < n; i += blockDim.x) kv_len[i] += add;
  __shared__ int64_t ps[64];
  for (int i = threadIdx.x; i < np; i += blockDim.x) {
    const int64_t p = pos[i] + inc;
    pos[i] = p;
    if (i < 64) ps[i] = p;
  }
  if (cur_cs == nullptr) return;
  __syncthreads();
  const int half = d >> 1;
  for (int idx = threadIdx.x; idx < np * half; idx += blockDim.x) {
    const int b = idx / half, i = idx - b * half;
    const int64_t p = b < 64 ? ps[b] : pos[b];
    const int64_t tp = p - pos0;
    if (rtab != nullptr && tp >= 0 && tp < ntab) {
      cur_cs[idx] = rtab[tp * half + i];
    } else {
      double sn, c;
      sincos((double)p * pow(theta, -2.0 * (double)i / (double)d), &sn, &c);
      cur_cs[idx] = make_double2(c, sn);
    }
  }
}

int decode_advance(int32_t* kv_len, int n, int add, int64_t* pos, int np, int inc, void* cur_cs,
                   const void* rtab, int64_t pos0, int64_t ntab, int d, double theta,
                   cudaStream_t s) {
  if (n == 0 && np == 0) return STAR_OK;
  if (cur_cs != nullptr && (d < 2 || (d & 1) || !(theta > 0)))
    return fail(STAR_ECONFIG, "decode_advance: bad head_dim / theta for the cos/sin refresh");
  decode_advance_kernel<<<1, 256, 0, s>>>(kv_len, n, add, pos, np, inc, (double2*)cur_cs,
                                          (const double2*)rtab, pos0, ntab, d, theta);
  STAR_LAUNCH_CHECK("decode_advance");
  return STAR_OK;
}

// ------------------------------------------------------------------ paged KV
// Vector width W bytes; each thread moves one W-byte chunk of one (row, head).
template <typename V>
__global__ void kv_copy_kernel(const char* __restrict__ ks, const char* __restrict__ vs,
                               char* __restrict__ kp, char* __restrict__ vp,
                               const int32_t* __restrict__ table, int64_t n_rows, int hkv,
                               int row_bytes, int64_t src_stride_bytes, int page_size,
                               int64_t row0, bool to_pages) {
  const int chunks = row_bytes / (int)sizeof(V);
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t total = n_rows * hkv * chunks;
  if (idx >= total) return;
  int c = (int)(idx % chunks);
  int64_t t = idx / chunks;
  int h = (int)(t % hkv);
  int64_t r = t / hkv;
  int64_t lr = row0 + r;
  int64_t page = table[lr / page_size];
  int slot = (int)(lr % page_size);
  int64_t poff = ((page * hkv + h) * page_size + slot) * (int64_t)row_bytes + c * sizeof(V);
  int64_t soff = r * src_stride_bytes + (int64_t)h * row_bytes + c * sizeof(V);
  if (to_pages) {
    *reinterpret_cast<V*>(kp + poff) = *reinterpret_cast<const V*>(ks + soff);
    *reinterpret_cast<V*>(vp + poff) = *reinterpret_cast<const V*>(vs + soff);
  } else {
    *reinterpret_cast<V*>(const_cast<char*>(ks) + soff) = *reinterpret_cast<const V*>(kp + poff);
    *reinterpret_cast<V*>(const_cast<char*>(vs) + soff) = *reinterpret_cast<const V*>(vp + poff);
  }
}

static int kv_copy(const void* ks, const void* vs, void* kp, void* vp, int dtype, int64_t n_rows,
                   int hkv, int d, int64_t src_stride, const int32_t* table, int page_size,
                   int64_t row0, bool to_pages, cudaStream_t s) {
  if (dtype != STAR_F32 && dtype != STAR_BF16)
    return fail(STAR_ECONFIG, "kv copy: unknown dtype %d", dtype);
  if (n_rows < 0 || hkv < 1 || d < 1 || page_size < 1 || row0 < 0)
    return fail(STAR_ESHAPE, "kv copy: bad shape");
  if (src_stride < (int64_t)hkv * d) return fail(STAR_ESHAPE, "kv copy: row stride < hkv*d");
  if (n_rows == 0) return STAR_OK;
  int es = dtype == STAR_F32 ? 4 : 2;
  int row_bytes = d * es;
  int64_t sb = src_stride * es;
  bool v16 = (row_bytes % 16 == 0) && (sb % 16 == 0) && ((uintptr_t)ks % 16 == 0) &&
             ((uintptr_t)vs % 16 == 0);
  int64_t chunks = v16 ? row_bytes / 16 : (row_bytes % 4 == 0 ? row_bytes / 4 : row_bytes / 2);
  int64_t total = n_rows * hkv * chunks;
  int grid = (int)((total + 255) / 256);
  if (v16)
    kv_copy_kernel<uint4><<<grid, 256, 0, s>>>((const char*)ks, (const char*)vs, (char*)kp,
                                               (char*)vp, table, n_rows, hkv, row_bytes, sb,
                                               page_size, row0, to_pages);
  else if (row_bytes % 4 == 0)
    kv_copy_kernel<uint32_t><<<grid, 256, 0, s>>>((const char*)ks, (const char*)vs, (char*)kp,
                                                  (char*)vp, table, n_rows, hkv, row_bytes, sb,
                                                  page_size, row0, to_pages);
  else
    kv_copy_kernel<uint16_t><<<grid, 256, 0, s>>>((const char*)ks, (const char*)vs, (char*)kp,
                                                  (char*)vp, table, n_rows, hkv, row_bytes, sb,
                                                  page_size, row0, to_pages);
  STAR_LAUNCH_CHECK("kv_copy");
  return STAR_OK;
}

int kv_write(const void* k, const void* v, int dtype, int64_t n_rows, int hkv, int d,
             int64_t src_stride, void* kp, void* vp, const int32_t* table, int page_size,
             int64_t row0, cudaStream_t s) {
  return kv_copy(k, v, kp, vp, dtype, n_rows, hkv, d, src_stride, table, page_size, row0, true, s);
}

int kv_read(const void* kp, const void* vp, int dtype, const int32_t* table, int page_size,
            int64_t row0, int64_t n_rows, int hkv, int d, void* kd, void* vd, cudaStream_t s) {
  return kv_copy(kd, vd, const_cast<void*>(kp), const_cast<void*>(vp), dtype, n_rows, hkv, d,
                 (int64_t)hkv * d, table, page_size, row0, false, s);
}

}  // namespace star
