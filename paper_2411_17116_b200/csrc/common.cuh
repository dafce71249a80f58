// Shared host/device helpers for the star-attention sm_100a library.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include <algorithm>

#include "../../include/star_attn.h"

namespace star {

// ---- error reporting (thread-local message, read through star_last_error) ----
void set_error(const char* fmt, ...);
int fail(int code, const char* fmt, ...);

#define STAR_CUDA_CHECK(expr)                                                              \
  do {                                                                                     \
    cudaError_t _e = (expr);                                                               \
    if (_e != cudaSuccess)                                                                 \
      return ::star::fail(STAR_ECUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), \
                          __FILE__, __LINE__);                                             \
  } while (0)

#define STAR_LAUNCH_CHECK(name)                                                            \
  do {                                                                                     \
    cudaError_t _e = cudaGetLastError();                                                   \
    if (_e != cudaSuccess)                                                                 \
      return ::star::fail(STAR_ECUDA, "launch of %s failed: %s", name, cudaGetErrorString(_e)); \
  } while (0)

int num_sms();

// ---- element conversion ----
template <typename T> struct Elem;
template <> struct Elem<float> {
  static __device__ __forceinline__ float load(const float* p) { return *p; }
  static __device__ __forceinline__ float to_f(float x) { return x; }
  static __device__ __forceinline__ float from_f(float x) { return x; }
};
template <> struct Elem<__nv_bfloat16> {
  static __device__ __forceinline__ float load(const __nv_bfloat16* p) { return __bfloat162float(*p); }
  static __device__ __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
  static __device__ __forceinline__ __nv_bfloat16 from_f(float x) { return __float2bfloat16_rn(x); }
};

__device__ __forceinline__ float bf16lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

// max segments per phase-1 launch (passed by value in the kernel parameter block)
constexpr int kMaxSegments = 64;

struct SegTable {
  int n;
  int64_t q_row0[kMaxSegments];   // first q row of segment (in the q/out tensors)
  int64_t k_row0[kMaxSegments];   // first k row of segment (in the k/v tensors)
  int32_t lq[kMaxSegments];
  int32_t lk[kMaxSegments];
  int32_t q_offset[kMaxSegments]; // absolute index of q row 0 relative to k row 0 (causal)
  int32_t tile_start[kMaxSegments + 1];  // cumulative q tiles
  // anchor dedup: the first dedup_tiles 128-row q tiles of every segment
  // s >= 1 repeat segment 0's rows exactly (first-block anchors); they are not launched —
  // segment 0's CTAs write their rows to every segment instead.
  int32_t dedup_tiles = 0;
  // first launched 128-row q tile of a segment (query-row ranges, star_phase1_fwd_range);
  // rows below it are neither computed nor written
  int32_t tile_lo[kMaxSegments] = {};
};

}  // namespace star
