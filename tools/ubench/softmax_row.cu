// Microbenchmark of K1's per-tile softmax instruction stream (128 scores per thread:
// FFMA2 scale-subtract, MUFU.EX2, bf16x2 pack, f32+=bf16 row sum), registers only.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 r;
  asm("{\n\t.reg .b64 a, b, c, d;\n\tmov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\tmov.b64 c, {%6, %7};\n\t"
      "fma.rn.f32x2 d, a, b, c;\n\tmov.b64 {%0, %1}, d;\n\t}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return r;
}
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ uint32_t pack(float lo, float hi) { uint32_t r; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo)); return r; }
__device__ __forceinline__ void acc2(float& a, float& b, uint32_t w) {
  asm("{\n\t.reg .b16 lo, hi;\n\tmov.b32 {lo, hi}, %2;\n\tadd.rn.f32.bf16 %0, lo, %0;\n\tadd.rn.f32.bf16 %1, hi, %1;\n\t}" : "+f"(a), "+f"(b) : "r"(w));
}

__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  float2 r;
  asm("{\n\t.reg .b64 a, b, d;\n\tmov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\t"
      "add.rn.f32x2 d, a, b;\n\tmov.b64 {%0, %1}, d;\n\t}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
__device__ __forceinline__ float2 poly_ex2x2(float2 x) {
  constexpr float kMagic = 12582912.0f;
  x.x = fmaxf(x.x, -125.f);
  x.y = fmaxf(x.y, -125.f);
  const float2 t = fadd2(x, make_float2(kMagic, kMagic));
  const float2 r = fadd2(t, make_float2(-kMagic, -kMagic));
  const float2 f = fadd2(x, make_float2(-r.x, -r.y));
  float2 p = ffma2(f, make_float2(0.05484800413f, 0.05484800413f), make_float2(0.24180661142f, 0.24180661142f));
  p = ffma2(p, f, make_float2(0.69324821234f, 0.69324821234f));
  p = ffma2(p, f, make_float2(0.99998867512f, 0.99998867512f));
  return make_float2(__int_as_float(__float_as_int(t.x) * 8388608 + __float_as_int(p.x)),
                     __int_as_float(__float_as_int(t.y) * 8388608 + __float_as_int(p.y)));
}

template <int MODE>
__global__ void kern(float* out, int iters, long long* cyc) {
  float sv[128];
#pragma unroll
  for (int i = 0; i < 128; ++i) sv[i] = 0.0071f * i + 0.001f * threadIdx.x;
  uint32_t chk = 0;
  float tot = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const float m = 0.3f + 1e-6f * it;
    const float2 sc2 = make_float2(1.44f, 1.44f), nm2 = make_float2(-m, -m);
    float2 rs[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      float p[32];
#pragma unroll
      for (int e = 0; e < 32; e += 2) {
        float2 x = ffma2(make_float2(sv[c * 32 + e], sv[c * 32 + e + 1]), sc2, nm2);
        const bool poly = MODE == 2 || MODE == 3 ? c >= 6 - MODE
                        : (MODE == 4 || MODE == 7) ? ((e >> 1) & 3) == 3
                        : MODE == 5 ? ((e >> 1) & 7) == 7 : false;
        if (poly) {  // MODE 2: chunk 3 on FMA; 3: chunks 2-3; 4: every 4th pair; 5: every 8th
          float2 q = poly_ex2x2(x);
          p[e] = q.x;
          p[e + 1] = q.y;
        } else {
          p[e] = ex2(x.x);
          p[e + 1] = ex2(x.y);
        }
      }
#pragma unroll
      for (int e = 0; e < 32; e += 2) {
        uint32_t w = pack(p[e], p[e + 1]);
        chk ^= w;
        if (MODE >= 6)
          rs[(e >> 1) & 1] = fadd2(rs[(e >> 1) & 1], make_float2(p[e], p[e + 1]));
        else if (MODE >= 1)
          acc2(rs[(e >> 1) & 1].x, rs[(e >> 1) & 1].y, w);
      }
    }
    tot += rs[0].x + rs[0].y + rs[1].x + rs[1].y;
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = tot + (float)chk;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  float* out; long long* cyc; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 8);
  const int iters = 2048;
  for (int mode = 0; mode < 8; ++mode)
    for (int wps = 1; wps <= 3; ++wps) {
      auto k = mode == 0 ? kern<0> : mode == 1 ? kern<1> : mode == 2 ? kern<2> : mode == 3 ? kern<3>
             : mode == 4 ? kern<4> : mode == 5 ? kern<5> : mode == 6 ? kern<6> : kern<7>;
      k<<<148, 128 * wps>>>(out, 8, cyc);
      k<<<148, 128 * wps>>>(out, iters, cyc);
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      printf("mode=%s warps/SMSP=%d: %.1f clk per 128-score row per warp (MUFU floor 1024 x warps)\n",
             mode == 0 ? "exp+pack" : mode == 1 ? "exp+pack+sum" : mode == 2 ? "+sum, 1/4 poly" : mode == 3 ? "+sum, 1/2 poly" : mode == 4 ? "+sum, 1/4 poly spread" : mode == 5 ? "+sum, 1/8 poly spread" : mode == 6 ? "fadd2 sum" : "fadd2 sum, 1/4 poly spread", wps, (double)c / iters);
    }
  return 0;
}
