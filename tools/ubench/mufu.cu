// Microbenchmark: per-SM-sub-partition throughput of MUFU.EX2, F2FP (bf16x2 pack),
// FHADD.BF16 (f32 += bf16) and FFMA2 on sm_100a; W warps per SMSP, 1 CTA per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }

template <int OP>
__global__ void kern(float* out, int iters, long long* cyc) {
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = 0.001f * (threadIdx.x + i);
  uint32_t w[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) w[i] = 0x3f803f80u + i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (OP == 0) a[i] = ex2(a[i]);
      if (OP == 1) { uint32_t r; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[(i + 1) & 15])); w[i] ^= r; }
      if (OP == 2) asm volatile("{\n\t.reg .b16 lo, hi;\n\tmov.b32 {lo, hi}, %1;\n\tadd.rn.f32.bf16 %0, lo, %0;\n\t}" : "+f"(a[i]) : "r"(w[i]));
      if (OP == 4) { uint32_t r; asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(r) : "r"(w[i])); w[i] = r ^ 0x00010001u; }
      if (OP == 5) { uint32_t r; asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(r) : "r"(w[i])); w[i] = r ^ 0x00010001u; }
      if (OP == 3) asm volatile("{\n\t.reg .b64 x;\n\tmov.b64 x, {%0, %1};\n\tfma.rn.f32x2 x, x, x, x;\n\tmov.b64 {%0, %1}, x;\n\t}" : "+f"(a[i]), "+f"(a[(i + 8) & 15]));
    }
  }
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i] + (float)w[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  float* out; long long* cyc; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 8);
  const char* names[6] = {"MUFU.EX2", "F2FP.BF16.PACK", "FHADD.BF16(f32+=bf16)", "FFMA2",
                          "EX2.F16x2 (2 results)", "EX2.BF16x2 (2 results)"};
  const int iters = 4096;
  for (int op = 0; op < 6; ++op)
    for (int wps = 1; wps <= 4; wps *= 2) {
      int threads = 128 * wps;
      auto k = op == 0 ? kern<0> : op == 1 ? kern<1> : op == 2 ? kern<2> : op == 3 ? kern<3>
             : op == 4 ? kern<4> : kern<5>;
      k<<<148, threads>>>(out, 16, cyc);
      k<<<148, threads>>>(out, iters, cyc);
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      double per_warp_instr = (double)c / (iters * 16.0 * wps);  // clk per warp-instruction per SMSP
      printf("%-24s warps/SMSP=%d  clk per warp-instr per SMSP = %.2f  (lanes/clk/SM = %.1f)\n", names[op], wps,
             per_warp_instr, 4 * 32 / per_warp_instr);
    }
  return 0;
}
