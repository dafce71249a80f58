// Microbenchmark: tcgen05.mma issue-to-completion rate per instruction on sm_100a, one CTA
// per SM, operands resident (zeros) in shared memory / TMEM.  Modes:
//   0  SS  M128 N128 K16, K-major A and B, one accumulator (K1 / K2q QK^T)
//   1  TS  M128 N128 K16, A from TMEM, B MN-major (K1 / K2q P.V)
//   2  SS  M128 N256 K16 (one MMA covering two 128-key tiles)
//   3  TS  alternating two accumulators
//   4  SS then TS, 8 + 16 (the K2q tile mix)
// 64 MMAs per commit + wait.  Reports clocks per MMA (peak 64 for M128 N128 K16 at 8192
// dense bf16 FLOP/clk/SM; 32 for N64, 128 for N256).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "sm100.cuh"

using namespace star::sm100;

__global__ void __launch_bounds__(128, 1) kern(int mode, int reps, long long* out) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 65536);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  for (int i = threadIdx.x; i < 65536 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  if (threadIdx.x < 32) tmem_alloc<512>(slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *slot;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    const uint32_t id128 = umma_idesc_bf16(128, 128, false, false);
    const uint32_t id256 = umma_idesc_bf16(128, 256, false, false);
    const uint32_t idts = umma_idesc_bf16(128, 128, false, true);
    long long t0 = 0;
    for (int it = 0; it < reps + 1; ++it) {
      if (it == 1) t0 = clock64();
      for (int kk = 0; kk < 64; ++kk) {
        const uint64_t ad = umma_desc_sw128(a + (kk & 3) * 32, 16, 1024);
        const uint64_t bd = umma_desc_sw128(b + (kk & 3) * 32, 16, 1024);
        const uint64_t bmn = umma_desc_sw128(b + (kk & 7) * 16 * 128, 16384, 1024);
        if (mode == 0) umma_bf16_ss(tbase, ad, bd, id128, 1u);
        if (mode == 1) umma_bf16_ts(tbase, tbase + 384 + (kk & 7) * 8, bmn, idts, 1u);
        if (mode == 2) umma_bf16_ss(tbase, ad, bd, id256, 1u);
        if (mode == 3) umma_bf16_ts(tbase + (kk & 1) * 128, tbase + 384 + (kk & 7) * 8, bmn, idts, 1u);
        if (mode == 4) {
          if ((kk % 24) < 8) umma_bf16_ss(tbase, ad, bd, id128, 1u);
          else umma_bf16_ts(tbase + 128, tbase + 384 + (kk & 7) * 8, bmn, idts, 1u);
        }
        if (mode == 5) umma_bf16_ss(tbase + (kk & 3) * 64, ad, bd, umma_idesc_bf16(128, 64, false, false), 1u);
        if (mode == 6) umma_bf16_ss(tbase + (kk & 1) * 128, ad, bd, id128, 1u);
      }
      umma_commit(bar);
      mbar_wait(bar, it & 1);
    }
    const long long t1 = clock64();
    out[blockIdx.x] = (t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_free<512>(tbase);
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 2048);
  const char* names[] = {"SS N128 one acc", "TS N128 one acc", "SS N256 one acc",
                         "TS N128 two accs", "SS x8 then TS x16 (K2q-like mix)",
                         "SS N64 four accs", "SS N128 two accs"};
  const int reps = 200;
  for (int mode = 0; mode < 7; ++mode) {
    kern<<<148, 128, 65536 + 2048>>>(mode, reps, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148;
    printf("%-34s %7.1f clk per MMA  (%s)\n", names[mode], avg / (reps * 64.0),
           cudaGetErrorString(e));
  }
  return 0;
}
