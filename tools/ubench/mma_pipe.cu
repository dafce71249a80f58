// Microbenchmark: tcgen05.mma execution rate when issued the way K1 issues it (the converged
// warp, one elect.sync per batch: umma_ss_d128_warp / umma_ts_x4_warp / umma_ts_x8_warp), and
// its sensitivity to what the other warps of the SM do meanwhile.  One CTA per SM, operands
// resident (zeros).  Issue modes:
//   0  SS M128 N128, K = 128 per batch (QK^T of one 128-key tile)
//   1  TS M128 N128, A from TMEM (P.V), 8 per batch
//   2  K1's mix per tile: P.V as two 4-MMA halves into O, then QK^T (8) into S
// Load on warps 1-3 while warp 0 issues:
//   0  none
//   1  shared-memory reads (ld.shared.v4 over the operand tiles)
//   2  shared-memory writes to a scratch region (what TMA fills of K/V cost)
//   3  TMEM loads (tcgen05.ld 32x32b.x32 + wait, as the softmax's row pass)
// Reports clocks per MMA (floor 64 for M128 N128 K16 at 8192 dense bf16 FLOP/clk/SM).
// usage: ./mma_pipe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "sm100.cuh"

using namespace star::sm100;

constexpr int kOps = 65536;           // operand tiles (A at 0, B at 32K)
constexpr int kScratch = 65536;       // write target of load mode 2
constexpr int kSmem = kOps + kScratch + 2048;

__global__ void __launch_bounds__(128, 1) kern(int mode, int load, int reps, long long* out,
                                               unsigned long long* sink) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + kOps + kScratch);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  volatile int* stop = reinterpret_cast<volatile int*>(bar + 2);
  for (int i = threadIdx.x; i < (kOps + kScratch) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
    *stop = 0;
  }
  if (threadIdx.x < 32) tmem_alloc<512>(slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    const uint32_t idss = umma_idesc_bf16(128, 128, false, false);
    const uint32_t idts = umma_idesc_bf16(128, 128, false, true);
    const uint64_t ad = umma_desc_sw128(a, 16, 1024);
    const uint64_t bd = umma_desc_sw128(b, 16, 1024);
    const uint64_t bmn = umma_desc_sw128(b, 16384, 1024);
    long long t0 = 0;
    for (int it = 0; it < reps + 1; ++it) {
      if (it == 1) t0 = clock64();
      for (int g = 0; g < 4; ++g) {  // 64 MMAs per commit
        if (mode == 0) {
          umma_ss_d128_warp(tbase, ad, bd, idss, 1u);
          umma_ss_d128_warp(tbase + 128, ad, bd, idss, 1u);
        } else if (mode == 1) {
          umma_ts_x8_warp(tbase + 256, tbase + 384, bmn, idts, 1u);
          umma_ts_x8_warp(tbase + 256, tbase + 416, bmn, idts, 1u);
        } else {
          umma_ts_x4_warp(tbase + 256, tbase + 384, bmn, idts, 1u);
          umma_ts_x4_warp(tbase + 256, tbase + 416, bmn, idts, 1u);
          umma_ss_d128_warp(tbase, ad, bd, idss, 0u);
        }
      }
      umma_commit_warp(bar);
      mbar_wait(bar, it & 1);
    }
    const long long t1 = clock64();
    if (lane == 0) {
      const int per = mode == 2 ? 4 * 16 : 4 * 16;
      out[blockIdx.x] = (t1 - t0) / per;  // clocks per MMA x reps
      *stop = 1;
    }
  } else if (load != 0) {
    unsigned long long acc = 0;
    const int w = warp - 1;
    int n = 0;
    while (!*stop) {
      if (load == 1) {
#pragma unroll 4
        for (int i = 0; i < 64; ++i) {
          const uint32_t ad = smem_u32(smem) + (((w * 2048 + i * 32 + lane) & 4095) << 4);
          uint32_t x, y, z, v;
          asm volatile("ld.volatile.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(x), "=r"(y), "=r"(z), "=r"(v) : "r"(ad));
          acc += x ^ v;
        }
      } else if (load == 2) {
#pragma unroll 4
        for (int i = 0; i < 64; ++i)
          asm volatile("st.volatile.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(
                           smem_u32(smem + kOps) + (((w * 1365 + i * 32 + lane) & 4095) << 4)),
                       "r"(i), "r"(n), "r"(0), "r"(0));
      } else {
        uint32_t r[32];
        // warps 1-3 read their TMEM lane quarter (w + 1) of the O columns
        tmem_ld32(tbase + ((uint32_t)((warp & 3) * 32) << 16) + 256 + (n & 3) * 32, r);
        tmem_wait_ld_tied(r);
        acc += r[0] ^ r[31];
      }
      ++n;
    }
    if (acc == 0x123456789ull) sink[0] = acc;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_free<512>(tbase);
}

int main() {
  long long* d;
  unsigned long long* sink;
  cudaMalloc(&d, 148 * 8);
  cudaMalloc(&sink, 8);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
  const char* modes[] = {"SS N128 (QK^T)", "TS N128 (P.V)", "K1 tile mix (4+4 TS, 8 SS)"};
  const char* loads[] = {"idle", "smem reads", "smem writes", "TMEM loads"};
  const int reps = 200;
  for (int mode = 0; mode < 3; ++mode)
    for (int load = 0; load < 4; ++load) {
      kern<<<148, 128, kSmem>>>(mode, load, reps, d, sink);
      cudaError_t e = cudaDeviceSynchronize();
      long long h[148];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < 148; ++i) avg += h[i];
      avg /= 148;
      printf("%-28s + %-12s %7.1f clk per MMA  (%s)\n", modes[mode], loads[load], avg / reps,
             cudaGetErrorString(e));
    }
  return 0;
}
