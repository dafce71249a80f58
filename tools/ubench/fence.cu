// Microbenchmark: cost of the release/acquire variants a peer-exchange producer/consumer can
// use on sm_100a.  One CTA of 256 threads stores 16.5 KB (a decode partial) into a buffer,
// then thread 0 publishes a flag with variant V; a second kernel in the same stream polls
// the flag with variant A and reads the data back.  Launch pairs are replayed from a CUDA
// graph; the time per pair is reported against the no-fence baseline.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void st_rel_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_rel_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_rlx_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acq_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_rlx_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_vol(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

constexpr int N = 4128;  // 32 x 129 floats

// V: 0 none (plain store of flag), 1 threadfence_system + st.release.sys, 2 st.release.sys,
//    3 threadfence (gpu) + st.relaxed.sys, 4 fence.acq_rel.sys + st.relaxed.sys,
//    5 st.release.gpu, 6 LL: (value, flag) 64-bit stores, no fence
template <int V>
__global__ void produce(float* data, uint2* ll, uint32_t* flag, uint32_t epoch) {
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    if (V == 6) {
      uint2 w = make_uint2(__float_as_uint(1.0f * i), epoch);
      asm volatile("st.volatile.global.v2.u32 [%0], {%1, %2};" ::"l"(ll + i), "r"(w.x), "r"(w.y) : "memory");
    } else {
      data[i] = 1.0f * i + epoch;
    }
  }
  if (V == 6) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    if (V == 0) *(volatile uint32_t*)flag = epoch;
    if (V == 1) { __threadfence_system(); st_rel_sys(flag, epoch); }
    if (V == 2) st_rel_sys(flag, epoch);
    if (V == 3) { __threadfence(); st_rlx_sys(flag, epoch); }
    if (V == 4) { asm volatile("fence.acq_rel.sys;" ::: "memory"); st_rlx_sys(flag, epoch); }
    if (V == 5) st_rel_gpu(flag, epoch);
  }
}

// A: 0 ld.volatile, 1 ld.acquire.sys, 2 ld.relaxed.sys + fence.acq_rel.sys, 3 LL poll
template <int A>
__global__ void consume(const float* data, const uint2* ll, const uint32_t* flag, uint32_t epoch,
                        float* sink) {
  float acc = 0.f;
  if (A == 3) {
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
      uint2 w;
      do {
        asm volatile("ld.volatile.global.v2.u32 {%0, %1}, [%2];" : "=r"(w.x), "=r"(w.y) : "l"(ll + i) : "memory");
      } while (w.y != epoch);
      acc += __uint_as_float(w.x);
    }
  } else {
    if (A == 0) while (ld_vol(flag) != epoch) {}
    if (A == 1) while (ld_acq_sys(flag) != epoch) {}
    if (A == 2) { while (ld_rlx_sys(flag) != epoch) {} asm volatile("fence.acq_rel.sys;" ::: "memory"); }
    for (int i = threadIdx.x; i < N; i += blockDim.x) acc += __ldcg(data + i);
  }
  if (acc == -1.f) *sink = acc;
}

template <int V, int A>
float run(float* data, uint2* ll, uint32_t* flag, float* sink, cudaStream_t s) {
  // epochs must advance per pair: graph of 20 pairs with epochs e0..e0+19 re-captured per rep
  static uint32_t e = 1;
  cudaGraph_t g;
  cudaGraphExec_t ge;
  const int pairs = 20, reps = 20;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float total = 0.f;
  for (int r = 0; r < reps + 2; ++r) {
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int p = 0; p < pairs; ++p, ++e) {
      produce<V><<<1, 256, 0, s>>>(data, ll, flag, e);
      consume<A><<<1, 256, 0, s>>>(data, ll, flag, e, sink);
    }
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphUpload(ge, s);
    cudaStreamSynchronize(s);
    cudaEventRecord(a, s);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(b, s);
    cudaStreamSynchronize(s);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (r >= 2) total += ms;
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
  }
  return total / (reps * pairs) * 1e3f;
}

int main() {
  float *data, *sink;
  uint2* ll;
  uint32_t* flag;
  cudaMalloc(&data, N * 4);
  cudaMalloc(&ll, N * 8);
  cudaMalloc(&flag, 4);
  cudaMalloc(&sink, 4);
  cudaMemset(flag, 0, 4);
  cudaMemset(ll, 0, N * 8);
  cudaStream_t s;
  cudaStreamCreate(&s);
  printf("us per produce+consume pair (graph replay):\n");
  printf("none/volatile                 %.2f\n", run<0, 0>(data, ll, flag, sink, s));
  printf("fence_sys+rel_sys/acq_sys     %.2f\n", run<1, 1>(data, ll, flag, sink, s));
  printf("rel_sys/acq_sys               %.2f\n", run<2, 1>(data, ll, flag, sink, s));
  printf("fence_gpu+rlx_sys/acq_sys     %.2f\n", run<3, 1>(data, ll, flag, sink, s));
  printf("fence_acqrel_sys+rlx/acq_sys  %.2f\n", run<4, 1>(data, ll, flag, sink, s));
  printf("rel_gpu/acq_sys               %.2f\n", run<5, 1>(data, ll, flag, sink, s));
  printf("rel_sys/rlx_sys+fence         %.2f\n", run<2, 2>(data, ll, flag, sink, s));
  printf("LL (value,flag) 64-bit        %.2f\n", run<6, 3>(data, ll, flag, sink, s));
  printf("none/acq_sys                  %.2f\n", run<0, 1>(data, ll, flag, sink, s));
  cudaError_t err = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(err));
  return 0;
}
