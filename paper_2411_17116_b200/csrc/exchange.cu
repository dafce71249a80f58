// Peer exchange of phase-2 partials (the fused C1; layout and protocol in exchange.cuh).
//
//  - star_ipc_*: map another rank's box into this process (CUDA IPC over NVLink/NVSwitch).
//  - exchange_push_kernel: deliver an already computed local partial (the fp32 check-mode
//    K2, or an empty cache's lse = -inf partial) into every box; the bf16 K2 pushes from
//    its own epilogue instead (phase2_mma.cu).
//  - exchange_merge_kernel (K3x): wait until every rank's words of the row carry the epoch
//    in flight, then fold the slots in ascending rank order with the merge rule of merge_partials
//    (ss/attention.py:154-173): s = logaddexp-reduce(lse_r), out = sum_r exp(lse_r - s) out_r,
//    weights in fp64; ranks with lse = -inf (empty caches, ss/sim.py:193-194) weigh 0.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "common.cuh"
#include "exchange.cuh"

namespace star {

PeerPush make_push(const ExchangeLayout& L, void* const* boxes, int rank) {
  PeerPush pp{};
  pp.L = L;
  pp.rank = rank;
  pp.merge = 0;
  for (int r = 0; r < L.world; ++r) pp.box[r] = boxes[r];
  return pp;
}

static int check_box(const ExchangeLayout& L, int64_t rows, int groups) {
  if (L.world < 1 || L.world > kMaxPeers)
    return fail(STAR_ENOTSUP, "exchange: world %d not in [1, %d]", L.world, kMaxPeers);
  if (L.rows < 1 || L.groups < 1 || L.d < 1) return fail(STAR_ESHAPE, "exchange: empty box");
  if (rows > L.rows || groups > L.groups)
    return fail(STAR_ESHAPE, "exchange: call needs %lld rows / %d groups, the box holds %lld / %d",
                (long long)rows, groups, (long long)L.rows, L.groups);
  return STAR_OK;
}

int check_exchange(const ExchangeLayout& L, void* const* boxes, int rank, int64_t rows,
                   int groups) {
  int rc = check_box(L, rows, groups);
  if (rc) return rc;
  if (rank < 0 || rank >= L.world) return fail(STAR_ECONFIG, "exchange: rank %d of %d", rank, L.world);
  if (boxes == nullptr) return fail(STAR_ESHAPE, "exchange: boxes is NULL");
  for (int r = 0; r < L.world; ++r)
    if (boxes[r] == nullptr) return fail(STAR_ESHAPE, "exchange: box of rank %d is NULL", r);
  return STAR_OK;
}

static int check_shape(int batch, int lq, int hq, int hkv, int d) {
  if (batch < 1 || lq < 1 || hq < 1 || hkv < 1 || hq % hkv || d < 1)
    return fail(STAR_ESHAPE, "exchange: bad shape (batch=%d lq=%d hq=%d hkv=%d d=%d)", batch, lq,
                hq, hkv, d);
  return STAR_OK;
}

// one CTA per (sequence, kv head) group: copy the group's rows into this rank's slot of
// every box as {value, epoch} words
__global__ void __launch_bounds__(256) exchange_push_kernel(const float* __restrict__ out,
                                                            const float* __restrict__ lse, int lq,
                                                            int hq, int hkv, int d,
                                                            const PeerPush pp) {
  const int g = blockIdx.x;
  const int b = g / hkv, kvh = g % hkv, G = hq / hkv;
  const int QR = G * lq;
  const uint32_t ep = exchange_epoch(pp);
  for (int e = threadIdx.x; e < QR * d; e += blockDim.x) {
    const int rr = e / d, c = e % d;
    const int64_t orow = ((int64_t)b * lq + rr / G) * hq + kvh * G + rr % G;
    put_out(pp, ep, false, nullptr, orow * d + c, __ldcg(out + orow * d + c));
    if (c == 0) put_lse(pp, ep, false, nullptr, orow, __ldcg(lse + orow));
  }
}

int push_partial(const float* out, const float* lse, int batch, int lq, int hq, int hkv, int d,
                 const PeerPush& pp, cudaStream_t s) {
  exchange_push_kernel<<<batch * hkv, 256, 0, s>>>(out, lse, lq, hq, hkv, d, pp);
  STAR_LAUNCH_CHECK("exchange_push");
  return STAR_OK;
}

constexpr int kXWarps = 8;

// K3x.  One warp per output row; lane j holds head-dim columns j, j + 32, ... (NW of them).
// The lanes poll their words of every rank's slot until all carry the epoch in flight, then
// fold the ranks in ascending order with fp64 weights like merge_partials.  The last CTA to
// finish advances the box's epoch counter (every CTA read it before arriving).
template <typename TO, int NW>
__global__ void __launch_bounds__(kXWarps * 32) exchange_merge_kernel(
    void* box, ExchangeLayout L, int64_t nrows, uint64_t timeout_ns, TO* __restrict__ out,
    float* __restrict__ lse) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = blockIdx.x * (int64_t)kXWarps + warp;
  uint32_t* hdr = L.header(box);
  const uint32_t epoch = next_epoch(__ldcg(hdr));
  const int par = (int)(epoch & 1u);
  const int d = L.d;
  if (row < nrows) {
    float ov[kMaxPeers][NW];
    float lv = -INFINITY;  // lane r < world: rank r's lse
    uint64_t t0 = 0;
    for (int r = 0; r < L.world; ++r) {
      const uint2* sl = L.slot(box, par, r);
      for (;;) {
        bool ok = true;
        uint2 w[NW + 1];
#pragma unroll
        for (int j = 0; j < NW; ++j)
          w[j] = (lane + 32 * j < d) ? ld_word(sl + row * d + lane + 32 * j) : make_uint2(0u, epoch);
        w[NW] = ld_word(sl + L.rows * d + row);
#pragma unroll
        for (int j = 0; j <= NW; ++j) ok &= w[j].y == epoch;
        if (__all_sync(0xffffffffu, ok)) {
#pragma unroll
          for (int j = 0; j < NW; ++j) ov[r][j] = __uint_as_float(w[j].x);
          if (lane == r) lv = __uint_as_float(w[NW].x);
          break;
        }
        if (t0 == 0) t0 = globaltimer_ns();
        if (globaltimer_ns() - t0 > timeout_ns) {
          if (lane == 0)
            printf("star exchange: rank %d never delivered row %lld of epoch %u (timeout)\n", r,
                   (long long)row, epoch);
          __trap();  // fail loudly instead of hanging the stream
        }
      }
    }
    double mx = (lane < L.world) ? (double)lv : -INFINITY;
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const double e = (lane < L.world && lv != -INFINITY) ? exp((double)lv - mx) : 0.0;
    double acc = e;
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    const float inv = acc > 0.0 ? (float)(1.0 / acc) : 0.f;
    float o[NW] = {};
    for (int r = 0; r < L.world; ++r) {
      const float w = __shfl_sync(0xffffffffu, (float)e, r);
#pragma unroll
      for (int j = 0; j < NW; ++j) o[j] = fmaf(w, ov[r][j], o[j]);
    }
#pragma unroll
    for (int j = 0; j < NW; ++j)
      if (lane + 32 * j < d) out[row * d + lane + 32 * j] = Elem<TO>::from_f(o[j] * inv);
    if (lse != nullptr && lane == 0) lse[row] = acc > 0.0 ? (float)(mx + log(acc)) : -INFINITY;
  }
  // every CTA has read the epoch before it arrives; the last arrival advances it
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(hdr + 1, 1u) == gridDim.x - 1) {
      hdr[1] = 0;
      hdr[0] = epoch;
      __threadfence();
    }
  }
}

static bool pdl_enabled() {  // STAR_EXCHANGE_PDL=0 turns the early launch off (measurement)
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("STAR_EXCHANGE_PDL");
    v = (e != nullptr && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

uint64_t spin_timeout_ns() {
  static uint64_t t = 0;
  if (t == 0) {
    const char* e = getenv("STAR_EXCHANGE_TIMEOUT_S");
    double s = e ? atof(e) : 30.0;
    if (!(s > 0)) s = 30.0;
    t = (uint64_t)(s * 1e9);
  }
  return t;
}

int exchange_push(const float* out, const float* lse, int batch, int lq, int hq, int hkv, int d,
                  void* const* boxes, const ExchangeLayout& L, int rank, cudaStream_t s) {
  int rc = check_shape(batch, lq, hq, hkv, d);
  if (rc) return rc;
  if (out == nullptr || lse == nullptr) return fail(STAR_ESHAPE, "exchange push: NULL partial");
  rc = check_exchange(L, boxes, rank, (int64_t)batch * lq * hq, batch * hkv);
  if (rc) return rc;
  return push_partial(out, lse, batch, lq, hq, hkv, d, make_push(L, boxes, rank), s);
}

int exchange_merge(void* box, const ExchangeLayout& L, int batch, int lq, int hq, int hkv, int d,
                   void* out, int out_dtype, float* lse, cudaStream_t s) {
  int rc = check_shape(batch, lq, hq, hkv, d);
  if (rc) return rc;
  if (out == nullptr || box == nullptr) return fail(STAR_ESHAPE, "exchange merge: NULL pointer");
  const int64_t nrows = (int64_t)batch * lq * hq;
  rc = check_box(L, nrows, batch * hkv);
  if (rc) return rc;
  if (d > 128) return fail(STAR_ENOTSUP, "exchange: head_dim %d > 128", d);
  const int grid = (int)((nrows + kXWarps - 1) / kXWarps);
  const uint64_t to = spin_timeout_ns();
  // Programmatic dependent launch: K3x may start while the producer kernel (K2 / push) is
  // still running — it needs none of its results beyond the epoch words it polls — so its
  // launch latency hides under K2 (K2 triggers at entry).  The header epoch it reads was
  // advanced by the previous K3x, which completed before the producer started.
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kXWarps * 32);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
#define STAR_XM(TO, NW) \
  cudaLaunchKernelEx(&cfg, exchange_merge_kernel<TO, NW>, box, L, nrows, to, (TO*)out, lse)
#define STAR_XM_D(TO) \
  do { if (d <= 32) STAR_XM(TO, 1); else if (d <= 64) STAR_XM(TO, 2); else STAR_XM(TO, 4); } while (0)
  if (out_dtype == STAR_F32)
    STAR_XM_D(float);
  else if (out_dtype == STAR_BF16)
    STAR_XM_D(__nv_bfloat16);
  else
    return fail(STAR_ECONFIG, "exchange merge: unknown dtype %d", out_dtype);
#undef STAR_XM_D
#undef STAR_XM
  STAR_LAUNCH_CHECK("exchange_merge");
  return STAR_OK;
}

// ---------------------------------------------------------------- CUDA IPC
static_assert(sizeof(cudaIpcMemHandle_t) == STAR_IPC_HANDLE_BYTES, "IPC handle size");

int ipc_get_handle(const void* ptr, void* handle, int64_t* offset) {
  if (ptr == nullptr || handle == nullptr || offset == nullptr)
    return fail(STAR_ESHAPE, "ipc: NULL argument");
  // the handle names the whole allocation; the caller's pointer may sit inside it
  static PFN_cuMemGetAddressRange_v3020 range = nullptr;
  if (range == nullptr) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        fn == nullptr)
      return fail(STAR_ECUDA, "ipc: cuMemGetAddressRange unavailable");
    range = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(fn);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, (CUdeviceptr)ptr) != CUDA_SUCCESS)
    return fail(STAR_ECUDA, "ipc: pointer %p is not device memory", ptr);
  cudaIpcMemHandle_t h;
  STAR_CUDA_CHECK(cudaIpcGetMemHandle(&h, (void*)base));
  memcpy(handle, &h, sizeof(h));
  *offset = (int64_t)((CUdeviceptr)ptr - base);
  return STAR_OK;
}

int ipc_open_handle(const void* handle, int64_t offset, void** ptr) {
  if (handle == nullptr || ptr == nullptr) return fail(STAR_ESHAPE, "ipc: NULL argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  void* base = nullptr;
  STAR_CUDA_CHECK(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
  *ptr = static_cast<char*>(base) + offset;
  return STAR_OK;
}

int ipc_close_handle(void* ptr, int64_t offset) {
  if (ptr == nullptr) return STAR_OK;
  STAR_CUDA_CHECK(cudaIpcCloseMemHandle(static_cast<char*>(ptr) - offset));
  return STAR_OK;
}

}  // namespace star
