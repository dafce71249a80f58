// Phase 1 (K1), variant "db64": 64-key tiles with double-buffered S/P in TMEM.
//
// Same semantics and boundary as phase1_tc.cu (causal_attention per anchor-augmented
// block, ss/attention.py:109-122 via ss/sim.py:108-123).  What changes is the TMEM plan:
// each of the NQ=2 q heads owns two 64-column S/P buffers plus its 128-column O, so the
// tensor core computes S_i(j+1) while the softmax warpgroup is still on S_i(j):
//   TMEM: [S0a S0b | S1a S1b | O0 | O1] = 2*(2*64) + 2*128 = 512 columns.
// MMA issue order per kv tile j and head i: PV_i(j) (A = P_i(j) from TMEM), then
// S_i(j+2) into the buffer P_i(j) occupied — safe because tcgen05.mma executes in
// issue order.  A 64-wide S row fits in registers, so the softmax reads TMEM once.
#include <cudaTypedefs.h>

#include "common.cuh"
#include "sm100.cuh"

namespace star {

using namespace sm100;

template <int D>
struct P1Cfg64 {
  static constexpr int NQ = 2;
  static constexpr int BM = 128, BN = 64;
  static constexpr int kQSlab = 128 * 128;          // [128 rows x 64 bf16]
  static constexpr int kKSlab = BN * 128;           // [64 rows x 64 bf16]
  static constexpr int kSlabs = D / 64;
  static constexpr int kQTile = kSlabs * kQSlab;
  static constexpr int kKTile = kSlabs * kKSlab;
  static constexpr int KST = 3, VST = 3;
  static constexpr int kQOff = 0;
  static constexpr int kKOff = kQOff + NQ * kQTile;
  static constexpr int kVOff = kKOff + KST * kKTile;
  static constexpr int kBarOff = kVOff + VST * kKTile;
  static constexpr int kNumBars = 1 + 2 * KST + 2 * VST + NQ * 2 + NQ * 2 + NQ;
  static constexpr int kSmem = kBarOff + kNumBars * 8 + 16 + 1024;
  static constexpr int kThreads = 64 + 128 * NQ;
  static constexpr int kSCols = 2 * BN;  // per head: two S/P buffers
  static_assert(NQ * (kSCols + D) <= 512, "TMEM budget");
  static_assert(kSmem <= 232448, "shared memory budget");
};

struct P1Params64 {
  SegTable segs;
  int hq, hkv;
  int64_t out_row_stride;
  int64_t lse_stride;
  float scale_log2;
  void* out;
  int out_f32;
  float* lse;
};

template <bool DIAG>
__device__ __forceinline__ void softmax_tile64(uint32_t s_tm, int lim, float sl2, float& m_run,
                                               float& alpha, float& rs, bool& need, bool first) {
  uint32_t a[32], b[32];
  tmem_ld32(s_tm, a);
  tmem_ld32(s_tm + 32, b);
  tmem_wait_ld();
  float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
  for (int e = 0; e < 32; ++e) {
    if (DIAG) {
      if (e > lim) a[e] = __float_as_uint(-INFINITY);
      if (e + 32 > lim) b[e] = __float_as_uint(-INFINITY);
    }
    m4[e & 3] = fmaxf(m4[e & 3], fmaxf(__uint_as_float(a[e]), __uint_as_float(b[e])));
  }
  const float mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])) * sl2;
  float m_use = m_run;
  alpha = 1.f;
  need = first || (mx > m_run + 8.f);
  if (need) {
    if (!first) alpha = ex2(m_run - mx);
    m_use = mx;
  }
  if (m_use == -INFINITY) m_use = 0.f;  // row with nothing visible yet (diagonal edge)
  const float2 sc2 = make_float2(sl2, sl2), nm2 = make_float2(-m_use, -m_use);
  float2 r2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
  uint32_t pk[2][16];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const uint32_t* v = h ? b : a;
#pragma unroll
    for (int e = 0; e < 32; e += 2) {
      const float2 x = ffma2(make_float2(__uint_as_float(v[e]), __uint_as_float(v[e + 1])), sc2, nm2);
      const uint32_t w = pack_bf16x2(ex2(x.x), ex2(x.y));  // ex2(-inf) = 0 for masked cells
      pk[h][e >> 1] = w;
      r2[(e >> 1) & 1] = fadd2(r2[(e >> 1) & 1], make_float2(bf16lo(w), bf16hi(w)));
    }
  }
  // P (bf16x2) over the consumed S columns: [0,16) <- cols 0..31, [16,32) <- cols 32..63
  tmem_st16(s_tm, pk[0]);
  tmem_st16(s_tm + 16, pk[1]);
  rs = (r2[0].x + r2[0].y) + (r2[1].x + r2[1].y);
  m_run = need ? m_use : m_run;
}

template <int D>
__global__ void __launch_bounds__(P1Cfg64<D>::kThreads, 1)
    phase1_tc64_kernel(const __grid_constant__ CUtensorMap tm_q,
                       const __grid_constant__ CUtensorMap tm_k,
                       const __grid_constant__ CUtensorMap tm_v,
                       const __grid_constant__ P1Params64 prm) {
  using C = P1Cfg64<D>;
  constexpr int NQ = C::NQ;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kBarOff);
  uint64_t* q_full = bars;
  uint64_t* k_full = q_full + 1;
  uint64_t* k_empty = k_full + C::KST;
  uint64_t* v_full = k_empty + C::KST;
  uint64_t* v_empty = v_full + C::VST;
  // Per-buffer S/P barriers: a softmax warpgroup may run one tile ahead of the MMA issuer,
  // so a single P barrier could be two phases ahead of its waiter and alias the parity.
  uint64_t* s_full = v_empty + C::VST;   // [NQ][2]
  uint64_t* p_full = s_full + NQ * 2;    // [NQ][2]
  uint64_t* o_done = p_full + NQ * 2;    // [NQ]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + NQ);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int y = blockIdx.y;
  int s = 0;
  while (s + 1 < prm.segs.n && prm.segs.tile_start[s + 1] <= y) ++s;
  const int ntq = prm.segs.tile_start[s + 1] - prm.segs.tile_start[s];
  const int qt = ntq - 1 - (y - prm.segs.tile_start[s]);
  const int G = prm.hq / prm.hkv;
  const int pairs = G / NQ;
  const int kvh = blockIdx.x / pairs;
  const int h0 = kvh * G + (blockIdx.x % pairs) * NQ;
  const int lq = prm.segs.lq[s];
  const int q_row0 = (int)prm.segs.q_row0[s];
  const int k_row0 = (int)prm.segs.k_row0[s];
  const int nkv = 2 * qt + 2;  // 64-key tiles up to the diagonal of the 128-row q tile

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < C::KST; ++i) { mbar_init(&k_full[i], 1); mbar_init(&k_empty[i], 1); }
    for (int i = 0; i < C::VST; ++i) { mbar_init(&v_full[i], 1); mbar_init(&v_empty[i], 1); }
    for (int i = 0; i < NQ; ++i) {
      mbar_init(&s_full[2 * i], 1);
      mbar_init(&s_full[2 * i + 1], 1);
      mbar_init(&p_full[2 * i], 4);
      mbar_init(&p_full[2 * i + 1], 4);
      mbar_init(&o_done[i], 1);
    }
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch(&tm_q);
      tma_prefetch(&tm_k);
      mbar_expect_tx(q_full, NQ * C::kQTile);
      for (int i = 0; i < NQ; ++i)
        for (int a = 0; a < C::kSlabs; ++a)
          tma_load_3d(smem + C::kQOff + i * C::kQTile + a * C::kQSlab, &tm_q, q_full, a * 64,
                      h0 + i, q_row0 + qt * C::BM);
      for (int j = 0; j < nkv; ++j) {
        const int st = j % C::KST;
        if (j >= C::KST) mbar_wait(&k_empty[st], ((j / C::KST) + 1) & 1);
        mbar_expect_tx(&k_full[st], C::kKTile);
        for (int a = 0; a < C::kSlabs; ++a)
          tma_load_3d(smem + C::kKOff + st * C::kKTile + a * C::kKSlab, &tm_k, &k_full[st], a * 64,
                      kvh, k_row0 + j * C::BN);
      }
    } else if (lane == 1) {
      tma_prefetch(&tm_v);
      for (int j = 0; j < nkv; ++j) {
        const int st = j % C::VST;
        if (j >= C::VST) mbar_wait(&v_empty[st], ((j / C::VST) + 1) & 1);
        mbar_expect_tx(&v_full[st], C::kKTile);
        for (int a = 0; a < C::kSlabs; ++a)
          tma_load_3d(smem + C::kVOff + st * C::kKTile + a * C::kKSlab, &tm_v, &v_full[st], a * 64,
                      kvh, k_row0 + j * C::BN);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_s = umma_idesc_bf16(128, C::BN, false, false);
      constexpr uint32_t idesc_o = umma_idesc_bf16(128, D, false, true);
      const uint32_t q_addr = smem_u32(smem + C::kQOff);
      const uint32_t k_addr = smem_u32(smem + C::kKOff);
      const uint32_t v_addr = smem_u32(smem + C::kVOff);
      auto s_col = [&](int i, int buf) { return tbase + i * C::kSCols + buf * C::BN; };
      auto issue_s = [&](int j) {  // S_i(j) for both heads from K tile j
        const int st = j % C::KST;
        mbar_wait(&k_full[st], (j / C::KST) & 1);
        tc_fence_after();
        for (int i = 0; i < NQ; ++i) {
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t qoff = (kk >> 2) * C::kQSlab + (kk & 3) * 32;
            const uint32_t koff = (kk >> 2) * C::kKSlab + (kk & 3) * 32;
            umma_bf16_ss(s_col(i, j & 1), umma_desc_sw128(q_addr + i * C::kQTile + qoff, 16, 1024),
                         umma_desc_sw128(k_addr + st * C::kKTile + koff, 16, 1024), idesc_s,
                         kk > 0 ? 1u : 0u);
          }
          umma_commit(&s_full[2 * i + (j & 1)]);
        }
        umma_commit(&k_empty[st]);
      };
      mbar_wait(q_full, 0);
      issue_s(0);
      issue_s(1);
      for (int j = 0; j < nkv; ++j) {
        const int vs = j % C::VST;
        mbar_wait(&v_full[vs], (j / C::VST) & 1);
        for (int i = 0; i < NQ; ++i) {
          mbar_wait(&p_full[2 * i + (j & 1)], (j >> 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < C::BN / 16; ++kk)
            umma_bf16_ts(tbase + NQ * C::kSCols + i * D, s_col(i, j & 1) + kk * 8,
                         umma_desc_sw128(v_addr + vs * C::kKTile + kk * 16 * 128, C::kKSlab, 1024),
                         idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
          umma_commit(&o_done[i]);
        }
        umma_commit(&v_empty[vs]);
        if (j + 2 < nkv) issue_s(j + 2);
      }
    }
  } else {
    const int i = (warp - 2) >> 2;
    const int wq = warp & 3;
    const int r = wq * 32 + lane;
    const int qrow = qt * C::BM + r;
    const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
    const uint32_t o_tm = tbase + lane_off + NQ * C::kSCols + i * D;
    const float sl2 = prm.scale_log2;
    float m_run = -INFINITY, l_run = 0.f;
    for (int j = 0; j < nkv; ++j) {
      const uint32_t s_tm = tbase + lane_off + i * C::kSCols + (j & 1) * C::BN;
      mbar_wait(&s_full[2 * i + (j & 1)], (j >> 1) & 1);
      tc_fence_after();
      const int lim = qrow - j * C::BN;
      float alpha, rs;
      bool need;
      if (j >= 2 * qt)
        softmax_tile64<true>(s_tm, lim, sl2, m_run, alpha, rs, need, j == 0);
      else
        softmax_tile64<false>(s_tm, lim, sl2, m_run, alpha, rs, need, j == 0);
      const bool rescale = j > 0 && __any_sync(0xffffffffu, need);
      if (j > 0 && (rescale || j == nkv - 1)) {
        // O must be stable (PV(j-1) done) before it is rescaled and before PV(j) adds to it.
        // At this point o_done has completed PV(j-2) (S(j) was issued after it) and PV(j) is
        // not issued yet, so the parity of phase j-1 is unambiguous.  The last tile waits
        // too, so that the epilogue's o_done wait below sees one of two phases only.
        mbar_wait(&o_done[i], (j - 1) & 1);
        tc_fence_after();
      }
      if (rescale) {
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
          uint32_t orr[32];
          tmem_ld32(o_tm + c * 32, orr);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 32; ++e) orr[e] = __float_as_uint(__uint_as_float(orr[e]) * alpha);
          tmem_st32(o_tm + c * 32, orr);
        }
      }
      tmem_wait_st();
      l_run = l_run * alpha + rs;
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[2 * i + (j & 1)]);
    }
    mbar_wait(&o_done[i], (nkv - 1) & 1);
    tc_fence_after();
    const float inv = 1.f / l_run;
    const bool row_ok = qrow < lq && prm.out != nullptr;
    const int64_t orow_off = (int64_t)(q_row0 + qrow) * prm.out_row_stride + (int64_t)(h0 + i) * D;
#pragma unroll
    for (int c = 0; c < D / 32; ++c) {
      uint32_t orr[32];
      tmem_ld32(o_tm + c * 32, orr);
      tmem_wait_ld();
      if (row_ok) {
        if (prm.out_f32) {
          float* orow = reinterpret_cast<float*>(prm.out) + orow_off;
#pragma unroll
          for (int e = 0; e < 32; e += 4)
            *reinterpret_cast<float4*>(orow + c * 32 + e) =
                make_float4(__uint_as_float(orr[e]) * inv, __uint_as_float(orr[e + 1]) * inv,
                            __uint_as_float(orr[e + 2]) * inv, __uint_as_float(orr[e + 3]) * inv);
        } else {
          __nv_bfloat16* orow = reinterpret_cast<__nv_bfloat16*>(prm.out) + orow_off;
#pragma unroll
          for (int e = 0; e < 32; e += 8) {
            uint4 w;
            w.x = pack_bf16x2(__uint_as_float(orr[e + 0]) * inv, __uint_as_float(orr[e + 1]) * inv);
            w.y = pack_bf16x2(__uint_as_float(orr[e + 2]) * inv, __uint_as_float(orr[e + 3]) * inv);
            w.z = pack_bf16x2(__uint_as_float(orr[e + 4]) * inv, __uint_as_float(orr[e + 5]) * inv);
            w.w = pack_bf16x2(__uint_as_float(orr[e + 6]) * inv, __uint_as_float(orr[e + 7]) * inv);
            *reinterpret_cast<uint4*>(orow + c * 32 + e) = w;
          }
        }
      }
    }
    if (qrow < lq && prm.lse != nullptr)
      prm.lse[(int64_t)(h0 + i) * prm.lse_stride + q_row0 + qrow] =
          (m_run + __log2f(l_run)) * 0.6931471805599453f;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    __syncwarp();
    tmem_free<512>(tbase);
  }
}

// ------------------------------------------------------------------ host
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder();

static int map3d(CUtensorMap* map, const void* base, int d, int heads, int64_t rows,
                 int64_t row_stride, int box_rows) {
  auto fn = tensor_map_encoder();
  if (fn == nullptr) return fail(STAR_ECUDA, "cuTensorMapEncodeTiled unavailable");
  if (((uintptr_t)base & 15) || ((row_stride * 2) & 15))
    return fail(STAR_ESHAPE, "TMA needs 16-byte aligned base and row stride");
  cuuint64_t dims[3] = {(cuuint64_t)d, (cuuint64_t)heads, (cuuint64_t)rows};
  cuuint64_t strides[2] = {(cuuint64_t)d * 2, (cuuint64_t)row_stride * 2};
  cuuint32_t box[3] = {64, 1, (cuuint32_t)box_rows};
  cuuint32_t estr[3] = {1, 1, 1};
  if (fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box,
         estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return fail(STAR_ECUDA, "cuTensorMapEncodeTiled failed");
  return STAR_OK;
}

int phase1_tc64(const void* q, const void* k, const void* v, SegTable& segs, int hq, int hkv,
                int64_t total_rows, int64_t qs, int64_t kvs, void* out, int out_f32, int64_t os,
                float* lse, int64_t lse_stride, cudaStream_t stream) {
  using C = P1Cfg64<128>;
  CUtensorMap tq, tk, tv;
  int rc;
  if ((rc = map3d(&tq, q, 128, hq, total_rows, qs, 128)) != STAR_OK) return rc;
  if ((rc = map3d(&tk, k, 128, hkv, total_rows, kvs, C::BN)) != STAR_OK) return rc;
  if ((rc = map3d(&tv, v, 128, hkv, total_rows, kvs, C::BN)) != STAR_OK) return rc;
  P1Params64 prm;
  prm.segs = segs;
  prm.hq = hq;
  prm.hkv = hkv;
  prm.out_row_stride = os;
  prm.lse_stride = lse_stride;
  prm.scale_log2 = (float)(1.4426950408889634 / sqrt(128.0));
  prm.out = out;
  prm.out_f32 = out_f32;
  prm.lse = lse;
  prm.segs.tile_start[0] = 0;
  for (int i = 0; i < segs.n; ++i)
    prm.segs.tile_start[i + 1] = prm.segs.tile_start[i] + (segs.lq[i] + C::BM - 1) / C::BM;
  const int tiles = prm.segs.tile_start[segs.n];
  if (tiles == 0) return STAR_OK;
  auto kern = phase1_tc64_kernel<128>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
  if (e != cudaSuccess) return fail(STAR_ECUDA, "phase1 smem attr: %s", cudaGetErrorString(e));
  dim3 grid(hkv * (hq / hkv / C::NQ), tiles);
  kern<<<grid, C::kThreads, C::kSmem, stream>>>(tq, tk, tv, prm);
  STAR_LAUNCH_CHECK("phase1_tc64");
  return STAR_OK;
}

}  // namespace star
