// Phase 1 (K1) on sm_100a tensor cores: causal flash attention over
// anchor-augmented blocks (segments), bf16 in, fp32 accumulation in TMEM.
//
// Reference semantics: causal_attention(q, k, v) per (block, layer, head)
// (ss/attention.py:109-122) inside _encode_block_channels (ss/sim.py:108-123);
// the online softmax is the tile-fold of streaming_causal_attention
// (ss/attention.py:176-210).
//
// CTA = one 128-row q tile of one segment for NQ query heads that share a kv
// head (GQA), so every K/V tile staged by TMA feeds NQ tensor-core pipelines.
// Warp roles:
//   warp 0      TMEM allocator; then lane 0 = TMA producer for K tiles and
//               lane 1 = TMA producer for V tiles (independent pipelines)
//   warp 1      tcgen05.mma issuer (one lane)
//   warps 2..   one 128-thread softmax warpgroup per q head: thread = q row =
//               TMEM lane.  S is read from TMEM in 32-column chunks (pass 1:
//               row max; pass 2: exp2, row sum, bf16 pack), and P is written
//               back into TMEM over the S columns already consumed; the P.V
//               MMA takes its A operand straight from TMEM, so P never touches
//               shared memory.  O stays in TMEM and is rescaled lazily (only
//               when the running max grows by more than 2^8 — exact, because
//               numerator and denominator share the stale max).
// TMEM columns: S_i / P_i at [i*BN, (i+1)*BN) (P packed bf16x2 in the first BN/2),
//               O_i at [NQ*BN + i*D, NQ*BN + (i+1)*D).
// MMA order per kv tile j: for each head i: PV_i(j) then S_i(j+1).  tcgen05.mma
// executes in issue order, so S_i(j+1) overwriting P_i(j) is safe, and the
// commit after S_i(j+1) also certifies PV_i(j) (O stable for the rescale).

#include <cudaTypedefs.h>
#include <stdlib.h>

#include "common.cuh"
#include "sm100.cuh"
#include "softmax_tc.cuh"

namespace star {

using namespace sm100;

template <int D, int NQ>
struct P1Cfg {
  static constexpr int BM = 128, BN = 128;
  static constexpr int kSlab = 128 * 128;          // [128 rows x 64 bf16] swizzled slab
  static constexpr int kSlabs = D / 64;            // slabs per [128 x D] tile
  static constexpr int kTile = kSlabs * kSlab;     // bytes of a [128 x D] bf16 tile
  static constexpr int KST = (D == 128) ? (NQ == 2 ? 2 : 3) : 3;  // K stages
  static constexpr int VST = (D == 128) ? (NQ == 2 ? 2 : 3) : 3;  // V stages
  static constexpr int kQOff = 0;
  static constexpr int kKOff = kQOff + NQ * kTile;
  static constexpr int kVOff = kKOff + KST * kTile;
  static constexpr int kBarOff = kVOff + VST * kTile;
  static constexpr int kNumBars = 1 + 2 * KST + 2 * VST + 4 * NQ + 4 * NQ;
  static constexpr int kSmem = kBarOff + kNumBars * 8 + 16 + 1024;  // + tmem slot + align slack
  static constexpr int kThreads = 64 + 128 * NQ;  // 2 control warps + softmax warpgroups
  // 12-warp layout (NQ == 2): softmax warpgroups 0-1, then warpgroup 2 = TMA producer, MMA
  // issuer and two idle warps; setmaxnreg moves registers from warpgroup 2 to the softmax
  static constexpr int kThreads12 = 384;
  static constexpr int kRegsCtl = 96, kRegsSoftmax = 200;
  // setmaxnreg.inc draws only on what .dec released (the CTA was launched at 168 per thread):
  // 4 warps x (168 - ctl) must cover 8 warps x (softmax - 168), or the softmax warps block
  static_assert(4 * (168 - kRegsCtl) >= 8 * (kRegsSoftmax - 168), "register pool");
  static constexpr int kTmemCols = (NQ * (BN + D) <= 256) ? 256 : 512;
  static_assert(NQ * (BN + D) <= 512, "TMEM budget");
  static_assert(kSmem <= 232448, "shared memory budget");
};

struct P1Params {
  SegTable segs;
  int hq, hkv, d;
  int64_t out_row_stride;
  int64_t lse_stride;
  float scale_log2;
  int seq;         // ping-pong the softmax warpgroups' exp sections (NQ == 2)
  void* out;       // bf16 or fp32 rows (out_f32)
  int out_f32;
  float* lse;
};

#ifndef STAR_K1_TRQ
#define STAR_K1_TRQ 2  // TMEM lane quarter (= SM sub-partition) whose lane 0 is traced
#endif
#ifdef STAR_K1_TRACE
// Timeline of CTA 0 (clock64): [head][tile][5] softmax events (S ready, max done, turn
// granted, exps done, P handed over) and [tile][head][2] MMA events (P seen, PV+S issued).
// Built only into the tracing library (make trace); tools/k1_trace.py reads it.
constexpr int kTrTiles = 256;
__device__ long long g_k1_trace[2 * kTrTiles * 5 + kTrTiles * 2 * 2 + 2 * kTrTiles * 4 * 2];
#define K1_TR(cond, idx) \
  do {                   \
    if (cond) g_k1_trace[idx] = clock64(); \
  } while (0)
#else
#define K1_TR(cond, idx) \
  do {                   \
  } while (0)
#endif
// per-row softmax helpers (row_max, exp_pack, tmem_ld_row128, ...): softmax_tc.cuh


template <int D, int NQ, int POLY, int SUM, bool SPLIT, bool L12 = false, int WAIT = 0,
          bool MW2 = false, int SWAIT = -1, bool BATCH = false, bool MC = false>
__global__ void __launch_bounds__(L12 ? P1Cfg<D, NQ>::kThreads12 : P1Cfg<D, NQ>::kThreads, 1)
    phase1_tc_kernel(const __grid_constant__ CUtensorMap tm_q,
                     const __grid_constant__ CUtensorMap tm_k,
                     const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ P1Params prm) {
  using C = P1Cfg<D, NQ>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-byte alignment for SWIZZLE_128B atoms
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kBarOff);
  uint64_t* q_full = bars;
  uint64_t* k_full = q_full + 1;
  uint64_t* k_empty = k_full + C::KST;
  uint64_t* v_full = k_empty + C::KST;
  uint64_t* v_empty = v_full + C::VST;
  uint64_t* s_full = v_empty + C::VST;
  uint64_t* p_full = s_full + NQ;
  uint64_t* o_done = p_full + NQ;
  uint64_t* seq_done = o_done + NQ;  // [NQ][4]: softmax warp (i, quarter) finished its exps
  uint64_t* p_half = seq_done + 4 * NQ;  // [NQ]: P of keys [0, BN/2) in TMEM (SPLIT)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(p_half + NQ);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // ---- work item from a 1-D raster: segment-major, then kv head, then q tile (heaviest
  // first), then the head pair — CTAs resident together share one kv head's K/V, which
  // stays L2-resident (a block's K/V over all kv heads exceeds the 126 MB L2) ----
  const int G = prm.hq / prm.hkv;
  const int pairs = G / NQ;
  const int per_tile = prm.hkv * pairs;  // CTAs per launched q tile
  const int bx = blockIdx.x;
  int s = 0;
  while (s + 1 < prm.segs.n && prm.segs.tile_start[s + 1] * per_tile <= bx) ++s;
  const int ntq = (prm.segs.lq[s] + C::BM - 1) / C::BM;
  const int launched = prm.segs.tile_start[s + 1] - prm.segs.tile_start[s];
  const int loc = bx - prm.segs.tile_start[s] * per_tile;  // [0, hkv * launched * pairs)
  const int kvh = loc / (launched * pairs);
  const int rem = loc - kvh * launched * pairs;
  const int qt = ntq - 1 - rem / pairs;
  const int h0 = kvh * G + (rem % pairs) * NQ;
  const int lq = prm.segs.lq[s];
  const int q_row0 = (int)prm.segs.q_row0[s];
  const int k_row0 = (int)prm.segs.k_row0[s];
  const int nkv = qt + 1;  // causal, q and k aligned at row 0 of the segment
  // MC: the CTA is one of a 2-CTA cluster whose CTAs run the two head pairs of the same
  // (segment, kv head, q tile) — the 1-D raster puts them at bx, bx + 1.  Each CTA loads one
  // 64-column slab of every K / V tile and multicasts it to both, so each tile leaves L2 once
  // per pair; a stage is refilled once BOTH CTAs' MMAs released it (empty count 2).
  static_assert(!MC || (D == 128 && NQ == 2 && !MW2), "multicast pairs two D = 128 head pairs");
  const uint32_t crank = MC ? cluster_ctarank() : 0u;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    // MW2: each q head's MMAs come from its own warp, and both release the K/V stages
    for (int i = 0; i < C::KST; ++i) { mbar_init(&k_full[i], 1); mbar_init(&k_empty[i], (MW2 || MC) ? 2 : 1); }
    for (int i = 0; i < C::VST; ++i) { mbar_init(&v_full[i], 1); mbar_init(&v_empty[i], (MW2 || MC) ? 2 : 1); }
    for (int i = 0; i < NQ; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 4);
      mbar_init(&p_half[i], 4);
      mbar_init(&o_done[i], 1);
      for (int w = 0; w < 4; ++w) mbar_init(&seq_done[i * 4 + w], 1);
    }
    fence_mbar_init();
  }
  static_assert(!L12 || NQ == 2, "12-warp layout pairs two softmax warpgroups");
  static_assert(!MW2 || L12, "two MMA warps need the 12-warp layout");
  // TMA producer warp (also the TMEM allocator) and MMA warp(s).  MW2 spreads the MMA issue
  // (each tcgen05.mma holds its SM sub-partition's dispatch for several cycles, which delays
  // the softmax warps sharing it) over sub-partitions 1 and 3, the producer on 0.
  const int ctl_warp0 = L12 ? 8 : 0;
  const bool is_producer = warp == ctl_warp0;
  const bool is_mma = MW2 ? (warp == 9 || warp == 11) : warp == ctl_warp0 + 1;
  if (is_producer) tmem_alloc<C::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  if (MC) cluster_sync();  // the peer's barriers are initialised before any multicast lands
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  // waits on the per-tile critical path (S ready, P handed over, MUFU turn)
  // MMA warp waits use WAIT, softmax waits SWAIT (defaults to WAIT)
  auto wait_mode = [](uint64_t* bar, uint32_t parity, int mode, int tag) {
    if (mode == 3)
      mbar_wait_dbg(bar, parity, tag);
    else if (mode == 1)
      mbar_wait_nohint(bar, parity);
    else if (mode == 2)
      mbar_wait_spin(bar, parity);
    else
      mbar_wait(bar, parity);
  };
  auto cwait = [&](uint64_t* bar, uint32_t parity, int tag = 0) { wait_mode(bar, parity, WAIT, tag); };
  auto swait = [&](uint64_t* bar, uint32_t parity, int tag = 0) {
    wait_mode(bar, parity, SWAIT < 0 ? WAIT : SWAIT, tag);
  };
  auto producer_role = [&]() {
    if (lane == 0) {
      // ================= K producer (+ Q once) =================
      tma_prefetch(&tm_q);
      tma_prefetch(&tm_k);
      mbar_expect_tx(q_full, NQ * C::kTile);
      for (int i = 0; i < NQ; ++i)
        for (int a = 0; a < C::kSlabs; ++a)
          tma_load_3d(smem + C::kQOff + i * C::kTile + a * C::kSlab, &tm_q, q_full, a * 64, h0 + i,
                      q_row0 + qt * C::BM);
      for (int j = 0; j < nkv; ++j) {
        const int st = j % C::KST;
        if (j >= C::KST) mbar_wait(&k_empty[st], ((j / C::KST) + 1) & 1);
        mbar_expect_tx(&k_full[st], C::kTile);
        if (MC)
          tma_load_3d_mc(smem + C::kKOff + st * C::kTile + crank * C::kSlab, &tm_k, &k_full[st],
                         crank * 64, kvh, k_row0 + j * C::BN, 0x3);
        else
          for (int a = 0; a < C::kSlabs; ++a)
            tma_load_3d(smem + C::kKOff + st * C::kTile + a * C::kSlab, &tm_k, &k_full[st], a * 64,
                        kvh, k_row0 + j * C::BN);
      }
    } else if (lane == 1) {
      // ================= V producer =================
      tma_prefetch(&tm_v);
      for (int j = 0; j < nkv; ++j) {
        const int st = j % C::VST;
        if (j >= C::VST) mbar_wait(&v_empty[st], ((j / C::VST) + 1) & 1);
        mbar_expect_tx(&v_full[st], C::kTile);
        if (MC)
          tma_load_3d_mc(smem + C::kVOff + st * C::kTile + crank * C::kSlab, &tm_v, &v_full[st],
                         crank * 64, kvh, k_row0 + j * C::BN, 0x3);
        else
          for (int a = 0; a < C::kSlabs; ++a)
            tma_load_3d(smem + C::kVOff + st * C::kTile + a * C::kSlab, &tm_v, &v_full[st], a * 64,
                        kvh, k_row0 + j * C::BN);
      }
    }
  };
  auto mma_role = [&](const int i0, const int i1) {
    // ================= MMA issuer =================
    {  // the whole warp, converged: one elected lane issues each MMA / commit
      constexpr uint32_t idesc_s = umma_idesc_bf16(128, C::BN, false, false);
      constexpr uint32_t idesc_o = umma_idesc_bf16(128, D, false, true);
      const uint32_t q_addr = smem_u32(smem + C::kQOff);
      const uint32_t k_addr = smem_u32(smem + C::kKOff);
      const uint32_t v_addr = smem_u32(smem + C::kVOff);
      auto issue_s = [&](int i, int st) {
        if (BATCH && D == 128) {
          umma_ss_d128_warp(tbase + i * C::BN, umma_desc_sw128(q_addr + i * C::kTile, 16, 1024),
                            umma_desc_sw128(k_addr + st * C::kTile, 16, 1024), idesc_s, 0u);
          umma_commit_warp(&s_full[i]);
          return;
        }
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * C::kSlab + (kk & 3) * 32;
          const uint64_t ad = umma_desc_sw128(q_addr + i * C::kTile + off, 16, 1024);
          const uint64_t bd = umma_desc_sw128(k_addr + st * C::kTile + off, 16, 1024);
          umma_bf16_ss_warp(tbase + i * C::BN, ad, bd, idesc_s, kk > 0 ? 1u : 0u);
        }
        umma_commit_warp(&s_full[i]);
      };
      mbar_wait(q_full, 0);
      mbar_wait(&k_full[0], 0);
      tc_fence_after();
      for (int i = i0; i < i1; ++i) issue_s(i, 0);
      auto release = [&](uint64_t* bar) {
        if (MC)
          umma_commit_mc_warp(bar, 0x3);
        else
          umma_commit_warp(bar);
      };
      if (C::KST < nkv) release(&k_empty[0]);
      for (int j = 0; j < nkv; ++j) {
        const int vs = j % C::VST;
        cwait(&v_full[vs], (j / C::VST) & 1, 7);
        const bool next = j + 1 < nkv;
        const int ks = (j + 1) % C::KST;
        if (next) cwait(&k_full[ks], ((j + 1) / C::KST) & 1, 8);
        for (int i = i0; i < i1; ++i) {
          if (SPLIT) {  // P.V over keys [0, BN/2) while the softmax still exponentiates the rest
            cwait(&p_half[i], j & 1, 2);
            tc_fence_after();
            if (BATCH && C::BN == 128) {
              umma_ts_x4_warp(tbase + NQ * C::BN + i * D, tbase + i * C::BN,
                              umma_desc_sw128(v_addr + vs * C::kTile, C::kSlab, 1024), idesc_o,
                              j > 0 ? 1u : 0u);
            } else
#pragma unroll
            for (int kk = 0; kk < C::BN / 32; ++kk) {
              const uint64_t bd = umma_desc_sw128(v_addr + vs * C::kTile + kk * 16 * 128, C::kSlab,
                                                  1024);
              umma_bf16_ts_warp(tbase + NQ * C::BN + i * D, tbase + i * C::BN + kk * 8, bd,
                                idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
            }
          }
          cwait(&p_full[i], j & 1, 3);
          K1_TR(bx == 0 && j < 256, 2 * 256 * 5 + (j * 2 + i) * 2);
          tc_fence_after();
          if (BATCH && C::BN == 128) {
            if (SPLIT)
              umma_ts_x4_warp(tbase + NQ * C::BN + i * D, tbase + i * C::BN + 32,
                              umma_desc_sw128(v_addr + vs * C::kTile + 4 * 16 * 128, C::kSlab, 1024),
                              idesc_o, 1u);
            else
              umma_ts_x8_warp(tbase + NQ * C::BN + i * D, tbase + i * C::BN,
                              umma_desc_sw128(v_addr + vs * C::kTile, C::kSlab, 1024), idesc_o,
                              j > 0 ? 1u : 0u);
          } else
#pragma unroll
          for (int kk = SPLIT ? C::BN / 32 : 0; kk < C::BN / 16; ++kk) {
            const uint64_t bd = umma_desc_sw128(v_addr + vs * C::kTile + kk * 16 * 128, C::kSlab,
                                                1024);
            umma_bf16_ts_warp(tbase + NQ * C::BN + i * D, tbase + i * C::BN + kk * 8, bd, idesc_o,
                         (j > 0 || kk > 0) ? 1u : 0u);
          }
          if (!next) umma_commit_warp(&o_done[i]);  // the epilogue's wait: the last P.V only
          if (next) issue_s(i, ks);
          K1_TR(bx == 0 && j < 256, 2 * 256 * 5 + (j * 2 + i) * 2 + 1);
        }
        // release a stage only if the producer will refill it (a commit nobody waits for
        // could still be in flight when the CTA exits)
        if (j + C::VST < nkv) release(&v_empty[vs]);
        if (next && j + 1 + C::KST < nkv) release(&k_empty[ks]);
      }
    }
  };
  auto softmax_role = [&](const int i) {
    // ================= softmax warpgroup i =================
    const int wq = warp & 3;  // TMEM lane quarter (a warp may only touch lanes 32*(warp%4)..)
    const int r = wq * 32 + lane;
    const int qrow = qt * C::BM + r;
    const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
    const uint32_t s_tm = tbase + lane_off + i * C::BN;
    const uint32_t o_tm = tbase + lane_off + NQ * C::BN + i * D;
    const float sl2 = prm.scale_log2;
    float m_run = -INFINITY, l_run = 0.f;

    for (int j = 0; j < nkv; ++j) {
      swait(&s_full[i], j & 1, 4);
      const bool tr = bx == 0 && wq == STAR_K1_TRQ && lane == 0 && j < 256;  // traced quarter
      K1_TR(tr, (i * 256 + j) * 5 + 0);
      K1_TR(bx == 0 && lane == 0 && j < 256, 2 * 256 * 5 + 256 * 2 * 2 + ((i * 256 + j) * 4 + wq) * 2);
      tc_fence_after();
      const bool diag = (j == qt);
      const int lim = qrow - j * C::BN;  // columns c <= lim are visible on the diagonal tile
      // ---- row max: the whole 128-column S row in registers (four tcgen05.ld, one wait) ----
      uint32_t sv[4][32];
      tmem_ld_row128(s_tm, sv);
      const float mx = (diag ? row_max_regs<true>(sv, lim) : row_max_regs<false>(sv, lim)) * sl2;
      K1_TR(tr, (i * 256 + j) * 5 + 1);
      float m_use = m_run, alpha = 1.f;
      const bool need = (j == 0) || (mx > m_run + 8.f);
      const bool warp_rescale = (j > 0) && __any_sync(0xffffffffu, need);
      if (need) {
        if (j > 0) alpha = ex2(m_run - mx);
        m_use = mx;
      }
      // ---- p = 2^(s*sl2 - m), row sum, bf16 P back into TMEM ----
      // Ping-pong: the two warps of one SM sub-partition (head 0 and head 1, same TMEM lane
      // quarter) take turns on its MUFU pipe — head 1 exponentiates tile j after head 0 has,
      // head 0 tile j after head 1's tile j-1 — so each runs at the full exp2 rate while the
      // other head's P.V + next S occupy the tensor pipe (anti-phase, not in-phase sharing).
      const bool seq = NQ == 2 && prm.seq;
      if (seq) {
        if (i == 1)
          swait(&seq_done[wq], j & 1, 5);
        else if (j > 0)
          swait(&seq_done[4 + wq], (j - 1) & 1, 6);
      }
      K1_TR(tr, (i * 256 + j) * 5 + 2);
      // O is stable here: s_full(j) was committed after PV(j-1).  It is rescaled before the
      // first P of this tile is handed over (mid-row under SPLIT, after the exps otherwise).
      auto rescale = [&]() {
        if (warp_rescale) {
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
      };
      auto half = [&]() {
        rescale();
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_half[i]);
        if (seq && prm.seq == 2 && lane == 0) mbar_arrive(&seq_done[i * 4 + wq]);  // mid-row turn
      };
      const float rs = diag ? exp_pack_regs<true, POLY, SUM, SPLIT>(sv, s_tm, lim, sl2, m_use, half)
                            : exp_pack_regs<false, POLY, SUM, SPLIT>(sv, s_tm, lim, sl2, m_use, half);
      K1_TR(tr, (i * 256 + j) * 5 + 3);
      if (seq && prm.seq != 2) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&seq_done[i * 4 + wq]);
      }
      if (!SPLIT) rescale();
      tmem_wait_st();
      l_run = l_run * alpha + rs;
      m_run = m_use;
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[i]);
      K1_TR(tr, (i * 256 + j) * 5 + 4);
      // every warp quarter: S seen and P handed over (skew across SM sub-partitions)
      K1_TR(bx == 0 && lane == 0 && j < 256, 2 * 256 * 5 + 256 * 2 * 2 + ((i * 256 + j) * 4 + wq) * 2 + 1);
    }
    // ---- epilogue: O / l -> rows; lse = ln(sum) + max ----
    mbar_wait(&o_done[i], 0);  // one phase: the commit after the last P.V
    tc_fence_after();
    const float inv = 1.f / l_run;
    const bool row_ok = qrow < lq && prm.out != nullptr;
    // segments receiving this row: itself, plus every deduplicated segment for anchor tiles
    const int n_dst = (s == 0 && qt < prm.segs.dedup_tiles) ? prm.segs.n : 1;
#pragma unroll
    for (int c = 0; c < D / 32; ++c) {
      uint32_t orr[32];
      tmem_ld32(o_tm + c * 32, orr);
      tmem_wait_ld();
      if (row_ok) {
        for (int t = 0; t < n_dst; ++t) {
          const int64_t orow_off = (int64_t)(prm.segs.q_row0[t == 0 ? s : t] + qrow) *
                                       prm.out_row_stride + (int64_t)(h0 + i) * D;
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
    }
    if (qrow < lq && prm.lse != nullptr) {
      const float lv = (m_run + __log2f(l_run)) * 0.6931471805599453f;
      for (int t = 0; t < n_dst; ++t)
        prm.lse[(int64_t)(h0 + i) * prm.lse_stride + prm.segs.q_row0[t == 0 ? s : t] + qrow] = lv;
    }
  };
  if (L12) {
    // setmaxnreg inside warpgroup-uniform branches (the warpgroup index is made provably
    // uniform by a shuffle), so ptxas allocates each role's code with its own budget
    const int wg = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 7), 0);
    if (wg == 2) {
      regs_dealloc<C::kRegsCtl>();
      if (is_producer)
        producer_role();
      else if (is_mma)
        MW2 ? mma_role(warp == 9 ? 0 : 1, warp == 9 ? 1 : 2) : mma_role(0, NQ);
    } else {
      regs_alloc<C::kRegsSoftmax>();
      softmax_role(wg);
    }
  } else {
    if (is_producer)
      producer_role();
    else if (is_mma)
      mma_role(0, NQ);
    else
      softmax_role((warp - 2) >> 2);
  }
  tc_fence_before();
  __syncthreads();
  if (MC) cluster_sync();  // no multicast or remote arrival targets an exited CTA
  if (is_producer) {
    __syncwarp();
    tmem_free<C::kTmemCols>(tbase);
  }
}

// ------------------------------------------------------------------ host
constexpr int kDefaultSeq = 0;  // MUFU ping-pong off: with a quarter of the exps on the FMA pipe it costs more than it saves

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (fn == nullptr) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) ==
            cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 3-D bf16 map over [rows][heads][d] with row stride (elements); box = 64 x 1 x 128.
static int make_map_3d(CUtensorMap* map, const void* base, int d, int heads, int64_t rows,
                       int64_t row_stride) {
  auto fn = tensor_map_encoder();
  if (fn == nullptr) return fail(STAR_ECUDA, "cuTensorMapEncodeTiled unavailable");
  if (((uintptr_t)base & 15) || ((row_stride * 2) & 15))
    return fail(STAR_ESHAPE, "TMA needs 16-byte aligned base and row stride (row_stride=%lld)",
                (long long)row_stride);
  cuuint64_t dims[3] = {(cuuint64_t)d, (cuuint64_t)heads, (cuuint64_t)rows};
  cuuint64_t strides[2] = {(cuuint64_t)d * 2, (cuuint64_t)row_stride * 2};
  cuuint32_t box[3] = {64, 1, 128};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(STAR_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return STAR_OK;
}

template <int D, int NQ>
static int launch_phase1_tc(const void* q, const void* k, const void* v, SegTable& segs, int hq,
                            int hkv, int64_t total_q_rows, int64_t total_kv_rows, int64_t qs,
                            int64_t kvs, void* out, int out_f32, int64_t os, float* lse,
                            int64_t lse_stride, cudaStream_t stream) {
  using C = P1Cfg<D, NQ>;
  CUtensorMap tq, tk, tv;
  int rc;
  if ((rc = make_map_3d(&tq, q, D, hq, total_q_rows, qs)) != STAR_OK) return rc;
  if ((rc = make_map_3d(&tk, k, D, hkv, total_kv_rows, kvs)) != STAR_OK) return rc;
  if ((rc = make_map_3d(&tv, v, D, hkv, total_kv_rows, kvs)) != STAR_OK) return rc;
  P1Params prm;
  prm.segs = segs;
  prm.hq = hq;
  prm.hkv = hkv;
  prm.d = D;
  prm.out_row_stride = os;
  prm.lse_stride = lse_stride;
  prm.scale_log2 = (float)(1.4426950408889634 / sqrt((double)D));
  prm.out = out;
  prm.out_f32 = out_f32;
  prm.lse = lse;
  prm.segs.tile_start[0] = 0;
  for (int i = 0; i < segs.n; ++i)
    prm.segs.tile_start[i + 1] = prm.segs.tile_start[i] + (segs.lq[i] + C::BM - 1) / C::BM -
                                 std::max(segs.tile_lo[i], i > 0 ? segs.dedup_tiles : 0);
  const int tiles = prm.segs.tile_start[segs.n];
  if (tiles == 0) return STAR_OK;
  // the product build instantiates the measured-best form: one-pass row in
  // registers, split P hand-off, fp32 FADD2 row sums, every 4th exponential pair on the FMA
  // pipe; NQ == 2 runs the 12-warp layout (setmaxnreg gives the softmax warpgroups 200
  // registers) with the MMA warp waiting without a suspend hint and issuing each MMA batch
  // under one elect
  prm.seq = kDefaultSeq;
  if (const char* sq = getenv("STAR_K1_SEQ")) prm.seq = atoi(sq);  // measurement knob
  using KernT = void (*)(const CUtensorMap, const CUtensorMap, const CUtensorMap, const P1Params);
  KernT kern;
  int threads;
  if constexpr (NQ == 2) {
    kern = phase1_tc_kernel<D, NQ, 4, 2, true, true, 1, false, 0, true>;
    threads = C::kThreads12;
  } else {
    kern = phase1_tc_kernel<D, NQ, 4, 2, true, false, 1, false, 0>;
    threads = C::kThreads;
  }
  // K/V tiles multicast across the two head pairs of a q tile (2-CTA cluster) when the GQA
  // ratio gives an even number of head pairs; STAR_K1_MC=0 turns it off (measurement knob)
  bool mc = false;
  if constexpr (NQ == 2 && D == 128) {
    const char* ev = getenv("STAR_K1_MC");
    if ((hq / hkv / NQ) % 2 == 0 && !(ev != nullptr && ev[0] == '0')) {
      kern = phase1_tc_kernel<D, NQ, 4, 2, true, true, 1, false, 0, true, true>;
      mc = true;
    }
  }
  if (const char* sv = getenv("STAR_K1_SM")) {  // measurement knob (tools/phase1_bench.py)
    if constexpr (NQ == 2) {  // the knob forms are single-CTA kernels
      if (mc) kern = phase1_tc_kernel<D, NQ, 4, 2, true, true, 1, false, 0, true>;
    }
    mc = false;
    const int vv = atoi(sv);
    if (vv == 1) {  // round-1 form: 10 warps, f32 += bf16 row sums, whole-P hand-off
      kern = phase1_tc_kernel<D, NQ, 0, 1, false>;
      threads = C::kThreads;
    }
    if constexpr (NQ == 2) {
      if (vv == 2) kern = phase1_tc_kernel<D, NQ, 0, 2, true, true, 1, false, 0>;
      if (vv == 3) kern = phase1_tc_kernel<D, NQ, 4, 2, true, true, 1, false, 0>;  // per-MMA elect
      if (vv == 4) kern = phase1_tc_kernel<D, NQ, 3, 2, true, true, 1, false, 0>;
      if (vv == 5) kern = phase1_tc_kernel<D, NQ, 2, 2, true, true, 1, false, 0>;
    }
  }
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
  if (e != cudaSuccess) return fail(STAR_ECUDA, "phase1 smem attr: %s", cudaGetErrorString(e));
  dim3 grid(tiles * hkv * (hq / hkv / NQ));
  if (mc) {
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = C::kSmem;
    cfg.stream = stream;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    // once per process: can a 2-CTA cluster of this kernel be resident at all (a partitioned
    // or shared GPU may not offer two free SMs of one GPC)?  If not, or if the cluster launch
    // is refused, the single-CTA kernel runs (same results, bit for bit)
    static int cluster_ok = -1;
    if (cluster_ok < 0) {
      int n = 0;
      cluster_ok = (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) == cudaSuccess && n > 0) ? 1 : 0;
      (void)cudaGetLastError();
    }
    e = cluster_ok ? cudaLaunchKernelEx(&cfg, kern, tq, tk, tv, prm) : cudaErrorNotSupported;
    if (e != cudaSuccess) {
      (void)cudaGetLastError();
      mc = false;
      if constexpr (NQ == 2) {
        kern = phase1_tc_kernel<D, NQ, 4, 2, true, true, 1, false, 0, true>;
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
        if (e != cudaSuccess) return fail(STAR_ECUDA, "phase1 smem attr: %s", cudaGetErrorString(e));
      }
    }
  }
  if (!mc) kern<<<grid, threads, C::kSmem, stream>>>(tq, tk, tv, prm);
  STAR_LAUNCH_CHECK("phase1_tc");
  return STAR_OK;
}

int phase1_tc(const void* q, const void* k, const void* v, SegTable& segs, int hq, int hkv, int d,
              int64_t total_rows, int64_t qs, int64_t kvs, void* out, int out_f32, int64_t os,
              float* lse, int64_t lse_stride, cudaStream_t stream) {
  const int G = hq / hkv;
  if (d == 128) {
    if (G % 2 == 0)
      return launch_phase1_tc<128, 2>(q, k, v, segs, hq, hkv, total_rows, total_rows, qs, kvs, out,
                                      out_f32, os, lse, lse_stride, stream);
    return launch_phase1_tc<128, 1>(q, k, v, segs, hq, hkv, total_rows, total_rows, qs, kvs, out,
                                    out_f32, os, lse, lse_stride, stream);
  }
  if (d == 64) {
    if (G % 2 == 0)
      return launch_phase1_tc<64, 2>(q, k, v, segs, hq, hkv, total_rows, total_rows, qs, kvs, out,
                                     out_f32, os, lse, lse_stride, stream);
    return launch_phase1_tc<64, 1>(q, k, v, segs, hq, hkv, total_rows, total_rows, qs, kvs, out, out_f32, os,
                                   lse, lse_stride, stream);
  }
  return fail(STAR_ENOTSUP, "phase1 tensor-core path needs head_dim 64 or 128, got %d", d);
}

// ------------------------------------------------------------------ debug GEMM
// C[128x128] = A[128xK] . B^T, one CTA, one stage per 64-wide K slab.  mode bit 0: B given
// MN-major ([K x 128]); bit 1: A staged into TMEM (the .kind::f16 [a_tmem] form the
// phase-1 P.V product uses).  Used by the tests to pin the UMMA descriptor / TMA swizzle /
// TMEM-operand conventions the attention kernel relies on.
__global__ void __launch_bounds__(128, 1)
    umma_gemm_kernel(const __grid_constant__ CUtensorMap tm_a,
                     const __grid_constant__ CUtensorMap tm_b, float* c, int K, int mode) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* a_s = smem;           // [128 x 64] slab
  unsigned char* b_s = smem + 16384;   // K-major: [128 x 64]; MN-major: 2 slabs of [64 x 64]
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 49152);
  uint64_t* mma_bar = bar + 1;
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b_mn = mode & 1, a_tm = (mode >> 1) & 1;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(mma_bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<256>(slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *slot;
  const int r = warp * 32 + lane;
  const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
  for (int kb = 0; kb < K / 64; ++kb) {
    if (threadIdx.x == 0) {
      mbar_expect_tx(bar, 16384 + 16384);
      tma_load_2d(a_s, &tm_a, bar, kb * 64, 0);
      if (!b_mn) {
        tma_load_2d(b_s, &tm_b, bar, kb * 64, 0);
      } else {
        tma_load_2d(b_s, &tm_b, bar, 0, kb * 64);
        tma_load_2d(b_s + 8192, &tm_b, bar, 64, kb * 64);
      }
    }
    mbar_wait(bar, kb & 1);
    if (a_tm) {
      // row r of the swizzled slab -> 32 packed columns of TMEM lane r
      uint32_t w[2][16];
      for (int ch = 0; ch < 8; ++ch) {
        const uint4 v = *reinterpret_cast<const uint4*>(a_s + r * 128 + ((ch ^ (r & 7)) << 4));
        w[ch >> 2][(ch & 3) * 4 + 0] = v.x;
        w[ch >> 2][(ch & 3) * 4 + 1] = v.y;
        w[ch >> 2][(ch & 3) * 4 + 2] = v.z;
        w[ch >> 2][(ch & 3) * 4 + 3] = v.w;
      }
      tmem_st16(tbase + lane_off + 128, w[0]);
      tmem_st16(tbase + lane_off + 144, w[1]);
      tmem_wait_st();
      tc_fence_before();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      tc_fence_after();
      const uint32_t idesc = umma_idesc_bf16(128, 128, false, b_mn != 0);
      for (int kk = 0; kk < 4; ++kk) {
        uint64_t bd = b_mn ? umma_desc_sw128(smem_u32(b_s) + kk * 16 * 128, 8192, 1024)
                           : umma_desc_sw128(smem_u32(b_s) + kk * 32, 16, 1024);
        if (a_tm) {
          umma_bf16_ts(tbase, tbase + 128 + kk * 8, bd, idesc, (kb > 0 || kk > 0) ? 1u : 0u);
        } else {
          uint64_t ad = umma_desc_sw128(smem_u32(a_s) + kk * 32, 16, 1024);
          umma_bf16_ss(tbase, ad, bd, idesc, (kb > 0 || kk > 0) ? 1u : 0u);
        }
      }
      umma_commit(mma_bar);
      mbar_wait(mma_bar, kb & 1);
    }
    __syncthreads();
  }
  tc_fence_after();
  for (int cc = 0; cc < 4; ++cc) {
    uint32_t v[32];
    tmem_ld32(tbase + lane_off + cc * 32, v);
    tmem_wait_ld();
    for (int e = 0; e < 32; ++e) c[r * 128 + cc * 32 + e] = __uint_as_float(v[e]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_free<256>(tbase);
}

int debug_umma_gemm(const void* a, const void* b, float* c, int K, int mode, cudaStream_t s) {
  const int b_mn = mode & 1;
  if (K < 64 || K % 64) return fail(STAR_ESHAPE, "debug gemm: K must be a multiple of 64");
  auto fn = tensor_map_encoder();
  if (fn == nullptr) return fail(STAR_ECUDA, "cuTensorMapEncodeTiled unavailable");
  CUtensorMap ta, tb;
  cuuint32_t estr[2] = {1, 1};
  {
    cuuint64_t dims[2] = {(cuuint64_t)K, 128};
    cuuint64_t str[1] = {(cuuint64_t)K * 2};
    cuuint32_t box[2] = {64, 128};
    if (fn(&ta, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(a), dims, str, box, estr,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
           CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return fail(STAR_ECUDA, "encode A failed");
  }
  {
    cuuint64_t dims[2];
    cuuint64_t str[1];
    cuuint32_t box[2] = {64, (cuuint32_t)(b_mn ? 64 : 128)};
    if (b_mn) {
      dims[0] = 128; dims[1] = (cuuint64_t)K; str[0] = 128 * 2;
    } else {
      dims[0] = (cuuint64_t)K; dims[1] = 128; str[0] = (cuuint64_t)K * 2;
    }
    if (fn(&tb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(b), dims, str, box, estr,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
           CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return fail(STAR_ECUDA, "encode B failed");
  }
  int smem = 49152 + 64 + 1024;
  cudaFuncSetAttribute(umma_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  umma_gemm_kernel<<<1, 128, smem, s>>>(ta, tb, c, K, mode);
  STAR_LAUNCH_CHECK("umma_gemm");
  return STAR_OK;
}

#ifdef STAR_K1_TRACE
int debug_k1_trace(long long* host, int n) {
  const int cap = (int)(sizeof(g_k1_trace) / sizeof(long long));
  if (n > cap) n = cap;
  return cudaMemcpyFromSymbol(host, g_k1_trace, n * sizeof(long long)) == cudaSuccess ? n : -4;
}
#endif

}  // namespace star

#ifdef STAR_K1_TRACE
extern "C" int star_debug_k1_trace(long long* host, int n) { return star::debug_k1_trace(host, n); }
#endif
