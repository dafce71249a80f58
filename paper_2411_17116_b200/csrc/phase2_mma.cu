// Phase 2 (K2), bf16 production path: split-KV partial attention over the paged
// cache, HBM-bound.  Reference semantics as in phase2.cu (partial_attention /
// _gather_merge, ss/attention.py:125-151, ss/sim.py:178-213).
//
// Design (B200): one CTA streams one key range ("split") of one (sequence, kv
// head).  A producer warp moves [TN x 64] K/V slabs with TMA (128B swizzle)
// into a STAGES-deep mbarrier ring; four consumer warps run the two small
// products on mma.sync m16n8k16 (bf16 in, fp32 accumulate) — the G query heads
// x lq query rows of the group are packed into the M=16 rows, so one K/V tile
// load serves every q head of the group.
//   KEYSPLIT (G*lq <= 16, decode): warp w takes keys [w*TN/4, (w+1)*TN/4) of
//     each tile with its own online softmax; the 4 warp partials are merged
//     in shared memory at the end of the split.
//   row mode (G*lq > 16, query encode): warp w takes q rows [16w, 16w+16) of a
//     64-row pass over every key of the tile.
#include <cudaTypedefs.h>
#include <limits.h>
#include <stdlib.h>

#include <array>
#include <mutex>
#include <unordered_map>

#include "common.cuh"
#include "exchange.cuh"
#include "sm100.cuh"
#include "softmax_tc.cuh"

namespace star {

using namespace sm100;

namespace p2 {

constexpr int TN = 64;       // keys per tile (must divide page_size)
constexpr int STAGES = 6;
// consumer warps: decode (KEYSPLIT) runs two groups of four that take alternate tiles, so
// every SM sub-partition has two independent mma.sync chains in flight; the query-encode
// row mode runs one group of four
template <bool KEYSPLIT>
struct Cons {
  static constexpr int NC = KEYSPLIT ? 8 : 4;   // consumer warps
  static constexpr int NG = NC / 4;             // tile groups
  static constexpr int kThreads = (NC + 1) * 32;
};

// ST stages of K + V (6: 192 KB in flight per SM).  ST must be EVEN in the decode mode: its two
// consumer groups take alternate tiles, and with an odd ring a group can reach a stage two
// phases ahead of the other's pending tile, where the mbarrier parity wait aliases (a 3-stage
// ring, tried for two CTAs per SM, failed the bit-exactness tests for that reason).
template <int D, int ST = STAGES>
struct Smem {
  static constexpr int kSlab = TN * 128;            // [TN rows x 64 bf16] swizzled
  static constexpr int kTile = (D / 64) * kSlab;    // one K (or V) tile
  static constexpr int kStage = 2 * kTile;          // K + V
  static constexpr int kBarOff = ST * kStage;
  static constexpr int kQOff = kBarOff + 2 * ST * 8;  // fused decode: rotated q [16][D] bf16
  static constexpr int kBytes = kQOff + 16 * D * 2 + 1024;
};

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                          uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// byte address of (row, 16-byte chunk) inside a [rows x 64 bf16] 128B-swizzled slab
__device__ __forceinline__ uint32_t swz(uint32_t slab, int row, int chunk) {
  return slab + row * 128 + (((chunk ^ row) & 7) << 4);
}

}  // namespace p2

#ifdef STAR_K1_TRACE
// K2 timeline (tracing library only, tools/k2_trace.py): per CTA, globaltimer ns at
// [0] entry, [1] first K/V tile landed (consumer warp 0), [2] main loop done (warp 0),
// [3] split partial stored (thread 0), [4] fix-up: all splits' words seen, [5] exit
// (thread 0), [6] fused exchange: every rank's words seen, [7] fused exchange: arrived,
// [8] kv_len loaded after griddepcontrol.wait (thread 0), [9] main loop done (warp 4, the
// other tile group), [10] every warp's loop done (decode merge, first barrier), [11] warp
// partials staged (second barrier).
constexpr int kK2TrSlots = 12;
constexpr int kK2TrCtas = 2048;
__device__ unsigned long long g_k2_trace[kK2TrCtas][kK2TrSlots];
__device__ __forceinline__ void k2_tr(int slot) {
  const int cta = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  if (cta < kK2TrCtas) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_k2_trace[cta][slot] = t;
  }
}
#define K2_TR(cond, slot) \
  do {                    \
    if (cond) k2_tr(slot); \
  } while (0)
// K2q timeline of CTA 0 (clock64): [tile][8] = softmax warp 0 lane 0: S seen, half max,
// maxima swapped, exps + packs done, P handed over; MMA lane: P seen, P.V issued, next S issued
__device__ long long g_k2q_trace[256][8];
#define K2Q_TR(cond, t, slot)                                                   \
  do {                                                                          \
    if ((cond) && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (t) < 256) \
      g_k2q_trace[t][slot] = clock64();                                         \
  } while (0)
#else
#define K2Q_TR(cond, t, slot) \
  do {                        \
  } while (0)
#define K2_TR(cond, slot) \
  do {                    \
  } while (0)
#endif

// Split-K fix-up: the last CTA of a (sequence, kv head) to finish folds the gridDim.x
// split partials (still L2-resident) with the merge rule and re-arms the counter.
// Consumer threads only (the producer has exited).  This tail is pure latency after the
// last split lands, so it is one round of L2 loads: each thread takes two output elements
// and loads the lse and out of 16 splits for both at once (64 loads in flight), folding
// further groups of 16 splits, if any, online (running max, as the kernel's tile fold).
template <int D, int NT>
__device__ void split_fixup(unsigned char* smem, int b, int kvh, int r_lo, int r_n, int lq,
                            int hq, int G,
                            const float* ws_out, const float* ws_lse, int64_t part_rows,
                            float* final_out, float* final_lse, int* counters,
                            const PeerPush& pp) {
  constexpr int PS = 16;  // splits per load round
  const int tid = threadIdx.x;
  const int nsp = gridDim.x;
  int* flag = reinterpret_cast<int*>(smem);
  named_barrier_sync(1, NT);  // every consumer's partial stores precede thread 0's release
  if (tid == 0) {
    __threadfence();
    const int old = atomicAdd(&counters[b * gridDim.y + blockIdx.y], 1);
    __threadfence();
    *flag = (old == nsp - 1);
  }
  named_barrier_sync(1, NT);
  if (!*flag) return;
  const uint32_t ep = pp.L.world ? exchange_epoch(pp) : 0u;
  for (int e0 = tid; e0 < r_n * D; e0 += 2 * NT) {
    int64_t orow[2];
    int c[2];
    bool ok[2];
    float m[2] = {-INFINITY, -INFINITY}, acc[2] = {0.f, 0.f}, o[2] = {0.f, 0.f};
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int e = e0 + k * NT;
      ok[k] = e < r_n * D;
      const int rr = r_lo + (ok[k] ? e : 0) / D;
      c[k] = (ok[k] ? e : 0) % D;
      orow[k] = ((int64_t)b * lq + rr / G) * hq + kvh * G + rr % G;
    }
    for (int p0 = 0; p0 < nsp; p0 += PS) {
      float lv[2][PS], ov[2][PS];
#pragma unroll
      for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int u = 0; u < PS; ++u) {
          const bool in = ok[k] && p0 + u < nsp;
          lv[k][u] = in ? __ldcg(ws_lse + (p0 + u) * part_rows + orow[k]) : -INFINITY;
          ov[k][u] = in ? __ldcg(ws_out + ((p0 + u) * part_rows + orow[k]) * D + c[k]) : 0.f;
        }
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        float mn = m[k];
#pragma unroll
        for (int u = 0; u < PS; ++u) mn = fmaxf(mn, lv[k][u]);
        if (mn == -INFINITY) continue;  // nothing visible yet (empty splits)
        const float sc = __expf(m[k] - mn);  // 0 while m is -inf
        acc[k] *= sc;
        o[k] *= sc;
#pragma unroll
        for (int u = 0; u < PS; ++u) {
          const float w = lv[k][u] == -INFINITY ? 0.f : __expf(lv[k][u] - mn);
          acc[k] += w;
          o[k] = fmaf(w, ov[k][u], o[k]);
        }
        m[k] = mn;
      }
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      if (!ok[k]) continue;
      put_out(pp, ep, false, final_out, orow[k] * D + c[k], acc[k] > 0.f ? o[k] / acc[k] : 0.f);
      if (c[k] == 0)
        put_lse(pp, ep, false, final_lse, orow[k],
                acc[k] > 0.f ? m[k] + __logf(acc[k]) : -INFINITY);
    }
  }
  if (tid == 0) counters[b * gridDim.y + blockIdx.y] = 0;  // re-arm for the next launch
}

// The whole peer exchange inside K2 (pp.merge; word mode, so every CTA of every rank is
// co-resident and a CTA waits only on the peers' CTAs of the same slice, never on an
// unscheduled CTA): after pushing its slice of the group's partial to every box, the CTA
// polls every rank's words of that slice in its own box and folds them in ascending rank
// order with the merge rule of merge_partials (fp64 weights, as K3x), writing the merged
// fp32 out / lse.  The last CTA of the grid to finish advances the box's epoch.
template <int D, int NT>
__device__ void exchange_merge_slice(int b, int kvh, int r_lo, int lq, int hq, int G, int lo,
                                     int hi,
                                     uint32_t ep, float* out, float* lse, const PeerPush& pp) {
  void* box = pp.box[pp.rank];
  const int par = (int)(ep & 1u);
  const int world = pp.L.world;
  for (int e = lo + (int)threadIdx.x; e < hi; e += NT) {
    const int rr = r_lo + e / D, c = e % D;
    const int64_t orow = ((int64_t)b * lq + rr / G) * hq + kvh * G + rr % G;
    float lv[kMaxPeers], ov[kMaxPeers];
    uint64_t t0 = 0;
    for (;;) {
      bool all = true;
#pragma unroll
      for (int r = 0; r < kMaxPeers; ++r) {
        if (r >= world) break;
        const uint2* sl = pp.L.slot(box, par, r);
        const uint2 wl = ld_word(sl + pp.L.rows * pp.L.d + orow);
        const uint2 wo = ld_word(sl + orow * D + c);
        all &= (wl.y == ep) & (wo.y == ep);
        lv[r] = __uint_as_float(wl.x);
        ov[r] = __uint_as_float(wo.x);
      }
      if (all) break;
      if (t0 == 0) t0 = globaltimer_ns();
      if (globaltimer_ns() - t0 > pp.timeout_ns) __trap();  // a peer never delivered
    }
    K2_TR(e == lo, 6);
    double mx = -INFINITY;
#pragma unroll
    for (int r = 0; r < kMaxPeers; ++r)
      if (r < world) mx = fmax(mx, (double)lv[r]);
    double acc = 0.0;
    float w[kMaxPeers];
#pragma unroll
    for (int r = 0; r < kMaxPeers; ++r) {
      if (r >= world) break;
      const double x = lv[r] == -INFINITY ? 0.0 : exp((double)lv[r] - mx);
      w[r] = (float)x;
      acc += x;
    }
    const float inv = acc > 0.0 ? (float)(1.0 / acc) : 0.f;
    float o = 0.f;
#pragma unroll
    for (int r = 0; r < kMaxPeers; ++r)
      if (r < world) o = fmaf(w[r], ov[r], o);
    out[orow * D + c] = o * inv;
    if (c == 0 && lse != nullptr) lse[orow] = acc > 0.0 ? (float)(mx + log(acc)) : -INFINITY;
  }
  // every CTA of the grid read the box epoch before pushing; the last to arrive advances it
  named_barrier_sync(1, NT);
  if (threadIdx.x == 0) {
    uint32_t* hdr = pp.L.header(box);
    const uint32_t total = gridDim.x * gridDim.y * gridDim.z;
    // no fence before the arrival: this CTA's read of the epoch completed long ago (its
    // value addressed the pushes and the polls above), so the arrival cannot overtake it
    if (atomicAdd(hdr + 1, 1u) == total - 1u) {
      hdr[1] = 0u;
      hdr[0] = ep;
      __threadfence();
    }
    K2_TR(true, 7);
  }
}

// Split fix-up without atomics or fences (word mode): every split CTA stores its partial as
// {value, epoch} words (8-byte single-copy-atomic vector stores); then EVERY split CTA of the
// (sequence, kv head) folds 1/nsp of the group's output elements, polling the words of all
// splits until they carry the launch's epoch.  The host picks this mode only when the whole
// grid is co-resident (one CTA per SM), so the spinning CTAs cannot starve a split that has
// not started.  Against the arrival-counter fix-up this removes the fence + atomic + fence
// round and spreads the one-CTA merge tail (two load rounds + fold) over the group
// (tools/k2_trace.py: 16K rows, last split stored -> exit 3.8 us -> see DESIGN §3 K2).
template <int D, int NT, int EG = 1>
__device__ void split_merge_words(int b, int kvh, int r_lo, int r_n, int lq, int hq, int G,
                                  const uint2* w_out,
                                  const uint2* w_lse, int64_t part_rows, uint32_t es,
                                  float* final_out, float* final_lse, uint32_t* grp_epoch,
                                  const PeerPush& pp) {
  // EG consecutive output elements of one row per thread (EG = 4: the query encode's 128-row
  // slices): the row's lse words are loaded once and the out words as 16-byte pairs, so each
  // thread has all its loads of a split round in flight together (EG = 1: the decode form).
  // The per-element arithmetic (and so the result) does not depend on EG.
  static_assert(EG == 1 || (EG == 4 && D % 4 == 0), "element groups of 1 or 4");
  // splits per load round (PS lse + PS x EG out words in flight; 8 x 4 keeps the query
  // encode's fold inside the registers the 12-warp layout leaves)
  constexpr int PS = EG == 1 ? 16 : 8;
  const int tid = threadIdx.x;
  const int nsp = gridDim.x;
  const int total = r_n * D;
  const int per = (total + nsp - 1) / nsp;
  const int lo = blockIdx.x * per, hi = min(total, lo + per);
  named_barrier_sync(1, NT);  // this CTA's own words are visible to its polls
  // every CTA reads the box epoch, also one whose slice is empty (lo >= hi): it still counts
  // as an arrival in exchange_merge_slice, and if it arrives last it stores this epoch back
  const uint32_t ep = pp.L.world ? exchange_epoch(pp) : 0u;
  // groups of EG elements aligned to EG (a group never crosses a row: D % EG == 0); only the
  // elements inside [lo, hi) are this CTA's
  const int g_lo = lo / EG, g_hi = (hi + EG - 1) / EG;
  for (int g = (lo < hi ? g_lo : g_hi) + tid; g < g_hi; g += NT) {
    const int e0 = g * EG;
    const int rr = r_lo + e0 / D, c = e0 % D;
    const int64_t orow = ((int64_t)b * lq + rr / G) * hq + kvh * G + rr % G;
    bool in[EG];
#pragma unroll
    for (int k = 0; k < EG; ++k) in[k] = e0 + k >= lo && e0 + k < hi;
    float m = -INFINITY, acc = 0.f, o[EG];
#pragma unroll
    for (int k = 0; k < EG; ++k) o[k] = 0.f;
    for (int p0 = 0; p0 < nsp; p0 += PS) {
      float lv[PS], ov[PS][EG];
      uint64_t t0 = 0;
      for (;;) {
        bool all = true;
#pragma unroll
        for (int u = 0; u < PS; ++u) {
          uint2 wl = make_uint2(__float_as_uint(-INFINITY), es);
          uint2 wo[EG];
#pragma unroll
          for (int k = 0; k < EG; ++k) wo[k] = make_uint2(0u, es);
          if (p0 + u < nsp) {
            wl = ld_word(w_lse + (p0 + u) * part_rows + orow);
            const uint2* src = w_out + ((p0 + u) * part_rows + orow) * D + c;
            if (EG == 4) {
              const uint4 a = ld_word4(src), bq = ld_word4(src + 2);
              wo[0] = make_uint2(a.x, a.y);
              wo[EG > 1 ? 1 : 0] = make_uint2(a.z, a.w);
              wo[EG > 2 ? 2 : 0] = make_uint2(bq.x, bq.y);
              wo[EG > 3 ? 3 : 0] = make_uint2(bq.z, bq.w);
            } else {
              wo[0] = ld_word(src);
            }
          }
          all &= (wl.y == es);
          lv[u] = __uint_as_float(wl.x);
#pragma unroll
          for (int k = 0; k < EG; ++k) {
            all &= (!in[k]) | (wo[k].y == es);
            ov[u][k] = __uint_as_float(wo[k].x);
          }
        }
        if (all) break;
        if (t0 == 0) t0 = globaltimer_ns();
        if (globaltimer_ns() - t0 > pp.timeout_ns) {  // a split never landed: fail loudly
          if ((threadIdx.x & 31) == 0)
            printf("star K2 split fold timed out: block (%d,%d,%d) row %d col %d epoch %u "
                   "splits %d-%d: lse word epoch %u\n", (int)blockIdx.x, (int)blockIdx.y,
                   (int)blockIdx.z, rr, c, es, p0, p0 + PS - 1,
                   (p0 < nsp) ? ld_word(w_lse + p0 * part_rows + orow).y : 0u);
          __trap();
        }
      }
      K2_TR(g == g_lo && p0 == 0, 4);
      float mn = m;
#pragma unroll
      for (int u = 0; u < PS; ++u) mn = fmaxf(mn, lv[u]);
      if (mn == -INFINITY) continue;  // nothing visible yet (empty splits)
      const float sc = __expf(m - mn);  // 0 while m is -inf
      acc *= sc;
#pragma unroll
      for (int k = 0; k < EG; ++k) o[k] *= sc;
#pragma unroll
      for (int u = 0; u < PS; ++u) {
        const float w = lv[u] == -INFINITY ? 0.f : __expf(lv[u] - mn);
        acc += w;
#pragma unroll
        for (int k = 0; k < EG; ++k) o[k] = fmaf(w, ov[u][k], o[k]);
      }
      m = mn;
    }
#pragma unroll
    for (int k = 0; k < EG; ++k)
      if (in[k]) put_out(pp, ep, false, final_out, orow * D + c + k, acc > 0.f ? o[k] / acc : 0.f);
    if (c == 0 && in[0]) put_lse(pp, ep, false, final_lse, orow, acc > 0.f ? m + __logf(acc) : -INFINITY);
  }
  // every split's words were seen, so every CTA of the group has read the epoch: advance it
  // for the next launch (all CTAs of the group store the same value)
  if (tid == 0) grp_epoch[b * gridDim.y + blockIdx.y] = es;
  if (pp.merge)
    exchange_merge_slice<D, NT>(b, kvh, r_lo, lq, hq, G, lo, hi, ep, final_out, final_lse, pp);
}

// The query encode's fold as a separate (not inlined) function: its registers then do not
// add to the 12-warp main loop's (inlined, the EG = 4 fold spilled there).  The decode kernel
// keeps the inlined fold: a call measured slower at short contexts.
template <int D, int NT, int EG>
__device__ __noinline__ void split_merge_words_call(int b, int kvh, int r_lo, int r_n, int lq, int hq,
                                                    int G, const uint2* w_out, const uint2* w_lse,
                                                    int64_t part_rows, uint32_t es, float* final_out,
                                                    float* final_lse, uint32_t* grp_epoch,
                                                    const PeerPush& pp) {
  split_merge_words<D, NT, EG>(b, kvh, r_lo, r_n, lq, hq, G, w_out, w_lse, part_rows, es, final_out,
                               final_lse, grp_epoch, pp);
}

// ---- fused decode append helpers (DecodeAppend, exchange.cuh) ----
// {cos, sin} of pair i at position p: the decode-position table entry when p is inside it,
// else formed in place with the fp64 expression of rope_kernel (bit-identical either way)
__device__ __noinline__ double2 rope_cs_slow(double theta, int64_t p, int i, int d) {
  double sn, c;
  sincos((double)p * pow(theta, -2.0 * (double)i / (double)d), &sn, &c);
  return make_double2(c, sn);
}
__device__ __forceinline__ double2 rope_cs(const DecodeAppend& ap, int64_t p, int i, int d) {
  const int64_t tp = p - ap.rtab_pos0;
  if (ap.rtab != nullptr && tp >= 0 && tp < ap.rtab_n)
    return reinterpret_cast<const double2*>(ap.rtab)[tp * (d >> 1) + i];
  return rope_cs_slow(ap.theta, p, i, d);  // off the table: the fp64 angle (slow, rare)
}
// rotate one adjacent bf16 pair (packed in a 32-bit word) in fp64, round as the append kernel
__device__ __forceinline__ uint32_t rope_pair_bf16(uint32_t w, double2 e) {
  const double x0 = __bfloat162float(__ushort_as_bfloat16((unsigned short)(w & 0xFFFFu)));
  const double x1 = __bfloat162float(__ushort_as_bfloat16((unsigned short)(w >> 16)));
  const __nv_bfloat16 y0 = __float2bfloat16_rn(__double2float_rn(x0 * e.x - x1 * e.y));
  const __nv_bfloat16 y1 = __float2bfloat16_rn(__double2float_rn(x0 * e.y + x1 * e.x));
  return (uint32_t)__bfloat16_as_ushort(y0) | ((uint32_t)__bfloat16_as_ushort(y1) << 16);
}
// the new row of kv head kvh, prefetched by the consumer warp that owns it: rotated k and raw
// v, lane l holding pairs l and l + 32 (the same rounding as kv_append_kernel)
template <int D>
struct NewRow {
  uint32_t k[D / 64], v[D / 64];
};
template <int D>
__device__ __forceinline__ NewRow<D> decode_new_row(const DecodeAppend& ap, int b, int kvh, int lane) {
  const int64_t p = ap.cur_cs != nullptr ? 0 : ap.pos[b];
  const uint32_t* kn = reinterpret_cast<const uint32_t*>(
      reinterpret_cast<const __nv_bfloat16*>(ap.k_new) + (int64_t)b * ap.kv_rs + (int64_t)kvh * D);
  const uint32_t* vn = reinterpret_cast<const uint32_t*>(
      reinterpret_cast<const __nv_bfloat16*>(ap.v_new) + (int64_t)b * ap.kv_rs + (int64_t)kvh * D);
  NewRow<D> nr;
  double2 cs[D / 64];
  uint32_t kw[D / 64];
  const int64_t tp = p - ap.rtab_pos0;
  const bool cur = ap.cur_cs != nullptr;
  const bool tab = cur || (ap.rtab != nullptr && tp >= 0 && tp < ap.rtab_n);
  const double2* src = cur ? reinterpret_cast<const double2*>(ap.cur_cs) + (int64_t)b * (D / 2)
                           : reinterpret_cast<const double2*>(ap.rtab) + tp * (D / 2);
#pragma unroll
  for (int u = 0; u < D / 64; ++u) {
    const int i = lane + 32 * u;  // pair index
    kw[u] = kn[i];
    nr.v[u] = vn[i];
    if (tab) cs[u] = src[i];
  }
  if (!tab)
#pragma unroll
    for (int u = 0; u < D / 64; ++u) cs[u] = rope_cs_slow(ap.theta, p, lane + 32 * u, D);
#pragma unroll
  for (int u = 0; u < D / 64; ++u) nr.k[u] = rope_pair_bf16(kw[u], cs[u]);
  return nr;
}
// write the new row into the cache (global, for the next tokens) and into row `r` of the
// staged K / V tile (swizzled smem), so this launch attends over it without a round trip
template <int D>
__device__ __forceinline__ void decode_put_row(const NewRow<D>& nr, const DecodeAppend& ap,
                                               int64_t pool_row, unsigned char* kb,
                                               unsigned char* vb, int r, int lane) {
  uint32_t* kd = reinterpret_cast<uint32_t*>(reinterpret_cast<__nv_bfloat16*>(ap.kp) + pool_row * D);
  uint32_t* vd = reinterpret_cast<uint32_t*>(reinterpret_cast<__nv_bfloat16*>(ap.vp) + pool_row * D);
#pragma unroll
  for (int u = 0; u < D / 64; ++u) {
    const int i = lane + 32 * u, c = 2 * i;  // pair i = elements c, c + 1
    kd[i] = nr.k[u];
    vd[i] = nr.v[u];
    const int slab = c >> 6, chunk = (c & 63) >> 3;
    const int off = slab * p2::TN * 128 + r * 128 + (((chunk ^ r) & 7) << 4) + (c & 7) * 2;
    *reinterpret_cast<uint32_t*>(kb + off) = nr.k[u];
    *reinterpret_cast<uint32_t*>(vb + off) = nr.v[u];
  }
}

template <int D, bool KEYSPLIT, int ST = p2::STAGES>
__global__ void __launch_bounds__(p2::Cons<KEYSPLIT>::kThreads) phase2_mma_kernel(
    const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
    const __nv_bfloat16* __restrict__ q, int lq, int hq, int hkv,
    const int32_t* __restrict__ page_table, int pages_per_seq, int page_size,
    const int32_t* __restrict__ kv_len, int own_tail, int64_t chunk, float* __restrict__ out,
    float* __restrict__ lse, int64_t part_stride_rows, float scale_log2,
    float* __restrict__ final_out, float* __restrict__ final_lse, int* __restrict__ counters,
    uint32_t* __restrict__ grp_epoch, const PeerPush pp, const DecodeAppend ap) {
  using namespace p2;
  using SM = Smem<D, ST>;
  static_assert(!KEYSPLIT || ST % 2 == 0, "decode mode: the ring depth must be even (see Smem)");
  constexpr int NC = Cons<KEYSPLIT>::NC, NG = Cons<KEYSPLIT>::NG;
  constexpr int NT_D = D / 8;  // n-tiles over head dim (P.V output)
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_align1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + SM::kBarOff);
  uint64_t* empty = full + ST;

  // row mode (G*lq > 16 query rows, e.g. a 32-token query encode) splits the group's rows
  // into 64-row blocks along grid.y, so every K/V tile is streamed once per split (the row
  // blocks of a split run side by side and share it through L2) instead of once per pass
  const int QRg = (hq / hkv) * lq;
  const int n_rb = KEYSPLIT ? 1 : (QRg + 63) / 64;
  const int split = blockIdx.x, kvh = blockIdx.y / n_rb, rb = blockIdx.y % n_rb, b = blockIdx.z;
  const int r_lo = KEYSPLIT ? 0 : rb * 64;
  const int r_n = KEYSPLIT ? QRg : min(64, QRg - r_lo);
  // a programmatic dependent (K3x of the peer exchange, which only polls the words this
  // kernel stores) may launch now and wait on SMs beside us instead of behind a kernel boundary
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  K2_TR(threadIdx.x == 0, 0);
  const int G = hq / hkv;
  const int QR = G * lq;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r0 = (int64_t)split * chunk;
  const int32_t* table = page_table + (int64_t)b * pages_per_seq;
  float* out_part = out + (int64_t)split * part_stride_rows * D;
  float* lse_part = lse + (int64_t)split * part_stride_rows;
  const int n_pass = 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 4);  // one group of four consumer warps per tile
    }
    fence_mbar_init();
  }
  if (warp == NC && lane == 0) {
    tma_prefetch(&tm_k);
    tma_prefetch(&tm_v);
  }
  __syncthreads();
  // Launched as a programmatic dependent (PDL) of the kernel before it (e.g. the decode
  // append that writes q's row and bumps kv_len): everything above overlapped that kernel;
  // nothing it writes is read before this point.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int64_t base_len = ld_after_wait(kv_len + b);
  const int64_t len = base_len + (ap.on ? ap.add : 0);
  const int64_t r1 = min(len, r0 + chunk);
  const int64_t tail0 = len - own_tail;
  const int ntiles = r1 > r0 ? (int)((r1 - r0 + TN - 1) / TN) : 0;
  K2_TR(threadIdx.x == 0 && ntiles >= 0, 8);

  if (warp == NC) {
    // ================= TMA producer =================
    // The whole warp resolves page-table entries 32 tiles at a time (lane l -> tile t0+l,
    // one coalesced load, the next group's load in flight while this group is issued);
    // lane 0 then issues the TMA loads back to back, so the ring fills without a
    // dependent table read in front of every tile.
    // bounded by the split's chunk, not by kv_len: the first table load does not wait for
    // the kv_len load (tiles past the sequence end are resolved but never issued)
    const int tiles_cap = (int)(chunk / TN);
    auto page_row = [&](int t) -> int {
      if (t >= tiles_cap) return 0;
      const int64_t row = r0 + (int64_t)t * TN;
      const int64_t pi = row / page_size;
      if (pi >= pages_per_seq) return 0;
      const int64_t page = table[pi];
      return (int)((page * hkv + kvh) * page_size + row % page_size);
    };
    int it = 0;
    for (int pass = 0; pass < n_pass; ++pass) {
      int cur = page_row(lane);
      for (int t0 = 0; t0 < ntiles; t0 += 32) {
        const int nxt = page_row(t0 + 32 + lane);
        const int cnt = min(32, ntiles - t0);
        for (int u = 0; u < cnt; ++u, ++it) {
          const int prow = __shfl_sync(0xffffffffu, cur, u);
          if (lane == 0) {
            const int st = it % ST;
            if (it >= ST) mbar_wait(&empty[st], ((it / ST) + 1) & 1);
            unsigned char* kb = smem + st * SM::kStage;
            mbar_expect_tx(&full[st], SM::kStage);
#pragma unroll
            for (int a = 0; a < D / 64; ++a) {
              tma_load_2d(kb + a * SM::kSlab, &tm_k, &full[st], a * 64, prow);
              tma_load_2d(kb + SM::kTile + a * SM::kSlab, &tm_v, &full[st], a * 64, prow);
            }
          }
          __syncwarp();
        }
        cur = nxt;
      }
    }
    return;
  }

  // ================= consumers =================
  // epoch of the peer exchange this CTA's final partial belongs to (one split per group)
  const uint32_t ep = (gridDim.x == 1 && pp.L.world > 0) ? exchange_epoch(pp) : 0u;
  // word-mode split fix-up: this split's partial goes out as {value, epoch} words
  const bool words = grp_epoch != nullptr && gridDim.x > 1;
  // read once per CTA (thread 0) before any word is stored, as K2q (see there)
  __shared__ uint32_t es_sh;
  if (threadIdx.x == 0)
    es_sh = words ? next_epoch(__ldcg(grp_epoch + b * gridDim.y + blockIdx.y)) : 0u;
  named_barrier_sync(1, NC * 32);
  const uint32_t es = es_sh;
  uint2* const w_out = reinterpret_cast<uint2*>(out);
  uint2* const w_lse = w_out + (int64_t)gridDim.x * part_stride_rows * D;
  uint2* const wsp_out = w_out + (int64_t)split * part_stride_rows * D;
  uint2* const wsp_lse = w_lse + (int64_t)split * part_stride_rows;
  const int g4 = lane >> 2, t4 = lane & 3;  // mma fragment coordinates
  const int grp = warp >> 2, wq4 = warp & 3;  // tile group, warp within the group
  for (int pass = 0; pass < n_pass; ++pass) {
    const int qbase = KEYSPLIT ? 0 : r_lo + pass * 64 + wq4 * 16;  // first q row of this warp
    // ---- Q A-fragments (16 rows x D) straight from global ----
    uint32_t qa[D / 16][4];
    {
      const int rA = qbase + g4, rB = qbase + g4 + 8;
      const __nv_bfloat16* qpA = nullptr;
      const __nv_bfloat16* qpB = nullptr;
      if (rA < QR) qpA = q + (((int64_t)b * lq + rA / G) * hq + kvh * G + rA % G) * D;
      if (rB < QR) qpB = q + (((int64_t)b * lq + rB / G) * hq + kvh * G + rB % G) * D;
      if (KEYSPLIT && ap.on) {
        // fused decode: the QR x D pre-RoPE rows of this group are rotated ONCE per CTA (one
        // pair per consumer thread, the append kernel's fp64 rotation) into shared memory;
        // every warp then takes its fragments from there.  lq == 1: row r is head kvh*G + r.
        uint32_t* qs = reinterpret_cast<uint32_t*>(smem + SM::kQOff);
        const __nv_bfloat16* qr = reinterpret_cast<const __nv_bfloat16*>(ap.q_raw) + (int64_t)b * ap.q_rs;
        const int64_t p = ap.cur_cs != nullptr ? 0 : ap.pos[b];
        for (int idx = threadIdx.x; idx < QR * (D / 2); idx += NC * 32) {
          const int r = idx / (D / 2), i = idx % (D / 2);
          const uint32_t raw = *reinterpret_cast<const uint32_t*>(qr + (int64_t)(kvh * G + r) * D + 2 * i);
          const double2 cs = ap.cur_cs != nullptr
                                 ? reinterpret_cast<const double2*>(ap.cur_cs)[(int64_t)b * (D / 2) + i]
                                 : rope_cs(ap, p, i, D);
          qs[idx] = rope_pair_bf16(raw, cs);
        }
        named_barrier_sync(1, NC * 32);
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
          const int c = ks * 16 + t4 * 2;
          const int rA2 = qbase + g4, rB2 = qbase + g4 + 8;
          qa[ks][0] = rA2 < QR ? qs[(rA2 * D + c) >> 1] : 0u;
          qa[ks][1] = rB2 < QR ? qs[(rB2 * D + c) >> 1] : 0u;
          qa[ks][2] = rA2 < QR ? qs[(rA2 * D + c + 8) >> 1] : 0u;
          qa[ks][3] = rB2 < QR ? qs[(rB2 * D + c + 8) >> 1] : 0u;
        }
      } else {
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
          const int c = ks * 16 + t4 * 2;
          qa[ks][0] = qpA ? *reinterpret_cast<const uint32_t*>(qpA + c) : 0u;
          qa[ks][1] = qpB ? *reinterpret_cast<const uint32_t*>(qpB + c) : 0u;
          qa[ks][2] = qpA ? *reinterpret_cast<const uint32_t*>(qpA + c + 8) : 0u;
          qa[ks][3] = qpB ? *reinterpret_cast<const uint32_t*>(qpB + c + 8) : 0u;
        }
      }
    }
    // query row index (for the own-tail mask) of my two fragment rows
    const int qiA = (qbase + g4) / G, qiB = (qbase + g4 + 8) / G;
    float o[NT_D][4];
#pragma unroll
    for (int n = 0; n < NT_D; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
    float mA = -INFINITY, mB = -INFINITY, lA = 0.f, lB = 0.f;

    constexpr int KW = KEYSPLIT ? TN / 4 : TN;  // keys per warp per tile
    constexpr int NT_K = KW / 8;                 // n-tiles over keys
    const int kofs = KEYSPLIT ? wq4 * KW : 0;
    // fused decode append: the warp whose keys hold row base_len (tile nt_new, key slot
    // r_new) prefetches the new row now and patches it into the staged tile (and the cache)
    int nt_new = -1, r_new = 0;
    NewRow<D> nrow{};
    if (KEYSPLIT && ap.on && ap.add && base_len >= r0 && base_len < r1) {
      const int tn = (int)((base_len - r0) / TN), rr = (int)((base_len - r0) % TN);
      if (tn % NG == grp && rr / KW == wq4) {
        nt_new = tn;
        r_new = rr;
        nrow = decode_new_row<D>(ap, b, kvh, lane);
      }
    }

    for (int t = grp; t < ntiles; t += NG) {
      const int it = pass * ntiles + t;  // the producer's running tile index
      const int st = it % ST;
      mbar_wait(&full[st], (it / ST) & 1);
      K2_TR(it == 0 && threadIdx.x == 0, 1);
      const uint32_t kbase = smem_u32(smem + st * SM::kStage);
      const uint32_t vbase = kbase + SM::kTile;
      const int64_t row0 = r0 + (int64_t)t * TN + kofs;
      if (t == ntiles - 1 && (r1 - r0) % TN != 0) {
        // rows past the split end may hold stale (even non-finite) data: zero their V rows so
        // the masked p = 0 never meets a NaN.  Warp w clears tile rows [16w, 16w+16).
        const int valid = (int)((r1 - r0) % TN);
        unsigned char* vb = smem + st * SM::kStage + SM::kTile;
        for (int e = lane; e < 16 * (D / 8); e += 32) {
          const int rr = wq4 * 16 + e / (D / 8), chunk = e % (D / 8);
          if (rr >= valid)
            *reinterpret_cast<uint4*>(vb + (chunk >> 3) * SM::kSlab + rr * 128 +
                                      (((chunk ^ rr) & 7) << 4)) = make_uint4(0, 0, 0, 0);
        }
        if (KEYSPLIT)
          __syncwarp();
        else
          named_barrier_sync(1, NC * 32);
      }
      if (KEYSPLIT && t == nt_new) {
        const int64_t row = r0 + (int64_t)t * TN + r_new;
        const int64_t pool_row = ((int64_t)table[row / page_size] * hkv + kvh) * page_size + row % page_size;
        decode_put_row<D>(nrow, ap, pool_row, smem + st * SM::kStage, smem + st * SM::kStage + SM::kTile,
                          r_new, lane);
        __syncwarp();
      }
      // ---- S = Q K^T  (16 x KW) ----
      float sc[NT_K][4];
#pragma unroll
      for (int n = 0; n < NT_K; ++n) sc[n][0] = sc[n][1] = sc[n][2] = sc[n][3] = 0.f;
#pragma unroll
      for (int n = 0; n < NT_K; ++n) {
        const int krow = kofs + n * 8 + (lane & 7);
#pragma unroll
        for (int ks = 0; ks < D / 16; ks += 2) {
          // 4 matrices: d chunks 2ks, 2ks+1, 2ks+2, 2ks+3 of keys krow
          const int chunk = ks * 2 + (lane >> 3);
          const uint32_t addr = swz(kbase + (chunk >> 3) * SM::kSlab, krow, chunk & 7);
          uint32_t b0, b1, b2, b3;
          ldsm_x4(addr, b0, b1, b2, b3);
          mma16816(sc[n], qa[ks], b0, b1);
          mma16816(sc[n], qa[ks + 1], b2, b3);
        }
      }
      // ---- mask + online softmax (rows A = g4, B = g4 + 8) ----
      float tmA = -INFINITY, tmB = -INFINITY;
#pragma unroll
      for (int n = 0; n < NT_K; ++n) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t key = row0 + n * 8 + t4 * 2 + e;
          bool visA = key < r1, visB = visA;
          if (own_tail > 0 && key >= tail0) {
            visA = visA && (key - tail0) <= qiA;
            visB = visB && (key - tail0) <= qiB;
          }
          sc[n][e] = visA ? sc[n][e] * scale_log2 : -INFINITY;
          sc[n][2 + e] = visB ? sc[n][2 + e] * scale_log2 : -INFINITY;
          tmA = fmaxf(tmA, sc[n][e]);
          tmB = fmaxf(tmB, sc[n][2 + e]);
        }
      }
      tmA = fmaxf(tmA, __shfl_xor_sync(0xffffffffu, tmA, 1));
      tmA = fmaxf(tmA, __shfl_xor_sync(0xffffffffu, tmA, 2));
      tmB = fmaxf(tmB, __shfl_xor_sync(0xffffffffu, tmB, 1));
      tmB = fmaxf(tmB, __shfl_xor_sync(0xffffffffu, tmB, 2));
      // lazy rescale (as in K1): keep the stale max unless the tile max exceeds it by > 2^8;
      // numerator and denominator share the max, so the result is exact.
      const bool needA = tmA > mA + 8.f, needB = tmB > mB + 8.f;
      const float nA = needA ? tmA : mA, nB = needB ? tmB : mB;
      const float aA = (!needA || mA == -INFINITY) ? 1.f : ex2(mA - nA);
      const float aB = (!needB || mB == -INFINITY) ? 1.f : ex2(mB - nB);
      const float uA = (nA == -INFINITY) ? 0.f : nA, uB = (nB == -INFINITY) ? 0.f : nB;
      // P split into bf16 hi + lo parts: the P.V product then carries ~16 mantissa bits of P
      // (decode is HBM-bound, the extra MMAs are free) instead of bf16's 8.
      float sA = 0.f, sB = 0.f;
      uint32_t pa[NT_K][2], pl[NT_K][2];
#pragma unroll
      for (int n = 0; n < NT_K; ++n) {
        const float p0 = ex2(sc[n][0] - uA), p1 = ex2(sc[n][1] - uA);
        const float p2v = ex2(sc[n][2] - uB), p3 = ex2(sc[n][3] - uB);
        sA += p0 + p1;
        sB += p2v + p3;
        pa[n][0] = pack_bf16x2(p0, p1);
        pa[n][1] = pack_bf16x2(p2v, p3);
        pl[n][0] = pack_bf16x2(p0 - bf16lo(pa[n][0]), p1 - bf16hi(pa[n][0]));
        pl[n][1] = pack_bf16x2(p2v - bf16lo(pa[n][1]), p3 - bf16hi(pa[n][1]));
      }
      lA = lA * aA + sA;
      lB = lB * aB + sB;
      mA = nA;
      mB = nB;
      if (__any_sync(0xffffffffu, needA || needB)) {
#pragma unroll
        for (int n = 0; n < NT_D; ++n) {
          o[n][0] *= aA;
          o[n][1] *= aA;
          o[n][2] *= aB;
          o[n][3] *= aB;
        }
      }
      // ---- O += P V  (P: 16 x KW, V: KW x D) ----
#pragma unroll
      for (int kk = 0; kk < KW / 16; ++kk) {
        const uint32_t a[4] = {pa[2 * kk][0], pa[2 * kk][1], pa[2 * kk + 1][0], pa[2 * kk + 1][1]};
        const uint32_t al[4] = {pl[2 * kk][0], pl[2 * kk][1], pl[2 * kk + 1][0], pl[2 * kk + 1][1]};
        const int vrow = kofs + kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
#pragma unroll
        for (int nd = 0; nd < NT_D; nd += 2) {
          // 4 matrices (trans): keys +0/+8 x d chunk nd, nd+1
          const int chunk = nd + (lane >> 4);
          const uint32_t addr = swz(vbase + (chunk >> 3) * SM::kSlab, vrow, chunk & 7);
          uint32_t b0, b1, b2, b3;
          ldsm_x4_t(addr, b0, b1, b2, b3);
          mma16816(o[nd], a, b0, b1);
          mma16816(o[nd + 1], a, b2, b3);
          mma16816(o[nd], al, b0, b1);
          mma16816(o[nd + 1], al, b2, b3);
        }
      }
      fence_proxy_async_smem();  // generic-proxy zeroing above vs the next TMA write
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
    K2_TR(threadIdx.x == 0, 2);
    K2_TR(threadIdx.x == 128, 9);
    // row sums across the quad
    lA += __shfl_xor_sync(0xffffffffu, lA, 1);
    lA += __shfl_xor_sync(0xffffffffu, lA, 2);
    lB += __shfl_xor_sync(0xffffffffu, lB, 1);
    lB += __shfl_xor_sync(0xffffffffu, lB, 2);

    if (KEYSPLIT) {
      // ---- merge the NC warp partials in shared memory (stage buffers are idle now) ----
      // rows padded by 8 floats: the 8 fragment rows of a store land in distinct banks;
      // only the G*lq valid rows of the 16 M rows are staged (4 of 16 in Llama-8B decode)
      constexpr int SR = D + 8;
      float* so = reinterpret_cast<float*>(smem);             // [NC][16][SR]
      float* sm = so + NC * 16 * SR;                          // [NC][16] max
      float* sl = sm + NC * 16;                               // [NC][16] sum
      float* sw = sl + NC * 16;                               // [NC][16] merge weight
      float* slse = sw + NC * 16;                             // [16] row lse
      named_barrier_sync(1, NC * 32);
      K2_TR(threadIdx.x == 0, 10);
#pragma unroll
      for (int n = 0; n < NT_D; ++n) {
        const int c = n * 8 + t4 * 2;
        if (g4 < QR)
          *reinterpret_cast<float2*>(so + (warp * 16 + g4) * SR + c) = make_float2(o[n][0], o[n][1]);
        if (g4 + 8 < QR)
          *reinterpret_cast<float2*>(so + (warp * 16 + g4 + 8) * SR + c) =
              make_float2(o[n][2], o[n][3]);
      }
      if (t4 == 0) {
        sm[warp * 16 + g4] = mA;
        sm[warp * 16 + g4 + 8] = mB;
        sl[warp * 16 + g4] = lA;
        sl[warp * 16 + g4 + 8] = lB;
      }
      named_barrier_sync(1, NC * 32);
      // one thread per row: the warp weights 2^(m_w - m) / l of the row (so the element pass
      // below is a weighted sum with no exponential, division or logarithm) and its lse
      if (threadIdx.x < QR) {
        const int rr = threadIdx.x;
        float m = -INFINITY;
#pragma unroll
        for (int w = 0; w < NC; ++w) m = fmaxf(m, sm[w * 16 + rr]);
        float f[NC], l = 0.f;
#pragma unroll
        for (int w = 0; w < NC; ++w) {
          f[w] = m > -INFINITY ? ex2(sm[w * 16 + rr] - m) : 0.f;
          l += sl[w * 16 + rr] * f[w];
        }
        const float inv = l > 0.f ? 1.f / l : 0.f;
#pragma unroll
        for (int w = 0; w < NC; ++w) sw[w * 16 + rr] = f[w] * inv;
        slse[rr] = l > 0.f ? (m + __log2f(l)) * 0.6931471805599453f : -INFINITY;
      }
      named_barrier_sync(1, NC * 32);
      K2_TR(threadIdx.x == 0, 11);
      // two adjacent columns per thread (one 16-byte word pair / float2 store)
      for (int e = threadIdx.x; e < QR * (D / 2); e += NC * 32) {
        const int rr = e / (D / 2), c = 2 * (e % (D / 2));
        float2 acc = make_float2(0.f, 0.f);
#pragma unroll
        for (int w = 0; w < NC; ++w) {
          const float2 ov = *reinterpret_cast<const float2*>(so + (w * 16 + rr) * SR + c);
          const float wt = sw[w * 16 + rr];
          acc.x = fmaf(ov.x, wt, acc.x);
          acc.y = fmaf(ov.y, wt, acc.y);
        }
        const int64_t orow = ((int64_t)b * lq + rr / G) * hq + kvh * G + rr % G;
        // one split: this is the final partial (pushed to every rank's box when exchanging)
        if (words) {
          st_word2(wsp_out + orow * D + c, acc, es);
          if (c == 0) st_word(wsp_lse + orow, slse[rr], es);
        } else {
          put_out2(pp, ep, gridDim.x > 1, out_part, orow * D + c, acc);
          if (c == 0) put_lse(pp, ep, gridDim.x > 1, lse_part, orow, slse[rr]);
        }
      }
    } else {
      // ---- each warp owns its 16 rows ----
      const int rows[2] = {qbase + g4, qbase + g4 + 8};
      const float ls[2] = {lA, lB}, ms[2] = {mA, mB};
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int rr = rows[h];
        if (rr >= QR) continue;
        const int64_t orow = ((int64_t)b * lq + rr / G) * hq + kvh * G + rr % G;
        const float inv = ls[h] > 0.f ? 1.f / ls[h] : 0.f;
#pragma unroll
        for (int n = 0; n < NT_D; ++n) {
          const int c = n * 8 + t4 * 2;
          const float2 v2 = make_float2(o[n][2 * h] * inv, o[n][2 * h + 1] * inv);
          if (words)
            st_word2(wsp_out + orow * D + c, v2, es);
          else
            put_out2(pp, ep, gridDim.x > 1, out_part, orow * D + c, v2);
        }
        if (t4 == 0) {
          const float vl = ls[h] > 0.f ? (ms[h] + __log2f(ls[h])) * 0.6931471805599453f : -INFINITY;
          if (words)
            st_word(wsp_lse + orow, vl, es);
          else
            put_lse(pp, ep, gridDim.x > 1, lse_part, orow, vl);
        }
      }
    }
  }
  K2_TR(threadIdx.x == 0, 3);
  if (words) {
    split_merge_words<D, NC * 32>(b, kvh, r_lo, r_n, lq, hq, G, w_out, w_lse, part_stride_rows, es,
                                  final_out, final_lse, grp_epoch, pp);
  } else if (gridDim.x > 1 && counters != nullptr) {
    split_fixup<D, NC * 32>(smem, b, kvh, r_lo, r_n, lq, hq, G, out, lse, part_stride_rows, final_out,
                            final_lse, counters, pp);
  }
  K2_TR(threadIdx.x == 0, 5);
}

// ------------------------------------------------------------------ K2q: tcgen05 query encode
// Phase-2 query encode (ss/sim.py:254-281 with own_tail = l_q; partial_attention on every
// other host): G*l_q in (16, 128] query rows per (sequence, kv head) — e.g. l_q = 32 at
// Llama-8B heads — are PACKED into one M = 128 tcgen05 tile (row r = token r/G, head r%G,
// loaded by one 3-D TMA box {64, G, l_q} per 64-column slab), so every 128-key K/V tile
// feeds one QK^T and one P.V of M = 128 on the tensor pipe instead of 16-row mma.sync
// fragments.  Keys come straight from the paged pool (two 64-key TMA boxes per tile through
// the page table, as K2).  One key range ("split") per CTA; the split partials fold by the
// word-mode fix-up (split_merge_words), which also pushes / merges the peer exchange.
// TMEM: S double-buffered (S_a | S_b | O = 384 of 512 columns), so QK^T of tile j+1 runs
// while the softmax of tile j does.  P goes back over its S buffer as a bf16 hi/lo pair
// (hi in columns [0,64), lo in [64,128)) and P.V runs on both halves: ≈16 mantissa bits of
// P, as K2's mma.sync path, which keeps the 2e-3 parity bound (bf16 P alone measured 2.04e-3
// at 5K keys).  Softmax as K1 (one thread per row = TMEM lane, lazy O rescale); padding rows
// past G*l_q and keys past the split end or the row's own-tail limit are masked.
// K2q's mbarrier waits: bounded and reporting (block, thread, site, parity) in a debug build
// (-DSTAR_K2Q_DEBUG, `make debug`), plain otherwise
#ifdef STAR_K2Q_DEBUG
#define K2Q_WAIT(tag, bar, par) mbar_wait_dbg(bar, par, 100 + (tag))
#else
#define K2Q_WAIT(tag, bar, par) mbar_wait(bar, par)
#endif
namespace p2q {
constexpr int BN = 128;                 // keys per tile
constexpr int kSlab = 128 * 128;        // [128 rows x 64 bf16] SW128 slab
constexpr int kTile = 2 * kSlab;        // [128 x 128] bf16
// K runs kSBuf tiles ahead of the softmax (QK^T of tile j+3 is issued right after P.V(j)),
// so it gets the deeper ring; P.V(j)'s V tile is needed one period after P(j)
constexpr int KST = 3, VST = 2;
constexpr int kQOff = 0;
constexpr int kKOff = kQOff + kTile;
constexpr int kVOff = kKOff + KST * kTile;
constexpr int kRedOff = kVOff + VST * kTile;      // [2 parity][2 half][128] f32 row maxima
constexpr int kLOff = kRedOff + 2 * 2 * 128 * 4;  // [2 half][128] f32 partial row sums
constexpr int kBarOff = kLOff + 2 * 128 * 4;
constexpr int kNumBars = 1 + 2 * KST + 2 * VST + 3 * 3 + 1;
constexpr int kSmem = kBarOff + kNumBars * 8 + 16 + 1024;
// warps 0-7 softmax: warp w owns TMEM lanes 32*(w%4).. (rows) and S columns of half w/4;
// warp 8 TMA, warp 9 MMA + TMEM allocation
constexpr int kSoftmaxThreads = 256;
constexpr int kThreads = kSoftmaxThreads + 64;
// 12-warp form: + two idle warps, so warpgroup 2 (TMA, MMA) can hand registers to the softmax
constexpr int kThreads12 = 384;
constexpr int kRegsCtl = 88, kRegsSoftmax = 208;
static_assert(4 * (168 - kRegsCtl) >= 8 * (kRegsSoftmax - 168), "register pool");
constexpr int kSBuf = 3;                // S buffers in TMEM (3 x 128 + O 128 = 512 columns)
constexpr int kOCol = kSBuf * BN;       // O after the S buffers
static_assert(kSmem <= 232448, "shared memory budget");
}  // namespace p2q

// One 64-column half of a row (columns colbase + [0, 64)): masked max of the raw scores.
template <bool DIAG>
__device__ __forceinline__ float row_max_half(const uint32_t (&sv)[2][32], int lim, int colbase) {
  float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
  for (int c = 0; c < 2; ++c)
#pragma unroll
    for (int e = 0; e < 32; e += 2) {
      float v0 = __uint_as_float(sv[c][e]), v1 = __uint_as_float(sv[c][e + 1]);
      if (DIAG) {
        if (colbase + c * 32 + e > lim) v0 = -INFINITY;
        if (colbase + c * 32 + e + 1 > lim) v1 = -INFINITY;
      }
      m4[(e >> 1) & 3] = fmaxf(m4[(e >> 1) & 3], fmaxf(v0, v1));
    }
  return fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
}

// P = hi + lo (both bf16) of 2^(s*sl2 - m) for one 64-column half row.  Layout over the
// half's own S columns: every 16 keys take 16 columns, hi (8 columns) then lo (8 columns),
// so a 32-key chunk is ONE 32-column tcgen05.st; P.V reads hi of keys [16g, 16g+16) at
// column 16g and lo at 16g + 8.  Returns the sum of hi + lo.
// FS: row sums as fp32 FADD2 over the unrounded p (half an instruction per element) instead of
// two FHADD.BF16 (hi and lo parts) per element
template <bool DIAG, bool FS>
__device__ __forceinline__ float exp_pack_hilo_half(const uint32_t (&sv)[2][32], uint32_t p_base,
                                                    int lim, int colbase, float sl2, float m) {
  float2 rsum[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
  const float2 sc2 = make_float2(sl2, sl2), nm2 = make_float2(-m, -m);
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    float p[32];
#pragma unroll
    for (int e = 0; e < 32; e += 2) {
      const float2 x = ffma2(make_float2(__uint_as_float(sv[c][e]), __uint_as_float(sv[c][e + 1])),
                             sc2, nm2);
      p[e] = ex2v(x.x);
      p[e + 1] = ex2v(x.y);
    }
    uint32_t w[32];
#pragma unroll
    for (int e = 0; e < 32; e += 2) {
      float p0 = p[e], p1 = p[e + 1];
      if (DIAG) {
        const int col = colbase + c * 32 + e;
        if (col > lim) p0 = 0.f;
        if (col + 1 > lim) p1 = 0.f;
      }
      const uint32_t wh = pack_bf16x2v(p0, p1);
      const uint32_t wl = pack_bf16x2v(p0 - bf16lo(wh), p1 - bf16hi(wh));
      const int g = e >> 4, k = (e & 15) >> 1;  // 16-key group in the chunk, pair in it
      w[g * 16 + k] = wh;
      w[g * 16 + 8 + k] = wl;
      float2& acc = rsum[(e >> 1) & 1];
      if (FS) {
        acc = fadd2(acc, make_float2(p0, p1));
      } else {
        acc_bf16x2(acc.x, acc.y, wh);
        acc_bf16x2(acc.x, acc.y, wl);
      }
    }
    tmem_st32(p_base + c * 32, w);
  }
  return (rsum[0].x + rsum[0].y) + (rsum[1].x + rsum[1].y);
}

template <bool FS, bool L12 = false>
__global__ void __launch_bounds__(L12 ? p2q::kThreads12 : p2q::kThreads, 1) phase2_qe_kernel(
    const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
    const __grid_constant__ CUtensorMap tm_v, int lq, int hq, int hkv,
    const int32_t* __restrict__ page_table, int pages_per_seq, int page_size,
    const int32_t* __restrict__ kv_len, int own_tail, int64_t chunk, uint2* __restrict__ w_out,
    int64_t part_rows, float scale_log2, float* __restrict__ final_out,
    float* __restrict__ final_lse, uint32_t* __restrict__ grp_epoch, const PeerPush pp) {
  using namespace p2q;
  constexpr int D = 128;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // the generic-pointer derivation is kept here: with smem_align1024 (LDS/STS for the
  // epilogue's staging) K2q measured 1.5% slower (query encode at 128K, l_q = 8 and 32)
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kBarOff);
  uint64_t* q_full = bars;
  uint64_t* k_full = q_full + 1;
  uint64_t* k_empty = k_full + KST;
  uint64_t* v_full = k_empty + KST;
  uint64_t* v_empty = v_full + VST;
  uint64_t* s_full = v_empty + VST;  // [kSBuf]
  uint64_t* p_full = s_full + kSBuf; // [kSBuf]
  uint64_t* o_done = p_full + kSBuf; // [kSBuf]: P.V(j) -> o_done[j % kSBuf] (the rescale)
  uint64_t* o_last = o_done + kSBuf; // the last P.V (the epilogue)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_last + 1);
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  const int split = blockIdx.x, kvh = blockIdx.y, b = blockIdx.z;
  const int G = hq / hkv;
  const int QR = G * lq;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r0 = (int64_t)split * chunk;
  const int32_t* table = page_table + (int64_t)b * pages_per_seq;
  uint2* const w_lse = w_out + (int64_t)gridDim.x * part_rows * D;

  // the Q tile's rows past G*l_q are never loaded: zero them (no garbage in their S rows)
  for (int e = threadIdx.x; e < kTile / 16; e += blockDim.x)
    reinterpret_cast<uint4*>(smem + kQOff)[e] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < KST; ++i) { mbar_init(&k_full[i], 1); mbar_init(&k_empty[i], 1); }
    for (int i = 0; i < VST; ++i) { mbar_init(&v_full[i], 1); mbar_init(&v_empty[i], 1); }
    for (int i = 0; i < kSBuf; ++i) { mbar_init(&s_full[i], 1); mbar_init(&p_full[i], 8); }
    for (int i = 0; i < kSBuf; ++i) mbar_init(&o_done[i], 1);
    mbar_init(o_last, 1);
    fence_mbar_init();
  }
  if (warp == 9) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  // programmatic dependent launch: the setup above overlapped the previous kernel
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // the word-mode epoch of this launch, read ONCE per CTA before any of its words is stored:
  // a CTA advances the group's epoch only after seeing every split's words, so every CTA of
  // the group has read it by then — a later re-read could see the advanced value (round 2:
  // the epilogue and the fold each re-read it, and a slow CTA folded against epoch + 1)
  __shared__ uint32_t es_cta_sh;
  if (threadIdx.x == 0)
    es_cta_sh = (grp_epoch != nullptr && gridDim.x > 1)
                    ? next_epoch(__ldcg(grp_epoch + b * gridDim.y + blockIdx.y)) : 0u;
  __syncthreads();
  const uint32_t es_cta = es_cta_sh;
  const int64_t len = ld_after_wait(kv_len + b);
  const int64_t r1 = min(len, r0 + chunk);
  const int64_t tail0 = len - own_tail;
  const int ntiles = r1 > r0 ? (int)((r1 - r0 + BN - 1) / BN) : 0;

  // pool row of the 64-key half `hh` of tile t (a half past the split end re-reads the
  // tile's first half, whose extra keys the softmax masks)
  auto key_row = [&](int t, int hh) -> int {
    int64_t row = r0 + (int64_t)t * BN + hh * 64;
    if (row >= r1) row = r0 + (int64_t)t * BN;
    const int32_t page = table[row / page_size];
    return (int)(((int64_t)page * hkv + kvh) * page_size + row % page_size);
  };

  auto producer_role = [&]() {
    if (ntiles > 0) {
      // ================= TMA producer: Q once, then K (one tile ahead) and V =================
      // The whole warp resolves page-table entries 32 half-tiles at a time (lane l -> half
      // w0 + l, one coalesced load); lane 0 issues the TMA loads.  K and V keep their own
      // windows (V trails K), so no TMA waits behind a dependent table read.
      if (lane == 0) {
        tma_prefetch(&tm_q);
        tma_prefetch(&tm_k);
        tma_prefetch(&tm_v);
        mbar_expect_tx(q_full, 2 * QR * 128);
        for (int a = 0; a < 2; ++a)
          tma_load_3d(smem + kQOff + a * kSlab, &tm_q, q_full, a * 64, kvh * G, b * lq);
      }
      const int nhalves = 2 * ntiles;
      auto half_row = [&](int h) -> int { return h < nhalves ? key_row(h >> 1, h & 1) : 0; };
      int kw0 = 0, vw0 = 0;
      int kcur = half_row(lane), vcur = kcur;
      int kt = 0, vt = 0;
      while (vt < ntiles) {
        const bool doK = kt < ntiles && kt <= vt + kSBuf;
        const int t = doK ? kt : vt;
        int& w0 = doK ? kw0 : vw0;
        int& cur = doK ? kcur : vcur;
        if (2 * t + 1 >= w0 + 32) {  // slide this window (warp-uniform)
          w0 = 2 * t;
          cur = half_row(w0 + lane);
        }
        const int pr0 = __shfl_sync(0xffffffffu, cur, 2 * t - w0);
        const int pr1 = __shfl_sync(0xffffffffu, cur, 2 * t + 1 - w0);
        if (lane == 0) {
          if (doK) {
            const int st = kt % KST;
            if (kt >= KST) K2Q_WAIT(1, &k_empty[st], ((kt / KST) + 1) & 1);
            mbar_expect_tx(&k_full[st], kTile);
            unsigned char* dst = smem + kKOff + st * kTile;
            for (int a = 0; a < 2; ++a) {
              tma_load_2d(dst + a * kSlab, &tm_k, &k_full[st], a * 64, pr0);
              tma_load_2d(dst + a * kSlab + 64 * 128, &tm_k, &k_full[st], a * 64, pr1);
            }
          } else {
            const int st = vt % VST;
            if (vt >= VST) K2Q_WAIT(2, &v_empty[st], ((vt / VST) + 1) & 1);
            mbar_expect_tx(&v_full[st], kTile);
            unsigned char* dst = smem + kVOff + st * kTile;
            for (int a = 0; a < 2; ++a) {
              tma_load_2d(dst + a * kSlab, &tm_v, &v_full[st], a * 64, pr0);
              tma_load_2d(dst + a * kSlab + 64 * 128, &tm_v, &v_full[st], a * 64, pr1);
            }
          }
        }
        __syncwarp();
        if (doK) ++kt; else ++vt;
      }
    }
  };
  auto mma_role = [&]() {
    // ================= MMA issuer =================
    // S(j) -> buffer j%2.  Order: S(0), S(1), then per tile j: P.V(j) (hi + lo halves of the
    // buffer), S(j+2) into the same buffer (in-order execution: P(j) is consumed first).
    if (ntiles > 0) {  // the whole warp (converged): one elected lane issues each MMA
      constexpr uint32_t idesc_s = umma_idesc_bf16(128, BN, false, false);
      constexpr uint32_t idesc_o = umma_idesc_bf16(128, D, false, true);
      const uint32_t q_addr = smem_u32(smem + kQOff);
      const uint32_t k_addr = smem_u32(smem + kKOff);
      const uint32_t v_addr = smem_u32(smem + kVOff);
      auto issue_s = [&](int t) {
        const int st = t % KST;
        K2Q_WAIT(3, &k_full[st], (t / KST) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * kSlab + (kk & 3) * 32;
          const uint64_t ad = umma_desc_sw128(q_addr + off, 16, 1024);
          const uint64_t bd = umma_desc_sw128(k_addr + st * kTile + off, 16, 1024);
          umma_bf16_ss_warp(tbase + (t % kSBuf) * BN, ad, bd, idesc_s, kk > 0 ? 1u : 0u);
        }
        umma_commit_warp(&s_full[t % kSBuf]);
        // release a stage only if the producer will refill it (commit only what is waited)
        if (t + KST < ntiles) umma_commit_warp(&k_empty[st]);
      };
      K2Q_WAIT(4, q_full, 0);
      for (int t = 0; t < kSBuf && t < ntiles; ++t) issue_s(t);
      for (int j = 0; j < ntiles; ++j) {
        const int vs = j % VST;
        K2Q_WAIT(5, &v_full[vs], (j / VST) & 1);
        K2Q_WAIT(6, &p_full[j % kSBuf], (j / kSBuf) & 1);
        tc_fence_after();
        K2Q_TR(true, j, 5);
        const uint32_t pb = tbase + (j % kSBuf) * BN;
#pragma unroll
        for (int kk = 0; kk < BN / 16; ++kk) {
          const uint64_t bd = umma_desc_sw128(v_addr + vs * kTile + kk * 16 * 128, kSlab, 1024);
#pragma unroll
          for (int h = 0; h < 2; ++h)  // hi at column 16kk, lo at 16kk + 8
            umma_bf16_ts_warp(tbase + kOCol, pb + kk * 16 + h * 8, bd, idesc_o,
                         (j > 0 || h > 0 || kk > 0) ? 1u : 0u);
        }
        K2Q_TR(true, j, 6);
        if (j + 1 < ntiles) {  // waited by a rescale of tile j+1
          // observe the barrier's previous phase (P.V(j - kSBuf), long complete) before arming
          // the next, so every phase is waited once (compute-sanitizer synccheck)
          if (j >= kSBuf) K2Q_WAIT(7, &o_done[j % kSBuf], ((j / kSBuf) - 1) & 1);
          umma_commit_warp(&o_done[j % kSBuf]);
        }
        if (j == ntiles - 1) umma_commit_warp(o_last);
        if (j + VST < ntiles) umma_commit_warp(&v_empty[vs]);
        if (j + kSBuf < ntiles) issue_s(j + kSBuf);
        K2Q_TR(true, j, 7);
      }
      // consume the last phase of every o_done barrier (a rescale waits on them only when
      // the running max jumps): no commit arrival is left unobserved when the CTA exits
      for (int i = 0; i < kSBuf; ++i) {
        const int n_i = ntiles - 1 > i ? (ntiles - 1 - i + kSBuf - 1) / kSBuf : 0;
        if (n_i > 0) K2Q_WAIT(8, &o_done[i], (n_i - 1) & 1);
      }
    }
  };
  auto softmax_role = [&]() {
    // ================= softmax: warps w and w+4 share the rows of TMEM lane quarter w%4,
    // each on one 64-column half of every S row (two warps per SM sub-partition keep its
    // MUFU pipe busy); the halves swap their row maxima through shared memory =================
    const int hf = warp >> 2;                  // column half
    const int r = (warp & 3) * 32 + lane;      // row = TMEM lane
    const int ti = r / G;  // token of this row (rows >= G*l_q are padding)
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t o_tm = tbase + lane_off + kOCol + hf * 64;  // this half's O columns
    float* red = reinterpret_cast<float*>(smem + kRedOff);   // [parity][half][row]
    float* lsum = reinterpret_cast<float*>(smem + kLOff);    // [half][row]
    const float sl2 = scale_log2;
    float m_run = -INFINITY, l_run = 0.f;  // l_run: this half's share of the row sum
    // last visible key of this row relative to the split start (the split end and the row's
    // own-tail causal limit); padding rows (r >= G*l_q) take no mask at all — their values
    // only ever reach their own O lanes, which are discarded — so a warp with padding rows
    // stays on the unmasked path
    const bool pad = r >= QR;
    const int last_rel = pad ? INT_MAX / 2 : (int)(min(r1 - 1, tail0 + ti) - r0);
    for (int j = 0; j < ntiles; ++j) {
      const uint32_t s_tm = tbase + lane_off + (j % kSBuf) * BN;
      K2Q_WAIT(9, &s_full[j % kSBuf], (j / kSBuf) & 1);
      tc_fence_after();
      K2Q_TR(threadIdx.x == 0, j, 0);
      const int64_t base = r0 + (int64_t)j * BN;
      const int lim = max(-1, min(BN, last_rel - j * BN));  // columns c > lim are invisible
      const bool masked = __any_sync(0xffffffffu, lim < hf * 64 + 63);
      uint32_t sv[2][32];
      tmem_ld32(s_tm + hf * 64, sv[0]);
      tmem_ld32(s_tm + hf * 64 + 32, sv[1]);
      tmem_wait_ld_tied(sv[0]);
      tmem_wait_ld_tied(sv[1]);
      const float mh = (masked ? row_max_half<true>(sv, lim, hf * 64)
                               : row_max_half<false>(sv, lim, hf * 64)) * sl2;
      K2Q_TR(threadIdx.x == 0, j, 1);
      red[((j & 1) * 2 + hf) * 128 + r] = mh;
      named_barrier_sync(2, kSoftmaxThreads);
      const float mx = fmaxf(mh, red[((j & 1) * 2 + (hf ^ 1)) * 128 + r]);
      K2Q_TR(threadIdx.x == 0, j, 2);
      float m_use = m_run, alpha = 1.f;
      const bool need = (j == 0) || (mx > m_run + 8.f);
      const bool warp_rescale = (j > 0) && __any_sync(0xffffffffu, need);
      if (need) {
        if (j > 0) alpha = ex2(m_run - mx);
        m_use = mx;
      }
      // rows with no visible key in this split (padding rows, or every key past the row's
      // own-tail limit): a finite m keeps their exp2 arguments finite
      if (pad || last_rel < 0) m_use = 0.f;
      // P of keys [64h, 64h+64) over this half's own S columns [64h, 64h+64)
      const uint32_t p_base = s_tm + hf * 64;
      const float rs = masked ? exp_pack_hilo_half<true, FS>(sv, p_base, lim, hf * 64, sl2, m_use)
                              : exp_pack_hilo_half<false, FS>(sv, p_base, lim, hf * 64, sl2, m_use);
      K2Q_TR(threadIdx.x == 0, j, 3);
      if (r1 - base < BN) {
        // keys past the split end: their V rows may hold stale (even non-finite) data and
        // P = 0 must not meet a NaN — zero them (half h clears V slab h) once the tile landed
        const int valid = (int)(r1 - base);
        K2Q_WAIT(10, &v_full[j % VST], (j / VST) & 1);
        if (r >= valid) {
          uint4* vrow = reinterpret_cast<uint4*>(smem + kVOff + (j % VST) * kTile + hf * kSlab + r * 128);
#pragma unroll
          for (int c = 0; c < 8; ++c) vrow[c] = make_uint4(0, 0, 0, 0);
        }
        fence_proxy_async_smem();
      }
      if (warp_rescale) {
        // O must hold P.V(j-1) before it is rescaled.  Its barrier o_done[(j-1) % kSBuf]
        // completes once per kSBuf tiles: P.V(j-1-kSBuf) is done (S(j) was issued after
        // P.V(j-kSBuf)) and P.V(j-1+kSBuf) cannot be (it needs a later P), so the parity of
        // ((j-1) / kSBuf) is unambiguous
        K2Q_WAIT(11, &o_done[(j - 1) % kSBuf], ((j - 1) / kSBuf) & 1);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < 2; ++c) {
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
      m_run = m_use;
      tc_fence_before();
      __syncwarp();
      K2Q_TR(threadIdx.x == 0, j, 4);
      if (lane == 0) mbar_arrive(&p_full[j % kSBuf]);
    }
    // ---- epilogue: this split's partial of row r (this half's 64 columns) as {value, epoch}
    // words; with one split (no fold) the final partial itself — local, or pushed ----
    lsum[hf * 128 + r] = l_run;
    named_barrier_sync(2, kSoftmaxThreads);
    const float l_row = l_run + lsum[(hf ^ 1) * 128 + r];
    const bool single = gridDim.x == 1;
    const uint32_t es = single ? 0u : es_cta;
    const uint32_t ep = (single && pp.L.world > 0) ? exchange_epoch(pp) : 0u;
    if (ntiles > 0) {
      // (not o_done's parity: P.V(ntiles-2) may still be in flight here, two phases behind)
      K2Q_WAIT(12, o_last, 0);
      tc_fence_after();
    }
    const bool row_ok = r < QR;
    const int64_t orow = ((int64_t)b * lq + ti) * hq + kvh * G + r % G;
    const float inv = l_row > 0.f ? 1.f / l_row : 0.f;
    uint2* wo = w_out + (int64_t)split * part_rows * D + orow * D + hf * 64;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      uint32_t orr[32];
      if (ntiles > 0) {
        tmem_ld32(o_tm + c * 32, orr);
        tmem_wait_ld();
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) orr[e] = 0u;
      }
      if (row_ok) {
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          const float2 v2 =
              make_float2(__uint_as_float(orr[e]) * inv, __uint_as_float(orr[e + 1]) * inv);
          if (single)
            put_out2(pp, ep, false, final_out, orow * D + hf * 64 + c * 32 + e, v2);
          else
            st_word2(wo + c * 32 + e, v2, es);
        }
      }
    }
    if (row_ok && hf == 0) {
      const float lv = l_row > 0.f ? (m_run + __log2f(l_row)) * 0.6931471805599453f : -INFINITY;
      if (single)
        put_lse(pp, ep, false, final_lse, orow, lv);
      else
        st_word(w_lse + (int64_t)split * part_rows + orow, lv, es);
    }
    tc_fence_before();
    if (gridDim.x > 1) {
      // word-mode fold of the splits (+ the peer exchange push / merge when asked); it reads
      // only global words, so it runs before the CTA-wide barrier that precedes the TMEM free
      // grouped loads once every thread has >= 4 elements of the slice (l_q = 32 at G = 4:
      // 1,024 per CTA); smaller slices keep one element per thread (more threads polling)
      if (QR * D >= 4 * kSoftmaxThreads * (int)gridDim.x)
        split_merge_words_call<D, kSoftmaxThreads, 4>(b, kvh, 0, QR, lq, hq, G, w_out, w_lse, part_rows,
                                                 es_cta, final_out, final_lse, grp_epoch, pp);
      else
        split_merge_words_call<D, kSoftmaxThreads, 1>(b, kvh, 0, QR, lq, hq, G, w_out, w_lse, part_rows,
                                                 es_cta, final_out, final_lse, grp_epoch, pp);
    }
  };
  if (L12) {
    // 12 warps: warpgroup 2 (TMA, MMA, two idle warps) gives registers to the softmax
    // warpgroups (setmaxnreg inside warpgroup-uniform branches, as K1)
    const int wg = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 7), 0);
    if (wg == 2) {
      regs_dealloc<kRegsCtl>();
      if (warp == 8)
        producer_role();
      else if (warp == 9)
        mma_role();
    } else {
      regs_alloc<kRegsSoftmax>();
      softmax_role();
    }
  } else {
    if (warp == 8)
      producer_role();
    else if (warp == 9)
      mma_role();
    else
      softmax_role();
  }
  __syncthreads();
  if (warp == 9) tmem_free<512>(tbase);
}

// ------------------------------------------------------------------ host
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder();

// K2 / K2q are launched as programmatic dependents of the kernel before them (their setup
// overlaps it; griddepcontrol.wait precedes every read of its outputs).  STAR_K2_PDL=0 turns
// it off (measurement).
static bool k2_pdl() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("STAR_K2_PDL");
    on = (e != nullptr && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

// STAR_K2_COOP=0 launches the word-mode grid without the cooperative attribute (measurement
// only: co-residency then rests on an otherwise idle GPU)
static bool k2_coop() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("STAR_K2_COOP");
    on = (e != nullptr && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

// K2q (tcgen05 query encode) takes 16 < G*l_q <= 128 packed rows at head_dim 128 over a pool
// of 64-key-aligned pages; STAR_K2_QE=0 turns it off (measurement)
bool phase2_qe_eligible(int qrows, int d, int page_size) {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("STAR_K2_QE");
    on = (e != nullptr && e[0] == '0') ? 0 : 1;
  }
  return on && d == 128 && qrows > 16 && qrows <= 128 && page_size % 64 == 0;
}

int phase2_mma(const void* q, int batch, int lq, int hq, int hkv, int d, const void* kp,
               const void* vp, int64_t num_pages, const int32_t* table, int pps, int page_size,
               const int32_t* kv_len, int own_tail, int64_t chunk, int n_splits, float* out,
               float* lse, float* final_out, float* final_lse, int* counters, PeerPush pp,
               int* merged, cudaStream_t s, const DecodeAppend* dap) {
  using namespace p2;
  if (merged != nullptr) *merged = 0;
  DecodeAppend ap{};
  if (dap != nullptr && dap->on) {
    ap = *dap;
    ap.kp = const_cast<void*>(kp);
    ap.vp = const_cast<void*>(vp);
    if (lq != 1 || (hq / hkv) > 16 || (d != 64 && d != 128))
      return fail(STAR_ENOTSUP, "fused decode append: lq must be 1 and G <= 16 (got lq=%d G=%d)", lq,
                  hq / hkv);
  }
  pp.timeout_ns = spin_timeout_ns();
  auto fn = tensor_map_encoder();
  if (fn == nullptr) return fail(STAR_ECUDA, "cuTensorMapEncodeTiled unavailable");
  if (page_size % TN) return fail(STAR_ECONFIG, "page_size must be a multiple of %d", TN);
  int64_t rows = num_pages * hkv * page_size;
  if (rows >= (1ll << 31)) return fail(STAR_ENOTSUP, "KV pool larger than 2^31 rows");
  CUtensorMap tk, tv;
  cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)rows};
  cuuint64_t str[1] = {(cuuint64_t)d * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)TN};
  cuuint32_t estr[2] = {1, 1};
  if (fn(&tk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(kp), dims, str, box, estr,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS ||
      fn(&tv, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(vp), dims, str, box, estr,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return fail(STAR_ECUDA, "phase2: tensor map encode failed");
  const int QR = (hq / hkv) * lq;
  const int stage_bytes = STAGES * (d == 128 ? Smem<128>::kStage : Smem<64>::kStage);
  if (n_splits > 1 && (int64_t)n_splits * QR * 4 + QR * 4 + 16 > stage_bytes)
    return fail(STAR_ECONFIG, "phase2: %d splits x %d query rows exceed the fix-up buffer", n_splits,
                QR);
  int n_rb = QR <= 16 ? 1 : (QR + 63) / 64;  // row blocks (see the kernel)
  dim3 grid(n_splits, hkv * n_rb, batch);
  // split fix-up: word mode (every split CTA polls the others' {value, epoch} words and
  // folds a slice of the group) when the whole grid is co-resident, so no spinning CTA can
  // starve one that has not started; else the arrival-counter fix-up.  STAR_K2_FIXUP=atomic forces the latter (measurement).
  static const bool force_atomic = getenv("STAR_K2_FIXUP") != nullptr && getenv("STAR_K2_FIXUP")[0] == 'a';
  uint32_t* grp_epoch = nullptr;
  // the tcgen05 query-encode kernel (K2q) for 16 < G*l_q <= 128 packed rows; it needs the
  // word-mode fix-up (co-resident grid), else the mma.sync row blocks run
  bool use_qe = false;
  if (counters != nullptr && n_splits > 1 && !force_atomic) {
    if (!ap.on && phase2_qe_eligible(QR, d, page_size) && (int64_t)n_splits * batch * hkv <= num_sms()) {
      use_qe = true;
      n_rb = 1;
      grid = dim3(n_splits, hkv, batch);
      grp_epoch = reinterpret_cast<uint32_t*>(counters) + kEpochOffsetWords;
    } else if ((int64_t)n_splits * batch * hkv * n_rb <= num_sms()) {  // 1 CTA / SM
      grp_epoch = reinterpret_cast<uint32_t*>(counters) + kEpochOffsetWords;
    }
  } else if (n_splits == 1 && !ap.on && phase2_qe_eligible(QR, d, page_size)) {
    // one split per (sequence, kv head): K2q writes the final partial, no fold (any grid)
    use_qe = true;
    n_rb = 1;
    grid = dim3(1, hkv, batch);
  }
  const float sl2 = (float)(1.4426950408889634 / sqrt((double)d));
  const int64_t part_rows = (int64_t)batch * lq * hq;
  // the in-kernel cross-rank merge needs the co-resident word-mode grid
  if (pp.merge && (grp_epoch == nullptr || pp.L.world == 0)) pp.merge = 0;
  if (merged != nullptr) *merged = pp.merge;
  bool reset_now = false;
  if (n_splits > 1 && counters != nullptr) {
    // A word's slot position depends on (batch, lq, hq, hkv, d) and word-mode epochs count
    // per (sequence, kv head): a workspace reused with another shape (or after the
    // arrival-counter mode wrote floats there) could hold stale words whose epoch equals
    // the new one.  Zero the header and this launch's partials whenever the workspace's
    // shape or mode changes (stream-ordered; once per change, e.g. query encode -> decode).
    static std::mutex mu;
    static std::unordered_map<const void*, std::array<int64_t, 7>> last;
    // n_splits is part of the signature: it moves the lse words and widens the zeroed range
    const std::array<int64_t, 7> sig = {batch, lq, hq, hkv, d, n_splits,
                                        (grp_epoch != nullptr ? 1 : 0) + (use_qe ? 2 : 0)};
    std::lock_guard<std::mutex> lock(mu);
    auto it = last.find(counters);
    if (it == last.end() || it->second != sig) {
      const size_t bytes = (size_t)16384 + (size_t)n_splits * part_rows * (d + 1) * 8;
      cudaError_t e = cudaMemsetAsync(counters, 0, bytes, s);
      if (e != cudaSuccess) return fail(STAR_ECUDA, "phase2 workspace reset: %s", cudaGetErrorString(e));
      last[counters] = sig;
      // a programmatic-dependent launch is not ordered after this memset (measured: with the
      // workspace address reused by another shape, the zeroing landed while the kernel's words
      // were in flight and the fold never completed) — this launch goes without PDL
      reset_now = true;
    }
  }
  if (use_qe) {
    // Q as [batch*lq rows][hq][d]: one box {64, G, lq} per 64-column slab = the packed tile
    CUtensorMap tq;
    const int G = hq / hkv;
    cuuint64_t qdims[3] = {(cuuint64_t)d, (cuuint64_t)hq, (cuuint64_t)batch * lq};
    cuuint64_t qstr[2] = {(cuuint64_t)d * 2, (cuuint64_t)hq * d * 2};
    cuuint32_t qbox[3] = {64, (cuuint32_t)G, (cuuint32_t)lq};
    cuuint32_t qestr[3] = {1, 1, 1};
    if (fn(&tq, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(q), qdims, qstr, qbox,
           qestr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return fail(STAR_ECUDA, "phase2 query encode: Q tensor map encode failed");
    static int fs = -1;  // STAR_K2Q_SUM=0: the round-1 FHADD.BF16 row sums (measurement knob)
    if (fs < 0) {
      const char* ev = getenv("STAR_K2Q_SUM");
      fs = (ev != nullptr && ev[0] == '0') ? 0 : 1;
    }
    static int l12 = -1;  // STAR_K2Q_L12=0: the 10-warp form (measurement knob)
    if (l12 < 0) {
      const char* ev = getenv("STAR_K2Q_L12");
      l12 = (ev != nullptr && ev[0] == '0') ? 0 : 1;
    }
    auto qek = fs ? (l12 ? phase2_qe_kernel<true, true> : phase2_qe_kernel<true, false>)
                  : (l12 ? phase2_qe_kernel<false, true> : phase2_qe_kernel<false, false>);
    cudaError_t e = cudaFuncSetAttribute(qek,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, p2q::kSmem);
    if (e != cudaSuccess) return fail(STAR_ECUDA, "phase2 qe smem attr: %s", cudaGetErrorString(e));
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (grp_epoch != nullptr && k2_coop()) {  // cooperative only for the word-mode fold
      attr[na].id = cudaLaunchAttributeCooperative;
      attr[na++].val.cooperative = 1;
    }
    if (k2_pdl() && !reset_now) {
      attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[na++].val.programmaticStreamSerializationAllowed = 1;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(l12 ? p2q::kThreads12 : p2q::kThreads);
    cfg.dynamicSmemBytes = p2q::kSmem;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = na;
    e = cudaLaunchKernelEx(&cfg, qek, tq, tk, tv, lq, hq, hkv, table, pps, page_size,
                           kv_len, own_tail, chunk, reinterpret_cast<uint2*>(out), part_rows, sl2,
                           final_out, final_lse, grp_epoch, pp);
    if (e != cudaSuccess) return fail(STAR_ECUDA, "phase2 qe launch: %s", cudaGetErrorString(e));
    return STAR_OK;
  }
  const bool keysplit = QR <= 16;
  // Word mode spins on other CTAs of the grid, so it is launched COOPERATIVELY: the driver
  // guarantees every CTA co-resident (also against kernels on other streams), and refuses the
  // launch instead of deadlocking if the grid cannot fit.
#define STAR_P2M_ST(DD, KS, SST)                                                                \
  do {                                                                                          \
    auto kern = phase2_mma_kernel<DD, KS, SST>;                                                 \
    const int bytes = Smem<DD, SST>::kBytes;                                                    \
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes); \
    if (e != cudaSuccess) return fail(STAR_ECUDA, "phase2 smem attr: %s", cudaGetErrorString(e)); \
    cudaLaunchAttribute attr[2];                                                                \
    int na = 0;                                                                                 \
    if (grp_epoch != nullptr && k2_coop()) {                                                    \
      attr[na].id = cudaLaunchAttributeCooperative;                                             \
      attr[na++].val.cooperative = 1;                                                           \
    }                                                                                           \
    if (k2_pdl() && !reset_now) {                                                                             \
      attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;                         \
      attr[na++].val.programmaticStreamSerializationAllowed = 1;                                \
    }                                                                                           \
    cudaLaunchConfig_t cfg = {};                                                                \
    cfg.gridDim = grid;                                                                         \
    cfg.blockDim = dim3(Cons<KS>::kThreads);                                                    \
    cfg.dynamicSmemBytes = bytes;                                                               \
    cfg.stream = s;                                                                             \
    cfg.attrs = attr;                                                                           \
    cfg.numAttrs = na;                                                                          \
    e = cudaLaunchKernelEx(&cfg, kern, tk, tv, (const __nv_bfloat16*)q, lq, hq, hkv, table, pps, \
                           page_size, kv_len, own_tail, chunk, out, lse, part_rows, sl2,        \
                           final_out, final_lse, counters, grp_epoch, pp, ap);                  \
    if (e != cudaSuccess) return fail(STAR_ECUDA, "phase2 launch: %s", cudaGetErrorString(e));  \
  } while (0)
#define STAR_P2M(DD, KS) STAR_P2M_ST(DD, KS, STAGES)
  if (d == 128) {
    if (keysplit) STAR_P2M(128, true); else STAR_P2M(128, false);
  } else if (d == 64) {
    if (keysplit) STAR_P2M(64, true); else STAR_P2M(64, false);
  } else {
    return fail(STAR_ENOTSUP, "phase2 bf16 path needs head_dim 64 or 128");
  }
#undef STAR_P2M
#undef STAR_P2M_ST
  STAR_LAUNCH_CHECK("phase2_mma");
  return STAR_OK;
}

#ifdef STAR_K1_TRACE
int debug_k2q_trace(long long* host, int n) {
  const int cap = 256 * 8;
  if (n > cap) n = cap;
  return cudaMemcpyFromSymbol(host, g_k2q_trace, n * sizeof(long long)) == cudaSuccess ? n : -4;
}
int debug_k2_trace(unsigned long long* host, int n) {
  const int cap = kK2TrCtas * kK2TrSlots;
  if (n > cap) n = cap;
  return cudaMemcpyFromSymbol(host, g_k2_trace, n * sizeof(unsigned long long)) == cudaSuccess ? n : -4;
}
#endif

}  // namespace star

#ifdef STAR_K1_TRACE
extern "C" int star_debug_k2_trace(unsigned long long* host, int n) {
  return star::debug_k2_trace(host, n);
}
#endif

#ifdef STAR_K1_TRACE
extern "C" int star_debug_k2q_trace(long long* host, int n) { return star::debug_k2q_trace(host, n); }
#endif
