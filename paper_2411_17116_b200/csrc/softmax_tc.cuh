// Per-row softmax building blocks over a 128-column S row in TMEM (one thread per row =
// TMEM lane), shared by the tcgen05 kernels: K1 (phase1_tc.cu) and the phase-2 query
// encode (phase2_mma.cu).  Masking (DIAG): columns c > lim are invisible.
#pragma once

#include "common.cuh"
#include "sm100.cuh"

namespace star {

using namespace sm100;


// 2^x for a pair on the FMA pipe (offloads the MUFU/XU pipe): x clamped to >= -125,
// x = n + f with n = round(x) (magic-number rounding), 2^f by a degree-3 minimax
// polynomial on [-1/2, 1/2] (max rel. error 2.1e-4, below bf16's 2^-9 rounding of P),
// then n is added to the exponent field with one IMAD.
__device__ __forceinline__ float2 poly_ex2x2(float2 x) {
  constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23
  x.x = fmaxf(x.x, -125.f);
  x.y = fmaxf(x.y, -125.f);
  const float2 t = fadd2(x, make_float2(kMagic, kMagic));
  const float2 r = fadd2(t, make_float2(-kMagic, -kMagic));
  const float2 f = fadd2(x, make_float2(-r.x, -r.y));
  float2 p = ffma2(f, make_float2(0.05484800413f, 0.05484800413f),
                   make_float2(0.24180661142f, 0.24180661142f));
  p = ffma2(p, f, make_float2(0.69324821234f, 0.69324821234f));
  p = ffma2(p, f, make_float2(0.99998867512f, 0.99998867512f));
  return make_float2(__int_as_float(__float_as_int(t.x) * 8388608 + __float_as_int(p.x)),
                     __int_as_float(__float_as_int(t.y) * 8388608 + __float_as_int(p.y)));
}

// volatile forms: the compiler keeps their relative (source) order, which here is the
// latency-hiding schedule (exponentials first, packs after)
__device__ __forceinline__ float ex2v(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack_bf16x2v(float lo, float hi) {
  uint32_t r;
  asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

// f32 += bf16 (one FHADD.BF16 per element, no unpack): the exact fp32 value of the
// bf16-rounded p joins the row sum.
__device__ __forceinline__ void acc_bf16x2(float& lo_acc, float& hi_acc, uint32_t w) {
  asm("{\n\t.reg .b16 lo, hi;\n\tmov.b32 {lo, hi}, %2;\n\t"
      "add.rn.f32.bf16 %0, lo, %0;\n\tadd.rn.f32.bf16 %1, hi, %1;\n\t}"
      : "+f"(lo_acc), "+f"(hi_acc)
      : "r"(w));
}

// One-pass softmax: the whole 128-column S row is loaded into registers once (four
// tcgen05.ld in flight together, one wait), reduced to its max, then exponentiated in
// place — no second TMEM read and a single exposed load latency per tile.
__device__ __forceinline__ void tmem_ld_row128(uint32_t s_tm, uint32_t (&sv)[4][32]) {
  tmem_ld32(s_tm, sv[0]);
  tmem_ld32(s_tm + 32, sv[1]);
  tmem_ld32(s_tm + 64, sv[2]);
  tmem_ld32(s_tm + 96, sv[3]);
  tmem_wait_ld_tied(sv[0]);
  tmem_wait_ld_tied(sv[1]);
  tmem_wait_ld_tied(sv[2]);
  tmem_wait_ld_tied(sv[3]);
}

template <bool DIAG>
__device__ __forceinline__ float row_max_regs(const uint32_t (&sv)[4][32], int lim) {
  float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
  for (int c = 0; c < 4; ++c)
#pragma unroll
    for (int e = 0; e < 32; e += 2) {
      float v0 = __uint_as_float(sv[c][e]), v1 = __uint_as_float(sv[c][e + 1]);
      if (DIAG) {
        if (c * 32 + e > lim) v0 = -INFINITY;
        if (c * 32 + e + 1 > lim) v1 = -INFINITY;
      }
      m4[(e >> 1) & 3] = fmaxf(m4[(e >> 1) & 3], fmaxf(v0, v1));
    }
  return fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
}

// Row-sum forms (SUM): 0 = fp32 FADD2 over the unpacked bf16-rounded p, 1 = f32 += bf16
// (FHADD.BF16, one per element), 2 = fp32 FADD2 over the unrounded p (half the instructions
// of 1; the bf16 quantisation of P then only enters the numerator, which measured the same
// error against the fp64 oracle, tests/test_tolerance.py).
// POLY (> 0): every POLY-th exponential pair runs on the FMA pipe (poly_ex2x2), spread
// evenly through the row so the FMA work fills the single warp's MUFU issue gaps.
// SPLIT: once the P of keys [0, 64) is stored, mid() runs (the caller hands that half over,
// so the P.V of those keys overlaps the exponentials of the rest); chunks 0-1 of S are dead
// by then, which leaves registers for whatever mid() needs.
struct NoMid {
  __device__ __forceinline__ void operator()() const {}
};
template <bool DIAG, int POLY, int SUM, bool SPLIT = false, class Mid = NoMid>
__device__ __forceinline__ float exp_pack_regs(const uint32_t (&sv)[4][32], uint32_t s_tm, int lim,
                                               float sl2, float m, const Mid& mid = Mid()) {
  float2 rsum[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
  const float2 sc2 = make_float2(sl2, sl2), nm2 = make_float2(-m, -m);
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    // all 32 exponentials of the chunk are issued back to back before any result is
    // consumed, so the MUFU pipe never idles behind its own latency (in-order issue)
    float p[32];
#pragma unroll
    for (int e = 0; e < 32; e += 2) {
      const float2 x = ffma2(make_float2(__uint_as_float(sv[c][e]), __uint_as_float(sv[c][e + 1])),
                             sc2, nm2);
      if (POLY > 0 && ((c * 16 + (e >> 1)) % (POLY > 0 ? POLY : 1)) == (POLY > 0 ? POLY - 1 : 0)) {
        const float2 q = poly_ex2x2(x);
        p[e] = q.x;
        p[e + 1] = q.y;
      } else {
        p[e] = ex2v(x.x);
        p[e + 1] = ex2v(x.y);
      }
    }
    uint32_t pk[16];
#pragma unroll
    for (int e = 0; e < 32; e += 2) {
      float p0 = p[e], p1 = p[e + 1];
      if (DIAG) {
        const int col = c * 32 + e;
        if (col > lim) p0 = 0.f;
        if (col + 1 > lim) p1 = 0.f;
      }
      const uint32_t w = pack_bf16x2v(p0, p1);
      pk[e >> 1] = w;
      float2& acc = rsum[(e >> 1) & 1];
      if (SUM == 1)
        acc_bf16x2(acc.x, acc.y, w);
      else if (SUM == 2)
        acc = fadd2(acc, make_float2(p0, p1));
      else
        acc = fadd2(acc, make_float2(bf16lo(w), bf16hi(w)));
    }
    tmem_st16(s_tm + c * 16, pk);
    if (SPLIT && c == 1) mid();
  }
  return (rsum[0].x + rsum[0].y) + (rsum[1].x + rsum[1].y);
}

}  // namespace star
