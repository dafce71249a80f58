// Peer exchange of phase-2 partials over NVLink peer memory (the fused form of C1).
//
// The reference gathers every host's (out, lse) partial to the query host and merges
// them in ascending host order (ss/sim.py:178-213, merge_partials ss/attention.py:154-173).
// Here every rank owns a "box" in its HBM, mapped into every other rank's address space
// (CUDA IPC).  The K2 epilogue that produces a (sequence, kv head) group's final partial
// stores it straight into slot `rank` of EVERY rank's box, and K3x (exchange_merge_kernel)
// on each rank merges the slots in ascending rank order.  No NCCL kernel, no staging copy:
// the transfer is the K2 epilogue's own stores.
//
// Low-latency word protocol (no fences, no flags): every 4-byte value travels in an 8-byte
// word {value, epoch} written with one vector store, which is single-copy atomic, so a
// reader that sees the current epoch in a word also sees its value.  A release/acquire flag
// protocol needs a system-scope fence per producer (MEMBAR.SYS), measured at ~1-3 us and
// serialising across SMs (tools/ubench/fence.cu, tools/exchange_bench.py); the words cost
// twice the bytes of a 16.5 KB partial instead, i.e. nothing on NVLink.
//
// Epochs live on the device: box header word 0 counts the exchanges this rank has
// completed (c); the exchange in flight is epoch e = c + 1 (a zeroed box holds epoch 0
// everywhere, so it is ready).  K2 / the push kernel read c from the rank's OWN box; the
// last CTA of K3x stores c + 1 after every CTA has read c.  Every rank runs the same
// sequence of exchanges, so the counters stay in step without host involvement — and a
// captured CUDA graph of a decode step replays correctly (no epoch in kernel parameters).
//
// Box layout (identical on every rank; parity p = e & 1 double-buffers the slots, so a rank
// that runs ahead to the next layer never overwrites a slot a slower rank still reads:
// writing parity p again requires every rank to have finished the merge of epoch e - 1):
//   u32 header[64]        [0] completed exchanges, [1] K3x CTA arrivals
//   u2  slots[2][world][part]   part = round_up(rows * d + rows, 2) words {value, epoch}
//       slot = [rows * d out words | rows lse words]
// rows is the box's CAPACITY (fixed for its lifetime, so calls of different shapes, e.g. a
// 32-row query encode followed by 1-row decodes, never move a slot under a rank that still
// reads the previous epoch); a call uses slot rows row = (b * lq + i) * hq + h <
// batch * lq * hq <= rows.  `groups` (batch * hkv capacity) bounds the callers' grids.
#pragma once

#include <stdint.h>

namespace star {

constexpr int kMaxPeers = 8;  // one NVSwitch node
// K2 workspace header: 2048 int32 arrival counters, then 2048 uint32 word-mode epochs
constexpr int kEpochOffsetWords = 2048;

struct ExchangeLayout {
  int world;
  int64_t rows;    // capacity: query rows (batch * lq * hq) per slot
  int d;
  int groups;      // capacity: (sequence, kv head) groups (batch * hkv)
  static constexpr int64_t kHeader = 256;
  __host__ __device__ int64_t part() const { return (rows * (d + 1) + 1) / 2 * 2; }  // words
  __host__ __device__ int64_t bytes() const { return kHeader + (int64_t)2 * world * part() * 8; }
  __host__ __device__ uint32_t* header(void* box) const { return static_cast<uint32_t*>(box); }
  __host__ __device__ uint2* slot(void* box, int parity, int src) const {
    return reinterpret_cast<uint2*>(static_cast<char*>(box) + kHeader) +
           ((int64_t)parity * world + src) * part();
  }
};

// What a producer kernel needs to deliver its final partial to every rank: the boxes of all
// ranks (box[rank] = its own, whose header holds the epoch) and the layout.
// L.world == 0: no exchange (write the local out / lse as usual).
struct PeerPush {
  void* box[kMaxPeers];
  ExchangeLayout L;
  int rank;
  // 1: the producer also merges every rank's partial of its slice (the whole exchange in
  // one kernel; only for a co-resident grid, see split_merge_words); 0: K3x merges
  int merge;
  // spin-wait bound of the word protocols (split fold and peer merge) before __trap: a
  // missing producer fails loudly instead of hanging the stream (STAR_EXCHANGE_TIMEOUT_S,
  // default 30 s; raise it under compute-sanitizer, which slows every CTA down)
  uint64_t timeout_ns;
};

// Fused decode append for K2 (lq = 1, bf16): instead of a separate star_kv_append launch,
// every K2 CTA rotates its q heads itself (RoPE at pos[b], cos/sin from the decode-position
// table) and the CTA whose key range holds row kv_len[b] writes the new row's rotated k and
// raw v into the paged cache right before its TMA reads that tile; K2 then attends over
// kv_len[b] + add rows.  The row counter is NOT advanced here (every CTA reads it): the
// decode step advances all layers' counters once per token (star_decode_advance).
// on == 0: plain K2 (q already rotated, no append).
struct DecodeAppend {
  const void* q_raw;    // [batch][hq][d] pre-RoPE (row stride q_rs elements)
  const void* k_new;    // [batch][hkv][d] pre-RoPE
  const void* v_new;    // [batch][hkv][d]
  int64_t q_rs, kv_rs;
  const int64_t* pos;   // [batch] positions of the new rows
  const void* rtab;     // double2 cos/sin table of positions [rtab_pos0, rtab_pos0 + rtab_n), or null
  const void* cur_cs;   // double2 [batch][d/2] cos/sin at pos[b] (star_decode_advance keeps it
                        // current), or null: read first, no dependent position load
  int64_t rtab_pos0, rtab_n;
  double theta;
  void* kp;             // the K / V pools K2 streams (the new row is written there)
  void* vp;
  int on;               // rotate q from q_raw
  int add;              // 1: append the row (write it, attend over kv_len + 1); 0: q only
};

// STAR_EXCHANGE_TIMEOUT_S (seconds, default 30), read once per process
uint64_t spin_timeout_ns();

__device__ __forceinline__ void st_word(uint2* p, float v, uint32_t e) {
  asm volatile("st.volatile.global.v2.u32 [%0], {%1, %2};" ::"l"(p), "r"(__float_as_uint(v)),
               "r"(e)
               : "memory");
}
__device__ __forceinline__ void st_word2(uint2* p, float2 v, uint32_t e) {  // p 16 B aligned
  asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p),
               "r"(__float_as_uint(v.x)), "r"(e), "r"(__float_as_uint(v.y)), "r"(e)
               : "memory");
}
__device__ __forceinline__ uint2 ld_word(const uint2* p) {
  uint2 w;
  asm volatile("ld.volatile.global.v2.u32 {%0, %1}, [%2];" : "=r"(w.x), "=r"(w.y) : "l"(p) : "memory");
  return w;
}
// two {value, epoch} words (16 bytes, p 16-byte aligned); each word's epoch is checked on its own
__device__ __forceinline__ uint4 ld_word4(const uint2* p) {
  uint4 w;
  asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w)
               : "l"(p)
               : "memory");
  return w;
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// epoch of the exchange in flight (completed exchanges of this rank + 1; kernel-boundary
// ordered after the previous K3x, which advanced the counter)
// Successor of an epoch counter: 0 (the value of a zeroed word) is never used, and the
// parity still alternates across the 32-bit wrap (0xFFFFFFFF -> 2).
__device__ __forceinline__ uint32_t next_epoch(uint32_t c) {
  const uint32_t e = c + 1u;
  return e == 0u ? 2u : e;
}
__device__ __forceinline__ uint32_t exchange_epoch(const PeerPush& pp) {
  return next_epoch(__ldcg(pp.L.header(pp.box[pp.rank])));
}

// final partial element stores: the local arrays (local_only, e.g. a split partial that the
// fix-up still folds, or no exchange), else this rank's slot (epoch e) in every box
__device__ __forceinline__ void put_out(const PeerPush& pp, uint32_t e, bool local_only,
                                        float* local, int64_t i, float v) {
  if (local_only || pp.L.world == 0) {
    local[i] = v;
    return;
  }
#pragma unroll
  for (int r = 0; r < kMaxPeers; ++r)
    if (r < pp.L.world) st_word(pp.L.slot(pp.box[r], e & 1u, pp.rank) + i, v, e);
}
__device__ __forceinline__ void put_out2(const PeerPush& pp, uint32_t e, bool local_only,
                                         float* local, int64_t i, float2 v) {  // i even
  if (local_only || pp.L.world == 0) {
    *reinterpret_cast<float2*>(local + i) = v;
    return;
  }
#pragma unroll
  for (int r = 0; r < kMaxPeers; ++r)
    if (r < pp.L.world) st_word2(pp.L.slot(pp.box[r], e & 1u, pp.rank) + i, v, e);
}
__device__ __forceinline__ void put_lse(const PeerPush& pp, uint32_t e, bool local_only,
                                        float* local, int64_t i, float v) {
  if (local_only || pp.L.world == 0) {
    local[i] = v;
    return;
  }
#pragma unroll
  for (int r = 0; r < kMaxPeers; ++r)
    if (r < pp.L.world)
      st_word(pp.L.slot(pp.box[r], e & 1u, pp.rank) + pp.L.rows * pp.L.d + i, v, e);
}

}  // namespace star
