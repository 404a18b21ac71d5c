// gat_common.cuh — device pieces shared by the sparse GAT kernels (gat.cu, gat2.cu): the work-item
// decoding of the segment plan, light-row tiles, the packed int8 -> fp32 conversion + FMA, IDP4A dots,
// the cp.async row-slice copies and the transposed 4-edge dot reduction.
#pragma once
#include "rowops.cuh"

namespace tango {

constexpr int WPB = 8;      // warps per block of the row kernels
constexpr int UNR = 8;      // gather pipeline depth (edges in flight per warp)

// ------------------------------------------------------------------ shared device pieces
struct Seg {
  int64_t vl, eb, ee;   // local row, edge range
  int slot;             // heavy segment slot (-1 for a whole light row)
  int c, base, nseg;    // chunk index, first slot and segment count of a heavy row
};

// Decode work item `item` of the space [0, hcount) heavy segments  U  [hcount, hcount + n) rows
// (the long heavy segments are handed out first).  Returns false for a row item that belongs to a
// heavy row (skipped).
__device__ __forceinline__ bool decode_item(int64_t item, int64_t hcount, const int64_t* ptr, const PlanDev& p,
                                            int chunk, Seg& s) {
  if (item >= hcount) {
    const int64_t r = item - hcount;
    s.vl = r;
    if (p.hbase[r] >= 0) return false;
    s.eb = ptr[r]; s.ee = ptr[r + 1]; s.slot = -1; s.c = 0; s.base = -1; s.nseg = 1;
    return true;
  }
  s.slot = (int)item;
  s.vl = p.hseg_row[s.slot];
  s.base = p.hbase[s.vl];
  s.c = s.slot - s.base;
  const int64_t beg = ptr[s.vl], end = ptr[s.vl + 1];
  s.nseg = (int)((end - beg + chunk - 1) / chunk);
  s.eb = beg + (int64_t)s.c * chunk;
  s.ee = min(end, s.eb + chunk);
  return true;
}
__device__ __forceinline__ int64_t load_count(const int32_t* c) { return (int64_t)*(volatile const int32_t*)c; }

// Dynamic work queue: lane 0 claims the next item index, broadcast to the warp.
__device__ __forceinline__ int64_t claim(int32_t* counter) {
  int it = 0;
  if ((threadIdx.x & 31) == 0) it = atomicAdd(counter, 1);
  return (int64_t)__shfl_sync(0xffffffffu, it, 0);
}
#define FOR_ITEMS(item, counter, nitems) for (int64_t item = claim(counter); item < (nitems); item = claim(counter))
#define FOR_ITEMS_FROM(item, counter, start, nitems) \
  for (int64_t item = (start) + claim(counter); item < (nitems); item = (start) + claim(counter))
// Batched claims for work queues of many small, uniform items (the v6 scalar passes: ~400 K hub segments
// per pass on Reddit-shaped graphs, where a per-item claim serialises on the counter's address): one
// same-address atomic per CLAIM_BATCH items.  Queues whose consecutive items belong to one hub row (the
// gather passes, the round-1 kernels) keep per-item claims so that a row's chunks spread over warps.
constexpr int CLAIM_BATCH = 4;
__device__ __forceinline__ int64_t claim_batch(int32_t* counter) {
  int it = 0;
  if ((threadIdx.x & 31) == 0) it = atomicAdd(counter, CLAIM_BATCH);
  return (int64_t)__shfl_sync(0xffffffffu, it, 0);
}
#define FOR_ITEMS4(item, counter, nitems)                                                                  \
  for (int64_t item##_b = claim_batch(counter); item##_b < (nitems); item##_b = claim_batch(counter))     \
    for (int64_t item = item##_b, item##_e = item##_b + CLAIM_BATCH < (int64_t)(nitems) ? item##_b + CLAIM_BATCH \
                                                                                      : (int64_t)(nitems); \
         item < item##_e; ++item)
#define FOR_ITEMS_FROM4(item, counter, start, nitems)                                                      \
  for (int64_t item##_b = (start) + claim_batch(counter); item##_b < (nitems);                            \
       item##_b = (start) + claim_batch(counter))                                                         \
    for (int64_t item = item##_b, item##_e = item##_b + CLAIM_BATCH < (int64_t)(nitems) ? item##_b + CLAIM_BATCH \
                                                                                      : (int64_t)(nitems); \
         item < item##_e; ++item)

template <int H>
__device__ __forceinline__ float head_pick(const float (&x)[H], int h) {
  float r = 0.0f;
#pragma unroll
  for (int k = 0; k < H; ++k) if (k == h) r = x[k];
  return r;
}

// ---- heavy-row helpers: every load of a batch is issued before the dependent arithmetic (hub rows
// span up to ~32 segments; the folds stay in canonical order, only the loads are hoisted).
template <int H>
__device__ __forceinline__ void load_qh(const int8_t* __restrict__ p, int8_t (&o)[H]) {
  if constexpr (H == 4) {
    const uint32_t w = __ldg(reinterpret_cast<const unsigned*>(p));
#pragma unroll
    for (int h = 0; h < 4; ++h) o[h] = (int8_t)(w >> (8 * h));
  } else if constexpr (H == 2) {
    const uint32_t w = __ldg(reinterpret_cast<const unsigned short*>(p));
    o[0] = (int8_t)w; o[1] = (int8_t)(w >> 8);
  } else {
#pragma unroll
    for (int h = 0; h < H; ++h) o[h] = p[h];
  }
}

// ------------------------------------------------------------------ light-row tiles
// A tile = 32 consecutive local rows, lane j owning row r0 + j.  Heavy rows inside the tile are
// skipped (their segments are separate work items).  The tile's light rows form ONE edge stream
// t = 0..T-1 (row after row, canonical order inside each row), so the per-row latency chain
// (row pointers -> indices -> attention inputs) is paid once per tile instead of once per row and
// the 8-deep gather pipeline runs across row boundaries; accumulators flush when the row changes.
constexpr int TILE = 32;

struct TileLane {
  int64_t r, eb;        // this lane's local row and its first edge
  int deg, off, end;    // degree (0 for heavy / absent rows), exclusive and inclusive scan
  bool light;           // row exists and is light
};

__device__ __forceinline__ TileLane tile_setup(const int64_t* __restrict__ ptr, const int32_t* __restrict__ hbase,
                                               int64_t r0, int64_t n, int& T, int lo = 0, int hi = 32) {
  const int lane = threadIdx.x & 31;
  TileLane L;
  L.r = r0 + lane;
  const bool has = L.r < n && lane >= lo && lane < hi;
  L.light = has && hbase[L.r] < 0;
  L.eb = has ? ptr[L.r] : 0;
  const int64_t ee = has ? ptr[L.r + 1] : 0;
  L.deg = L.light ? (int)(ee - L.eb) : 0;
  int x = L.deg;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  L.end = x;
  L.off = x - L.deg;
  T = __shfl_sync(0xffffffffu, x, 31);
  return L;
}
// lane (row) of stream position t: the smallest j with end_j > t (rows of degree 0 are skipped)
__device__ __forceinline__ int tile_row(int t, int end) {
  int pos = 0;
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) {
    const int ev = __shfl_sync(0xffffffffu, end, pos + s - 1);
    if (ev <= t) pos += s;
  }
  return pos & 31;
}
// next row (lane) after `cur` with edges, -1 if none
__device__ __forceinline__ int tile_next(unsigned act, int cur) {
  const unsigned rest = cur >= 31 ? 0u : (act & ~((2u << cur) - 1u));
  return rest ? __ffs(rest) - 1 : -1;
}


__device__ __forceinline__ void amax_flush(unsigned* slot, float amax_loc) {
  amax_loc = warp_max(amax_loc);
  if ((threadIdx.x & 31) == 0 && slot) atomicMax(slot, __float_as_uint(amax_loc));
}


// ---- packed fp32x2 helpers (sm_100a FADD2 / FFMA2: IEEE rn per half, bit-identical to scalar ops)
__device__ __forceinline__ uint64_t pk2(uint32_t lo, uint32_t hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(lo), "r"(hi));
  return r;
}
__device__ __forceinline__ uint64_t pkf(float x) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %1};" : "=l"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ void unpk(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
// acc = fma(al, (float)q[k], acc) for the 4 codes of one word: PRMT builds 2^23+128+q, FADD2 removes
// the bias exactly, FFMA2 accumulates (sm_100a packed fp32: IEEE rn per half, bit-identical to fmaf)
__device__ __forceinline__ float2 codes2(uint32_t wx, uint32_t s0, uint32_t s1) {
  return __fadd2_rn(make_float2(__uint_as_float(__byte_perm(wx, 0x4B000000u, s0)),
                                __uint_as_float(__byte_perm(wx, 0x4B000000u, s1))),
                    make_float2(-8388736.0f, -8388736.0f));
}
// the same for 4 excess-128 codes (q + 128): the PRMT already yields 2^23 + 128 + q, no sign flip
// (tried: the top byte through IMAD.HI on the FMA pipe to unload the ALU pipe — 25 % slower gathers)
__device__ __forceinline__ void fma4_biased(uint32_t word, float2 al2, float2& a01, float2& a23) {
  a01 = __ffma2_rn(al2, codes2(word, 0x7440u, 0x7441u), a01);
  a23 = __ffma2_rn(al2, codes2(word, 0x7442u, 0x7443u), a23);
}
// Σ_k a_k·b_k over 4 byte lanes with a unsigned (excess-128 codes) and b signed
__device__ __forceinline__ int dp4a_us(uint32_t a, uint32_t b, int c) {
  int d;
  asm("dp4a.u32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
// exact q_x·q_y of this lane's slice where x holds excess-128 codes and y plain codes:
// Σ (q_x + 128)·q_y − 128·Σ q_y
template <int VPL>
__device__ __forceinline__ int row_dot_biased(const Row<VPL>& x, const Row<VPL>& y, int ysum) {
  int acc = 0;
#pragma unroll
  for (int i = 0; i < VPL / 4; ++i) acc = dp4a_us(x.w[i], y.w[i], acc);
  return acc - 128 * ysum;
}
// Σ (q_x + 128)·q_y of this lane's slice without the correction (applied after a cross-lane reduction)
template <int VPL>
__device__ __forceinline__ int row_dot_raw(const Row<VPL>& x, const Row<VPL>& y) {
  int acc = 0;
#pragma unroll
  for (int i = 0; i < VPL / 4; ++i) acc = dp4a_us(x.w[i], y.w[i], acc);
  return acc;
}
// Σ of this lane's plain codes (for the correction above); flips excess-128 codes to plain first
template <int VPL>
__device__ __forceinline__ int row_sum_plain(Row<VPL>& y, bool flip) {
  int s = 0;
#pragma unroll
  for (int i = 0; i < VPL / 4; ++i) {
    if (flip) y.w[i] ^= 0x80808080u;
    s = __dp4a((int)y.w[i], 0x01010101, s);
  }
  return s;
}

__device__ __forceinline__ void fma4_codes(uint32_t word, float2 al2, float2& a01, float2& a23) {
  const uint32_t wx = word ^ 0x80808080u;
  a01 = __ffma2_rn(al2, codes2(wx, 0x7440u, 0x7441u), a01);
  a23 = __ffma2_rn(al2, codes2(wx, 0x7442u, 0x7443u), a23);
}
template <bool BIASED>
__device__ __forceinline__ void fma4_any(uint32_t word, float2 al2, float2& a01, float2& a23) {
  if constexpr (BIASED) fma4_biased(word, al2, a01, a23);
  else fma4_codes(word, al2, a01, a23);
}


// ================================================================== cp.async gather engine
// Each lane copies its own VPL-byte slice of a gathered row into a per-warp shared-memory ring of R
// rows (cp.async.cg: L2 only, no register held while in flight), waits with cp.async.wait_group and
// reads back only the bytes it copied itself (no cross-lane synchronisation).  The next 32-edge
// chunk's indices and α are loaded one chunk ahead so the ring streams across chunk boundaries.
__device__ __forceinline__ void cp_async_bytes16(uint32_t saddr, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_bytes8(uint32_t saddr, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(saddr), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_bytes4(uint32_t saddr, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(saddr), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int VPL>
__device__ __forceinline__ void cp_row_slice(uint32_t saddr, const int8_t* g) {
  if constexpr (VPL == 16) cp_async_bytes16(saddr, g);
  else if constexpr (VPL == 8) cp_async_bytes8(saddr, g);
  else cp_async_bytes4(saddr, g);
}
template <int VPL>
__device__ __forceinline__ Row<VPL> lds_row_slice(uint32_t saddr) {
  Row<VPL> r;
  if constexpr (VPL == 16) {
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]) : "r"(saddr));
  } else if constexpr (VPL == 8) {
    asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(r.w[0]), "=r"(r.w[1]) : "r"(saddr));
  } else {
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r.w[0]) : "r"(saddr));
  }
  return r;
}

constexpr int AGG_RING = 16;

// 4-edge transposed reduction of per-lane partial dots over the LPH lanes of a head: afterwards the
// lane holds the full (exact, integer) dot of edge k = (lane & LPH/2 ? 2 : 0) + (lane & LPH/4 ? 1 : 0)
// of the group; 4 shuffles instead of 4 * log2(LPH).
template <int LPH>
__device__ __forceinline__ int group_dot_reduce(const int (&d)[4], int& k) {
  const int lane = threadIdx.x & 31;
  const bool hi = lane & (LPH / 2), mid = lane & (LPH / 4);
  const int x0 = (hi ? d[2] : d[0]) + __shfl_xor_sync(0xffffffffu, hi ? d[0] : d[2], LPH / 2);
  const int x1 = (hi ? d[3] : d[1]) + __shfl_xor_sync(0xffffffffu, hi ? d[1] : d[3], LPH / 2);
  int y = (mid ? x1 : x0) + __shfl_xor_sync(0xffffffffu, mid ? x0 : x1, LPH / 4);
#pragma unroll
  for (int o = LPH / 8; o > 0; o >>= 1) y += __shfl_xor_sync(0xffffffffu, y, o);
  k = (hi ? 2 : 0) + (mid ? 1 : 0);
  return y;
}


}  // namespace tango
