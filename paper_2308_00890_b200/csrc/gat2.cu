// gat2.cu — the single-GPU sparse half of the quantized GAT layer, v6 dataflow.
//
// Paper: ③ SDDMM-add + LeakyReLU, ④ edge softmax (FP32 per P:604-615),
// ⑤ SPMM, ⑤′ SPMM on the reversed graph, ⑤″ SDDMM-dot on codes (P:252-255,
// P:875-876), ④′ softmax backward, ③′/③″ incidence SPMM, ②′ (R23).
//
// Values are exactly those of the oracle (canonical chunked sums Σᶜ of reading R14, pinned fp32 ops);
// only WHERE each value is computed differs from the round-1 kernels (gat.cu):
//   * No edge-sized α array: every pass recomputes α[e,h] = exp_p(lrelu(e_pre) − m[v,h]) / den[v,h]
//     from the int8 q_S, q_D rows and the per-node m, den — bit-identical to the stored value.
//   * Forward = two kernels: F-stats (m, den per destination; hub rows by a whole CTA, light rows by
//     warp tiles) and F-agg (⑤ with α recomputed; hub segments folded by the last finishing warp).
//   * Backward = ONE row-gather pass instead of two: the SOURCE pass P1 gathers q_G[v] along out-edges
//     of u and computes both ⑤′ (α·q_G[v] into ∂H′_agg[u]) and ⑤″ (∂α[e] = q_G[v]·q_H′[u] on codes, u's
//     row held in registers), writing ∂α in out-CSR order (coalesced).  P2 (destination rows, no row
//     gather; ∂α through the in-CSR -> out-CSR position map) folds P = Σᶜ fmaf(∂α, α) and
//     ∂D = Σᶜ ∂E_pre; P3 (source rows, no row gather) folds ∂S = Σᶜ ∂E_pre and finalizes
//     ∂H′ = (∂H′_agg + ∂S·a_src) + ∂D·a_dst.  For the Reddit-shaped layer this removes one 58.8 GB
//     pass of int8 row gathers (the former destination-side SDDMM-dot).
#include "gat_common.cuh"

namespace tango {

namespace {

// ------------------------------------------------------------------ small helpers
template <int H>
__device__ __forceinline__ void ld_h(const float* __restrict__ p, float (&o)[H]) {
  if constexpr (H == 4) {
    const float4 v = *reinterpret_cast<const float4*>(p);
    o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
  } else if constexpr (H == 8) {
    const float4 v = *reinterpret_cast<const float4*>(p), w = *reinterpret_cast<const float4*>(p + 4);
    o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w; o[4] = w.x; o[5] = w.y; o[6] = w.z; o[7] = w.w;
  } else if constexpr (H == 2) {
    const float2 v = *reinterpret_cast<const float2*>(p);
    o[0] = v.x; o[1] = v.y;
  } else {
#pragma unroll
    for (int h = 0; h < H; ++h) o[h] = p[h];
  }
}
template <int H>
__device__ __forceinline__ void st_h(float* __restrict__ p, const float (&o)[H]) {
  if constexpr (H == 4) {
    *reinterpret_cast<float4*>(p) = make_float4(o[0], o[1], o[2], o[3]);
  } else if constexpr (H == 8) {
    *reinterpret_cast<float4*>(p) = make_float4(o[0], o[1], o[2], o[3]);
    *reinterpret_cast<float4*>(p + 4) = make_float4(o[4], o[5], o[6], o[7]);
  } else if constexpr (H == 2) {
    *reinterpret_cast<float2*>(p) = make_float2(o[0], o[1]);
  } else {
#pragma unroll
    for (int h = 0; h < H; ++h) p[h] = o[h];
  }
}

// order-preserving unsigned key of a float (never −0 or NaN here: el = lrelu(e_pre) and e_pre is a sum
// of two products of finite values, which is never −0)
__device__ __forceinline__ unsigned fkey(float x) {
  const unsigned b = __float_as_uint(x);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float fkey_dec(unsigned k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k);
}

// per-destination data of the edge softmax: q_D row, m, den
template <int H>
struct DstSm {
  int8_t qd[H];
  float m[H], den[H];
};
template <int H>
__device__ __forceinline__ DstSm<H> load_dst(const G2Args& a, int64_t vg) {
  DstSm<H> d;
  load_qh<H>(a.qD + vg * H, d.qd);
  ld_h<H>(a.m + vg * H, d.m);
  ld_h<H>(a.den + vg * H, d.den);
  return d;
}
// the same from the packed per-node record (one 64-B block at H = 4: m, den in the first sector, P and q_D
// in the second), for gathers of another node's data
template <int H>
__device__ __forceinline__ DstSm<H> load_rec(const G2Args& a, int64_t v) {
  DstSm<H> d;
  const float* r = a.nrec + v * a.nrs;
  ld_h<H>(r, d.m);
  ld_h<H>(r + H, d.den);
  load_qh<H>(reinterpret_cast<const int8_t*>(r + 3 * H), d.qd);
  return d;
}
// the record's fields as loaded (q_D still packed), unpacked where α is computed, so that a gather issued a
// chunk ahead is not consumed (byte extraction) right after it is issued
template <int H>
struct RecRaw {
  float m[H], den[H];
  uint32_t qw[(H + 3) / 4];
};
template <int H>
__device__ __forceinline__ RecRaw<H> load_rec_raw(const G2Args& a, int64_t v) {
  RecRaw<H> r;
  const float* p = a.nrec + v * a.nrs;
  ld_h<H>(p, r.m);
  ld_h<H>(p + H, r.den);
  const uint32_t* q = reinterpret_cast<const uint32_t*>(p + 3 * H);
  if constexpr (H == 1) r.qw[0] = *reinterpret_cast<const uint8_t*>(q);
  else if constexpr (H == 2) r.qw[0] = *reinterpret_cast<const uint16_t*>(q);
  else {
#pragma unroll
    for (int k = 0; k < (H + 3) / 4; ++k) r.qw[k] = q[k];
  }
  return r;
}
template <int H>
__device__ __forceinline__ DstSm<H> rec_unpack(const RecRaw<H>& r) {
  DstSm<H> d;
#pragma unroll
  for (int h = 0; h < H; ++h) {
    d.m[h] = r.m[h];
    d.den[h] = r.den[h];
    d.qd[h] = (int8_t)(r.qw[h >> 2] >> (8 * (h & 3)));
  }
  return d;
}
template <int H>
__device__ __forceinline__ void rec_put(const G2Args& a, int64_t v, int field, const float (&x)[H]) {
  st_h<H>(a.nrec + v * a.nrs + field * H, x);
}
__device__ __forceinline__ void rec_put1(const G2Args& a, int64_t v, int field, int h, float x) {
  a.nrec[v * a.nrs + field * a.d.heads + h] = x;
}
template <int H>
__device__ __forceinline__ void rec_put_qd(const G2Args& a, int64_t v) {
  int8_t* r = reinterpret_cast<int8_t*>(a.nrec + v * a.nrs + 3 * H);
#pragma unroll
  for (int h = 0; h < H; ++h) r[h] = a.qD[v * H + h];
}

// e_pre (③, two rn multiplies + one rn add) and α (④: exp_p(el − m) / den), all heads
template <int H>
__device__ __forceinline__ void alpha_rec(const int8_t (&qs)[H], const DstSm<H>& d, float sS, float sD, float slope,
                                          float (&ep)[H], float (&al)[H]) {
#pragma unroll
  for (int h = 0; h < H; ++h) {
    ep[h] = sddmm_add1(qs[h], sS, d.qd[h], sD);
    al[h] = __fdiv_rn(exp_p(__fsub_rn(lrelu(ep[h], slope), d.m[h])), d.den[h]);
  }
}

template <int H>
__device__ __forceinline__ int8_t head_pick_i8(const int8_t (&x)[H], int h) {
  int8_t r = 0;
#pragma unroll
  for (int k = 0; k < H; ++k) if (k == h) r = x[k];
  return r;
}

// P1's record of an edge at its in-CSR slot for P2: {∂α[H], α[H] with the LeakyReLU branch in its sign bit},
// 2H floats = one full 32-B sector at H = 4 (no partial-sector read-modify-write in L2 / DRAM)
template <int H>
__device__ __forceinline__ void put_rec(float* rec, int64_t slot, const float (&dal)[H], const float* sa_lane,
                                        uint32_t sg) {
  float al[H];
#pragma unroll
  for (int h = 0; h < H; ++h) {
    const float x = sa_lane[h * 32];
    al[h] = (sg >> h) & 1u ? x : -x;
  }
  if constexpr (H == 4) {   // one 256-bit streaming store: the whole sector in one L2 write (no partial-sector
                            // fill), evict-first so the write streams do not push the gathered table out of L2
    asm volatile("st.global.cs.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(rec + slot * 8), "f"(dal[0]), "f"(dal[1]),
                 "f"(dal[2]), "f"(dal[3]), "f"(al[0]), "f"(al[1]), "f"(al[2]), "f"(al[3])
                 : "memory");
  } else {
    st_h<H>(rec + slot * 2 * H, dal);
    st_h<H>(rec + slot * 2 * H + H, al);
  }
}
// P1's signed α of an out-edge at its out-CSR position (for P3, coalesced, streaming)
template <int H>
__device__ __forceinline__ void put_alpha(float* dst, const float* sa_lane, uint32_t sg) {
  float al[H];
#pragma unroll
  for (int h = 0; h < H; ++h) {
    const float x = sa_lane[h * 32];
    al[h] = (sg >> h) & 1u ? x : -x;
  }
  if constexpr (H == 4) __stcs(reinterpret_cast<float4*>(dst), make_float4(al[0], al[1], al[2], al[3]));
  else st_h<H>(dst, al);
}
template <int H>
__device__ __forceinline__ uint32_t ep_sign_bits(const float (&ep)[H]) {
  uint32_t sg = 0;
#pragma unroll
  for (int h = 0; h < H; ++h) sg |= (ep[h] > 0.0f ? 1u : 0u) << h;
  return sg;
}

// α with the LeakyReLU branch in its sign bit (negative: e_pre <= 0), stored by F-agg for the destination
// pass P2 (which then neither gathers q_S nor recomputes α); α >= 0, so |stored| = α exactly
template <int H>
__device__ __forceinline__ void store_alpha(float* dst, const float (&al)[H], const float (&ep)[H]) {
  float o[H];
#pragma unroll
  for (int h = 0; h < H; ++h) o[h] = ep[h] > 0.0f ? al[h] : -al[h];
  st_h<H>(dst, o);
}

template <int H>
__host__ __device__ constexpr int hbatch() { return H >= 8 ? 32 : 64; }   // edges per staged batch of a hub chunk

// ------------------------------------------------------------------ light tiles: segmented sums
// A light sub-tile's rows form one edge stream t = 0..T-1 (TileLane).  For each 32-position batch every
// lane computes the per-head values of its position; the row's owner lane then adds its row's part
// of the batch sequentially (a light row is a single chunk of the canonical sum, reading R14).
struct TileCtx {
  TileLane L;
  int T;
  int64_t r0;
};
__device__ __forceinline__ int64_t tile_edge(const TileCtx& t, int pos, int& row) {
  row = tile_row(pos < t.T ? pos : t.T - 1, t.L.end);
  return __shfl_sync(0xffffffffu, t.L.eb, row) + (pos - __shfl_sync(0xffffffffu, t.L.off, row));
}

// sequential per-row fold of a staged 32-position batch: plain adds (FMA = false) of x, or fmaf(x, y, ·)
template <int H, bool FMA>
__device__ __forceinline__ void tile_fold(const TileCtx& t, int base, const float (*sx)[H], const float (*sy)[H],
                                          float (&acc)[H]) {
  const int cnt = t.T - base < 32 ? t.T - base : 32;
  const int lo = (t.L.off > base ? t.L.off : base) - base;
  const int hi = (t.L.end < base + cnt ? t.L.end : base + cnt) - base;
  for (int i = lo; i < hi; ++i)
#pragma unroll
    for (int h = 0; h < H; ++h) acc[h] = FMA ? __fmaf_rn(sx[i][h], sy[i][h], acc[h]) : __fadd_rn(acc[h], sx[i][h]);
}

// ------------------------------------------------------------------ hub rows: per-segment partials
// A hub row (degree > C_E) is cut into its canonical chunks ("segments", reading R14), each an
// independent warp work item.  A segment's per-edge values are computed lane-parallel, two edges per
// lane per batch of 64 (both edges' loads issued before either is used), staged in the warp's buffer,
// and lane h < H adds head h's values of the batch in edge order: the chunk partial of Σᶜ.  The warp
// whose segment completes the row last (atomic count per row) folds the row's partials in chunk order
// (total = p_0, total = total + p_c) — bit-identical to the oracle's left-to-right fold.
constexpr int SB = 64;   // edges per staged batch
template <int H, bool FMA, typename LD, typename CV>
__device__ __forceinline__ float seg_partial(int64_t eb, int64_t ee, float (*bx)[H], float (*by)[H], LD&& ld,
                                             CV&& cv) {
  const int lane = threadIdx.x & 31;
  float acc = 0.0f;   // lane h < H: head h
  const int cnt = (int)(ee - eb);
  // the next batch's loads are issued before this batch's sequential sums (latency overlap)
  auto l0 = ld(eb + (lane < cnt ? lane : 0));
  auto l1 = ld(eb + (lane + 32 < cnt ? lane + 32 : 0));
  for (int b0 = 0; b0 < cnt; b0 += SB) {
    const int bc = cnt - b0 < SB ? cnt - b0 : SB;
    const bool v0 = lane < bc, v1 = lane + 32 < bc;
    float x[H], y[H];
    if (v0) {
      cv(l0, x, y);
#pragma unroll
      for (int h = 0; h < H; ++h) { bx[lane][h] = x[h]; if (FMA) by[lane][h] = y[h]; }
    }
    if (v1) {
      cv(l1, x, y);
#pragma unroll
      for (int h = 0; h < H; ++h) { bx[lane + 32][h] = x[h]; if (FMA) by[lane + 32][h] = y[h]; }
    }
    __syncwarp();
    const int nb = b0 + SB;
    if (nb < cnt) {
      l0 = ld(eb + nb + (nb + lane < cnt ? lane : 0));
      l1 = ld(eb + nb + (nb + lane + 32 < cnt ? lane + 32 : 0));
    }
    if (lane < H) {
      int i = 0;
      for (; i + 4 <= bc; i += 4) {
        const float x0 = bx[i][lane], x1 = bx[i + 1][lane], x2 = bx[i + 2][lane], x3 = bx[i + 3][lane];
        if (FMA) {
          const float y0 = by[i][lane], y1 = by[i + 1][lane], y2 = by[i + 2][lane], y3 = by[i + 3][lane];
          acc = __fmaf_rn(x0, y0, acc); acc = __fmaf_rn(x1, y1, acc);
          acc = __fmaf_rn(x2, y2, acc); acc = __fmaf_rn(x3, y3, acc);
        } else {
          acc = __fadd_rn(acc, x0); acc = __fadd_rn(acc, x1); acc = __fadd_rn(acc, x2); acc = __fadd_rn(acc, x3);
        }
      }
      for (; i < bc; ++i) acc = FMA ? __fmaf_rn(bx[i][lane], by[i][lane], acc) : __fadd_rn(acc, bx[i][lane]);
    }
    __syncwarp();
  }
  return acc;
}
// true (whole warp) for the warp that finished the row's last segment; resets the row's counter
__device__ __forceinline__ bool seg_last(int32_t* cnt, int64_t row, int nseg) {
  if (nseg == 1) return true;
  __threadfence();
  int d = 0;
  if ((threadIdx.x & 31) == 0) d = atomicAdd(cnt + row, 1);
  d = __shfl_sync(0xffffffffu, d, 0);
  if (d != nseg - 1) return false;
  __threadfence();
  if ((threadIdx.x & 31) == 0) cnt[row] = 0;
  return true;
}
// chunk-order fold of a row's per-segment partials [slot][H] (L2 reads: written by other SMs); lane h < H
// returns head h's total
template <int H>
__device__ __forceinline__ float seg_fold(const float* part, int base, int nseg) {
  const int lane = threadIdx.x & 31;
  float tot = 0.0f;
  for (int j0 = 0; j0 < nseg; j0 += 32 / H) {
    // lanes load 32/H segments x H heads at once: lane = jj * H + h
    const int jj = lane / H, h = lane % H, j = j0 + jj;
    const float v = j < nseg ? __ldcg(part + (int64_t)(base + j) * H + h) : 0.0f;
    const int cnt = nseg - j0 < 32 / H ? nseg - j0 : 32 / H;
    for (int k = 0; k < cnt; ++k) {
      const float y = __shfl_sync(0xffffffffu, v, k * H + (lane % H));
      tot = (j0 + k == 0) ? y : __fadd_rn(tot, y);
    }
  }
  return tot;   // valid in every lane for head lane % H
}
template <int H>
__device__ __forceinline__ float seg_fold_max(const float* part, int base, int nseg) {
  const int lane = threadIdx.x & 31;
  float m = -INFINITY;
  for (int j = lane / H; j < nseg; j += 32 / H) m = fmaxf(m, __ldcg(part + (int64_t)(base + j) * H + lane % H));
#pragma unroll
  for (int o = 16; o >= H; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  return m;   // every lane: max for head lane % H
}

}  // namespace

// ================================================================== F-stats: m, den per destination
// FS1 (hub segments): segment max of el = lrelu(e_pre), folded into the row's m by an atomic max on
// order-preserving keys (max is order-free: no partials, no fold).
// FS2 (hub segments, then light sub-tiles): segment Σ exp_p(el − m) partial, folded in chunk order by the
// row's last segment into den; a light sub-tile computes m and den of its rows in two lane-parallel passes
// (per-row max by a segmented lane scan, Σ by the row's owner lane in edge order).
template <int H>
__global__ void __launch_bounds__(256, 4) k2_fstats1(const G2Args a) {
  const int lane = threadIdx.x & 31;
  const Scale scS = scale_from_amax(amax_load(a.amax_S), a.bits);
  const Scale scD = scale_from_amax(amax_load(a.amax_D), a.bits);
  const int64_t hc = load_count(a.pin.counts);
  FOR_ITEMS4(si, a.work + 0, hc) {
    Seg s;
    decode_item(si, hc, a.g.in_ptr, a.pin, a.g.chunk, s);
    const int64_t vg = a.g.row_begin + s.vl;
    int8_t qd[H];
    load_qh<H>(a.qD + vg * H, qd);
    if (a.slope > 0.0f) {
      // e_pre (two rn products and one rn add, sS > 0) and LeakyReLU (slope > 0) are monotone
      // non-decreasing in q_S[u], so max over the edges of el = lrelu(e_pre(max q_S)): the max is taken on
      // the int8 codes (SIMD byte max over all heads at once) and converted once — the same value as the
      // oracle's max of the el (no ±0 ties: el = −0 needs slope 0)
      constexpr int NW = (H + 3) / 4;
      uint32_t mw[NW];
#pragma unroll
      for (int k = 0; k < NW; ++k) mw[k] = 0x80808080u;
      for (int64_t b = s.eb; b < s.ee; b += 256) {   // a whole C_E = 256 chunk per round trip pair
        int u[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) u[k] = b + 32 * k + lane < s.ee ? __ldg(a.g.in_src + b + 32 * k + lane) : -1;
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (u[k] >= 0) {
            const int8_t* q = a.qS + (int64_t)u[k] * H;
            if constexpr (H == 1) mw[0] = __vmaxs4(mw[0], 0x80808000u | (uint32_t)(uint8_t)__ldg(q));
            else if constexpr (H == 2)
              mw[0] = __vmaxs4(mw[0], 0x80800000u | (uint32_t)__ldg(reinterpret_cast<const unsigned short*>(q)));
            else {
#pragma unroll
              for (int w = 0; w < NW; ++w) mw[w] = __vmaxs4(mw[w], __ldg(reinterpret_cast<const unsigned*>(q) + w));
            }
          }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int w = 0; w < NW; ++w) mw[w] = __vmaxs4(mw[w], __shfl_xor_sync(0xffffffffu, mw[w], o));
      if (lane < H) {
        const int code = (int8_t)(mw[lane >> 2] >> (8 * (lane & 3)));
        const float m = lrelu(sddmm_add1((int8_t)code, scS.s, head_pick_i8<H>(qd, lane), scD.s), a.slope);
        atomicMax(reinterpret_cast<unsigned*>(a.nrec + vg * a.nrs) + lane, fkey(m));
      }
      continue;
    }
    float mx[H];
#pragma unroll
    for (int h = 0; h < H; ++h) mx[h] = -INFINITY;
    for (int64_t b = s.eb; b < s.ee; b += 128) {
      int u[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) u[k] = b + 32 * k + lane < s.ee ? a.g.in_src[b + 32 * k + lane] : -1;
      int8_t qs[4][H];
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (u[k] >= 0) load_qh<H>(a.qS + (int64_t)u[k] * H, qs[k]);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (u[k] >= 0)
#pragma unroll
          for (int h = 0; h < H; ++h) mx[h] = fmaxf(mx[h], lrelu(sddmm_add1(qs[k][h], scS.s, qd[h], scD.s), a.slope));
    }
#pragma unroll
    for (int h = 0; h < H; ++h) mx[h] = warp_max(mx[h]);
    // max is order-free: every segment folds its maximum into the row's m field of the node record
    // (order-preserving unsigned keys; the record is zeroed at the start of the forward, below any key)
    if (lane < H) atomicMax(reinterpret_cast<unsigned*>(a.nrec + vg * a.nrs) + lane, fkey(head_pick<H>(mx, lane)));
  }
}

template <int H>
__global__ void __launch_bounds__(256, 4) k2_fstats2(const G2Args a) {
  __shared__ float sbx[8][SB][H];
  __shared__ float tmx[8][32][H];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Scale scS = scale_from_amax(amax_load(a.amax_S), a.bits);
  const Scale scD = scale_from_amax(amax_load(a.amax_D), a.bits);
  const int64_t n = a.g.n_local, hc = load_count(a.pin.counts), nitems = hc + load_count(a.pin.counts + 2);
  FOR_ITEMS_FROM4(item, a.work + 3, a.hub_fs ? hc : 0, nitems) {
    if (item < hc) {   // ---- hub segment (staged form; k2_fstats2_hub(m) when hub_fs)
      Seg s;
      decode_item(item, hc, a.g.in_ptr, a.pin, a.g.chunk, s);
      const int64_t vg = a.g.row_begin + s.vl;
      int8_t qd[H];
      load_qh<H>(a.qD + vg * H, qd);
      float m[H];
#pragma unroll
      for (int h = 0; h < H; ++h) m[h] = fkey_dec(reinterpret_cast<const unsigned*>(a.nrec + vg * a.nrs)[h]);
      struct L { int8_t qs[H]; };
      const float part = seg_partial<H, false>(
          s.eb, s.ee, sbx[w], nullptr,
          [&](int64_t e) { L l; load_qh<H>(a.qS + (int64_t)a.g.in_src[e] * H, l.qs); return l; },
          [&](const L& l, float (&x)[H], float (&)[H]) {
#pragma unroll
            for (int h = 0; h < H; ++h)
              x[h] = exp_p(__fsub_rn(lrelu(sddmm_add1(l.qs[h], scS.s, qd[h], scD.s), a.slope), m[h]));
          });
      if (lane < H) __stcg(a.h2 + (int64_t)s.slot * H + lane, part);
      if (!seg_last(a.hcnt, s.vl, s.nseg)) continue;
      const float den = seg_fold<H>(a.h2, s.base, s.nseg);
      if (lane < H) {   // the row's m (as a float) and den; every segment of the row has read the keys
        a.m[vg * H + lane] = head_pick<H>(m, lane);
        rec_put1(a, vg, 0, lane, head_pick<H>(m, lane));
        a.den[vg * H + lane] = den;
        rec_put1(a, vg, 1, lane, den);
      }
      if (lane == 0) rec_put_qd<H>(a, vg);
      continue;
    }
    // ---- light sub-tile
    const int32_t code = a.pin.tiles[item - hc];
    TileCtx t;
    t.r0 = (int64_t)(code >> 10) * TILE;
    t.L = tile_setup(a.g.in_ptr, a.pin.hbase, t.r0, n, t.T, (code >> 5) & 31, (code & 31) + 1);
    const int64_t vgl = a.g.row_begin + t.L.r;
    float (*tbuf)[H] = reinterpret_cast<float (*)[H]>(&sbx[w][0][0]);
    int qdj[H];
#pragma unroll
    for (int h = 0; h < H; ++h) {
      qdj[h] = t.L.light ? (int)a.qD[vgl * H + h] : 0;
      tmx[w][lane][h] = -INFINITY;
    }
    __syncwarp();
    auto el_at = [&](int pos, float (&el)[H], int& row) {
      const int64_t e = tile_edge(t, pos, row);
      int qdr[H];
#pragma unroll
      for (int h = 0; h < H; ++h) qdr[h] = __shfl_sync(0xffffffffu, qdj[h], row);
      if (pos < t.T) {
        int8_t qs[H];
        load_qh<H>(a.qS + (int64_t)a.g.in_src[e] * H, qs);
#pragma unroll
        for (int h = 0; h < H; ++h) el[h] = lrelu(sddmm_add1(qs[h], scS.s, (int8_t)qdr[h], scD.s), a.slope);
      } else {
#pragma unroll
        for (int h = 0; h < H; ++h) el[h] = -INFINITY;
      }
    };
    for (int base = 0; base < t.T; base += 32) {   // pass A: per-row max (segmented lane scan)
      float el[H];
      int row;
      el_at(base + lane, el, row);
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int ro = __shfl_up_sync(0xffffffffu, row, o);
#pragma unroll
        for (int h = 0; h < H; ++h) {
          const float y = __shfl_up_sync(0xffffffffu, el[h], o);
          if (lane >= o && ro == row) el[h] = fmaxf(el[h], y);
        }
      }
      const int rn = __shfl_down_sync(0xffffffffu, row, 1);
      if (base + lane < t.T && (lane == 31 || rn != row || base + lane + 1 >= t.T))
#pragma unroll
        for (int h = 0; h < H; ++h) tmx[w][row][h] = fmaxf(tmx[w][row][h], el[h]);
      __syncwarp();
    }
    float mown[H], den[H];
#pragma unroll
    for (int h = 0; h < H; ++h) {
      mown[h] = (t.L.light && t.L.deg > 0) ? tmx[w][lane][h] : 0.0f;
      den[h] = 0.0f;
    }
    for (int base = 0; base < t.T; base += 32) {   // pass B: Σ exp_p(el − m) by the row owner
      float el[H];
      int row;
      el_at(base + lane, el, row);
      float mr[H];
#pragma unroll
      for (int h = 0; h < H; ++h) mr[h] = __shfl_sync(0xffffffffu, mown[h], row);
      if (base + lane < t.T)
#pragma unroll
        for (int h = 0; h < H; ++h) tbuf[lane][h] = exp_p(__fsub_rn(el[h], mr[h]));
      __syncwarp();
      tile_fold<H, false>(t, base, tbuf, nullptr, den);
      __syncwarp();
    }
    if (t.L.light) {
      st_h<H>(a.m + vgl * H, mown);
      st_h<H>(a.den + vgl * H, den);
      rec_put<H>(a, vgl, 0, mown);
      rec_put<H>(a, vgl, 1, den);
      rec_put_qd<H>(a, vgl);
    }
  }
}

// ================================================================== gather engine (v8: cp.async, 8-edge groups)
// One warp streams a heavy segment (one row, ≤ C_E edges) or a light sub-tile (≤ 32 rows).  Each lane
// copies its own 16-B (VPL-byte) slice of every gathered row into a per-warp ring of RING = 16 rows
// (two groups of GR = 8 edges) with cp.async (L2 only, evict_last: the gathered table is the one
// structure worth keeping in L2), waits for the group with cp.async.wait_group and reads back only its
// own bytes (no cross-lane synchronisation).  A group is always 8 edges: positions past the end of the
// stream gather row 0 with α = +0, exact no-ops (fmaf(+0, q, acc) == acc; acc is never −0), so the hot
// loop has no per-edge predicates; every group (possibly empty past the end) is committed, so
// wait_group<1> always means "the current group has landed".  Per-edge attributes (gather row, α per
// head, tile row, ...) are computed lane-parallel for 32-edge chunks: gather rows two chunks ahead,
// attributes one chunk ahead, stashed in per-warp shared memory ([head][edge] for α).
constexpr int GR = 8;       // edges per group
constexpr int RING = 16;    // ring rows per warp (two groups)

template <int VPL>
__host__ __device__ constexpr int g8_ring_bytes() { return RING * 32 * VPL; }

__device__ __forceinline__ uint64_t l2_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
template <int VPL>
__device__ __forceinline__ void cp_slice_hint(uint32_t saddr, const int8_t* g, uint64_t pol) {
  if constexpr (VPL == 16)
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(saddr), "l"(g), "l"(pol) : "memory");
  else if constexpr (VPL == 8)   // (the cache-hint form of the 8- and 4-byte copies faults on sm_100a)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(saddr), "l"(g) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(saddr), "l"(g) : "memory");
}
// issue group g (rows sidx[8g .. 8g+7] of the chunk double buffer) into ring half g & 1, then commit
template <int VPL>
__device__ __forceinline__ void g8_fill(uint32_t ring_lane, const int8_t* lane_base, uint32_t ld, const int* sidx, int g,
                                        bool any, uint64_t pol) {
  if (any) {
    const int* ix = sidx + (((8 * g) >> 5) & 1) * 32 + ((8 * g) & 31);
    const int4 x0 = *reinterpret_cast<const int4*>(ix), x1 = *reinterpret_cast<const int4*>(ix + 4);
    const int iv[GR] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
    const uint32_t s0 = ring_lane + (uint32_t)(g & 1) * (GR * 32 * VPL);
#pragma unroll
    for (int j = 0; j < GR; ++j)   // base + row * ld as one 32 x 32 -> 64-bit IMAD.WIDE.U32
      cp_slice_hint<VPL>(s0 + j * 32 * VPL,
                         reinterpret_cast<const int8_t*>((uint64_t)lane_base + (uint64_t)(uint32_t)iv[j] * ld), pol);
  }
  cp_commit();
}
template <int VPL>
__device__ __forceinline__ void g8_rows(uint32_t ring_lane, int g, Row<VPL> (&r)[GR]) {
  const uint32_t s0 = ring_lane + (uint32_t)(g & 1) * (GR * 32 * VPL);
#pragma unroll
  for (int j = 0; j < GR; ++j) r[j] = lds_row_slice<VPL>(s0 + j * 32 * VPL);
}

// ================================================================== F-agg: ⑤ with α recomputed
// H_out[v] = (Σᶜ fmaf(α[e], q_H′[u]))·s_H′ over v's in-edges; α = exp_p(lrelu(e_pre) − m[v]) / den[v].
template <int H, int VPL>
__host__ __device__ constexpr int fa_warp_smem() {   // ring | α [2][H][32] | rows [2][32] | tile rows [2][32]
  return g8_ring_bytes<VPL>() + 2 * H * 32 * 4 + 2 * 32 * 4 + 2 * 32;
}
template <int H, int VPL>
__global__ void __launch_bounds__(256, 3) k2_fagg(const G2Args a) {
  constexpr int HD = 32 * VPL, WS = fa_warp_smem<H, VPL>();
  extern __shared__ __align__(16) uint8_t dsm[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int myh = lane / (32 / H);
  uint8_t* wsm = dsm + w * ((WS + 15) & ~15);
  float* sa = reinterpret_cast<float*>(wsm + g8_ring_bytes<VPL>());   // [2][H][32]
  int* sidx = reinterpret_cast<int*>(sa + 2 * H * 32);                // [2][32]
  uint8_t* srow = reinterpret_cast<uint8_t*>(sidx + 64);             // [2][32]
  const uint32_t ring_lane = smem_u32(wsm) + lane * VPL;
  const int8_t* lane_base = a.qHp + lane * VPL;
  const uint32_t ld32 = (uint32_t)a.ldHp;
  const uint64_t pol = l2_evict_last();
  const Scale scH = scale_from_amax(amax_load(a.amax_Hp), a.bits);
  const Scale scS = scale_from_amax(amax_load(a.amax_S), a.bits);
  const Scale scD = scale_from_amax(amax_load(a.amax_D), a.bits);
  const int64_t n = a.g.n_local, hc = load_count(a.pin.counts);
  const int64_t nitems = hc + load_count(a.pin.counts + 2);
  float amax_loc = 0.0f;
  FOR_ITEMS(it, a.work + 2, nitems - hc) {   // light sub-tiles (hub rows: k2_fagg_seg)
    const int64_t item = hc + it;
    constexpr bool tile = true;
    Seg s;
    s.eb = 0; s.vl = 0; s.slot = -1; s.nseg = 1;
    TileCtx t;
    t.r0 = 0;
    if (!tile) {
      decode_item(item, hc, a.g.in_ptr, a.pin, a.g.chunk, s);
      t.T = (int)(s.ee - s.eb);
      t.L.eb = 0; t.L.off = 0; t.L.end = 0;
    } else {
      const int32_t code = a.pin.tiles[item - hc];
      t.r0 = (int64_t)(code >> 10) * TILE;
      t.L = tile_setup(a.g.in_ptr, a.pin.hbase, t.r0, n, t.T, (code >> 5) & 31, (code & 31) + 1);
      unsigned zm = __ballot_sync(0xffffffffu, t.L.light && t.L.deg == 0);
      while (zm) {   // light rows without in-edges: H_out = 0
        const int j = __ffs(zm) - 1;
        zm &= zm - 1;
        float4* dst = reinterpret_cast<float4*>(a.Hout + (t.r0 + j) * HD + lane * VPL);
#pragma unroll
        for (int k = 0; k < VPL / 4; ++k) __stcs(dst + k, make_float4(0.0f, 0.0f, 0.0f, 0.0f));
      }
    }
    const int T = t.T;
    if (T == 0) continue;
    DstSm<H> dseg;
    if (!tile) dseg = load_dst<H>(a, a.g.row_begin + s.vl);
    // stream position -> (edge, tile row); gather row u (0 past the end)
    auto pos_of = [&](int c, int& row) -> int64_t {
      const int pos = c * 32 + lane;
      if (tile) return tile_edge(t, pos, row);
      row = 0;
      return s.eb + (pos < T ? pos : T - 1);
    };
    auto alpha_of = [&](int c, int u, int row, int64_t e, float (&al)[H]) {
#pragma unroll
      for (int h = 0; h < H; ++h) al[h] = 0.0f;
      if (c * 32 + lane < T) {
        const DstSm<H> d = tile ? load_dst<H>(a, a.g.row_begin + t.r0 + row) : dseg;
        int8_t qs[H];
        load_qh<H>(a.qS + (int64_t)u * H, qs);
        float ep[H];
        alpha_rec<H>(qs, d, scS.s, scD.s, a.slope, ep, al);
        if (a.alpha_st) store_alpha<H>(a.alpha_st + e * H, al, ep);
      }
    };
    auto stash = [&](int c, int row, const float (&al)[H]) {
      const int b = c & 1;
#pragma unroll
      for (int h = 0; h < H; ++h) sa[(b * H + h) * 32 + lane] = al[h];
      srow[b * 32 + lane] = (uint8_t)row;
    };
    const int nch = (T + 31) >> 5, ng = (T + GR - 1) / GR;
    // prologue: chunk 0 attributes, chunk 1 gather rows, first two groups
    int row1, u1 = 0;
    {
      int row0;
      const int64_t e0 = pos_of(0, row0);
      const int u0 = lane < T ? __ldcs(a.g.in_src + e0) : 0;
      float al0[H];
      alpha_of(0, u0, row0, e0, al0);
      stash(0, row0, al0);
      sidx[lane] = u0;
      const int64_t e1 = pos_of(1, row1);
      if (32 + lane < T) u1 = __ldcs(a.g.in_src + e1);
      sidx[32 + lane] = u1;
    }
    __syncwarp();
    g8_fill<VPL>(ring_lane, lane_base, ld32, sidx, 0, true, pol);
    g8_fill<VPL>(ring_lane, lane_base, ld32, sidx, 1, 1 < ng, pol);
    float2 acc[VPL / 2];
#pragma unroll
    for (int k = 0; k < VPL / 2; ++k) acc[k] = make_float2(0.0f, 0.0f);
    auto flush = [&](int j) {   // tile row j done: H_out = acc · s_H′
      float4* dst = reinterpret_cast<float4*>(a.Hout + (t.r0 + j) * HD + lane * VPL);
      const float2 sH2 = make_float2(scH.s, scH.s);
#pragma unroll
      for (int k = 0; k < VPL / 4; ++k) {
        const float2 o01 = __fmul2_rn(acc[2 * k], sH2), o23 = __fmul2_rn(acc[2 * k + 1], sH2);
        amax_loc = fmaxf(amax_loc, fmaxf(fmaxf(fabsf(o01.x), fabsf(o01.y)), fmaxf(fabsf(o23.x), fabsf(o23.y))));
        __stcs(dst + k, make_float4(o01.x, o01.y, o23.x, o23.y));
        acc[2 * k] = make_float2(0.0f, 0.0f);
        acc[2 * k + 1] = make_float2(0.0f, 0.0f);
      }
    };
    int cur = tile ? -1 : 0;
    for (int c = 0; c < nch; ++c) {
      // loads for chunk c + 2's gather rows and chunk c + 1's attributes, used after this chunk's groups
      int row2;
      const int64_t e2 = pos_of(c + 2, row2);
      const int u2 = (c + 2) * 32 + lane < T ? __ldcs(a.g.in_src + e2) : 0;
      int8_t qs1[H];
      int row1x = 0;
      const int64_t e1x = pos_of(c + 1, row1x);
      DstSm<H> d1 = dseg;
      if ((c + 1) * 32 + lane < T) {
        load_qh<H>(a.qS + (int64_t)u1 * H, qs1);
        if (tile) d1 = load_dst<H>(a, a.g.row_begin + t.r0 + row1x);
      }
      const int b = c & 1;
      const float* sac = sa + (b * H + myh) * 32;
      for (int i0 = 0; i0 < 32; i0 += GR) {
        const int t0 = c * 32 + i0;
        if (t0 >= T) break;
        const int g = t0 / GR;
        cp_wait<1>();
        const uint32_t s0 = ring_lane + (uint32_t)(g & 1) * (GR * 32 * VPL);
        const float4 a4 = *reinterpret_cast<const float4*>(sac + i0);
        const float4 b4 = *reinterpret_cast<const float4*>(sac + i0 + 4);
        const float al[GR] = {a4.x, a4.y, a4.z, a4.w, b4.x, b4.y, b4.z, b4.w};
        bool same = true;
        uint32_t rw0 = 0, rw1 = 0;
        if (tile) {
          rw0 = *reinterpret_cast<const uint32_t*>(srow + b * 32 + i0);
          rw1 = *reinterpret_cast<const uint32_t*>(srow + b * 32 + i0 + 4);
          same = (int)(rw0 & 0xffu) == cur && (int)(rw1 >> 24) == cur;
        }
        if (same) {
#pragma unroll
          for (int j = 0; j < GR; ++j) {
            const Row<VPL> rj = lds_row_slice<VPL>(s0 + j * 32 * VPL);
            const float2 al2 = make_float2(al[j], al[j]);
#pragma unroll
            for (int q = 0; q < VPL / 4; ++q) fma4_biased(rj.w[q], al2, acc[2 * q], acc[2 * q + 1]);
          }
        } else {
#pragma unroll
          for (int j = 0; j < GR; ++j) {
            const int rowj = (int)(((j < 4 ? rw0 : rw1) >> (8 * (j & 3))) & 0xffu);
            if (rowj != cur) {
              if (cur >= 0) flush(cur);
              cur = rowj;
            }
            const Row<VPL> rj = lds_row_slice<VPL>(s0 + j * 32 * VPL);
            const float2 al2 = make_float2(al[j], al[j]);
#pragma unroll
            for (int q = 0; q < VPL / 4; ++q) fma4_biased(rj.w[q], al2, acc[2 * q], acc[2 * q + 1]);
          }
        }
        g8_fill<VPL>(ring_lane, lane_base, ld32, sidx, g + 2, g + 2 < ng, pol);
      }
      // attributes of chunk c + 1 (buffer (c+1)&1, last read by chunk c − 1) and rows of chunk c + 2
      // (buffer c&1: chunk c's rows were last read by the refill after its first group)
      __syncwarp();
      if (c + 1 < nch) {
        float al1[H];
#pragma unroll
        for (int h = 0; h < H; ++h) al1[h] = 0.0f;
        if ((c + 1) * 32 + lane < T) {
          float ep[H];
          alpha_rec<H>(qs1, d1, scS.s, scD.s, a.slope, ep, al1);
          if (a.alpha_st) store_alpha<H>(a.alpha_st + e1x * H, al1, ep);
        }
        stash(c + 1, row1x, al1);
        sidx[b * 32 + lane] = u2;
      }
      __syncwarp();
      u1 = u2;
      (void)row2;
    }
    if (tile) {
      if (cur >= 0) flush(cur);
      continue;
    }
    // heavy segment: partial -> scratch; the row's last segment folds the partials in chunk order
    {
      float4* dst = reinterpret_cast<float4*>(a.hagg + (int64_t)s.slot * HD + lane * VPL);
#pragma unroll
      for (int k = 0; k < VPL / 4; ++k)
        __stcg(dst + k, make_float4(acc[2 * k].x, acc[2 * k].y, acc[2 * k + 1].x, acc[2 * k + 1].y));
    }
    if (!seg_last(a.hcnt, s.vl, s.nseg)) continue;
    float tot[VPL];
    {
      const float* p0 = a.hagg + (int64_t)s.base * HD + lane * VPL;
#pragma unroll
      for (int k = 0; k < VPL / 4; ++k) {
        const float4 v = __ldcg(reinterpret_cast<const float4*>(p0) + k);
        tot[4 * k] = v.x; tot[4 * k + 1] = v.y; tot[4 * k + 2] = v.z; tot[4 * k + 3] = v.w;
      }
      for (int j = 1; j < s.nseg; ++j) {
        const float4* pj = reinterpret_cast<const float4*>(p0 + (int64_t)j * HD);
#pragma unroll
        for (int k = 0; k < VPL / 4; ++k) {
          const float4 v = __ldcg(pj + k);
          tot[4 * k] = __fadd_rn(tot[4 * k], v.x); tot[4 * k + 1] = __fadd_rn(tot[4 * k + 1], v.y);
          tot[4 * k + 2] = __fadd_rn(tot[4 * k + 2], v.z); tot[4 * k + 3] = __fadd_rn(tot[4 * k + 3], v.w);
        }
      }
    }
    float4* dst = reinterpret_cast<float4*>(a.Hout + s.vl * HD + lane * VPL);
#pragma unroll
    for (int k = 0; k < VPL / 4; ++k) {
      float o[4];
#pragma unroll
      for (int z = 0; z < 4; ++z) {
        o[z] = __fmul_rn(tot[4 * k + z], scH.s);
        amax_loc = fmaxf(amax_loc, fabsf(o[z]));
      }
      __stcs(dst + k, make_float4(o[0], o[1], o[2], o[3]));
    }
  }
  amax_flush(a.amax_out, amax_loc);
}

// ================================================================== F-agg, hub rows: segment pieces
// A hub row (degree > C_E) is cut into its canonical chunks.  A row of at most SPIECE chunks (the common hub
// on Reddit-like graphs) is one warp item that folds its chunk partials itself in registers (total = p_0,
// total = total + p_c) and writes no partials; a longer row is spread chunk by chunk over warps whose
// partials go to scratch, and the row's last finishing item folds them in chunk order — the same
// left-to-right fold as the oracle's Σᶜ.
constexpr int SPIECE = 4;

// groups of one piece: 8 edges; a chunk boundary can only fall on a group start when C_E % 8 == 0 (the
// FAST form); other C_E (parity tests use 3, 7, 64 ...) check every edge
template <int VPL>
struct PieceFold {
  float tot[VPL];
  int nfold;
  __device__ __forceinline__ void fold(float2 (&acc)[VPL / 2]) {
#pragma unroll
    for (int k = 0; k < VPL / 2; ++k) {
      tot[2 * k] = nfold == 0 ? acc[k].x : __fadd_rn(tot[2 * k], acc[k].x);
      tot[2 * k + 1] = nfold == 0 ? acc[k].y : __fadd_rn(tot[2 * k + 1], acc[k].y);
      acc[k] = make_float2(0.0f, 0.0f);
    }
    ++nfold;
  }
};

template <int H, int VPL>
__host__ __device__ constexpr int fs_warp_smem_seg() {   // ring | α [2][H][32] | gather offsets [2][32]
  return g8_ring_bytes<VPL>() + 2 * H * 32 * 4 + 2 * 32 * 4;
}

// chunks in a row's piece 0: the whole row when it has at most SPIECE chunks (folded in registers, no
// partials), else the first chunk only (long rows stay spread over many warps)
__device__ __forceinline__ int piece0(int nseg) { return nseg <= SPIECE ? nseg : 1; }

// last item of a split hub row: fold piece 0's partial (slot base) with the partials of chunks
// 1 .. nseg-1 (slots base + c), in chunk order; every lane its VPL columns
template <int VPL>
__device__ __forceinline__ void fold_tail(const float* hagg, int64_t base, int nseg, float (&tot)[VPL]) {
  constexpr int HD = 32 * VPL;
  const float* p0 = hagg + base * HD + (threadIdx.x & 31) * VPL;
#pragma unroll
  for (int k = 0; k < VPL / 4; ++k) {
    const float4 v = __ldcg(reinterpret_cast<const float4*>(p0) + k);
    tot[4 * k] = v.x; tot[4 * k + 1] = v.y; tot[4 * k + 2] = v.z; tot[4 * k + 3] = v.w;
  }
  for (int j = 1; j < nseg; ++j) {
    const float4* pj = reinterpret_cast<const float4*>(p0 + (int64_t)j * HD);
#pragma unroll
    for (int k = 0; k < VPL / 4; ++k) {
      const float4 v = __ldcg(pj + k);
      tot[4 * k] = __fadd_rn(tot[4 * k], v.x); tot[4 * k + 1] = __fadd_rn(tot[4 * k + 1], v.y);
      tot[4 * k + 2] = __fadd_rn(tot[4 * k + 2], v.z); tot[4 * k + 3] = __fadd_rn(tot[4 * k + 3], v.w);
    }
  }
}
template <int VPL>
__device__ __forceinline__ void store_partial(float* dst_row, const float* x) {
  float4* d = reinterpret_cast<float4*>(dst_row + (threadIdx.x & 31) * VPL);
#pragma unroll
  for (int k = 0; k < VPL / 4; ++k) __stcg(d + k, make_float4(x[4 * k], x[4 * k + 1], x[4 * k + 2], x[4 * k + 3]));
}
// true for the warp whose item completes a split row (nseg > SPIECE: one item per chunk)
__device__ __forceinline__ bool piece_last(int32_t* cnt, int64_t row, int nseg) { return seg_last(cnt, row, nseg); }

template <int H, int VPL>
__global__ void __launch_bounds__(256, 3) k2_fagg_seg(const G2Args a) {
  constexpr int HD = 32 * VPL, WS = fs_warp_smem_seg<H, VPL>();
  extern __shared__ __align__(16) uint8_t dsm[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int myh = lane / (32 / H);
  uint8_t* wsm = dsm + w * ((WS + 15) & ~15);
  float* sa = reinterpret_cast<float*>(wsm + g8_ring_bytes<VPL>());   // [2][H][32]
  int* sidx = reinterpret_cast<int*>(sa + 2 * H * 32);                // [2][32]
  const uint32_t ring_lane = smem_u32(wsm) + lane * VPL;
  const int8_t* lane_base = a.qHp + lane * VPL;
  const uint32_t ld32 = (uint32_t)a.ldHp;
  const uint64_t pol = l2_evict_last();
  const Scale scH = scale_from_amax(amax_load(a.amax_Hp), a.bits);
  const Scale scS = scale_from_amax(amax_load(a.amax_S), a.bits);
  const Scale scD = scale_from_amax(amax_load(a.amax_D), a.bits);
  const int64_t hc = load_count(a.pin.counts);
  const int C = a.g.chunk;
  const bool fast = (C % GR) == 0;
  float amax_loc = 0.0f;
  FOR_ITEMS(si, a.work + 1, hc) {
    Seg s;
    decode_item(si, hc, a.g.in_ptr, a.pin, a.g.chunk, s);
    const int k0 = piece0(s.nseg);
    if (s.c > 0 && s.c < k0) continue;                // part of the row's piece 0
    const int kseg = s.c == 0 ? k0 : 1;
    const int64_t rend = a.g.in_ptr[s.vl + 1];
    const int64_t eb = s.eb, ee = eb + (int64_t)kseg * C < rend ? eb + (int64_t)kseg * C : rend;
    const int T = (int)(ee - eb);
    const DstSm<H> d = load_dst<H>(a, a.g.row_begin + s.vl);
    auto alpha_of = [&](int c, const int8_t (&qs)[H], float (&al)[H]) {
#pragma unroll
      for (int h = 0; h < H; ++h) al[h] = 0.0f;
      if (c * 32 + lane < T) {
        float ep[H];
        alpha_rec<H>(qs, d, scS.s, scD.s, a.slope, ep, al);
        if (a.alpha_st) store_alpha<H>(a.alpha_st + (eb + c * 32 + lane) * H, al, ep);
      }
    };
    auto stash = [&](int c, const float (&al)[H]) {
      const int b = c & 1;
#pragma unroll
      for (int h = 0; h < H; ++h) sa[(b * H + h) * 32 + lane] = al[h];
    };
    auto edge_u = [&](int c) -> int { return c * 32 + lane < T ? __ldcs(a.g.in_src + eb + c * 32 + lane) : 0; };
    const int nch = (T + 31) >> 5, ng = (T + GR - 1) / GR;
    int u1;
    {
      const int u0 = edge_u(0);
      int8_t qs0[H];
      load_qh<H>(a.qS + (int64_t)u0 * H, qs0);
      float al0[H];
      alpha_of(0, qs0, al0);
      stash(0, al0);
      sidx[lane] = u0;
      u1 = edge_u(1);
      sidx[32 + lane] = u1;
    }
    __syncwarp();
    g8_fill<VPL>(ring_lane, lane_base, ld32, sidx, 0, true, pol);
    g8_fill<VPL>(ring_lane, lane_base, ld32, sidx, 1, 1 < ng, pol);
    float2 acc[VPL / 2];
#pragma unroll
    for (int k = 0; k < VPL / 2; ++k) acc[k] = make_float2(0.0f, 0.0f);
    PieceFold<VPL> pf;
    pf.nfold = 0;
    int nextf = C;   // next chunk boundary of the piece (FAST form: group starts only)
    for (int c = 0; c < nch; ++c) {
      const int u2 = edge_u(c + 2);
      int8_t qs1[H];
      load_qh<H>(a.qS + (int64_t)u1 * H, qs1);
      const float* sac = sa + ((c & 1) * H + myh) * 32;
      for (int i0 = 0; i0 < 32; i0 += GR) {
        const int t0 = c * 32 + i0;
        if (t0 >= T) break;
        const int g = t0 / GR;
        cp_wait<1>();
        const uint32_t s0 = ring_lane + (uint32_t)(g & 1) * (GR * 32 * VPL);
        const float4 a4 = *reinterpret_cast<const float4*>(sac + i0);
        const float4 b4 = *reinterpret_cast<const float4*>(sac + i0 + 4);
        const float al[GR] = {a4.x, a4.y, a4.z, a4.w, b4.x, b4.y, b4.z, b4.w};
        if (fast) {
          if (t0 == nextf) {
            pf.fold(acc);
            nextf += C;
          }
#pragma unroll
          for (int j = 0; j < GR; ++j) {
            const Row<VPL> rj = lds_row_slice<VPL>(s0 + j * 32 * VPL);
            const float2 al2 = make_float2(al[j], al[j]);
#pragma unroll
            for (int q = 0; q < VPL / 4; ++q) fma4_biased(rj.w[q], al2, acc[2 * q], acc[2 * q + 1]);
          }
        } else {
#pragma unroll
          for (int j = 0; j < GR; ++j) {
            if (t0 + j > 0 && t0 + j < T && (t0 + j) % C == 0) pf.fold(acc);
            const Row<VPL> rj = lds_row_slice<VPL>(s0 + j * 32 * VPL);
            const float2 al2 = make_float2(al[j], al[j]);
#pragma unroll
            for (int q = 0; q < VPL / 4; ++q) fma4_biased(rj.w[q], al2, acc[2 * q], acc[2 * q + 1]);
          }
        }
        g8_fill<VPL>(ring_lane, lane_base, ld32, sidx, g + 2, g + 2 < ng, pol);
      }
      __syncwarp();
      if (c + 1 < nch) {
        float al1[H];
        alpha_of(c + 1, qs1, al1);
        stash(c + 1, al1);
        sidx[(c & 1) * 32 + lane] = u2;
      }
      __syncwarp();
      u1 = u2;
    }
    pf.fold(acc);   // the last chunk's partial
    float* out_row = nullptr;
    if (s.nseg <= SPIECE) {
      out_row = a.Hout + s.vl * HD;   // the whole row in this piece
    } else {
      store_partial<VPL>(a.hagg + (int64_t)(s.c == 0 ? s.base : s.base + s.c) * HD, pf.tot);
      if (!piece_last(a.hcnt, s.vl, s.nseg)) continue;
      fold_tail<VPL>(a.hagg, s.base, s.nseg, pf.tot);
      out_row = a.Hout + s.vl * HD;
    }
    float4* dst = reinterpret_cast<float4*>(out_row + lane * VPL);
#pragma unroll
    for (int k = 0; k < VPL / 4; ++k) {
      float o[4];
#pragma unroll
      for (int z = 0; z < 4; ++z) {
        o[z] = __fmul_rn(pf.tot[4 * k + z], scH.s);
        amax_loc = fmaxf(amax_loc, fabsf(o[z]));
      }
      __stcs(dst + k, make_float4(o[0], o[1], o[2], o[3]));
    }
  }
  amax_flush(a.amax_out, amax_loc);
}

// ================================================================== P1: source rows, ⑤′ + ⑤″
// Per out-edge e' = (u → v): gather q_G[v] (excess-128 codes); ∂α[e'] = i2f(q_G[v]·q_H′[u])·s_G s_H′ (u's
// row in registers as plain codes, exact IDP4A dot + 4-edge transposed reduction); acc += α·q_G[v] with α
// recomputed.  ∂α is written in out-CSR order (dal_out, coalesced; the destination pass P2 reads it through
// the in-CSR -> out-CSR position map).  Rows: ∂H′_agg = acc·s_G into dHp (finalized by P3).
template <int H, int VPL>
__host__ __device__ constexpr int bs_warp_smem() {
  // ring | α [2][H][32] | rows [2][32] | out-CSR slots [2][32] | ∂α [H][32] | tile rows
  return g8_ring_bytes<VPL>() + 2 * H * 32 * 4 + 2 * 2 * 32 * 4 + H * 32 * 4 + 2 * 32;
}
template <int H, int VPL, int NW>
__global__ void __launch_bounds__(NW * 32, 20 / NW) k2_bsrc1(const G2Args a) {
  constexpr int HD = 32 * VPL, LPH = 32 / H, WS = bs_warp_smem<H, VPL>();
  extern __shared__ __align__(16) uint8_t dsm[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int myh = lane / LPH;
  uint8_t* wsm = dsm + w * ((WS + 15) & ~15);
  float* sa = reinterpret_cast<float*>(wsm + g8_ring_bytes<VPL>());   // [2][H][32] α
  int* sidx = reinterpret_cast<int*>(sa + 2 * H * 32);                // [2][32] gather rows (v)
  int* seo = sidx + 64;                                               // [2][32] out-CSR position
  float* sd = reinterpret_cast<float*>(seo + 64);                     // [H][32] ∂α of the chunk
  uint8_t* srow = reinterpret_cast<uint8_t*>(sd + H * 32);           // [2][32]
  const uint32_t ring_lane = smem_u32(wsm) + lane * VPL;
  const int8_t* lane_base = a.qG + lane * VPL;
  const uint32_t ld32 = (uint32_t)a.ldG;
  const uint64_t pol = l2_evict_last();
  const Scale scH = scale_from_amax(amax_load(a.amax_Hp), a.bits);
  const Scale scG = scale_from_amax(amax_load(a.amax_G), a.bits);
  const Scale scS = scale_from_amax(amax_load(a.amax_S), a.bits);
  const Scale scD = scale_from_amax(amax_load(a.amax_D), a.bits);
  const float sGH = __fmul_rn(scG.s, scH.s);
  const int64_t n = a.g.n_local, hc = load_count(a.pout.counts);
  const int64_t nitems = hc + load_count(a.pout.counts + 2);
  const int8_t* obase = a.qHp + lane * VPL;      // own: q_H′[u] (excess-128 -> flipped to plain)
  FOR_ITEMS(it, a.work + 7, nitems - hc) {   // light sub-tiles (hub rows: k2_bsrc1_seg)
    const int64_t item = hc + it;
    constexpr bool tile = true;
    Seg s;
    s.eb = 0; s.vl = 0; s.slot = -1; s.nseg = 1;
    TileCtx t;
    t.r0 = 0;
    if (!tile) {
      decode_item(item, hc, a.g.out_ptr, a.pout, a.g.chunk, s);
      t.T = (int)(s.ee - s.eb);
      t.L.eb = 0; t.L.off = 0; t.L.end = 0; t.L.deg = 0; t.L.light = false;
      t.r0 = s.vl;
    } else {
      const int32_t code = a.pout.tiles[item - hc];
      t.r0 = (int64_t)(code >> 10) * TILE;
      t.L = tile_setup(a.g.out_ptr, a.pout.hbase, t.r0, n, t.T, (code >> 5) & 31, (code & 31) + 1);
      unsigned zm = __ballot_sync(0xffffffffu, t.L.light && t.L.deg == 0);
      while (zm) {   // light rows without out-edges: ∂H′_agg = 0
        const int j = __ffs(zm) - 1;
        zm &= zm - 1;
        float4* dst = reinterpret_cast<float4*>(a.dHp + (t.r0 + j) * HD + lane * VPL);
#pragma unroll
        for (int k = 0; k < VPL / 4; ++k) dst[k] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
      }
    }
    const int T = t.T;
    if (T == 0) continue;
    const int64_t ug0 = a.g.row_begin + t.r0;
    int qsj[H];   // own row's q_S (tile lane j: row j; segment: the row)
    {
      const int64_t ugl = tile ? ug0 + lane : ug0;
      const bool ok = tile ? t.L.light : true;
#pragma unroll
      for (int h = 0; h < H; ++h) qsj[h] = ok ? (int)a.qS[ugl * H + h] : 0;
    }
    auto pos_of = [&](int c, int& row) -> int64_t {
      const int pos = c * 32 + lane;
      if (tile) return tile_edge(t, pos, row);
      row = 0;
      return s.eb + (pos < T ? pos : T - 1);
    };
    // attributes of a chunk: α (needs v's softmax data), in-CSR slot, out-CSR slot, tile row
    struct AttrIn { RecRaw<H> r; };
    auto attr_load = [&](int c, int v, int64_t e) {
      AttrIn x;
      (void)e;
      if (c * 32 + lane < T) x.r = load_rec_raw<H>(a, v);
      return x;
    };
    auto attrs = [&](int c, int row, const AttrIn& x, float (&al)[H], uint32_t& sg) {
      int8_t qs[H];
#pragma unroll
      for (int h = 0; h < H; ++h) qs[h] = (int8_t)(tile ? __shfl_sync(0xffffffffu, qsj[h], row) : qsj[h]);
#pragma unroll
      for (int h = 0; h < H; ++h) al[h] = 0.0f;
      sg = 0;
      if (c * 32 + lane < T) {
        float ep[H];
        alpha_rec<H>(qs, rec_unpack<H>(x.r), scS.s, scD.s, a.slope, ep, al);
        sg = ep_sign_bits<H>(ep);
      }
    };
    auto stash = [&](int c, int row, int64_t e, const float (&al)[H]) {
      const int b = c & 1;
#pragma unroll
      for (int h = 0; h < H; ++h) sa[(b * H + h) * 32 + lane] = al[h];
      srow[b * 32 + lane] = (uint8_t)row;
      seo[b * 32 + lane] = (int)e;
    };
    const int nch = (T + 31) >> 5, ng = (T + GR - 1) / GR;
    int row1, v1 = 0;
    uint32_t sg_cur = 0, sg_nxt = 0;   // LeakyReLU branch bits of the lane's edge of chunk c / c + 1
    int64_t e1;
    {
      int row0;
      const int64_t e0 = pos_of(0, row0);
      const int v0 = lane < T ? __ldcs(a.g.out_dst + e0) : 0;
      float al0[H];
      const AttrIn x0 = attr_load(0, v0, e0);
      attrs(0, row0, x0, al0, sg_cur);
      stash(0, row0, e0, al0);
      sidx[lane] = v0;
      e1 = pos_of(1, row1);
      if (32 + lane < T) v1 = __ldcs(a.g.out_dst + e1);
      sidx[32 + lane] = v1;
    }
    __syncwarp();
    g8_fill<VPL>(ring_lane, lane_base, ld32, sidx, 0, true, pol);
    g8_fill<VPL>(ring_lane, lane_base, ld32, sidx, 1, 1 < ng, pol);
    // own q_H′[u] slice per row (plain codes + their sum for the excess-128 dot), prefetched a row ahead
    const unsigned act = tile ? __ballot_sync(0xffffffffu, t.L.deg > 0) : 1u;
    int nxt = act ? __ffs(act) - 1 : -1;
    Row<VPL> ow{}, ow_nxt{};
    int osum = 0;
    if (nxt >= 0) ow_nxt = load_row<VPL>(obase + (ug0 + nxt) * a.ldHp);
    int cur = -1;
    if (!tile) {
      cur = 0;
      ow = ow_nxt;
      osum = row_sum_plain<VPL>(ow, true);
    }
    float2 acc[VPL / 2];
#pragma unroll
    for (int k = 0; k < VPL / 2; ++k) acc[k] = make_float2(0.0f, 0.0f);
    auto flush = [&](int j) {   // tile row j done: ∂H′_agg = acc · s_G
      float4* dst = reinterpret_cast<float4*>(a.dHp + (t.r0 + j) * HD + lane * VPL);
      const float2 s2 = make_float2(scG.s, scG.s);
#pragma unroll
      for (int k = 0; k < VPL / 4; ++k) {
        const float2 o01 = __fmul2_rn(acc[2 * k], s2), o23 = __fmul2_rn(acc[2 * k + 1], s2);
        dst[k] = make_float4(o01.x, o01.y, o23.x, o23.y);
        acc[2 * k] = make_float2(0.0f, 0.0f);
        acc[2 * k + 1] = make_float2(0.0f, 0.0f);
      }
    };
    auto row_change = [&](int rj) {
      if (cur >= 0) flush(cur);
      cur = rj;
      ow = ow_nxt;
      osum = row_sum_plain<VPL>(ow, true);
      nxt = tile_next(act, cur);
      if (nxt >= 0) ow_nxt = load_row<VPL>(obase + (ug0 + nxt) * a.ldHp);
    };
    for (int c = 0; c < nch; ++c) {
      int row2;
      const int64_t e2 = pos_of(c + 2, row2);
      const int v2 = (c + 2) * 32 + lane < T ? __ldcs(a.g.out_dst + e2) : 0;
      const AttrIn x1 = attr_load(c + 1, v1, e1);
      const int b = c & 1;
      const int ein = (a.rec && c * 32 + lane < T) ? __ldcs(a.g.out_eid + seo[b * 32 + lane]) : 0;
      const float* sac = sa + (b * H + myh) * 32;
      for (int i0 = 0; i0 < 32; i0 += GR) {
        const int t0 = c * 32 + i0;
        if (t0 >= T) break;
        const int g = t0 / GR;
        cp_wait<1>();
        const uint32_t s0 = ring_lane + (uint32_t)(g & 1) * (GR * 32 * VPL);
        const float4 a4 = *reinterpret_cast<const float4*>(sac + i0);
        const float4 b4 = *reinterpret_cast<const float4*>(sac + i0 + 4);
        const float al[GR] = {a4.x, a4.y, a4.z, a4.w, b4.x, b4.y, b4.z, b4.w};
        int d[GR];
        bool same = true;
        uint32_t rw0 = 0, rw1 = 0;
        if (tile) {
          rw0 = *reinterpret_cast<const uint32_t*>(srow + b * 32 + i0);
          rw1 = *reinterpret_cast<const uint32_t*>(srow + b * 32 + i0 + 4);
          same = (int)(rw0 & 0xffu) == cur && (int)(rw1 >> 24) == cur;
        }
        if (same) {
#pragma unroll
          for (int j = 0; j < GR; ++j) {
            const Row<VPL> rj = lds_row_slice<VPL>(s0 + j * 32 * VPL);
            d[j] = row_dot_biased<VPL>(rj, ow, osum);
            const float2 al2 = make_float2(al[j], al[j]);
#pragma unroll
            for (int q = 0; q < VPL / 4; ++q) fma4_biased(rj.w[q], al2, acc[2 * q], acc[2 * q + 1]);
          }
        } else {
#pragma unroll
          for (int j = 0; j < GR; ++j) {
            const int rowj = (int)(((j < 4 ? rw0 : rw1) >> (8 * (j & 3))) & 0xffu);
            if (rowj != cur) row_change(rowj);
            const Row<VPL> rj = lds_row_slice<VPL>(s0 + j * 32 * VPL);
            d[j] = row_dot_biased<VPL>(rj, ow, osum);
            const float2 al2 = make_float2(al[j], al[j]);
#pragma unroll
            for (int q = 0; q < VPL / 4; ++q) fma4_biased(rj.w[q], al2, acc[2 * q], acc[2 * q + 1]);
          }
        }
        {
          int k;
          const int d0[4] = {d[0], d[1], d[2], d[3]}, d1[4] = {d[4], d[5], d[6], d[7]};
          const int x0 = group_dot_reduce<LPH>(d0, k);
          const int x1 = group_dot_reduce<LPH>(d1, k);
          sd[myh * 32 + i0 + k] = __fmul_rn(__int2float_rn(x0), sGH);
          sd[myh * 32 + i0 + 4 + k] = __fmul_rn(__int2float_rn(x1), sGH);
        }
        g8_fill<VPL>(ring_lane, lane_base, ld32, sidx, g + 2, g + 2 < ng, pol);
      }
      __syncwarp();
      if (c * 32 + lane < T) {   // ∂α of this chunk: out-CSR order (coalesced) and the edge's in-CSR slot
        float o[H];
#pragma unroll
        for (int h = 0; h < H; ++h) o[h] = sd[h * 32 + lane];
        if constexpr (H == 4)
          __stcs(reinterpret_cast<float4*>(a.dal_out + (int64_t)seo[b * 32 + lane] * H), make_float4(o[0], o[1], o[2], o[3]));
        else
          st_h<H>(a.dal_out + (int64_t)seo[b * 32 + lane] * H, o);
        if (a.scatter_in) st_h<H>(a.dal_in + (int64_t)__ldcs(a.g.out_eid + seo[b * 32 + lane]) * H, o);
        if (a.rec) put_rec<H>(a.rec, ein, o, sa + b * H * 32 + lane, sg_cur);
        if (a.al_out) put_alpha<H>(a.al_out + (int64_t)seo[b * 32 + lane] * H, sa + b * H * 32 + lane, sg_cur);

      }
      __syncwarp();
      if (c + 1 < nch) {
        float al1[H];
        attrs(c + 1, row1, x1, al1, sg_nxt);
        sg_cur = sg_nxt;
        stash(c + 1, row1, e1, al1);
        sidx[b * 32 + lane] = v2;
      }
      __syncwarp();
      v1 = v2; e1 = e2; row1 = row2;
    }
    if (tile) {
      if (cur >= 0) flush(cur);
      continue;
    }
    {
      float4* dst = reinterpret_cast<float4*>(a.hagg + (int64_t)s.slot * HD + lane * VPL);
#pragma unroll
      for (int k = 0; k < VPL / 4; ++k)
        __stcg(dst + k, make_float4(acc[2 * k].x, acc[2 * k].y, acc[2 * k + 1].x, acc[2 * k + 1].y));
    }
    if (!seg_last(a.hcnt, s.vl, s.nseg)) continue;
    float tot[VPL];
    {
      const float* p0 = a.hagg + (int64_t)s.base * HD + lane * VPL;
#pragma unroll
      for (int k = 0; k < VPL / 4; ++k) {
        const float4 v = __ldcg(reinterpret_cast<const float4*>(p0) + k);
        tot[4 * k] = v.x; tot[4 * k + 1] = v.y; tot[4 * k + 2] = v.z; tot[4 * k + 3] = v.w;
      }
      for (int j = 1; j < s.nseg; ++j) {
        const float4* pj = reinterpret_cast<const float4*>(p0 + (int64_t)j * HD);
#pragma unroll
        for (int k = 0; k < VPL / 4; ++k) {
          const float4 v = __ldcg(pj + k);
          tot[4 * k] = __fadd_rn(tot[4 * k], v.x); tot[4 * k + 1] = __fadd_rn(tot[4 * k + 1], v.y);
          tot[4 * k + 2] = __fadd_rn(tot[4 * k + 2], v.z); tot[4 * k + 3] = __fadd_rn(tot[4 * k + 3], v.w);
        }
      }
    }
    float4* dst = reinterpret_cast<float4*>(a.dHp + s.vl * HD + lane * VPL);
#pragma unroll
    for (int k = 0; k < VPL / 4; ++k)
      dst[k] = make_float4(__fmul_rn(tot[4 * k], scG.s), __fmul_rn(tot[4 * k + 1], scG.s),
                           __fmul_rn(tot[4 * k + 2], scG.s), __fmul_rn(tot[4 * k + 3], scG.s));
  }
}

// ================================================================== P1, hub rows: segment pieces
// As k2_fagg_seg for the source pass: piece 0 folds the row's first SPIECE out-CSR chunks in registers,
// further chunks write partials folded by the row's last item; u's own q_H′ row (the ⑤″ dot operand) is
// fixed for the whole piece, and the piece's ∂α are written coalesced at their out-CSR positions.
template <int H, int VPL>
__host__ __device__ constexpr int bs_warp_smem_seg() {   // ring | α [2][H][32] | rows [2][32] | ∂α [H][32]
  return g8_ring_bytes<VPL>() + 2 * H * 32 * 4 + 2 * 32 * 4 + H * 32 * 4;
}
template <int H, int VPL, int NW>
__global__ void __launch_bounds__(NW * 32, 20 / NW) k2_bsrc1_seg(const G2Args a) {
  constexpr int HD = 32 * VPL, LPH = 32 / H, WS = bs_warp_smem_seg<H, VPL>();
  extern __shared__ __align__(16) uint8_t dsm[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int myh = lane / LPH;
  uint8_t* wsm = dsm + w * ((WS + 15) & ~15);
  float* sa = reinterpret_cast<float*>(wsm + g8_ring_bytes<VPL>());   // [2][H][32] α
  int* sidx = reinterpret_cast<int*>(sa + 2 * H * 32);                // [2][32] gather rows (v)
  float* sd = reinterpret_cast<float*>(sidx + 64);                    // [H][32] ∂α of the chunk
  const uint32_t ring_lane = smem_u32(wsm) + lane * VPL;
  const int8_t* lane_base = a.qG + lane * VPL;
  const uint32_t ld32 = (uint32_t)a.ldG;
  const uint64_t pol = l2_evict_last();
  const Scale scH = scale_from_amax(amax_load(a.amax_Hp), a.bits);
  const Scale scG = scale_from_amax(amax_load(a.amax_G), a.bits);
  const Scale scS = scale_from_amax(amax_load(a.amax_S), a.bits);
  const Scale scD = scale_from_amax(amax_load(a.amax_D), a.bits);
  const float sGH = __fmul_rn(scG.s, scH.s);
  const int64_t hc = load_count(a.pout.counts);
  const int C = a.g.chunk;
  const bool fast = (C % GR) == 0;
  FOR_ITEMS(si, a.work + 2, hc) {
    Seg s;
    decode_item(si, hc, a.g.out_ptr, a.pout, a.g.chunk, s);
    const int k0 = piece0(s.nseg);
    if (s.c > 0 && s.c < k0) continue;
    const int kseg = s.c == 0 ? k0 : 1;
    const int64_t rend = a.g.out_ptr[s.vl + 1];
    const int64_t eb = s.eb, ee = eb + (int64_t)kseg * C < rend ? eb + (int64_t)kseg * C : rend;
    const int T = (int)(ee - eb);
    const int64_t ug = a.g.row_begin + s.vl;
    int8_t qs[H];
    load_qh<H>(a.qS + ug * H, qs);
    Row<VPL> ow = load_row<VPL>(a.qHp + ug * a.ldHp + lane * VPL);
    int osum_h = row_sum_plain<VPL>(ow, true);   // -> Σ of the head's plain own codes (all its lanes)
#pragma unroll
    for (int o = LPH / 2; o > 0; o >>= 1) osum_h += __shfl_xor_sync(0xffffffffu, osum_h, o);
    auto edge_v = [&](int c) -> int { return c * 32 + lane < T ? __ldcs(a.g.out_dst + eb + c * 32 + lane) : 0; };
    auto alpha_of = [&](int c, const DstSm<H>& d, float (&al)[H], uint32_t& sg) {
#pragma unroll
      for (int h = 0; h < H; ++h) al[h] = 0.0f;
      sg = 0;
      if (c * 32 + lane < T) {
        float ep[H];
        alpha_rec<H>(qs, d, scS.s, scD.s, a.slope, ep, al);
        sg = ep_sign_bits<H>(ep);
      }
    };
    auto stash = [&](int c, const float (&al)[H]) {
      const int b = c & 1;
#pragma unroll
      for (int h = 0; h < H; ++h) sa[(b * H + h) * 32 + lane] = al[h];
    };
    const int nch = (T + 31) >> 5, ng = (T + GR - 1) / GR;
    int v1;
    uint32_t sg_cur = 0, sg_nxt = 0;   // LeakyReLU branch bits of the lane's edge of chunk c / c + 1
    {
      const int v0 = edge_v(0);
      DstSm<H> d0;
      if (lane < T) d0 = load_rec<H>(a, v0);
      float al0[H];
      alpha_of(0, d0, al0, sg_cur);
      stash(0, al0);
      sidx[lane] = v0;
      v1 = edge_v(1);
      sidx[32 + lane] = v1;
    }
    __syncwarp();
    g8_fill<VPL>(ring_lane, lane_base, ld32, sidx, 0, true, pol);
    g8_fill<VPL>(ring_lane, lane_base, ld32, sidx, 1, 1 < ng, pol);
    float2 acc[VPL / 2];
#pragma unroll
    for (int k = 0; k < VPL / 2; ++k) acc[k] = make_float2(0.0f, 0.0f);
    PieceFold<VPL> pf;
    pf.nfold = 0;
    int nextf = C;   // next chunk boundary of the piece (FAST form: group starts only)
    for (int c = 0; c < nch; ++c) {
      const int v2 = edge_v(c + 2);
      RecRaw<H> r1;
      if ((c + 1) * 32 + lane < T) r1 = load_rec_raw<H>(a, v1);
      // in-CSR slot of this chunk's edge (scatter of ∂α), loaded here so the store at the chunk end does not wait
      const int ein = ((a.scatter_in || a.rec) && c * 32 + lane < T) ? __ldcs(a.g.out_eid + eb + c * 32 + lane) : 0;
      const float* sac = sa + ((c & 1) * H + myh) * 32;
      for (int i0 = 0; i0 < 32; i0 += GR) {
        const int t0 = c * 32 + i0;
        if (t0 >= T) break;
        const int g = t0 / GR;
        cp_wait<1>();
        const uint32_t s0 = ring_lane + (uint32_t)(g & 1) * (GR * 32 * VPL);
        const float4 a4 = *reinterpret_cast<const float4*>(sac + i0);
        const float4 b4 = *reinterpret_cast<const float4*>(sac + i0 + 4);
        const float al[GR] = {a4.x, a4.y, a4.z, a4.w, b4.x, b4.y, b4.z, b4.w};
        int dd[GR];
        // per edge: the lane's raw IDP4A sum on excess-128 codes; the −128·Σq_H′ correction is applied once
        // per edge after the reduction over the head's lanes (osum_h: the head's Σ of plain own codes)
        if (fast) {
          if (t0 == nextf) {
            pf.fold(acc);
            nextf += C;
          }
#pragma unroll
          for (int j = 0; j < GR; ++j) {
            const Row<VPL> rj = lds_row_slice<VPL>(s0 + j * 32 * VPL);
            dd[j] = row_dot_raw<VPL>(rj, ow);
            const float2 al2 = make_float2(al[j], al[j]);
#pragma unroll
            for (int q = 0; q < VPL / 4; ++q) fma4_biased(rj.w[q], al2, acc[2 * q], acc[2 * q + 1]);
          }
        } else {
#pragma unroll
          for (int j = 0; j < GR; ++j) {
            if (t0 + j > 0 && t0 + j < T && (t0 + j) % C == 0) pf.fold(acc);
            const Row<VPL> rj = lds_row_slice<VPL>(s0 + j * 32 * VPL);
            dd[j] = row_dot_raw<VPL>(rj, ow);
            const float2 al2 = make_float2(al[j], al[j]);
#pragma unroll
            for (int q = 0; q < VPL / 4; ++q) fma4_biased(rj.w[q], al2, acc[2 * q], acc[2 * q + 1]);
          }
        }
        {
          int k;
          const int d0[4] = {dd[0], dd[1], dd[2], dd[3]}, d1x[4] = {dd[4], dd[5], dd[6], dd[7]};
          const int x0 = group_dot_reduce<LPH>(d0, k) - 128 * osum_h;
          const int x1 = group_dot_reduce<LPH>(d1x, k) - 128 * osum_h;
          sd[myh * 32 + i0 + k] = __fmul_rn(__int2float_rn(x0), sGH);
          sd[myh * 32 + i0 + 4 + k] = __fmul_rn(__int2float_rn(x1), sGH);
        }
        g8_fill<VPL>(ring_lane, lane_base, ld32, sidx, g + 2, g + 2 < ng, pol);
      }
      __syncwarp();
      if (c * 32 + lane < T) {   // ∂α of this chunk at its out-CSR positions (coalesced)
        float o[H];
#pragma unroll
        for (int h = 0; h < H; ++h) o[h] = sd[h * 32 + lane];
        float4 o4;
        if constexpr (H == 4) {
          o4 = make_float4(o[0], o[1], o[2], o[3]);
          __stcs(reinterpret_cast<float4*>(a.dal_out + (eb + c * 32 + lane) * H), o4);
        } else {
          st_h<H>(a.dal_out + (eb + c * 32 + lane) * H, o);
        }
        if (a.scatter_in) st_h<H>(a.dal_in + (int64_t)ein * H, o);
        if (a.rec) put_rec<H>(a.rec, ein, o, sa + (c & 1) * H * 32 + lane, sg_cur);
        if (a.al_out) put_alpha<H>(a.al_out + (eb + c * 32 + lane) * H, sa + (c & 1) * H * 32 + lane, sg_cur);
      }
      __syncwarp();
      if (c + 1 < nch) {
        float al1[H];
        const DstSm<H> d1 = rec_unpack<H>(r1);
        alpha_of(c + 1, d1, al1, sg_nxt);
        sg_cur = sg_nxt;
        stash(c + 1, al1);
        sidx[(c & 1) * 32 + lane] = v2;
      }
      __syncwarp();
      v1 = v2;
    }
    pf.fold(acc);
    if (s.nseg > SPIECE) {
      store_partial<VPL>(a.hagg + (int64_t)(s.c == 0 ? s.base : s.base + s.c) * HD, pf.tot);
      if (!piece_last(a.hcnt, s.vl, s.nseg)) continue;
      fold_tail<VPL>(a.hagg, s.base, s.nseg, pf.tot);
    }
    float4* dst = reinterpret_cast<float4*>(a.dHp + s.vl * HD + lane * VPL);
#pragma unroll
    for (int k = 0; k < VPL / 4; ++k)
      dst[k] = make_float4(__fmul_rn(pf.tot[4 * k], scG.s), __fmul_rn(pf.tot[4 * k + 1], scG.s),
                           __fmul_rn(pf.tot[4 * k + 2], scG.s), __fmul_rn(pf.tot[4 * k + 3], scG.s));
  }
}

// ================================================================== P2: destination rows, ④′ + ③″
// P[v] = Σᶜ fmaf(∂α, α) over in-edges (in-CSR order), ∂E = α(∂α − P[v]), ∂E_pre = e_pre > 0 ? ∂E : ∂E·slope,
// ∂D[v] = Σᶜ ∂E_pre.  ∂α = dal_out[in2out[e]] (written by P1), α recomputed; P2a also stores the gathered ∂α
// of hub rows in in-CSR order (dal_in), so that P2b reads it coalesced.
// P2a: hub segments (P partials, folded by the row's last segment) and light sub-tiles (P and ∂D);
// P2b: hub segments (∂D partials with the row's P, folded likewise).
template <int H>
struct EdgeIn { int8_t qs[H]; float da[H], st[H]; };   // st: α stored by F-agg (sign = LeakyReLU branch)

// α and the branch from F-agg's stored signed α
template <int H>
__device__ __forceinline__ void alpha_from_st(const float (&st)[H], float (&ep)[H], float (&al)[H]) {
#pragma unroll
  for (int h = 0; h < H; ++h) {
    al[h] = fabsf(st[h]);
    ep[h] = signbit(st[h]) ? -1.0f : 1.0f;
  }
}

template <int H>
__global__ void __launch_bounds__(256, 3) k2_bdst_a(const G2Args a) {
  __shared__ float sbx[8][SB][H];
  __shared__ float sby[8][SB][H];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Scale scS = scale_from_amax(amax_load(a.amax_S), a.bits);
  const Scale scD = scale_from_amax(amax_load(a.amax_D), a.bits);
  const int64_t n = a.g.n_local, hc = load_count(a.pin.counts), nitems = hc + load_count(a.pin.counts + 2);
  FOR_ITEMS_FROM4(item, a.work + 3, a.hub_p2 ? hc : 0, nitems) {
    if (item < hc) {   // ---- hub segment: P partial (staged form; k2_bdst_a_hub(m) when hub_p2)
      Seg s;
      decode_item(item, hc, a.g.in_ptr, a.pin, a.g.chunk, s);
      const int64_t vg = a.g.row_begin + s.vl;
      const DstSm<H> d = load_dst<H>(a, vg);
      const float part = seg_partial<H, true>(
          s.eb, s.ee, sbx[w], sby[w],
          [&](int64_t e) {
            EdgeIn<H> l;
            if (a.rec) {   // P1's record: ∂α and signed α at the in-CSR slot
              ld_h<H>(a.rec + e * 2 * H, l.da);
              ld_h<H>(a.rec + e * 2 * H + H, l.st);
              return l;
            }
            if (a.alpha_st) ld_h<H>(a.alpha_st + e * H, l.st);
            else load_qh<H>(a.qS + (int64_t)a.g.in_src[e] * H, l.qs);
            if (a.scatter_in) {
              ld_h<H>(a.dal_in + e * H, l.da);   // scattered into in-CSR order by P1
            } else {
              ld_h<H>(a.dal_out + (int64_t)__ldcs(a.in2out + e) * H, l.da);
              st_h<H>(a.dal_in + e * H, l.da);   // ∂α in in-CSR order for P2b (coalesced)
            }
            return l;
          },
          [&](const EdgeIn<H>& l, float (&x)[H], float (&y)[H]) {
            float ep[H];
            if (a.alpha_st || a.rec) alpha_from_st<H>(l.st, ep, y);
            else alpha_rec<H>(l.qs, d, scS.s, scD.s, a.slope, ep, y);
#pragma unroll
            for (int h = 0; h < H; ++h) x[h] = l.da[h];
          });
      if (lane < H) __stcg(a.h1 + (int64_t)s.slot * H + lane, part);
      if (!seg_last(a.hcnt, s.vl, s.nseg)) continue;
      const float P = seg_fold<H>(a.h1, s.base, s.nseg);
      if (lane < H) {
        a.P[vg * H + lane] = P;
        rec_put1(a, vg, 2, lane, P);
      }
      continue;
    }
    // ---- light sub-tile: P and ∂D of its rows
    const int32_t code = a.pin.tiles[item - hc];
    TileCtx t;
    t.r0 = (int64_t)(code >> 10) * TILE;
    t.L = tile_setup(a.g.in_ptr, a.pin.hbase, t.r0, n, t.T, (code >> 5) & 31, (code & 31) + 1);
    const int64_t vgl = a.g.row_begin + t.L.r;
    float (*tbx)[H] = reinterpret_cast<float (*)[H]>(&sbx[w][0][0]);
    float (*tby)[H] = reinterpret_cast<float (*)[H]>(&sby[w][0][0]);
    DstSm<H> dj;
    if (t.L.light) dj = load_dst<H>(a, vgl);
    else {
#pragma unroll
      for (int h = 0; h < H; ++h) { dj.qd[h] = 0; dj.m[h] = 0.0f; dj.den[h] = 1.0f; }
    }
    auto edge_vals = [&](int pos, float (&da)[H], float (&al)[H], float (&ep)[H], int& row) {
      const int64_t e = tile_edge(t, pos, row);
      DstSm<H> d;
#pragma unroll
      for (int h = 0; h < H; ++h) {
        d.qd[h] = (int8_t)__shfl_sync(0xffffffffu, (int)dj.qd[h], row);
        d.m[h] = __shfl_sync(0xffffffffu, dj.m[h], row);
        d.den[h] = __shfl_sync(0xffffffffu, dj.den[h], row);
      }
      if (pos < t.T && a.rec) {
        float st[H];
        ld_h<H>(a.rec + e * 2 * H, da);
        ld_h<H>(a.rec + e * 2 * H + H, st);
        alpha_from_st<H>(st, ep, al);
      } else if (pos < t.T) {
        if (a.scatter_in) ld_h<H>(a.dal_in + e * H, da);
        else ld_h<H>(a.dal_out + (int64_t)__ldcs(a.in2out + e) * H, da);
        if (a.alpha_st) {
          float st[H];
          ld_h<H>(a.alpha_st + e * H, st);
          alpha_from_st<H>(st, ep, al);
        } else {
          int8_t qs[H];
          load_qh<H>(a.qS + (int64_t)a.g.in_src[e] * H, qs);
          alpha_rec<H>(qs, d, scS.s, scD.s, a.slope, ep, al);
        }
      }
    };
    float P[H], dD[H];
#pragma unroll
    for (int h = 0; h < H; ++h) { P[h] = 0.0f; dD[h] = 0.0f; }
    for (int base = 0; base < t.T; base += 32) {
      float da[H], al[H], ep[H];
      int row;
      edge_vals(base + lane, da, al, ep, row);
      if (base + lane < t.T)
#pragma unroll
        for (int h = 0; h < H; ++h) { tbx[lane][h] = da[h]; tby[lane][h] = al[h]; }
      __syncwarp();
      tile_fold<H, true>(t, base, tbx, tby, P);
      __syncwarp();
    }
    for (int base = 0; base < t.T; base += 32) {
      float da[H], al[H], ep[H];
      int row;
      edge_vals(base + lane, da, al, ep, row);
      float Pr[H];
#pragma unroll
      for (int h = 0; h < H; ++h) Pr[h] = __shfl_sync(0xffffffffu, P[h], row);
      if (base + lane < t.T)
#pragma unroll
        for (int h = 0; h < H; ++h) {
          const float dE = __fmul_rn(al[h], __fsub_rn(da[h], Pr[h]));
          tbx[lane][h] = ep[h] > 0.0f ? dE : __fmul_rn(dE, a.slope);
        }
      __syncwarp();
      tile_fold<H, false>(t, base, tbx, nullptr, dD);
      __syncwarp();
    }
    if (t.L.light) {
      st_h<H>(a.P + vgl * H, P);
      st_h<H>(a.dD + vgl * H, dD);
      rec_put<H>(a, vgl, 2, P);
    }
  }
}

template <int H>
__global__ void __launch_bounds__(256, 4) k2_bdst_b(const G2Args a) {
  __shared__ float sbx[8][SB][H];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Scale scS = scale_from_amax(amax_load(a.amax_S), a.bits);
  const Scale scD = scale_from_amax(amax_load(a.amax_D), a.bits);
  const int64_t hc = load_count(a.pin.counts);
  FOR_ITEMS4(si, a.work + 4, hc) {
    Seg s;
    decode_item(si, hc, a.g.in_ptr, a.pin, a.g.chunk, s);
    const int64_t vg = a.g.row_begin + s.vl;
    const DstSm<H> d = load_dst<H>(a, vg);
    float P[H];
    ld_h<H>(a.P + vg * H, P);
    const float part = seg_partial<H, false>(
        s.eb, s.ee, sbx[w], nullptr,
        [&](int64_t e) {
          EdgeIn<H> l;
          if (a.rec) {
            ld_h<H>(a.rec + e * 2 * H, l.da);
            ld_h<H>(a.rec + e * 2 * H + H, l.st);
            return l;
          }
          if (a.alpha_st) ld_h<H>(a.alpha_st + e * H, l.st);
          else load_qh<H>(a.qS + (int64_t)a.g.in_src[e] * H, l.qs);
          ld_h<H>(a.dal_in + e * H, l.da);
          return l;
        },
        [&](const EdgeIn<H>& l, float (&x)[H], float (&)[H]) {
          float ep[H], al[H];
          if (a.alpha_st || a.rec) alpha_from_st<H>(l.st, ep, al);
          else alpha_rec<H>(l.qs, d, scS.s, scD.s, a.slope, ep, al);
#pragma unroll
          for (int h = 0; h < H; ++h) {
            const float dE = __fmul_rn(al[h], __fsub_rn(l.da[h], P[h]));
            x[h] = ep[h] > 0.0f ? dE : __fmul_rn(dE, a.slope);
          }
        });
    if (lane < H) __stcg(a.h2 + (int64_t)s.slot * H + lane, part);
    if (!seg_last(a.hcnt, s.vl, s.nseg)) continue;
    const float dD = seg_fold<H>(a.h2, s.base, s.nseg);
    if (lane < H) a.dD[vg * H + lane] = dD;
  }
}

// ================================================================== P3: source rows, ③′ + ②′
// ∂S[u] = Σᶜ ∂E_pre over out-edges (out-CSR order), ∂E_pre recomputed from ∂α (dal_out), α, P[v]; then
// ∂H′[u] = (∂H′_agg[u] + ∂S·a_src) + ∂D[u]·a_dst in place over dHp (one warp per row), amax(∂H′).
template <int H, int VPL>
__device__ __forceinline__ void src_finalize_row(const G2Args& a, int64_t ul, const float (&dS)[H], float& amax_loc) {
  constexpr int HD = 32 * VPL, LPH = 32 / H;
  const int lane = threadIdx.x & 31;
  const int64_t ug = a.g.row_begin + ul;
  const int myh = lane / LPH;
  const float dSh = head_pick<H>(dS, myh);
  const float dD = a.dD[ug * H + myh];
  const int c0 = lane * VPL;
  float4* p = reinterpret_cast<float4*>(a.dHp + ul * HD + c0);
  const float4* as = reinterpret_cast<const float4*>(a.a_src + c0);
  const float4* ad = reinterpret_cast<const float4*>(a.a_dst + c0);
#pragma unroll
  for (int k = 0; k < VPL / 4; ++k) {
    const float4 g4 = p[k], s4 = __ldg(as + k), d4 = __ldg(ad + k);
    const float v[4] = {g4.x, g4.y, g4.z, g4.w}, sv[4] = {s4.x, s4.y, s4.z, s4.w}, dv[4] = {d4.x, d4.y, d4.z, d4.w};
    float o[4];
#pragma unroll
    for (int z = 0; z < 4; ++z) {
      const float t2 = __fadd_rn(v[z], __fmul_rn(dSh, sv[z]));
      o[z] = __fadd_rn(t2, __fmul_rn(dD, dv[z]));
      amax_loc = fmaxf(amax_loc, fabsf(o[z]));
    }
    p[k] = make_float4(o[0], o[1], o[2], o[3]);
  }
}

template <int H>
struct EdgeOut { int64_t e; int v; float da[H]; };

template <int H, int VPL>
__global__ void __launch_bounds__(256, 3) k2_bsrc2(const G2Args a) {
  __shared__ float sbx[8][SB][H];
  __shared__ float tS[8][32][H];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Scale scS = scale_from_amax(amax_load(a.amax_S), a.bits);
  const Scale scD = scale_from_amax(amax_load(a.amax_D), a.bits);
  const int64_t n = a.g.n_local, hc = load_count(a.pout.counts), nitems = hc + load_count(a.pout.counts + 2);
  float amax_loc = 0.0f;
  // ∂E_pre of out-edge e' = (u → v) with u's q_S; α from P1's out-CSR copy (al_out, signed) when present
  auto dEp = [&](int64_t e, int v, const float (&da)[H], const int8_t (&qs)[H], float (&x)[H]) {
    float ep[H], al[H], Pv[H];
    ld_h<H>(a.nrec + (int64_t)v * a.nrs + 2 * H, Pv);
    if (a.al_out) {
      float st[H];
      ld_h<H>(a.al_out + e * H, st);
      alpha_from_st<H>(st, ep, al);
    } else {
      const DstSm<H> d = load_rec<H>(a, v);
      alpha_rec<H>(qs, d, scS.s, scD.s, a.slope, ep, al);
    }
#pragma unroll
    for (int h = 0; h < H; ++h) {
      const float dE = __fmul_rn(al[h], __fsub_rn(da[h], Pv[h]));
      x[h] = ep[h] > 0.0f ? dE : __fmul_rn(dE, a.slope);
    }
  };
  FOR_ITEMS_FROM4(item, a.work + 6, a.hub_p3 ? hc : 0, nitems) {
    if (item < hc) {   // ---- hub segment: ∂S partial; the row's last segment folds and finalizes (staged form)
      Seg s;
      decode_item(item, hc, a.g.out_ptr, a.pout, a.g.chunk, s);
      const int64_t ug = a.g.row_begin + s.vl;
      int8_t qs[H];
      load_qh<H>(a.qS + ug * H, qs);
      const float part = seg_partial<H, false>(
          s.eb, s.ee, sbx[w], nullptr,
          [&](int64_t e) {
            EdgeOut<H> l;
            l.e = e;
            l.v = a.g.out_dst[e];
            ld_h<H>(a.dal_out + e * H, l.da);
            return l;
          },
          [&](const EdgeOut<H>& l, float (&x)[H], float (&)[H]) { dEp(l.e, l.v, l.da, qs, x); });
      if (lane < H) __stcg(a.hs + (int64_t)s.slot * H + lane, part);
      if (!seg_last(a.hcnt, s.vl, s.nseg)) continue;
      const float tot = seg_fold<H>(a.hs, s.base, s.nseg);
      float dS[H];
#pragma unroll
      for (int h = 0; h < H; ++h) dS[h] = __shfl_sync(0xffffffffu, tot, h);
      if (lane < H) a.dS[ug * H + lane] = tot;
      src_finalize_row<H, VPL>(a, s.vl, dS, amax_loc);
      continue;
    }
    // ---- light sub-tile
    const int32_t code = a.pout.tiles[item - hc];
    TileCtx t;
    t.r0 = (int64_t)(code >> 10) * TILE;
    t.L = tile_setup(a.g.out_ptr, a.pout.hbase, t.r0, n, t.T, (code >> 5) & 31, (code & 31) + 1);
    const int64_t ugl = a.g.row_begin + t.L.r;
    float (*tbx)[H] = reinterpret_cast<float (*)[H]>(&sbx[w][0][0]);
    int qsj[H];
#pragma unroll
    for (int h = 0; h < H; ++h) qsj[h] = t.L.light ? (int)a.qS[ugl * H + h] : 0;
    float dS[H];
#pragma unroll
    for (int h = 0; h < H; ++h) dS[h] = 0.0f;
    for (int base = 0; base < t.T; base += 32) {
      int row;
      const int64_t e = tile_edge(t, base + lane, row);
      int8_t qs[H];
#pragma unroll
      for (int h = 0; h < H; ++h) qs[h] = (int8_t)__shfl_sync(0xffffffffu, qsj[h], row);
      if (base + lane < t.T) {
        float da[H], x[H];
        ld_h<H>(a.dal_out + e * H, da);
        dEp(e, a.g.out_dst[e], da, qs, x);
#pragma unroll
        for (int h = 0; h < H; ++h) tbx[lane][h] = x[h];
      }
      __syncwarp();
      tile_fold<H, false>(t, base, tbx, nullptr, dS);
      __syncwarp();
    }
    if (t.L.light) st_h<H>(a.dS + ugl * H, dS);
#pragma unroll
    for (int h = 0; h < H; ++h) tS[w][lane][h] = dS[h];
    __syncwarp();
    const unsigned lm = __ballot_sync(0xffffffffu, t.L.light);   // finalize the light rows, a warp per row
    for (unsigned mm = lm; mm; mm &= mm - 1) {
      const int j = __ffs(mm) - 1;
      float dSj[H];
#pragma unroll
      for (int h = 0; h < H; ++h) dSj[h] = tS[w][j][h];
      src_finalize_row<H, VPL>(a, t.r0 + j, dSj, amax_loc);
    }
    __syncwarp();
  }
  amax_flush(a.amax_dHp, amax_loc);
}

// ================================================================== hub segments, one lane per (segment, head)
// The per-edge scalar passes over hub rows (F-stats Σ, P2's P and ∂D, P3's ∂S) as lane-parallel chunk sums: a
// warp claims SPW = 32/H consecutive hub segments (canonical chunks of C_E edges, reading R14) and lane
// L = k·H + h computes segment k's partial of head h sequentially in edge order, all 32 lanes busy (the
// staged form, seg_partial, sums on H lanes only).  Each group of H lanes stores its segment's partials
// (coalesced), and the group that completes a row (atomic count per row) folds the row's partials in chunk
// order (total = p_0, total = total + p_c) — the oracle's left-to-right Σᶜ.
struct LaneSeg {
  int64_t slot, row, eb, ee;
  int base, nseg;
  bool ok;
};
template <int H>
__device__ __forceinline__ LaneSeg lane_seg(int64_t first, int64_t hc, const int64_t* __restrict__ ptr,
                                            const PlanDev& p, int C) {
  LaneSeg s;
  s.slot = first + (threadIdx.x & 31) / H;
  s.ok = s.slot < hc;
  s.row = 0; s.eb = 0; s.ee = 0; s.base = 0; s.nseg = 1;
  if (s.ok) {
    s.row = p.hseg_row[s.slot];
    s.base = p.hbase[s.row];
    const int64_t beg = ptr[s.row], end = ptr[s.row + 1];
    s.nseg = (int)((end - beg + C - 1) / C);
    s.eb = beg + (s.slot - s.base) * (int64_t)C;
    s.ee = s.eb + C < end ? s.eb + C : end;
  }
  return s;
}
// after the group's partials are stored: true for the (whole) group whose segment completed its row; the
// row's counter is reset for the next pass.  Every lane of the warp must call it.
template <int H>
__device__ __forceinline__ bool lane_seg_last(int32_t* cnt, const LaneSeg& s) {
  const int lane = threadIdx.x & 31;
  __threadfence();
  int d = -1;
  if (s.ok && (lane % H) == 0) d = atomicAdd(cnt + s.row, 1);
  d = __shfl_sync(0xffffffffu, d, lane & ~(H - 1));
  const bool last = s.ok && d == s.nseg - 1;
  if (last) {
    __threadfence();
    if ((lane % H) == 0) cnt[s.row] = 0;
  }
  return last;
}
// chunk-order fold of the row's partials part[(base + j)·H + h], j = 0 .. nseg-1 (L2 reads)
template <int H>
__device__ __forceinline__ float lane_seg_fold(const float* part, const LaneSeg& s) {
  const int h = (threadIdx.x & 31) % H;
  const float* p = part + (int64_t)s.base * H + h;
  float tot = __ldcg(p);
  int j = 1;
  for (; j + 4 <= s.nseg; j += 4) {
    const float x0 = __ldcg(p + (int64_t)j * H), x1 = __ldcg(p + (int64_t)(j + 1) * H);
    const float x2 = __ldcg(p + (int64_t)(j + 2) * H), x3 = __ldcg(p + (int64_t)(j + 3) * H);
    tot = __fadd_rn(tot, x0); tot = __fadd_rn(tot, x1); tot = __fadd_rn(tot, x2); tot = __fadd_rn(tot, x3);
  }
  for (; j < s.nseg; ++j) tot = __fadd_rn(tot, __ldcg(p + (int64_t)j * H));
  return tot;
}
// Software pipeline over a lane's segment: the index loads of batch k+2 and the dependent loads of batch k+1
// are issued before batch k is used (in edge order), so both load latencies overlap the arithmetic.
// fi(e) -> I (independent loads of edge e), fd(I, e) -> D (loads that need I), fu(D) (the sequential use).
template <int U, typename I, typename D, typename FI, typename FD, typename FU>
__device__ __forceinline__ void lane_pipe(int64_t eb, int64_t ee, FI&& fi, FD&& fd, FU&& fu) {
  I ia[U], ib[U];
  D dc[U], dn[U];
#pragma unroll
  for (int j = 0; j < U; ++j)
    if (eb + j < ee) ia[j] = fi(eb + j);
#pragma unroll
  for (int j = 0; j < U; ++j)
    if (eb + j < ee) dc[j] = fd(ia[j], eb + j);
#pragma unroll
  for (int j = 0; j < U; ++j)
    if (eb + U + j < ee) ia[j] = fi(eb + U + j);
  for (int64_t e0 = eb; e0 < ee; e0 += U) {
#pragma unroll
    for (int j = 0; j < U; ++j)
      if (e0 + 2 * U + j < ee) ib[j] = fi(e0 + 2 * U + j);
#pragma unroll
    for (int j = 0; j < U; ++j)
      if (e0 + U + j < ee) dn[j] = fd(ia[j], e0 + U + j);
#pragma unroll
    for (int j = 0; j < U; ++j)
      if (e0 + j < ee) fu(dc[j]);
#pragma unroll
    for (int j = 0; j < U; ++j) {
      dc[j] = dn[j];
      ia[j] = ib[j];
    }
  }
}

// claim SPW segments per warp; the loop body sees `first` (the warp's first slot)
#define FOR_LANE_SEGS(first, counter, hc, SPW)                                                     \
  for (int64_t first = claim_n(counter, SPW); first < (hc); first = claim_n(counter, SPW))

__device__ __forceinline__ int64_t claim_n(int32_t* counter, int n) {
  int it = 0;
  if ((threadIdx.x & 31) == 0) it = atomicAdd(counter, n);
  return (int64_t)__shfl_sync(0xffffffffu, it, 0);
}

// ---- F-stats Σ over hub segments: den partial Σ exp_p(el − m), m from FS1's keys in the node record
template <int H>
__global__ void __launch_bounds__(256, 3) k2_fstats2_hub(const G2Args a) {
  constexpr int SPW = 32 / H;
  const int h = (threadIdx.x & 31) % H;
  const Scale scS = scale_from_amax(amax_load(a.amax_S), a.bits);
  const Scale scD = scale_from_amax(amax_load(a.amax_D), a.bits);
  const int64_t hc = load_count(a.pin.counts);
  FOR_LANE_SEGS(first, a.work + 8, hc, SPW) {
    const LaneSeg s = lane_seg<H>(first, hc, a.g.in_ptr, a.pin, a.g.chunk);
    const int64_t vg = a.g.row_begin + s.row;
    float m = 0.0f, acc = 0.0f;
    int qd = 0;
    if (s.ok) {
      m = fkey_dec(reinterpret_cast<const unsigned*>(a.nrec + vg * a.nrs)[h]);
      qd = a.qD[vg * H + h];
      lane_pipe<8, int, int>(
          s.eb, s.ee, [&](int64_t e) { return (int)__ldg(a.g.in_src + e); },
          [&](int u, int64_t) { return (int)a.qS[(int64_t)u * H + h]; },
          [&](int qs) {
            acc = __fadd_rn(acc, exp_p(__fsub_rn(lrelu(sddmm_add1((int8_t)qs, scS.s, (int8_t)qd, scD.s), a.slope), m)));
          });
      __stcg(a.h2 + s.slot * H + h, acc);
    }
    if (lane_seg_last<H>(a.hcnt, s)) {   // the row's m (as a float) and den; every segment has read the keys
      const float den = lane_seg_fold<H>(a.h2, s);
      a.m[vg * H + h] = m;
      rec_put1(a, vg, 0, h, m);
      a.den[vg * H + h] = den;
      rec_put1(a, vg, 1, h, den);
      reinterpret_cast<int8_t*>(a.nrec + vg * a.nrs + 3 * H)[h] = (int8_t)qd;
    }
  }
}

// α of one in-edge for head h: e_pre (③) and exp_p(lrelu(e_pre) − m) / den (④)
__device__ __forceinline__ float alpha1(int qs, int qd, float sS, float sD, float slope, float m, float den, float& ep) {
  ep = sddmm_add1((int8_t)qs, sS, (int8_t)qd, sD);
  return __fdiv_rn(exp_p(__fsub_rn(lrelu(ep, slope), m)), den);
}
struct UDa { int u; float da; };
struct QDa { int qs; float da; };

// ---- P2a over hub segments: P partial Σ fmaf(∂α, α); ∂α in in-CSR order (scattered there by P1), or gathered
// through the in2out map and stored in in-CSR order for P2b
template <int H>
__global__ void __launch_bounds__(256, 3) k2_bdst_a_hub(const G2Args a) {
  constexpr int SPW = 32 / H;
  const int h = (threadIdx.x & 31) % H;
  const Scale scS = scale_from_amax(amax_load(a.amax_S), a.bits);
  const Scale scD = scale_from_amax(amax_load(a.amax_D), a.bits);
  const int64_t hc = load_count(a.pin.counts);
  FOR_LANE_SEGS(first, a.work + 9, hc, SPW) {
    const LaneSeg s = lane_seg<H>(first, hc, a.g.in_ptr, a.pin, a.g.chunk);
    const int64_t vg = a.g.row_begin + s.row;
    if (s.ok) {
      const float m = a.m[vg * H + h], den = a.den[vg * H + h];
      const int qd = a.qD[vg * H + h];
      float acc = 0.0f;
      lane_pipe<4, UDa, QDa>(
          s.eb, s.ee,
          [&](int64_t e) {
            UDa x;
            x.u = __ldg(a.g.in_src + e);
            if (a.rec) {
              x.da = __ldcs(a.rec + e * 2 * H + h);
            } else if (a.scatter_in) {
              x.da = __ldcs(a.dal_in + e * H + h);
            } else {
              x.da = a.dal_out[(int64_t)__ldg(a.in2out + e) * H + h];
              a.dal_in[e * H + h] = x.da;   // for P2b (coalesced)
            }
            return x;
          },
          [&](const UDa& x, int64_t) { return QDa{(int)a.qS[(int64_t)x.u * H + h], x.da}; },
          [&](const QDa& y) {
            float ep;
            acc = __fmaf_rn(y.da, alpha1(y.qs, qd, scS.s, scD.s, a.slope, m, den, ep), acc);
          });
      __stcg(a.h1 + s.slot * H + h, acc);
    }
    if (lane_seg_last<H>(a.hcnt, s)) {
      const float P = lane_seg_fold<H>(a.h1, s);
      a.P[vg * H + h] = P;
      rec_put1(a, vg, 2, h, P);
    }
  }
}

// ---- P2b over hub segments: ∂D partial Σ ∂E_pre, ∂E_pre = α(∂α − P[v]) · lrelu′(e_pre)
template <int H>
__global__ void __launch_bounds__(256, 3) k2_bdst_b_hub(const G2Args a) {
  constexpr int SPW = 32 / H;
  const int h = (threadIdx.x & 31) % H;
  const Scale scS = scale_from_amax(amax_load(a.amax_S), a.bits);
  const Scale scD = scale_from_amax(amax_load(a.amax_D), a.bits);
  const int64_t hc = load_count(a.pin.counts);
  FOR_LANE_SEGS(first, a.work + 10, hc, SPW) {
    const LaneSeg s = lane_seg<H>(first, hc, a.g.in_ptr, a.pin, a.g.chunk);
    const int64_t vg = a.g.row_begin + s.row;
    if (s.ok) {
      const float m = a.m[vg * H + h], den = a.den[vg * H + h], P = a.P[vg * H + h];
      const int qd = a.qD[vg * H + h];
      float acc = 0.0f;
      lane_pipe<4, UDa, QDa>(
          s.eb, s.ee,
          [&](int64_t e) {
            return UDa{(int)__ldg(a.g.in_src + e), a.rec ? __ldcs(a.rec + e * 2 * H + h) : __ldcs(a.dal_in + e * H + h)};
          },
          [&](const UDa& x, int64_t) { return QDa{(int)a.qS[(int64_t)x.u * H + h], x.da}; },
          [&](const QDa& y) {
            float ep;
            const float al = alpha1(y.qs, qd, scS.s, scD.s, a.slope, m, den, ep);
            const float dE = __fmul_rn(al, __fsub_rn(y.da, P));
            acc = __fadd_rn(acc, ep > 0.0f ? dE : __fmul_rn(dE, a.slope));
          });
      __stcg(a.h2 + s.slot * H + h, acc);
    }
    if (lane_seg_last<H>(a.hcnt, s)) a.dD[vg * H + h] = lane_seg_fold<H>(a.h2, s);
  }
}

// ---- P3 over hub segments (out-CSR): ∂S partial Σ ∂E_pre over u's out-edges, v's m, den, P, q_D from the
// node record; the group that completes u's row writes ∂S[u], then the warp finalizes the completed rows'
// ∂H′ = (∂H′_agg + ∂S·a_src) + ∂D·a_dst (one warp per row)
struct VDa { int v; float da; };
struct RecH { float m, den, P, da; int qd; };
template <int H, int VPL>
__global__ void __launch_bounds__(256, 2) k2_bsrc2_hub(const G2Args a) {
  constexpr int SPW = 32 / H;
  const int lane = threadIdx.x & 31, h = lane % H;
  const Scale scS = scale_from_amax(amax_load(a.amax_S), a.bits);
  const Scale scD = scale_from_amax(amax_load(a.amax_D), a.bits);
  const int64_t hc = load_count(a.pout.counts);
  float amax_loc = 0.0f;
  FOR_LANE_SEGS(first, a.work + 11, hc, SPW) {
    const LaneSeg s = lane_seg<H>(first, hc, a.g.out_ptr, a.pout, a.g.chunk);
    const int64_t ug = a.g.row_begin + s.row;
    if (s.ok) {
      const int qs = a.qS[ug * H + h];
      float acc = 0.0f;
      lane_pipe<4, VDa, RecH>(
          s.eb, s.ee, [&](int64_t e) { return VDa{(int)__ldg(a.g.out_dst + e), __ldcs(a.dal_out + e * H + h)}; },
          [&](const VDa& x, int64_t) {
            const float* r = a.nrec + (int64_t)x.v * a.nrs;
            return RecH{r[h], r[H + h], r[2 * H + h], x.da, (int)reinterpret_cast<const int8_t*>(r + 3 * H)[h]};
          },
          [&](const RecH& y) {
            float ep;
            const float al = alpha1(qs, y.qd, scS.s, scD.s, a.slope, y.m, y.den, ep);
            const float dE = __fmul_rn(al, __fsub_rn(y.da, y.P));
            acc = __fadd_rn(acc, ep > 0.0f ? dE : __fmul_rn(dE, a.slope));
          });
      __stcg(a.hs + s.slot * H + h, acc);
    }
    const bool last = lane_seg_last<H>(a.hcnt, s);
    float dS = 0.0f;
    if (last) {
      dS = lane_seg_fold<H>(a.hs, s);
      a.dS[ug * H + h] = dS;
    }
    // finalize the rows completed by this warp's groups, the whole warp per row
    unsigned done = __ballot_sync(0xffffffffu, last && h == 0);
    while (done) {
      const int g0 = __ffs(done) - 1;
      done &= done - 1;
      float dSr[H];
#pragma unroll
      for (int k = 0; k < H; ++k) dSr[k] = __shfl_sync(0xffffffffu, dS, g0 + k);
      const int64_t rl = __shfl_sync(0xffffffffu, s.row, g0);
      src_finalize_row<H, VPL>(a, rl, dSr, amax_loc);
    }
  }
  amax_flush(a.amax_dHp, amax_loc);
}

// ================================================================== hub segments, multi-segment staged sums
// The per-edge scalar passes over hub rows with all 32 lanes busy in BOTH halves of the staged form: a warp
// claims SPW = 32/H consecutive hub segments (canonical chunks); per batch of 32 positions lane L computes
// position L of every one of the SPW segments (coalesced loads per segment) and stages the per-head values
// in shared memory [seg][pos][H]; then lane L = k·H + h adds segment k's staged values of head h in edge
// order (the chunk partial of Σᶜ).  Partials, the row's last-finisher fold and the P3 finalize are those of
// the lane form above.
template <int H, bool FMA, typename CV>
__device__ __forceinline__ float seg_multi(const LaneSeg& s, float* __restrict__ bx, float* __restrict__ by, CV&& cv) {
  constexpr int SPW = 32 / H;
  const int lane = threadIdx.x & 31, k = lane / H, h = lane % H;
  const int mylen = s.ok ? (int)(s.ee - s.eb) : 0;
  int maxlen = mylen;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) maxlen = max(maxlen, __shfl_xor_sync(0xffffffffu, maxlen, o));
  float acc = 0.0f;
  for (int b0 = 0; b0 < maxlen; b0 += 32) {
#pragma unroll 2
    for (int t = 0; t < SPW; ++t) {   // segment t: its start, length and row from its group leader
      const int ebt = __shfl_sync(0xffffffffu, (int)s.eb, t * H);
      const int lent = __shfl_sync(0xffffffffu, mylen, t * H);
      const int rowt = __shfl_sync(0xffffffffu, (int)s.row, t * H);
      if (b0 + lane < lent) {
        float x[H], y[H];
        cv(rowt, (int64_t)ebt + b0 + lane, x, y);
#pragma unroll
        for (int hh = 0; hh < H; ++hh) {
          bx[(t * 32 + lane) * H + hh] = x[hh];
          if (FMA) by[(t * 32 + lane) * H + hh] = y[hh];
        }
      }
    }
    __syncwarp();
    const int cnt = mylen - b0 < 32 ? mylen - b0 : 32;
    const float* px = bx + (k * 32) * H + h;
    const float* py = by + (k * 32) * H + h;
    int i = 0;
    for (; i + 4 <= cnt; i += 4) {
      const float x0 = px[i * H], x1 = px[(i + 1) * H], x2 = px[(i + 2) * H], x3 = px[(i + 3) * H];
      if (FMA) {
        const float y0 = py[i * H], y1 = py[(i + 1) * H], y2 = py[(i + 2) * H], y3 = py[(i + 3) * H];
        acc = __fmaf_rn(x0, y0, acc); acc = __fmaf_rn(x1, y1, acc);
        acc = __fmaf_rn(x2, y2, acc); acc = __fmaf_rn(x3, y3, acc);
      } else {
        acc = __fadd_rn(acc, x0); acc = __fadd_rn(acc, x1); acc = __fadd_rn(acc, x2); acc = __fadd_rn(acc, x3);
      }
    }
    for (; i < cnt; ++i) acc = FMA ? __fmaf_rn(px[i * H], py[i * H], acc) : __fadd_rn(acc, px[i * H]);
    __syncwarp();
  }
  return acc;
}

template <int H>
__global__ void __launch_bounds__(256, 3) k2_fstats2_hubm(const G2Args a) {
  constexpr int SPW = 32 / H;
  __shared__ float sbx[8][SPW * 32 * H];
  const int w = threadIdx.x >> 5, h = (threadIdx.x & 31) % H;
  const Scale scS = scale_from_amax(amax_load(a.amax_S), a.bits);
  const Scale scD = scale_from_amax(amax_load(a.amax_D), a.bits);
  const int64_t hc = load_count(a.pin.counts);
  FOR_LANE_SEGS(first, a.work + 8, hc, SPW) {
    const LaneSeg s = lane_seg<H>(first, hc, a.g.in_ptr, a.pin, a.g.chunk);
    const int64_t vg = a.g.row_begin + s.row;
    const float acc = seg_multi<H, false>(s, sbx[w], nullptr, [&](int rowt, int64_t e, float (&x)[H], float (&)[H]) {
      const int64_t rg = a.g.row_begin + rowt;
      int8_t qd[H], qs[H];
      load_qh<H>(a.qD + rg * H, qd);
      load_qh<H>(a.qS + (int64_t)__ldg(a.g.in_src + e) * H, qs);
      const unsigned* mk = reinterpret_cast<const unsigned*>(a.nrec + rg * a.nrs);
#pragma unroll
      for (int hh = 0; hh < H; ++hh)
        x[hh] = exp_p(__fsub_rn(lrelu(sddmm_add1(qs[hh], scS.s, qd[hh], scD.s), a.slope), fkey_dec(mk[hh])));
    });
    float m = 0.0f;
    if (s.ok) {
      m = fkey_dec(reinterpret_cast<const unsigned*>(a.nrec + vg * a.nrs)[h]);
      __stcg(a.h2 + s.slot * H + h, acc);
    }
    if (lane_seg_last<H>(a.hcnt, s)) {
      const float den = lane_seg_fold<H>(a.h2, s);
      a.m[vg * H + h] = m;
      rec_put1(a, vg, 0, h, m);
      a.den[vg * H + h] = den;
      rec_put1(a, vg, 1, h, den);
      reinterpret_cast<int8_t*>(a.nrec + vg * a.nrs + 3 * H)[h] = a.qD[vg * H + h];
    }
  }
}

template <int H>
__global__ void __launch_bounds__(128, 6) k2_bdst_a_hubm(const G2Args a) {   // 4-warp blocks (x and y staged)
  constexpr int SPW = 32 / H;
  __shared__ float sbx[4][SPW * 32 * H];
  __shared__ float sby[4][SPW * 32 * H];
  const int w = threadIdx.x >> 5, h = (threadIdx.x & 31) % H;
  const Scale scS = scale_from_amax(amax_load(a.amax_S), a.bits);
  const Scale scD = scale_from_amax(amax_load(a.amax_D), a.bits);
  const int64_t hc = load_count(a.pin.counts);
  FOR_LANE_SEGS(first, a.work + 9, hc, SPW) {
    const LaneSeg s = lane_seg<H>(first, hc, a.g.in_ptr, a.pin, a.g.chunk);
    const int64_t vg = a.g.row_begin + s.row;
    const float acc = seg_multi<H, true>(s, sbx[w], sby[w], [&](int rowt, int64_t e, float (&x)[H], float (&y)[H]) {
      float ep[H];
      if (a.rec) {
        float st[H];
        ld_h<H>(a.rec + e * 2 * H, x);
        ld_h<H>(a.rec + e * 2 * H + H, st);
        alpha_from_st<H>(st, ep, y);
        return;
      }
      if (a.scatter_in) {
        ld_h<H>(a.dal_in + e * H, x);
      } else {
        ld_h<H>(a.dal_out + (int64_t)__ldcs(a.in2out + e) * H, x);
        st_h<H>(a.dal_in + e * H, x);   // for P2b (coalesced)
      }
      if (a.alpha_st) {
        float st[H];
        ld_h<H>(a.alpha_st + e * H, st);
        alpha_from_st<H>(st, ep, y);
      } else {
        int8_t qs[H];
        load_qh<H>(a.qS + (int64_t)__ldg(a.g.in_src + e) * H, qs);
        alpha_rec<H>(qs, load_dst<H>(a, a.g.row_begin + rowt), scS.s, scD.s, a.slope, ep, y);
      }
    });
    if (s.ok) __stcg(a.h1 + s.slot * H + h, acc);
    if (lane_seg_last<H>(a.hcnt, s)) {
      const float P = lane_seg_fold<H>(a.h1, s);
      a.P[vg * H + h] = P;
      rec_put1(a, vg, 2, h, P);
    }
  }
}

template <int H>
__global__ void __launch_bounds__(256, 3) k2_bdst_b_hubm(const G2Args a) {
  constexpr int SPW = 32 / H;
  __shared__ float sbx[8][SPW * 32 * H];
  const int w = threadIdx.x >> 5, h = (threadIdx.x & 31) % H;
  const Scale scS = scale_from_amax(amax_load(a.amax_S), a.bits);
  const Scale scD = scale_from_amax(amax_load(a.amax_D), a.bits);
  const int64_t hc = load_count(a.pin.counts);
  FOR_LANE_SEGS(first, a.work + 10, hc, SPW) {
    const LaneSeg s = lane_seg<H>(first, hc, a.g.in_ptr, a.pin, a.g.chunk);
    const int64_t vg = a.g.row_begin + s.row;
    const float acc = seg_multi<H, false>(s, sbx[w], nullptr, [&](int rowt, int64_t e, float (&x)[H], float (&)[H]) {
      const int64_t rg = a.g.row_begin + rowt;
      float da[H], P[H], ep[H], al[H];
      ld_h<H>(a.P + rg * H, P);
      if (a.rec) {
        float st[H];
        ld_h<H>(a.rec + e * 2 * H, da);
        ld_h<H>(a.rec + e * 2 * H + H, st);
        alpha_from_st<H>(st, ep, al);
      } else if (a.alpha_st) {
        ld_h<H>(a.dal_in + e * H, da);
        float st[H];
        ld_h<H>(a.alpha_st + e * H, st);
        alpha_from_st<H>(st, ep, al);
      } else {
        ld_h<H>(a.dal_in + e * H, da);
        int8_t qs[H];
        load_qh<H>(a.qS + (int64_t)__ldg(a.g.in_src + e) * H, qs);
        alpha_rec<H>(qs, load_dst<H>(a, rg), scS.s, scD.s, a.slope, ep, al);
      }
#pragma unroll
      for (int hh = 0; hh < H; ++hh) {
        const float dE = __fmul_rn(al[hh], __fsub_rn(da[hh], P[hh]));
        x[hh] = ep[hh] > 0.0f ? dE : __fmul_rn(dE, a.slope);
      }
    });
    if (s.ok) __stcg(a.h2 + s.slot * H + h, acc);
    if (lane_seg_last<H>(a.hcnt, s)) a.dD[vg * H + h] = lane_seg_fold<H>(a.h2, s);
  }
}

template <int H, int VPL>
__global__ void __launch_bounds__(256, 3) k2_bsrc2_hubm(const G2Args a) {
  constexpr int SPW = 32 / H;
  __shared__ float sbx[8][SPW * 32 * H];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, h = lane % H;
  const Scale scS = scale_from_amax(amax_load(a.amax_S), a.bits);
  const Scale scD = scale_from_amax(amax_load(a.amax_D), a.bits);
  const int64_t hc = load_count(a.pout.counts);
  float amax_loc = 0.0f;
  FOR_LANE_SEGS(first, a.work + 11, hc, SPW) {
    const LaneSeg s = lane_seg<H>(first, hc, a.g.out_ptr, a.pout, a.g.chunk);
    const int64_t ug = a.g.row_begin + s.row;
    const float acc = seg_multi<H, false>(s, sbx[w], nullptr, [&](int rowt, int64_t e, float (&x)[H], float (&)[H]) {
      const int v = __ldg(a.g.out_dst + e);
      float da[H], Pv[H], ep[H], al[H];
      ld_h<H>(a.dal_out + e * H, da);
      ld_h<H>(a.nrec + (int64_t)v * a.nrs + 2 * H, Pv);
      if (a.al_out) {   // P1's signed α in out-CSR order
        float st[H];
        ld_h<H>(a.al_out + e * H, st);
        alpha_from_st<H>(st, ep, al);
      } else {
        int8_t qs[H];
        load_qh<H>(a.qS + (a.g.row_begin + rowt) * H, qs);
        alpha_rec<H>(qs, load_rec<H>(a, v), scS.s, scD.s, a.slope, ep, al);
      }
#pragma unroll
      for (int hh = 0; hh < H; ++hh) {
        const float dE = __fmul_rn(al[hh], __fsub_rn(da[hh], Pv[hh]));
        x[hh] = ep[hh] > 0.0f ? dE : __fmul_rn(dE, a.slope);
      }
    });
    if (s.ok) __stcg(a.hs + s.slot * H + h, acc);
    const bool last = lane_seg_last<H>(a.hcnt, s);
    float dS = 0.0f;
    if (last) {
      dS = lane_seg_fold<H>(a.hs, s);
      a.dS[ug * H + h] = dS;
    }
    unsigned done = __ballot_sync(0xffffffffu, last && h == 0);
    while (done) {
      const int g0 = __ffs(done) - 1;
      done &= done - 1;
      float dSr[H];
#pragma unroll
      for (int k2 = 0; k2 < H; ++k2) dSr[k2] = __shfl_sync(0xffffffffu, dS, g0 + k2);
      const int64_t rl = __shfl_sync(0xffffffffu, s.row, g0);
      src_finalize_row<H, VPL>(a, rl, dSr, amax_loc);
    }
  }
  amax_flush(a.amax_dHp, amax_loc);
}

// ================================================================== ∂a, deterministic (reading R39)
// ∂a_src[j] = Σᶜ_u fmaf(∂S[u,h], deq(q_H′)[u,j], ·) with chunks of DA_CHUNK global rows folded left to
// right (R33's order); block b computes chunk b's partials for all 2·HD outputs (one sequential fmaf chain
// per output and thread), the last block to finish folds the partials in chunk order.
constexpr int DA_CHUNK = 1024;
// Block (chunk, 128-column slice): one thread per column carries the ∂a_src and ∂a_dst chains of its column
// over the chunk's rows; the slice of every row (128 codes) and the rows' ∂S | ∂D are staged through a
// ring of 32-row tiles with cp.async.  A second kernel folds the chunk partials of every output left to right.
constexpr int DA_COLS = 128, DA_TR = 32, DA_NT = 4;
template <int H, int VPL>
__global__ void __launch_bounds__(DA_COLS) k2_attn_part(const G2Args a) {
  constexpr int HD = 32 * VPL;
  __shared__ __align__(16) int8_t sq[DA_NT][DA_TR][DA_COLS];
  __shared__ float ssd[DA_NT][DA_TR][2 * H];
  const Scale scH = scale_from_amax(amax_load(a.amax_Hp), a.bits);
  const int flip = a.codes_biased ? 128 : 0;   // stored excess-128 -> plain codes
  const int nsl = HD / DA_COLS;
  const int64_t ch = blockIdx.x / nsl;
  const int c0 = (blockIdx.x % nsl) * DA_COLS;
  const int tid = threadIdx.x, col = c0 + tid, h = col / (HD / H);
  const int64_t u0 = ch * DA_CHUNK, u1 = u0 + DA_CHUNK < a.g.n_local ? u0 + DA_CHUNK : a.g.n_local;
  const int ntile = (int)((u1 - u0 + DA_TR - 1) / DA_TR);
  auto issue = [&](int k) {
    const int64_t r0 = u0 + (int64_t)k * DA_TR;
    const int rows = u1 - r0 < DA_TR ? (int)(u1 - r0) : DA_TR;
    for (int i = tid; i < rows * (DA_COLS / 16); i += DA_COLS) {
      const int r = i / (DA_COLS / 16), c = i % (DA_COLS / 16);
      cp_async_bytes16(smem_u32(&sq[k % DA_NT][r][c * 16]), a.qHp + (a.g.row_begin + r0 + r) * a.ldHp + c0 + c * 16);
    }
    for (int i = tid; i < rows * 2 * H; i += DA_COLS) {
      const int r = i / (2 * H), c = i % (2 * H);
      const int64_t ug = a.g.row_begin + r0 + r;
      ssd[k % DA_NT][r][c] = c < H ? a.dS[ug * H + c] : a.dD[ug * H + c - H];
    }
    cp_commit();
  };
  float ps = 0.0f, pd = 0.0f;
#pragma unroll
  for (int k = 0; k < DA_NT - 1; ++k) {
    if (k < ntile) issue(k);
    else cp_commit();
  }
  for (int k = 0; k < ntile; ++k) {
    if (k + DA_NT - 1 < ntile) issue(k + DA_NT - 1);
    else cp_commit();
    cp_wait<DA_NT - 1>();
    __syncthreads();
    const int rows = u1 - (u0 + (int64_t)k * DA_TR) < DA_TR ? (int)(u1 - (u0 + (int64_t)k * DA_TR)) : DA_TR;
    const int b = k % DA_NT;
#pragma unroll 8
    for (int r = 0; r < rows; ++r) {
      const int q = (int)(uint8_t)sq[b][r][tid] - flip;   // plain code (two's complement if not biased)
      const float hp = __fmul_rn(__int2float_rn(flip ? q : (int)(int8_t)sq[b][r][tid]), scH.s);
      ps = __fmaf_rn(ssd[b][r][h], hp, ps);
      pd = __fmaf_rn(ssd[b][r][H + h], hp, pd);
    }
    __syncthreads();
  }
  cp_wait<0>();
  __stcg(a.da_part + ch * 2 * HD + col, ps);
  __stcg(a.da_part + ch * 2 * HD + HD + col, pd);
}
// output j (∂a_src then ∂a_dst): total = p_0, total = total + p_c over the chunks (R39), loads batched
template <int H, int VPL>
__global__ void __launch_bounds__(128) k2_attn_fold(const G2Args a) {
  constexpr int HD = 32 * VPL;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= 2 * HD) return;
  const int64_t nch = (a.g.n_local + DA_CHUNK - 1) / DA_CHUNK;
  float tot = 0.0f;
  for (int64_t c0 = 0; c0 < nch; c0 += 16) {
    float p[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) p[k] = c0 + k < nch ? __ldcg(a.da_part + (c0 + k) * 2 * HD + j) : 0.0f;
#pragma unroll
    for (int k = 0; k < 16; ++k)
      if (c0 + k < nch) tot = (c0 + k == 0) ? p[k] : __fadd_rn(tot, p[k]);
  }
  (j < HD ? a.da_src : a.da_dst)[j % HD] = tot;
}

// ================================================================== in-CSR -> out-CSR position map
__global__ void k2_in2out(const int32_t* __restrict__ out_eid, int64_t e, int32_t* __restrict__ in2out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < e; i += (int64_t)gridDim.x * blockDim.x)
    in2out[out_eid[i]] = (int32_t)i;
}
cudaError_t launch_gat2_in2out(const int32_t* out_eid, int64_t e, int32_t* in2out, cudaStream_t st) {
  if (e == 0) return cudaSuccess;
  ProfScope p("plan_in2out", st);
  const int64_t blocks = (e + 255) / 256;
  k2_in2out<<<(unsigned)(blocks < (int64_t)num_sms() * 16 ? blocks : (int64_t)num_sms() * 16), 256, 0, st>>>(out_eid, e,
                                                                                                          in2out);
  return cudaGetLastError();
}

// ================================================================== launchers
static int grid_items(int64_t items, int per_sm) {
  int64_t g = items;
  const int64_t cap = (int64_t)num_sms() * per_sm;
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

bool gat2_supported(const GraphDev& g, int heads, int hd) {
  const int vpl = hd / 32;
  return g.out_eid && g.row_begin == 0 && g.n_local == g.n_global && g.chunk <= 256 &&
         (vpl == 4 || vpl == 8 || vpl == 16) && (heads == 1 || heads == 2 || heads == 4 || heads == 8) &&
         hd % heads == 0 && (hd / heads) % (vpl) == 0 && 32 % heads == 0;
}

#define G2_CASES(X) X(1, 4) X(1, 8) X(1, 16) X(2, 4) X(2, 8) X(2, 16) X(4, 4) X(4, 8) X(4, 16) X(8, 4) X(8, 8) X(8, 16)

static cudaError_t fork2(cudaStream_t st, const SideStream* x) {
  if (!x || x->s == st) return cudaSuccess;
  cudaError_t e = cudaEventRecord(x->fork, st);
  return e == cudaSuccess ? cudaStreamWaitEvent(x->s, x->fork, 0) : e;
}
static cudaError_t join2(cudaStream_t st, const SideStream* x) {
  if (!x || x->s == st) return cudaSuccess;
  cudaError_t e = cudaEventRecord(x->join, x->s);
  return e == cudaSuccess ? cudaStreamWaitEvent(st, x->join, 0) : e;
}

// hub-row pieces on the side stream (when given) beside the light sub-tiles on st
cudaError_t launch_gat2_fwd(const G2Args& a, cudaStream_t st, const SideStream* x) {
  cudaStream_t sh = (x && x->s) ? x->s : st;
  const int hv = a.d.heads * 100 + a.d.hd / 32;
  bool ok = false;
  cudaError_t e = cudaSuccess;
#define X(H_, V_)                                                                                    \
  if (hv == H_ * 100 + V_) {                                                                         \
    ok = true;                                                                                       \
    constexpr int smem = 8 * ((fa_warp_smem<H_, V_>() + 15) & ~15);                                   \
    constexpr int smem_s = 8 * ((fs_warp_smem_seg<H_, V_>() + 15) & ~15);                             \
    static bool attr = false;                                                                        \
    if (!attr) {                                                                                     \
      cudaFuncSetAttribute(k2_fagg<H_, V_>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);      \
      cudaFuncSetAttribute(k2_fagg_seg<H_, V_>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_s); \
      attr = true;                                                                                   \
    }                                                                                                \
    { ProfScope p("gat_fwd_stats1", st); k2_fstats1<H_><<<grid_items((a.pin.cap + 7) / 8, 4), 256, 0, st>>>(a); } \
    if (a.hub_fs) { /* hub segments on the side stream beside the light sub-tiles */                   \
      e = fork2(st, x);                                                                              \
      { ProfScope p("gat_fwd_stats_hub", sh); if (a.hub_fs == 2) k2_fstats2_hubm<H_><<<grid_items((a.pin.cap + 63) / 64, 3), 256, 0, sh>>>(a); else k2_fstats2_hub<H_><<<grid_items((a.pin.cap + 63) / 64, 4), 256, 0, sh>>>(a); } \
      { ProfScope p("gat_fwd_stats", st); k2_fstats2<H_><<<grid_items((a.pin.cap + a.pin.tcap + 7) / 8, 4), 256, 0, st>>>(a); } \
      if (e == cudaSuccess) e = join2(st, x);                                                        \
    } else { ProfScope p("gat_fwd_stats", st); k2_fstats2<H_><<<grid_items((a.pin.cap + a.pin.tcap + 7) / 8, 4), 256, 0, st>>>(a); } \
    if (e == cudaSuccess) e = fork2(st, x);                                                          \
    { ProfScope p("gat_fwd_agg_hub", sh); k2_fagg_seg<H_, V_><<<grid_items((a.pin.cap + 7) / 8, 3), 256, smem_s, sh>>>(a); } \
    { ProfScope p("gat_fwd_agg", st); k2_fagg<H_, V_><<<grid_items((a.pin.tcap + 7) / 8, 3), 256, smem, st>>>(a); } \
    if (e == cudaSuccess) e = join2(st, x);                                                          \
  }
  G2_CASES(X)
#undef X
  if (!ok) return cudaErrorInvalidValue;
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_gat2_bwd(const G2Args& a, cudaStream_t st, const SideStream* x) {
  cudaStream_t sh = (x && x->s) ? x->s : st;
  const int hv = a.d.heads * 100 + a.d.hd / 32;
  bool ok = false;
  cudaError_t e = cudaSuccess;
#define X(H_, V_)                                                                                    \
  if (hv == H_ * 100 + V_) {                                                                         \
    ok = true;                                                                                       \
    constexpr int NW = 4, smem = NW * ((bs_warp_smem<H_, V_>() + 15) & ~15);                          \
    constexpr int smem_s = NW * ((bs_warp_smem_seg<H_, V_>() + 15) & ~15);                           \
    static bool attr = false;                                                                        \
    if (!attr) {                                                                                     \
      cudaFuncSetAttribute(k2_bsrc1<H_, V_, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
      cudaFuncSetAttribute(k2_bsrc1_seg<H_, V_, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_s); \
      attr = true;                                                                                   \
    }                                                                                                \
    e = fork2(st, x);                                                                                \
    { ProfScope p("gat_bwd_src_hub", sh); k2_bsrc1_seg<H_, V_, NW><<<grid_items((a.pout.cap + NW - 1) / NW, 20 / NW), NW * 32, smem_s, sh>>>(a); } \
    { ProfScope p("gat_bwd_src", st); k2_bsrc1<H_, V_, NW><<<grid_items((a.pout.tcap + NW - 1) / NW, 20 / NW), NW * 32, smem, st>>>(a); } \
    if (e == cudaSuccess) e = join2(st, x);                                                          \
    if (a.hub_p2) { /* P2 hub segments on the side stream beside the light sub-tiles */                \
      if (e == cudaSuccess) e = fork2(st, x);                                                        \
      { ProfScope p("gat_bwd_dst_hub", sh); if (a.hub_p2 == 2) k2_bdst_a_hubm<H_><<<grid_items((a.pin.cap + 31) / 32, 6), 128, 0, sh>>>(a); else k2_bdst_a_hub<H_><<<grid_items((a.pin.cap + 63) / 64, 4), 256, 0, sh>>>(a); } \
      { ProfScope p("gat_bwd_dst", st); k2_bdst_a<H_><<<grid_items((a.pin.cap + a.pin.tcap + 7) / 8, 4), 256, 0, st>>>(a); } \
      if (e == cudaSuccess) e = join2(st, x);                                                        \
      { ProfScope p("gat_bwd_dst2", st); if (a.hub_p2 == 2) k2_bdst_b_hubm<H_><<<grid_items((a.pin.cap + 63) / 64, 3), 256, 0, st>>>(a); else k2_bdst_b_hub<H_><<<grid_items((a.pin.cap + 63) / 64, 4), 256, 0, st>>>(a); } \
    } else {                                                                                         \
      { ProfScope p("gat_bwd_dst", st); k2_bdst_a<H_><<<grid_items((a.pin.cap + a.pin.tcap + 7) / 8, 4), 256, 0, st>>>(a); } \
      { ProfScope p("gat_bwd_dst2", st); k2_bdst_b<H_><<<grid_items((a.pin.cap + 7) / 8, 4), 256, 0, st>>>(a); } \
    }                                                                                                \
    if (a.hub_p3) { /* P3 hub segments on the side stream beside the light sub-tiles */                \
      if (e == cudaSuccess) e = fork2(st, x);                                                        \
      { ProfScope p("gat_bwd_src2_hub", sh); if (a.hub_p3 == 2) k2_bsrc2_hubm<H_, V_><<<grid_items((a.pout.cap + 63) / 64, 3), 256, 0, sh>>>(a); else k2_bsrc2_hub<H_, V_><<<grid_items((a.pout.cap + 63) / 64, 4), 256, 0, sh>>>(a); } \
      { ProfScope p("gat_bwd_src2", st); k2_bsrc2<H_, V_><<<grid_items((a.pout.cap + a.pout.tcap + 7) / 8, 4), 256, 0, st>>>(a); } \
      if (e == cudaSuccess) e = join2(st, x);                                                        \
    } else {                                                                                         \
      { ProfScope p("gat_bwd_src2", st); k2_bsrc2<H_, V_><<<grid_items((a.pout.cap + a.pout.tcap + 7) / 8, 4), 256, 0, st>>>(a); } \
    }                                                                                                \
  }
  G2_CASES(X)
#undef X
  if (!ok) return cudaErrorInvalidValue;
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_gat2_attn_grad(const G2Args& a, cudaStream_t st) {
  const int hv = a.d.heads * 100 + a.d.hd / 32;
  const int64_t nch = (a.g.n_local + DA_CHUNK - 1) / DA_CHUNK;
  bool ok = false;
#define X(H_, V_)                                                                                    \
  if (hv == H_ * 100 + V_) {                                                                         \
    ok = true;                                                                                       \
    if (nch > 0) {                                                                                   \
      ProfScope p("gat_bwd_attn_grad", st);                                                          \
      k2_attn_part<H_, V_><<<(unsigned)(nch * (32 * V_ / DA_COLS)), DA_COLS, 0, st>>>(a);            \
    }                                                                                                \
    { ProfScope p("gat_bwd_attn_fold", st); k2_attn_fold<H_, V_><<<(2 * 32 * V_ + 127) / 128, 128, 0, st>>>(a); } \
  }
  G2_CASES(X)
#undef X
  if (!ok) return cudaErrorInvalidValue;
  return cudaGetLastError();
}

}  // namespace tango
