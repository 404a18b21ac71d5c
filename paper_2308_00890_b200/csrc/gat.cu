// gat.cu — the sparse half of the quantized GAT layer as fused, segment-parallel row kernels.
//
// Paper: ③ SDDMM-add + LeakyReLU, ④ edge softmax (FP32 per P:604-615),
// ⑤ SPMM, ⑤′ SPMM on the reversed graph, ⑤″ SDDMM-dot on codes
// (P:252-255), ④′ softmax backward, ③′/③″ incidence SPMM (P:276,
// P:821-832), ②′ (reading R23).
//
// B200 design:
//  * A node row of HD int8 codes is split across the 32 lanes of a warp (VPL = HD/32 codes per
//    lane, 16 B at HD = 512), so one warp-wide 16-B load gathers a whole 512-B source row.
//  * Work items are SEGMENTS: a row with deg <= C_E is one segment (processed end to end by one
//    warp); a row with deg > C_E ("heavy", the power-law hubs) is cut at the canonical chunk
//    boundaries of reading R14 into ceil(deg/C_E) segments processed by different warps, whose
//    partial sums are folded afterwards in chunk order — bit-identical to the oracle's Σᶜ.
//    A per-call plan kernel lists heavy rows and assigns their segments scratch slots.
//  * Per-edge scalars (α, ∂α, e_pre) are computed lane-parallel over 32-edge batches and staged
//    in shared memory; α, ∂α and ∂E are recomputed from per-node data (reading R30), so the only
//    edge-sized arrays are the CSR indices and one fp32 ∂α scratch (backward destination pass).
//  * Row gathers are software-pipelined 8 edges deep (8 x 16-B loads in flight per lane).
#include "rowops.cuh"

namespace tango {

constexpr int WPB = 8;      // warps per block of the row kernels
constexpr int UNR = 8;      // gather pipeline depth (edges in flight per warp)

// ------------------------------------------------------------------ plan
// hbase[v] = first scratch slot of heavy row v's segments (or -1), hseg_row[slot] = v,
// hrow[i] = i-th heavy row; counts[0] = #heavy segments, counts[1] = #heavy rows (pre-zeroed).
__global__ void k_plan(const int64_t* __restrict__ ptr, int64_t n, int chunk, PlanDev p) {
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= n) return;
  const int64_t deg = ptr[v + 1] - ptr[v];
  if (deg > chunk) {
    const int nseg = (int)((deg + chunk - 1) / chunk);
    const int base = atomicAdd(&p.counts[0], nseg);
    p.hbase[v] = base;
    for (int c = 0; c < nseg; ++c) p.hseg_row[base + c] = (int32_t)v;
    p.hrow[atomicAdd(&p.counts[1], 1)] = (int32_t)v;
  } else {
    p.hbase[v] = -1;
  }
}
cudaError_t launch_plan(const int64_t* ptr, int64_t n, int chunk, const PlanDev& p, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  ProfScope ps("plan", st);
  k_plan<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(ptr, n, chunk, p);
  return cudaGetLastError();
}

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

template <int H>
__device__ __forceinline__ float head_pick(const float (&x)[H], int h) {
  float r = 0.0f;
#pragma unroll
  for (int k = 0; k < H; ++k) if (k == h) r = x[k];
  return r;
}

// max over the segment of el = lrelu(e_pre) (lane-parallel; order-free), all lanes get the result
template <int H>
__device__ __forceinline__ void seg_max(const int32_t* __restrict__ src, int64_t eb, int64_t ee,
                                        const int8_t* __restrict__ qS, float sS, const int8_t (&qd)[H], float sD,
                                        float slope, float (&mx)[H]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int h = 0; h < H; ++h) mx[h] = -INFINITY;
  for (int64_t e = eb + lane; e < ee; e += 32) {
    const int64_t u = src[e];
#pragma unroll
    for (int h = 0; h < H; ++h) mx[h] = fmaxf(mx[h], lrelu(sddmm_add1(qS[u * H + h], sS, qd[h], sD), slope));
  }
#pragma unroll
  for (int h = 0; h < H; ++h) mx[h] = warp_max(mx[h]);
}

// Σ over the segment of exp_p(el - m), sequential in edge order (one chunk: no folding).
// Returns the sum for head `lane` in lanes < H.
template <int H>
__device__ __forceinline__ float seg_sum_exp(const int32_t* __restrict__ src, int64_t eb, int64_t ee,
                                             const int8_t* __restrict__ qS, float sS, const int8_t (&qd)[H],
                                             float sD, float slope, const float (&mx)[H], float (*buf)[H]) {
  const int lane = threadIdx.x & 31;
  float part = 0.0f;
  for (int64_t base = eb; base < ee; base += 32) {
    const int cnt = (int)(ee - base < 32 ? ee - base : 32);
    if (lane < cnt) {
      const int64_t u = src[base + lane];
#pragma unroll
      for (int h = 0; h < H; ++h)
        buf[lane][h] = exp_p(__fsub_rn(lrelu(sddmm_add1(qS[u * H + h], sS, qd[h], sD), slope), mx[h]));
    }
    __syncwarp();
    if (lane < H)
      for (int i = 0; i < cnt; ++i) part = __fadd_rn(part, buf[i][lane]);
    __syncwarp();
  }
  return part;
}

// m = max over a heavy row's segment maxima, den = left fold of its segment sums (lane h), broadcast
template <int H>
__device__ __forceinline__ void heavy_row_stats(const float* __restrict__ hmax, const float* __restrict__ hden,
                                                int base, int nseg, float (&mx)[H], float (&den)[H]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int h = 0; h < H; ++h) mx[h] = -INFINITY;
  for (int j = lane; j < nseg; j += 32)
#pragma unroll
    for (int h = 0; h < H; ++h) mx[h] = fmaxf(mx[h], hmax[(int64_t)(base + j) * H + h]);
#pragma unroll
  for (int h = 0; h < H; ++h) mx[h] = warp_max(mx[h]);
  if (hden) {
    float tot = 0.0f;
    if (lane < H) {
      tot = hden[(int64_t)base * H + lane];
      for (int j = 1; j < nseg; ++j) tot = __fadd_rn(tot, hden[(int64_t)(base + j) * H + lane]);
    }
#pragma unroll
    for (int h = 0; h < H; ++h) den[h] = __shfl_sync(0xffffffffu, tot, h);
  }
}

// exact int8 -> fp32 of byte k of a word pre-XORed with 0x80808080: 2^23 + 128 + q - (2^23 + 128)
__device__ __forceinline__ float bx2f(uint32_t wx, int k) {
  return __fsub_rn(__uint_as_float(__byte_perm(wx, 0x4B000000u, 0x7440u | (uint32_t)k)), 8388736.0f);
}

// part[k] += α[e] * q_X[w_e][lane*VPL + k] over the segment's 32-edge batch (α staged in abuf[i][myh]),
// rows gathered 8 deep.  `idx` holds the other endpoint of edge (base + lane).
template <int VPL>
__device__ __forceinline__ void gather_fma_batch(const int8_t* __restrict__ xbase, int64_t ldx, int idx, int cnt,
                                                 const float* __restrict__ acol /* &abuf[0][myh] */, int astride,
                                                 float (&part)[VPL]) {
  for (int i0 = 0; i0 < cnt; i0 += UNR) {
    Row<VPL> r[UNR];
#pragma unroll
    for (int j = 0; j < UNR; ++j) {
      const int w = __shfl_sync(0xffffffffu, idx, (i0 + j) & 31);
      if (i0 + j < cnt) r[j] = load_row<VPL>(xbase + (int64_t)w * ldx);
    }
#pragma unroll
    for (int j = 0; j < UNR; ++j) {
      if (i0 + j < cnt) {
        const float al = acol[(i0 + j) * astride];
#pragma unroll
        for (int q = 0; q < (VPL + 3) / 4; ++q) {
          const uint32_t wx = r[j].w[q] ^ 0x80808080u;
#pragma unroll
          for (int k = 0; k < 4 && q * 4 + k < VPL; ++k) part[q * 4 + k] = __fmaf_rn(al, bx2f(wx, k), part[q * 4 + k]);
        }
      }
    }
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
                                               int64_t r0, int64_t n, int& T) {
  const int lane = threadIdx.x & 31;
  TileLane L;
  L.r = r0 + lane;
  const bool has = L.r < n;
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

// ================================================================== forward
// FS: light rows -> m, den (final);  heavy segments -> segment max (hmax)
template <int H>
__global__ void __launch_bounds__(256) k_fwd_stats(const GatFwdArgs a) {
  __shared__ float sh[WPB][32][H];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Scale scS = scale_from_amax(amax_load(a.amax_S), a.bits);
  const Scale scD = scale_from_amax(amax_load(a.amax_D), a.bits);
  const int64_t hc = load_count(a.plan.counts), nitems = a.g.n_local + hc;
  FOR_ITEMS(item, a.work + 0, nitems) {
    Seg s;
    if (!decode_item(item, hc, a.g.in_ptr, a.plan, a.g.chunk, s)) continue;
    const int64_t vg = a.g.row_begin + s.vl;
    int8_t qd[H];
#pragma unroll
    for (int h = 0; h < H; ++h) qd[h] = a.qD[vg * H + h];
    float mx[H];
    seg_max<H>(a.g.in_src, s.eb, s.ee, a.qS, scS.s, qd, scD.s, a.slope, mx);
    if (s.slot >= 0) {
      if (lane < H) a.hmax[(int64_t)s.slot * H + lane] = head_pick<H>(mx, lane);
      continue;
    }
    if (s.ee == s.eb)
#pragma unroll
      for (int h = 0; h < H; ++h) mx[h] = 0.0f;
    const float den = seg_sum_exp<H>(a.g.in_src, s.eb, s.ee, a.qS, scS.s, qd, scD.s, a.slope, mx, sh[w]);
    if (lane < H) {
      a.m[vg * H + lane] = head_pick<H>(mx, lane);
      a.den[vg * H + lane] = den;
    }
  }
}

// FS2: heavy segments -> segment Σ exp_p(el - m) (hden), m from all segment maxima of the row
template <int H>
__global__ void __launch_bounds__(256) k_fwd_stats2(const GatFwdArgs a) {
  __shared__ float sh[WPB][32][H];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Scale scS = scale_from_amax(amax_load(a.amax_S), a.bits);
  const Scale scD = scale_from_amax(amax_load(a.amax_D), a.bits);
  const int64_t hcnt = load_count(a.plan.counts);
  FOR_ITEMS(si, a.work + 1, hcnt) {
    Seg s;
    decode_item(si, hcnt, a.g.in_ptr, a.plan, a.g.chunk, s);
    const int64_t vg = a.g.row_begin + s.vl;
    int8_t qd[H];
#pragma unroll
    for (int h = 0; h < H; ++h) qd[h] = a.qD[vg * H + h];
    float mx[H], dummy[H];
    heavy_row_stats<H>(a.hmax, nullptr, s.base, s.nseg, mx, dummy);
    const float part = seg_sum_exp<H>(a.g.in_src, s.eb, s.ee, a.qS, scS.s, qd, scD.s, a.slope, mx, sh[w]);
    if (lane < H) a.hden[si * H + lane] = part;
  }
}


// FA on a tile of light rows: α per edge (lane-parallel), aggregation streamed across rows.
template <int H, int VPL>
__device__ __forceinline__ void fwd_agg_tile(const GatFwdArgs& a, int64_t r0, float (*buf)[H], int* rb,
                                             float sS, float sD, float sH, float& amax_loc) {
  constexpr int LPH = 32 / H;
  constexpr int HD = 32 * VPL;
  const int lane = threadIdx.x & 31, myh = lane / LPH;
  int T;
  const TileLane L = tile_setup(a.g.in_ptr, a.plan.hbase, r0, a.g.n_local, T);
  const int64_t vg = a.g.row_begin + L.r;
  float mj[H], dj[H];
  int qdj[H];
#pragma unroll
  for (int h = 0; h < H; ++h) {
    mj[h] = L.deg > 0 ? a.m[vg * H + h] : 0.0f;
    dj[h] = L.deg > 0 ? a.den[vg * H + h] : 0.0f;
    qdj[h] = L.deg > 0 ? (int)a.qD[vg * H + h] : 0;
  }
  unsigned zm = __ballot_sync(0xffffffffu, L.light && L.deg == 0);
  while (zm) {   // light rows without in-edges: H_out = 0
    const int j = __ffs(zm) - 1;
    zm &= zm - 1;
    float* dst = a.Hout + (r0 + j) * HD + lane * VPL;
#pragma unroll
    for (int k = 0; k < VPL; ++k) dst[k] = 0.0f;
  }
  const int8_t* xbase = a.qHp + lane * VPL;
  float part[VPL];
#pragma unroll
  for (int k = 0; k < VPL; ++k) part[k] = 0.0f;
  int cur = -1;
  auto flush = [&](int j) {
    float* dst = a.Hout + (r0 + j) * HD + lane * VPL;
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const float o = __fmul_rn(part[k], sH);
      amax_loc = fmaxf(amax_loc, fabsf(o));
      dst[k] = o;
      part[k] = 0.0f;
    }
  };
  for (int base = 0; base < T; base += 32) {
    const int cnt = T - base < 32 ? T - base : 32;
    const int t = base + lane;
    const int row = tile_row(t, L.end);
    const int64_t ebr = __shfl_sync(0xffffffffu, L.eb, row);
    const int offr = __shfl_sync(0xffffffffu, L.off, row);
    float mr[H], dr[H];
    int qdr[H];
#pragma unroll
    for (int h = 0; h < H; ++h) {
      mr[h] = __shfl_sync(0xffffffffu, mj[h], row);
      dr[h] = __shfl_sync(0xffffffffu, dj[h], row);
      qdr[h] = __shfl_sync(0xffffffffu, qdj[h], row);
    }
    int u = 0;
    if (lane < cnt) {
      u = a.g.in_src[ebr + (t - offr)];
#pragma unroll
      for (int h = 0; h < H; ++h)
        buf[lane][h] = __fdiv_rn(
            exp_p(__fsub_rn(lrelu(sddmm_add1(a.qS[(int64_t)u * H + h], sS, (int8_t)qdr[h], sD), a.slope), mr[h])),
            dr[h]);
      rb[lane] = row;
    }
    __syncwarp();
    for (int i0 = 0; i0 < cnt; i0 += UNR) {
      Row<VPL> rr[UNR];
#pragma unroll
      for (int j = 0; j < UNR; ++j) {
        const int w = __shfl_sync(0xffffffffu, u, (i0 + j) & 31);
        if (i0 + j < cnt) rr[j] = load_row<VPL>(xbase + (int64_t)w * a.ldHp);
      }
#pragma unroll
      for (int j = 0; j < UNR; ++j) {
        if (i0 + j < cnt) {
          const int ri = rb[i0 + j];
          if (ri != cur) {
            if (cur >= 0) flush(cur);
            cur = ri;
          }
          const float al = buf[i0 + j][myh];
#pragma unroll
          for (int q = 0; q < (VPL + 3) / 4; ++q) {
            const uint32_t wx = rr[j].w[q] ^ 0x80808080u;
#pragma unroll
            for (int k = 0; k < 4 && q * 4 + k < VPL; ++k) part[q * 4 + k] = __fmaf_rn(al, bx2f(wx, k), part[q * 4 + k]);
          }
        }
      }
    }
    __syncwarp();
  }
  if (cur >= 0) flush(cur);
}

// FA: α = exp_p(el - m)/den and the aggregation Σ fmaf(α, q_H′[u]) per segment;
// light rows finish H_out, heavy segments leave a partial in hagg.
template <int H, int VPL>
__global__ void __launch_bounds__(256, 2) k_fwd_agg(const GatFwdArgs a) {
  constexpr int LPH = 32 / H;
  constexpr int HD = 32 * VPL;
  __shared__ float sh[WPB][32][H];
  __shared__ unsigned sh_amax;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int myh = lane / LPH;
  float (*buf)[H] = sh[w];
  if (threadIdx.x == 0) sh_amax = 0u;
  __syncthreads();
  const Scale scS = scale_from_amax(amax_load(a.amax_S), a.bits);
  const Scale scD = scale_from_amax(amax_load(a.amax_D), a.bits);
  const Scale scH = scale_from_amax(amax_load(a.amax_Hp), a.bits);
  const int64_t hc = load_count(a.plan.counts), nitems = hc + (a.g.n_local + TILE - 1) / TILE;
  const int8_t* xbase = a.qHp + lane * VPL;
  float amax_loc = 0.0f;
  __shared__ int sh_rb[WPB][32];
  FOR_ITEMS(item, a.work + 2, nitems) {
    if (item >= hc) {
      fwd_agg_tile<H, VPL>(a, (item - hc) * TILE, buf, sh_rb[w], scS.s, scD.s, scH.s, amax_loc);
      continue;
    }
    Seg s;
    if (!decode_item(item, hc, a.g.in_ptr, a.plan, a.g.chunk, s)) continue;
    const int64_t vg = a.g.row_begin + s.vl;
    int8_t qd[H];
    float mx[H], den[H];
#pragma unroll
    for (int h = 0; h < H; ++h) qd[h] = a.qD[vg * H + h];
    if (s.slot < 0) {
#pragma unroll
      for (int h = 0; h < H; ++h) { mx[h] = a.m[vg * H + h]; den[h] = a.den[vg * H + h]; }
    } else {
      heavy_row_stats<H>(a.hmax, a.hden, s.base, s.nseg, mx, den);
    }
    float part[VPL];
#pragma unroll
    for (int k = 0; k < VPL; ++k) part[k] = 0.0f;
    for (int64_t base = s.eb; base < s.ee; base += 32) {
      const int cnt = (int)(s.ee - base < 32 ? s.ee - base : 32);
      int u = 0;
      if (lane < cnt) {
        u = a.g.in_src[base + lane];
#pragma unroll
        for (int h = 0; h < H; ++h)
          buf[lane][h] = __fdiv_rn(
              exp_p(__fsub_rn(lrelu(sddmm_add1(a.qS[(int64_t)u * H + h], scS.s, qd[h], scD.s), a.slope), mx[h])),
              den[h]);
      }
      __syncwarp();
      gather_fma_batch<VPL>(xbase, a.ldHp, u, cnt, &buf[0][myh], H, part);
      __syncwarp();
    }
    if (s.slot < 0) {
      float out[VPL];
#pragma unroll
      for (int k = 0; k < VPL; ++k) { out[k] = __fmul_rn(part[k], scH.s); amax_loc = fmaxf(amax_loc, fabsf(out[k])); }
      float* dst = a.Hout + s.vl * HD + lane * VPL;
#pragma unroll
      for (int k = 0; k < VPL; ++k) dst[k] = out[k];
    } else {
      float* dst = a.hagg + (int64_t)s.slot * HD + lane * VPL;
#pragma unroll
      for (int k = 0; k < VPL; ++k) dst[k] = part[k];
    }
  }
  if (a.amax_out) {
    amax_loc = warp_max(amax_loc);
    if (lane == 0) atomicMax(&sh_amax, __float_as_uint(amax_loc));
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(a.amax_out, sh_amax);
  }
}

// FC: heavy rows — fold segment partials in chunk order, write m, den, H_out
template <int H, int VPL>
__global__ void __launch_bounds__(256) k_fwd_combine(const GatFwdArgs a) {
  constexpr int HD = 32 * VPL;
  __shared__ unsigned sh_amax;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) sh_amax = 0u;
  __syncthreads();
  const Scale scH = scale_from_amax(amax_load(a.amax_Hp), a.bits);
  const int64_t hrows = load_count(a.plan.counts + 1);
  float amax_loc = 0.0f;
  FOR_ITEMS(r, a.work + 3, hrows) {
    const int64_t vl = a.plan.hrow[r];
    const int64_t vg = a.g.row_begin + vl;
    const int base = a.plan.hbase[vl];
    const int64_t deg = a.g.in_ptr[vl + 1] - a.g.in_ptr[vl];
    const int nseg = (int)((deg + a.g.chunk - 1) / a.g.chunk);
    float mx[H], den[H];
    heavy_row_stats<H>(a.hmax, a.hden, base, nseg, mx, den);
    if (lane < H) {
      a.m[vg * H + lane] = head_pick<H>(mx, lane);
      a.den[vg * H + lane] = head_pick<H>(den, lane);
    }
    float tot[VPL];
    const float* src = a.hagg + (int64_t)base * HD + lane * VPL;
#pragma unroll
    for (int k = 0; k < VPL; ++k) tot[k] = src[k];
    for (int j = 1; j < nseg; ++j) {
      const float* p = src + (int64_t)j * HD;
#pragma unroll
      for (int k = 0; k < VPL; ++k) tot[k] = __fadd_rn(tot[k], p[k]);
    }
    float* dst = a.Hout + vl * HD + lane * VPL;
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const float o = __fmul_rn(tot[k], scH.s);
      amax_loc = fmaxf(amax_loc, fabsf(o));
      dst[k] = o;
    }
  }
  if (a.amax_out) {
    amax_loc = warp_max(amax_loc);
    if (lane == 0) atomicMax(&sh_amax, __float_as_uint(amax_loc));
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(a.amax_out, sh_amax);
  }
}

// ================================================================== backward, destination side
// Pass 1 over a segment of v's in-edges: ∂α = i2f(q_G[v]·q_H′[u]) (s_G s_H′) -> dalpha scratch,
// P partial = Σ fmaf(∂α, α) (sequential, leader lane of each head).  Returns P partial in leaders.
template <int H, int VPL>
__device__ __forceinline__ float bwd_dst_pass1(const GatBwdArgs& a, const Seg& s, const int8_t (&qd)[H],
                                               const float (&mh)[H], const float (&dh)[H], const Row<VPL>& gw,
                                               float sS, float sD, float sGH, float (*ba)[H], float (*bd)[H]) {
  constexpr int LPH = 32 / H;
  const int lane = threadIdx.x & 31;
  const int myh = lane / LPH;
  const bool leader = (lane % LPH) == 0;
  float P = 0.0f;
  const int8_t* hbase = a.qHp + lane * VPL;
  for (int64_t base = s.eb; base < s.ee; base += 32) {
    const int cnt = (int)(s.ee - base < 32 ? s.ee - base : 32);
    int u = 0;
    if (lane < cnt) {
      u = a.g.in_src[base + lane];
#pragma unroll
      for (int h = 0; h < H; ++h)
        ba[lane][h] = __fdiv_rn(
            exp_p(__fsub_rn(lrelu(sddmm_add1(a.qS[(int64_t)u * H + h], sS, qd[h], sD), a.slope), mh[h])), dh[h]);
    }
    __syncwarp();
    for (int i0 = 0; i0 < cnt; i0 += UNR) {
      Row<VPL> r[UNR];
#pragma unroll
      for (int j = 0; j < UNR; ++j) {
        const int w = __shfl_sync(0xffffffffu, u, (i0 + j) & 31);
        if (i0 + j < cnt) r[j] = load_row<VPL>(hbase + (int64_t)w * a.ldHp);
      }
#pragma unroll
      for (int j = 0; j < UNR; ++j) {
        if (i0 + j < cnt) {
          int dot = row_dot<VPL>(gw, r[j]);
#pragma unroll
          for (int o = 1; o < LPH; o <<= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
          if (leader) {
            const float dal = __fmul_rn(__int2float_rn(dot), sGH);
            P = __fmaf_rn(dal, ba[i0 + j][myh], P);
            bd[i0 + j][myh] = dal;
          }
        }
      }
    }
    __syncwarp();
    for (int idx = lane; idx < cnt * H; idx += 32) a.dalpha[base * H + idx] = bd[idx / H][idx % H];
    __syncwarp();
  }
  return P;
}

// Pass 2 over a segment: ∂E = α(∂α − P[v]), ∂E_pre (LeakyReLU backward), Σ ∂E_pre (lane h).
template <int H>
__device__ __forceinline__ float bwd_dst_pass2(const GatBwdArgs& a, const Seg& s, const int8_t (&qd)[H],
                                               const float (&mh)[H], const float (&dh)[H], const float (&P)[H],
                                               float sS, float sD, float (*ba)[H]) {
  const int lane = threadIdx.x & 31;
  float part = 0.0f;
  for (int64_t base = s.eb; base < s.ee; base += 32) {
    const int cnt = (int)(s.ee - base < 32 ? s.ee - base : 32);
    if (lane < cnt) {
      const int64_t e = base + lane;
      const int64_t u = a.g.in_src[e];
#pragma unroll
      for (int h = 0; h < H; ++h) {
        const float ep = sddmm_add1(a.qS[u * H + h], sS, qd[h], sD);
        const float al = __fdiv_rn(exp_p(__fsub_rn(lrelu(ep, a.slope), mh[h])), dh[h]);
        const float dE = __fmul_rn(al, __fsub_rn(a.dalpha[e * H + h], P[h]));
        ba[lane][h] = ep > 0.0f ? dE : __fmul_rn(dE, a.slope);
      }
    }
    __syncwarp();
    if (lane < H)
      for (int i = 0; i < cnt; ++i) part = __fadd_rn(part, ba[i][lane]);
    __syncwarp();
  }
  return part;
}


// BD1 on a tile of light destination rows: pass 1 streams ∂α (IDP4A dot with the row's q_G slice,
// prefetched one row ahead) and P; pass 2 re-streams the tile for ∂E_pre and ∂D (lane j = row j).
template <int H, int VPL>
__device__ __forceinline__ void bwd_dst1_tile(const GatBwdArgs& a, int64_t r0, float (*ba)[H], float (*bd)[H],
                                              int* rb, float (*pt)[H], float sS, float sD, float sGH) {
  constexpr int LPH = 32 / H;
  const int lane = threadIdx.x & 31, myh = lane / LPH;
  const bool leader = (lane % LPH) == 0;
  int T;
  const TileLane L = tile_setup(a.g.in_ptr, a.pin.hbase, r0, a.g.n_local, T);
  const int64_t vg = a.g.row_begin + L.r;
  float mj[H], dj[H];
  int qdj[H];
#pragma unroll
  for (int h = 0; h < H; ++h) {
    mj[h] = L.deg > 0 ? a.m[vg * H + h] : 0.0f;
    dj[h] = L.deg > 0 ? a.den[vg * H + h] : 0.0f;
    qdj[h] = L.deg > 0 ? (int)a.qD[vg * H + h] : 0;
  }
  if (L.light && L.deg == 0) {
#pragma unroll
    for (int h = 0; h < H; ++h) { a.P[vg * H + h] = 0.0f; a.dD[vg * H + h] = 0.0f; }
  }
  const unsigned act = __ballot_sync(0xffffffffu, L.deg > 0);
  const int8_t* gbase = a.qG + lane * VPL;
  const int8_t* hbase = a.qHp + lane * VPL;
  const int64_t vg0 = a.g.row_begin + r0;
  int nxt = act ? __ffs(act) - 1 : -1;
  Row<VPL> gw_nxt{}, gw{};
  if (nxt >= 0) gw_nxt = load_row<VPL>(gbase + (vg0 + nxt) * a.ldG);
  float P = 0.0f;
  int cur = -1;
  // ---- pass 1
  for (int base = 0; base < T; base += 32) {
    const int cnt = T - base < 32 ? T - base : 32;
    const int t = base + lane;
    const int row = tile_row(t, L.end);
    const int64_t ebr = __shfl_sync(0xffffffffu, L.eb, row);
    const int offr = __shfl_sync(0xffffffffu, L.off, row);
    float mr[H], dr[H];
    int qdr[H];
#pragma unroll
    for (int h = 0; h < H; ++h) {
      mr[h] = __shfl_sync(0xffffffffu, mj[h], row);
      dr[h] = __shfl_sync(0xffffffffu, dj[h], row);
      qdr[h] = __shfl_sync(0xffffffffu, qdj[h], row);
    }
    int u = 0;
    const int64_t e = ebr + (t - offr);
    if (lane < cnt) {
      u = a.g.in_src[e];
#pragma unroll
      for (int h = 0; h < H; ++h)
        ba[lane][h] = __fdiv_rn(
            exp_p(__fsub_rn(lrelu(sddmm_add1(a.qS[(int64_t)u * H + h], sS, (int8_t)qdr[h], sD), a.slope), mr[h])),
            dr[h]);
      rb[lane] = row;
    }
    __syncwarp();
    for (int i0 = 0; i0 < cnt; i0 += UNR) {
      Row<VPL> rr[UNR];
#pragma unroll
      for (int j = 0; j < UNR; ++j) {
        const int w = __shfl_sync(0xffffffffu, u, (i0 + j) & 31);
        if (i0 + j < cnt) rr[j] = load_row<VPL>(hbase + (int64_t)w * a.ldHp);
      }
#pragma unroll
      for (int j = 0; j < UNR; ++j) {
        if (i0 + j < cnt) {
          const int ri = rb[i0 + j];
          if (ri != cur) {
            if (cur >= 0 && leader) pt[cur][myh] = P;
            P = 0.0f;
            cur = ri;
            gw = gw_nxt;
            nxt = tile_next(act, cur);
            if (nxt >= 0) gw_nxt = load_row<VPL>(gbase + (vg0 + nxt) * a.ldG);
          }
          int dot = row_dot<VPL>(gw, rr[j]);
#pragma unroll
          for (int o = 1; o < LPH; o <<= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
          if (leader) {
            const float dal = __fmul_rn(__int2float_rn(dot), sGH);
            P = __fmaf_rn(dal, ba[i0 + j][myh], P);
            bd[i0 + j][myh] = dal;
          }
        }
      }
    }
    __syncwarp();
    if (lane < cnt) {
#pragma unroll
      for (int h = 0; h < H; ++h) a.dalpha[e * H + h] = bd[lane][h];
    }
    __syncwarp();
  }
  if (cur >= 0 && leader) pt[cur][myh] = P;
  __syncwarp();
  // ---- pass 2
  float dDp[H];
#pragma unroll
  for (int h = 0; h < H; ++h) dDp[h] = 0.0f;
  for (int base = 0; base < T; base += 32) {
    const int cnt = T - base < 32 ? T - base : 32;
    const int t = base + lane;
    const int row = tile_row(t, L.end);
    const int64_t ebr = __shfl_sync(0xffffffffu, L.eb, row);
    const int offr = __shfl_sync(0xffffffffu, L.off, row);
    float mr[H], dr[H];
    int qdr[H];
#pragma unroll
    for (int h = 0; h < H; ++h) {
      mr[h] = __shfl_sync(0xffffffffu, mj[h], row);
      dr[h] = __shfl_sync(0xffffffffu, dj[h], row);
      qdr[h] = __shfl_sync(0xffffffffu, qdj[h], row);
    }
    if (lane < cnt) {
      const int64_t e = ebr + (t - offr);
      const int64_t u = a.g.in_src[e];
#pragma unroll
      for (int h = 0; h < H; ++h) {
        const float ep = sddmm_add1(a.qS[u * H + h], sS, (int8_t)qdr[h], sD);
        const float al = __fdiv_rn(exp_p(__fsub_rn(lrelu(ep, a.slope), mr[h])), dr[h]);
        const float dE = __fmul_rn(al, __fsub_rn(a.dalpha[e * H + h], pt[row][h]));
        ba[lane][h] = ep > 0.0f ? dE : __fmul_rn(dE, a.slope);
      }
    }
    __syncwarp();
    const int lo = (L.off > base ? L.off : base) - base;
    const int hi = (L.end < base + cnt ? L.end : base + cnt) - base;
    for (int i = lo; i < hi; ++i)
#pragma unroll
      for (int h = 0; h < H; ++h) dDp[h] = __fadd_rn(dDp[h], ba[i][h]);
    __syncwarp();
  }
  if (L.deg > 0) {
#pragma unroll
    for (int h = 0; h < H; ++h) { a.P[vg * H + h] = pt[lane][h]; a.dD[vg * H + h] = dDp[h]; }
  }
  __syncwarp();
}

// BD1: light rows -> ∂α, P, ∂D final; heavy segments -> ∂α, P partial (hP)
template <int H, int VPL>
__global__ void __launch_bounds__(256, 2) k_bwd_dst1(const GatBwdArgs a) {
  constexpr int LPH = 32 / H;
  __shared__ float sh_a[WPB][32][H];
  __shared__ float sh_d[WPB][32][H];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Scale scS = scale_from_amax(amax_load(a.amax_S), a.bits);
  const Scale scD = scale_from_amax(amax_load(a.amax_D), a.bits);
  const Scale scH = scale_from_amax(amax_load(a.amax_Hp), a.bits);
  const Scale scG = scale_from_amax(amax_load(a.amax_G), a.bits);
  const float sGH = __fmul_rn(scG.s, scH.s);
  const int64_t hc = load_count(a.pin.counts), nitems = hc + (a.g.n_local + TILE - 1) / TILE;
  __shared__ int sh_rb[WPB][32];
  __shared__ float sh_pt[WPB][32][H];
  FOR_ITEMS(item, a.work + 0, nitems) {
    if (item >= hc) {
      bwd_dst1_tile<H, VPL>(a, (item - hc) * TILE, sh_a[w], sh_d[w], sh_rb[w], sh_pt[w], scS.s, scD.s, sGH);
      continue;
    }
    Seg s;
    if (!decode_item(item, hc, a.g.in_ptr, a.pin, a.g.chunk, s)) continue;
    const int64_t vg = a.g.row_begin + s.vl;
    int8_t qd[H];
    float mh[H], dh[H];
#pragma unroll
    for (int h = 0; h < H; ++h) { qd[h] = a.qD[vg * H + h]; mh[h] = a.m[vg * H + h]; dh[h] = a.den[vg * H + h]; }
    const Row<VPL> gw = load_row<VPL>(a.qG + vg * a.ldG + lane * VPL);
    const float Pl = bwd_dst_pass1<H, VPL>(a, s, qd, mh, dh, gw, scS.s, scD.s, sGH, sh_a[w], sh_d[w]);
    if (s.slot >= 0) {
      if ((lane % LPH) == 0) a.hP[(int64_t)s.slot * H + lane / LPH] = Pl;
      continue;
    }
    float P[H];
#pragma unroll
    for (int h = 0; h < H; ++h) P[h] = __shfl_sync(0xffffffffu, Pl, h * LPH);
    const float dD = bwd_dst_pass2<H>(a, s, qd, mh, dh, P, scS.s, scD.s, sh_a[w]);
    if (lane < H) {
      a.P[vg * H + lane] = head_pick<H>(P, lane);
      a.dD[vg * H + lane] = dD;
    }
  }
}

// BD2: heavy segments -> P (fold of hP; segment 0 writes it), ∂D partial (hdD)
template <int H>
__global__ void __launch_bounds__(256) k_bwd_dst2(const GatBwdArgs a) {
  __shared__ float sh_a[WPB][32][H];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Scale scS = scale_from_amax(amax_load(a.amax_S), a.bits);
  const Scale scD = scale_from_amax(amax_load(a.amax_D), a.bits);
  const int64_t hcnt = load_count(a.pin.counts);
  FOR_ITEMS(si, a.work + 1, hcnt) {
    Seg s;
    decode_item(si, hcnt, a.g.in_ptr, a.pin, a.g.chunk, s);
    const int64_t vg = a.g.row_begin + s.vl;
    int8_t qd[H];
    float mh[H], dh[H], P[H];
#pragma unroll
    for (int h = 0; h < H; ++h) { qd[h] = a.qD[vg * H + h]; mh[h] = a.m[vg * H + h]; dh[h] = a.den[vg * H + h]; }
    float tot = 0.0f;
    if (lane < H) {
      tot = a.hP[(int64_t)s.base * H + lane];
      for (int j = 1; j < s.nseg; ++j) tot = __fadd_rn(tot, a.hP[(int64_t)(s.base + j) * H + lane]);
      if (s.c == 0) a.P[vg * H + lane] = tot;
    }
#pragma unroll
    for (int h = 0; h < H; ++h) P[h] = __shfl_sync(0xffffffffu, tot, h);
    const float dDp = bwd_dst_pass2<H>(a, s, qd, mh, dh, P, scS.s, scD.s, sh_a[w]);
    if (lane < H) a.hdD[si * H + lane] = dDp;
  }
}

// BD3: heavy rows -> ∂D = fold of hdD
template <int H>
__global__ void __launch_bounds__(256) k_bwd_dst3(const GatBwdArgs a) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t hrows = load_count(a.pin.counts + 1);
  if (t >= hrows * H) return;
  const int64_t vl = a.pin.hrow[t / H];
  const int h = (int)(t % H);
  const int base = a.pin.hbase[vl];
  const int64_t deg = a.g.in_ptr[vl + 1] - a.g.in_ptr[vl];
  const int nseg = (int)((deg + a.g.chunk - 1) / a.g.chunk);
  float tot = a.hdD[(int64_t)base * H + h];
  for (int j = 1; j < nseg; ++j) tot = __fadd_rn(tot, a.hdD[(int64_t)(base + j) * H + h]);
  a.dD[(a.g.row_begin + vl) * H + h] = tot;
}

// ================================================================== backward, source side
// One segment of u's out-edges: recompute α, e_pre, ∂α, ∂E_pre per out-edge (u→v) from per-node
// data; ∂S partial (leaders) and the ⑤′ aggregation partial Σ fmaf(α, q_G[v]).
template <int H, int VPL>
__device__ __forceinline__ float bwd_src_seg(const GatBwdArgs& a, const Seg& s, const int8_t (&qs)[H],
                                             const Row<VPL>& hw, float sS, float sD, float sGH, float (*ba)[H],
                                             float (*be)[H], float (*bp)[H], float (&part)[VPL]) {
  constexpr int LPH = 32 / H;
  const int lane = threadIdx.x & 31;
  const int myh = lane / LPH;
  const bool leader = (lane % LPH) == 0;
  float dS = 0.0f;
  const int8_t* gbase = a.qG + lane * VPL;
  for (int64_t base = s.eb; base < s.ee; base += 32) {
    const int cnt = (int)(s.ee - base < 32 ? s.ee - base : 32);
    int v = 0;
    if (lane < cnt) {
      v = a.g.out_dst[base + lane];
#pragma unroll
      for (int h = 0; h < H; ++h) {
        const int64_t k = (int64_t)v * H + h;
        const float ep = sddmm_add1(qs[h], sS, a.qD[k], sD);
        ba[lane][h] = __fdiv_rn(exp_p(__fsub_rn(lrelu(ep, a.slope), a.m[k])), a.den[k]);
        be[lane][h] = ep;
        bp[lane][h] = a.P[k];
      }
    }
    __syncwarp();
    for (int i0 = 0; i0 < cnt; i0 += UNR) {
      Row<VPL> r[UNR];
#pragma unroll
      for (int j = 0; j < UNR; ++j) {
        const int vv = __shfl_sync(0xffffffffu, v, (i0 + j) & 31);
        if (i0 + j < cnt) r[j] = load_row<VPL>(gbase + (int64_t)vv * a.ldG);
      }
#pragma unroll
      for (int j = 0; j < UNR; ++j) {
        if (i0 + j < cnt) {
          int dot = row_dot<VPL>(r[j], hw);
#pragma unroll
          for (int o = 1; o < LPH; o <<= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
          const float al = ba[i0 + j][myh];
          if (leader) {
            const float dal = __fmul_rn(__int2float_rn(dot), sGH);
            const float dE = __fmul_rn(al, __fsub_rn(dal, bp[i0 + j][myh]));
            dS = __fadd_rn(dS, be[i0 + j][myh] > 0.0f ? dE : __fmul_rn(dE, a.slope));
          }
#pragma unroll
          for (int q = 0; q < (VPL + 3) / 4; ++q) {
            const uint32_t wx = r[j].w[q] ^ 0x80808080u;
#pragma unroll
            for (int k = 0; k < 4 && q * 4 + k < VPL; ++k) part[q * 4 + k] = __fmaf_rn(al, bx2f(wx, k), part[q * 4 + k]);
          }
        }
      }
    }
    __syncwarp();
  }
  return dS;
}

// ②′ finalize of source row u: ∂H′ = (agg·s_G + ∂S·a_src) + ∂D·a_dst ; ∂S stored for the ∂a pass
template <int VPL>
__device__ __forceinline__ void bwd_src_finalize(const GatBwdArgs& a, int64_t ul, int64_t ug, int myh, float dS,
                                                 const float (&sum)[VPL], float sG, float& amax_loc, int H) {
  constexpr int HD = 32 * VPL;
  const int lane = threadIdx.x & 31;
  const float dD = a.dD[ug * H + myh];
  float* dst = a.dHp + ul * HD + lane * VPL;
  const float* asrc = a.a_src + lane * VPL;
  const float* adst = a.a_dst + lane * VPL;
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    const float agg = __fmul_rn(sum[k], sG);
    const float t2 = __fadd_rn(agg, __fmul_rn(dS, __ldg(asrc + k)));
    const float o = __fadd_rn(t2, __fmul_rn(dD, __ldg(adst + k)));
    amax_loc = fmaxf(amax_loc, fabsf(o));
    dst[k] = o;
  }
  if ((lane % (32 / H)) == 0) a.dS[ug * H + myh] = dS;
}

__device__ __forceinline__ void amax_flush(unsigned* slot, float amax_loc) {
  amax_loc = warp_max(amax_loc);
  if ((threadIdx.x & 31) == 0 && slot) atomicMax(slot, __float_as_uint(amax_loc));
}

// BS on a tile of light source rows: per out-edge (u→v) recompute α, e_pre, ∂α, ∂E_pre; stream
// the q_G[v] gathers across rows (own q_H′[u] slice prefetched one row ahead); finalize at row change.
template <int H, int VPL>
__device__ __forceinline__ void bwd_src_tile(const GatBwdArgs& a, int64_t r0, float (*ba)[H], float (*be)[H],
                                             float (*bp)[H], int* rb, float sS, float sD, float sGH, float sG,
                                             float& amax_loc) {
  constexpr int LPH = 32 / H;
  const int lane = threadIdx.x & 31, myh = lane / LPH;
  const bool leader = (lane % LPH) == 0;
  int T;
  const TileLane L = tile_setup(a.g.out_ptr, a.pout.hbase, r0, a.g.n_local, T);
  const int64_t ug0 = a.g.row_begin + r0;
  int qsj[H];
#pragma unroll
  for (int h = 0; h < H; ++h) qsj[h] = L.deg > 0 ? (int)a.qS[(ug0 + lane) * H + h] : 0;
  const int8_t* gbase = a.qG + lane * VPL;
  const int8_t* hbase = a.qHp + lane * VPL;
  float zero[VPL];
#pragma unroll
  for (int k = 0; k < VPL; ++k) zero[k] = 0.0f;
  unsigned zm = __ballot_sync(0xffffffffu, L.light && L.deg == 0);
  while (zm) {   // light rows without out-edges: ∂H′ = (0 + 0·a_src) + ∂D·a_dst
    const int j = __ffs(zm) - 1;
    zm &= zm - 1;
    bwd_src_finalize<VPL>(a, r0 + j, ug0 + j, myh, 0.0f, zero, sG, amax_loc, H);
  }
  const unsigned act = __ballot_sync(0xffffffffu, L.deg > 0);
  int nxt = act ? __ffs(act) - 1 : -1;
  Row<VPL> hw_nxt{}, hw{};
  if (nxt >= 0) hw_nxt = load_row<VPL>(hbase + (ug0 + nxt) * a.ldHp);
  float part[VPL];
#pragma unroll
  for (int k = 0; k < VPL; ++k) part[k] = 0.0f;
  float dS = 0.0f;
  int cur = -1;
  auto flush = [&](int j) {
    const float dSb = __shfl_sync(0xffffffffu, dS, myh * LPH);
    bwd_src_finalize<VPL>(a, r0 + j, ug0 + j, myh, dSb, part, sG, amax_loc, H);
#pragma unroll
    for (int k = 0; k < VPL; ++k) part[k] = 0.0f;
    dS = 0.0f;
  };
  for (int base = 0; base < T; base += 32) {
    const int cnt = T - base < 32 ? T - base : 32;
    const int t = base + lane;
    const int row = tile_row(t, L.end);
    const int64_t ebr = __shfl_sync(0xffffffffu, L.eb, row);
    const int offr = __shfl_sync(0xffffffffu, L.off, row);
    int qsr[H];
#pragma unroll
    for (int h = 0; h < H; ++h) qsr[h] = __shfl_sync(0xffffffffu, qsj[h], row);
    int v = 0;
    if (lane < cnt) {
      v = a.g.out_dst[ebr + (t - offr)];
#pragma unroll
      for (int h = 0; h < H; ++h) {
        const int64_t k = (int64_t)v * H + h;
        const float ep = sddmm_add1((int8_t)qsr[h], sS, a.qD[k], sD);
        ba[lane][h] = __fdiv_rn(exp_p(__fsub_rn(lrelu(ep, a.slope), a.m[k])), a.den[k]);
        be[lane][h] = ep;
        bp[lane][h] = a.P[k];
      }
      rb[lane] = row;
    }
    __syncwarp();
    for (int i0 = 0; i0 < cnt; i0 += UNR) {
      Row<VPL> rr[UNR];
#pragma unroll
      for (int j = 0; j < UNR; ++j) {
        const int vv = __shfl_sync(0xffffffffu, v, (i0 + j) & 31);
        if (i0 + j < cnt) rr[j] = load_row<VPL>(gbase + (int64_t)vv * a.ldG);
      }
#pragma unroll
      for (int j = 0; j < UNR; ++j) {
        if (i0 + j < cnt) {
          const int ri = rb[i0 + j];
          if (ri != cur) {
            if (cur >= 0) flush(cur);
            cur = ri;
            hw = hw_nxt;
            nxt = tile_next(act, cur);
            if (nxt >= 0) hw_nxt = load_row<VPL>(hbase + (ug0 + nxt) * a.ldHp);
          }
          int dot = row_dot<VPL>(rr[j], hw);
#pragma unroll
          for (int o = 1; o < LPH; o <<= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
          const float al = ba[i0 + j][myh];
          if (leader) {
            const float dal = __fmul_rn(__int2float_rn(dot), sGH);
            const float dE = __fmul_rn(al, __fsub_rn(dal, bp[i0 + j][myh]));
            dS = __fadd_rn(dS, be[i0 + j][myh] > 0.0f ? dE : __fmul_rn(dE, a.slope));
          }
#pragma unroll
          for (int q = 0; q < (VPL + 3) / 4; ++q) {
            const uint32_t wx = rr[j].w[q] ^ 0x80808080u;
#pragma unroll
            for (int k = 0; k < 4 && q * 4 + k < VPL; ++k) part[q * 4 + k] = __fmaf_rn(al, bx2f(wx, k), part[q * 4 + k]);
          }
        }
      }
    }
    __syncwarp();
  }
  if (cur >= 0) flush(cur);
}

// BS: light out-rows (tiles) -> ∂H′ final; heavy out-segments -> ∂S, aggregation partials
template <int H, int VPL>
__global__ void __launch_bounds__(256, 2) k_bwd_src(const GatBwdArgs a) {
  constexpr int LPH = 32 / H;
  constexpr int HD = 32 * VPL;
  __shared__ float sh_a[WPB][32][H];
  __shared__ float sh_e[WPB][32][H];
  __shared__ float sh_p[WPB][32][H];
  __shared__ int sh_rb[WPB][32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Scale scS = scale_from_amax(amax_load(a.amax_S), a.bits);
  const Scale scD = scale_from_amax(amax_load(a.amax_D), a.bits);
  const Scale scH = scale_from_amax(amax_load(a.amax_Hp), a.bits);
  const Scale scG = scale_from_amax(amax_load(a.amax_G), a.bits);
  const float sGH = __fmul_rn(scG.s, scH.s);
  float amax_loc = 0.0f;
  const int64_t hc = load_count(a.pout.counts), nitems = hc + (a.g.n_local + TILE - 1) / TILE;
  FOR_ITEMS(item, a.work + 2, nitems) {
    if (item >= hc) {
      bwd_src_tile<H, VPL>(a, (item - hc) * TILE, sh_a[w], sh_e[w], sh_p[w], sh_rb[w], scS.s, scD.s, sGH, scG.s,
                           amax_loc);
      continue;
    }
    Seg s;
    decode_item(item, hc, a.g.out_ptr, a.pout, a.g.chunk, s);
    const int64_t ug = a.g.row_begin + s.vl;
    int8_t qs[H];
#pragma unroll
    for (int h = 0; h < H; ++h) qs[h] = a.qS[ug * H + h];
    const Row<VPL> hw = load_row<VPL>(a.qHp + ug * a.ldHp + lane * VPL);
    float part[VPL];
#pragma unroll
    for (int k = 0; k < VPL; ++k) part[k] = 0.0f;
    const float dSl = bwd_src_seg<H, VPL>(a, s, qs, hw, scS.s, scD.s, sGH, sh_a[w], sh_e[w], sh_p[w], part);
    if ((lane % LPH) == 0) a.hdS[(int64_t)s.slot * H + lane / LPH] = dSl;
    float* dst = a.hagg + (int64_t)s.slot * HD + lane * VPL;
#pragma unroll
    for (int k = 0; k < VPL; ++k) dst[k] = part[k];
  }
  amax_flush(a.amax_dHp, amax_loc);
}

// BC: heavy out-rows -> fold ∂S and aggregation partials in chunk order, finalize ∂H′
template <int H, int VPL>
__global__ void __launch_bounds__(256) k_bwd_src_combine(const GatBwdArgs a) {
  constexpr int LPH = 32 / H;
  constexpr int HD = 32 * VPL;
  const int lane = threadIdx.x & 31;
  const int myh = lane / LPH;
  const Scale scG = scale_from_amax(amax_load(a.amax_G), a.bits);
  float amax_loc = 0.0f;
  const int64_t hrows = load_count(a.pout.counts + 1);
  FOR_ITEMS(r, a.work + 3, hrows) {
    const int64_t ul = a.pout.hrow[r];
    const int64_t ug = a.g.row_begin + ul;
    const int base = a.pout.hbase[ul];
    const int64_t deg = a.g.out_ptr[ul + 1] - a.g.out_ptr[ul];
    const int nseg = (int)((deg + a.g.chunk - 1) / a.g.chunk);
    float dS = a.hdS[(int64_t)base * H + myh];
    for (int j = 1; j < nseg; ++j) dS = __fadd_rn(dS, a.hdS[(int64_t)(base + j) * H + myh]);
    float tot[VPL];
    const float* src = a.hagg + (int64_t)base * HD + lane * VPL;
#pragma unroll
    for (int k = 0; k < VPL; ++k) tot[k] = src[k];
    for (int j = 1; j < nseg; ++j) {
      const float* p = src + (int64_t)j * HD;
#pragma unroll
      for (int k = 0; k < VPL; ++k) tot[k] = __fadd_rn(tot[k], p[k]);
    }
    bwd_src_finalize<VPL>(a, ul, ug, myh, dS, tot, scG.s, amax_loc, H);
  }
  amax_flush(a.amax_dHp, amax_loc);
}

// ②′ for the attention vectors (reading R23): ∂a_src[j] = Σ_u ∂S[u,h(j)]·deq(q_H′)[u,j],
// ∂a_dst likewise with ∂D.  A streaming reduction over the owned rows (q_H′ read once, coalesced);
// summation order is free (fp32 atomics), checked against the oracle within the derived bound.
template <int H, int VPL>
__global__ void __launch_bounds__(256) k_bwd_attn_grad(const GatBwdArgs a) {
  constexpr int LPH = 32 / H;
  constexpr int HD = 32 * VPL;
  __shared__ float sh_da[2][HD];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int myh = lane / LPH;
  for (int j = threadIdx.x; j < 2 * HD; j += blockDim.x) (&sh_da[0][0])[j] = 0.0f;
  __syncthreads();
  const Scale scH = scale_from_amax(amax_load(a.amax_Hp), a.bits);
  float das[VPL], dad[VPL];
#pragma unroll
  for (int k = 0; k < VPL; ++k) { das[k] = 0.0f; dad[k] = 0.0f; }
  for (int64_t ul = (int64_t)blockIdx.x * WPB + w; ul < a.g.n_local; ul += (int64_t)gridDim.x * WPB) {
    const int64_t ug = a.g.row_begin + ul;
    const float dS = a.dS[ug * H + myh];
    const float dD = a.dD[ug * H + myh];
    const Row<VPL> hw = load_row<VPL>(a.qHp + ug * a.ldHp + lane * VPL);
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const float hp = __fmul_rn(row_f<VPL>(hw, k), scH.s);
      das[k] = __fmaf_rn(dS, hp, das[k]);
      dad[k] = __fmaf_rn(dD, hp, dad[k]);
    }
  }
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    atomicAdd(&sh_da[0][lane * VPL + k], das[k]);
    atomicAdd(&sh_da[1][lane * VPL + k], dad[k]);
  }
  __syncthreads();
  for (int j = threadIdx.x; j < HD; j += blockDim.x) {
    atomicAdd(a.da_src + j, sh_da[0][j]);
    atomicAdd(a.da_dst + j, sh_da[1][j]);
  }
}

// ------------------------------------------------------------------ dispatch
static int item_grid(int64_t items) {
  int64_t g = (items + WPB - 1) / WPB;
  const int64_t cap = (int64_t)num_sms() * 4;     // >= resident blocks; the work queue balances
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

#define TANGO_HV_CASES(X) X(1, 2) X(1, 4) X(1, 8) X(1, 16) X(2, 2) X(2, 4) X(2, 8) X(2, 16) \
                          X(4, 2) X(4, 4) X(4, 8) X(4, 16) X(8, 2) X(8, 4) X(8, 8) X(8, 16)

cudaError_t launch_gat_fwd(const GatFwdArgs& a, cudaStream_t st) {
  if (a.g.n_local == 0) return cudaSuccess;
  const int hv = a.d.heads * 100 + a.d.hd / 32;
  const int64_t items = a.g.n_local + a.plan.cap;
  bool ok = false;
#define X(H_, V_)                                                                                  \
  if (hv == H_ * 100 + V_) {                                                                       \
    ok = true;                                                                                     \
    { ProfScope p("gat_fwd_stats", st);  k_fwd_stats<H_><<<item_grid(items), 256, 0, st>>>(a); }   \
    { ProfScope p("gat_fwd_stats2", st); k_fwd_stats2<H_><<<item_grid(a.plan.cap), 256, 0, st>>>(a); } \
    { ProfScope p("gat_fwd_agg", st);    k_fwd_agg<H_, V_><<<item_grid(items), 256, 0, st>>>(a); }  \
    { ProfScope p("gat_fwd_combine", st); k_fwd_combine<H_, V_><<<item_grid(a.g.n_local), 256, 0, st>>>(a); } \
  }
  TANGO_HV_CASES(X)
#undef X
  if (!ok) return cudaErrorInvalidValue;
  return cudaGetLastError();
}

cudaError_t launch_gat_bwd_dst(const GatBwdArgs& a, cudaStream_t st) {
  if (a.g.n_local == 0) return cudaSuccess;
  const int hv = a.d.heads * 100 + a.d.hd / 32;
  const int64_t items = a.g.n_local + a.pin.cap;
  bool ok = false;
#define X(H_, V_)                                                                                  \
  if (hv == H_ * 100 + V_) {                                                                       \
    ok = true;                                                                                     \
    { ProfScope p("gat_bwd_dst1", st); k_bwd_dst1<H_, V_><<<item_grid(items), 256, 0, st>>>(a); }  \
    { ProfScope p("gat_bwd_dst2", st); k_bwd_dst2<H_><<<item_grid(a.pin.cap), 256, 0, st>>>(a); }  \
    { ProfScope p("gat_bwd_dst3", st);                                                             \
      k_bwd_dst3<H_><<<(unsigned)((a.g.n_local * H_ + 255) / 256), 256, 0, st>>>(a); }            \
  }
  TANGO_HV_CASES(X)
#undef X
  if (!ok) return cudaErrorInvalidValue;
  return cudaGetLastError();
}

cudaError_t launch_gat_bwd_src(const GatBwdArgs& a, cudaStream_t st) {
  if (a.g.n_local == 0) return cudaSuccess;
  const int hv = a.d.heads * 100 + a.d.hd / 32;
  const int64_t items = a.g.n_local + a.pout.cap;
  bool ok = false;
#define X(H_, V_)                                                                                  \
  if (hv == H_ * 100 + V_) {                                                                       \
    ok = true;                                                                                     \
    { ProfScope p("gat_bwd_src", st); k_bwd_src<H_, V_><<<item_grid(items), 256, 0, st>>>(a); }    \
    { ProfScope p("gat_bwd_src_combine", st);                                                      \
      k_bwd_src_combine<H_, V_><<<item_grid(a.g.n_local), 256, 0, st>>>(a); }                     \
    { ProfScope p("gat_bwd_attn_grad", st);                                                        \
      k_bwd_attn_grad<H_, V_><<<num_sms() * 2, 256, 0, st>>>(a); }                                 \
  }
  TANGO_HV_CASES(X)
#undef X
  if (!ok) return cudaErrorInvalidValue;
  return cudaGetLastError();
}

}  // namespace tango
