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
//  * Light rows are processed in tiles of 32 consecutive rows streamed as one edge sequence, and
//    the three gather passes are split into head groups (one warp per group of WC = 32*VPL columns)
//    so a warp gathers one 128-B line per edge with a 16-deep pipeline at low register cost.
#include "gat_common.cuh"
#include <cstdlib>
#include <cstring>

namespace tango {


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

// Edge-balanced sub-tiles of light rows: each 32-row block is cut into runs of rows whose first
// edge falls in the same BIN-edge window, so a work item holds at most BIN + C_E edges.  Items are
// encoded (block << 10) | (lo << 5) | (hi - 1) for rows [32*block + lo, 32*block + hi).
constexpr int TILE_BIN = 128;
__global__ void k_plan_tiles(const int64_t* __restrict__ ptr, int64_t n, PlanDev p) {
  const int lane = threadIdx.x & 31;
  const int64_t b = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (b * 32 >= n) return;
  const int64_t r = b * 32 + lane;
  const bool has = r < n;
  const bool light = has && p.hbase[r] < 0;
  const int deg = light ? (int)(ptr[r + 1] - ptr[r]) : 0;
  int cum = deg;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, cum, o);
    if (lane >= o) cum += y;
  }
  const int key = (cum - deg) / TILE_BIN;
  const int prev = __shfl_up_sync(0xffffffffu, key, 1);
  const unsigned starts = __ballot_sync(0xffffffffu, has && (lane == 0 || key != prev));
  const unsigned valid = __ballot_sync(0xffffffffu, has);
  const int nrun = __popc(starts);
  int slot = 0;
  if (lane == 0) slot = atomicAdd(&p.counts[2], nrun);
  slot = __shfl_sync(0xffffffffu, slot, 0);
  if (starts & (1u << lane)) {
    const unsigned later = lane >= 31 ? 0u : (starts & ~((2u << lane) - 1u));
    const int hi = later ? __ffs(later) - 1 : 32 - __clz(valid);
    const int idx = __popc(starts & ((1u << lane) - 1u));
    p.tiles[slot + idx] = (int32_t)((b << 10) | (lane << 5) | (hi - 1));
  }
}
cudaError_t launch_plan_tiles(const int64_t* ptr, int64_t n, const PlanDev& p, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  ProfScope ps("plan_tiles", st);
  const int64_t blocks = (n + 31) / 32;
  k_plan_tiles<<<(unsigned)((blocks * 32 + 255) / 256), 256, 0, st>>>(ptr, n, p);
  return cudaGetLastError();
}


constexpr int SEGB = 8;   // 32-edge chunks loaded per batch (256 edges)
template <int H>
__host__ __device__ constexpr int segb() { return H >= 8 ? 4 : SEGB; }   // staging fits 48 KB static smem

// max over the segment of el = lrelu(e_pre) (lane-parallel; order-free), all lanes get the result
template <int H>
__device__ __forceinline__ void seg_max(const int32_t* __restrict__ src, int64_t eb, int64_t ee,
                                        const int8_t* __restrict__ qS, float sS, const int8_t (&qd)[H], float sD,
                                        float slope, float (&mx)[H]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int h = 0; h < H; ++h) mx[h] = -INFINITY;
  for (int64_t base = eb; base < ee; base += 32 * SEGB) {
    int u[SEGB];
#pragma unroll
    for (int i = 0; i < SEGB; ++i) {
      const int64_t e = base + i * 32 + lane;
      u[i] = e < ee ? src[e] : -1;
    }
    int8_t qs[SEGB][H];
#pragma unroll
    for (int i = 0; i < SEGB; ++i)
      if (u[i] >= 0) load_qh<H>(qS + (int64_t)u[i] * H, qs[i]);
#pragma unroll
    for (int i = 0; i < SEGB; ++i)
      if (u[i] >= 0)
#pragma unroll
        for (int h = 0; h < H; ++h) mx[h] = fmaxf(mx[h], lrelu(sddmm_add1(qs[i][h], sS, qd[h], sD), slope));
  }
#pragma unroll
  for (int h = 0; h < H; ++h) mx[h] = warp_max(mx[h]);
}

// Σ over the segment of exp_p(el - m), sequential in edge order (one chunk: no folding).
// Returns the sum for head `lane` in lanes < H.  Stores ex with the sign of e_pre (the LeakyReLU
// branch) into sx[e][h] (stride 2H).  buf: per-warp [32*SEGB][H] staging.
template <int H>
__device__ __forceinline__ float seg_sum_exp(const int32_t* __restrict__ src, int64_t eb, int64_t ee,
                                             const int8_t* __restrict__ qS, float sS, const int8_t (&qd)[H],
                                             float sD, float slope, const float (&mx)[H], float (*buf)[H],
                                             float* __restrict__ sx) {
  const int lane = threadIdx.x & 31;
  float part = 0.0f;
  for (int64_t base = eb; base < ee; base += 32 * segb<H>()) {
    int u[segb<H>()];
#pragma unroll
    for (int i = 0; i < segb<H>(); ++i) {
      const int64_t e = base + i * 32 + lane;
      u[i] = e < ee ? src[e] : -1;
    }
    int8_t qs[segb<H>()][H];
#pragma unroll
    for (int i = 0; i < segb<H>(); ++i)
      if (u[i] >= 0) load_qh<H>(qS + (int64_t)u[i] * H, qs[i]);
#pragma unroll
    for (int i = 0; i < segb<H>(); ++i) {
      if (u[i] < 0) continue;
      const int64_t e = base + i * 32 + lane;
      float o[H];
#pragma unroll
      for (int h = 0; h < H; ++h) {
        const float ep = sddmm_add1(qs[i][h], sS, qd[h], sD);
        const float ex = exp_p(__fsub_rn(lrelu(ep, slope), mx[h]));
        buf[i * 32 + lane][h] = ex;
        o[h] = ep > 0.0f ? ex : -ex;
      }
      if constexpr (H == 4) {
        *reinterpret_cast<float4*>(sx + e * 8) = make_float4(o[0], o[1], o[2], o[3]);
      } else {
#pragma unroll
        for (int h = 0; h < H; ++h) sx[e * 2 * H + h] = o[h];
      }
    }
    __syncwarp();
    const int cnt = (int)(ee - base < 32 * segb<H>() ? ee - base : 32 * segb<H>());
    if (lane < H)
      for (int i = 0; i < cnt; ++i) part = __fadd_rn(part, buf[i][lane]);
    __syncwarp();
  }
  return part;
}

// Left fold x[base + 0] + x[base + 1] + ... (segment order) of per-segment scalars [slot][H], all
// heads, all lanes get the result.  Lanes load one segment each; the fold runs over shuffles.
template <int H>
__device__ __forceinline__ void fold_segments(const float* __restrict__ x, int base, int nseg, float (&tot)[H]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int h = 0; h < H; ++h) tot[h] = 0.0f;
  for (int j0 = 0; j0 < nseg; j0 += 32) {
    const int j = j0 + lane;
    float v[H];
#pragma unroll
    for (int h = 0; h < H; ++h) v[h] = j < nseg ? x[(int64_t)(base + j) * H + h] : 0.0f;
    const int cnt = nseg - j0 < 32 ? nseg - j0 : 32;
    for (int i = 0; i < cnt; ++i)
#pragma unroll
      for (int h = 0; h < H; ++h) {
        const float y = __shfl_sync(0xffffffffu, v[h], i);
        tot[h] = (j0 + i == 0) ? y : __fadd_rn(tot[h], y);
      }
  }
}

// Left fold of nseg per-segment row slices (this lane's VPL floats at src + j*stride), 4 in flight
template <int VPL>
__device__ __forceinline__ void fold_rows(const float* __restrict__ src, int64_t stride, int nseg,
                                          float (&tot)[VPL]) {
#pragma unroll
  for (int k = 0; k < VPL; ++k) tot[k] = src[k];
  for (int j = 1; j < nseg; j += 4) {
    float b[4][VPL];
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (j + q < nseg) {
        const float* p = src + (j + q) * stride;
        if constexpr (VPL % 4 == 0) {
#pragma unroll
          for (int k = 0; k < VPL / 4; ++k) {
            const float4 v = *reinterpret_cast<const float4*>(p + 4 * k);
            b[q][4 * k] = v.x; b[q][4 * k + 1] = v.y; b[q][4 * k + 2] = v.z; b[q][4 * k + 3] = v.w;
          }
        } else {
#pragma unroll
          for (int k = 0; k < VPL; ++k) b[q][k] = p[k];
        }
      }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (j + q < nseg)
#pragma unroll
        for (int k = 0; k < VPL; ++k) tot[k] = __fadd_rn(tot[k], b[q][k]);
  }
}

// m = max over a heavy row's segment maxima, den = left fold of its segment sums, all lanes
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
  if (hden) fold_segments<H>(hden, base, nseg, den);
}

// exact int8 -> fp32 of byte k of a word pre-XORed with 0x80808080: 2^23 + 128 + q - (2^23 + 128)
__device__ __forceinline__ float bx2f(uint32_t wx, int k) {
  return __fsub_rn(__uint_as_float(__byte_perm(wx, 0x4B000000u, 0x7440u | (uint32_t)k)), 8388736.0f);
}

// ================================================================== forward

// FS (tiles): heavy segments -> segment max (hmax); light sub-tiles -> m, den and α for every edge.
// Lane = edge of the tile's stream: the per-row max is a segmented lane scan (order-free), the per-row
// Σ exp_p(el − m) is folded sequentially in edge order by the row's owner lane (canonical order; a
// light row is one chunk), then α = |ex| / den keeps the sign of e_pre.  Tiles of up to FS_TC edges
// keep el / ex, the row and the edge id of every stream position in shared memory (one global pass);
// longer tiles recompute them per pass.
constexpr int FS_TC = 384;
template <int H>
__host__ __device__ constexpr int fs_warp_smem() { return FS_TC * H * 4 + FS_TC * 4 + FS_TC + 2 * 32 * H * 4; }

template <int H>
__global__ void __launch_bounds__(256) k_fwd_stats_t(const GatFwdArgs a) {
  extern __shared__ __align__(16) uint8_t fsm[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* wsm = fsm + w * fs_warp_smem<H>();
  float (*cx)[H] = reinterpret_cast<float (*)[H]>(wsm);                          // [FS_TC][H] el -> ex
  int* ce = reinterpret_cast<int*>(wsm + FS_TC * H * 4);                          // [FS_TC] edge id
  float (*smx)[H] = reinterpret_cast<float (*)[H]>(wsm + FS_TC * H * 4 + FS_TC * 4);        // [32][H]
  float (*sbuf)[H] = smx + 32;                                                    // [32][H]
  uint8_t* crow = wsm + FS_TC * H * 4 + FS_TC * 4 + 2 * 32 * H * 4;               // [FS_TC]
  const Scale scS = scale_from_amax(amax_load(a.amax_S), a.bits);
  const Scale scD = scale_from_amax(amax_load(a.amax_D), a.bits);
  const int64_t n = a.g.n_local, hc = load_count(a.plan.counts);
  const int64_t nitems = hc + load_count(a.plan.counts + 2);
  const int64_t i_lo = a.part == 2 ? hc : 0, i_hi = a.part == 1 ? hc : nitems;   // hub / light split
  FOR_ITEMS(it, a.work + 0 + (a.part == 1 ? 8 : 0), i_hi - i_lo) {
    const int64_t item = i_lo + it;
    if (item < hc) {
      Seg s;
      decode_item(item, hc, a.g.in_ptr, a.plan, a.g.chunk, s);
      const int64_t vg = a.g.row_begin + s.vl;
      int8_t qd[H];
#pragma unroll
      for (int h = 0; h < H; ++h) qd[h] = a.qD[vg * H + h];
      float mx[H];
      seg_max<H>(a.g.in_src, s.eb, s.ee, a.qS, scS.s, qd, scD.s, a.slope, mx);
      if (lane < H) a.hmax[(int64_t)s.slot * H + lane] = head_pick<H>(mx, lane);
      continue;
    }
    const int32_t code = a.plan.tiles[item - hc];
    const int64_t r0 = (int64_t)(code >> 10) * TILE;
    int T;
    const TileLane L = tile_setup(a.g.in_ptr, a.plan.hbase, r0, n, T, (code >> 5) & 31, (code & 31) + 1);
    const int64_t vg = a.g.row_begin + L.r;
    const bool cached = T <= FS_TC;
    int qdj[H];
#pragma unroll
    for (int h = 0; h < H; ++h) {
      qdj[h] = L.light ? (int)a.qD[vg * H + h] : 0;
      smx[lane][h] = -INFINITY;
    }
    __syncwarp();
    const int tlast = T - 1, nch = (T + 31) >> 5;
    auto edge_of = [&](int t, int& row) -> int64_t {
      row = tile_row(t < T ? t : tlast, L.end);
      return __shfl_sync(0xffffffffu, L.eb, row) + (t - __shfl_sync(0xffffffffu, L.off, row));
    };
    // el of stream position t (lane), computed from the graph (pass A, or any pass when not cached)
    auto el_of = [&](int t, int row, int64_t e, float (&ep)[H]) {
      int qdr[H];
#pragma unroll
      for (int h = 0; h < H; ++h) qdr[h] = __shfl_sync(0xffffffffu, qdj[h], row);
      if (t < T) {
        int8_t qs[H];
        load_qh<H>(a.qS + (int64_t)a.g.in_src[e] * H, qs);
#pragma unroll
        for (int h = 0; h < H; ++h) ep[h] = sddmm_add1(qs[h], scS.s, (int8_t)qdr[h], scD.s);
      }
    };
    // pass A: e_pre, per-row max of el = lrelu(e_pre)
    for (int c = 0; c < nch; ++c) {
      const int t = c * 32 + lane;
      int row;
      const int64_t e = edge_of(t, row);
      float ep[H], el[H];
      el_of(t, row, e, ep);
#pragma unroll
      for (int h = 0; h < H; ++h) el[h] = t < T ? lrelu(ep[h], a.slope) : -INFINITY;
      if (cached && t < T) {
#pragma unroll
        for (int h = 0; h < H; ++h) cx[t][h] = ep[h];
        ce[t] = (int)e;
        crow[t] = (uint8_t)row;
      }
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int ro = __shfl_up_sync(0xffffffffu, row, o);
#pragma unroll
        for (int h = 0; h < H; ++h) {
          const float v = __shfl_up_sync(0xffffffffu, el[h], o);
          if (lane >= o && ro == row) el[h] = fmaxf(el[h], v);
        }
      }
      const int rn = __shfl_down_sync(0xffffffffu, row, 1);
      if (lane == 31 || rn != row)
#pragma unroll
        for (int h = 0; h < H; ++h) smx[row][h] = fmaxf(smx[row][h], el[h]);
      __syncwarp();
    }
    float mown[H], den[H];
#pragma unroll
    for (int h = 0; h < H; ++h) { mown[h] = (L.light && L.deg > 0) ? smx[lane][h] : 0.0f; den[h] = 0.0f; }
    // pass B: ex = exp_p(el − m) with the sign of e_pre, den = sequential sum by the row owner
    for (int c = 0; c < nch; ++c) {
      const int base = c * 32, t = base + lane;
      const int cnt = T - base < 32 ? T - base : 32;
      int row;
      int64_t e = 0;
      float ep[H];
      if (cached) {
        row = crow[t < T ? t : tlast];
        if (t < T)
#pragma unroll
          for (int h = 0; h < H; ++h) ep[h] = cx[t][h];
      } else {
        e = edge_of(t, row);
        el_of(t, row, e, ep);
      }
      float mr[H];
#pragma unroll
      for (int h = 0; h < H; ++h) mr[h] = __shfl_sync(0xffffffffu, mown[h], row);
      if (t < T) {
        float sx[H];
#pragma unroll
        for (int h = 0; h < H; ++h) {
          const float ex = exp_p(__fsub_rn(lrelu(ep[h], a.slope), mr[h]));
          sbuf[lane][h] = ex;
          sx[h] = ep[h] > 0.0f ? ex : -ex;
        }
        if (cached) {
#pragma unroll
          for (int h = 0; h < H; ++h) cx[t][h] = sx[h];
        } else if constexpr (H == 4) {
          *reinterpret_cast<float4*>(a.alpha + e * 8) = make_float4(sx[0], sx[1], sx[2], sx[3]);
        } else {
#pragma unroll
          for (int h = 0; h < H; ++h) a.alpha[e * 2 * H + h] = sx[h];
        }
      }
      __syncwarp();
      const int lo = (L.off > base ? L.off : base) - base;
      const int hi = (L.end < base + cnt ? L.end : base + cnt) - base;
      for (int i = lo; i < hi; ++i)
#pragma unroll
        for (int h = 0; h < H; ++h) den[h] = __fadd_rn(den[h], sbuf[i][h]);
      __syncwarp();
    }
    if (L.light) {
#pragma unroll
      for (int h = 0; h < H; ++h) { a.m[vg * H + h] = mown[h]; a.den[vg * H + h] = den[h]; }
    }
    // pass C: α = |ex| / den with the sign of e_pre
    for (int c = 0; c < nch; ++c) {
      const int t = c * 32 + lane;
      int row;
      int64_t e;
      if (cached) {
        row = crow[t < T ? t : tlast];
        e = t < T ? ce[t] : 0;
      } else {
        e = edge_of(t, row);
      }
      float dr[H];
#pragma unroll
      for (int h = 0; h < H; ++h) dr[h] = __shfl_sync(0xffffffffu, den[h], row);
      if (t < T) {
        float xs[H], o[H];
        if (cached) {
#pragma unroll
          for (int h = 0; h < H; ++h) xs[h] = cx[t][h];
        } else {
#pragma unroll
          for (int h = 0; h < H; ++h) xs[h] = a.alpha[e * 2 * H + h];
        }
#pragma unroll
        for (int h = 0; h < H; ++h) {
          const float al = __fdiv_rn(fabsf(xs[h]), dr[h]);
          o[h] = signbit(xs[h]) ? -al : al;
        }
        if constexpr (H == 4) {
          *reinterpret_cast<float4*>(a.alpha + e * 8) = make_float4(o[0], o[1], o[2], o[3]);
        } else {
#pragma unroll
          for (int h = 0; h < H; ++h) a.alpha[e * 2 * H + h] = o[h];
        }
      }
    }
    __syncwarp();
  }
}

// FS2: heavy segments -> segment Σ exp_p(el - m) (hden), m from all segment maxima of the row
template <int H>
__global__ void __launch_bounds__(256) k_fwd_stats2(const GatFwdArgs a) {
  __shared__ float sh[WPB][32 * segb<H>()][H];
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
    const float part = seg_sum_exp<H>(a.g.in_src, s.eb, s.ee, a.qS, scS.s, qd, scD.s, a.slope, mx, sh[w], a.alpha);
    if (lane < H) a.hden[si * H + lane] = part;
  }
}

// FS3: heavy segments -> α = ex / den with den the chunk-ordered fold of the row's segment sums
template <int H>
__global__ void __launch_bounds__(256) k_fwd_alpha3(const GatFwdArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t hcnt = load_count(a.plan.counts);
  FOR_ITEMS(si, a.work + 4, hcnt) {
    Seg s;
    decode_item(si, hcnt, a.g.in_ptr, a.plan, a.g.chunk, s);
    float mx[H], den[H];
    heavy_row_stats<H>(a.hmax, a.hden, s.base, s.nseg, mx, den);
    for (int64_t base = s.eb; base < s.ee; base += 32 * SEGB) {
      float x[SEGB][H];
#pragma unroll
      for (int i = 0; i < SEGB; ++i) {
        const int64_t e = base + i * 32 + lane;
        if (e < s.ee)
#pragma unroll
          for (int h = 0; h < H; ++h) x[i][h] = a.alpha[e * 2 * H + h];
      }
#pragma unroll
      for (int i = 0; i < SEGB; ++i) {
        const int64_t e = base + i * 32 + lane;
        if (e < s.ee)
#pragma unroll
          for (int h = 0; h < H; ++h) {
            const float al = __fdiv_rn(fabsf(x[i][h]), den[h]);
            a.alpha[e * 2 * H + h] = signbit(x[i][h]) ? -al : al;
          }
      }
    }
  }
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

// ================================================================== column-group gather kernels
// A warp owns one head group: WC = 32*VPL consecutive columns holding HPW whole heads (D = WC/HPW),
// for a tile of light rows or for one heavy segment.  Work item = (tile or segment) x (group), so a
// warp gathers WC bytes (one 128-B line at D = 128) per edge with VPL accumulators per lane: few
// registers, many resident warps and a 16-deep gather pipeline.  Heads are independent in every
// gather pass (α, ∂α, P, ∂E, ∂S, ∂D are per head), so the canonical per-row order is unchanged.
template <int VPL>
struct CGCfg {
  static constexpr int WORDS = (VPL + 3) / 4;
  static constexpr int UNRC = WORDS == 1 ? 16 : (WORDS == 2 ? 8 : 4);
};

// ---- FA: aggregation ⑤ per (tile | heavy segment, head group)
// Streamed aggregation of one 32-edge chunk: rows q_X[w_i] gathered through a rolling ring of RING
// loads in flight; edge i of the chunk uses weight sa[i][myh] and (if rb) belongs to row rb[i].
template <int H, int VPL, int RING, typename F>
__device__ __forceinline__ void agg_chunk(const int8_t* __restrict__ xbase, int64_t ldx, int w_l, int cnt,
                                          const float (*sa)[H], const int* rb, int& cur, float2 (&acc)[VPL / 2],
                                          F&& on_row) {
  constexpr int WORDS = VPL / 4 > 0 ? VPL / 4 : 1;
  const int myh = (threadIdx.x & 31) / (32 / H);
  Row<VPL> ring[RING];
#pragma unroll
  for (int j = 0; j < RING; ++j) {
    const int w = __shfl_sync(0xffffffffu, w_l, j);
    if (j < cnt) ring[j] = load_row<VPL>(xbase + (int64_t)w * ldx);
  }
  // rolling ring: a RING-wide unrolled body inside a runtime loop keeps RING rows in flight with
  // small code (the fully unrolled 32-edge body overflowed the instruction cache)
  for (int i0 = 0; i0 < cnt; i0 += RING) {
#pragma unroll
    for (int j = 0; j < RING; ++j) {
      const int i = i0 + j;
      if (i < cnt) {
        if (rb) {
          const int ri = rb[i];
          if (ri != cur) { on_row(ri); cur = ri; }
        }
        const float al = sa[i][myh];
        const float2 al2 = make_float2(al, al);
        if constexpr (VPL >= 4) {
#pragma unroll
          for (int q = 0; q < WORDS; ++q) fma4_codes(ring[j].w[q], al2, acc[2 * q], acc[2 * q + 1]);
        } else {   // VPL == 2: two codes in the low half-word
          acc[0] = __ffma2_rn(al2, codes2(ring[j].w[0] ^ 0x80808080u, 0x7440u, 0x7441u), acc[0]);
        }
        // refill the consumed slot (no register copy of the in-flight row)
        const int nx = i + RING;
        const int w = __shfl_sync(0xffffffffu, w_l, nx & 31);
        if (nx < cnt) ring[j] = load_row<VPL>(xbase + (int64_t)w * ldx);
      }
    }
  }
}

// evict-first (streaming) stores for outputs that are not re-read by this pass: keep L2 for the
// gathered int8 table
__device__ __forceinline__ void st_cs(float* p, float v) { __stcs(p, v); }

// FA: ⑤ H_out = (Σ fmaf(α, q_H′[u])) * s_H′ over (heavy segment | tile of light rows); α is read from
// the stored (signed) α of the stats passes, so the chunk attributes are two coalesced loads.
template <int H, int VPL>
__global__ void __launch_bounds__(256, 3) k_fwd_agg2(const GatFwdArgs a) {
  constexpr int HD = 32 * VPL;
  constexpr int RING = VPL >= 16 ? 4 : 8;
  __shared__ float sh_a[WPB][32][H];
  __shared__ int sh_rb[WPB][32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Scale scH = scale_from_amax(amax_load(a.amax_Hp), a.bits);
  const int64_t n = a.g.n_local, hc = load_count(a.plan.counts);
  const int64_t nitems = hc + load_count(a.plan.counts + 2);
  const int8_t* xbase = a.qHp + lane * VPL;
  float amax_loc = 0.0f;
  float2 acc[VPL / 2];
  auto zero_acc = [&]() {
#pragma unroll
    for (int k = 0; k < VPL / 2; ++k) acc[k] = make_float2(0.0f, 0.0f);
  };
  FOR_ITEMS(item, a.work + 2, nitems) {
    zero_acc();
    if (item < hc) {   // ------------------------------------------------ heavy segment -> hagg
      Seg s;
      decode_item(item, hc, a.g.in_ptr, a.plan, a.g.chunk, s);
      int cur = 0;
      for (int64_t base = s.eb; base < s.ee; base += 32) {
        const int cnt = (int)(s.ee - base < 32 ? s.ee - base : 32);
        int u = 0;
        if (lane < cnt) {
          u = a.g.in_src[base + lane];
#pragma unroll
          for (int h = 0; h < H; ++h) sh_a[w][lane][h] = fabsf(a.alpha[(base + lane) * 2 * H + h]);
        }
        __syncwarp();
        agg_chunk<H, VPL, RING>(xbase, a.ldHp, u, cnt, sh_a[w], nullptr, cur, acc, [](int) {});
        __syncwarp();
      }
      float* dst = a.hagg + (int64_t)s.slot * HD + lane * VPL;
#pragma unroll
      for (int k = 0; k < VPL / 2; ++k) { dst[2 * k] = acc[k].x; dst[2 * k + 1] = acc[k].y; }
      continue;
    }
    // --------------------------------------------------------------- sub-tile of light rows
    const int32_t code = a.plan.tiles[item - hc];
    const int64_t r0 = (int64_t)(code >> 10) * TILE;
    int T;
    const TileLane L = tile_setup(a.g.in_ptr, a.plan.hbase, r0, n, T, (code >> 5) & 31, (code & 31) + 1);
    unsigned zm = __ballot_sync(0xffffffffu, L.light && L.deg == 0);
    while (zm) {   // light rows without in-edges: H_out = 0
      const int j = __ffs(zm) - 1;
      zm &= zm - 1;
      float* dst = a.Hout + (r0 + j) * HD + lane * VPL;
#pragma unroll
      for (int k = 0; k < VPL; ++k) dst[k] = 0.0f;
    }
    int cur = -1;
    auto flush = [&](int j) {
      float* dst = a.Hout + (r0 + j) * HD + lane * VPL;
#pragma unroll
      for (int k = 0; k < VPL / 2; ++k) {
        const float x = __fmul_rn(acc[k].x, scH.s), y = __fmul_rn(acc[k].y, scH.s);
        amax_loc = fmaxf(amax_loc, fmaxf(fabsf(x), fabsf(y)));
        st_cs(dst + 2 * k, x);
        st_cs(dst + 2 * k + 1, y);
        acc[k] = make_float2(0.0f, 0.0f);
      }
    };
    for (int base = 0; base < T; base += 32) {
      const int cnt = T - base < 32 ? T - base : 32;
      const int t = base + lane;
      const int row = tile_row(t, L.end);
      const int64_t e = __shfl_sync(0xffffffffu, L.eb, row) + (t - __shfl_sync(0xffffffffu, L.off, row));
      int u = 0;
      if (lane < cnt) {
        u = a.g.in_src[e];
#pragma unroll
        for (int h = 0; h < H; ++h) sh_a[w][lane][h] = fabsf(a.alpha[e * 2 * H + h]);
        sh_rb[w][lane] = row;
      }
      __syncwarp();
      agg_chunk<H, VPL, RING>(xbase, a.ldHp, u, cnt, sh_a[w], sh_rb[w], cur, acc, [&](int) {
        if (cur >= 0) flush(cur);
      });
      __syncwarp();
    }
    if (cur >= 0) flush(cur);
  }
  amax_flush(a.amax_out, amax_loc);
}



// FA (VPL >= 4): ⑤ H_out = (Σ fmaf(α, q_H′[u])) * s_H′ over (heavy segment | light sub-tile)
// ================================================================== gather engine v4
// One warp streams a heavy segment or a light sub-tile: the 32-edge chunk attributes (gather index,
// tile row, |α| per head, optional per-edge addend x per head) are loaded one chunk ahead into
// registers and stashed in per-warp shared memory as [head][edge] so a group of 4 edges reads them
// with one LDS.128 each; rows are gathered by cp.async into a ring of AGG_RING slots whose refill
// indices also come from shared memory (one LDS.128 per 4 edges, no shuffles).  The tail group is
// padded with α = +0, x = +0 and the last row: fmaf(+0, q, acc) == acc and acc + (+0) == acc for
// every acc these sums can hold (never -0), so padding is exact and the group loop is branch-free.
// The gathered tables hold excess-128 codes (gat_codes_biased), converted without a sign flip.
template <int H, int VPL, bool HAS_X>
__host__ __device__ constexpr int g4_warp_smem() {
  return AGG_RING * 32 * VPL + 2 * H * 32 * 4 * (HAS_X ? 2 : 1) + 2 * 32 * 4 + 2 * 32;
}

template <int H, int VPL, bool HAS_X, typename AttrF, typename RowF>
__device__ __forceinline__ int g4_stream(uint8_t* wsm, const int8_t* __restrict__ xbase, uint32_t ld32, bool tile,
                                         int64_t seg_eb, const TileLane& L, int T, AttrF&& attr, RowF&& on_row,
                                         float2 (&acc)[VPL / 2], float& xs) {
  constexpr int R = AGG_RING, RB = 32 * VPL;
  const int lane = threadIdx.x & 31, myh = lane / (32 / H);
  float* sa = reinterpret_cast<float*>(wsm + R * RB);                       // [2][H][32] |α|
  float* sx = sa + 2 * H * 32;                                              // [2][H][32] x (HAS_X)
  int* sidx = reinterpret_cast<int*>(wsm + R * RB + 2 * H * 32 * 4 * (HAS_X ? 2 : 1));   // [2][32]
  uint8_t* srow = reinterpret_cast<uint8_t*>(sidx + 64);                   // [2][32]
  const uint32_t ring_s = smem_u32(wsm) + lane * VPL;
  const int tlast = T - 1;
  auto load = [&](int c, int& idx, int& row, float (&al)[H], float (&x)[H]) {
    const int t = c * 32 + lane;
    int64_t e;
    if (tile) {
      row = tile_row(t < T ? t : tlast, L.end);
      e = __shfl_sync(0xffffffffu, L.eb, row) + (t - __shfl_sync(0xffffffffu, L.off, row));
    } else {
      row = 0;
      e = seg_eb + t;
    }
    idx = 0;
#pragma unroll
    for (int h = 0; h < H; ++h) { al[h] = 0.0f; x[h] = 0.0f; }
    if (t < T) attr(e, idx, al, x);
  };
  auto stash = [&](int b, int row, const float (&al)[H], const float (&x)[H]) {
#pragma unroll
    for (int h = 0; h < H; ++h) {
      sa[(b * H + h) * 32 + lane] = al[h];
      if constexpr (HAS_X) sx[(b * H + h) * 32 + lane] = x[h];
    }
    srow[b * 32 + lane] = (uint8_t)row;
  };
  auto group = [&](const Row<VPL> (&r)[4], float4 a4, float4 x4, uint32_t rw, int& cur) {
    const float al[4] = {a4.x, a4.y, a4.z, a4.w};
    const float xv[4] = {x4.x, x4.y, x4.z, x4.w};
    if ((int)(rw >> 24) == cur) {   // rows are non-decreasing: the whole group continues the row
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 al2 = make_float2(al[j], al[j]);
#pragma unroll
        for (int q = 0; q < VPL / 4; ++q) fma4_biased(r[j].w[q], al2, acc[2 * q], acc[2 * q + 1]);
        if constexpr (HAS_X) xs = __fadd_rn(xs, xv[j]);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int rj = (int)((rw >> (8 * j)) & 0xffu);
        if (rj != cur) {
          if (cur >= 0) on_row(cur);
          cur = rj;
        }
        const float2 al2 = make_float2(al[j], al[j]);
#pragma unroll
        for (int q = 0; q < VPL / 4; ++q) fma4_biased(r[j].w[q], al2, acc[2 * q], acc[2 * q + 1]);
        if constexpr (HAS_X) xs = __fadd_rn(xs, xv[j]);
      }
    }
  };
  {
    int idxA, rowA;
    float alA[H], xA[H];
    load(0, idxA, rowA, alA, xA);
    stash(0, rowA, alA, xA);
    sidx[lane] = (int)((uint32_t)idxA * ld32);   // byte offset of the gathered row
  }
  __syncwarp();
#pragma unroll
  for (int g = 0; g < R / 4; ++g) {   // ring prologue: edges 0 .. R-1, one commit group per 4 edges
    const int4 nx = *reinterpret_cast<const int4*>(sidx + 4 * g);
    const int nv[4] = {nx.x, nx.y, nx.z, nx.w};
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (4 * g + j < T) cp_row_slice<VPL>(ring_s + (4 * g + j) * RB, xbase + (uint32_t)nv[j]);
    cp_commit();
  }
  int cur = tile ? -1 : 0;
  const int nch = (T + 31) >> 5;
  for (int c = 0; c < nch; ++c) {
    int idxB, rowB;
    float alB[H], xB[H];
    load(c + 1, idxB, rowB, alB, xB);   // next chunk, in flight while this chunk streams
    const int cb = c & 1;
    const float* sac = sa + (cb * H + myh) * 32;
    const float* sxc = sx + (cb * H + myh) * 32;
    const uint8_t* src_ = srow + cb * 32;
    for (int i0 = 0; i0 < 32; i0 += 4) {
      const int t0 = c * 32 + i0;
      if (t0 >= T) break;
      if (i0 == 12) {   // refills from group 16 on read the next chunk's indices
        sidx[(cb ^ 1) * 32 + lane] = (int)((uint32_t)idxB * ld32);
        __syncwarp();
      }
      cp_wait<R / 4 - 1>();   // the 4 rows of this group have landed
      const uint32_t slot0 = ring_s + (uint32_t)(t0 & (R - 1)) * RB;
      Row<VPL> r[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) r[j] = lds_row_slice<VPL>(slot0 + j * RB);
      const float4 a4 = *reinterpret_cast<const float4*>(sac + i0);
      float4 x4 = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
      if constexpr (HAS_X) x4 = *reinterpret_cast<const float4*>(sxc + i0);
      const uint32_t rw = *reinterpret_cast<const uint32_t*>(src_ + i0);
      group(r, a4, x4, rw, cur);
      const int tn0 = t0 + R;   // refill the 4 consumed slots with edges t0+R .. t0+R+3
      const int4 nx = *reinterpret_cast<const int4*>(sidx + ((tn0 >> 5) & 1) * 32 + (tn0 & 31));
      const int nv[4] = {nx.x, nx.y, nx.z, nx.w};
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (tn0 + j < T) cp_row_slice<VPL>(slot0 + j * RB, xbase + (uint32_t)nv[j]);   // N*ld < 2^32
      cp_commit();
    }
    __syncwarp();
    stash(cb ^ 1, rowB, alB, xB);
    __syncwarp();
  }
  cp_wait<0>();
  __syncwarp();
  return cur;
}

// FA (VPL >= 4): ⑤ H_out = (Σ fmaf(α, q_H′[u])) * s_H′ over (heavy segment | light sub-tile)
template <int H, int VPL>
__global__ void __launch_bounds__(256, 3) k_fwd_agg4(const GatFwdArgs a) {
  constexpr int HD = 32 * VPL;
  extern __shared__ __align__(16) uint8_t dsm[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* wsm = dsm + w * g4_warp_smem<H, VPL, false>();
  const Scale scH = scale_from_amax(amax_load(a.amax_Hp), a.bits);
  const int64_t n = a.g.n_local, hc = load_count(a.plan.counts);
  const int64_t nitems = hc + load_count(a.plan.counts + 2);
  const int8_t* xbase = a.qHp + lane * VPL;
  const uint32_t ld32 = (uint32_t)a.ldHp;
  float amax_loc = 0.0f;
  const int64_t i_lo = a.part == 2 ? hc : 0, i_hi = a.part == 1 ? hc : nitems;   // hub / light split
  FOR_ITEMS(it, a.work + 2 + (a.part == 1 ? 8 : 0), i_hi - i_lo) {
    const int64_t item = i_lo + it;
    const bool tile = item >= hc;
    Seg s;
    s.eb = 0;
    TileLane L;
    int64_t r0 = 0;
    int T;
    if (!tile) {
      decode_item(item, hc, a.g.in_ptr, a.plan, a.g.chunk, s);
      T = (int)(s.ee - s.eb);
      L.eb = 0; L.off = 0; L.end = 0;
    } else {
      const int32_t code = a.plan.tiles[item - hc];
      r0 = (int64_t)(code >> 10) * TILE;
      L = tile_setup(a.g.in_ptr, a.plan.hbase, r0, n, T, (code >> 5) & 31, (code & 31) + 1);
      unsigned zm = __ballot_sync(0xffffffffu, L.light && L.deg == 0);
      while (zm) {   // light rows without in-edges: H_out = 0
        const int j = __ffs(zm) - 1;
        zm &= zm - 1;
        float4* dst = reinterpret_cast<float4*>(a.Hout + (r0 + j) * HD + lane * VPL);
#pragma unroll
        for (int k = 0; k < VPL / 4; ++k) __stcs(dst + k, make_float4(0.0f, 0.0f, 0.0f, 0.0f));
      }
    }
    float2 acc[VPL / 2];
#pragma unroll
    for (int k = 0; k < VPL / 2; ++k) acc[k] = make_float2(0.0f, 0.0f);
    float xs = 0.0f;
    auto flush = [&](int j) {
      float4* dst = reinterpret_cast<float4*>(a.Hout + (r0 + j) * HD + lane * VPL);
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
    auto attr = [&](int64_t e, int& u, float (&al)[H], float (&)[H]) {
      u = a.g.in_src[e];
      if constexpr (H == 4) {
        const float4 v = *reinterpret_cast<const float4*>(a.alpha + e * 8);
        al[0] = fabsf(v.x); al[1] = fabsf(v.y); al[2] = fabsf(v.z); al[3] = fabsf(v.w);
      } else {
#pragma unroll
        for (int h = 0; h < H; ++h) al[h] = fabsf(a.alpha[e * 2 * H + h]);
      }
    };
    const int cur = g4_stream<H, VPL, false>(wsm, xbase, ld32, tile, s.eb, L, T, attr, flush, acc, xs);
    if (tile) {
      if (cur >= 0) flush(cur);
    } else {
      float4* dst = reinterpret_cast<float4*>(a.hagg + (int64_t)s.slot * HD + lane * VPL);
#pragma unroll
      for (int k = 0; k < VPL / 4; ++k)
        dst[k] = make_float4(acc[2 * k].x, acc[2 * k].y, acc[2 * k + 1].x, acc[2 * k + 1].y);
    }
  }
  amax_flush(a.amax_out, amax_loc);
}


// ================================================================== gather engine v5 (TMA gather4)
// As v4, but the rows are gathered by the TMA engine: one elected lane issues
// cp.async.bulk.tensor.2d.tile::gather4 per group of 4 edges (4 rows of HD bytes land contiguously in
// a ring slot, completion on the slot's mbarrier), so consumer lanes spend no issue slots on
// addresses.  Ring: G slots of 4 rows per warp; slot/phase follow a per-warp running group counter.


// FA (VPL >= 4, TMA gather): ⑤ H_out = (Σ fmaf(α, q_H′[u])) * s_H′ over (heavy segment | light sub-tile)
// ================================================================== backward gather kernels (cp.async engine)
template <int H, int VPL>
__host__ __device__ constexpr int bwd3_warp_smem() {
  // ring + α[2][32][H] + (∂α | P[v])[2][32][H] + row[2][32] + edge[2][32] + P-tile[32][H]
  return AGG_RING * 32 * VPL + 2 * 32 * H * 4 * 2 + 2 * 32 * 4 * 2 + 32 * H * 4;
}

// exact i8·i8 dot of this lane's slice, reduced over the LPH lanes of its head
template <int VPL, int LPH>
__device__ __forceinline__ int head_dot(const Row<VPL>& x, const Row<VPL>& y) {
  int dot = row_dot<VPL>(x, y);
#pragma unroll
  for (int o = 1; o < LPH; o <<= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
  return dot;
}

// BD1: ⑤″ ∂α = i2f(q_G[v]·q_H′[u]) (s_G s_H′) (IDP4A on codes), ④′ P = Σ fmaf(∂α, α) per
// destination row (heavy segments: P partials), then for light rows ∂E_pre and ∂D.
// ②′ finalize of source row u (full row): ∂H′ = (agg·s_G + ∂S·a_src) + ∂D·a_dst ; ∂S stored
template <int VPL>
__device__ __forceinline__ void src_finalize_full(const GatBwdArgs& a, int64_t ul, int64_t ug, int myh, int H,
                                                  float dS, float2 (&acc)[VPL / 2], float sG, float& amax_loc) {
  constexpr int HD = 32 * VPL;
  const int lane = threadIdx.x & 31;
  const float dD = a.dD[ug * H + myh];
  const int c0 = lane * VPL;
  float* dst = a.dHp + ul * HD + c0;
#pragma unroll
  for (int k = 0; k < VPL / 2; ++k) {
    float v2[2] = {acc[k].x, acc[k].y};
#pragma unroll
    for (int z = 0; z < 2; ++z) {
      const int col = c0 + 2 * k + z;
      const float agg = __fmul_rn(v2[z], sG);
      const float t2 = __fadd_rn(agg, __fmul_rn(dS, __ldg(a.a_src + col)));
      const float o = __fadd_rn(t2, __fmul_rn(dD, __ldg(a.a_dst + col)));
      amax_loc = fmaxf(amax_loc, fabsf(o));
      dst[2 * k + z] = o;
    }
    acc[k] = make_float2(0.0f, 0.0f);
  }
  if ((lane % (32 / H)) == 0) a.dS[ug * H + myh] = dS;
}

// BS: ⑤′ ∂H′_agg = Σ fmaf(α, q_G[v]) over out-edges, ③′ ∂S = Σ ∂E_pre, ②′ finalize (light rows);
// heavy out-segments leave ∂S / aggregation partials.  α comes from the stored signed α via out_eid
// when available (one GPU), otherwise it is recomputed from per-node data.
template <int H, int VPL, bool B>
__global__ void __launch_bounds__(256, 2) k_bwd_src_v3(const GatBwdArgs a) {
  constexpr int HD = 32 * VPL, R = AGG_RING, RB = 32 * VPL, LPH = 32 / H;
  extern __shared__ __align__(16) uint8_t dsm[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int myh = lane / LPH;
  const bool leader = (lane % LPH) == 0;
  uint8_t* wsm = dsm + w * bwd3_warp_smem<H, VPL>();
  float (*sa)[32][H] = reinterpret_cast<float (*)[32][H]>(wsm + R * RB);                 // signed α
  float (*sp)[32][H] = reinterpret_cast<float (*)[32][H]>(wsm + R * RB + 2 * 32 * H * 4);  // P[v]
  int (*srb)[32] = reinterpret_cast<int (*)[32]>(wsm + R * RB + 4 * 32 * H * 4);
  const uint32_t ring_s = smem_u32(wsm) + lane * VPL;
  const Scale scS = scale_from_amax(amax_load(a.amax_S), a.bits);
  const Scale scD = scale_from_amax(amax_load(a.amax_D), a.bits);
  const Scale scH = scale_from_amax(amax_load(a.amax_Hp), a.bits);
  const Scale scG = scale_from_amax(amax_load(a.amax_G), a.bits);
  const float sGH = __fmul_rn(scG.s, scH.s);
  const int64_t n = a.g.n_local, hc = load_count(a.pout.counts);
  const int64_t nitems = hc + load_count(a.pout.counts + 2);
  const int8_t* gbase = a.qG + lane * VPL;
  const int8_t* hbase = a.qHp + lane * VPL;
  const uint32_t ld32 = (uint32_t)a.ldG;
  const bool use_eid = a.g.out_eid != nullptr;
  float amax_loc = 0.0f;
  FOR_ITEMS(item, a.work + 2, nitems) {
    const bool tile = item >= hc;
    Seg s;
    TileLane L;
    int64_t r0 = 0;
    int T;
    if (!tile) {
      decode_item(item, hc, a.g.out_ptr, a.pout, a.g.chunk, s);
      T = (int)(s.ee - s.eb);
      L.eb = 0; L.off = 0; L.end = 0; L.deg = 0; L.light = false;
      r0 = s.vl;
    } else {
      const int32_t code = a.pout.tiles[item - hc];
      r0 = (int64_t)(code >> 10) * TILE;
      L = tile_setup(a.g.out_ptr, a.pout.hbase, r0, n, T, (code >> 5) & 31, (code & 31) + 1);
    }
    const int64_t ug0 = a.g.row_begin + r0;
    int qsj[H];   // own q_S of lane j's row (recompute path)
#pragma unroll
    for (int h = 0; h < H; ++h) qsj[h] = (!use_eid && (tile ? L.deg > 0 : lane == 0)) ? (int)a.qS[(ug0 + lane) * H + h] : 0;
    float2 acc[VPL / 2];
#pragma unroll
    for (int k = 0; k < VPL / 2; ++k) acc[k] = make_float2(0.0f, 0.0f);
    if (tile) {
      unsigned zm = __ballot_sync(0xffffffffu, L.light && L.deg == 0);
      while (zm) {   // light rows without out-edges: ∂H′ = (0 + 0·a_src) + ∂D·a_dst
        const int j = __ffs(zm) - 1;
        zm &= zm - 1;
        src_finalize_full<VPL>(a, r0 + j, ug0 + j, myh, H, 0.0f, acc, scG.s, amax_loc);
      }
    }
    auto attrs = [&](int c, int& v, float (&al)[H], float (&pv)[H], int& row) {
      const int t = c * 32 + lane;
      int64_t e;
      if (tile) {
        row = tile_row(t, L.end);
        e = __shfl_sync(0xffffffffu, L.eb, row) + (t - __shfl_sync(0xffffffffu, L.off, row));
      } else {
        row = 0;
        e = s.eb + t;
      }
      int qsr[H];
#pragma unroll
      for (int h = 0; h < H; ++h) qsr[h] = __shfl_sync(0xffffffffu, qsj[h], row);
      v = 0;
#pragma unroll
      for (int h = 0; h < H; ++h) { al[h] = 0.0f; pv[h] = 0.0f; }
      if (t < T) {
        v = a.g.out_dst[e];
        if (use_eid) {   // one GPU: α and ∂E_pre of the destination-side passes, by in-CSR edge id
          const int64_t eid = a.g.out_eid[e];
#pragma unroll
          for (int h = 0; h < H; ++h) { al[h] = a.alpha[eid * 2 * H + h]; pv[h] = a.alpha[eid * 2 * H + H + h]; }
        } else {
#pragma unroll
          for (int h = 0; h < H; ++h) {
            const int64_t k = (int64_t)v * H + h;
            const float ep = sddmm_add1((int8_t)qsr[h], scS.s, a.qD[k], scD.s);
            const float al_ = __fdiv_rn(exp_p(__fsub_rn(lrelu(ep, a.slope), a.m[k])), a.den[k]);
            al[h] = ep > 0.0f ? al_ : -al_;
          }
        }
        if (!use_eid) {
#pragma unroll
          for (int h = 0; h < H; ++h) pv[h] = a.P[(int64_t)v * H + h];
        }
      }
    };
    const unsigned act = tile ? __ballot_sync(0xffffffffu, L.deg > 0) : 1u;
    int nxt = act ? __ffs(act) - 1 : -1;
    Row<VPL> hw{}, hw_nxt{};
    int hsum = 0;   // Σ of the own q_H′ slice in plain codes (excess-128 correction of the dots)
    if (nxt >= 0) hw_nxt = load_row<VPL>(hbase + (ug0 + nxt) * a.ldHp);
    int vA, rowA;
    float alA[H], pA[H];
    attrs(0, vA, alA, pA, rowA);
#pragma unroll
    for (int h = 0; h < H; ++h) { sa[0][lane][h] = alA[h]; sp[0][lane][h] = pA[h]; }
    srb[0][lane] = rowA;
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const int vv = __shfl_sync(0xffffffffu, vA, j);
      if (j < T) cp_row_slice<VPL>(ring_s + j * RB, gbase + (uint32_t)vv * ld32);
      if ((j & 3) == 3) cp_commit();
    }
    float dS = 0.0f;
    int cur = -1;
    const int nch = (T + 31) >> 5;
    for (int c = 0; c < nch; ++c) {
      int vB, rowB;
      float alB[H], pB[H];
      attrs(c + 1, vB, alB, pB, rowB);
      __syncwarp();
      const int cb = c & 1;
      for (int i0 = 0; i0 < 32; i0 += 4) {
        const int t0 = c * 32 + i0;
        if (t0 >= T) break;
        cp_wait<R / 4 - 1>();
        const uint32_t slot0 = ring_s + (uint32_t)(t0 & (R - 1)) * RB;
        Row<VPL> r[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) r[j] = lds_row_slice<VPL>(slot0 + j * RB);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (t0 + j < T) {
            const int ri = tile ? srb[cb][i0 + j] : 0;
            if (ri != cur) {
              if (cur >= 0) {
                const float dSb = __shfl_sync(0xffffffffu, dS, myh * LPH);
                src_finalize_full<VPL>(a, r0 + cur, ug0 + cur, myh, H, dSb, acc, scG.s, amax_loc);
                dS = 0.0f;
              }
              cur = ri;
              hw = hw_nxt;
              if constexpr (B) hsum = row_sum_plain<VPL>(hw, true);
              nxt = tile ? tile_next(act, cur) : -1;
              if (nxt >= 0) hw_nxt = load_row<VPL>(hbase + (ug0 + nxt) * a.ldHp);
            }
            const float x = sa[cb][i0 + j][myh];
            const float al = fabsf(x);
            if (use_eid) {   // ∂E_pre read from the destination pass
              if (leader) dS = __fadd_rn(dS, sp[cb][i0 + j][myh]);
            } else {         // recompute ∂α = q_G[v]·q_H′[u] and ∂E_pre (partitioned graphs)
              int dot;
              if constexpr (B) {
                dot = row_dot_biased<VPL>(r[j], hw, hsum);
#pragma unroll
                for (int o = 1; o < LPH; o <<= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
              } else {
                dot = head_dot<VPL, LPH>(r[j], hw);
              }
              if (leader) {
                const float dal = __fmul_rn(__int2float_rn(dot), sGH);
                const float dE = __fmul_rn(al, __fsub_rn(dal, sp[cb][i0 + j][myh]));
                dS = __fadd_rn(dS, signbit(x) ? __fmul_rn(dE, a.slope) : dE);
              }
            }
            const float2 al2 = make_float2(al, al);
#pragma unroll
            for (int q = 0; q < VPL / 4; ++q) fma4_any<B>(r[j].w[q], al2, acc[2 * q], acc[2 * q + 1]);
          }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int tn = t0 + R + j;
          const int va = __shfl_sync(0xffffffffu, vA, tn & 31);
          const int vb = __shfl_sync(0xffffffffu, vB, tn & 31);
          const uint32_t vn = (uint32_t)(tn < (c + 1) * 32 ? va : vb);
          if (tn < T) cp_row_slice<VPL>(slot0 + j * RB, gbase + vn * ld32);
        }
        cp_commit();
      }
      __syncwarp();
#pragma unroll
      for (int h = 0; h < H; ++h) { sa[cb ^ 1][lane][h] = alB[h]; sp[cb ^ 1][lane][h] = pB[h]; }
      srb[cb ^ 1][lane] = rowB;
      vA = vB;
      __syncwarp();
    }
    cp_wait<0>();
    __syncwarp();
    if (!tile) {
      if (leader) a.hdS[(int64_t)s.slot * H + myh] = dS;
      float* dst = a.hagg + (int64_t)s.slot * HD + lane * VPL;
#pragma unroll
      for (int k = 0; k < VPL / 2; ++k) { dst[2 * k] = acc[k].x; dst[2 * k + 1] = acc[k].y; }
      continue;
    }
    if (cur >= 0) {
      const float dSb = __shfl_sync(0xffffffffu, dS, myh * LPH);
      src_finalize_full<VPL>(a, r0 + cur, ug0 + cur, myh, H, dSb, acc, scG.s, amax_loc);
    }
  }
  amax_flush(a.amax_dHp, amax_loc);
}

template <int H, int VPL>
__host__ __device__ constexpr int dst4_warp_smem() {
  // ring | |α| [2][H][32] | gather idx [2][32] | row [2][32] u8 | ∂α [H][32] (pass 2: [32][H]) | P [32][H]
  return AGG_RING * 32 * VPL + 2 * H * 32 * 4 + 2 * 32 * 4 + 2 * 32 + H * 32 * 4 + 32 * H * 4;
}

// BD1 (v4 engine): ⑤″ ∂α = i2f(q_G[v]·q_H′[u]) (s_G s_H′), ④′ P = Σ fmaf(∂α, α) in edge order per
// destination row (heavy segments: P partials), then for light rows ∂E_pre and ∂D (pass 2).
template <int H, int VPL, int NW, bool B>
__global__ void __maxnreg__(80) k_bwd_dst1_v4(const GatBwdArgs a) {
  constexpr int R = AGG_RING, RB = 32 * VPL, LPH = 32 / H;
  extern __shared__ __align__(16) uint8_t dsm[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int myh = lane / LPH;
  const bool leader = (lane % LPH) == 0;
  uint8_t* wsm = dsm + w * dst4_warp_smem<H, VPL>();
  float* sa = reinterpret_cast<float*>(wsm + R * RB);                 // [2][H][32]
  int* sidx = reinterpret_cast<int*>(sa + 2 * H * 32);                // [2][32]
  uint8_t* srow = reinterpret_cast<uint8_t*>(sidx + 64);             // [2][32]
  float* sd = reinterpret_cast<float*>(srow + 64);                    // [H][32]
  float (*pt)[H] = reinterpret_cast<float (*)[H]>(sd + H * 32);       // [32][H]
  const uint32_t ring_s = smem_u32(wsm) + lane * VPL;
  const Scale scH = scale_from_amax(amax_load(a.amax_Hp), a.bits);
  const Scale scG = scale_from_amax(amax_load(a.amax_G), a.bits);
  const float sGH = __fmul_rn(scG.s, scH.s);
  const int64_t n = a.g.n_local, hc = load_count(a.pin.counts);
  const int64_t nitems = hc + load_count(a.pin.counts + 2);
  const int8_t* xbase = a.qHp + lane * VPL;
  const int8_t* gbase = a.qG + lane * VPL;
  const uint32_t ld32 = (uint32_t)a.ldHp;
  const int64_t i_lo = a.part == 2 ? hc : 0, i_hi = a.part == 1 ? hc : nitems;   // hub / light split
  FOR_ITEMS(it, a.work + 0 + (a.part == 1 ? 8 : 0), i_hi - i_lo) {
    const int64_t item = i_lo + it;
    const bool tile = item >= hc;
    Seg s;
    s.eb = 0;
    TileLane L;
    int64_t r0 = 0;
    int T;
    if (!tile) {
      decode_item(item, hc, a.g.in_ptr, a.pin, a.g.chunk, s);
      T = (int)(s.ee - s.eb);
      L.eb = 0; L.off = 0; L.end = 0; L.deg = 0; L.light = false;
    } else {
      const int32_t code = a.pin.tiles[item - hc];
      r0 = (int64_t)(code >> 10) * TILE;
      L = tile_setup(a.g.in_ptr, a.pin.hbase, r0, n, T, (code >> 5) & 31, (code & 31) + 1);
      if (L.light && L.deg == 0) {
        const int64_t vg = a.g.row_begin + L.r;
#pragma unroll
        for (int h = 0; h < H; ++h) { a.P[vg * H + h] = 0.0f; a.dD[vg * H + h] = 0.0f; }
      }
    }
    const int tlast = T - 1;
    auto load = [&](int c, int& u, int& row, int64_t& e, float (&al)[H]) {
      const int t = c * 32 + lane;
      if (tile) {
        row = tile_row(t < T ? t : tlast, L.end);
        e = __shfl_sync(0xffffffffu, L.eb, row) + (t - __shfl_sync(0xffffffffu, L.off, row));
      } else {
        row = 0;
        e = s.eb + t;
      }
      u = 0;
#pragma unroll
      for (int h = 0; h < H; ++h) al[h] = 0.0f;
      if (t < T) {
        u = a.g.in_src[e];
        if constexpr (H == 4) {
          const float4 v = *reinterpret_cast<const float4*>(a.alpha + e * 8);
          al[0] = fabsf(v.x); al[1] = fabsf(v.y); al[2] = fabsf(v.z); al[3] = fabsf(v.w);
        } else {
#pragma unroll
          for (int h = 0; h < H; ++h) al[h] = fabsf(a.alpha[e * 2 * H + h]);
        }
      }
    };
    auto stash = [&](int b, int row, const float (&al)[H]) {
#pragma unroll
      for (int h = 0; h < H; ++h) sa[(b * H + h) * 32 + lane] = al[h];
      srow[b * 32 + lane] = (uint8_t)row;
    };
    // own q_G[v] slice per row, prefetched one row ahead
    const unsigned act = tile ? __ballot_sync(0xffffffffu, L.deg > 0) : 1u;
    const int64_t vg0 = a.g.row_begin + (tile ? r0 : s.vl);
    int nxt = act ? __ffs(act) - 1 : -1;
    Row<VPL> gw{}, gw_nxt{};
    int gsum = 0;   // Σ of the own q_G slice in plain codes (excess-128 correction of the dots)
    if (nxt >= 0) gw_nxt = load_row<VPL>(gbase + (vg0 + nxt) * a.ldG);
    int64_t eA;
    {
      int uA, rowA;
      float alA[H];
      load(0, uA, rowA, eA, alA);
      stash(0, rowA, alA);
      sidx[lane] = (int)((uint32_t)uA * ld32);   // byte offset of the gathered row
    }
    __syncwarp();
#pragma unroll
    for (int g = 0; g < R / 4; ++g) {
      const int4 nx = *reinterpret_cast<const int4*>(sidx + 4 * g);
      const int nv[4] = {nx.x, nx.y, nx.z, nx.w};
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (4 * g + j < T) cp_row_slice<VPL>(ring_s + (4 * g + j) * RB, xbase + (uint32_t)nv[j]);
      cp_commit();
    }
    float P = 0.0f;
    int cur = -1, pcur = -1;
    if (!tile) {   // a heavy segment is one row
      cur = 0; pcur = 0;
      gw = gw_nxt;
      if constexpr (B) gsum = row_sum_plain<VPL>(gw, true);
    }
    const int nch = (T + 31) >> 5;
    for (int c = 0; c < nch; ++c) {
      int uB, rowB;
      int64_t eB;
      float alB[H];
      load(c + 1, uB, rowB, eB, alB);
      const int cb = c & 1;
      const float* sac = sa + (cb * H + myh) * 32;
      const uint8_t* src_ = srow + cb * 32;
      for (int i0 = 0; i0 < 32; i0 += 4) {
        const int t0 = c * 32 + i0;
        if (t0 >= T) break;
        if (i0 == 12) {
          sidx[(cb ^ 1) * 32 + lane] = (int)((uint32_t)uB * ld32);
          __syncwarp();
        }
        cp_wait<R / 4 - 1>();
        const uint32_t slot0 = ring_s + (uint32_t)(t0 & (R - 1)) * RB;
        Row<VPL> r[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) r[j] = lds_row_slice<VPL>(slot0 + j * RB);
        const float4 a4 = *reinterpret_cast<const float4*>(sac + i0);
        const uint32_t rw = *reinterpret_cast<const uint32_t*>(src_ + i0);
        int d[4];
        const bool same = (int)(rw >> 24) == cur;
        if (same) {
#pragma unroll
          for (int j = 0; j < 4; ++j) d[j] = B ? row_dot_biased<VPL>(r[j], gw, gsum) : row_dot<VPL>(gw, r[j]);
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int rj = (int)((rw >> (8 * j)) & 0xffu);
            if (rj != cur) {
              cur = rj;
              gw = gw_nxt;
              if constexpr (B) gsum = row_sum_plain<VPL>(gw, true);
              nxt = tile_next(act, cur);
              if (nxt >= 0) gw_nxt = load_row<VPL>(gbase + (vg0 + nxt) * a.ldG);
            }
            d[j] = B ? row_dot_biased<VPL>(r[j], gw, gsum) : row_dot<VPL>(gw, r[j]);
          }
        }
        int k;
        const int dot = group_dot_reduce<LPH>(d, k);
        sd[myh * 32 + i0 + k] = __fmul_rn(__int2float_rn(dot), sGH);
        __syncwarp();
        const float4 d4 = *reinterpret_cast<const float4*>(sd + myh * 32 + i0);
        const float dal[4] = {d4.x, d4.y, d4.z, d4.w}, al[4] = {a4.x, a4.y, a4.z, a4.w};
        if (same) {
#pragma unroll
          for (int j = 0; j < 4; ++j) P = __fmaf_rn(dal[j], al[j], P);
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int rj = (int)((rw >> (8 * j)) & 0xffu);
            if (rj != pcur) {
              if (pcur >= 0 && leader) pt[pcur][myh] = P;
              P = 0.0f;
              pcur = rj;
            }
            P = __fmaf_rn(dal[j], al[j], P);
          }
        }
        const int tn0 = t0 + R;
        const int4 nx = *reinterpret_cast<const int4*>(sidx + ((tn0 >> 5) & 1) * 32 + (tn0 & 31));
        const int nv[4] = {nx.x, nx.y, nx.z, nx.w};
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (tn0 + j < T) cp_row_slice<VPL>(slot0 + j * RB, xbase + (uint32_t)nv[j]);
        cp_commit();
      }
      __syncwarp();
      if (c * 32 + lane < T) {   // ∂α of this chunk -> scratch (edge-major)
        if constexpr (H == 4) {
          *reinterpret_cast<float4*>(a.dalpha + eA * 4) = make_float4(sd[lane], sd[32 + lane], sd[64 + lane], sd[96 + lane]);
        } else {
#pragma unroll
          for (int h = 0; h < H; ++h) a.dalpha[eA * H + h] = sd[h * 32 + lane];
        }
      }
      __syncwarp();
      stash(cb ^ 1, rowB, alB);
      eA = eB;
      __syncwarp();
    }
    cp_wait<0>();
    __syncwarp();
    if (!tile) {
      if (leader) a.hP[(int64_t)s.slot * H + myh] = P;
      continue;
    }
    if (pcur >= 0 && leader) pt[pcur][myh] = P;
    __syncwarp();
    // ---- pass 2 (light rows): ∂E = α(∂α − P[v]), ∂E_pre, ∂D = Σ ∂E_pre (lane j folds row j)
    float (*sdx)[H] = reinterpret_cast<float (*)[H]>(sd);   // [32][H]
    float dDp[H];
#pragma unroll
    for (int h = 0; h < H; ++h) dDp[h] = 0.0f;
    for (int base = 0; base < T; base += 32) {
      const int cnt = T - base < 32 ? T - base : 32;
      const int t = base + lane;
      const int row = tile_row(t < T ? t : tlast, L.end);
      const int64_t e = __shfl_sync(0xffffffffu, L.eb, row) + (t - __shfl_sync(0xffffffffu, L.off, row));
      if (lane < cnt) {
        float x[H], dl[H], o[H];
        if constexpr (H == 4) {
          const float4 xv = *reinterpret_cast<const float4*>(a.alpha + e * 8);
          const float4 dv = *reinterpret_cast<const float4*>(a.dalpha + e * 4);
          x[0] = xv.x; x[1] = xv.y; x[2] = xv.z; x[3] = xv.w;
          dl[0] = dv.x; dl[1] = dv.y; dl[2] = dv.z; dl[3] = dv.w;
        } else {
#pragma unroll
          for (int h = 0; h < H; ++h) { x[h] = a.alpha[e * 2 * H + h]; dl[h] = a.dalpha[e * H + h]; }
        }
#pragma unroll
        for (int h = 0; h < H; ++h) {
          const float dE = __fmul_rn(fabsf(x[h]), __fsub_rn(dl[h], pt[row][h]));
          o[h] = signbit(x[h]) ? __fmul_rn(dE, a.slope) : dE;
          sdx[lane][h] = o[h];
        }
        if constexpr (H == 4) {
          *reinterpret_cast<float4*>(a.alpha_dE + e * 8 + 4) = make_float4(o[0], o[1], o[2], o[3]);
        } else {
#pragma unroll
          for (int h = 0; h < H; ++h) a.alpha_dE[e * 2 * H + H + h] = o[h];
        }
      }
      __syncwarp();
      const int lo = (L.off > base ? L.off : base) - base;
      const int hi = (L.end < base + cnt ? L.end : base + cnt) - base;
      for (int i = lo; i < hi; ++i)
#pragma unroll
        for (int h = 0; h < H; ++h) dDp[h] = __fadd_rn(dDp[h], sdx[i][h]);
      __syncwarp();
    }
    if (L.deg > 0) {
      const int64_t vg = a.g.row_begin + L.r;
#pragma unroll
      for (int h = 0; h < H; ++h) { a.P[vg * H + h] = pt[lane][h]; a.dD[vg * H + h] = dDp[h]; }
    }
    __syncwarp();
  }
}

// ②′ finalize of one source row (vectorized): ∂H′ = (agg·s_G + ∂S·a_src) + ∂D·a_dst
template <int H, int VPL>
__device__ __forceinline__ void src_finalize4(const GatBwdArgs& a, int64_t ul, int64_t ug, int myh, bool leader,
                                              float dS, float2 (&acc)[VPL / 2], float sG, float& amax_loc) {
  constexpr int HD = 32 * VPL;
  const int lane = threadIdx.x & 31;
  const float dD = a.dD[ug * H + myh];
  const int c0 = lane * VPL;
  float4* dst = reinterpret_cast<float4*>(a.dHp + ul * HD + c0);
  const float4* as = reinterpret_cast<const float4*>(a.a_src + c0);
  const float4* ad = reinterpret_cast<const float4*>(a.a_dst + c0);
#pragma unroll
  for (int k = 0; k < VPL / 4; ++k) {
    const float4 s4 = __ldg(as + k), d4 = __ldg(ad + k);
    const float v[4] = {acc[2 * k].x, acc[2 * k].y, acc[2 * k + 1].x, acc[2 * k + 1].y};
    const float sv[4] = {s4.x, s4.y, s4.z, s4.w}, dv[4] = {d4.x, d4.y, d4.z, d4.w};
    float o[4];
#pragma unroll
    for (int z = 0; z < 4; ++z) {   // scalar: ptxas contracts packed FMUL2 + FADD2 into FFMA2
      const float t2 = __fadd_rn(__fmul_rn(v[z], sG), __fmul_rn(dS, sv[z]));
      o[z] = __fadd_rn(t2, __fmul_rn(dD, dv[z]));
      amax_loc = fmaxf(amax_loc, fabsf(o[z]));
    }
    dst[k] = make_float4(o[0], o[1], o[2], o[3]);
    acc[2 * k] = make_float2(0.0f, 0.0f);
    acc[2 * k + 1] = make_float2(0.0f, 0.0f);
  }
  if (leader) a.dS[ug * H + myh] = dS;
}

// BS (one GPU, out_eid present): ⑤′ ∂H′_agg = Σ fmaf(|α|, q_G[v]) and ③′ ∂S = Σ ∂E_pre over out-edges,
// with |α| and ∂E_pre read through the edge-id map from the packed [E][2H] array; ②′ finalize.
template <int H, int VPL, int NW>
__global__ void __maxnreg__(96) k_bwd_src4(const GatBwdArgs a) {
  constexpr int HD = 32 * VPL;
  extern __shared__ __align__(16) uint8_t dsm[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int myh = lane / (32 / H);
  const bool leader = (lane % (32 / H)) == 0;
  uint8_t* wsm = dsm + w * g4_warp_smem<H, VPL, true>();
  const Scale scG = scale_from_amax(amax_load(a.amax_G), a.bits);
  const int64_t n = a.g.n_local, hc = load_count(a.pout.counts);
  const int64_t nitems = hc + load_count(a.pout.counts + 2);
  const int8_t* gbase = a.qG + lane * VPL;
  const uint32_t ld32 = (uint32_t)a.ldG;
  float amax_loc = 0.0f;
  const int64_t i_lo = a.part == 2 ? hc : 0, i_hi = a.part == 1 ? hc : nitems;   // hub / light split
  FOR_ITEMS(it, a.work + 2 + (a.part == 1 ? 8 : 0), i_hi - i_lo) {
    const int64_t item = i_lo + it;
    const bool tile = item >= hc;
    Seg s;
    s.eb = 0;
    TileLane L;
    int64_t r0 = 0;
    int T;
    float2 acc[VPL / 2];
#pragma unroll
    for (int k = 0; k < VPL / 2; ++k) acc[k] = make_float2(0.0f, 0.0f);
    if (!tile) {
      decode_item(item, hc, a.g.out_ptr, a.pout, a.g.chunk, s);
      T = (int)(s.ee - s.eb);
      L.eb = 0; L.off = 0; L.end = 0;
      r0 = s.vl;
    } else {
      const int32_t code = a.pout.tiles[item - hc];
      r0 = (int64_t)(code >> 10) * TILE;
      L = tile_setup(a.g.out_ptr, a.pout.hbase, r0, n, T, (code >> 5) & 31, (code & 31) + 1);
      unsigned zm = __ballot_sync(0xffffffffu, L.light && L.deg == 0);
      while (zm) {   // light rows without out-edges: ∂H′ = (0 + 0·a_src) + ∂D·a_dst
        const int j = __ffs(zm) - 1;
        zm &= zm - 1;
        src_finalize4<H, VPL>(a, r0 + j, a.g.row_begin + r0 + j, myh, leader, 0.0f, acc, scG.s, amax_loc);
      }
    }
    const int64_t ug0 = a.g.row_begin + r0;
    float dS = 0.0f;
    auto flush = [&](int j) {
      src_finalize4<H, VPL>(a, r0 + j, ug0 + j, myh, leader, dS, acc, scG.s, amax_loc);
      dS = 0.0f;
    };
    auto attr = [&](int64_t e, int& v, float (&al)[H], float (&x)[H]) {
      v = a.g.out_dst[e];
      const int64_t eid = a.g.out_eid[e];
      if constexpr (H == 4) {
        const float4 p = *reinterpret_cast<const float4*>(a.alpha + eid * 8);
        const float4 q = *reinterpret_cast<const float4*>(a.alpha + eid * 8 + 4);
        al[0] = fabsf(p.x); al[1] = fabsf(p.y); al[2] = fabsf(p.z); al[3] = fabsf(p.w);
        x[0] = q.x; x[1] = q.y; x[2] = q.z; x[3] = q.w;
      } else {
#pragma unroll
        for (int h = 0; h < H; ++h) { al[h] = fabsf(a.alpha[eid * 2 * H + h]); x[h] = a.alpha[eid * 2 * H + H + h]; }
      }
    };
    const int cur = g4_stream<H, VPL, true>(wsm, gbase, ld32, tile, s.eb, L, T, attr, flush, acc, dS);
    if (tile) {
      if (cur >= 0) flush(cur);
    } else {
      if (leader) a.hdS[(int64_t)s.slot * H + myh] = dS;
      float4* dst = reinterpret_cast<float4*>(a.hagg + (int64_t)s.slot * HD + lane * VPL);
#pragma unroll
      for (int k = 0; k < VPL / 4; ++k)
        dst[k] = make_float4(acc[2 * k].x, acc[2 * k].y, acc[2 * k + 1].x, acc[2 * k + 1].y);
    }
  }
  amax_flush(a.amax_dHp, amax_loc);
}

// BS (one GPU, out_eid present, TMA gather): ⑤′ ∂H′_agg, ③′ ∂S over out-edges, ②′ finalize
// ---- BD1: ⑤″ ∂α (IDP4A on codes) + ④′ P (+ ∂E_pre, ∂D for light rows) per (tile | segment, group)
template <int VPL, int HPW>
__device__ __forceinline__ int cg_dot(const Row<VPL>& x, const Row<VPL>& y) {
  int dot = row_dot<VPL>(x, y);
#pragma unroll
  for (int o = 1; o < 32 / HPW; o <<= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
  return dot;
}

template <int VPL, int HPW>
__global__ void __launch_bounds__(256) k_bwd_dst1_cg(const GatBwdArgs a) {
  constexpr int WC = 32 * VPL, LPH = 32 / HPW, UNRC = CGCfg<VPL>::UNRC;
  __shared__ float sh_a[WPB][32][HPW];
  __shared__ float sh_d[WPB][32][HPW];
  __shared__ float sh_pt[WPB][32][HPW];
  __shared__ int sh_rb[WPB][32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int lh = lane / LPH;
  const bool leader = (lane % LPH) == 0;
  const int H = a.d.heads, HD = a.d.hd, NG = HD / WC;
  const Scale scS = scale_from_amax(amax_load(a.amax_S), a.bits);
  const Scale scD = scale_from_amax(amax_load(a.amax_D), a.bits);
  const Scale scH = scale_from_amax(amax_load(a.amax_Hp), a.bits);
  const Scale scG = scale_from_amax(amax_load(a.amax_G), a.bits);
  const float sGH = __fmul_rn(scG.s, scH.s);
  const int64_t n = a.g.n_local, hc = load_count(a.pin.counts);
  const int64_t nitems = (hc + (n + TILE - 1) / TILE) * NG;
  float (*ba)[HPW] = sh_a[w];
  float (*bd)[HPW] = sh_d[w];
  FOR_ITEMS(item, a.work + 0, nitems) {
    const int64_t wi = item / NG;
    const int g = (int)(item - wi * NG), h0 = g * HPW;
    const int8_t* hbase = a.qHp + g * WC + lane * VPL;
    const int8_t* gbase = a.qG + g * WC + lane * VPL;
    if (wi < hc) {   // ----------------------------------------------- heavy segment: ∂α, P partial
      Seg s;
      decode_item(wi, hc, a.g.in_ptr, a.pin, a.g.chunk, s);
      const int64_t vg = a.g.row_begin + s.vl;
      float mr[HPW], dr[HPW];
      int qdr[HPW];
#pragma unroll
      for (int k = 0; k < HPW; ++k) {
        mr[k] = a.m[vg * H + h0 + k]; dr[k] = a.den[vg * H + h0 + k]; qdr[k] = (int)a.qD[vg * H + h0 + k];
      }
      const Row<VPL> gw = load_row<VPL>(gbase + vg * a.ldG);
      float P = 0.0f;
      for (int64_t base = s.eb; base < s.ee; base += 32) {
        const int cnt = (int)(s.ee - base < 32 ? s.ee - base : 32);
        int u = 0;
        if (lane < cnt) {
          u = a.g.in_src[base + lane];
#pragma unroll
          for (int k = 0; k < HPW; ++k)
            ba[lane][k] = __fdiv_rn(exp_p(__fsub_rn(lrelu(sddmm_add1(a.qS[(int64_t)u * H + h0 + k], scS.s,
                                                                     (int8_t)qdr[k], scD.s), a.slope), mr[k])), dr[k]);
        }
        __syncwarp();
        for (int i0 = 0; i0 < cnt; i0 += UNRC) {
          Row<VPL> rr[UNRC];
#pragma unroll
          for (int j = 0; j < UNRC; ++j) {
            const int wv = __shfl_sync(0xffffffffu, u, (i0 + j) & 31);
            if (i0 + j < cnt) rr[j] = load_row<VPL>(hbase + (int64_t)wv * a.ldHp);
          }
#pragma unroll
          for (int j = 0; j < UNRC; ++j) {
            if (i0 + j < cnt) {
              const int dot = cg_dot<VPL, HPW>(gw, rr[j]);
              if (leader) {
                const float dal = __fmul_rn(__int2float_rn(dot), sGH);
                P = __fmaf_rn(dal, ba[i0 + j][lh], P);
                bd[i0 + j][lh] = dal;
              }
            }
          }
        }
        __syncwarp();
        if (lane < cnt) {
#pragma unroll
          for (int k = 0; k < HPW; ++k) a.dalpha[(base + lane) * H + h0 + k] = bd[lane][k];
        }
        __syncwarp();
      }
      if (leader) a.hP[(int64_t)s.slot * H + h0 + lh] = P;
      continue;
    }
    // ------------------------------------------------------------- tile of light rows
    const int64_t r0 = (wi - hc) * TILE;
    int T;
    const TileLane L = tile_setup(a.g.in_ptr, a.pin.hbase, r0, n, T);
    const int64_t vg = a.g.row_begin + L.r;
    float mj[HPW], dj[HPW];
    int qdj[HPW];
#pragma unroll
    for (int k = 0; k < HPW; ++k) {
      mj[k] = L.deg > 0 ? a.m[vg * H + h0 + k] : 0.0f;
      dj[k] = L.deg > 0 ? a.den[vg * H + h0 + k] : 0.0f;
      qdj[k] = L.deg > 0 ? (int)a.qD[vg * H + h0 + k] : 0;
    }
    if (L.light && L.deg == 0) {
#pragma unroll
      for (int k = 0; k < HPW; ++k) { a.P[vg * H + h0 + k] = 0.0f; a.dD[vg * H + h0 + k] = 0.0f; }
    }
    const unsigned act = __ballot_sync(0xffffffffu, L.deg > 0);
    const int64_t vg0 = a.g.row_begin + r0;
    int nxt = act ? __ffs(act) - 1 : -1;
    Row<VPL> gw_nxt{}, gw{};
    if (nxt >= 0) gw_nxt = load_row<VPL>(gbase + (vg0 + nxt) * a.ldG);
    float P = 0.0f;
    int cur = -1;
    for (int base = 0; base < T; base += 32) {     // pass 1
      const int cnt = T - base < 32 ? T - base : 32;
      const int t = base + lane;
      const int row = tile_row(t, L.end);
      const int64_t e = __shfl_sync(0xffffffffu, L.eb, row) + (t - __shfl_sync(0xffffffffu, L.off, row));
      float mr[HPW], dr[HPW];
      int qdr[HPW];
#pragma unroll
      for (int k = 0; k < HPW; ++k) {
        mr[k] = __shfl_sync(0xffffffffu, mj[k], row);
        dr[k] = __shfl_sync(0xffffffffu, dj[k], row);
        qdr[k] = __shfl_sync(0xffffffffu, qdj[k], row);
      }
      int u = 0;
      if (lane < cnt) {
        u = a.g.in_src[e];
#pragma unroll
        for (int k = 0; k < HPW; ++k)
          ba[lane][k] = __fdiv_rn(exp_p(__fsub_rn(lrelu(sddmm_add1(a.qS[(int64_t)u * H + h0 + k], scS.s,
                                                                   (int8_t)qdr[k], scD.s), a.slope), mr[k])), dr[k]);
        sh_rb[w][lane] = row;
      }
      __syncwarp();
      for (int i0 = 0; i0 < cnt; i0 += UNRC) {
        Row<VPL> rr[UNRC];
#pragma unroll
        for (int j = 0; j < UNRC; ++j) {
          const int wv = __shfl_sync(0xffffffffu, u, (i0 + j) & 31);
          if (i0 + j < cnt) rr[j] = load_row<VPL>(hbase + (int64_t)wv * a.ldHp);
        }
#pragma unroll
        for (int j = 0; j < UNRC; ++j) {
          if (i0 + j < cnt) {
            const int ri = sh_rb[w][i0 + j];
            if (ri != cur) {
              if (cur >= 0 && leader) sh_pt[w][cur][lh] = P;
              P = 0.0f;
              cur = ri;
              gw = gw_nxt;
              nxt = tile_next(act, cur);
              if (nxt >= 0) gw_nxt = load_row<VPL>(gbase + (vg0 + nxt) * a.ldG);
            }
            const int dot = cg_dot<VPL, HPW>(gw, rr[j]);
            if (leader) {
              const float dal = __fmul_rn(__int2float_rn(dot), sGH);
              P = __fmaf_rn(dal, ba[i0 + j][lh], P);
              bd[i0 + j][lh] = dal;
            }
          }
        }
      }
      __syncwarp();
      if (lane < cnt) {
#pragma unroll
        for (int k = 0; k < HPW; ++k) a.dalpha[e * H + h0 + k] = bd[lane][k];
      }
      __syncwarp();
    }
    if (cur >= 0 && leader) sh_pt[w][cur][lh] = P;
    __syncwarp();
    float dDp[HPW];
#pragma unroll
    for (int k = 0; k < HPW; ++k) dDp[k] = 0.0f;
    for (int base = 0; base < T; base += 32) {     // pass 2: ∂E_pre, ∂D
      const int cnt = T - base < 32 ? T - base : 32;
      const int t = base + lane;
      const int row = tile_row(t, L.end);
      const int64_t e = __shfl_sync(0xffffffffu, L.eb, row) + (t - __shfl_sync(0xffffffffu, L.off, row));
      float mr[HPW], dr[HPW];
      int qdr[HPW];
#pragma unroll
      for (int k = 0; k < HPW; ++k) {
        mr[k] = __shfl_sync(0xffffffffu, mj[k], row);
        dr[k] = __shfl_sync(0xffffffffu, dj[k], row);
        qdr[k] = __shfl_sync(0xffffffffu, qdj[k], row);
      }
      if (lane < cnt) {
        const int64_t u = a.g.in_src[e];
#pragma unroll
        for (int k = 0; k < HPW; ++k) {
          const float ep = sddmm_add1(a.qS[u * H + h0 + k], scS.s, (int8_t)qdr[k], scD.s);
          const float al = __fdiv_rn(exp_p(__fsub_rn(lrelu(ep, a.slope), mr[k])), dr[k]);
          const float dE = __fmul_rn(al, __fsub_rn(a.dalpha[e * H + h0 + k], sh_pt[w][row][k]));
          ba[lane][k] = ep > 0.0f ? dE : __fmul_rn(dE, a.slope);
          a.alpha_dE[e * 2 * H + H + h0 + k] = ba[lane][k];   // ∂E_pre beside α
        }
      }
      __syncwarp();
      const int lo = (L.off > base ? L.off : base) - base;
      const int hi = (L.end < base + cnt ? L.end : base + cnt) - base;
      for (int i = lo; i < hi; ++i)
#pragma unroll
        for (int k = 0; k < HPW; ++k) dDp[k] = __fadd_rn(dDp[k], ba[i][k]);
      __syncwarp();
    }
    if (L.deg > 0) {
#pragma unroll
      for (int k = 0; k < HPW; ++k) { a.P[vg * H + h0 + k] = sh_pt[w][lane][k]; a.dD[vg * H + h0 + k] = dDp[k]; }
    }
    __syncwarp();
  }
}

// ---- BS: ⑤′ + ③′ + ②′ per (tile | heavy segment, group) over out-edges (u→v)
// finalize of row u for the group's columns: ∂H′ = (agg·s_G + ∂S·a_src) + ∂D·a_dst ; ∂S stored
template <int VPL, int HPW>
__device__ __forceinline__ void cg_src_finalize(const GatBwdArgs& a, int64_t ul, int64_t ug, int g, float dS,
                                                float (&part)[VPL], float sG, float& amax_loc) {
  constexpr int WC = 32 * VPL, LPH = 32 / HPW;
  const int lane = threadIdx.x & 31, lh = lane / LPH;
  const int H = a.d.heads, HD = a.d.hd, h = g * HPW + lh;
  const float dD = a.dD[ug * H + h];
  const int c0 = g * WC + lane * VPL;
  float* dst = a.dHp + ul * HD + c0;
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    const float agg = __fmul_rn(part[k], sG);
    const float t2 = __fadd_rn(agg, __fmul_rn(dS, __ldg(a.a_src + c0 + k)));
    const float o = __fadd_rn(t2, __fmul_rn(dD, __ldg(a.a_dst + c0 + k)));
    amax_loc = fmaxf(amax_loc, fabsf(o));
    dst[k] = o;
    part[k] = 0.0f;
  }
  if ((lane % LPH) == 0) a.dS[ug * H + h] = dS;
}

template <int VPL, int HPW>
__global__ void __launch_bounds__(256) k_bwd_src_cg(const GatBwdArgs a) {
  constexpr int WC = 32 * VPL, LPH = 32 / HPW, UNRC = CGCfg<VPL>::UNRC;
  __shared__ float sh_a[WPB][32][HPW];
  __shared__ float sh_e[WPB][32][HPW];
  __shared__ float sh_p[WPB][32][HPW];
  __shared__ int sh_rb[WPB][32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int lh = lane / LPH;
  const bool leader = (lane % LPH) == 0;
  const int H = a.d.heads, HD = a.d.hd, NG = HD / WC;
  const Scale scS = scale_from_amax(amax_load(a.amax_S), a.bits);
  const Scale scD = scale_from_amax(amax_load(a.amax_D), a.bits);
  const Scale scH = scale_from_amax(amax_load(a.amax_Hp), a.bits);
  const Scale scG = scale_from_amax(amax_load(a.amax_G), a.bits);
  const float sGH = __fmul_rn(scG.s, scH.s);
  const int64_t n = a.g.n_local, hc = load_count(a.pout.counts);
  const int64_t nitems = (hc + (n + TILE - 1) / TILE) * NG;
  float (*ba)[HPW] = sh_a[w];
  float (*be)[HPW] = sh_e[w];
  float (*bp)[HPW] = sh_p[w];
  float amax_loc = 0.0f;
  FOR_ITEMS(item, a.work + 2, nitems) {
    const int64_t wi = item / NG;
    const int g = (int)(item - wi * NG), h0 = g * HPW;
    const int8_t* hbase = a.qHp + g * WC + lane * VPL;
    const int8_t* gbase = a.qG + g * WC + lane * VPL;
    float part[VPL];
#pragma unroll
    for (int k = 0; k < VPL; ++k) part[k] = 0.0f;
    float dS = 0.0f;
    // one 32-edge batch of out-edges: per-edge α, e_pre, P[v] (lane-parallel), then the q_G gathers
    auto batch = [&](int cnt, int v, const int (&qsr)[HPW], const int* rb, int& cur, Row<VPL>& hw, auto&& on_row) {
      if ((threadIdx.x & 31) < cnt) {
#pragma unroll
        for (int k = 0; k < HPW; ++k) {
          const int64_t kk = (int64_t)v * H + h0 + k;
          const float ep = sddmm_add1((int8_t)qsr[k], scS.s, a.qD[kk], scD.s);
          ba[lane][k] = __fdiv_rn(exp_p(__fsub_rn(lrelu(ep, a.slope), a.m[kk])), a.den[kk]);
          be[lane][k] = ep;
          bp[lane][k] = a.P[kk];
        }
      }
      __syncwarp();
      for (int i0 = 0; i0 < cnt; i0 += UNRC) {
        Row<VPL> rr[UNRC];
#pragma unroll
        for (int j = 0; j < UNRC; ++j) {
          const int vv = __shfl_sync(0xffffffffu, v, (i0 + j) & 31);
          if (i0 + j < cnt) rr[j] = load_row<VPL>(gbase + (int64_t)vv * a.ldG);
        }
#pragma unroll
        for (int j = 0; j < UNRC; ++j) {
          if (i0 + j < cnt) {
            if (rb) {
              const int ri = rb[i0 + j];
              if (ri != cur) { on_row(ri); cur = ri; }
            }
            const int dot = cg_dot<VPL, HPW>(rr[j], hw);
            const float al = ba[i0 + j][lh];
            if (leader) {
              const float dal = __fmul_rn(__int2float_rn(dot), sGH);
              const float dE = __fmul_rn(al, __fsub_rn(dal, bp[i0 + j][lh]));
              dS = __fadd_rn(dS, be[i0 + j][lh] > 0.0f ? dE : __fmul_rn(dE, a.slope));
            }
#pragma unroll
            for (int q = 0; q < CGCfg<VPL>::WORDS; ++q) {
              const uint32_t wx = rr[j].w[q] ^ 0x80808080u;
#pragma unroll
              for (int k = 0; k < 4 && q * 4 + k < VPL; ++k) part[q * 4 + k] = __fmaf_rn(al, bx2f(wx, k), part[q * 4 + k]);
            }
          }
        }
      }
      __syncwarp();
    };
    if (wi < hc) {   // ----------------------------------------------- heavy segment: partials
      Seg s;
      decode_item(wi, hc, a.g.out_ptr, a.pout, a.g.chunk, s);
      const int64_t ug = a.g.row_begin + s.vl;
      int qs[HPW];
#pragma unroll
      for (int k = 0; k < HPW; ++k) qs[k] = (int)a.qS[ug * H + h0 + k];
      Row<VPL> hw = load_row<VPL>(hbase + ug * a.ldHp);
      int cur = 0;
      for (int64_t base = s.eb; base < s.ee; base += 32) {
        const int cnt = (int)(s.ee - base < 32 ? s.ee - base : 32);
        const int v = lane < cnt ? a.g.out_dst[base + lane] : 0;
        batch(cnt, v, qs, nullptr, cur, hw, [](int) {});
      }
      if (leader) a.hdS[(int64_t)s.slot * H + h0 + lh] = dS;
      float* dst = a.hagg + (int64_t)s.slot * HD + g * WC + lane * VPL;
#pragma unroll
      for (int k = 0; k < VPL; ++k) dst[k] = part[k];
      continue;
    }
    // ------------------------------------------------------------- tile of light source rows
    const int64_t r0 = (wi - hc) * TILE;
    int T;
    const TileLane L = tile_setup(a.g.out_ptr, a.pout.hbase, r0, n, T);
    const int64_t ug0 = a.g.row_begin + r0;
    int qsj[HPW];
#pragma unroll
    for (int k = 0; k < HPW; ++k) qsj[k] = L.deg > 0 ? (int)a.qS[(ug0 + lane) * H + h0 + k] : 0;
    unsigned zm = __ballot_sync(0xffffffffu, L.light && L.deg == 0);
    while (zm) {   // light rows without out-edges: ∂H′ = (0 + 0·a_src) + ∂D·a_dst
      const int j = __ffs(zm) - 1;
      zm &= zm - 1;
      cg_src_finalize<VPL, HPW>(a, r0 + j, ug0 + j, g, 0.0f, part, scG.s, amax_loc);
    }
    const unsigned act = __ballot_sync(0xffffffffu, L.deg > 0);
    int nxt = act ? __ffs(act) - 1 : -1;
    Row<VPL> hw_nxt{}, hw{};
    if (nxt >= 0) hw_nxt = load_row<VPL>(hbase + (ug0 + nxt) * a.ldHp);
    int cur = -1;
    auto on_row = [&](int ri) {
      if (cur >= 0) {
        const float dSb = __shfl_sync(0xffffffffu, dS, lh * LPH);
        cg_src_finalize<VPL, HPW>(a, r0 + cur, ug0 + cur, g, dSb, part, scG.s, amax_loc);
        dS = 0.0f;
      }
      hw = hw_nxt;
      nxt = tile_next(act, ri);
      if (nxt >= 0) hw_nxt = load_row<VPL>(hbase + (ug0 + nxt) * a.ldHp);
    };
    for (int base = 0; base < T; base += 32) {
      const int cnt = T - base < 32 ? T - base : 32;
      const int t = base + lane;
      const int row = tile_row(t, L.end);
      const int64_t e = __shfl_sync(0xffffffffu, L.eb, row) + (t - __shfl_sync(0xffffffffu, L.off, row));
      int qsr[HPW];
#pragma unroll
      for (int k = 0; k < HPW; ++k) qsr[k] = __shfl_sync(0xffffffffu, qsj[k], row);
      int v = 0;
      if (lane < cnt) {
        v = a.g.out_dst[e];
        sh_rb[w][lane] = row;
      }
      batch(cnt, v, qsr, sh_rb[w], cur, hw, on_row);
    }
    if (cur >= 0) {
      const float dSb = __shfl_sync(0xffffffffu, dS, lh * LPH);
      cg_src_finalize<VPL, HPW>(a, r0 + cur, ug0 + cur, g, dSb, part, scG.s, amax_loc);
    }
  }
  amax_flush(a.amax_dHp, amax_loc);
}

// FC: heavy rows — fold segment partials in chunk order, write m, den, H_out
template <int H, int VPL>
__global__ void __launch_bounds__(256) k_fwd_combine(const GatFwdArgs a) {
  constexpr int HD = 32 * VPL;
  __shared__ unsigned sh_amax;
  const int lane = threadIdx.x & 31;
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
    fold_rows<VPL>(a.hagg + (int64_t)base * HD + lane * VPL, HD, nseg, tot);
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

// ∂E = |α|(∂α − P[v]), ∂E_pre (stored beside α) and the segment's sequential Σ ∂E_pre (returned in
// lanes < H), from the stored signed α (its sign bit is the LeakyReLU branch of e_pre).
template <int H>
__device__ __forceinline__ float bwd_dst_pass2(const GatBwdArgs& a, const Seg& s, const float (&P)[H],
                                               float (*buf)[H]) {
  const int lane = threadIdx.x & 31;
  float part = 0.0f;
  for (int64_t base = s.eb; base < s.ee; base += 32 * segb<H>()) {
    float x[segb<H>()][H], dl[segb<H>()][H];
#pragma unroll
    for (int i = 0; i < segb<H>(); ++i) {
      const int64_t e = base + i * 32 + lane;
      if (e < s.ee)
#pragma unroll
        for (int h = 0; h < H; ++h) { x[i][h] = a.alpha[e * 2 * H + h]; dl[i][h] = a.dalpha[e * H + h]; }
    }
#pragma unroll
    for (int i = 0; i < segb<H>(); ++i) {
      const int64_t e = base + i * 32 + lane;
      if (e < s.ee)
#pragma unroll
        for (int h = 0; h < H; ++h) {
          const float dE = __fmul_rn(fabsf(x[i][h]), __fsub_rn(dl[i][h], P[h]));
          const float o = signbit(x[i][h]) ? __fmul_rn(dE, a.slope) : dE;
          buf[i * 32 + lane][h] = o;
          a.alpha_dE[e * 2 * H + H + h] = o;
        }
    }
    __syncwarp();
    const int cnt = (int)(s.ee - base < 32 * segb<H>() ? s.ee - base : 32 * segb<H>());
    if (lane < H)
      for (int i = 0; i < cnt; ++i) part = __fadd_rn(part, buf[i][lane]);
    __syncwarp();
  }
  return part;
}

// BD2: heavy segments -> P (fold of hP; segment 0 writes it), ∂D partial (hdD)
template <int H>
__global__ void __launch_bounds__(256) k_bwd_dst2(const GatBwdArgs a) {
  __shared__ float sh_a[WPB][32 * segb<H>()][H];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t hcnt = load_count(a.pin.counts);
  FOR_ITEMS(si, a.work + 1, hcnt) {
    Seg s;
    decode_item(si, hcnt, a.g.in_ptr, a.pin, a.g.chunk, s);
    const int64_t vg = a.g.row_begin + s.vl;
    float P[H];
    fold_segments<H>(a.hP, s.base, s.nseg, P);
    if (s.c == 0 && lane < H) a.P[vg * H + lane] = head_pick<H>(P, lane);
    const float dDp = bwd_dst_pass2<H>(a, s, P, sh_a[w]);
    if (lane < H) a.hdD[si * H + lane] = dDp;
  }
}

// BD3: heavy rows -> ∂D = fold of hdD (one warp per heavy row)
template <int H>
__global__ void __launch_bounds__(256) k_bwd_dst3(const GatBwdArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t hrows = load_count(a.pin.counts + 1);
  FOR_ITEMS(r, a.work + 5, hrows) {
    const int64_t vl = a.pin.hrow[r];
    const int base = a.pin.hbase[vl];
    const int64_t deg = a.g.in_ptr[vl + 1] - a.g.in_ptr[vl];
    const int nseg = (int)((deg + a.g.chunk - 1) / a.g.chunk);
    float tot[H];
    fold_segments<H>(a.hdD, base, nseg, tot);
    if (lane < H) a.dD[(a.g.row_begin + vl) * H + lane] = head_pick<H>(tot, lane);
  }
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
    float dSh[H];
    fold_segments<H>(a.hdS, base, nseg, dSh);
    const float dS = head_pick<H>(dSh, myh);
    float tot[VPL];
    fold_rows<VPL>(a.hagg + (int64_t)base * HD + lane * VPL, HD, nseg, tot);
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
  constexpr int RU = 8;   // rows in flight per warp
  __shared__ float sh_da[WPB][2][HD];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int myh = lane / LPH;
  const Scale scH = scale_from_amax(amax_load(a.amax_Hp), a.bits);
  const uint32_t flip = a.codes_biased ? 0u : 0x80808080u;   // to excess-128 for the PRMT conversion
  float das[VPL], dad[VPL];
#pragma unroll
  for (int k = 0; k < VPL; ++k) { das[k] = 0.0f; dad[k] = 0.0f; }
  // each warp streams a contiguous range of rows, RU rows per step
  const int64_t nw = (int64_t)gridDim.x * WPB, wid = (int64_t)blockIdx.x * WPB + w;
  const int64_t per = (a.g.n_local + nw - 1) / nw;
  const int64_t rb = wid * per, re = rb + per < a.g.n_local ? rb + per : a.g.n_local;
  for (int64_t ul0 = rb; ul0 < re; ul0 += RU) {
    Row<VPL> hw[RU];
    float dS[RU], dD[RU];
#pragma unroll
    for (int i = 0; i < RU; ++i) {
      const int64_t ul = ul0 + i < re ? ul0 + i : rb;
      const int64_t ug = a.g.row_begin + ul;
      dS[i] = ul0 + i < re ? a.dS[ug * H + myh] : 0.0f;
      dD[i] = ul0 + i < re ? a.dD[ug * H + myh] : 0.0f;
      hw[i] = load_row<VPL>(a.qHp + ug * a.ldHp + lane * VPL);
    }
#pragma unroll
    for (int i = 0; i < RU; ++i) {
      if constexpr (VPL < 4) {
#pragma unroll
        for (int k = 0; k < VPL; ++k) {
          const float hp = __fmul_rn(row_f<VPL>(hw[i], k), scH.s);
          das[k] = __fmaf_rn(dS[i], hp, das[k]);
          dad[k] = __fmaf_rn(dD[i], hp, dad[k]);
        }
        continue;
      }
      const float2 s2 = make_float2(dS[i], dS[i]), d2 = make_float2(dD[i], dD[i]);
#pragma unroll
      for (int q = 0; q < VPL / 4; ++q) {
        const uint32_t wx = hw[i].w[q] ^ flip;
#pragma unroll
        for (int z = 0; z < 2; ++z) {
          const float2 c = codes2(wx, z ? 0x7442u : 0x7440u, z ? 0x7443u : 0x7441u);
          const float2 hp = make_float2(__fmul_rn(c.x, scH.s), __fmul_rn(c.y, scH.s));
          const float2 sa = __ffma2_rn(s2, hp, make_float2(das[4 * q + 2 * z], das[4 * q + 2 * z + 1]));
          const float2 da = __ffma2_rn(d2, hp, make_float2(dad[4 * q + 2 * z], dad[4 * q + 2 * z + 1]));
          das[4 * q + 2 * z] = sa.x; das[4 * q + 2 * z + 1] = sa.y;
          dad[4 * q + 2 * z] = da.x; dad[4 * q + 2 * z + 1] = da.y;
        }
      }
    }
  }
#pragma unroll
  for (int k = 0; k < VPL; ++k) { sh_da[w][0][lane * VPL + k] = das[k]; sh_da[w][1][lane * VPL + k] = dad[k]; }
  __syncthreads();
  for (int j = threadIdx.x; j < 2 * HD; j += blockDim.x) {
    float t = 0.0f;
#pragma unroll
    for (int v = 0; v < WPB; ++v) t = __fadd_rn(t, (&sh_da[v][0][0])[j]);
    atomicAdd((j < HD ? a.da_src : a.da_dst) + (j % HD), t);
  }
}

// ------------------------------------------------------------------ dispatch
static int item_grid(int64_t items) {
  int64_t g = (items + WPB - 1) / WPB;
  const int64_t cap = (int64_t)num_sms() * 8;     // >= resident blocks; the work queue balances
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

// Heavy-row kernels: the number of heavy segments / rows is a device count (plan); a grid of 2
// blocks per SM keeps the work-queue claims cheap.  The hub chain runs beside the light sub-tiles,
// so its own occupancy matters little: 4 or 8 blocks per SM made the serialised products hub
// kernels 1.4x faster but the overlapped layer no faster (46.1 vs 46.6 ms) and arxiv slower
// (1.418 vs 1.409 ms).  TANGO_HUB_BLOCKS_PER_SM overrides the default of 2.
static int heavy_grid(int64_t cap) {
  static int per_sm = [] {
    const char* e = getenv("TANGO_HUB_BLOCKS_PER_SM");
    const int v = e ? atoi(e) : 2;
    return v > 0 ? v : 2;
  }();
  const int g = item_grid(cap);
  const int c = num_sms() * per_sm;
  return g < c ? g : c;
}

bool gat_codes_biased(int heads, int hd) { return hd / 32 >= 4 && heads <= 8; }

// (H, HD/32) for the row-wide kernels, (VPL, HPW) head-group shape for the gather kernels
#define TANGO_HV_CASES(X) X(1, 2) X(1, 4) X(1, 8) X(1, 16) X(2, 2) X(2, 4) X(2, 8) X(2, 16) \
                          X(4, 2) X(4, 4) X(4, 8) X(4, 16) X(8, 2) X(8, 4) X(8, 8) X(8, 16)
#define TANGO_CG_CASES(X) X(1, 4) X(1, 2) X(1, 1) X(2, 1) X(4, 1) X(8, 1) X(16, 1)

static bool cg_shape(int D, int& vpl, int& hpw) {
  if (D >= 32 && D % 32 == 0) {
    vpl = D / 32; hpw = 1;
    return vpl == 1 || vpl == 2 || vpl == 4 || vpl == 8 || vpl == 16;
  }
  if (D == 16) { vpl = 1; hpw = 2; return true; }
  if (D == 8) { vpl = 1; hpw = 4; return true; }
  return false;
}
bool gat_shape_supported(int heads, int head_dim) {
  int v, p;
  return cg_shape(head_dim, v, p);
}

// ---- hub / light split: the hub-row chain (segment statistics, folds) runs on a side stream beside
// the light sub-tiles, which need none of it (v4 engine, VPL >= 4).
static cudaError_t fork_to(cudaStream_t st, const SideStream& x) {
  cudaError_t e = cudaEventRecord(x.fork, st);
  return e == cudaSuccess ? cudaStreamWaitEvent(x.s, x.fork, 0) : e;
}
static cudaError_t join_from(cudaStream_t st, const SideStream& x) {
  cudaError_t e = cudaEventRecord(x.join, x.s);
  return e == cudaSuccess ? cudaStreamWaitEvent(st, x.join, 0) : e;
}

static cudaError_t launch_gat_fwd_split(const GatFwdArgs& a, cudaStream_t st, const SideStream& x) {
  const int hv = a.d.heads * 100 + a.d.hd / 32;
  GatFwdArgs ah = a, al = a;
  ah.part = 1;
  al.part = 2;
  cudaError_t e = fork_to(st, x);
  if (e != cudaSuccess) return e;
  bool ok = false;
#define X(H_, V_)                                                                                  \
  if (hv == H_ * 100 + V_ && V_ >= 4) {                                                            \
    ok = true;                                                                                     \
    constexpr int VV = V_ >= 4 ? V_ : 4;                                                           \
    constexpr int fsm = 8 * fs_warp_smem<H_>();                                                    \
    constexpr int smem = 8 * g4_warp_smem<H_, VV, false>();                                        \
    static bool attr_set = false;                                                                  \
    if (!attr_set) {                                                                               \
      cudaFuncSetAttribute(k_fwd_stats_t<H_>, cudaFuncAttributeMaxDynamicSharedMemorySize, fsm);   \
      cudaFuncSetAttribute(k_fwd_agg4<H_, VV>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
      attr_set = true;                                                                             \
    }                                                                                              \
    { ProfScope p("gat_fwd_stats_hub", x.s); k_fwd_stats_t<H_><<<heavy_grid(a.plan.cap), 256, fsm, x.s>>>(ah); } \
    { ProfScope p("gat_fwd_stats2", x.s); k_fwd_stats2<H_><<<heavy_grid(a.plan.cap), 256, 0, x.s>>>(ah); } \
    { ProfScope p("gat_fwd_alpha3", x.s); k_fwd_alpha3<H_><<<heavy_grid(a.plan.cap), 256, 0, x.s>>>(ah); } \
    { ProfScope p("gat_fwd_agg_hub", x.s); k_fwd_agg4<H_, VV><<<heavy_grid(a.plan.cap), 256, smem, x.s>>>(ah); } \
    { ProfScope p("gat_fwd_combine", x.s); k_fwd_combine<H_, V_><<<heavy_grid(a.plan.cap), 256, 0, x.s>>>(ah); } \
    { ProfScope p("gat_fwd_stats", st); k_fwd_stats_t<H_><<<item_grid(a.plan.tcap), 256, fsm, st>>>(al); } \
    { ProfScope p("gat_fwd_agg", st); k_fwd_agg4<H_, VV><<<item_grid(a.plan.tcap), 256, smem, st>>>(al); } \
  }
  TANGO_HV_CASES(X)
#undef X
  if (!ok) return cudaErrorInvalidValue;
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  return join_from(st, x);
}

static cudaError_t launch_gat_bwd_dst_split(const GatBwdArgs& a, cudaStream_t st, const SideStream& x) {
  const int hv = a.d.heads * 100 + a.d.hd / 32;
  GatBwdArgs ah = a, al = a;
  ah.part = 1;
  al.part = 2;
  cudaError_t e = fork_to(st, x);
  if (e != cudaSuccess) return e;
  bool ok = false;
#define X(H_, V_)                                                                                  \
  if (hv == H_ * 100 + V_ && V_ >= 4 && H_ <= 8) {                                                 \
    ok = true;                                                                                     \
    constexpr int VV = V_ >= 4 ? V_ : 4;                                                           \
    constexpr int NW = 7, smem4 = NW * dst4_warp_smem<H_, VV>();                                   \
    static bool attr_set = false;                                                                  \
    if (!attr_set) {                                                                               \
      cudaFuncSetAttribute(k_bwd_dst1_v4<H_, VV, NW, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem4); cudaFuncSetAttribute(k_bwd_dst1_v4<H_, VV, NW, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem4); \
      attr_set = true;                                                                             \
    }                                                                                              \
    { ProfScope p("gat_bwd_dst1_hub", x.s);                                                        \
      if (a.codes_biased) k_bwd_dst1_v4<H_, VV, NW, true><<<heavy_grid(a.pin.cap), NW * 32, smem4, x.s>>>(ah); else k_bwd_dst1_v4<H_, VV, NW, false><<<heavy_grid(a.pin.cap), NW * 32, smem4, x.s>>>(ah); }             \
    { ProfScope p("gat_bwd_dst2", x.s); k_bwd_dst2<H_><<<heavy_grid(a.pin.cap), 256, 0, x.s>>>(ah); } \
    { ProfScope p("gat_bwd_dst3", x.s); k_bwd_dst3<H_><<<heavy_grid(a.pin.cap), 256, 0, x.s>>>(ah); } \
    { ProfScope p("gat_bwd_dst1", st);                                                             \
      if (a.codes_biased) k_bwd_dst1_v4<H_, VV, NW, true><<<item_grid(a.pin.tcap), NW * 32, smem4, st>>>(al); else k_bwd_dst1_v4<H_, VV, NW, false><<<item_grid(a.pin.tcap), NW * 32, smem4, st>>>(al); }              \
  }
  TANGO_HV_CASES(X)
#undef X
  if (!ok) return cudaErrorInvalidValue;
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  return join_from(st, x);
}

static cudaError_t launch_gat_bwd_src_split(const GatBwdArgs& a, cudaStream_t st, const SideStream& x) {
  const int hv = a.d.heads * 100 + a.d.hd / 32;
  GatBwdArgs ah = a, al = a;
  ah.part = 1;
  al.part = 2;
  cudaError_t e = fork_to(st, x);
  if (e != cudaSuccess) return e;
  bool ok = false;
#define X(H_, V_)                                                                                  \
  if (hv == H_ * 100 + V_ && V_ >= 4) {                                                            \
    ok = true;                                                                                     \
    constexpr int VV = V_ >= 4 ? V_ : 4;                                                           \
    constexpr int NW = 4, smem4 = NW * g4_warp_smem<H_, VV, true>();                               \
    static bool attr_set = false;                                                                  \
    if (!attr_set) {                                                                               \
      cudaFuncSetAttribute(k_bwd_src4<H_, VV, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem4); \
      attr_set = true;                                                                             \
    }                                                                                              \
    { ProfScope p("gat_bwd_src_hub", x.s);                                                         \
      k_bwd_src4<H_, VV, NW><<<heavy_grid(a.pout.cap), NW * 32, smem4, x.s>>>(ah); }               \
    { ProfScope p("gat_bwd_src_combine", x.s);                                                     \
      k_bwd_src_combine<H_, V_><<<heavy_grid(a.pout.cap), 256, 0, x.s>>>(ah); }                    \
    { ProfScope p("gat_bwd_src", st);                                                              \
      k_bwd_src4<H_, VV, NW><<<item_grid(a.pout.tcap), NW * 32, smem4, st>>>(al); }                \
  }
  TANGO_HV_CASES(X)
#undef X
  if (!ok) return cudaErrorInvalidValue;
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  return join_from(st, x);
}

cudaError_t launch_gat_fwd(const GatFwdArgs& a, cudaStream_t st, const SideStream* aux) {
  if (a.g.n_local == 0) return cudaSuccess;
  if (aux && a.d.hd / 32 >= 4) return launch_gat_fwd_split(a, st, *aux);
  const int hv = a.d.heads * 100 + a.d.hd / 32;
  int vpl, hpw;
  if (!cg_shape(a.d.head_dim, vpl, hpw)) return cudaErrorInvalidValue;
  const int64_t cg_items = (a.plan.cap + (a.g.n_local + TILE - 1) / TILE) * (a.d.hd / (32 * vpl));
  bool ok = false;
#define X(H_, V_)                                                                                  \
  if (hv == H_ * 100 + V_) {                                                                       \
    ok = true;                                                                                     \
    { ProfScope p("gat_fwd_stats", st);                                                            \
      constexpr int fsm = 8 * fs_warp_smem<H_>();                                                  \
      static bool fs_attr = false;                                                                 \
      if (!fs_attr) {                                                                              \
        cudaFuncSetAttribute(k_fwd_stats_t<H_>, cudaFuncAttributeMaxDynamicSharedMemorySize, fsm); \
        fs_attr = true;                                                                            \
      }                                                                                            \
      k_fwd_stats_t<H_><<<item_grid(a.plan.cap + a.plan.tcap), 256, fsm, st>>>(a); }               \
    { ProfScope p("gat_fwd_stats2", st); k_fwd_stats2<H_><<<heavy_grid(a.plan.cap), 256, 0, st>>>(a); } \
  }
  TANGO_HV_CASES(X)
#undef X
  if (!ok) return cudaErrorInvalidValue;
  (void)cg_items;
  ok = false;
#define X(H_, V_)                                                                                  \
  if (hv == H_ * 100 + V_) {                                                                       \
    ok = true;                                                                                     \
    { ProfScope p("gat_fwd_alpha3", st); k_fwd_alpha3<H_><<<heavy_grid(a.plan.cap), 256, 0, st>>>(a); } \
    { ProfScope p("gat_fwd_agg", st);                                                              \
      if (V_ >= 4) {                                                                               \
        constexpr int smem = 8 * g4_warp_smem<H_, (V_ >= 4 ? V_ : 4), false>();                     \
        static bool attr_set = false;                                                              \
        if (!attr_set) {                                                                           \
          cudaFuncSetAttribute(k_fwd_agg4<H_, (V_ >= 4 ? V_ : 4)>,                                 \
                               cudaFuncAttributeMaxDynamicSharedMemorySize, smem);                 \
          attr_set = true;                                                                         \
        }                                                                                          \
        k_fwd_agg4<H_, (V_ >= 4 ? V_ : 4)><<<item_grid(a.plan.cap + a.plan.tcap), 256, smem, st>>>(a); \
      } else {                                                                                     \
        k_fwd_agg2<H_, V_><<<item_grid(a.plan.cap + a.plan.tcap), 256, 0, st>>>(a);               \
      } }                                                                                          \
    { ProfScope p("gat_fwd_combine", st);                                                          \
      k_fwd_combine<H_, V_><<<heavy_grid(a.plan.cap), 256, 0, st>>>(a); }                           \
  }
  TANGO_HV_CASES(X)
#undef X
  return cudaGetLastError();
}

cudaError_t launch_gat_bwd_dst(const GatBwdArgs& a, cudaStream_t st, const SideStream* aux) {
  if (a.g.n_local == 0) return cudaSuccess;
  if (aux && a.d.hd / 32 >= 4 && a.d.heads <= 8) return launch_gat_bwd_dst_split(a, st, *aux);
  int vpl, hpw;
  if (!cg_shape(a.d.head_dim, vpl, hpw)) return cudaErrorInvalidValue;
  const int64_t cg_items = (a.pin.cap + (a.g.n_local + TILE - 1) / TILE) * (a.d.hd / (32 * vpl));
  bool ok = false;
  const int hv = a.d.heads * 100 + a.d.hd / 32;
  if (a.d.hd / 32 >= 4) {
#define X(H_, V_)                                                                                  \
    if (hv == H_ * 100 + V_ && V_ >= 4) {                                                          \
      ok = true;                                                                                   \
      constexpr int VV = V_ >= 4 ? V_ : 4;                                                          \
      ProfScope p("gat_bwd_dst1", st);                                                             \
      if (H_ <= 8) {                                                                               \
        constexpr int NW = 7, smem4 = NW * dst4_warp_smem<H_, VV>();                               \
        static bool attr4_set = false;                                                             \
        if (!attr4_set) {                                                                          \
          cudaFuncSetAttribute(k_bwd_dst1_v4<H_, VV, NW, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem4); cudaFuncSetAttribute(k_bwd_dst1_v4<H_, VV, NW, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem4); \
          attr4_set = true;                                                                        \
        }                                                                                          \
        if (a.codes_biased) k_bwd_dst1_v4<H_, VV, NW, true><<<item_grid(a.pin.cap + a.pin.tcap), NW * 32, smem4, st>>>(a); else k_bwd_dst1_v4<H_, VV, NW, false><<<item_grid(a.pin.cap + a.pin.tcap), NW * 32, smem4, st>>>(a);   \
      }                                                                                            \
    }
    TANGO_HV_CASES(X)
#undef X
  } else {
#define X(V_, P_)                                                                                  \
    if (vpl == V_ && hpw == P_) {                                                                  \
      ok = true;                                                                                   \
      ProfScope p("gat_bwd_dst1", st);                                                             \
      k_bwd_dst1_cg<V_, P_><<<item_grid(cg_items), 256, 0, st>>>(a);                                \
    }
    TANGO_CG_CASES(X)
#undef X
  }
  if (!ok) return cudaErrorInvalidValue;
  ok = false;
#define X(H_, V_)                                                                                  \
  if (hv == H_ * 100 + V_) {                                                                       \
    ok = true;                                                                                     \
    { ProfScope p("gat_bwd_dst2", st); k_bwd_dst2<H_><<<heavy_grid(a.pin.cap), 256, 0, st>>>(a); }  \
    { ProfScope p("gat_bwd_dst3", st);                                                             \
      k_bwd_dst3<H_><<<heavy_grid(a.pin.cap), 256, 0, st>>>(a); }                                         \
  }
  TANGO_HV_CASES(X)
#undef X
  if (!ok) return cudaErrorInvalidValue;
  return cudaGetLastError();
}

cudaError_t launch_gat_bwd_src(const GatBwdArgs& a, cudaStream_t st, const SideStream* aux) {
  if (a.g.n_local == 0) return cudaSuccess;
  if (aux && a.d.hd / 32 >= 4 && a.g.out_eid) return launch_gat_bwd_src_split(a, st, *aux);
  int vpl, hpw;
  if (!cg_shape(a.d.head_dim, vpl, hpw)) return cudaErrorInvalidValue;
  const int64_t cg_items = (a.pout.cap + (a.g.n_local + TILE - 1) / TILE) * (a.d.hd / (32 * vpl));
  bool ok = false;
  const int hv = a.d.heads * 100 + a.d.hd / 32;
  if (a.d.hd / 32 >= 4) {
#define X(H_, V_)                                                                                  \
    if (hv == H_ * 100 + V_ && V_ >= 4) {                                                          \
      ok = true;                                                                                   \
      constexpr int VV = V_ >= 4 ? V_ : 4;                                                          \
      constexpr int smem = 8 * bwd3_warp_smem<H_, VV>();                                           \
      static bool attr_set = false;                                                                \
      if (!attr_set) {                                                                             \
        cudaFuncSetAttribute(k_bwd_src_v3<H_, VV, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
        cudaFuncSetAttribute(k_bwd_src_v3<H_, VV, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
        attr_set = true;                                                                           \
      }                                                                                            \
      ProfScope p("gat_bwd_src", st);                                                              \
      if (a.g.out_eid) {                                                                           \
        constexpr int NW = 4, smem4 = NW * g4_warp_smem<H_, VV, true>();                           \
        static bool attr4_set = false;                                                             \
        if (!attr4_set) {                                                                          \
          cudaFuncSetAttribute(k_bwd_src4<H_, VV, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem4); \
          attr4_set = true;                                                                        \
        }                                                                                          \
        k_bwd_src4<H_, VV, NW><<<item_grid(a.pout.cap + a.pout.tcap), NW * 32, smem4, st>>>(a);  \
      } else {                                                                                     \
        if (a.codes_biased) k_bwd_src_v3<H_, VV, true><<<item_grid(a.pout.cap + a.pout.tcap), 256, smem, st>>>(a); \
        else k_bwd_src_v3<H_, VV, false><<<item_grid(a.pout.cap + a.pout.tcap), 256, smem, st>>>(a);  \
      }                                                                                            \
    }
    TANGO_HV_CASES(X)
#undef X
  } else {
#define X(V_, P_)                                                                                  \
    if (vpl == V_ && hpw == P_) {                                                                  \
      ok = true;                                                                                   \
      ProfScope p("gat_bwd_src", st);                                                              \
      k_bwd_src_cg<V_, P_><<<item_grid(cg_items), 256, 0, st>>>(a);                                 \
    }
    TANGO_CG_CASES(X)
#undef X
  }
  if (!ok) return cudaErrorInvalidValue;
  ok = false;
#define X(H_, V_)                                                                                  \
  if (hv == H_ * 100 + V_) {                                                                       \
    ok = true;                                                                                     \
    { ProfScope p("gat_bwd_src_combine", st);                                                      \
      k_bwd_src_combine<H_, V_><<<heavy_grid(a.pout.cap), 256, 0, st>>>(a); }                     \
  }
  TANGO_HV_CASES(X)
#undef X
  if (!ok) return cudaErrorInvalidValue;
  return cudaGetLastError();
}

// ②′ for the attention vectors (∂a_src, ∂a_dst); needs ∂S, ∂D of the owned rows (after the source pass)
cudaError_t launch_gat_attn_grad(const GatBwdArgs& a, cudaStream_t st) {
  if (a.g.n_local == 0) return cudaSuccess;
  const int hv = a.d.heads * 100 + a.d.hd / 32;
  bool ok = false;
#define X(H_, V_)                                                                                  \
  if (hv == H_ * 100 + V_) {                                                                       \
    ok = true;                                                                                     \
    ProfScope p("gat_bwd_attn_grad", st);                                                          \
    k_bwd_attn_grad<H_, V_><<<num_sms() * 4, 256, 0, st>>>(a);                                     \
  }
  TANGO_HV_CASES(X)
#undef X
  if (!ok) return cudaErrorInvalidValue;
  return cudaGetLastError();
}

}  // namespace tango
