// gat.cu — the sparse half of the quantized GAT layer as fused destination / source row kernels,
// plus the unfused primitives exposed by the C ABI (tango_sddmm_q, tango_edge_softmax, ...).
//
// Paper: ③ SDDMM-add + LeakyReLU, ④ edge softmax (FP32 per P:604-615),
// ⑤ SPMM, ⑤′ SPMM on the reversed graph, ⑤″ SDDMM-dot on codes
// (P:252-255), ④′ softmax backward, ③′/③″ incidence SPMM (P:276,
// P:821-832), ②′ (reading R23).
//
// B200 design: one warp per node row.  A node row of HD int8 codes is split
// across the 32 lanes (VPL = HD/32 codes per lane, 16 B per lane at HD = 512), so one warp-wide
// 16-B load gathers a whole 512-B source row: coalesced, vectorised, one L2 sector per 32 B.
// Per-edge scalars (α, ∂α, e_pre) are computed lane-parallel over 32-edge batches and staged in
// shared memory; every reduction that feeds a value compared bit-for-bit with the oracle runs
// sequentially in the canonical edge order with the chunked sum Σᶜ (reading R14).  α, ∂α and
// ∂E are recomputed from per-node data instead of being stored per edge (reading R30), so the
// only edge-sized arrays are the CSR indices and one fp32 ∂α scratch in the backward dst pass.
#include "kernels.h"

namespace tango {

// ------------------------------------------------------------------ helpers
template <int VPL>
struct Row {
  uint32_t w[(VPL + 3) / 4];
};
template <int VPL>
__device__ __forceinline__ Row<VPL> load_row(const int8_t* p) {
  Row<VPL> r;
  if constexpr (VPL == 16) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(p));
    r.w[0] = v.x; r.w[1] = v.y; r.w[2] = v.z; r.w[3] = v.w;
  } else if constexpr (VPL == 8) {
    const uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
    r.w[0] = v.x; r.w[1] = v.y;
  } else if constexpr (VPL == 4) {
    r.w[0] = __ldg(reinterpret_cast<const unsigned*>(p));
  } else if constexpr (VPL == 2) {
    r.w[0] = (uint32_t)__ldg(reinterpret_cast<const unsigned short*>(p));
  } else {
    r.w[0] = (uint32_t)__ldg(reinterpret_cast<const unsigned char*>(p));
  }
  return r;
}
template <int VPL>
__device__ __forceinline__ float row_f(const Row<VPL>& r, int k) {
  return i8_to_f(r.w[k >> 2], k & 3);
}
template <int VPL>
__device__ __forceinline__ int row_dot(const Row<VPL>& a, const Row<VPL>& b) {
  int acc = 0;
  if constexpr (VPL >= 4) {
#pragma unroll
    for (int i = 0; i < VPL / 4; ++i) acc = __dp4a((int)a.w[i], (int)b.w[i], acc);
  } else {
#pragma unroll
    for (int k = 0; k < VPL; ++k)
      acc += (int)(int8_t)((a.w[0] >> (8 * k)) & 0xFF) * (int)(int8_t)((b.w[0] >> (8 * k)) & 0xFF);
  }
  return acc;
}
__device__ __forceinline__ float i8f(int8_t v) { return __int2float_rn((int)v); }

// Chunked sum state (reading R14): partial sums restart every C_E list elements.
struct CSum {
  float total, part;
  bool folded;
  __device__ __forceinline__ void init() { total = 0.0f; part = 0.0f; folded = false; }
  __device__ __forceinline__ void fold() {
    total = folded ? __fadd_rn(total, part) : part;
    part = 0.0f;
    folded = true;
  }
  __device__ __forceinline__ float finish(int64_t len) const {
    if (len == 0) return 0.0f;
    return folded ? __fadd_rn(total, part) : part;
  }
};

// e_pre for edge (u -> v), head h (reading: two rn multiplies, one rn add, order a + b)
__device__ __forceinline__ float sddmm_add1(int8_t qs, float sS, int8_t qd, float sD) {
  return __fadd_rn(__fmul_rn(i8f(qs), sS), __fmul_rn(i8f(qd), sD));
}

// ================================================================== fused forward, destination rows
// F5 (③ + ④) and F6 (⑤) for one destination row per warp:
//   pass 1: m = max el (lane-parallel over edges, butterfly max — order-free)
//   pass 2: den = Σᶜ exp_p(el - m) (lane-parallel exp, sequential chunked sum by lane h)
//   pass 3: α = ex/den (lane-parallel), H_out = (Σᶜ fmaf(α, q_H′[u])) * s_H′ (lanes over features)
template <int H, int VPL>
__global__ void __launch_bounds__(256) k_gat_fwd_dst(const GatFwdDstArgs a) {
  constexpr int WPB = 8;
  constexpr int LPH = 32 / H;  // lanes per head
  __shared__ float sh_val[WPB][32][H];
  __shared__ int sh_red;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float(*buf)[H] = sh_val[w];
  const int myh = lane / LPH;
  const Scale scS = scale_from_amax(amax_load(a.amax_S), a.bits);
  const Scale scD = scale_from_amax(amax_load(a.amax_D), a.bits);
  const Scale scH = scale_from_amax(amax_load(a.amax_Hp), a.bits);
  const float slope = a.slope;
  const int chunk = a.g.chunk;
  constexpr int HD = 32 * VPL;
  float amax_loc = 0.0f;
  if (threadIdx.x == 0) sh_red = 0;
  for (int64_t vl = (int64_t)blockIdx.x * WPB + w; vl < a.g.n_local; vl += (int64_t)gridDim.x * WPB) {
    const int64_t vg = a.g.row_begin + vl;
    const int64_t beg = a.g.in_ptr[vl], end = a.g.in_ptr[vl + 1], deg = end - beg;
    int8_t qd[H];
#pragma unroll
    for (int h = 0; h < H; ++h) qd[h] = a.qD[vg * H + h];
    // ---- pass 1: max
    float mx[H];
#pragma unroll
    for (int h = 0; h < H; ++h) mx[h] = -INFINITY;
    for (int64_t base = beg; base < end; base += 32) {
      const int64_t e = base + lane;
      if (e < end) {
        const int64_t u = a.g.in_src[e];
#pragma unroll
        for (int h = 0; h < H; ++h) mx[h] = fmaxf(mx[h], lrelu(sddmm_add1(a.qS[u * H + h], scS.s, qd[h], scD.s), slope));
      }
    }
#pragma unroll
    for (int h = 0; h < H; ++h) { mx[h] = warp_max(mx[h]); if (deg == 0) mx[h] = 0.0f; }
    // ---- pass 2: den
    CSum cs; cs.init();
    int left = chunk;
    for (int64_t base = beg; base < end; base += 32) {
      const int cnt = (int)(end - base < 32 ? end - base : 32);
      if (lane < cnt) {
        const int64_t u = a.g.in_src[base + lane];
#pragma unroll
        for (int h = 0; h < H; ++h)
          buf[lane][h] = exp_p(__fsub_rn(lrelu(sddmm_add1(a.qS[u * H + h], scS.s, qd[h], scD.s), slope), mx[h]));
      }
      __syncwarp();
      if (lane < H) {
        for (int i = 0; i < cnt; ++i) {
          if (left == 0) { cs.fold(); left = chunk; }
          cs.part = __fadd_rn(cs.part, buf[i][lane]);
          --left;
        }
      }
      __syncwarp();
    }
    const float den_mine = (lane < H) ? cs.finish(deg) : 0.0f;
    float den[H];
#pragma unroll
    for (int h = 0; h < H; ++h) den[h] = __shfl_sync(0xffffffffu, den_mine, h);
    // ---- pass 3: α and aggregation
    float tot[VPL], part[VPL];
#pragma unroll
    for (int k = 0; k < VPL; ++k) { tot[k] = 0.0f; part[k] = 0.0f; }
    bool folded = false;
    left = chunk;
    const int8_t* qbase = a.qHp + lane * VPL;
    for (int64_t base = beg; base < end; base += 32) {
      const int cnt = (int)(end - base < 32 ? end - base : 32);
      int u_reg = 0;
      if (lane < cnt) {
        u_reg = a.g.in_src[base + lane];
#pragma unroll
        for (int h = 0; h < H; ++h)
          buf[lane][h] = __fdiv_rn(
              exp_p(__fsub_rn(lrelu(sddmm_add1(a.qS[(int64_t)u_reg * H + h], scS.s, qd[h], scD.s), slope), mx[h])),
              den[h]);
      }
      __syncwarp();
      int i = 0;
      for (; i + 4 <= cnt; i += 4) {
        Row<VPL> r[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int u = __shfl_sync(0xffffffffu, u_reg, i + j);
          r[j] = load_row<VPL>(qbase + (int64_t)u * a.ldHp);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (left == 0) {
#pragma unroll
            for (int k = 0; k < VPL; ++k) { tot[k] = folded ? __fadd_rn(tot[k], part[k]) : part[k]; part[k] = 0.0f; }
            folded = true; left = chunk;
          }
          const float al = buf[i + j][myh];
#pragma unroll
          for (int k = 0; k < VPL; ++k) part[k] = __fmaf_rn(al, row_f<VPL>(r[j], k), part[k]);
          --left;
        }
      }
      for (; i < cnt; ++i) {
        const int u = __shfl_sync(0xffffffffu, u_reg, i);
        const Row<VPL> r = load_row<VPL>(qbase + (int64_t)u * a.ldHp);
        if (left == 0) {
#pragma unroll
          for (int k = 0; k < VPL; ++k) { tot[k] = folded ? __fadd_rn(tot[k], part[k]) : part[k]; part[k] = 0.0f; }
          folded = true; left = chunk;
        }
        const float al = buf[i][myh];
#pragma unroll
        for (int k = 0; k < VPL; ++k) part[k] = __fmaf_rn(al, row_f<VPL>(r, k), part[k]);
        --left;
      }
      __syncwarp();
    }
    float out[VPL];
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const float s = deg == 0 ? 0.0f : (folded ? __fadd_rn(tot[k], part[k]) : part[k]);
      out[k] = __fmul_rn(s, scH.s);
      amax_loc = fmaxf(amax_loc, fabsf(out[k]));
    }
    float* dst = a.Hout + vl * HD + lane * VPL;
    if constexpr (VPL % 4 == 0) {
#pragma unroll
      for (int k = 0; k < VPL; k += 4) *reinterpret_cast<float4*>(dst + k) = make_float4(out[k], out[k + 1], out[k + 2], out[k + 3]);
    } else {
#pragma unroll
      for (int k = 0; k < VPL; ++k) dst[k] = out[k];
    }
    if (lane < H) {
      float mm = 0.0f;
#pragma unroll
      for (int h = 0; h < H; ++h) if (lane == h) mm = mx[h];
      a.m[vg * H + lane] = mm;
      a.den[vg * H + lane] = den_mine;
    }
  }
  if (a.amax_out) {
    amax_loc = warp_max(amax_loc);
    __syncthreads();
    if (lane == 0) atomicMax(reinterpret_cast<unsigned*>(&sh_red), __float_as_uint(amax_loc));
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(a.amax_out, (unsigned)sh_red);
  }
}

// ================================================================== fused backward, destination rows
// B2 ⑤″ ∂α = i2f(q_G[v]·q_H′[u]) * (s_G s_H′) (IDP4A, exact), B3 ④′ P and ∂E_pre, B4 ③″ ∂D.
template <int H, int VPL>
__global__ void __launch_bounds__(256) k_gat_bwd_dst(const GatBwdDstArgs a) {
  constexpr int WPB = 8;
  constexpr int LPH = 32 / H;
  __shared__ float sh_a[WPB][32][H];
  __shared__ float sh_d[WPB][32][H];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float(*ba)[H] = sh_a[w];
  float(*bd)[H] = sh_d[w];
  const int myh = lane / LPH;
  const bool leader = (lane % LPH) == 0;
  const Scale scS = scale_from_amax(amax_load(a.amax_S), a.bits);
  const Scale scD = scale_from_amax(amax_load(a.amax_D), a.bits);
  const Scale scH = scale_from_amax(amax_load(a.amax_Hp), a.bits);
  const Scale scG = scale_from_amax(amax_load(a.amax_G), a.bits);
  const float sGH = __fmul_rn(scG.s, scH.s);
  const float slope = a.slope;
  const int chunk = a.g.chunk;
  for (int64_t vl = (int64_t)blockIdx.x * WPB + w; vl < a.g.n_local; vl += (int64_t)gridDim.x * WPB) {
    const int64_t vg = a.g.row_begin + vl;
    const int64_t beg = a.g.in_ptr[vl], end = a.g.in_ptr[vl + 1], deg = end - beg;
    int8_t qd[H];
    float mh[H], dh[H];
#pragma unroll
    for (int h = 0; h < H; ++h) { qd[h] = a.qD[vg * H + h]; mh[h] = a.m[vg * H + h]; dh[h] = a.den[vg * H + h]; }
    const Row<VPL> gw = load_row<VPL>(a.qG + vg * a.ldG + lane * VPL);
    // ---- pass 1: ∂α per edge, P = Σᶜ fmaf(∂α, α)
    CSum cp; cp.init();
    int left = chunk;
    for (int64_t base = beg; base < end; base += 32) {
      const int cnt = (int)(end - base < 32 ? end - base : 32);
      int u_reg = 0;
      if (lane < cnt) {
        u_reg = a.g.in_src[base + lane];
#pragma unroll
        for (int h = 0; h < H; ++h)
          ba[lane][h] = __fdiv_rn(
              exp_p(__fsub_rn(lrelu(sddmm_add1(a.qS[(int64_t)u_reg * H + h], scS.s, qd[h], scD.s), slope), mh[h])),
              dh[h]);
      }
      __syncwarp();
      for (int i = 0; i < cnt; ++i) {
        const int u = __shfl_sync(0xffffffffu, u_reg, i);
        const Row<VPL> hw = load_row<VPL>(a.qHp + (int64_t)u * a.ldHp + lane * VPL);
        int dot = row_dot<VPL>(gw, hw);
#pragma unroll
        for (int o = 1; o < LPH; o <<= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
        const float dal = __fmul_rn(__int2float_rn(dot), sGH);
        if (left == 0) { cp.fold(); left = chunk; }
        if (leader) {
          cp.part = __fmaf_rn(dal, ba[i][myh], cp.part);
          bd[i][myh] = dal;
        }
        --left;
      }
      __syncwarp();
      for (int idx = lane; idx < cnt * H; idx += 32) a.dalpha[base * H + idx] = bd[idx / H][idx % H];
      __syncwarp();
    }
    const float P_lead = cp.finish(deg);
    float P[H];
#pragma unroll
    for (int h = 0; h < H; ++h) P[h] = __shfl_sync(0xffffffffu, P_lead, h * LPH);
    // ---- pass 2: ∂E_pre and ∂D = Σᶜ ∂E_pre
    CSum cd; cd.init();
    left = chunk;
    for (int64_t base = beg; base < end; base += 32) {
      const int cnt = (int)(end - base < 32 ? end - base : 32);
      if (lane < cnt) {
        const int64_t e = base + lane;
        const int64_t u = a.g.in_src[e];
#pragma unroll
        for (int h = 0; h < H; ++h) {
          const float ep = sddmm_add1(a.qS[u * H + h], scS.s, qd[h], scD.s);
          const float al = __fdiv_rn(exp_p(__fsub_rn(lrelu(ep, slope), mh[h])), dh[h]);
          const float dE = __fmul_rn(al, __fsub_rn(a.dalpha[e * H + h], P[h]));
          ba[lane][h] = ep > 0.0f ? dE : __fmul_rn(dE, slope);
        }
      }
      __syncwarp();
      if (lane < H) {
        for (int i = 0; i < cnt; ++i) {
          if (left == 0) { cd.fold(); left = chunk; }
          cd.part = __fadd_rn(cd.part, ba[i][lane]);
          --left;
        }
      }
      __syncwarp();
    }
    if (lane < H) {
      float pm = 0.0f;
#pragma unroll
      for (int h = 0; h < H; ++h) if (lane == h) pm = P[h];
      a.P[vg * H + lane] = pm;
      a.dD[vg * H + lane] = cd.finish(deg);
    }
  }
}

// ================================================================== fused backward, source rows
// B5 ⑤′ ∂H′_agg = (Σᶜ over out-edges fmaf(α, q_G[v])) * s_G, B6 ③′ ∂S = Σᶜ ∂E_pre, B7 ②′ ∂H′ and ∂a.
// α, ∂α and ∂E_pre of each out-edge are recomputed from per-node data (q_S[u], q_D[v], m[v], den[v],
// P[v]) and the two gathered rows q_G[v], q_H′[u] — bit-identical to the destination-side values.
template <int H, int VPL>
__global__ void __launch_bounds__(256) k_gat_bwd_src(const GatBwdSrcArgs a) {
  constexpr int WPB = 8;
  constexpr int LPH = 32 / H;
  constexpr int HD = 32 * VPL;
  __shared__ float sh_a[WPB][32][H];
  __shared__ float sh_e[WPB][32][H];
  __shared__ float sh_p[WPB][32][H];
  __shared__ float sh_da[2][HD];
  __shared__ unsigned sh_amax;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float(*ba)[H] = sh_a[w];
  float(*be)[H] = sh_e[w];
  float(*bp)[H] = sh_p[w];
  const int myh = lane / LPH;
  const bool leader = (lane % LPH) == 0;
  for (int j = threadIdx.x; j < 2 * HD; j += blockDim.x) (&sh_da[0][0])[j] = 0.0f;
  if (threadIdx.x == 0) sh_amax = 0u;
  __syncthreads();
  const Scale scS = scale_from_amax(amax_load(a.amax_S), a.bits);
  const Scale scD = scale_from_amax(amax_load(a.amax_D), a.bits);
  const Scale scH = scale_from_amax(amax_load(a.amax_Hp), a.bits);
  const Scale scG = scale_from_amax(amax_load(a.amax_G), a.bits);
  const float sGH = __fmul_rn(scG.s, scH.s);
  const float slope = a.slope;
  const int chunk = a.g.chunk;
  float asrc[VPL], adst[VPL], das[VPL], dad[VPL];
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    asrc[k] = a.a_src[lane * VPL + k];
    adst[k] = a.a_dst[lane * VPL + k];
    das[k] = 0.0f; dad[k] = 0.0f;
  }
  float amax_loc = 0.0f;
  for (int64_t ul = (int64_t)blockIdx.x * WPB + w; ul < a.g.n_local; ul += (int64_t)gridDim.x * WPB) {
    const int64_t ug = a.g.row_begin + ul;
    const int64_t beg = a.g.out_ptr[ul], end = a.g.out_ptr[ul + 1], deg = end - beg;
    int8_t qs[H];
#pragma unroll
    for (int h = 0; h < H; ++h) qs[h] = a.qS[ug * H + h];
    const Row<VPL> hw = load_row<VPL>(a.qHp + ug * a.ldHp + lane * VPL);
    CSum cs; cs.init();
    float tot[VPL], part[VPL];
#pragma unroll
    for (int k = 0; k < VPL; ++k) { tot[k] = 0.0f; part[k] = 0.0f; }
    bool folded = false;
    int left = chunk;
    const int8_t* gbase = a.qG + lane * VPL;
    for (int64_t base = beg; base < end; base += 32) {
      const int cnt = (int)(end - base < 32 ? end - base : 32);
      int v_reg = 0;
      if (lane < cnt) {
        v_reg = a.g.out_dst[base + lane];
#pragma unroll
        for (int h = 0; h < H; ++h) {
          const int64_t k = (int64_t)v_reg * H + h;
          const float ep = sddmm_add1(qs[h], scS.s, a.qD[k], scD.s);
          ba[lane][h] = __fdiv_rn(exp_p(__fsub_rn(lrelu(ep, slope), a.m[k])), a.den[k]);
          be[lane][h] = ep;
          bp[lane][h] = a.P[k];
        }
      }
      __syncwarp();
      for (int i = 0; i < cnt; ++i) {
        const int v = __shfl_sync(0xffffffffu, v_reg, i);
        const Row<VPL> gw = load_row<VPL>(gbase + (int64_t)v * a.ldG);
        int dot = row_dot<VPL>(gw, hw);
#pragma unroll
        for (int o = 1; o < LPH; o <<= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
        if (left == 0) {
          cs.fold();
#pragma unroll
          for (int k = 0; k < VPL; ++k) { tot[k] = folded ? __fadd_rn(tot[k], part[k]) : part[k]; part[k] = 0.0f; }
          folded = true; left = chunk;
        }
        const float al = ba[i][myh];
        if (leader) {
          const float dal = __fmul_rn(__int2float_rn(dot), sGH);
          const float dE = __fmul_rn(al, __fsub_rn(dal, bp[i][myh]));
          const float dEp = be[i][myh] > 0.0f ? dE : __fmul_rn(dE, slope);
          cs.part = __fadd_rn(cs.part, dEp);
        }
#pragma unroll
        for (int k = 0; k < VPL; ++k) part[k] = __fmaf_rn(al, row_f<VPL>(gw, k), part[k]);
        --left;
      }
      __syncwarp();
    }
    const float dS_lead = cs.finish(deg);
    const float dS = __shfl_sync(0xffffffffu, dS_lead, myh * LPH);
    const float dD = a.dD[ug * H + myh];
    float outv[VPL];
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const float sum = deg == 0 ? 0.0f : (folded ? __fadd_rn(tot[k], part[k]) : part[k]);
      const float agg = __fmul_rn(sum, scG.s);
      const float t2 = __fadd_rn(agg, __fmul_rn(dS, asrc[k]));
      outv[k] = __fadd_rn(t2, __fmul_rn(dD, adst[k]));
      amax_loc = fmaxf(amax_loc, fabsf(outv[k]));
      const float hp = __fmul_rn(row_f<VPL>(hw, k), scH.s);
      das[k] = __fmaf_rn(dS, hp, das[k]);
      dad[k] = __fmaf_rn(dD, hp, dad[k]);
    }
    float* dst = a.dHp + ul * HD + lane * VPL;
    if constexpr (VPL % 4 == 0) {
#pragma unroll
      for (int k = 0; k < VPL; k += 4) *reinterpret_cast<float4*>(dst + k) = make_float4(outv[k], outv[k + 1], outv[k + 2], outv[k + 3]);
    } else {
#pragma unroll
      for (int k = 0; k < VPL; ++k) dst[k] = outv[k];
    }
  }
  // ∂a: block reduction in shared memory, then one global atomic per column per block (tolerance-checked)
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    atomicAdd(&sh_da[0][lane * VPL + k], das[k]);
    atomicAdd(&sh_da[1][lane * VPL + k], dad[k]);
  }
  amax_loc = warp_max(amax_loc);
  if (lane == 0) atomicMax(&sh_amax, __float_as_uint(amax_loc));
  __syncthreads();
  for (int j = threadIdx.x; j < HD; j += blockDim.x) {
    atomicAdd(a.da_src + j, sh_da[0][j]);
    atomicAdd(a.da_dst + j, sh_da[1][j]);
  }
  if (threadIdx.x == 0 && a.amax_dHp) atomicMax(a.amax_dHp, sh_amax);
}

// ------------------------------------------------------------------ dispatch of the fused kernels
static int rows_grid(int64_t rows) {
  int64_t g = (rows + 7) / 8;
  const int64_t cap = (int64_t)num_sms() * 16;
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

#define TANGO_DISPATCH_HV(H_, VPL_, KERNEL, ARGS, ST, N)                                      \
  switch (H_ * 100 + VPL_) {                                                                   \
    case 102: KERNEL<1, 2><<<rows_grid(N), 256, 0, ST>>>(ARGS); break;                        \
    case 104: KERNEL<1, 4><<<rows_grid(N), 256, 0, ST>>>(ARGS); break;                        \
    case 108: KERNEL<1, 8><<<rows_grid(N), 256, 0, ST>>>(ARGS); break;                        \
    case 116: KERNEL<1, 16><<<rows_grid(N), 256, 0, ST>>>(ARGS); break;                       \
    case 202: KERNEL<2, 2><<<rows_grid(N), 256, 0, ST>>>(ARGS); break;                        \
    case 204: KERNEL<2, 4><<<rows_grid(N), 256, 0, ST>>>(ARGS); break;                        \
    case 208: KERNEL<2, 8><<<rows_grid(N), 256, 0, ST>>>(ARGS); break;                        \
    case 216: KERNEL<2, 16><<<rows_grid(N), 256, 0, ST>>>(ARGS); break;                       \
    case 402: KERNEL<4, 2><<<rows_grid(N), 256, 0, ST>>>(ARGS); break;                        \
    case 404: KERNEL<4, 4><<<rows_grid(N), 256, 0, ST>>>(ARGS); break;                        \
    case 408: KERNEL<4, 8><<<rows_grid(N), 256, 0, ST>>>(ARGS); break;                        \
    case 416: KERNEL<4, 16><<<rows_grid(N), 256, 0, ST>>>(ARGS); break;                       \
    case 802: KERNEL<8, 2><<<rows_grid(N), 256, 0, ST>>>(ARGS); break;                        \
    case 804: KERNEL<8, 4><<<rows_grid(N), 256, 0, ST>>>(ARGS); break;                        \
    case 808: KERNEL<8, 8><<<rows_grid(N), 256, 0, ST>>>(ARGS); break;                        \
    case 816: KERNEL<8, 16><<<rows_grid(N), 256, 0, ST>>>(ARGS); break;                       \
    default: return cudaErrorInvalidValue;                                                    \
  }

cudaError_t launch_gat_fwd_dst(const GatFwdDstArgs& a, cudaStream_t st) {
  if (a.g.n_local == 0) return cudaSuccess;
  ProfScope ps("gat_fwd_dst", st);
  TANGO_DISPATCH_HV(a.d.heads, a.d.hd / 32, k_gat_fwd_dst, a, st, a.g.n_local);
  return cudaGetLastError();
}
cudaError_t launch_gat_bwd_dst(const GatBwdDstArgs& a, cudaStream_t st) {
  if (a.g.n_local == 0) return cudaSuccess;
  ProfScope ps("gat_bwd_dst", st);
  TANGO_DISPATCH_HV(a.d.heads, a.d.hd / 32, k_gat_bwd_dst, a, st, a.g.n_local);
  return cudaGetLastError();
}
cudaError_t launch_gat_bwd_src(const GatBwdSrcArgs& a, cudaStream_t st) {
  if (a.g.n_local == 0) return cudaSuccess;
  ProfScope ps("gat_bwd_src", st);
  TANGO_DISPATCH_HV(a.d.heads, a.d.hd / 32, k_gat_bwd_src, a, st, a.g.n_local);
  return cudaGetLastError();
}

// ================================================================== unfused primitives
// One thread per (row, head) or (row, column), sequential over the row's edges in canonical order:
// the same arithmetic as the fused kernels, laid out for clarity rather than speed.

__global__ void k_sddmm_add(GraphDev g, int heads, const int8_t* qS, const float* sS, const int8_t* qD,
                            const float* sD, float slope, float* e_pre, float* el) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (tid >= g.n_local * heads) return;
  const int64_t vl = tid / heads;
  const int h = (int)(tid % heads);
  const int64_t vg = g.row_begin + vl;
  const float s1 = *sS, s2 = *sD;
  for (int64_t e = g.in_ptr[vl]; e < g.in_ptr[vl + 1]; ++e) {
    const int64_t u = g.in_src[e];
    const float x = sddmm_add1(qS[u * heads + h], s1, qD[vg * heads + h], s2);
    if (e_pre) e_pre[e * heads + h] = x;
    if (el) el[e * heads + h] = lrelu(x, slope);
  }
}

__global__ void k_sddmm_dot(GraphDev g, int heads, int hd_total, const int8_t* qA, int64_t lda, const float* sA,
                            const int8_t* qB, int64_t ldb, const float* sB, float* out, int32_t* acc_out) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (tid >= g.n_local * heads) return;
  const int64_t vl = tid / heads;
  const int h = (int)(tid % heads);
  const int64_t vg = g.row_begin + vl;
  const int D = hd_total / heads;
  const float s = __fmul_rn(*sA, *sB);
  for (int64_t e = g.in_ptr[vl]; e < g.in_ptr[vl + 1]; ++e) {
    const int64_t u = g.in_src[e];
    int acc = 0;
    for (int d = 0; d < D; ++d) acc += (int)qA[vg * lda + h * D + d] * (int)qB[u * ldb + h * D + d];
    if (out) out[e * heads + h] = __fmul_rn(__int2float_rn(acc), s);
    if (acc_out) acc_out[e * heads + h] = acc;
  }
}

__global__ void k_edge_softmax(GraphDev g, int heads, const float* el, float* m, float* den, float* alpha) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (tid >= g.n_local * heads) return;
  const int64_t vl = tid / heads;
  const int h = (int)(tid % heads);
  const int64_t b = g.in_ptr[vl], e1 = g.in_ptr[vl + 1], len = e1 - b;
  float mx = -INFINITY;
  for (int64_t e = b; e < e1; ++e) mx = fmaxf(mx, el[e * heads + h]);
  if (len == 0) mx = 0.0f;
  CSum cs; cs.init();
  int left = g.chunk;
  for (int64_t e = b; e < e1; ++e) {
    if (left == 0) { cs.fold(); left = g.chunk; }
    cs.part = __fadd_rn(cs.part, exp_p(__fsub_rn(el[e * heads + h], mx)));
    --left;
  }
  const float dn = cs.finish(len);
  for (int64_t e = b; e < e1; ++e) alpha[e * heads + h] = __fdiv_rn(exp_p(__fsub_rn(el[e * heads + h], mx)), dn);
  if (m) m[(g.row_begin + vl) * heads + h] = mx;
  if (den) den[(g.row_begin + vl) * heads + h] = dn;
}

__global__ void k_softmax_bwd(GraphDev g, int heads, const float* alpha, const float* dalpha, const float* e_pre,
                              float slope, float* P, float* dEp) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (tid >= g.n_local * heads) return;
  const int64_t vl = tid / heads;
  const int h = (int)(tid % heads);
  const int64_t b = g.in_ptr[vl], e1 = g.in_ptr[vl + 1];
  CSum cs; cs.init();
  int left = g.chunk;
  for (int64_t e = b; e < e1; ++e) {
    if (left == 0) { cs.fold(); left = g.chunk; }
    cs.part = __fmaf_rn(dalpha[e * heads + h], alpha[e * heads + h], cs.part);
    --left;
  }
  const float p = cs.finish(e1 - b);
  if (P) P[(g.row_begin + vl) * heads + h] = p;
  for (int64_t e = b; e < e1; ++e) {
    const float dE = __fmul_rn(alpha[e * heads + h], __fsub_rn(dalpha[e * heads + h], p));
    dEp[e * heads + h] = e_pre[e * heads + h] > 0.0f ? dE : __fmul_rn(dE, slope);
  }
}

__global__ void k_edge_sum(GraphDev g, int dir, int heads, const float* x, float* out) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (tid >= g.n_local * heads) return;
  const int64_t vl = tid / heads;
  const int h = (int)(tid % heads);
  const int64_t* ptr = dir ? g.out_ptr : g.in_ptr;
  const int64_t b = ptr[vl], e1 = ptr[vl + 1];
  CSum cs; cs.init();
  int left = g.chunk;
  for (int64_t p = b; p < e1; ++p) {
    const int64_t eid = dir ? (int64_t)g.out_eid[p] : p;
    if (left == 0) { cs.fold(); left = g.chunk; }
    cs.part = __fadd_rn(cs.part, x[eid * heads + h]);
    --left;
  }
  out[vl * heads + h] = cs.finish(e1 - b);
}

__global__ void k_spmm_w(GraphDev g, int dir, int heads, int cols, const float* w, const int8_t* qX, int64_t ldx,
                         const float* sX, float* out) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (tid >= g.n_local * cols) return;
  const int64_t vl = tid / cols;
  const int j = (int)(tid % cols);
  const int h = j / (cols / heads);
  const int64_t* ptr = dir ? g.out_ptr : g.in_ptr;
  const int64_t b = ptr[vl], e1 = ptr[vl + 1];
  CSum cs; cs.init();
  int left = g.chunk;
  for (int64_t p = b; p < e1; ++p) {
    const int64_t eid = dir ? (int64_t)g.out_eid[p] : p;
    const int64_t other = dir ? (int64_t)g.out_dst[p] : (int64_t)g.in_src[p];
    if (left == 0) { cs.fold(); left = g.chunk; }
    cs.part = __fmaf_rn(w[eid * heads + h], i8f(qX[other * ldx + j]), cs.part);
    --left;
  }
  out[vl * cols + j] = __fmul_rn(cs.finish(e1 - b), *sX);
}

// Unweighted int32 SPMM (GCN; exact, order-free).  Warp per row, lanes over columns (coalesced rows).
// out = ((float)sum * s_X) * rowscale[row] (optional), amax over |out| (optional).
__global__ void __launch_bounds__(256) k_spmm_sum(GraphDev g, int dir, int cols, const int8_t* qX, int64_t ldx,
                                                  const float* sX, const float* rowscale, float* out,
                                                  int32_t* out_i32, unsigned* amax_out) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float s = sX ? *sX : 1.0f;
  float amax_loc = 0.0f;
  for (int64_t vl = (int64_t)blockIdx.x * 8 + w; vl < g.n_local; vl += (int64_t)gridDim.x * 8) {
    const int64_t* ptr = dir ? g.out_ptr : g.in_ptr;
    const int32_t* nbr = dir ? g.out_dst : g.in_src;
    const int64_t b = ptr[vl], e1 = ptr[vl + 1];
    const float rs = rowscale ? rowscale[vl] : 1.0f;
    for (int j0 = 0; j0 < cols; j0 += 32) {
      const int j = j0 + lane;
      int acc = 0;
      if (j < cols)
        for (int64_t p = b; p < e1; ++p) acc += (int)qX[(int64_t)nbr[p] * ldx + j];
      if (j < cols) {
        if (out_i32) out_i32[vl * cols + j] = acc;
        if (out) {
          float v = __fmul_rn(__int2float_rn(acc), s);
          if (rowscale) v = __fmul_rn(v, rs);
          out[vl * cols + j] = v;
          amax_loc = fmaxf(amax_loc, fabsf(v));
        }
      }
    }
  }
  if (amax_out) {
    amax_loc = warp_max(amax_loc);
    if (lane == 0) atomicMax(amax_out, __float_as_uint(amax_loc));
  }
}

// GCN normalisation (reading R26): ns = 1/sqrt(out_deg), nd = 1/sqrt(in_deg); 0 for degree 0.
__global__ void k_gcn_norms(GraphDev g, float* ns, float* nd) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= g.n_local) return;
  const int64_t di = g.in_ptr[i + 1] - g.in_ptr[i];
  const int64_t dout = g.out_ptr[i + 1] - g.out_ptr[i];
  nd[i] = di > 0 ? __fdiv_rn(1.0f, __fsqrt_rn((float)di)) : 0.0f;
  ns[i] = dout > 0 ? __fdiv_rn(1.0f, __fsqrt_rn((float)dout)) : 0.0f;
}

static int flat_grid(int64_t n) {
  int64_t g = (n + 255) / 256;
  return (int)(g < 1 ? 1 : g);
}

cudaError_t launch_sddmm_add(const GraphDev& g, int heads, const int8_t* qS, const float* sS, const int8_t* qD,
                             const float* sD, float slope, float* e_pre, float* el, cudaStream_t st) {
  if (g.n_local == 0) return cudaSuccess;
  ProfScope ps("sddmm_add", st);
  k_sddmm_add<<<flat_grid(g.n_local * heads), 256, 0, st>>>(g, heads, qS, sS, qD, sD, slope, e_pre, el);
  return cudaGetLastError();
}
cudaError_t launch_sddmm_dot(const GraphDev& g, int heads, int hd_total, const int8_t* qA, int64_t lda,
                             const float* sA, const int8_t* qB, int64_t ldb, const float* sB, float* out,
                             int32_t* acc, cudaStream_t st) {
  if (g.n_local == 0) return cudaSuccess;
  ProfScope ps("sddmm_dot", st);
  k_sddmm_dot<<<flat_grid(g.n_local * heads), 256, 0, st>>>(g, heads, hd_total, qA, lda, sA, qB, ldb, sB, out, acc);
  return cudaGetLastError();
}
cudaError_t launch_edge_softmax(const GraphDev& g, int heads, const float* el, float* m, float* den, float* alpha,
                                cudaStream_t st) {
  if (g.n_local == 0) return cudaSuccess;
  ProfScope ps("edge_softmax", st);
  k_edge_softmax<<<flat_grid(g.n_local * heads), 256, 0, st>>>(g, heads, el, m, den, alpha);
  return cudaGetLastError();
}
cudaError_t launch_softmax_bwd(const GraphDev& g, int heads, const float* alpha, const float* dalpha,
                               const float* e_pre, float slope, float* P, float* dEp, cudaStream_t st) {
  if (g.n_local == 0) return cudaSuccess;
  ProfScope ps("softmax_bwd", st);
  k_softmax_bwd<<<flat_grid(g.n_local * heads), 256, 0, st>>>(g, heads, alpha, dalpha, e_pre, slope, P, dEp);
  return cudaGetLastError();
}
cudaError_t launch_edge_sum(const GraphDev& g, int dir, int heads, const float* x, float* out, cudaStream_t st) {
  if (g.n_local == 0) return cudaSuccess;
  ProfScope ps("edge_sum", st);
  k_edge_sum<<<flat_grid(g.n_local * heads), 256, 0, st>>>(g, dir, heads, x, out);
  return cudaGetLastError();
}
cudaError_t launch_spmm_w(const GraphDev& g, int dir, int heads, int cols, const float* w, const int8_t* qX,
                          int64_t ldx, const float* sX, float* out, cudaStream_t st) {
  if (g.n_local == 0) return cudaSuccess;
  ProfScope ps("spmm_w", st);
  k_spmm_w<<<flat_grid(g.n_local * cols), 256, 0, st>>>(g, dir, heads, cols, w, qX, ldx, sX, out);
  return cudaGetLastError();
}
cudaError_t launch_spmm_sum(const GraphDev& g, int dir, int cols, const int8_t* qX, int64_t ldx, const float* sX,
                            const float* rowscale, float* out, int32_t* out_i32, unsigned* amax_out,
                            cudaStream_t st) {
  if (g.n_local == 0) return cudaSuccess;
  ProfScope ps("spmm_sum", st);
  k_spmm_sum<<<rows_grid(g.n_local), 256, 0, st>>>(g, dir, cols, qX, ldx, sX, rowscale, out, out_i32, amax_out);
  return cudaGetLastError();
}
cudaError_t launch_gcn_norms(const GraphDev& g, float* ns, float* nd, cudaStream_t st) {
  if (g.n_local == 0) return cudaSuccess;
  ProfScope ps("gcn_norms", st);
  k_gcn_norms<<<flat_grid(g.n_local), 256, 0, st>>>(g, ns, nd);
  return cudaGetLastError();
}

}  // namespace tango
