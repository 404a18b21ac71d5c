// prims.cu — the unfused sparse primitives of the C ABI (tango_sddmm_q, tango_edge_softmax,
// tango_softmax_bwd, tango_edge_sum, tango_spmm_q) and the GCN helpers.  tango_edge_sum (the paper's
// incidence SPMM, Table 2), tango_spmm_q and tango_spmm_q8 are row-block kernels with chunk items; the others run one
// thread per (row, head) or (row, column), sequential over the row's edges in canonical order: the
// same arithmetic as the fused kernels of gat.cu / gat2.cu, laid out for clarity rather than speed.
// Paper: ③ P:204-209, ④ P:212-217, ⑤/⑤′ P:224-251, ⑤″ P:252-255, ④′ P:258-264,
// ③′/③″ P:276 and P:821-832, GCN P:347-348.
#include "gat_common.cuh"

namespace tango {
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

// ---------------------------------------------------------------------------- incidence SPMM (③′ / ③″)
// out[v,h] = Σᶜ x[e,h] over v's in-edges (dir 0, contiguous in-CSR edge records: a streaming read) or
// out-edges (dir 1, records out_eid[p]: a gather of F-float rows), reading R14.
// Row blocks: block b owns rows [256·b, 256·b + 256) (no plan, no search); its rows are cut into canonical
// chunks ("items", ≤ C_E edges), so a hub row's chunks are spread over the block's 8 warps.  A
// group of GW = ceil(F / VW) lanes sums one item sequentially, each lane VW consecutive columns (float4 /
// float2 / float loads), so a group's load of one edge record is one contiguous 4F-byte run; 16 floats
// per lane are in flight (16 / VW records) and the blocks run at 4 per SM (32 warps).  A
// row with one chunk is written directly, a hub row's chunk partials go to shared memory and are folded
// left to right (total = p_0, total += p_c) after a barrier.  Rows are taken in batches of at most
// ES_ROWS rows and es_slots(F) items; a row with more chunks than one batch holds is folded window by
// window (running totals in shared memory — the same left-to-right order).
constexpr int ES_THREADS = 256, ES_ROWS = 256;

__host__ __device__ inline int es_slots(int F) {
  const int s = 4096 / F;
  return s > 1024 ? 1024 : (s < 8 ? 8 : s);
}

template <int VW> struct VecF;
template <> struct VecF<1> { using T = float; };
template <> struct VecF<2> { using T = float2; };
template <> struct VecF<4> { using T = float4; };
template <int VW>
__device__ __forceinline__ void vadd(float (&acc)[VW], const typename VecF<VW>::T& v) {
  if constexpr (VW == 1) {
    acc[0] = __fadd_rn(acc[0], v);
  } else if constexpr (VW == 2) {
    acc[0] = __fadd_rn(acc[0], v.x); acc[1] = __fadd_rn(acc[1], v.y);
  } else {
    acc[0] = __fadd_rn(acc[0], v.x); acc[1] = __fadd_rn(acc[1], v.y);
    acc[2] = __fadd_rn(acc[2], v.z); acc[3] = __fadd_rn(acc[3], v.w);
  }
}

template <int DIR, int VW>
__global__ void __launch_bounds__(ES_THREADS, 2) k_edge_sum_w(GraphDev g, int F, int64_t epb, int64_t E,
                                                          const float* __restrict__ x, float* __restrict__ out) {
  using V = typename VecF<VW>::T;
  extern __shared__ __align__(16) float es_part[];               // [slots + 1][F]
  __shared__ int s_pre[ES_ROWS];                                 // inclusive prefix of chunk counts (items)
  __shared__ int s_slot[ES_ROWS];                                // inclusive prefix of partial slots
  const int64_t* __restrict__ ptr = DIR ? g.out_ptr : g.in_ptr;
  const int32_t* __restrict__ eid = g.out_eid;
  const int64_t n = g.n_local, C = g.chunk;
  const int slots = es_slots(F);
  (void)epb; (void)E;
  const int64_t r0 = (int64_t)blockIdx.x * ES_ROWS, r1 = r0 + ES_ROWS < n ? r0 + ES_ROWS : n;   // the block's rows
  const int nv = (F + VW - 1) / VW;                 // vectors per record
  const int GW = nv < 32 ? nv : 32, GPW = 32 / GW, ncb = (nv + 31) / 32;
  const int lane = threadIdx.x & 31, grp = (threadIdx.x >> 5) * GPW + lane / GW, gl = lane % GW;
  const bool lane_ok = lane / GW < GPW;
  const int ngroups = (ES_THREADS / 32) * GPW;
  const V* __restrict__ xv = reinterpret_cast<const V*>(x);
  auto chunks = [&](int64_t r) -> int64_t {
    const int64_t d = ptr[r + 1] - ptr[r];
    return d <= C ? 1 : (d + C - 1) / C;
  };
  // sequential sum of list positions [pb, pe) (pe - pb <= C) for the lane's vector vi (columns VW·vi ..):
  // 32 floats per lane in flight (U = 32 / VW records; 2 blocks per SM at 128 registers), then added in order
  auto chunk_sum = [&](int64_t pb, int64_t pe, int vi, float (&acc)[VW]) {
    constexpr int U = 32 / VW;
#pragma unroll
    for (int k = 0; k < VW; ++k) acc[k] = 0.0f;
    for (int64_t p = pb; p < pe; p += U) {
      V v[U];
#pragma unroll
      for (int j = 0; j < U; ++j) {
        if (p + j < pe) {
          const int64_t e = DIR ? (int64_t)__ldg(eid + p + j) : p + j;
          v[j] = __ldg(xv + e * nv + vi);
        }
      }
#pragma unroll
      for (int j = 0; j < U; ++j)
        if (p + j < pe) vadd<VW>(acc, v[j]);
    }
  };
  auto put = [&](float* dst, int vi, const float (&acc)[VW]) {   // columns VW·vi .. of one row (F floats)
#pragma unroll
    for (int k = 0; k < VW; ++k)
      if (vi * VW + k < F) dst[vi * VW + k] = acc[k];
  };
  int64_t row = r0;
  while (row < r1) {
    const int64_t rr = row + threadIdx.x;
    const int64_t c = (threadIdx.x < ES_ROWS && rr < r1) ? chunks(rr) : 0;
    // two prefixes over the batch's rows: items (chunks of every row) and partial slots (chunks of the
    // multi-chunk rows only: a single-chunk row writes its output directly and needs no slot)
    int v = (int)(c < (1 << 20) ? c : (1 << 20));
    int ws = c > 1 ? (int)(c > slots ? slots + 1 : c) : 0;
    s_pre[threadIdx.x] = v;
    s_slot[threadIdx.x] = ws;
    __syncthreads();
    for (int off = 1; off < ES_ROWS; off <<= 1) {
      const int add = threadIdx.x >= off ? s_pre[threadIdx.x - off] : 0;
      const int adw = threadIdx.x >= off ? s_slot[threadIdx.x - off] : 0;
      __syncthreads();
      v += add;
      ws += adw;
      s_pre[threadIdx.x] = v;
      s_slot[threadIdx.x] = ws;
      __syncthreads();
    }
    // rows of the batch: the slot prefix is non-decreasing, so the cut is a count
    const int nb = __syncthreads_count(rr < r1 && ws <= slots);
    if (nb == 0) {
      // one row with more chunks than a batch: windows of `slots` chunks, folded in order
      const int64_t pb0 = ptr[row], pe0 = ptr[row + 1], nch = (pe0 - pb0 + C - 1) / C;
      float* tot = es_part + (int64_t)slots * F;   // running totals of the row [F]
      for (int64_t w0 = 0; w0 < nch; w0 += slots) {
        const int wn = (int)(nch - w0 < slots ? nch - w0 : slots);
        for (int u = grp; u < wn * ncb; u += ngroups) {
          const int it = u / ncb, vi = (u % ncb) * 32 + gl;
          if (!lane_ok || vi >= nv) continue;
          const int64_t pb = pb0 + (w0 + it) * C, pe = pb + C < pe0 ? pb + C : pe0;
          float acc[VW];
          chunk_sum(pb, pe, vi, acc);
          put(es_part + it * F, vi, acc);
        }
        __syncthreads();
        for (int h = threadIdx.x; h < F; h += ES_THREADS) {
          float t = w0 == 0 ? es_part[h] : __fadd_rn(tot[h], es_part[h]);
          for (int it = 1; it < wn; ++it) t = __fadd_rn(t, es_part[it * F + h]);
          tot[h] = t;
          if (w0 + wn == nch) out[row * F + h] = t;
        }
        __syncthreads();
      }
      row += 1;
      continue;
    }
    const int nitems = s_pre[nb - 1];
    for (int u = grp; u < nitems * ncb; u += ngroups) {
      const int it = u / ncb, vi = (u % ncb) * 32 + gl;
      int a = 0, b = nb - 1;   // first j with s_pre[j] > it
      while (a < b) {
        const int m = (a + b) >> 1;
        if (s_pre[m] > it) b = m; else a = m + 1;
      }
      const int j = a, k = it - (j ? s_pre[j - 1] : 0);
      const int64_t r = row + j, pb0 = ptr[r], pe0 = ptr[r + 1];
      const int64_t pb = pb0 + (int64_t)k * C, pe = pb + C < pe0 ? pb + C : pe0;
      if (!lane_ok || vi >= nv) continue;
      float acc[VW];
      chunk_sum(pb, pe, vi, acc);
      const int slot = (j ? s_slot[j - 1] : 0) + k;
      put(pe0 - pb0 <= C ? out + r * F : es_part + slot * F, vi, acc);   // single-chunk row: direct
    }
    __syncthreads();
    // fold the multi-chunk rows of the batch
    for (int t = threadIdx.x; t < nb * F; t += ES_THREADS) {
      const int j = t / F, h = t % F;
      const int i0 = j ? s_slot[j - 1] : 0, i1 = s_slot[j];
      if (i1 - i0 < 2) continue;
      float tot = es_part[i0 * F + h];
      for (int it = i0 + 1; it < i1; ++it) tot = __fadd_rn(tot, es_part[it * F + h]);
      out[(row + j) * F + h] = tot;
    }
    __syncthreads();
    row += nb;
  }
}

// ---------------------------------------------------------------------------- weighted SPMM ⑤ / ⑤′
// out[v,j] = ((Σᶜ fmaf(w[e,h(j)], i2f(q_X[u_e,j]))) · s_X) [· row_scale[v]] over v's in-edges (dir 0, u_e =
// source) or out-edges (dir 1, u_e = destination, weight w[out_eid[p]]), R14.  The
// same row blocks and chunk items as tango_edge_sum; a WARP sums one (item, 32·V-column pass): per 32-edge
// batch the lanes load the batch's gather rows and weights in parallel into per-warp shared memory, then
// every lane streams its V columns (V = 16: one 16-B load, 4: one word, 1: bytes) of each gathered row, 8
// rows in flight, with the exact int8 -> fp32 conversion (PRMT + FADD2) and packed FFMA2 in edge order
// (bit-identical to fmaf).  Multi-chunk rows fold their chunk partials left to right after a barrier.
template <int V>
__host__ __device__ constexpr int sw_cols() { return 32 * V; }
template <int V>
__host__ __device__ constexpr int sw_slots() { return V == 16 ? 16 : 64; }

template <int DIR, int V>
__global__ void __launch_bounds__(ES_THREADS) k_spmm_w_fast(GraphDev g, int heads, int cols, int64_t epb, int64_t E,
                                                           const float* __restrict__ w, const int8_t* __restrict__ qX,
                                                           int64_t ldx, const float* __restrict__ sX,
                                                           const float* __restrict__ rowscale, float* __restrict__ out,
                                                           unsigned* amax_out) {
  extern __shared__ __align__(16) float sw_dyn[];
  constexpr int SW_COLS = sw_cols<V>();
  float* part = sw_dyn;                                            // [slots][SW_COLS]
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int* su = reinterpret_cast<int*>(part + (sw_slots<V>() + 1) * SW_COLS) + wid * 32 * (1 + heads);   // [32] rows
  float* swt = reinterpret_cast<float*>(su + 32);                                           // [32][heads]
  __shared__ int s_pre[ES_ROWS];    // inclusive prefix of chunk counts (items)
  __shared__ int s_slot[ES_ROWS];   // inclusive prefix of partial slots (multi-chunk rows)
  const int64_t* __restrict__ ptr = DIR ? g.out_ptr : g.in_ptr;
  const int32_t* __restrict__ nbr = DIR ? g.out_dst : g.in_src;
  const int64_t n = g.n_local, C = g.chunk;
  const int slots = sw_slots<V>();
  const int D = cols / heads, npass = (cols + SW_COLS - 1) / SW_COLS;
  const float s = *sX;
  float amax_loc = 0.0f;
  (void)epb; (void)E;
  const int64_t r0 = (int64_t)blockIdx.x * ES_ROWS, r1 = r0 + ES_ROWS < n ? r0 + ES_ROWS : n;   // the block's rows
  auto chunks = [&](int64_t r) -> int64_t {
    const int64_t d = ptr[r + 1] - ptr[r];
    return d <= C ? 1 : (d + C - 1) / C;
  };
  auto finish = [&](int64_t r, int j, float acc) {   // (Σᶜ)·s_X [· row_scale] -> out, amax
    float v = __fmul_rn(acc, s);
    if (rowscale) v = __fmul_rn(v, rowscale[r]);
    out[r * cols + j] = v;
    amax_loc = fmaxf(amax_loc, fabsf(v));
  };
  // chunk sum of list positions [pb, pe) for the lane's columns j0 .. j0+V-1 of pass cp -> acc[V]
  auto chunk_sum = [&](int64_t pb, int64_t pe, int j0, float (&acc)[V]) {
#pragma unroll
    for (int c = 0; c < V; ++c) acc[c] = 0.0f;
    int hc[V];
#pragma unroll
    for (int c = 0; c < V; ++c) hc[c] = (j0 + c < cols) ? (j0 + c) / D : 0;
    for (int64_t b0 = pb; b0 < pe; b0 += 32) {
      const int nb = (int)(pe - b0 < 32 ? pe - b0 : 32);
      __syncwarp();
      if (lane < nb) {
        const int64_t p = b0 + lane;
        const int64_t e = DIR ? (int64_t)g.out_eid[p] : p;
        su[lane] = nbr[p];
        for (int h = 0; h < heads; ++h) swt[lane * heads + h] = w[e * heads + h];
      }
      __syncwarp();
      for (int i0 = 0; i0 < nb; i0 += 8) {
        uint32_t word[8][(V + 3) / 4];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
#pragma unroll
          for (int k = 0; k < (V + 3) / 4; ++k) word[i][k] = 0u;
          if (i0 + i < nb) {
            const int8_t* row = qX + (int64_t)su[i0 + i] * ldx;
            if constexpr (V == 16) {
              if (j0 < cols) {
                const uint4 x = __ldg(reinterpret_cast<const uint4*>(row + j0));
                word[i][0] = x.x; word[i][1] = x.y; word[i][2] = x.z; word[i][3] = x.w;
              }
            } else if constexpr (V == 4) {
              if (j0 < cols) word[i][0] = __ldg(reinterpret_cast<const unsigned*>(row + j0));
            } else {
              if (j0 < cols) word[i][0] = (uint32_t)(uint8_t)__ldg(row + j0);
            }
          }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (i0 + i < nb) {
            const float* wr = swt + (i0 + i) * heads;
            if constexpr (V >= 4) {   // D % 4 == 0: a word's 4 columns share one head
#pragma unroll
              for (int k = 0; k < V / 4; ++k) {
                const float wk = wr[hc[4 * k]];
                float2 a01 = make_float2(acc[4 * k], acc[4 * k + 1]), a23 = make_float2(acc[4 * k + 2], acc[4 * k + 3]);
                fma4_codes(word[i][k], make_float2(wk, wk), a01, a23);
                acc[4 * k] = a01.x; acc[4 * k + 1] = a01.y; acc[4 * k + 2] = a23.x; acc[4 * k + 3] = a23.y;
              }
            } else {
              acc[0] = __fmaf_rn(wr[hc[0]], __int2float_rn((int)(int8_t)word[i][0]), acc[0]);
            }
          }
        }
      }
    }
  };
  int64_t row = r0;
  while (row < r1) {
    const int64_t rr = row + threadIdx.x;
    const int64_t c = (threadIdx.x < ES_ROWS && rr < r1) ? chunks(rr) : 0;
    // items of every row, partial slots of the multi-chunk rows only (as in tango_edge_sum)
    int v = (int)(c < (1 << 20) ? c : (1 << 20));
    int ws = c > 1 ? (int)(c > slots ? slots + 1 : c) : 0;
    s_pre[threadIdx.x] = v;
    s_slot[threadIdx.x] = ws;
    __syncthreads();
    for (int off = 1; off < ES_ROWS; off <<= 1) {
      const int add = threadIdx.x >= off ? s_pre[threadIdx.x - off] : 0;
      const int adw = threadIdx.x >= off ? s_slot[threadIdx.x - off] : 0;
      __syncthreads();
      v += add;
      ws += adw;
      s_pre[threadIdx.x] = v;
      s_slot[threadIdx.x] = ws;
      __syncthreads();
    }
    const int nb = __syncthreads_count(rr < r1 && ws <= slots);
    if (nb == 0) {   // one row with more chunks than the partial slots: windows, folded in order
      const int64_t pb0 = ptr[row], pe0 = ptr[row + 1], nch = (pe0 - pb0 + C - 1) / C;
      float* wtot = part + (int64_t)slots * SW_COLS;   // running totals of the pass's columns
      for (int cp = 0; cp < npass; ++cp) {
        for (int64_t w0 = 0; w0 < nch; w0 += slots) {
          const int wn = (int)(nch - w0 < slots ? nch - w0 : slots);
          for (int it = wid; it < wn; it += ES_THREADS / 32) {
            const int64_t pb = pb0 + (w0 + it) * C, pe = pb + C < pe0 ? pb + C : pe0;
            float acc[V];
            chunk_sum(pb, pe, cp * SW_COLS + lane * V, acc);
#pragma unroll
            for (int q = 0; q < V; ++q) part[it * SW_COLS + lane * V + q] = acc[q];
          }
          __syncthreads();
          for (int t = threadIdx.x; t < SW_COLS; t += ES_THREADS) {
            float tot = w0 == 0 ? part[t] : __fadd_rn(wtot[t], part[t]);
            for (int it = 1; it < wn; ++it) tot = __fadd_rn(tot, part[it * SW_COLS + t]);
            wtot[t] = tot;
          }
          __syncthreads();
        }
        for (int t = threadIdx.x; t < SW_COLS; t += ES_THREADS)
          if (cp * SW_COLS + t < cols) finish(row, cp * SW_COLS + t, wtot[t]);
        __syncthreads();
      }
      row += 1;
      continue;
    }
    const int nitems = s_pre[nb - 1];
    for (int cp = 0; cp < npass; ++cp) {
      for (int it = wid; it < nitems; it += ES_THREADS / 32) {
        int a = 0, b = nb - 1;
        while (a < b) {
          const int m = (a + b) >> 1;
          if (s_pre[m] > it) b = m; else a = m + 1;
        }
        const int j = a, k = it - (j ? s_pre[j - 1] : 0);
        const int64_t r = row + j, pb0 = ptr[r], pe0 = ptr[r + 1];
        const int64_t pb = pb0 + (int64_t)k * C, pe = pb + C < pe0 ? pb + C : pe0;
        const int j0 = cp * SW_COLS + lane * V;
        float acc[V];
        chunk_sum(pb, pe, j0, acc);
        if (pe0 - pb0 <= C) {
#pragma unroll
          for (int q = 0; q < V; ++q)
            if (j0 + q < cols) finish(r, j0 + q, acc[q]);
        } else {
          const int slot = (j ? s_slot[j - 1] : 0) + k;
#pragma unroll
          for (int q = 0; q < V; ++q) part[slot * SW_COLS + lane * V + q] = acc[q];
        }
      }
      __syncthreads();
      for (int t = threadIdx.x; t < nb * SW_COLS; t += ES_THREADS) {
        const int jr = t / SW_COLS, col = cp * SW_COLS + t % SW_COLS;
        const int i0 = jr ? s_slot[jr - 1] : 0, i1 = s_slot[jr];
        if (i1 - i0 < 2 || col >= cols) continue;
        float tot = part[i0 * SW_COLS + t % SW_COLS];
        for (int it = i0 + 1; it < i1; ++it) tot = __fadd_rn(tot, part[it * SW_COLS + t % SW_COLS]);
        finish(row + jr, col, tot);
      }
      __syncthreads();
    }
    row += nb;
  }
  if (amax_out) {
    amax_loc = warp_max(amax_loc);
    if (lane == 0) atomicMax(amax_out, __float_as_uint(amax_loc));
  }
}

// ---------------------------------------------------------------------------- int8-α SPMM (NEXT-4)
// acc[v,j] = Σ q_α[e,h(j)]·q_X[w_e,j] (exact int32, order-free), out = i2f(acc)·fl(s_α·s_X) (orc_spmm_q8).
// The same row blocks and chunk items as tango_spmm_q; a warp sums one (item, 128-column pass): per
// 32-edge batch the lanes stage the batch's gather rows and α codes ([head][edge] bytes) in shared memory;
// every lane then takes its 4 columns (one 32-bit word) of 4 gathered rows at a time, transposes the 4x4
// bytes (8 PRMT) and adds 4 IDP4A dots against the 4 edges' α codes of its head — 16 products in 12
// instructions instead of the fp32 path's 2 per product.  Integer sums are order-free, so a multi-chunk row
// adds its chunks with int32 atomics (out_i32 zeroed first); a second pass writes the fp32 output.
constexpr int Q8_COLS = 128;   // 4 columns per lane

__device__ __forceinline__ void transpose4(uint32_t r0, uint32_t r1, uint32_t r2, uint32_t r3, uint32_t (&t)[4]) {
  const uint32_t a = __byte_perm(r0, r1, 0x5140), b = __byte_perm(r2, r3, 0x5140);
  const uint32_t c = __byte_perm(r0, r1, 0x7362), d = __byte_perm(r2, r3, 0x7362);
  t[0] = __byte_perm(a, b, 0x5410); t[1] = __byte_perm(a, b, 0x7632);
  t[2] = __byte_perm(c, d, 0x5410); t[3] = __byte_perm(c, d, 0x7632);
}

template <int DIR>
__global__ void __launch_bounds__(ES_THREADS) k_spmm_q8(GraphDev g, int heads, int cols, int64_t epb, int64_t E,
                                                       const int8_t* __restrict__ qa, const int8_t* __restrict__ qX,
                                                       int64_t ldx, int32_t* __restrict__ out_i32) {
  extern __shared__ __align__(16) uint8_t q8_dyn[];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int* su = reinterpret_cast<int*>(q8_dyn) + wid * 32;                                    // [32] rows
  uint8_t* sa = q8_dyn + (ES_THREADS / 32) * 32 * 4 + wid * 32 * heads;                  // [heads][32]
  __shared__ int s_pre[ES_ROWS];
  const int64_t* __restrict__ ptr = DIR ? g.out_ptr : g.in_ptr;
  const int32_t* __restrict__ nbr = DIR ? g.out_dst : g.in_src;
  const int64_t n = g.n_local, C = g.chunk;
  const int D = cols / heads, npass = (cols + Q8_COLS - 1) / Q8_COLS;
  (void)epb; (void)E;
  const int64_t r0 = (int64_t)blockIdx.x * ES_ROWS, r1 = r0 + ES_ROWS < n ? r0 + ES_ROWS : n;   // the block's rows
  auto chunks = [&](int64_t r) -> int64_t {
    const int64_t d = ptr[r + 1] - ptr[r];
    return d <= C ? 1 : (d + C - 1) / C;
  };
  // integer dot sums of list positions [pb, pe) for the lane's 4 columns j0 .. j0+3 (one head: D % 4 == 0)
  auto chunk_dot = [&](int64_t pb, int64_t pe, int j0, int (&acc)[4]) {
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[c] = 0;
    const int h = j0 < cols ? j0 / D : 0;
    for (int64_t b0 = pb; b0 < pe; b0 += 32) {
      const int nb = (int)(pe - b0 < 32 ? pe - b0 : 32);
      __syncwarp();
      {
        const int64_t p = b0 + lane;
        const bool in = lane < nb;
        const int64_t e = in ? (DIR ? (int64_t)g.out_eid[p] : p) : 0;
        su[lane] = in ? nbr[p] : 0;
        for (int k = 0; k < heads; ++k) sa[k * 32 + lane] = in ? (uint8_t)qa[e * heads + k] : 0;   // pad: α code 0
      }
      __syncwarp();
      for (int i0 = 0; i0 < nb; i0 += 4) {
        uint32_t w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
          w[i] = j0 < cols ? __ldg(reinterpret_cast<const unsigned*>(qX + (int64_t)su[i0 + i] * ldx + j0)) : 0u;
        uint32_t t[4];
        transpose4(w[0], w[1], w[2], w[3], t);
        const int wa = *reinterpret_cast<const int*>(sa + h * 32 + i0);
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[c] = __dp4a((int)t[c], wa, acc[c]);
      }
    }
  };
  int64_t row = r0;
  while (row < r1) {
    const int64_t rr = row + threadIdx.x;
    // rows per batch: up to ES_ROWS, no item cap (multi-chunk rows add their chunks atomically)
    const int64_t c = (threadIdx.x < ES_ROWS && rr < r1) ? chunks(rr) : 0;
    int v = (int)(c > (1 << 20) ? (1 << 20) : c);
    s_pre[threadIdx.x] = v;
    __syncthreads();
    for (int off = 1; off < ES_ROWS; off <<= 1) {
      const int add = threadIdx.x >= off ? s_pre[threadIdx.x - off] : 0;
      __syncthreads();
      v += add;
      s_pre[threadIdx.x] = v;
      __syncthreads();
    }
    const int nb = (int)((r1 - row) < ES_ROWS ? (r1 - row) : ES_ROWS);
    const int nitems = s_pre[nb - 1];
    for (int cp = 0; cp < npass; ++cp) {
      for (int it = wid; it < nitems; it += ES_THREADS / 32) {
        int a = 0, b = nb - 1;
        while (a < b) {
          const int m = (a + b) >> 1;
          if (s_pre[m] > it) b = m; else a = m + 1;
        }
        const int j = a, k = it - (j ? s_pre[j - 1] : 0);
        const int64_t r = row + j, pb0 = ptr[r], pe0 = ptr[r + 1];
        const int64_t pb = pb0 + (int64_t)k * C, pe = pb + C < pe0 ? pb + C : pe0;
        const int j0 = cp * Q8_COLS + lane * 4;
        int acc[4];
        chunk_dot(pb, pe, j0, acc);
        if (j0 < cols) {
          if (pe0 - pb0 <= C) {
            *reinterpret_cast<int4*>(out_i32 + r * cols + j0) = make_int4(acc[0], acc[1], acc[2], acc[3]);
          } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) atomicAdd(out_i32 + r * cols + j0 + q, acc[q]);
          }
        }
      }
    }
    __syncthreads();
    row += nb;
  }
}

__global__ void k_i32_to_f32(const int32_t* __restrict__ acc, int64_t count, const float* sa, const float* sx,
                             float* __restrict__ out) {
  const float s = __fmul_rn(*sa, *sx);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __fmul_rn(__int2float_rn(acc[i]), s);
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
cudaError_t launch_edge_sum(const GraphDev& g, int dir, int heads, const float* x, float* out, int64_t e_list,
                            cudaStream_t st) {
  if (g.n_local == 0) return cudaSuccess;
  ProfScope ps("edge_sum", st);
  // edges per block: about 8 blocks per SM, at least 256, at most 16 Ki edges
  const int64_t e = e_list > 0 ? e_list : 1;
  int64_t epb = e / ((int64_t)num_sms() * 8);
  epb = epb < 256 ? 256 : (epb > 16384 ? 16384 : epb);
  const int64_t blocks = (g.n_local + ES_ROWS - 1) / ES_ROWS;   // row blocks
  const size_t smem = (size_t)(es_slots(heads) + 1) * heads * 4;
  const uintptr_t xa = reinterpret_cast<uintptr_t>(x);
  const int vw = (heads % 4 == 0 && xa % 16 == 0) ? 4 : (heads % 2 == 0 && xa % 8 == 0) ? 2 : 1;
  void (*f)(GraphDev, int, int64_t, int64_t, const float*, float*) =
      dir ? (vw == 4 ? k_edge_sum_w<1, 4> : vw == 2 ? k_edge_sum_w<1, 2> : k_edge_sum_w<1, 1>)
          : (vw == 4 ? k_edge_sum_w<0, 4> : vw == 2 ? k_edge_sum_w<0, 2> : k_edge_sum_w<0, 1>);
  if (smem > 48 * 1024) {
    const cudaError_t err = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
  }
  f<<<(unsigned)blocks, ES_THREADS, smem, st>>>(g, heads, epb, e_list, x, out);
  return cudaGetLastError();
}
cudaError_t launch_spmm_w(const GraphDev& g, int dir, int heads, int cols, const float* w, const int8_t* qX,
                          int64_t ldx, const float* sX, const float* rowscale, float* out, unsigned* amax_out,
                          int64_t e_list, cudaStream_t st) {
  if (g.n_local == 0) return cudaSuccess;
  ProfScope ps("spmm_w", st);
  const int64_t blocks = (g.n_local + ES_ROWS - 1) / ES_ROWS;   // row blocks
  const int D = cols / heads;
  const uintptr_t qa = reinterpret_cast<uintptr_t>(qX);
  const int v = (D % 16 == 0 && ldx % 16 == 0 && qa % 16 == 0) ? 16 : (D % 4 == 0 && ldx % 4 == 0 && qa % 4 == 0) ? 4 : 1;
  void (*f)(GraphDev, int, int, int64_t, int64_t, const float*, const int8_t*, int64_t, const float*, const float*,
            float*, unsigned*);
  size_t cols_pass;
  int slots;
  if (v == 16) { f = dir ? k_spmm_w_fast<1, 16> : k_spmm_w_fast<0, 16>; cols_pass = sw_cols<16>(); slots = sw_slots<16>(); }
  else if (v == 4) { f = dir ? k_spmm_w_fast<1, 4> : k_spmm_w_fast<0, 4>; cols_pass = sw_cols<4>(); slots = sw_slots<4>(); }
  else { f = dir ? k_spmm_w_fast<1, 1> : k_spmm_w_fast<0, 1>; cols_pass = sw_cols<1>(); slots = sw_slots<1>(); }
  const size_t smem = (size_t)(slots + 1) * cols_pass * 4 + (size_t)(ES_THREADS / 32) * 32 * (1 + heads) * 4;
  if (smem > 48 * 1024) {
    const cudaError_t err = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
  }
  f<<<(unsigned)blocks, ES_THREADS, smem, st>>>(g, heads, cols, 0, e_list, w, qX, ldx, sX, rowscale, out, amax_out);
  return cudaGetLastError();
}
cudaError_t launch_spmm_q8(const GraphDev& g, int dir, int heads, int cols, const int8_t* qa, const float* sa,
                           const int8_t* qX, int64_t ldx, const float* sX, int32_t* out_i32, float* out,
                           int64_t e_list, cudaStream_t st) {
  if (g.n_local == 0) return cudaSuccess;
  cudaError_t err = cudaMemsetAsync(out_i32, 0, (size_t)g.n_local * cols * 4, st);
  if (err != cudaSuccess) return err;
  {
    ProfScope ps("spmm_q8", st);
    const int64_t e = e_list > 0 ? e_list : 1;
    int64_t epb = e / ((int64_t)num_sms() * 4);
    epb = epb < 256 ? 256 : (epb > 16384 ? 16384 : epb);
    const int64_t blocks = (g.n_local + ES_ROWS - 1) / ES_ROWS;   // row blocks
    const size_t smem = (size_t)(ES_THREADS / 32) * 32 * (4 + heads);
    auto f = dir ? k_spmm_q8<1> : k_spmm_q8<0>;
    if (smem > 48 * 1024) {
      err = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (err != cudaSuccess) return err;
    }
    f<<<(unsigned)blocks, ES_THREADS, smem, st>>>(g, heads, cols, epb, e_list, qa, qX, ldx, out_i32);
    err = cudaGetLastError();
    if (err != cudaSuccess) return err;
  }
  if (out) {
    ProfScope ps("spmm_q8_out", st);
    const int64_t count = g.n_local * (int64_t)cols;
    int64_t gr = (count + 255) / 256;
    if (gr > (int64_t)num_sms() * 8) gr = (int64_t)num_sms() * 8;
    k_i32_to_f32<<<(unsigned)gr, 256, 0, st>>>(out_i32, count, sa, sX, out);
    err = cudaGetLastError();
  }
  return err;
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
