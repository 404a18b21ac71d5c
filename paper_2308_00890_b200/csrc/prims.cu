// prims.cu — the unfused sparse primitives of the C ABI (tango_sddmm_q, tango_edge_softmax,
// tango_softmax_bwd, tango_edge_sum, tango_spmm_q) and the GCN helpers.  One thread per
// (row, head) or (row, column), sequential over the row's edges in canonical order: the same
// arithmetic as the fused kernels of gat.cu, laid out for clarity rather than speed.
// Paper: ③ P:204-209, ④ P:212-217, ⑤/⑤′ P:224-251, ⑤″ P:252-255, ④′ P:258-264,
// ③′/③″ P:276 and P:821-832, GCN P:347-348.
#include "rowops.cuh"

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
