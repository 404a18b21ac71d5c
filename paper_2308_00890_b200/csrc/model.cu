// model.cu — NEXT-1: the training step around the quantized GAT layer.
//
//  * tango_sgemm            full-precision GEMM with the pinned K-chunked FMA order (reading R33)
//  * tango_gat_out_fwd/bwd  the FP32 final GAT layer ("full precision for the layer before the
//                           Softmax", §3.2 Eq.7-8), heads averaged + bias (R35)
//  * tango_bias_act_fwd/bwd hidden-layer bias + ReLU with the next quantizer's amax (R34)
//  * tango_cross_entropy    mean cross-entropy over labelled rows (R36)
//  * tango_sgd_update       W <- W - lr*dW on the FP32 masters (Eq.6, R37)
//
// Every value compared bit for bit with the oracle is computed with explicit round-to-nearest
// intrinsics in the order the readings fix; only the attention-vector gradients (atomics) and the
// loss scalar (logf, double atomics) are order-free and compared within a tolerance.
#include <algorithm>
#include <cstdio>
#include <cstring>

#include "../../include/tango.h"
#include "rowops.cuh"

namespace tango {

constexpr int kCK = 1024;   // R33: chunk of the full-precision contractions and column sums

static int grid_1d(int64_t n, int threads = 256) {
  int64_t g = (n + threads - 1) / threads;
  const int64_t cap = (int64_t)num_sms() * 32;
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

// ------------------------------------------------------------------ full-precision GEMM (R33)
// C[m][n] = sequential fmaf chain over k in [kbeg, kend) of A(m,k)*B(k,n), starting from 0.
// A(m,k) = TA ? A[k*lda + m] : A[m*lda + k];  B(k,n) = TB ? B[n*ldb + k] : B[k*ldb + n].
// Block z covers chunk z (k in [z*kCK, (z+1)*kCK)) and writes C + z*M*N; with one chunk that is C.
// 64x64 tile, BK = 16, 256 threads with 4x4 outputs each; the next k-tile is prefetched into
// registers while the current one is consumed from shared memory.
constexpr int SG_BM = 64, SG_BN = 64, SG_BK = 16, SG_PAD = 4;

template <bool TA, bool TB>
__global__ void __launch_bounds__(256) k_sgemm(const float* __restrict__ A, int64_t lda, const float* __restrict__ B,
                                               int64_t ldb, int64_t M, int64_t N, int64_t K,
                                               float* __restrict__ C) {
  __shared__ __align__(16) float As[SG_BK][SG_BM + SG_PAD];
  __shared__ __align__(16) float Bs[SG_BK][SG_BN + SG_PAD];
  const int t = threadIdx.x;
  const int64_t m0 = (int64_t)blockIdx.y * SG_BM, n0 = (int64_t)blockIdx.x * SG_BN;
  const int64_t kbeg = (int64_t)blockIdx.z * kCK;
  const int64_t kend = min(K, kbeg + kCK);
  float* Cz = C + (int64_t)blockIdx.z * M * N;

  float ra[4], rb[4];
  auto load = [&](int64_t k0) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int i = t + 256 * r;
      int mm, kk;
      if (TA) { kk = i / SG_BM; mm = i % SG_BM; } else { mm = i / SG_BK; kk = i % SG_BK; }
      const int64_t gm = m0 + mm, gk = k0 + kk;
      ra[r] = (gm < M && gk < kend) ? (TA ? __ldg(A + gk * lda + gm) : __ldg(A + gm * lda + gk)) : 0.0f;
      int nn, kb;
      if (TB) { nn = i / SG_BK; kb = i % SG_BK; } else { kb = i / SG_BN; nn = i % SG_BN; }
      const int64_t gn = n0 + nn, gkb = k0 + kb;
      rb[r] = (gn < N && gkb < kend) ? (TB ? __ldg(B + gn * ldb + gkb) : __ldg(B + gkb * ldb + gn)) : 0.0f;
    }
  };
  auto store = [&]() {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int i = t + 256 * r;
      int mm, kk;
      if (TA) { kk = i / SG_BM; mm = i % SG_BM; } else { mm = i / SG_BK; kk = i % SG_BK; }
      As[kk][mm] = ra[r];
      int nn, kb;
      if (TB) { nn = i / SG_BK; kb = i % SG_BK; } else { kb = i / SG_BN; nn = i % SG_BN; }
      Bs[kb][nn] = rb[r];
    }
  };

  const int ty = t / 16, tx = t % 16;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;

  if (kbeg < kend) load(kbeg);
  for (int64_t k0 = kbeg; k0 < kend; k0 += SG_BK) {
    __syncthreads();
    store();
    __syncthreads();
    if (k0 + SG_BK < kend) load(k0 + SG_BK);
    const int kmax = (kend - k0 < SG_BK) ? (int)(kend - k0) : SG_BK;
    if (kmax == SG_BK) {
#pragma unroll
      for (int kk = 0; kk < SG_BK; ++kk) {
        const float4 a = *reinterpret_cast<const float4*>(&As[kk][ty * 4]);
        const float4 b = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
        const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = __fmaf_rn(av[i], bv[j], acc[i][j]);
      }
    } else {
      for (int kk = 0; kk < kmax; ++kk) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = __fmaf_rn(As[kk][ty * 4 + i], Bs[kk][tx * 4 + j], acc[i][j]);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t gm = m0 + ty * 4 + i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t gn = n0 + tx * 4 + j;
      if (gn < N) Cz[gm * N + gn] = acc[i][j];
    }
  }
}

// Left-to-right fold of chunk partials (R14/R33): out[i] = ((p0 + p1) + p2) + ...
__global__ void k_fold(const float* __restrict__ ws, int64_t count, int nchunks, float* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    float t = ws[i];
    for (int c = 1; c < nchunks; ++c) t = __fadd_rn(t, ws[(int64_t)c * count + i]);
    out[i] = t;
  }
}

static inline int64_t nchunks_of(int64_t K) { return K <= kCK ? 1 : (K + kCK - 1) / kCK; }

static size_t sgemm_ws_bytes(int64_t M, int64_t N, int64_t K) {
  const int64_t nc = nchunks_of(K);
  return nc > 1 ? (size_t)nc * (size_t)M * (size_t)N * sizeof(float) : 0;
}

static cudaError_t launch_sgemm(const float* A, int64_t lda, bool ta, const float* B, int64_t ldb, bool tb, int64_t M,
                                int64_t N, int64_t K, float* C, float* ws, cudaStream_t st) {
  if (M == 0 || N == 0) return cudaSuccess;
  const int64_t nc = nchunks_of(K);
  float* dst = nc > 1 ? ws : C;
  dim3 grid((unsigned)((N + SG_BN - 1) / SG_BN), (unsigned)((M + SG_BM - 1) / SG_BM), (unsigned)nc);
  {
    ProfScope ps("sgemm", st);
    if (!ta && !tb) k_sgemm<false, false><<<grid, 256, 0, st>>>(A, lda, B, ldb, M, N, K, dst);
    else if (ta && !tb) k_sgemm<true, false><<<grid, 256, 0, st>>>(A, lda, B, ldb, M, N, K, dst);
    else if (!ta && tb) k_sgemm<false, true><<<grid, 256, 0, st>>>(A, lda, B, ldb, M, N, K, dst);
    else k_sgemm<true, true><<<grid, 256, 0, st>>>(A, lda, B, ldb, M, N, K, dst);
  }
  if (nc > 1) {
    ProfScope ps("sgemm_fold", st);
    k_fold<<<grid_1d(M * N), 256, 0, st>>>(ws, M * N, (int)nc, C);
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------ column sums over rows (R33)
// Thread per (column, 1024-row chunk): plain sequential adds; partial per chunk, folded after.
// MODE 0: x -> partials.  MODE 1 (ReLU backward, R34): d = a > 0 ? da : 0 written to dx, |d| max
// into amax, and d summed.
template <int MODE>
__global__ void __launch_bounds__(256) k_colsum(const float* __restrict__ x, const float* __restrict__ da,
                                                int64_t rows, int64_t cols, float* __restrict__ dst,
                                                float* __restrict__ dx, unsigned* amax) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t c = blockIdx.y;
  const int64_t r0 = c * kCK, r1 = min(rows, r0 + kCK);
  float part = 0.0f, mx = 0.0f;
  if (j < cols) {
    constexpr int U = 16;
    int64_t r = r0;
    for (; r + U <= r1; r += U) {
      float v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t i = (r + u) * cols + j;
        if (MODE == 0) v[u] = __ldg(x + i);
        else { const float a = __ldg(x + i), d = __ldg(da + i); v[u] = a > 0.0f ? d : 0.0f; dx[i] = v[u]; }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        part = __fadd_rn(part, v[u]);
        if (MODE == 1) mx = fmaxf(mx, fabsf(v[u]));
      }
    }
    for (; r < r1; ++r) {
      const int64_t i = r * cols + j;
      float v;
      if (MODE == 0) v = __ldg(x + i);
      else { const float a = __ldg(x + i), d = __ldg(da + i); v = a > 0.0f ? d : 0.0f; dx[i] = v; }
      part = __fadd_rn(part, v);
      if (MODE == 1) mx = fmaxf(mx, fabsf(v));
    }
    dst[c * cols + j] = part;
  }
  if (MODE == 1) {
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    if ((threadIdx.x & 31) == 0 && amax) atomicMax(amax, __float_as_uint(mx));
  }
}

static size_t colsum_ws_bytes(int64_t rows, int64_t cols) {
  const int64_t nc = nchunks_of(rows);
  return nc > 1 ? (size_t)nc * (size_t)cols * sizeof(float) : 0;
}

template <int MODE>
static cudaError_t launch_colsum(const float* x, const float* da, int64_t rows, int64_t cols, float* out, float* ws,
                                 float* dx, float* amax, cudaStream_t st) {
  if (cols == 0) return cudaSuccess;
  if (amax) {
    cudaError_t e = cudaMemsetAsync(amax, 0, sizeof(float), st);
    if (e != cudaSuccess) return e;
  }
  if (rows == 0) return cudaMemsetAsync(out, 0, cols * sizeof(float), st);
  const int64_t nc = nchunks_of(rows);
  float* dst = nc > 1 ? ws : out;
  dim3 grid((unsigned)((cols + 255) / 256), (unsigned)nc);
  {
    ProfScope ps(MODE == 0 ? "colsum" : "bias_relu_bwd", st);
    k_colsum<MODE><<<grid, 256, 0, st>>>(x, da, rows, cols, dst, dx, reinterpret_cast<unsigned*>(amax));
  }
  if (nc > 1) {
    ProfScope ps("colsum_fold", st);
    k_fold<<<grid_1d(cols), 256, 0, st>>>(ws, cols, (int)nc, out);
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------ bias + ReLU forward (R34)
__global__ void __launch_bounds__(256) k_bias_relu_fwd(const float* __restrict__ x, const float* __restrict__ b,
                                                       int64_t rows, int64_t cols, float* __restrict__ y,
                                                       unsigned* amax) {
  float mx = 0.0f;
  const int64_t n = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float v = __fadd_rn(__ldg(x + i), __ldg(b + i % cols));
    const float a = v > 0.0f ? v : 0.0f;
    y[i] = a;
    mx = fmaxf(mx, a);
  }
  mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
  mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
  mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
  mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
  mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
  if ((threadIdx.x & 31) == 0 && amax) atomicMax(amax, __float_as_uint(mx));
}

// ------------------------------------------------------------------ cross-entropy (R36)
// Warp per row; the exps of a row are staged in shared memory and summed by lane 0 in class order.
constexpr int XE_MAXC = 1024;
__global__ void __launch_bounds__(128) k_xent(const float* __restrict__ z, const int32_t* __restrict__ labels,
                                              int64_t rows, int C, float inv_dummy, float n_lab,
                                              float* __restrict__ dz, double* loss_acc, int32_t* status) {
  extern __shared__ float sh[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* ex = sh + warp * C;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t v = blockIdx.x * (int64_t)(blockDim.x >> 5) + warp; v < rows; v += nw) {
    const int32_t y = labels[v];
    const float* zr = z + v * C;
    float* dr = dz + v * C;
    if (y >= C) {
      if (lane == 0 && status) atomicCAS(status, 0, (int32_t)TANGO_ERR_INVALID_ARG);
      for (int c = lane; c < C; c += 32) dr[c] = 0.0f;
      continue;
    }
    if (y < 0) {
      for (int c = lane; c < C; c += 32) dr[c] = 0.0f;
      continue;
    }
    float m = -INFINITY;
    for (int c = lane; c < C; c += 32) m = fmaxf(m, zr[c]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    for (int c = lane; c < C; c += 32) ex[c] = exp_p(__fsub_rn(zr[c], m));
    __syncwarp();
    float ssum = 0.0f;
    if (lane == 0) {
      for (int c = 0; c < C; ++c) ssum = __fadd_rn(ssum, ex[c]);
      const float lv = __fsub_rn(__fadd_rn(m, logf(ssum)), zr[y]);
      atomicAdd(loss_acc, (double)lv);
    }
    ssum = __shfl_sync(0xffffffffu, ssum, 0);
    for (int c = lane; c < C; c += 32) {
      const float p = __fdiv_rn(ex[c], ssum);
      const float t = __fsub_rn(p, c == y ? 1.0f : 0.0f);
      dr[c] = __fdiv_rn(t, n_lab);
    }
    __syncwarp();
  }
}
__global__ void k_xent_finish(double* loss, double n_lab) {
  if (threadIdx.x == 0 && blockIdx.x == 0) *loss = n_lab > 0 ? *loss / n_lab : 0.0;
}

// ------------------------------------------------------------------ SGD on the FP32 masters (R37)
constexpr int SGD_MAX = 32;
struct SgdList {
  float* w[SGD_MAX];
  const float* g[SGD_MAX];
  int64_t off[SGD_MAX + 1];
  int n;
};
__global__ void __launch_bounds__(256) k_sgd(SgdList L, float lr) {
  const int64_t total = L.off[L.n];
  int t = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    while (i >= L.off[t + 1]) ++t;
    const int64_t k = i - L.off[t];
    L.w[t][k] = __fsub_rn(L.w[t][k], __fmul_rn(lr, L.g[t][k]));
  }
}

// ------------------------------------------------------------------ FP32 final GAT layer (R35)
// S, D per (row, head): sequential fmaf over the head's C columns (R10 in FP32)
__global__ void k_out_sd(const float* __restrict__ Hp, int64_t n, int heads, int C, const float* __restrict__ a_src,
                         const float* __restrict__ a_dst, float* __restrict__ S, float* __restrict__ D) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (tid >= n * heads) return;
  const int64_t v = tid / heads;
  const int h = (int)(tid % heads);
  const float* r = Hp + v * (int64_t)heads * C + (int64_t)h * C;
  float s = 0.0f, d = 0.0f;
  for (int c = 0; c < C; ++c) {
    s = __fmaf_rn(r[c], a_src[h * C + c], s);
    d = __fmaf_rn(r[c], a_dst[h * C + c], d);
  }
  S[tid] = s;
  D[tid] = d;
}

// ③ in FP32: e_pre = S[u] + D[v], el = LeakyReLU(e_pre) (thread per (row, head), in-CSR order)
__global__ void k_out_el(GraphDev g, int heads, const float* __restrict__ S, const float* __restrict__ D, float slope,
                         float* __restrict__ e_pre, float* __restrict__ el) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (tid >= g.n_local * heads) return;
  const int64_t v = tid / heads;
  const int h = (int)(tid % heads);
  const float dv = D[v * heads + h];
  for (int64_t e = g.in_ptr[v]; e < g.in_ptr[v + 1]; ++e) {
    const float x = __fadd_rn(S[(int64_t)g.in_src[e] * heads + h], dv);
    e_pre[e * heads + h] = x;
    el[e * heads + h] = x > 0.0f ? x : __fmul_rn(x, slope);
  }
}

// ⑤ + head mean + bias: warp per destination row; column j of head h = j / C sums
// Σᶜ fmaf(α[e,h], H′[u,j]) over the in-edges (R14), then logits = ((Σ_h agg) / heads) + b.
constexpr int OUT_MAXHC = 1024;
__global__ void __launch_bounds__(256) k_out_agg(GraphDev g, int heads, int C, const float* __restrict__ alpha,
                                                 const float* __restrict__ Hp, const float* __restrict__ bias,
                                                 float* __restrict__ logits) {
  extern __shared__ float sh[];
  const int HC = heads * C;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* agg = sh + warp * HC;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t v = blockIdx.x * (int64_t)(blockDim.x >> 5) + warp; v < g.n_local; v += nw) {
    const int64_t b = g.in_ptr[v], e1 = g.in_ptr[v + 1];
    for (int j = lane; j < HC; j += 32) {
      const int h = j / C;
      CSum cs; cs.init();
      int left = g.chunk;
      for (int64_t e = b; e < e1; ++e) {
        if (left == 0) { cs.fold(); left = g.chunk; }
        cs.part = __fmaf_rn(alpha[e * heads + h], Hp[(int64_t)g.in_src[e] * HC + j], cs.part);
        --left;
      }
      agg[j] = cs.finish(e1 - b);
    }
    __syncwarp();
    for (int c = lane; c < C; c += 32) {
      float t = agg[c];
      for (int h = 1; h < heads; ++h) t = __fadd_rn(t, agg[h * C + c]);
      t = __fdiv_rn(t, (float)heads);
      logits[v * C + c] = __fadd_rn(t, bias[c]);
    }
    __syncwarp();
  }
}

// G = ∂logits / heads (the gradient reaching every head's aggregation)
__global__ void k_out_g(const float* __restrict__ dz, int64_t count, float heads, float* __restrict__ G) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    G[i] = __fdiv_rn(dz[i], heads);
}

// ⑤″ in FP32: ∂α[e,h] = Σ_c fmaf(G[v,c], H′[u,h,c]) sequential in c
__global__ void k_out_dalpha(GraphDev g, int heads, int C, const float* __restrict__ G, const float* __restrict__ Hp,
                             float* __restrict__ dalpha) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (tid >= g.n_local * heads) return;
  const int64_t v = tid / heads;
  const int h = (int)(tid % heads);
  const int HC = heads * C;
  const float* gv = G + v * C;
  for (int64_t e = g.in_ptr[v]; e < g.in_ptr[v + 1]; ++e) {
    const float* hu = Hp + (int64_t)g.in_src[e] * HC + (int64_t)h * C;
    float acc = 0.0f;
    for (int c = 0; c < C; ++c) acc = __fmaf_rn(gv[c], hu[c], acc);
    dalpha[e * heads + h] = acc;
  }
}

// ⑤′ + ②′ in FP32: warp per source row u; ∂H′_agg[u,j] = Σᶜ over out-edges fmaf(α[eid,h], G[v,c]),
// ∂H′ = (∂H′_agg + ∂S·a_src) + ∂D·a_dst (R23)
__global__ void __launch_bounds__(256) k_out_dhp(GraphDev g, int heads, int C, const float* __restrict__ alpha,
                                                 const float* __restrict__ G, const float* __restrict__ dS,
                                                 const float* __restrict__ dD, const float* __restrict__ a_src,
                                                 const float* __restrict__ a_dst, float* __restrict__ dHp) {
  const int HC = heads * C;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t u = blockIdx.x * (int64_t)(blockDim.x >> 5) + warp; u < g.n_local; u += nw) {
    const int64_t b = g.out_ptr[u], e1 = g.out_ptr[u + 1];
    for (int j = lane; j < HC; j += 32) {
      const int h = j / C, c = j - h * C;
      CSum cs; cs.init();
      int left = g.chunk;
      for (int64_t p = b; p < e1; ++p) {
        if (left == 0) { cs.fold(); left = g.chunk; }
        const int64_t eid = g.out_eid[p];
        cs.part = __fmaf_rn(alpha[eid * heads + h], G[(int64_t)g.out_dst[p] * C + c], cs.part);
        --left;
      }
      const float agg = cs.finish(e1 - b);
      const float t1 = __fmul_rn(dS[u * heads + h], a_src[j]);
      const float t2 = __fadd_rn(agg, t1);
      const float t3 = __fmul_rn(dD[u * heads + h], a_dst[j]);
      dHp[u * HC + j] = __fadd_rn(t2, t3);
    }
  }
}

// ∂a_src[j] = Σ_u ∂S[u,h]·H′[u,j], ∂a_dst likewise (fp32 per thread, then atomics: order-free,
// compared within the DESIGN.md §3 bound)
__global__ void __launch_bounds__(256) k_out_da(const float* __restrict__ Hp, int64_t n, int heads, int C,
                                                const float* __restrict__ dS, const float* __restrict__ dD,
                                                float* __restrict__ da_src, float* __restrict__ da_dst) {
  const int HC = heads * C;
  for (int j0 = 0; j0 < HC; j0 += blockDim.x) {
    const int j = j0 + threadIdx.x;
    if (j >= HC) break;
    const int h = j / C;
    float as = 0.0f, ad = 0.0f;
    for (int64_t u = blockIdx.x; u < n; u += gridDim.x) {
      const float x = Hp[u * HC + j];
      as = __fmaf_rn(dS[u * heads + h], x, as);
      ad = __fmaf_rn(dD[u * heads + h], x, ad);
    }
    atomicAdd(da_src + j, as);
    atomicAdd(da_dst + j, ad);
  }
}

}  // namespace tango

using namespace tango;

#define M_TRY_CUDA(x)                                                                                  \
  do {                                                                                                 \
    cudaError_t e_ = (x);                                                                              \
    if (e_ != cudaSuccess) {                                                                           \
      fprintf(stderr, "[tango] CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return TANGO_ERR_CUDA;                                                                           \
    }                                                                                                  \
  } while (0)

namespace {
struct OutLayout {
  int64_t n, e, F, H, C, HC;
  size_t off_Hp, off_S, off_D, off_epre, off_el, off_alpha, off_m, off_den, off_G, off_dalpha, off_dEp, off_P,
      off_dD, off_dS, off_dHp, off_ws, total;
};
inline size_t al256(size_t x) { return (x + 255) & ~size_t(255); }
bool out_layout(const tango_graph* G, const tango_gat_out_params* p, OutLayout* L) {
  if (!G || !p) return false;
  if (p->in_feats <= 0 || p->heads <= 0 || p->classes <= 0) return false;
  L->n = G->row_end - G->row_begin;
  L->e = G->e_in;
  L->F = p->in_feats; L->H = p->heads; L->C = p->classes; L->HC = L->H * L->C;
  const int64_t n = L->n, e = L->e, H = L->H, HC = L->HC, F = L->F;
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o = al256(o + bytes); return r; };
  L->off_Hp = take(4 * n * HC);
  L->off_S = take(4 * n * H);
  L->off_D = take(4 * n * H);
  L->off_epre = take(4 * e * H);
  L->off_el = take(4 * e * H);
  L->off_alpha = take(4 * e * H);
  L->off_m = take(4 * n * H);
  L->off_den = take(4 * n * H);
  L->off_G = take(4 * n * L->C);
  L->off_dalpha = take(4 * e * H);
  L->off_dEp = take(4 * e * H);
  L->off_P = take(4 * n * H);
  L->off_dD = take(4 * n * H);
  L->off_dS = take(4 * n * H);
  L->off_dHp = take(4 * n * HC);
  size_t ws = sgemm_ws_bytes(F, HC, n);
  ws = std::max(ws, sgemm_ws_bytes(n, F, HC));
  ws = std::max(ws, colsum_ws_bytes(n, L->C));
  L->off_ws = take(ws > 0 ? ws : 4);
  L->total = o;
  return true;
}
GraphDev dev_graph(const tango_graph* G) {
  GraphDev g;
  g.n_local = G->row_end - G->row_begin;
  g.row_begin = G->row_begin;
  g.n_global = G->n_global;
  g.in_ptr = G->in_ptr; g.in_src = G->in_src;
  g.out_ptr = G->out_ptr; g.out_dst = G->out_dst; g.out_eid = G->out_eid;
  g.chunk = G->chunk_edges > 0 ? G->chunk_edges : 256;
  return g;
}
tango_status check_out(const tango_graph* G, const tango_gat_out_params* p) {
  if (!G || !p || !p->W || !p->a_src || !p->a_dst || !p->bias) return TANGO_ERR_INVALID_ARG;
  if (p->in_feats <= 0 || p->heads <= 0 || p->classes <= 0) return TANGO_ERR_SHAPE;
  if ((int64_t)p->heads * p->classes > OUT_MAXHC) return TANGO_ERR_UNSUPPORTED;
  // one GPU: the final layer runs on the whole graph (partitioning is NEXT-3)
  if (G->row_begin != 0 || G->row_end != G->n_global) return TANGO_ERR_UNSUPPORTED;
  if (G->n_global > 0 && (!G->in_ptr || !G->out_ptr)) return TANGO_ERR_INVALID_ARG;
  if (G->e_in > 0 && (!G->in_src || !G->out_dst || !G->out_eid)) return TANGO_ERR_INVALID_ARG;
  if (G->e_in != G->e_out) return TANGO_ERR_SHAPE;
  if (p->neg_slope != p->neg_slope) return TANGO_ERR_INVALID_ARG;
  return TANGO_OK;
}
}  // namespace

extern "C" {

size_t tango_sgemm_workspace_bytes(int64_t M, int64_t N, int64_t K) {
  if (M < 0 || N < 0 || K < 0) return 0;
  return sgemm_ws_bytes(M, N, K);
}

tango_status tango_sgemm(const float* A, int64_t lda, int32_t a_layout, const float* B, int64_t ldb, int32_t b_layout,
                         int64_t M, int64_t N, int64_t K, float* C, void* workspace, size_t ws_bytes,
                         cudaStream_t stream) {
  if (M < 0 || N < 0 || K < 0) return TANGO_ERR_SHAPE;
  if (a_layout != TANGO_K_MAJOR && a_layout != TANGO_MN_MAJOR) return TANGO_ERR_INVALID_ARG;
  if (b_layout != TANGO_K_MAJOR && b_layout != TANGO_MN_MAJOR) return TANGO_ERR_INVALID_ARG;
  if (M == 0 || N == 0) return TANGO_OK;
  if (!C || (K > 0 && (!A || !B))) return TANGO_ERR_INVALID_ARG;
  const bool ta = a_layout == TANGO_MN_MAJOR, tb = b_layout == TANGO_K_MAJOR;
  if (lda < (ta ? M : K) || ldb < (tb ? K : N)) return TANGO_ERR_SHAPE;
  if ((M + SG_BM - 1) / SG_BM > 65535 || nchunks_of(K) > 65535) return TANGO_ERR_UNSUPPORTED;
  const size_t need = sgemm_ws_bytes(M, N, K);
  if (need > 0 && (!workspace || ws_bytes < need)) return TANGO_ERR_INVALID_ARG;
  M_TRY_CUDA(launch_sgemm(A, lda, ta, B, ldb, tb, M, N, K, C, static_cast<float*>(workspace), stream));
  return TANGO_OK;
}

size_t tango_colsum_workspace_bytes(int64_t rows, int64_t cols) {
  if (rows < 0 || cols < 0) return 0;
  return colsum_ws_bytes(rows, cols);
}

tango_status tango_colsum(const float* x, int64_t rows, int64_t cols, float* out, void* workspace, size_t ws_bytes,
                          cudaStream_t stream) {
  if (rows < 0 || cols < 0) return TANGO_ERR_SHAPE;
  if (cols == 0) return TANGO_OK;
  if (!out || (rows > 0 && !x)) return TANGO_ERR_INVALID_ARG;
  const size_t need = colsum_ws_bytes(rows, cols);
  if (need > 0 && (!workspace || ws_bytes < need)) return TANGO_ERR_INVALID_ARG;
  M_TRY_CUDA(launch_colsum<0>(x, nullptr, rows, cols, out, static_cast<float*>(workspace), nullptr, nullptr, stream));
  return TANGO_OK;
}

tango_status tango_bias_act_fwd(const float* x, const float* bias, int64_t rows, int64_t cols, float* y,
                                float* amax_out, cudaStream_t stream) {
  if (rows < 0 || cols < 0) return TANGO_ERR_SHAPE;
  if (amax_out) M_TRY_CUDA(cudaMemsetAsync(amax_out, 0, sizeof(float), stream));
  if (rows == 0 || cols == 0) return TANGO_OK;
  if (!x || !bias || !y) return TANGO_ERR_INVALID_ARG;
  {
    ProfScope ps("bias_relu_fwd", stream);
    k_bias_relu_fwd<<<grid_1d(rows * cols), 256, 0, stream>>>(x, bias, rows, cols, y,
                                                              reinterpret_cast<unsigned*>(amax_out));
  }
  M_TRY_CUDA(cudaGetLastError());
  return TANGO_OK;
}

tango_status tango_bias_act_bwd(const float* y, const float* dy, int64_t rows, int64_t cols, float* dx, float* dbias,
                                float* amax_dx, void* workspace, size_t ws_bytes, cudaStream_t stream) {
  if (rows < 0 || cols < 0) return TANGO_ERR_SHAPE;
  if (cols == 0) return TANGO_OK;
  if (!dbias || (rows > 0 && (!y || !dy || !dx))) return TANGO_ERR_INVALID_ARG;
  const size_t need = colsum_ws_bytes(rows, cols);
  if (need > 0 && (!workspace || ws_bytes < need)) return TANGO_ERR_INVALID_ARG;
  M_TRY_CUDA(launch_colsum<1>(y, dy, rows, cols, dbias, static_cast<float*>(workspace), dx, amax_dx, stream));
  return TANGO_OK;
}

tango_status tango_cross_entropy(const float* logits, const int32_t* labels, int64_t rows, int32_t classes,
                                 int64_t n_labeled, float* dlogits, double* loss_out, int32_t* dev_status,
                                 cudaStream_t stream) {
  if (rows < 0 || classes <= 0 || n_labeled < 0 || n_labeled > rows) return TANGO_ERR_SHAPE;
  if (classes > XE_MAXC) return TANGO_ERR_UNSUPPORTED;
  if (!loss_out) return TANGO_ERR_INVALID_ARG;
  M_TRY_CUDA(cudaMemsetAsync(loss_out, 0, sizeof(double), stream));
  if (rows == 0) return TANGO_OK;
  if (!logits || !labels || !dlogits) return TANGO_ERR_INVALID_ARG;
  {
    ProfScope ps("cross_entropy", stream);
    const size_t smem = 4 * sizeof(float) * (size_t)classes;
    k_xent<<<grid_1d(rows, 4), 128, smem, stream>>>(logits, labels, rows, classes, 0.0f,
                                                    n_labeled > 0 ? (float)n_labeled : 1.0f, dlogits, loss_out,
                                                    dev_status);
  }
  {
    ProfScope ps("cross_entropy_finish", stream);
    k_xent_finish<<<1, 32, 0, stream>>>(loss_out, (double)n_labeled);
  }
  M_TRY_CUDA(cudaGetLastError());
  return TANGO_OK;
}

tango_status tango_sgd_update(const tango_sgd_tensor* tensors, int32_t count, float lr, cudaStream_t stream) {
  if (count < 0 || count > SGD_MAX) return TANGO_ERR_UNSUPPORTED;
  if (count == 0) return TANGO_OK;
  if (!tensors) return TANGO_ERR_INVALID_ARG;
  SgdList L;
  memset(&L, 0, sizeof(L));
  L.n = count;
  L.off[0] = 0;
  for (int i = 0; i < count; ++i) {
    if (tensors[i].count < 0) return TANGO_ERR_SHAPE;
    if (tensors[i].count > 0 && (!tensors[i].w || !tensors[i].g)) return TANGO_ERR_INVALID_ARG;
    L.w[i] = tensors[i].w;
    L.g[i] = tensors[i].g;
    L.off[i + 1] = L.off[i] + tensors[i].count;
  }
  if (L.off[count] == 0) return TANGO_OK;
  {
    ProfScope ps("sgd", stream);
    k_sgd<<<grid_1d(L.off[count]), 256, 0, stream>>>(L, lr);
  }
  M_TRY_CUDA(cudaGetLastError());
  return TANGO_OK;
}

size_t tango_gat_out_ctx_bytes(const tango_graph* G, const tango_gat_out_params* p) {
  OutLayout L;
  if (check_out(G, p) != TANGO_OK || !out_layout(G, p, &L)) return 0;
  return L.total;
}

tango_status tango_gat_out_fwd(const tango_graph* G, const tango_gat_out_params* p, const float* H, void* ctx,
                               size_t ctx_bytes, float* logits, cudaStream_t stream) {
  tango_status s = check_out(G, p);
  if (s != TANGO_OK) return s;
  OutLayout L;
  out_layout(G, p, &L);
  if (!ctx || ctx_bytes < L.total) return TANGO_ERR_INVALID_ARG;
  if (L.n == 0) return TANGO_OK;
  if (!H || !logits) return TANGO_ERR_INVALID_ARG;
  char* c = static_cast<char*>(ctx);
  float* Hp = reinterpret_cast<float*>(c + L.off_Hp);
  float* S = reinterpret_cast<float*>(c + L.off_S);
  float* D = reinterpret_cast<float*>(c + L.off_D);
  float* epre = reinterpret_cast<float*>(c + L.off_epre);
  float* el = reinterpret_cast<float*>(c + L.off_el);
  float* alpha = reinterpret_cast<float*>(c + L.off_alpha);
  float* m = reinterpret_cast<float*>(c + L.off_m);
  float* den = reinterpret_cast<float*>(c + L.off_den);
  float* ws = reinterpret_cast<float*>(c + L.off_ws);
  const GraphDev g = dev_graph(G);
  const int H_ = (int)L.H, C_ = (int)L.C;
  // ① H′ = H·W (R33)
  M_TRY_CUDA(launch_sgemm(H, L.F, false, p->W, L.HC, false, L.n, L.HC, L.F, Hp, ws, stream));
  {
    ProfScope ps("out_sd", stream);
    k_out_sd<<<(unsigned)((L.n * H_ + 255) / 256), 256, 0, stream>>>(Hp, L.n, H_, C_, p->a_src, p->a_dst, S, D);
  }
  {
    ProfScope ps("out_el", stream);
    k_out_el<<<(unsigned)((L.n * H_ + 255) / 256), 256, 0, stream>>>(g, H_, S, D, p->neg_slope, epre, el);
  }
  M_TRY_CUDA(launch_edge_softmax(g, H_, el, m, den, alpha, stream));
  {
    ProfScope ps("out_agg", stream);
    const size_t smem = 8 * sizeof(float) * (size_t)L.HC;
    k_out_agg<<<grid_1d(L.n, 8), 256, smem, stream>>>(g, H_, C_, alpha, Hp, p->bias, logits);
  }
  M_TRY_CUDA(cudaGetLastError());
  return TANGO_OK;
}

tango_status tango_gat_out_bwd(const tango_graph* G, const tango_gat_out_params* p, void* ctx, size_t ctx_bytes,
                               const float* H, const float* dlogits, float* dH, float* dW, float* da_src,
                               float* da_dst, float* dbias, cudaStream_t stream) {
  tango_status s = check_out(G, p);
  if (s != TANGO_OK) return s;
  OutLayout L;
  out_layout(G, p, &L);
  if (!ctx || ctx_bytes < L.total) return TANGO_ERR_INVALID_ARG;
  if (!dW || !da_src || !da_dst || !dbias) return TANGO_ERR_INVALID_ARG;
  if (L.n > 0 && (!H || !dlogits)) return TANGO_ERR_INVALID_ARG;
  char* c = static_cast<char*>(ctx);
  float* Hp = reinterpret_cast<float*>(c + L.off_Hp);
  float* epre = reinterpret_cast<float*>(c + L.off_epre);
  float* alpha = reinterpret_cast<float*>(c + L.off_alpha);
  float* Gm = reinterpret_cast<float*>(c + L.off_G);
  float* dalpha = reinterpret_cast<float*>(c + L.off_dalpha);
  float* dEp = reinterpret_cast<float*>(c + L.off_dEp);
  float* P = reinterpret_cast<float*>(c + L.off_P);
  float* dD = reinterpret_cast<float*>(c + L.off_dD);
  float* dS = reinterpret_cast<float*>(c + L.off_dS);
  float* dHp = reinterpret_cast<float*>(c + L.off_dHp);
  float* ws = reinterpret_cast<float*>(c + L.off_ws);
  const GraphDev g = dev_graph(G);
  const int H_ = (int)L.H, C_ = (int)L.C;
  M_TRY_CUDA(cudaMemsetAsync(da_src, 0, sizeof(float) * L.HC, stream));
  M_TRY_CUDA(cudaMemsetAsync(da_dst, 0, sizeof(float) * L.HC, stream));
  // ∂b = Σᶜ_v ∂logits (R33)
  M_TRY_CUDA(launch_colsum<0>(dlogits, nullptr, L.n, L.C, dbias, ws, nullptr, nullptr, stream));
  if (L.n == 0) {
    M_TRY_CUDA(cudaMemsetAsync(dW, 0, sizeof(float) * L.F * L.HC, stream));
    return TANGO_OK;
  }
  {
    ProfScope ps("out_g", stream);
    k_out_g<<<grid_1d(L.n * L.C), 256, 0, stream>>>(dlogits, L.n * L.C, (float)H_, Gm);
  }
  {
    ProfScope ps("out_dalpha", stream);
    k_out_dalpha<<<(unsigned)((L.n * H_ + 255) / 256), 256, 0, stream>>>(g, H_, C_, Gm, Hp, dalpha);
  }
  M_TRY_CUDA(launch_softmax_bwd(g, H_, alpha, dalpha, epre, p->neg_slope, P, dEp, stream));
  M_TRY_CUDA(launch_edge_sum(g, 0, H_, dEp, dD, stream));
  M_TRY_CUDA(launch_edge_sum(g, 1, H_, dEp, dS, stream));
  {
    ProfScope ps("out_dhp", stream);
    k_out_dhp<<<grid_1d(L.n, 8), 256, 0, stream>>>(g, H_, C_, alpha, Gm, dS, dD, p->a_src, p->a_dst, dHp);
  }
  {
    ProfScope ps("out_da", stream);
    k_out_da<<<num_sms() * 2, 256, 0, stream>>>(Hp, L.n, H_, C_, dS, dD, da_src, da_dst);
  }
  // ①′ ∂H = ∂H′·Wᵀ (K = H·C), ∂W = Hᵀ·∂H′ (K = n, chunked) (R33)
  if (dH) M_TRY_CUDA(launch_sgemm(dHp, L.HC, false, p->W, L.HC, true, L.n, L.F, L.HC, dH, ws, stream));
  M_TRY_CUDA(launch_sgemm(H, L.F, true, dHp, L.HC, false, L.F, L.HC, L.n, dW, ws, stream));
  return TANGO_OK;
}

tango_status tango_gat_out_ctx_get_view(const tango_graph* G, const tango_gat_out_params* p, void* ctx,
                                        tango_gat_out_ctx_view* view) {
  tango_status s = check_out(G, p);
  if (s != TANGO_OK) return s;
  if (!ctx || !view) return TANGO_ERR_INVALID_ARG;
  OutLayout L;
  out_layout(G, p, &L);
  char* c = static_cast<char*>(ctx);
  view->Hp = reinterpret_cast<float*>(c + L.off_Hp);
  view->S = reinterpret_cast<float*>(c + L.off_S);
  view->D = reinterpret_cast<float*>(c + L.off_D);
  view->e_pre = reinterpret_cast<float*>(c + L.off_epre);
  view->alpha = reinterpret_cast<float*>(c + L.off_alpha);
  view->m = reinterpret_cast<float*>(c + L.off_m);
  view->den = reinterpret_cast<float*>(c + L.off_den);
  view->G = reinterpret_cast<float*>(c + L.off_G);
  view->dalpha = reinterpret_cast<float*>(c + L.off_dalpha);
  view->dE_pre = reinterpret_cast<float*>(c + L.off_dEp);
  view->P = reinterpret_cast<float*>(c + L.off_P);
  view->dD = reinterpret_cast<float*>(c + L.off_dD);
  view->dS = reinterpret_cast<float*>(c + L.off_dS);
  view->dHp = reinterpret_cast<float*>(c + L.off_dHp);
  return TANGO_OK;
}

}  // extern "C"
