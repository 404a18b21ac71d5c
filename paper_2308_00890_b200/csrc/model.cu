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

// Large-tile variant: BM = 128 rows x BN (128 or 160) columns per block, BK = 8, 256 threads as
// 16 x 16 with 8 x (BN/16) outputs each; double-buffered shared memory (one barrier per k-tile),
// 16-B global loads where the operand is aligned and the tile in bounds.  Same per-output chain.
constexpr int SG2_BM = 128;

template <bool TA, bool TB, int BN, int SG2_BK = (BN == 128 ? 16 : 8)>
__global__ void __launch_bounds__(256, 2) k_sgemm2(const float* __restrict__ A, int64_t lda, const float* __restrict__ B,
                                                   int64_t ldb, int64_t M, int64_t N, int64_t K,
                                                   float* __restrict__ C) {
  constexpr int BM = SG2_BM, BK = SG2_BK, TN = BN / 16, TM = BM / 16;
  constexpr int A4 = BM * BK / 4, B4 = BN * BK / 4;          // float4 slots per tile
  __shared__ __align__(16) float As[2][BK][BM];
  __shared__ __align__(16) float Bs[2][BK][BN];
  const int t = threadIdx.x;
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
  const int64_t kbeg = (int64_t)blockIdx.z * kCK;
  const int64_t kend = min(K, kbeg + kCK);
  float* Cz = C + (int64_t)blockIdx.z * M * N;
  const bool avec = ((lda & 3) == 0) && ((reinterpret_cast<uintptr_t>(A) & 15) == 0);
  const bool bvec = ((ldb & 3) == 0) && ((reinterpret_cast<uintptr_t>(B) & 15) == 0);

  float4 ra[(A4 + 255) / 256], rb[(B4 + 255) / 256];
  // slot i of A: TA (A[k][m]): k = i / (BM/4), m4 = i % (BM/4);  !TA (A[m][k]): m = i / (BK/4), k4 = i % (BK/4)
  const bool mn_in = avec && bvec && m0 + BM <= M && n0 + BN <= N;
  auto load = [&](int64_t k0) {
    if (mn_in && k0 + BK <= kend) {   // interior tile: unpredicated 16-B loads
#pragma unroll
      for (int r = 0; r < (A4 + 255) / 256; ++r) {
        const int i = t + 256 * r;
        if (i < A4) {
          if (TA) ra[r] = __ldg(reinterpret_cast<const float4*>(A + (k0 + i / (BM / 4)) * lda + m0 + (i % (BM / 4)) * 4));
          else ra[r] = __ldg(reinterpret_cast<const float4*>(A + (m0 + i / (BK / 4)) * lda + k0 + (i % (BK / 4)) * 4));
        }
      }
#pragma unroll
      for (int r = 0; r < (B4 + 255) / 256; ++r) {
        const int i = t + 256 * r;
        if (i < B4) {
          if (!TB) rb[r] = __ldg(reinterpret_cast<const float4*>(B + (k0 + i / (BN / 4)) * ldb + n0 + (i % (BN / 4)) * 4));
          else rb[r] = __ldg(reinterpret_cast<const float4*>(B + (n0 + i / (BK / 4)) * ldb + k0 + (i % (BK / 4)) * 4));
        }
      }
      return;
    }
#pragma unroll
    for (int r = 0; r < (A4 + 255) / 256; ++r) {
      const int i = t + 256 * r;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (i < A4) {
        if (TA) {
          const int kk = i / (BM / 4), mm = (i % (BM / 4)) * 4;
          const int64_t gk = k0 + kk, gm = m0 + mm;
          if (gk < kend) {
            const float* p = A + gk * lda + gm;
            if (avec && gm + 3 < M) v = __ldg(reinterpret_cast<const float4*>(p));
            else {
              v.x = gm < M ? __ldg(p) : 0.f; v.y = gm + 1 < M ? __ldg(p + 1) : 0.f;
              v.z = gm + 2 < M ? __ldg(p + 2) : 0.f; v.w = gm + 3 < M ? __ldg(p + 3) : 0.f;
            }
          }
        } else {
          const int mm = i / (BK / 4), kk = (i % (BK / 4)) * 4;
          const int64_t gm = m0 + mm, gk = k0 + kk;
          if (gm < M) {
            const float* p = A + gm * lda + gk;
            if (avec && gk + 3 < kend) v = __ldg(reinterpret_cast<const float4*>(p));
            else {
              v.x = gk < kend ? __ldg(p) : 0.f; v.y = gk + 1 < kend ? __ldg(p + 1) : 0.f;
              v.z = gk + 2 < kend ? __ldg(p + 2) : 0.f; v.w = gk + 3 < kend ? __ldg(p + 3) : 0.f;
            }
          }
        }
      }
      ra[r] = v;
    }
#pragma unroll
    for (int r = 0; r < (B4 + 255) / 256; ++r) {
      const int i = t + 256 * r;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (i < B4) {
        if (!TB) {   // B[k][n]
          const int kk = i / (BN / 4), nn = (i % (BN / 4)) * 4;
          const int64_t gk = k0 + kk, gn = n0 + nn;
          if (gk < kend) {
            const float* p = B + gk * ldb + gn;
            if (bvec && gn + 3 < N) v = __ldg(reinterpret_cast<const float4*>(p));
            else {
              v.x = gn < N ? __ldg(p) : 0.f; v.y = gn + 1 < N ? __ldg(p + 1) : 0.f;
              v.z = gn + 2 < N ? __ldg(p + 2) : 0.f; v.w = gn + 3 < N ? __ldg(p + 3) : 0.f;
            }
          }
        } else {     // B[n][k]
          const int nn = i / (BK / 4), kk = (i % (BK / 4)) * 4;
          const int64_t gn = n0 + nn, gk = k0 + kk;
          if (gn < N) {
            const float* p = B + gn * ldb + gk;
            if (bvec && gk + 3 < kend) v = __ldg(reinterpret_cast<const float4*>(p));
            else {
              v.x = gk < kend ? __ldg(p) : 0.f; v.y = gk + 1 < kend ? __ldg(p + 1) : 0.f;
              v.z = gk + 2 < kend ? __ldg(p + 2) : 0.f; v.w = gk + 3 < kend ? __ldg(p + 3) : 0.f;
            }
          }
        }
      }
      rb[r] = v;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int r = 0; r < (A4 + 255) / 256; ++r) {
      const int i = t + 256 * r;
      if (i >= A4) continue;
      if (TA) {
        const int kk = i / (BM / 4), mm = (i % (BM / 4)) * 4;
        *reinterpret_cast<float4*>(&As[buf][kk][mm]) = ra[r];
      } else {
        const int mm = i / (BK / 4), kk = (i % (BK / 4)) * 4;
        As[buf][kk][mm] = ra[r].x; As[buf][kk + 1][mm] = ra[r].y;
        As[buf][kk + 2][mm] = ra[r].z; As[buf][kk + 3][mm] = ra[r].w;
      }
    }
#pragma unroll
    for (int r = 0; r < (B4 + 255) / 256; ++r) {
      const int i = t + 256 * r;
      if (i >= B4) continue;
      if (!TB) {
        const int kk = i / (BN / 4), nn = (i % (BN / 4)) * 4;
        *reinterpret_cast<float4*>(&Bs[buf][kk][nn]) = rb[r];
      } else {
        const int nn = i / (BK / 4), kk = (i % (BK / 4)) * 4;
        Bs[buf][kk][nn] = rb[r].x; Bs[buf][kk + 1][nn] = rb[r].y;
        Bs[buf][kk + 2][nn] = rb[r].z; Bs[buf][kk + 3][nn] = rb[r].w;
      }
    }
  };

  const int ty = t / 16, tx = t % 16;
  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.0f;

  int buf = 0;
  if (kbeg < kend) {
    load(kbeg);
    store(0);
  }
  __syncthreads();
  for (int64_t k0 = kbeg; k0 < kend; k0 += BK) {
    const bool more = k0 + BK < kend;
    if (more) load(k0 + BK);
    const int kmax = (kend - k0 < BK) ? (int)(kend - k0) : BK;
    if (kmax == BK) {
#pragma unroll
      for (int kk = 0; kk < BK; ++kk) {
        float a[TM], b[TN];
#pragma unroll
        for (int i = 0; i < TM; i += 4) {
          const float4 v = *reinterpret_cast<const float4*>(&As[buf][kk][ty * TM + i]);
          a[i] = v.x; a[i + 1] = v.y; a[i + 2] = v.z; a[i + 3] = v.w;
        }
#pragma unroll
        for (int j = 0; j < TN; j += 2) {
          const float2 v = *reinterpret_cast<const float2*>(&Bs[buf][kk][tx * TN + j]);
          b[j] = v.x; b[j + 1] = v.y;
        }
        // packed FFMA2 (fma.rn.f32x2: two IEEE fmas per instruction, the 3-register FFMA issues at
        // half rate): acc[i][j..j+1] = fma({a_i, a_i}, {b_j, b_j+1}, acc[i][j..j+1]) — the same
        // per-output chain as the scalar form
#pragma unroll
        for (int i = 0; i < TM; ++i) {
          uint64_t a2;
          asm("mov.b64 %0, {%1, %1};" : "=l"(a2) : "f"(a[i]));
#pragma unroll
          for (int j = 0; j < TN; j += 2) {
            uint64_t b2, c2;
            asm("mov.b64 %0, {%1, %2};" : "=l"(b2) : "f"(b[j]), "f"(b[j + 1]));
            asm("mov.b64 %0, {%1, %2};" : "=l"(c2) : "f"(acc[i][j]), "f"(acc[i][j + 1]));
            asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(c2) : "l"(a2), "l"(b2));
            asm("mov.b64 {%0, %1}, %2;" : "=f"(acc[i][j]), "=f"(acc[i][j + 1]) : "l"(c2));
          }
        }
      }
    } else {
      for (int kk = 0; kk < kmax; ++kk) {
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j)
            acc[i][j] = __fmaf_rn(As[buf][kk][ty * TM + i], Bs[buf][kk][tx * TN + j], acc[i][j]);
      }
    }
    if (more) store(buf ^ 1);
    __syncthreads();
    buf ^= 1;
  }
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int64_t gm = m0 + ty * TM + i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int64_t gn = n0 + tx * TN + j;
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
  if (M < 64) {
    dim3 grid((unsigned)((N + SG_BN - 1) / SG_BN), (unsigned)((M + SG_BM - 1) / SG_BM), (unsigned)nc);
    ProfScope ps("sgemm", st);
    if (!ta && !tb) k_sgemm<false, false><<<grid, 256, 0, st>>>(A, lda, B, ldb, M, N, K, dst);
    else if (ta && !tb) k_sgemm<true, false><<<grid, 256, 0, st>>>(A, lda, B, ldb, M, N, K, dst);
    else if (!ta && tb) k_sgemm<false, true><<<grid, 256, 0, st>>>(A, lda, B, ldb, M, N, K, dst);
    else k_sgemm<true, true><<<grid, 256, 0, st>>>(A, lda, B, ldb, M, N, K, dst);
  } else {
    // 160-wide column tiles when they cover N with less waste than 128-wide ones
    const int64_t w128 = (N + 127) / 128 * 128, w160 = (N + 159) / 160 * 160;
    const bool n160 = w160 < w128;
    const int bn = n160 ? 160 : 128;
    dim3 grid((unsigned)((N + bn - 1) / bn), (unsigned)((M + SG2_BM - 1) / SG2_BM), (unsigned)nc);
    ProfScope ps("sgemm", st);
#define SG2(TA_, TB_)                                                                              \
    if (n160) k_sgemm2<TA_, TB_, 160><<<grid, 256, 0, st>>>(A, lda, B, ldb, M, N, K, dst);         \
    else k_sgemm2<TA_, TB_, 128><<<grid, 256, 0, st>>>(A, lda, B, ldb, M, N, K, dst);
    if (!ta && !tb) { SG2(false, false) }
    else if (ta && !tb) { SG2(true, false) }
    else if (!ta && tb) { SG2(false, true) }
    else { SG2(true, true) }
#undef SG2
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
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if ((cols & 3) == 0 && ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15) == 0) {
    // 16-B path: 4 consecutive columns of one row per step, streaming loads / stores
    const int64_t n4 = n >> 2;
    for (int64_t i = tid; i < n4; i += stride) {
      const float4 v = __ldcs(reinterpret_cast<const float4*>(x) + i);
      const int64_t j = (i << 2) % cols;
      float4 a;
      a.x = __fadd_rn(v.x, __ldg(b + j));
      a.y = __fadd_rn(v.y, __ldg(b + j + 1));
      a.z = __fadd_rn(v.z, __ldg(b + j + 2));
      a.w = __fadd_rn(v.w, __ldg(b + j + 3));
      a.x = a.x > 0.0f ? a.x : 0.0f; a.y = a.y > 0.0f ? a.y : 0.0f;
      a.z = a.z > 0.0f ? a.z : 0.0f; a.w = a.w > 0.0f ? a.w : 0.0f;
      reinterpret_cast<float4*>(y)[i] = a;
      mx = fmaxf(mx, fmaxf(fmaxf(a.x, a.y), fmaxf(a.z, a.w)));
    }
  } else {
    for (int64_t i = tid; i < n; i += stride) {
      const float v = __fadd_rn(__ldg(x + i), __ldg(b + i % cols));
      const float a = v > 0.0f ? v : 0.0f;
      y[i] = a;
      mx = fmaxf(mx, a);
    }
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
                                              int64_t rows, int C, float n_lab,
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

// The final layer's per-row chunked sums (R14) are split by row weight: a LIGHT row (degree
// <= C_E) is one chunk and is summed by one thread / one warp sequentially; a HEAVY row (degree >
// C_E) is handled by one block whose threads compute the chunk partials in parallel and fold them
// left to right (the same value the sequential definition gives).  The heavy-row lists of the
// in- and out-CSR and the in-CSR destination of every edge come from k_out_plan.
constexpr int OUT_MAXHC = 1024;
constexpr int OUT_PART = 4096;   // shared-memory partials per pass of a heavy-row block

__global__ void __launch_bounds__(256) k_out_plan(GraphDev g, int32_t* __restrict__ in_dst, int32_t* __restrict__ hin,
                                                  int32_t* __restrict__ hout, int32_t* counts) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t v = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); v < g.n_local; v += nw) {
    const int64_t b = g.in_ptr[v], e1 = g.in_ptr[v + 1];
    for (int64_t e = b + lane; e < e1; e += 32) in_dst[e] = (int32_t)v;
    if (lane == 0) {
      if (e1 - b > g.chunk) hin[atomicAdd(counts + 0, 1)] = (int32_t)v;
      if (g.out_ptr[v + 1] - g.out_ptr[v] > g.chunk) hout[atomicAdd(counts + 1, 1)] = (int32_t)v;
    }
  }
}

// ③ in FP32: e_pre = S[u] + D[v], el = LeakyReLU(e_pre); thread per edge (all heads)
__global__ void k_out_el(int64_t e_in, int heads, const int32_t* __restrict__ in_src,
                         const int32_t* __restrict__ in_dst, const float* __restrict__ S, const float* __restrict__ D,
                         float slope, float* __restrict__ e_pre, float* __restrict__ el) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < e_in; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t u = in_src[e], v = in_dst[e];
    for (int h = 0; h < heads; ++h) {
      const float x = __fadd_rn(S[u * heads + h], D[v * heads + h]);
      e_pre[e * heads + h] = x;
      el[e * heads + h] = x > 0.0f ? x : __fmul_rn(x, slope);
    }
  }
}

// Chunked sums of one heavy row inside a block: for every head h, total_h = Σᶜ over the row's
// list positions i in [0, len) of the accumulation acc = op(acc, i, h) (chunks of `chunk`
// positions, partials folded left to right).  Results in out_h[h] (shared).  All threads call it.
template <class Op>
__device__ void heavy_row_sums(int64_t len, int chunk, int heads, Op op, float* part, float* out_h) {
  const int64_t nch = (len + chunk - 1) / chunk;
  const int grp = OUT_PART / heads;
  float total = 0.0f;
  for (int64_t c0 = 0; c0 < nch; c0 += grp) {
    const int64_t nc = min((int64_t)grp, nch - c0);
    for (int64_t it = threadIdx.x; it < nc * heads; it += blockDim.x) {
      const int64_t c = c0 + it / heads;
      const int h = (int)(it % heads);
      const int64_t i0 = c * chunk, i1 = min(len, i0 + chunk);
      float acc = 0.0f;
#pragma unroll 8
      for (int64_t i = i0; i < i1; ++i) acc = op(acc, i, h);
      part[it] = acc;
    }
    __syncthreads();
    if (threadIdx.x < heads) {
      for (int64_t c = 0; c < nc; ++c) {
        const float p = part[c * heads + threadIdx.x];
        total = (c0 + c == 0) ? p : __fadd_rn(total, p);
      }
    }
    __syncthreads();
  }
  if (threadIdx.x < heads) out_h[threadIdx.x] = total;
  __syncthreads();
}

__device__ __forceinline__ float block_max(float v, float* red) {
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  float r = -INFINITY;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r = fmaxf(r, red[w]);
  __syncthreads();
  return r;
}

// ④ edge softmax, light rows: thread per (row, head), one sequential chunk
__global__ void k_out_softmax_light(GraphDev g, int heads, const float* __restrict__ el, float* __restrict__ m,
                                    float* __restrict__ den, float* __restrict__ alpha) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (tid >= g.n_local * heads) return;
  const int64_t v = tid / heads;
  const int h = (int)(tid % heads);
  const int64_t b = g.in_ptr[v], e1 = g.in_ptr[v + 1];
  if (e1 - b > g.chunk) return;
  float mx = -INFINITY;
  for (int64_t e = b; e < e1; ++e) mx = fmaxf(mx, el[e * heads + h]);
  if (e1 == b) mx = 0.0f;
  float dn = 0.0f;
  for (int64_t e = b; e < e1; ++e) dn = __fadd_rn(dn, exp_p(__fsub_rn(el[e * heads + h], mx)));
  for (int64_t e = b; e < e1; ++e) alpha[e * heads + h] = __fdiv_rn(exp_p(__fsub_rn(el[e * heads + h], mx)), dn);
  m[tid] = mx;
  den[tid] = dn;
}

// ④ edge softmax, heavy rows: block per row
__global__ void __launch_bounds__(256) k_out_softmax_heavy(GraphDev g, int heads, const int32_t* __restrict__ hin,
                                                           const int32_t* counts, const float* __restrict__ el,
                                                           float* __restrict__ m, float* __restrict__ den,
                                                           float* __restrict__ alpha) {
  __shared__ float part[OUT_PART];
  __shared__ float red[32];
  __shared__ float mh[32], dh[32];
  for (int i = blockIdx.x; i < counts[0]; i += gridDim.x) {
    const int64_t v = hin[i];
    const int64_t b = g.in_ptr[v], len = g.in_ptr[v + 1] - b;
    for (int h = 0; h < heads; ++h) {
      float mx = -INFINITY;
      for (int64_t k = threadIdx.x; k < len; k += blockDim.x) mx = fmaxf(mx, el[(b + k) * heads + h]);
      mx = block_max(mx, red);
      if (threadIdx.x == 0) mh[h] = mx;
    }
    __syncthreads();
    heavy_row_sums(len, g.chunk, heads,
                   [&](float acc, int64_t k, int h) {
                     return __fadd_rn(acc, exp_p(__fsub_rn(el[(b + k) * heads + h], mh[h])));
                   }, part, dh);
    for (int64_t it = threadIdx.x; it < len * heads; it += blockDim.x) {
      const int h = (int)(it % heads);
      const int64_t e = b + it / heads;
      alpha[e * heads + h] = __fdiv_rn(exp_p(__fsub_rn(el[e * heads + h], mh[h])), dh[h]);
    }
    if (threadIdx.x < heads) {
      m[v * heads + threadIdx.x] = mh[threadIdx.x];
      den[v * heads + threadIdx.x] = dh[threadIdx.x];
    }
    __syncthreads();
  }
}

// Column sums of rows gathered along a CSR row: out[v, j] = Σᶜ over the row's list positions p of
// fmaf(w(p, h(j)), X[r(p), c(j)]) with h = j / C, and c = j (IN: X = H′ rows of width HC, weights
// α[e,h], r = in_src) or c = j % C (OUT: X = G rows of width C, weights α[out_eid,h], r = out_dst).
// alpha == nullptr: unweighted, acc + X (the FP32 GCN aggregation, heads = 1).
template <bool OUT>
struct GatherRow {
  const int64_t* ptr; const int32_t* idx; const int32_t* eid;
  const float* alpha; const float* X; int heads, C, HC, ldx;
  __device__ __forceinline__ int64_t edge(int64_t p) const { return OUT ? (int64_t)eid[p] : p; }
  __device__ __forceinline__ int col(int j) const { return OUT ? j % C : j; }
};

// light rows: warp per row, NC columns per lane (j = lane + 32 t)
template <bool OUT, bool WGT, int NC>
__global__ void __launch_bounds__(256) k_out_gather_light(GatherRow<OUT> R, int64_t n, int chunk,
                                                          float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  int h[NC], c[NC];
  bool ok[NC];
#pragma unroll
  for (int t = 0; t < NC; ++t) {
    const int j = lane + 32 * t;
    ok[t] = j < R.HC;
    h[t] = ok[t] ? j / R.C : 0;
    c[t] = ok[t] ? R.col(j) : 0;
  }
  for (int64_t v = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); v < n; v += nw) {
    const int64_t b = R.ptr[v], e1 = R.ptr[v + 1];
    if (e1 - b > chunk) continue;
    float acc[NC];
#pragma unroll
    for (int t = 0; t < NC; ++t) acc[t] = 0.0f;
    // two list entries per step, all loads of both issued before either is accumulated
    int64_t p = b;
    for (; p + 1 < e1; p += 2) {
      const int64_t ea = R.edge(p), eb = R.edge(p + 1);
      const float* xa = R.X + (int64_t)__ldg(R.idx + p) * R.ldx;
      const float* xb = R.X + (int64_t)__ldg(R.idx + p + 1) * R.ldx;
      float va[NC], vb[NC], wa[NC], wb[NC];
#pragma unroll
      for (int t = 0; t < NC; ++t) {
        va[t] = ok[t] ? __ldg(xa + c[t]) : 0.0f;
        vb[t] = ok[t] ? __ldg(xb + c[t]) : 0.0f;
        if constexpr (WGT) {
          wa[t] = ok[t] ? __ldg(R.alpha + ea * R.heads + h[t]) : 0.0f;
          wb[t] = ok[t] ? __ldg(R.alpha + eb * R.heads + h[t]) : 0.0f;
        }
      }
#pragma unroll
      for (int t = 0; t < NC; ++t) {
        if constexpr (WGT) {
          acc[t] = __fmaf_rn(wa[t], va[t], acc[t]);
          acc[t] = __fmaf_rn(wb[t], vb[t], acc[t]);
        } else {
          acc[t] = __fadd_rn(acc[t], va[t]);
          acc[t] = __fadd_rn(acc[t], vb[t]);
        }
      }
    }
    if (p < e1) {
      const int64_t e = R.edge(p);
      const float* xr = R.X + (int64_t)__ldg(R.idx + p) * R.ldx;
#pragma unroll
      for (int t = 0; t < NC; ++t)
        if (ok[t]) {
          if constexpr (WGT) acc[t] = __fmaf_rn(__ldg(R.alpha + e * R.heads + h[t]), __ldg(xr + c[t]), acc[t]);
          else acc[t] = __fadd_rn(acc[t], __ldg(xr + c[t]));
        }
    }
#pragma unroll
    for (int t = 0; t < NC; ++t)
      if (ok[t]) out[v * R.HC + lane + 32 * t] = acc[t];
  }
}

// heavy rows: block per (row, 32-column slab); warps compute chunk partials, lane = column
template <bool OUT>
__global__ void __launch_bounds__(256) k_out_gather_heavy(GatherRow<OUT> R, const int32_t* __restrict__ hrows,
                                                          const int32_t* count, int chunk, float* __restrict__ out) {
  constexpr int PASS = 64;
  __shared__ float part[PASS][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const int nslab = (R.HC + 31) / 32;
  for (int64_t item = blockIdx.x; item < (int64_t)count[0] * nslab; item += gridDim.x) {
    const int64_t v = hrows[item / nslab];
    const int j = (int)(item % nslab) * 32 + lane;
    const bool ok = j < R.HC;
    const int h = ok ? j / R.C : 0, c = ok ? R.col(j) : 0;
    const int64_t b = R.ptr[v], len = R.ptr[v + 1] - b;
    const int64_t nch = (len + chunk - 1) / chunk;
    float total = 0.0f;
    for (int64_t c0 = 0; c0 < nch; c0 += PASS) {
      const int64_t nc = min((int64_t)PASS, nch - c0);
      for (int64_t k = warp; k < nc; k += nwarp) {
        const int64_t p0 = b + (c0 + k) * chunk, p1 = min(b + len, p0 + chunk);
        float acc = 0.0f;
        if (ok) {
#pragma unroll 4
          for (int64_t p = p0; p < p1; ++p) {
            const float x = R.X[(int64_t)R.idx[p] * R.ldx + c];
            acc = R.alpha ? __fmaf_rn(R.alpha[R.edge(p) * R.heads + h], x, acc) : __fadd_rn(acc, x);
          }
        }
        part[k][lane] = acc;
      }
      __syncthreads();
      if (warp == 0)
        for (int64_t k = 0; k < nc; ++k) total = (c0 + k == 0) ? part[k][lane] : __fadd_rn(total, part[k][lane]);
      __syncthreads();
    }
    if (warp == 0 && ok) out[v * R.HC + j] = total;
  }
}

template <bool OUT>
static cudaError_t launch_gather(const GatherRow<OUT>& R, int64_t n, int chunk, const int32_t* hrows,
                                 const int32_t* count, float* out, cudaStream_t st, const char* light_name = nullptr,
                                 const char* heavy_name = nullptr) {
  const int nc = (R.HC + 31) / 32;
  const int grid = grid_1d(n, 8);
  {
    ProfScope ps(light_name ? light_name : (OUT ? "out_dhp_light" : "out_agg_light"), st);
#define GL(NC_)                                                                                   \
    if (R.alpha) k_out_gather_light<OUT, true, NC_><<<grid, 256, 0, st>>>(R, n, chunk, out);       \
    else k_out_gather_light<OUT, false, NC_><<<grid, 256, 0, st>>>(R, n, chunk, out);
    switch (nc) {
      case 1: GL(1) break;
      case 2: GL(2) break;
      case 3: GL(3) break;
      case 4: GL(4) break;
      case 5: GL(5) break;
      case 6: GL(6) break;
      case 7: GL(7) break;
      case 8: GL(8) break;
      default: GL(32) break;
    }
#undef GL
  }
  {
    ProfScope ps(heavy_name ? heavy_name : (OUT ? "out_dhp_heavy" : "out_agg_heavy"), st);
    k_out_gather_heavy<OUT><<<num_sms() * 4, 256, 0, st>>>(R, hrows, count, chunk, out);
  }
  return cudaGetLastError();
}

// logits[v,c] = ((Σ_h agg[v,h,c], head order) / heads) + bias[c]
__global__ void k_out_logits(const float* __restrict__ agg, int64_t n, int heads, int C, const float* __restrict__ bias,
                             float* __restrict__ logits) {
  const int HC = heads * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * C; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = i / C;
    const int c = (int)(i % C);
    float t = agg[v * HC + c];
    for (int h = 1; h < heads; ++h) t = __fadd_rn(t, agg[v * HC + h * C + c]);
    logits[i] = __fadd_rn(__fdiv_rn(t, (float)heads), bias[c]);
  }
}

// Wt[j][f] = W[f][j] (so that ∂H = ∂H′·Wᵀ reads its B operand row-major: 16-B shared stores)
__global__ void k_transpose(const float* __restrict__ W, int64_t rows, int64_t cols, float* __restrict__ Wt) {
  __shared__ float tile[32][33];
  const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t r = r0 + i, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[i][threadIdx.x] = W[r * cols + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t c = c0 + i, r = r0 + threadIdx.x;
    if (r < rows && c < cols) Wt[c * rows + r] = tile[threadIdx.x][i];
  }
}

// G = ∂logits / heads (the gradient reaching every head's aggregation)
__global__ void k_out_g(const float* __restrict__ dz, int64_t count, float heads, float* __restrict__ G) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    G[i] = __fdiv_rn(dz[i], heads);
}

// ⑤″ in FP32: ∂α[e,h] = Σ_c fmaf(G[v,c], H′[u,h,c]) sequential in c; thread per (edge, head)
__global__ void k_out_dalpha(int64_t e_in, int heads, int C, const int32_t* __restrict__ in_src,
                             const int32_t* __restrict__ in_dst, const float* __restrict__ G,
                             const float* __restrict__ Hp, float* __restrict__ dalpha) {
  const int HC = heads * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < e_in * heads;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i / heads;
    const int h = (int)(i % heads);
    const float* gv = G + (int64_t)in_dst[e] * C;
    const float* hu = Hp + (int64_t)in_src[e] * HC + (int64_t)h * C;
    float acc = 0.0f;
    int c = 0;
    if ((C & 3) == 0) {   // rows 16-B aligned: 4 terms per load, still one sequential chain over c
#pragma unroll 2
      for (; c < C; c += 4) {
        const float4 gq = __ldg(reinterpret_cast<const float4*>(gv + c));
        const float4 hq = __ldg(reinterpret_cast<const float4*>(hu + c));
        acc = __fmaf_rn(gq.x, hq.x, acc);
        acc = __fmaf_rn(gq.y, hq.y, acc);
        acc = __fmaf_rn(gq.z, hq.z, acc);
        acc = __fmaf_rn(gq.w, hq.w, acc);
      }
    }
    for (; c < C; ++c) acc = __fmaf_rn(gv[c], hu[c], acc);
    dalpha[i] = acc;
  }
}

// ④′ + LeakyReLU′ + ③″ (∂D over in-edges), light rows: thread per (row, head)
__global__ void k_out_sbwd_light(GraphDev g, int heads, const float* __restrict__ alpha,
                                 const float* __restrict__ dalpha, const float* __restrict__ e_pre, float slope,
                                 float* __restrict__ P, float* __restrict__ dEp, float* __restrict__ dD) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (tid >= g.n_local * heads) return;
  const int64_t v = tid / heads;
  const int h = (int)(tid % heads);
  const int64_t b = g.in_ptr[v], e1 = g.in_ptr[v + 1];
  if (e1 - b > g.chunk) return;
  float p = 0.0f;
  for (int64_t e = b; e < e1; ++e) p = __fmaf_rn(dalpha[e * heads + h], alpha[e * heads + h], p);
  float dd = 0.0f;
  for (int64_t e = b; e < e1; ++e) {
    const int64_t k = e * heads + h;
    const float dE = __fmul_rn(alpha[k], __fsub_rn(dalpha[k], p));
    const float x = e_pre[k] > 0.0f ? dE : __fmul_rn(dE, slope);
    dEp[k] = x;
    dd = __fadd_rn(dd, x);
  }
  P[tid] = p;
  dD[tid] = dd;
}

__global__ void __launch_bounds__(256) k_out_sbwd_heavy(GraphDev g, int heads, const int32_t* __restrict__ hin,
                                                        const int32_t* counts, const float* __restrict__ alpha,
                                                        const float* __restrict__ dalpha,
                                                        const float* __restrict__ e_pre, float slope,
                                                        float* __restrict__ P, float* __restrict__ dEp,
                                                        float* __restrict__ dD) {
  __shared__ float part[OUT_PART];
  __shared__ float ph[32], dh[32];
  for (int i = blockIdx.x; i < counts[0]; i += gridDim.x) {
    const int64_t v = hin[i];
    const int64_t b = g.in_ptr[v], len = g.in_ptr[v + 1] - b;
    heavy_row_sums(len, g.chunk, heads,
                   [&](float acc, int64_t k, int h) {
                     return __fmaf_rn(dalpha[(b + k) * heads + h], alpha[(b + k) * heads + h], acc);
                   }, part, ph);
    for (int64_t it = threadIdx.x; it < len * heads; it += blockDim.x) {
      const int64_t k = b * heads + it;
      const int h = (int)(it % heads);
      const float dE = __fmul_rn(alpha[k], __fsub_rn(dalpha[k], ph[h]));
      dEp[k] = e_pre[k] > 0.0f ? dE : __fmul_rn(dE, slope);
    }
    __syncthreads();
    heavy_row_sums(len, g.chunk, heads,
                   [&](float acc, int64_t k, int h) { return __fadd_rn(acc, dEp[(b + k) * heads + h]); }, part, dh);
    if (threadIdx.x < heads) {
      P[v * heads + threadIdx.x] = ph[threadIdx.x];
      dD[v * heads + threadIdx.x] = dh[threadIdx.x];
    }
    __syncthreads();
  }
}

// ③′ ∂S over out-edges (out order, edge values by out_eid): light thread per (row, head), heavy block per row
__global__ void k_out_dS_light(GraphDev g, int heads, const float* __restrict__ dEp, float* __restrict__ dS) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (tid >= g.n_local * heads) return;
  const int64_t u = tid / heads;
  const int h = (int)(tid % heads);
  const int64_t b = g.out_ptr[u], e1 = g.out_ptr[u + 1];
  if (e1 - b > g.chunk) return;
  float s = 0.0f;
  for (int64_t p = b; p < e1; ++p) s = __fadd_rn(s, dEp[(int64_t)g.out_eid[p] * heads + h]);
  dS[tid] = s;
}
__global__ void __launch_bounds__(256) k_out_dS_heavy(GraphDev g, int heads, const int32_t* __restrict__ hout,
                                                      const int32_t* counts, const float* __restrict__ dEp,
                                                      float* __restrict__ dS) {
  __shared__ float part[OUT_PART];
  __shared__ float sh[32];
  for (int i = blockIdx.x; i < counts[1]; i += gridDim.x) {
    const int64_t u = hout[i];
    const int64_t b = g.out_ptr[u], len = g.out_ptr[u + 1] - b;
    heavy_row_sums(len, g.chunk, heads,
                   [&](float acc, int64_t k, int h) {
                     return __fadd_rn(acc, dEp[(int64_t)g.out_eid[b + k] * heads + h]);
                   }, part, sh);
    if (threadIdx.x < heads) dS[u * heads + threadIdx.x] = sh[threadIdx.x];
    __syncthreads();
  }
}

// ②′: ∂H′ = (∂H′_agg + ∂S·a_src) + ∂D·a_dst (R23), in place on the aggregated buffer
__global__ void k_out_dhp_combine(float* __restrict__ dHp, int64_t n, int heads, int C, const float* __restrict__ dS,
                                  const float* __restrict__ dD, const float* __restrict__ a_src,
                                  const float* __restrict__ a_dst) {
  const int HC = heads * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * HC; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t u = i / HC;
    const int j = (int)(i % HC), h = j / C;
    const float t1 = __fmul_rn(dS[u * heads + h], a_src[j]);
    const float t2 = __fadd_rn(dHp[i], t1);
    const float t3 = __fmul_rn(dD[u * heads + h], a_dst[j]);
    dHp[i] = __fadd_rn(t2, t3);
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

// FP32 GCN final layer row scalings (R26 norms folded into rows, R35 bias)
// MODE 0: out = x·ns[u]   MODE 1: out = x·nd[v] + b   MODE 2: out = x·nd[v]
template <int MODE>
__global__ void k_gcn_rowscale(const float* __restrict__ x, int64_t n, int C, const float* __restrict__ sc,
                               const float* __restrict__ bias, float* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * C; i += (int64_t)gridDim.x * blockDim.x) {
    const float t = __fmul_rn(x[i], sc[i / C]);
    out[i] = MODE == 1 ? __fadd_rn(t, bias[i % C]) : t;
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
      off_dD, off_dS, off_dHp, off_agg, off_indst, off_hin, off_hout, off_cnt, off_Wt, off_ws, total;
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
  L->off_agg = take(4 * n * HC);
  L->off_indst = take(4 * e);
  L->off_hin = take(4 * n);
  L->off_hout = take(4 * n);
  L->off_cnt = take(4 * 8);
  L->off_Wt = take(4 * F * HC);
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
  if ((M + SG_BM - 1) / SG_BM > 65535 || nchunks_of(K) > 65535) return TANGO_ERR_UNSUPPORTED;   // grid y / z
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
    k_xent<<<grid_1d(rows, 4), 128, smem, stream>>>(logits, labels, rows, classes,
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
  float* agg = reinterpret_cast<float*>(c + L.off_agg);
  int32_t* in_dst = reinterpret_cast<int32_t*>(c + L.off_indst);
  int32_t* hin = reinterpret_cast<int32_t*>(c + L.off_hin);
  int32_t* hout = reinterpret_cast<int32_t*>(c + L.off_hout);
  int32_t* cnt = reinterpret_cast<int32_t*>(c + L.off_cnt);
  const GraphDev g = dev_graph(G);
  const int H_ = (int)L.H, C_ = (int)L.C;
  // plan: in-CSR destinations, heavy rows (degree > C_E) of both CSRs
  M_TRY_CUDA(cudaMemsetAsync(cnt, 0, 8 * sizeof(int32_t), stream));
  {
    ProfScope ps("out_plan", stream);
    k_out_plan<<<grid_1d(L.n, 8), 256, 0, stream>>>(g, in_dst, hin, hout, cnt);
  }
  // ① H′ = H·W (R33)
  M_TRY_CUDA(launch_sgemm(H, L.F, false, p->W, L.HC, false, L.n, L.HC, L.F, Hp, ws, stream));
  {
    ProfScope ps("out_sd", stream);
    k_out_sd<<<(unsigned)((L.n * H_ + 255) / 256), 256, 0, stream>>>(Hp, L.n, H_, C_, p->a_src, p->a_dst, S, D);
  }
  if (L.e > 0) {
    ProfScope ps("out_el", stream);
    k_out_el<<<grid_1d(L.e), 256, 0, stream>>>(L.e, H_, G->in_src, in_dst, S, D, p->neg_slope, epre, el);
  }
  {
    ProfScope ps("out_softmax_light", stream);
    k_out_softmax_light<<<(unsigned)((L.n * H_ + 255) / 256), 256, 0, stream>>>(g, H_, el, m, den, alpha);
  }
  {
    ProfScope ps("out_softmax_heavy", stream);
    k_out_softmax_heavy<<<num_sms() * 2, 256, 0, stream>>>(g, H_, hin, cnt, el, m, den, alpha);
  }
  GatherRow<false> R{G->in_ptr, G->in_src, nullptr, alpha, Hp, H_, C_, (int)L.HC, (int)L.HC};
  M_TRY_CUDA(launch_gather<false>(R, L.n, g.chunk, hin, cnt, agg, stream));
  {
    ProfScope ps("out_logits", stream);
    k_out_logits<<<grid_1d(L.n * L.C), 256, 0, stream>>>(agg, L.n, H_, C_, p->bias, logits);
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
  int32_t* in_dst = reinterpret_cast<int32_t*>(c + L.off_indst);
  int32_t* hin = reinterpret_cast<int32_t*>(c + L.off_hin);
  int32_t* hout = reinterpret_cast<int32_t*>(c + L.off_hout);
  int32_t* cnt = reinterpret_cast<int32_t*>(c + L.off_cnt);
  if (L.e > 0) {
    ProfScope ps("out_dalpha", stream);
    k_out_dalpha<<<grid_1d(L.e * H_), 256, 0, stream>>>(L.e, H_, C_, G->in_src, in_dst, Gm, Hp, dalpha);
  }
  {
    ProfScope ps("out_sbwd_light", stream);
    k_out_sbwd_light<<<(unsigned)((L.n * H_ + 255) / 256), 256, 0, stream>>>(g, H_, alpha, dalpha, epre,
                                                                               p->neg_slope, P, dEp, dD);
  }
  {
    ProfScope ps("out_sbwd_heavy", stream);
    k_out_sbwd_heavy<<<num_sms() * 2, 256, 0, stream>>>(g, H_, hin, cnt, alpha, dalpha, epre, p->neg_slope, P, dEp,
                                                        dD);
  }
  {
    ProfScope ps("out_dS_light", stream);
    k_out_dS_light<<<(unsigned)((L.n * H_ + 255) / 256), 256, 0, stream>>>(g, H_, dEp, dS);
  }
  {
    ProfScope ps("out_dS_heavy", stream);
    k_out_dS_heavy<<<num_sms() * 2, 256, 0, stream>>>(g, H_, hout, cnt, dEp, dS);
  }
  GatherRow<true> R{G->out_ptr, G->out_dst, G->out_eid, alpha, Gm, H_, C_, (int)L.HC, C_};
  M_TRY_CUDA(launch_gather<true>(R, L.n, g.chunk, hout, cnt + 1, dHp, stream));
  {
    ProfScope ps("out_dhp_combine", stream);
    k_out_dhp_combine<<<grid_1d(L.n * L.HC), 256, 0, stream>>>(dHp, L.n, H_, C_, dS, dD, p->a_src, p->a_dst);
  }
  {
    ProfScope ps("out_da", stream);
    k_out_da<<<num_sms() * 2, 256, 0, stream>>>(Hp, L.n, H_, C_, dS, dD, da_src, da_dst);
  }
  // ①′ ∂H = ∂H′·Wᵀ (K = H·C), ∂W = Hᵀ·∂H′ (K = n, chunked) (R33)
  if (dH) {
    float* Wt = reinterpret_cast<float*>(c + L.off_Wt);
    {
      ProfScope ps("transpose", stream);
      k_transpose<<<dim3((unsigned)((L.HC + 31) / 32), (unsigned)((L.F + 31) / 32)), dim3(32, 8), 0, stream>>>(
          p->W, L.F, L.HC, Wt);
    }
    M_TRY_CUDA(launch_sgemm(dHp, L.HC, false, Wt, L.F, false, L.n, L.F, L.HC, dH, ws, stream));
  }
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
  view->agg = reinterpret_cast<float*>(c + L.off_agg);
  return TANGO_OK;
}

}  // extern "C"

// ------------------------------------------------------------------ FP32 final GCN layer (R26, R35)
namespace {
struct GcnOutLayout {
  int64_t n, e, F, C;
  size_t off_Y, off_Ys, off_agg, off_Gs, off_aggb, off_dY, off_ns, off_nd, off_indst, off_hin, off_hout, off_cnt,
      off_ws, total;
};
bool gcn_out_layout(const tango_graph* G, const tango_gcn_out_params* p, GcnOutLayout* L) {
  if (!G || !p || p->in_feats <= 0 || p->classes <= 0) return false;
  L->n = G->row_end - G->row_begin;
  L->e = G->e_in;
  L->F = p->in_feats;
  L->C = p->classes;
  const int64_t n = L->n, C = L->C;
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o = al256(o + bytes); return r; };
  L->off_Y = take(4 * n * C);
  L->off_Ys = take(4 * n * C);
  L->off_agg = take(4 * n * C);
  L->off_Gs = take(4 * n * C);
  L->off_aggb = take(4 * n * C);
  L->off_dY = take(4 * n * C);
  L->off_ns = take(4 * n);
  L->off_nd = take(4 * n);
  L->off_indst = take(4 * L->e);
  L->off_hin = take(4 * n);
  L->off_hout = take(4 * n);
  L->off_cnt = take(4 * 8);
  size_t ws = std::max(sgemm_ws_bytes(L->F, C, n), sgemm_ws_bytes(n, L->F, C));
  ws = std::max(ws, colsum_ws_bytes(n, C));
  L->off_ws = take(ws > 0 ? ws : 4);
  L->total = o;
  return true;
}
tango_status check_gcn_out(const tango_graph* G, const tango_gcn_out_params* p) {
  if (!G || !p || !p->W || !p->bias) return TANGO_ERR_INVALID_ARG;
  if (p->in_feats <= 0 || p->classes <= 0) return TANGO_ERR_SHAPE;
  if (p->classes > OUT_MAXHC) return TANGO_ERR_UNSUPPORTED;
  if (G->row_begin != 0 || G->row_end != G->n_global) return TANGO_ERR_UNSUPPORTED;
  if (G->n_global > 0 && (!G->in_ptr || !G->out_ptr)) return TANGO_ERR_INVALID_ARG;
  if (G->e_in > 0 && (!G->in_src || !G->out_dst || !G->out_eid)) return TANGO_ERR_INVALID_ARG;
  if (G->e_in != G->e_out) return TANGO_ERR_SHAPE;
  return TANGO_OK;
}
template <class T>
T* at(void* ctx, size_t off) { return reinterpret_cast<T*>(static_cast<char*>(ctx) + off); }
}  // namespace

extern "C" {

size_t tango_gcn_out_ctx_bytes(const tango_graph* G, const tango_gcn_out_params* p) {
  GcnOutLayout L;
  if (check_gcn_out(G, p) != TANGO_OK || !gcn_out_layout(G, p, &L)) return 0;
  return L.total;
}

tango_status tango_gcn_out_fwd(const tango_graph* G, const tango_gcn_out_params* p, const float* X, void* ctx,
                               size_t ctx_bytes, float* logits, cudaStream_t stream) {
  tango_status s = check_gcn_out(G, p);
  if (s != TANGO_OK) return s;
  GcnOutLayout L;
  gcn_out_layout(G, p, &L);
  if (!ctx || ctx_bytes < L.total) return TANGO_ERR_INVALID_ARG;
  if (L.n == 0) return TANGO_OK;
  if (!X || !logits) return TANGO_ERR_INVALID_ARG;
  const GraphDev g = dev_graph(G);
  const int C = (int)L.C;
  float *Y = at<float>(ctx, L.off_Y), *Ys = at<float>(ctx, L.off_Ys), *agg = at<float>(ctx, L.off_agg);
  float *ns = at<float>(ctx, L.off_ns), *nd = at<float>(ctx, L.off_nd), *ws = at<float>(ctx, L.off_ws);
  int32_t* cnt = at<int32_t>(ctx, L.off_cnt);
  M_TRY_CUDA(cudaMemsetAsync(cnt, 0, 8 * sizeof(int32_t), stream));
  {
    ProfScope ps("out_plan", stream);
    k_out_plan<<<grid_1d(L.n, 8), 256, 0, stream>>>(g, at<int32_t>(ctx, L.off_indst), at<int32_t>(ctx, L.off_hin),
                                                    at<int32_t>(ctx, L.off_hout), cnt);
  }
  M_TRY_CUDA(launch_gcn_norms(g, ns, nd, stream));
  M_TRY_CUDA(launch_sgemm(X, L.F, false, p->W, C, false, L.n, C, L.F, Y, ws, stream));
  {
    ProfScope ps("gcn_out_scale", stream);
    k_gcn_rowscale<0><<<grid_1d(L.n * C), 256, 0, stream>>>(Y, L.n, C, ns, nullptr, Ys);
  }
  GatherRow<false> R{G->in_ptr, G->in_src, nullptr, nullptr, Ys, 1, C, C, C};
  M_TRY_CUDA(launch_gather<false>(R, L.n, g.chunk, at<int32_t>(ctx, L.off_hin), cnt, agg, stream, "gcn_out_agg_light",
                                  "gcn_out_agg_heavy"));
  {
    ProfScope ps("gcn_out_scale", stream);
    k_gcn_rowscale<1><<<grid_1d(L.n * C), 256, 0, stream>>>(agg, L.n, C, nd, p->bias, logits);
  }
  M_TRY_CUDA(cudaGetLastError());
  return TANGO_OK;
}

tango_status tango_gcn_out_bwd(const tango_graph* G, const tango_gcn_out_params* p, void* ctx, size_t ctx_bytes,
                               const float* X, const float* dlogits, float* dX, float* dW, float* dbias,
                               cudaStream_t stream) {
  tango_status s = check_gcn_out(G, p);
  if (s != TANGO_OK) return s;
  GcnOutLayout L;
  gcn_out_layout(G, p, &L);
  if (!ctx || ctx_bytes < L.total) return TANGO_ERR_INVALID_ARG;
  if (!dW || !dbias) return TANGO_ERR_INVALID_ARG;
  if (L.n > 0 && (!X || !dlogits)) return TANGO_ERR_INVALID_ARG;
  const GraphDev g = dev_graph(G);
  const int C = (int)L.C;
  float *Gs = at<float>(ctx, L.off_Gs), *aggb = at<float>(ctx, L.off_aggb), *dY = at<float>(ctx, L.off_dY);
  float *ns = at<float>(ctx, L.off_ns), *nd = at<float>(ctx, L.off_nd), *ws = at<float>(ctx, L.off_ws);
  int32_t* cnt = at<int32_t>(ctx, L.off_cnt);
  M_TRY_CUDA(launch_colsum<0>(dlogits, nullptr, L.n, C, dbias, ws, nullptr, nullptr, stream));
  if (L.n == 0) {
    M_TRY_CUDA(cudaMemsetAsync(dW, 0, sizeof(float) * L.F * C, stream));
    return TANGO_OK;
  }
  {
    ProfScope ps("gcn_out_scale", stream);
    k_gcn_rowscale<2><<<grid_1d(L.n * C), 256, 0, stream>>>(dlogits, L.n, C, nd, nullptr, Gs);
  }
  GatherRow<true> R{G->out_ptr, G->out_dst, G->out_eid, nullptr, Gs, 1, C, C, C};
  M_TRY_CUDA(launch_gather<true>(R, L.n, g.chunk, at<int32_t>(ctx, L.off_hout), cnt + 1, aggb, stream,
                                 "gcn_out_aggb_light", "gcn_out_aggb_heavy"));
  {
    ProfScope ps("gcn_out_scale", stream);
    k_gcn_rowscale<0><<<grid_1d(L.n * C), 256, 0, stream>>>(aggb, L.n, C, ns, nullptr, dY);
  }
  if (dX) M_TRY_CUDA(launch_sgemm(dY, C, false, p->W, C, true, L.n, L.F, C, dX, ws, stream));
  M_TRY_CUDA(launch_sgemm(X, L.F, true, dY, C, false, L.F, C, L.n, dW, ws, stream));
  return TANGO_OK;
}

tango_status tango_gcn_out_ctx_get_view(const tango_graph* G, const tango_gcn_out_params* p, void* ctx,
                                        tango_gcn_out_ctx_view* view) {
  tango_status s = check_gcn_out(G, p);
  if (s != TANGO_OK) return s;
  if (!ctx || !view) return TANGO_ERR_INVALID_ARG;
  GcnOutLayout L;
  gcn_out_layout(G, p, &L);
  view->Y = at<float>(ctx, L.off_Y);
  view->Ys = at<float>(ctx, L.off_Ys);
  view->agg = at<float>(ctx, L.off_agg);
  view->Gs = at<float>(ctx, L.off_Gs);
  view->aggb = at<float>(ctx, L.off_aggb);
  view->dY = at<float>(ctx, L.off_dY);
  return TANGO_OK;
}

}  // extern "C"
