// gemm_tc.cu — quantization-aware int8 GEMM on the 5th-generation tensor cores (sm_100a).
//
// Paper: §3.2 Fig.4 (int8 x int8 -> int32 result, dequantized in-kernel, the output
// scale derived inside the GEMM) and P:736-739 §3.3 (GEMM with fused quantization / dequantization).
// B200 design: the paper's DP4A CUDA-core tiling is replaced by
//   * TMA (cp.async.bulk.tensor, SWIZZLE_128B) loads of int8 tiles into a 4-stage smem ring,
//   * one elected thread issuing tcgen05.mma.cta_group::1.kind::i8 (M=128, N<=256, K=32 per op)
//     into a double-buffered int32 accumulator in TMEM,
//   * 4 epilogue warps draining TMEM with tcgen05.ld and applying the fused epilogue
//     (dequantize, per-head S/D dots, amax, Philox stochastic-rounding re-quantization,
//      fp32 store, or int64 split-K reduction),
// in a persistent kernel (grid = #SMs) with warp specialisation: warp 0 TMA, warp 1 MMA,
// warps 2-5 epilogue.  Operands may be K-major or MN-major (∂W = Hᵀ·∂H′ reads both MN-major).
#include <cudaTypedefs.h>

#include <cstdio>
#include <mutex>

#include "kernels.h"

namespace tango {

constexpr int BM = 128;            // rows per tile (TMEM lanes)
constexpr int BKB = 128;           // K bytes per pipeline stage (one 128-B swizzle row)
constexpr int STAGES = 4;
constexpr int A_BYTES = BM * BKB;  // 16 KB
constexpr int B_BYTES_MAX = 256 * BKB;
constexpr int STAGE_BYTES = A_BYTES + B_BYTES_MAX;
constexpr int EPI_WARPS = 8;       // two per TMEM sub-partition, each owning a column group of the N tile
constexpr int GEMM_THREADS = 64 + 32 * EPI_WARPS;
constexpr int TR_LD = 17;          // EPI_STORE transpose tile: 32 rows x 16 columns (+1 pad) per epilogue warp
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 4096 + 1024 + EPI_WARPS * 32 * TR_LD * 4 + 1024;   // + alignment slack

struct KParams {
  int64_t M, N, K;
  int BN, n_tiles_m, n_tiles_n, splits, kb_per_split, total_kb, nblk_b;
  int a_mn, b_mn, col_groups;   // epilogue column groups per sub-partition (1..3; whole heads with dots)
  int64_t total_tiles;
  uint32_t idesc, stage_tx, tmem_cols;
  const float* sA; const float* sB; const float* rowscale;
  unsigned* amax_slot;
  const float* a_src; const float* a_dst; int head_dim; float* S; float* Dd; int heads;
  unsigned* amax_S; unsigned* amax_D;
  uint32_t code_xor;   // EPI_QUANT: 0x80808080 stores excess-128 codes (q + 128) for the gather kernels
  const unsigned* amax_in; int bits; PhiloxKey key; uint32_t step; uint32_t tag; int64_t g_row0;
  int8_t* q_out; int64_t ldq; float* scale_out; int32_t* status;
  void* C; int64_t ldc;
  int c_pair;   // EPI_STORE: even ldc and 8-B aligned C -> float2 stores
};

// dequantized epilogue value: v = i2f(acc) * (s_A s_B) [* rowscale]  (two roundings)
__device__ __forceinline__ float deq(uint32_t acc, float sAB, bool has_rs, float rs) {
  float v = __fmul_rn(__int2float_rn((int)acc), sAB);
  return has_rs ? __fmul_rn(v, rs) : v;
}

template <int MODE, bool RS>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    k_gemm_i8(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const __grid_constant__ KParams p) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned by pointer arithmetic on the shared array (keeps the shared address space visible)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* sm_asrc = reinterpret_cast<float*>(smem + STAGES * STAGE_BYTES + 1024);
  float* sm_adst = sm_asrc + 256;
  float* sm_tr = reinterpret_cast<float*>(smem + STAGES * STAGE_BYTES + 4096 + 1024);

  const int warp = warp_id();
  const int lane = lane_id();

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 32 * EPI_WARPS); }
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) { tma_prefetch_desc(&tmA); tma_prefetch_desc(&tmB); }
  if (warp == 1) tmem_alloc(tmem_slot, p.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------- TMA producer
    if (lane == 0) {
      int stage = 0; uint32_t phase = 0;
      for (int64_t t = blockIdx.x; t < p.total_tiles; t += gridDim.x) {
        const int sp = (int)(t % p.splits);
        const int64_t mn = t / p.splits;
        const int nt = (int)(mn % p.n_tiles_n);
        const int mt = (int)(mn / p.n_tiles_n);
        const int kb0 = sp * p.kb_per_split;
        const int kb1 = min(p.total_kb, kb0 + p.kb_per_split);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], p.stage_tx);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          uint8_t* sb = sa + A_BYTES;
          if (!p.a_mn) tma_load_2d(sa, &tmA, &full[stage], kb * BKB, mt * BM);
          else tma_load_2d(sa, &tmA, &full[stage], mt * BM, kb * BKB);
          if (!p.b_mn) {
            tma_load_2d(sb, &tmB, &full[stage], kb * BKB, nt * p.BN);
          } else {
            for (int blk = 0; blk < p.nblk_b; ++blk)
              tma_load_2d(sb + blk * (BKB * 128), &tmB, &full[stage], nt * p.BN + blk * 128, kb * BKB);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------- MMA issuer (one thread)
    if (lane == 0) {
      int stage = 0; uint32_t phase = 0;
      uint32_t lt = 0;
      for (int64_t t = blockIdx.x; t < p.total_tiles; t += gridDim.x, ++lt) {
        const int sp = (int)(t % p.splits);
        const int kb0 = sp * p.kb_per_split;
        const int kb1 = min(p.total_kb, kb0 + p.kb_per_split);
        const uint32_t buf = lt & 1, tph = (lt >> 1) & 1;
        mbar_wait(&tempty[buf], tph ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + buf * (uint32_t)p.BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * STAGE_BYTES);
          const uint32_t sb = sa + A_BYTES;
#pragma unroll
          for (int kk = 0; kk < BKB / 32; ++kk) {
            const uint64_t ad = p.a_mn ? make_sdesc(sa + kk * 32 * 128, A_BYTES, 1024, 2)
                                       : make_sdesc(sa + kk * 32, 16, 1024, 2);
            const uint64_t bd = p.b_mn ? make_sdesc(sb + kk * 32 * 128, BKB * 128, 1024, 2)
                                       : make_sdesc(sb + kk * 32, 16, 1024, 2);
            mma_i8(d_tmem, ad, bd, p.idesc, (kb > kb0 || kk > 0) ? 1u : 0u);
          }
          mma_commit(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        mma_commit(&tfull[buf]);
      }
    }
  } else {
    // ------------------------------------------------------------- epilogue (warps 2..9)
    const int ew = warp - 2;                  // 0 .. EPI_WARPS-1
    const int sub = warp & 3;                 // TMEM sub-partition this warp may access
    const int grp = ew >> 2;                  // column group of the N tile (idle if >= col_groups)
    const int rin = sub * 32 + lane;          // row within the tile
    const int nch = p.BN / 32;
    const int c_lo = grp < p.col_groups ? (grp * nch) / p.col_groups : 0;
    const int c_hi = grp < p.col_groups ? ((grp + 1) * nch) / p.col_groups : 0;
    const float sAB = (p.sA && p.sB) ? __fmul_rn(*p.sA, *p.sB) : 1.0f;
    constexpr bool has_rs = RS;   // per-row multiplier (GCN), a template parameter: no select per element
    Scale qs = {1.0f, 1.0f, false};
    if (MODE == EPI_QUANT) {
      qs = scale_from_amax(amax_load(p.amax_in), p.bits);
      if (blockIdx.x == 0 && threadIdx.x == 64) {
        if (p.scale_out) *p.scale_out = qs.s;
        if (qs.bad && p.status) atomicExch(p.status, ST_NONFINITE);
      }
    }
    const int qmax = (1 << (p.bits - 1)) - 1;
    float amax_v = 0.0f, amax_s = 0.0f, amax_d = 0.0f;
    const bool dots = (MODE == EPI_AMAX) && (p.a_src != nullptr);
    const bool fast_heads = dots && (p.head_dim % 32 == 0);
    uint32_t lt = 0;
    int loaded_nt = -1;
    for (int64_t t = blockIdx.x; t < p.total_tiles; t += gridDim.x, ++lt) {
      const int64_t mn = t / p.splits;
      const int nt = (int)(mn % p.n_tiles_n);
      const int mt = (int)(mn / p.n_tiles_n);
      const uint32_t buf = lt & 1, tph = (lt >> 1) & 1;
      if (dots && nt != loaded_nt) {
        // stage this N-tile's attention vectors in smem (epilogue warps only: named barrier 1)
        asm volatile("bar.sync 1, %0;" ::"n"(32 * EPI_WARPS) : "memory");
        for (int j = threadIdx.x - 64; j < p.BN; j += 32 * EPI_WARPS) {
          const int64_t col = (int64_t)nt * p.BN + j;
          sm_asrc[j] = col < p.N ? p.a_src[col] : 0.0f;
          sm_adst[j] = col < p.N ? p.a_dst[col] : 0.0f;
        }
        asm volatile("bar.sync 1, %0;" ::"n"(32 * EPI_WARPS) : "memory");
        loaded_nt = nt;
      }
      mbar_wait(&tfull[buf], tph);
      tc_fence_after();
      const int64_t row = (int64_t)mt * BM + rin;
      const bool row_ok = row < p.M;
      const float rs = (has_rs && row_ok) ? p.rowscale[row] : 1.0f;
      const uint32_t tbase = tmem_base + ((uint32_t)(sub * 32) << 16) + buf * (uint32_t)p.BN;
      float s_acc = 0.0f, d_acc = 0.0f;
      int dcount = 0;
      const int cph = fast_heads ? p.head_dim / 32 : 1;   // 32-column chunks per head
      int hcnt = fast_heads ? (c_lo % cph) : 0;
      int h_next = fast_heads ? (int)(((int64_t)nt * p.BN + c_lo * 32) / p.head_dim) : 0;
      for (int c = c_lo; c < c_hi; ++c) {
        uint32_t r[32];
        tmem_ld32(tbase + c * 32, r);
        tmem_ld_wait();
        const int64_t col0 = (int64_t)nt * p.BN + c * 32;
        const bool full_chunk = col0 + 32 <= p.N;
        if constexpr (MODE == EPI_AMAX) {
          if (full_chunk && (fast_heads || !dots)) {
            float v[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = deq(r[i], sAB, has_rs, rs);
            if (row_ok) {
#pragma unroll
              for (int i = 0; i < 32; ++i) amax_v = fmaxf(amax_v, fabsf(v[i]));
            }
            if (dots) {
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                s_acc = __fmaf_rn(v[i], sm_asrc[c * 32 + i], s_acc);
                d_acc = __fmaf_rn(v[i], sm_adst[c * 32 + i], d_acc);
              }
              if (++hcnt == cph) {   // the chunk closes a head (head_dim % 32 == 0 here)
                hcnt = 0;
                const int h = h_next++;
                if (row_ok) {
                  p.S[row * p.heads + h] = s_acc;
                  p.Dd[row * p.heads + h] = d_acc;
                  amax_s = fmaxf(amax_s, fabsf(s_acc));
                  amax_d = fmaxf(amax_d, fabsf(d_acc));
                }
                s_acc = 0.0f; d_acc = 0.0f;
              }
            }
          } else {
            for (int i = 0; i < 32; ++i) {
              const int64_t col = col0 + i;
              if (col >= p.N) break;
              const float v = deq(r[i], sAB, has_rs, rs);
              if (row_ok) amax_v = fmaxf(amax_v, fabsf(v));
              if (dots) {
                s_acc = __fmaf_rn(v, sm_asrc[c * 32 + i], s_acc);
                d_acc = __fmaf_rn(v, sm_adst[c * 32 + i], d_acc);
                if (++dcount == p.head_dim) {
                  if (row_ok) {
                    const int h = (int)(col / p.head_dim);
                    p.S[row * p.heads + h] = s_acc;
                    p.Dd[row * p.heads + h] = d_acc;
                    amax_s = fmaxf(amax_s, fabsf(s_acc));
                    amax_d = fmaxf(amax_d, fabsf(d_acc));
                  }
                  s_acc = 0.0f; d_acc = 0.0f; dcount = 0;
                }
              }
            }
          }
        } else if constexpr (MODE == EPI_QUANT) {
          uint32_t packed[8];
#pragma unroll
          for (int g8 = 0; g8 < 4; ++g8) {
            const int64_t g = (p.g_row0 + row) * p.N + col0 + g8 * 8;   // N % 8 == 0
            const SR8 rnd = sr_draw8((uint64_t)(g >> 3), p.tag, p.step, p.key);
            float v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = deq(r[g8 * 8 + k], sAB, has_rs, rs);
            const uint2 pk = sr_quant8(v, qs.r, rnd, qmax);
            const bool in = col0 + g8 * 8 < p.N;   // N % 8 == 0: whole groups are in or out
            packed[g8 * 2] = in ? pk.x ^ p.code_xor : 0u; packed[g8 * 2 + 1] = in ? pk.y ^ p.code_xor : 0u;
          }
          if (row_ok && col0 < p.ldq) {
            uint4* dst = reinterpret_cast<uint4*>(p.q_out + row * p.ldq + col0);
            dst[0] = make_uint4(packed[0], packed[1], packed[2], packed[3]);
            dst[1] = make_uint4(packed[4], packed[5], packed[6], packed[7]);
          }
        } else if constexpr (MODE == EPI_STORE) {
          // lane = row: transpose the 32 x 32 chunk through shared memory in two 16-column halves so that
          // every store instruction writes two rows' 16 consecutive columns (64 contiguous bytes per row,
          // whole sectors) instead of one 16-B piece of 32 different rows; any ldc / C alignment works
          float* Cf = reinterpret_cast<float*>(p.C);
          float* tr = sm_tr + ew * (32 * TR_LD);
          const int64_t rowbase = (int64_t)mt * BM + sub * 32;
#pragma unroll
          for (int hf = 0; hf < 2; ++hf) {
#pragma unroll
            for (int i = 0; i < 16; ++i) tr[lane * TR_LD + i] = deq(r[hf * 16 + i], sAB, has_rs, rs);
            __syncwarp();
            if (p.c_pair) {   // 8-B aligned rows (even ldc, 8-B aligned C): float2 stores, 4 rows x 16 columns each
              const int c2 = (lane & 7) * 2, rq = lane >> 3;
              const int64_t col = col0 + hf * 16 + c2;
#pragma unroll
              for (int j = 0; j < 32; j += 4) {
                const int64_t rr = rowbase + j + rq;
                const float x0 = tr[(j + rq) * TR_LD + c2], x1 = tr[(j + rq) * TR_LD + c2 + 1];
                if (rr < p.M) {
                  if (col + 1 < p.N) *reinterpret_cast<float2*>(Cf + rr * p.ldc + col) = make_float2(x0, x1);
                  else if (col < p.N) Cf[rr * p.ldc + col] = x0;
                }
              }
            } else {
              const int cl = lane & 15, rh = lane >> 4;
              const int64_t col = col0 + hf * 16 + cl;
#pragma unroll
              for (int j = 0; j < 32; j += 2) {
                const int64_t rr = rowbase + j + rh;
                if (rr < p.M && col < p.N) Cf[rr * p.ldc + col] = tr[(j + rh) * TR_LD + cl];
              }
            }
            __syncwarp();
          }
        } else if constexpr (MODE == EPI_I32) {   // transposed through shared memory as EPI_STORE
          int32_t* Ci = reinterpret_cast<int32_t*>(p.C);
          int32_t* tr = reinterpret_cast<int32_t*>(sm_tr) + ew * (32 * TR_LD);
          const int64_t rowbase = (int64_t)mt * BM + sub * 32;
          const int cl = lane & 15, rh = lane >> 4;
#pragma unroll
          for (int hf = 0; hf < 2; ++hf) {
#pragma unroll
            for (int i = 0; i < 16; ++i) tr[lane * TR_LD + i] = (int32_t)r[hf * 16 + i];
            __syncwarp();
            const int64_t col = col0 + hf * 16 + cl;
#pragma unroll
            for (int j = 0; j < 32; j += 2) {
              const int64_t rr = rowbase + j + rh;
              if (rr < p.M && col < p.N) Ci[rr * p.ldc + col] = tr[(j + rh) * TR_LD + cl];
            }
            __syncwarp();
          }
        } else {  // EPI_ATOMIC64
          unsigned long long* C64 = reinterpret_cast<unsigned long long*>(p.C);
          if (row_ok) {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (col0 + i < p.N && r[i] != 0u)
                atomicAdd(C64 + row * p.ldc + col0 + i, (unsigned long long)(long long)(int32_t)r[i]);
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[buf]);
    }
    if (MODE == EPI_AMAX) {
      amax_v = warp_max(amax_v);
      if (lane == 0 && p.amax_slot) atomic_max_abs(p.amax_slot, amax_v);
      if (dots) {
        amax_s = warp_max(amax_s);
        amax_d = warp_max(amax_d);
        if (lane == 0) {
          if (p.amax_S) atomic_max_abs(p.amax_S, amax_s);
          if (p.amax_D) atomic_max_abs(p.amax_D, amax_d);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, p.tmem_cols);
  }
}

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  return fn;
}

static bool make_map(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint64_t stride_bytes,
                     uint32_t box_inner, uint32_t box_outer) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {stride_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Row-gather map for TMA tile::gather4 (gat.cu): the int8 table [rows][ld] viewed as uint32
// [rows][ld/4] with a {row_bytes/4, 1} box, no swizzle — one gather4 lands 4 rows of row_bytes
// contiguously in shared memory.
bool make_row_gather_map(CUtensorMap* m, const void* base, uint64_t rows, uint64_t row_bytes, uint64_t ld_bytes) {
  auto fn = encode_fn();
  if (!fn || row_bytes % 16 || ld_bytes % 16 || row_bytes / 4 > 256 || rows == 0) return false;
  cuuint64_t dims[2] = {ld_bytes / 4, rows};
  cuuint64_t strides[1] = {ld_bytes};
  cuuint32_t box[2] = {(cuuint32_t)(row_bytes / 4), 1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

cudaError_t launch_gemm(const GemmArgs& a, cudaStream_t st) {
  if (a.M <= 0 || a.N <= 0) return cudaSuccess;
  KParams p{};
  p.M = a.M; p.N = a.N; p.K = a.K;
  int BN = (int)((a.N + 31) / 32 * 32);
  if (BN > 256) BN = 256;
  if (a.mode == EPI_AMAX && a.a_src && (BN % a.head_dim) != 0) {
    // a tile must hold whole heads: shrink BN to a multiple of head_dim (head_dim divides 256 in practice)
    BN = (256 / a.head_dim) * a.head_dim;
    if (BN % 32) return cudaErrorInvalidValue;
  }
  p.BN = BN;
  p.n_tiles_m = (int)((a.M + BM - 1) / BM);
  p.n_tiles_n = (int)((a.N + BN - 1) / BN);
  p.total_kb = (int)((a.K + BKB - 1) / BKB);
  if (p.total_kb == 0) p.total_kb = 1;   // K = 0: one zero-filled block keeps the pipeline uniform
  p.splits = a.splits > 1 ? a.splits : 1;
  p.kb_per_split = (p.total_kb + p.splits - 1) / p.splits;
  p.splits = (p.total_kb + p.kb_per_split - 1) / p.kb_per_split;
  p.nblk_b = (BN + 127) / 128;
  p.a_mn = a.a_mn; p.b_mn = a.b_mn;
  {   // as many column groups as the epilogue warps allow; with head dots every group holds whole heads
    const int nch = BN / 32;
    const bool dots = a.mode == EPI_AMAX && a.a_src;
    int g = EPI_WARPS / 4;
    for (; g > 1; --g) {
      if (g > nch) continue;
      if (dots && (nch % g || ((BN / g) % a.head_dim) != 0)) continue;
      break;
    }
    p.col_groups = g;
  }
  p.total_tiles = (int64_t)p.n_tiles_m * p.n_tiles_n * p.splits;
  p.idesc = make_idesc_i8(BM, BN, a.a_mn, a.b_mn);
  p.stage_tx = A_BYTES + (a.b_mn ? p.nblk_b * BKB * 128 : BN * BKB);
  uint32_t cols = 32;
  while (cols < (uint32_t)(2 * BN)) cols <<= 1;
  p.tmem_cols = cols;
  p.sA = a.sA; p.sB = a.sB; p.rowscale = a.rowscale;
  p.amax_slot = a.amax_slot; p.a_src = a.a_src; p.a_dst = a.a_dst; p.head_dim = a.head_dim > 0 ? a.head_dim : 1;
  p.S = a.S; p.Dd = a.Dd; p.heads = a.heads; p.amax_S = a.amax_S; p.amax_D = a.amax_D;
  p.amax_in = a.amax_in; p.bits = a.bits > 0 ? a.bits : 8; p.key = philox_key(a.seed); p.code_xor = a.code_xor; p.step = a.step; p.tag = a.tag;
  p.g_row0 = a.g_row0; p.q_out = a.q_out; p.ldq = a.ldq; p.scale_out = a.scale_out; p.status = a.status;
  p.C = a.C; p.ldc = a.ldc;
  p.c_pair = (a.ldc % 2 == 0) && ((reinterpret_cast<uintptr_t>(a.C) & 7) == 0);

  CUtensorMap tA, tB;
  bool ok;
  if (!a.a_mn) ok = make_map(&tA, a.A, (uint64_t)a.lda, (uint64_t)a.M, (uint64_t)a.lda, BKB, BM);
  else ok = make_map(&tA, a.A, (uint64_t)a.lda, (uint64_t)a.K, (uint64_t)a.lda, 128, BKB);
  if (!ok) return cudaErrorInvalidValue;
  if (!a.b_mn) ok = make_map(&tB, a.B, (uint64_t)a.ldb, (uint64_t)a.N, (uint64_t)a.ldb, BKB, (uint32_t)BN);
  else ok = make_map(&tB, a.B, (uint64_t)a.ldb, (uint64_t)a.K, (uint64_t)a.ldb, 128, BKB);
  if (!ok) return cudaErrorInvalidValue;

  int64_t grid = p.total_tiles < num_sms() ? p.total_tiles : num_sms();
  static const char* names[] = {"gemm_amax", "gemm_quant", "gemm_store", "gemm_i32", "gemm_splitk_i64"};
  ProfScope ps(names[a.mode], st);
  switch (a.mode) {
#define LAUNCH(M_)                                                                                   \
  case M_: {                                                                                         \
    static std::once_flag once_##M_;                                                                 \
    std::call_once(once_##M_, [] {                                                                   \
      cudaFuncSetAttribute(k_gemm_i8<M_, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES); \
      cudaFuncSetAttribute(k_gemm_i8<M_, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);  \
    });                                                                                              \
    if (p.rowscale) k_gemm_i8<M_, true><<<(unsigned)grid, GEMM_THREADS, SMEM_BYTES, st>>>(tA, tB, p);  \
    else k_gemm_i8<M_, false><<<(unsigned)grid, GEMM_THREADS, SMEM_BYTES, st>>>(tA, tB, p);           \
    break;                                                                                           \
  }
    LAUNCH(EPI_AMAX) LAUNCH(EPI_QUANT) LAUNCH(EPI_STORE) LAUNCH(EPI_I32) LAUNCH(EPI_ATOMIC64)
#undef LAUNCH
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// dW = (float)acc64 * (sA*sB)  (reading R27: int64 reduction, one rounding)
__global__ void k_finalize_dw(const int64_t* __restrict__ acc, int64_t count, const float* sA, const float* sB,
                              float* __restrict__ out) {
  const float s = __fmul_rn(*sA, *sB);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __fmul_rn(__ll2float_rn(acc[i]), s);
}
cudaError_t launch_finalize_dw(const int64_t* acc, int64_t count, const float* sA, const float* sB, float* out,
                               cudaStream_t st) {
  if (count == 0) return cudaSuccess;
  int grid = (int)((count + 255) / 256);
  if (grid > 4 * num_sms()) grid = 4 * num_sms();
  ProfScope ps("finalize_dw", st);
  k_finalize_dw<<<grid, 256, 0, st>>>(acc, count, sA, sB, out);
  return cudaGetLastError();
}

}  // namespace tango
