// int4.cu — NEXT-4: sub-byte node features for the SDDMM primitives
// (§4.4, Fig.18a "INT4 SDDMM").  Codes are the B = 4 stochastic-rounding codes of the
// quantizer (qmax = 7, the same Philox stream and element index as tango_quantize with bits = 4),
// stored packed: element 2i of a row in the low nibble of byte i, element 2i+1 in the high nibble,
// 4-bit two's complement.
//
// The SDDMM-dot works on packed words without unpacking to bytes: for a 32-bit word w of 8 nibbles,
// (w << 4) & 0xF0F0F0F0 holds the even codes and w & 0xF0F0F0F0 the odd codes, each as a signed
// byte equal to 16·q; one IDP4A on each gives 256·Σ q_a q_b exactly, so the row dot is the exact
// integer Σ_d q_a q_b after a division by 256 (all terms are multiples of 256, |Σ| < 2^31).
// The same warp-per-destination-row kernel serves 8-bit codes (one IDP4A per word), so int8 and int4
// are compared on one design.
#include "../../include/tango.h"
#include "rowops.cuh"

namespace tango {

// pack the int8 codes of 8 consecutive elements (two words of 4 bytes) into 8 nibbles
__device__ __forceinline__ uint32_t nib_pack8(uint2 c) {
  auto half = [](uint32_t w) {
    return (w & 0xFu) | ((w >> 4) & 0xF0u) | ((w >> 8) & 0xF00u) | ((w >> 12) & 0xF000u);
  };
  return half(c.x) | (half(c.y) << 16);
}

// SR quantization to packed 4-bit codes: one Philox call per group of 8 elements (reading R4/R5)
__global__ void __launch_bounds__(256) k_quantize_pack4(const float* __restrict__ x, int64_t rows, int64_t cols,
                                                        int64_t g0, const unsigned* __restrict__ amax_slot,
                                                        const PhiloxKey key, uint32_t step, uint32_t tag,
                                                        uint8_t* __restrict__ q, int64_t ldb,
                                                        float* __restrict__ scale_out, int32_t* __restrict__ status) {
  const Scale sc = scale_from_amax(amax_load(amax_slot), 4);
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (tid == 0) {
    if (scale_out) *scale_out = sc.s;
    if (sc.bad && status) atomicExch(status, ST_NONFINITE);
  }
  const int64_t gpr = cols >> 3;                 // groups per row (cols % 8 == 0)
  const int64_t groups = rows * gpr;
  for (int64_t k = tid; k < groups; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = k / gpr, jg = k - i * gpr;
    const float* src = x + i * cols + jg * 8;
    const float4 a = __ldg(reinterpret_cast<const float4*>(src)), b = __ldg(reinterpret_cast<const float4*>(src) + 1);
    const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    const SR8 rnd = sr_draw8((uint64_t)((g0 + i * cols + jg * 8) >> 3), tag, step, key);
    const uint2 c = sr_quant8(v, sc.r, rnd, 7);
    *reinterpret_cast<uint32_t*>(q + i * ldb + jg * 4) = nib_pack8(c);
  }
}

// words of one row: WBITS = 8 -> 4 codes per word, 4 -> 8 codes per word
template <int BITS>
__device__ __forceinline__ int word_dot(uint32_t a, uint32_t b) {
  if (BITS == 8) return __dp4a((int)a, (int)b, 0);
  const int lo = __dp4a((int)((a << 4) & 0xF0F0F0F0u), (int)((b << 4) & 0xF0F0F0F0u), 0);
  return __dp4a((int)(a & 0xF0F0F0F0u), (int)(b & 0xF0F0F0F0u), lo);   // 256 · Σ q_a q_b over 8 codes
}

// Edge runs: the work is split into runs of consecutive in-CSR positions (not rows), so a hub row
// is spread over many warps; the destination row of a position is found by a binary search of
// in_ptr at the start of a run and by walking forward from there.
__device__ __forceinline__ int64_t row_of(const int64_t* __restrict__ ptr, int64_t n, int64_t e) {
  int64_t lo = 0, hi = n;            // largest v with ptr[v] <= e  (ptr[0] = 0 <= e < ptr[n])
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (__ldg(ptr + mid) <= e) lo = mid; else hi = mid;
  }
  return lo;
}

// ⑤″ SDDMM-dot on BITS-bit codes, one warp per run of RUN in-edges, lanes over the 32-bit words of a
// row (word l + 32c, c < NCH), GRP edges' rows loaded before any is reduced.  With gsz = words per
// head (a power of two): gsz <= 32 -> the lanes of a head reduce with shuffles per 32-word chunk;
// gsz > 32 -> a head spans gsz/32 chunks, summed in-lane first.  Integer sums (order-free).
// out[e,h] = i2f(Σ_d qA[v] qB[u]) · (sA·sB).
constexpr int DOT_RUN = 64;
template <int BITS, int NCH, int GSZ, int DOT_GRP = (NCH <= 2 ? 8 : 4)>
__global__ void __launch_bounds__(256) k_sddmm_dot_e(GraphDev g, int heads, int words, const uint32_t* __restrict__ A,
                                                     int64_t lda_w, const float* sA, const uint32_t* __restrict__ B,
                                                     int64_t ldb_w, const float* sB, float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  constexpr int gsz = GSZ;
  const float s = __fmul_rn(*sA, *sB);
  const int64_t E = g.in_ptr[g.n_local];
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t item = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); item * DOT_RUN < E; item += nw) {
    const int64_t e0 = item * DOT_RUN, e1 = min(E, e0 + DOT_RUN);
    int64_t v = row_of(g.in_ptr, g.n_local, e0);
    int64_t vend = __ldg(g.in_ptr + v + 1);
    // the run's source ids, one per lane (two rounds of 32), broadcast by shuffles below
    const int32_t idx0 = e0 + lane < e1 ? __ldg(g.in_src + e0 + lane) : 0;
    const int32_t idx1 = e0 + 32 + lane < e1 ? __ldg(g.in_src + e0 + 32 + lane) : 0;
    for (int64_t eb = e0; eb < e1; eb += DOT_GRP) {
      uint32_t wa[DOT_GRP][NCH], wb[DOT_GRP][NCH];
#pragma unroll
      for (int k = 0; k < DOT_GRP; ++k) {
        const int64_t e = eb + k;
        if (e < e1) {
          while (vend <= e) { ++v; vend = __ldg(g.in_ptr + v + 1); }
        }
        const uint32_t* arow = A + (g.row_begin + v) * lda_w;
        const int o = (int)(e - e0);
        const int32_t u = __shfl_sync(0xffffffffu, o < 32 ? idx0 : idx1, o & 31);
        const uint32_t* brow = B + (int64_t)(e < e1 ? u : 0) * ldb_w;
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          const int w = c * 32 + lane;
          const bool ok = e < e1 && w < words;
          wa[k][c] = ok ? __ldg(arow + w) : 0u;
          wb[k][c] = ok ? __ldg(brow + w) : 0u;
        }
      }
      if constexpr (GSZ >= DOT_GRP && GSZ <= 32) {
        // transposed reduction: the DOT_GRP partial dots of a lane are reduce-scattered over the GSZ
        // lanes of its head (halving exchanges), so a group of edges costs ~DOT_GRP shuffles per
        // 32-word chunk instead of DOT_GRP·log2(GSZ); lane bit o of each halving step selects
        // which half (which edges) the lane keeps.
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          int val[DOT_GRP];
#pragma unroll
          for (int k = 0; k < DOT_GRP; ++k) val[k] = word_dot<BITS>(wa[k][c], wb[k][c]);
          int kidx = 0;
#pragma unroll
          for (int n = DOT_GRP, o = GSZ / 2; n > 1; n >>= 1, o >>= 1) {
            const bool upper = (lane & o) != 0;
#pragma unroll
            for (int i = 0; i < n / 2; ++i) {
              const int send = upper ? val[i] : val[i + n / 2];
              const int keep = upper ? val[i + n / 2] : val[i];
              val[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
            }
            kidx = kidx * 2 + (upper ? 1 : 0);
          }
#pragma unroll
          for (int o = GSZ / (2 * DOT_GRP); o >= 1; o >>= 1) val[0] += __shfl_xor_sync(0xffffffffu, val[0], o);
          const int w = c * 32 + lane;
          const int64_t e = eb + kidx;
          if (w < words && (lane & (GSZ / DOT_GRP - 1)) == 0 && e < e1)
            out[e * heads + w / GSZ] = __fmul_rn(__int2float_rn(BITS == 8 ? val[0] : val[0] / 256), s);
        }
        continue;
      }
#pragma unroll
      for (int k = 0; k < DOT_GRP; ++k) {
        const int64_t e = eb + k;
        if (e >= e1) continue;
        if constexpr (GSZ <= 32) {
#pragma unroll
          for (int c = 0; c < NCH; ++c) {
            int x = word_dot<BITS>(wa[k][c], wb[k][c]);
#pragma unroll
            for (int o = 1; o < GSZ; o <<= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
            const int w = c * 32 + lane;
            if (w < words && (lane & (gsz - 1)) == 0)
              out[e * heads + w / gsz] = __fmul_rn(__int2float_rn(BITS == 8 ? x : x / 256), s);
          }
        } else {
          constexpr int per = GSZ / 32;   // chunks per head
          int x = 0;
#pragma unroll
          for (int c = 0; c < NCH; ++c) {
            x += word_dot<BITS>(wa[k][c], wb[k][c]);
            if ((c + 1) % per == 0) {
#pragma unroll
              for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
              if (lane == 0 && c * 32 < words)
                out[e * heads + (c * 32) / gsz] = __fmul_rn(__int2float_rn(BITS == 8 ? x : x / 256), s);
              x = 0;
            }
          }
        }
      }
    }
  }
}

// ③ SDDMM-add on BITS-bit codes of S [N][heads] and D [n][heads]: one warp per run of 32·ADD_PER
// in-edges, lane per edge (all heads); each lane walks its destination row forward from the run's.
template <int BITS>
__device__ __forceinline__ int code_at(const uint8_t* row, int h) {
  if (BITS == 8) return (int)(int8_t)row[h];
  const uint8_t byte = row[h >> 1];
  const int nib = (h & 1) ? (byte >> 4) : (byte & 0xF);
  return nib >= 8 ? nib - 16 : nib;
}
constexpr int ADD_PER = 8;
template <int BITS>
__global__ void __launch_bounds__(256) k_sddmm_add_e(GraphDev g, int heads, const uint8_t* __restrict__ S,
                                                     int64_t lds, const float* sS, const uint8_t* __restrict__ D,
                                                     int64_t ldd, const float* sD, float slope,
                                                     float* __restrict__ e_pre, float* __restrict__ el) {
  const float s1 = *sS, s2 = *sD;
  const int lane = threadIdx.x & 31;
  const int64_t E = g.in_ptr[g.n_local];
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t item = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); item * 32 * ADD_PER < E;
       item += nw) {
    const int64_t e0 = item * 32 * ADD_PER;
    int64_t v = row_of(g.in_ptr, g.n_local, min(E - 1, e0 + lane));
    int64_t vend = __ldg(g.in_ptr + v + 1);
#pragma unroll 2
    for (int i = 0; i < ADD_PER; ++i) {
      const int64_t e = e0 + lane + 32 * i;
      if (e >= E) continue;
      while (vend <= e) { ++v; vend = __ldg(g.in_ptr + v + 1); }
      const uint8_t* srow = S + (int64_t)__ldg(g.in_src + e) * lds;
      const uint8_t* drow = D + (g.row_begin + v) * ldd;
      for (int h = 0; h < heads; ++h) {
        const float x = __fadd_rn(__fmul_rn(__int2float_rn(code_at<BITS>(srow, h)), s1),
                                  __fmul_rn(__int2float_rn(code_at<BITS>(drow, h)), s2));
        if (e_pre) e_pre[e * heads + h] = x;
        if (el) el[e * heads + h] = x > 0.0f ? x : __fmul_rn(x, slope);
      }
    }
  }
}

static int warp_grid(int64_t warps) {
  int64_t g = (warps + 7) / 8;
  const int64_t cap = (int64_t)num_sms() * 16;
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace tango

using namespace tango;

namespace {
GraphDev graph_dev(const tango_graph* G) {
  GraphDev g;
  g.n_local = G->row_end - G->row_begin;
  g.row_begin = G->row_begin;
  g.n_global = G->n_global;
  g.in_ptr = G->in_ptr; g.in_src = G->in_src;
  g.out_ptr = G->out_ptr; g.out_dst = G->out_dst; g.out_eid = G->out_eid;
  g.chunk = G->chunk_edges > 0 ? G->chunk_edges : 256;
  return g;
}
}  // namespace

extern "C" {

tango_status tango_quantize_int4(const float* x, int64_t rows, int64_t cols, int64_t global_row0,
                                 const float* amax_hint, tango_rng rng, uint8_t* q, int64_t ld_bytes, float* scale_out,
                                 float* amax_out, int32_t* dev_status, cudaStream_t stream) {
  if (rows < 0 || cols < 0 || global_row0 < 0) return TANGO_ERR_SHAPE;
  if ((cols & 7) != 0 || ld_bytes < cols / 2 || (ld_bytes & 3) != 0) return TANGO_ERR_SHAPE;
  if (!scale_out || !amax_out) return TANGO_ERR_INVALID_ARG;
  if (rows > 0 && cols > 0 && (!x || !q)) return TANGO_ERR_INVALID_ARG;
  if ((reinterpret_cast<uintptr_t>(x) & 15) != 0 || (reinterpret_cast<uintptr_t>(q) & 3) != 0)
    return TANGO_ERR_INVALID_ARG;
  unsigned* slot = reinterpret_cast<unsigned*>(amax_out);
  if (amax_hint) {
    if (cudaMemcpyAsync(slot, amax_hint, sizeof(float), cudaMemcpyDeviceToDevice, stream) != cudaSuccess)
      return TANGO_ERR_CUDA;
  } else {
    if (cudaMemsetAsync(slot, 0, sizeof(float), stream) != cudaSuccess) return TANGO_ERR_CUDA;
    if (launch_absmax(x, rows, cols, nullptr, slot, stream) != cudaSuccess) return TANGO_ERR_CUDA;
  }
  const int64_t groups = rows * (cols >> 3);
  int64_t grid = (groups + 255) / 256;
  if (grid > (int64_t)num_sms() * 16) grid = (int64_t)num_sms() * 16;
  if (grid < 1) grid = 1;
  {
    ProfScope ps("quantize_int4", stream);
    k_quantize_pack4<<<(unsigned)grid, 256, 0, stream>>>(x, rows, cols, global_row0 * cols, slot,
                                                         philox_key(rng.seed), rng.step, rng.tag, q, ld_bytes,
                                                         scale_out, dev_status);
  }
  return cudaGetLastError() == cudaSuccess ? TANGO_OK : TANGO_ERR_CUDA;
}

tango_status tango_sddmm_qn(const tango_graph* G, int32_t op, int32_t bits, const void* Xsrc, int64_t ld_src,
                            const float* s_src, const void* Xdst, int64_t ld_dst, const float* s_dst, int32_t heads,
                            int32_t cols, float slope, float* out0, float* out1, cudaStream_t stream) {
  if (!G || !Xsrc || !Xdst || !s_src || !s_dst || !out0) return TANGO_ERR_INVALID_ARG;
  if (bits != 8 && bits != 4) return TANGO_ERR_BITS;
  if (heads <= 0 || cols <= 0 || cols % heads != 0) return TANGO_ERR_SHAPE;
  if (G->row_end < G->row_begin || G->n_global < G->row_end) return TANGO_ERR_SHAPE;
  const GraphDev g = graph_dev(G);
  if (g.n_local == 0) return TANGO_OK;
  if (!G->in_ptr || (G->e_in > 0 && !G->in_src)) return TANGO_ERR_INVALID_ARG;
  const int64_t row_bytes = bits == 8 ? cols : (cols + 1) / 2;
  if (ld_src < row_bytes || ld_dst < row_bytes) return TANGO_ERR_SHAPE;
  if (op == TANGO_SDDMM_DOT) {
    const int per_word = 32 / bits;
    const int words = cols / per_word;
    const int gsz = words / (heads > 0 ? heads : 1);
    if (cols % per_word != 0 || words % heads != 0 || words > 128 || (gsz & (gsz - 1)) != 0 || (ld_src & 3) != 0 ||
        (ld_dst & 3) != 0)
      return TANGO_ERR_UNSUPPORTED;
    ProfScope ps(bits == 8 ? "sddmm_dot_i8" : "sddmm_dot_i4", stream);
    const uint32_t* A = static_cast<const uint32_t*>(Xdst);
    const uint32_t* B = static_cast<const uint32_t*>(Xsrc);
    const int nch = (words + 31) / 32;
    const int grid = warp_grid((G->e_in + DOT_RUN - 1) / DOT_RUN);
#define DOTW(BITS_, NCH_, GSZ_) \
    k_sddmm_dot_e<BITS_, NCH_, GSZ_><<<grid, 256, 0, stream>>>(g, heads, words, A, ld_dst / 4, s_dst, B, ld_src / 4, \
                                                            s_src, out0)
#define DOTG(BITS_, NCH_)                                             \
    switch (gsz) {                                                    \
      case 1: DOTW(BITS_, NCH_, 1); break;                            \
      case 2: DOTW(BITS_, NCH_, 2); break;                            \
      case 4: DOTW(BITS_, NCH_, 4); break;                            \
      case 8: DOTW(BITS_, NCH_, 8); break;                            \
      case 16: DOTW(BITS_, NCH_, 16); break;                          \
      case 32: DOTW(BITS_, NCH_, 32); break;                          \
      case 64: DOTW(BITS_, NCH_, 64); break;                          \
      default: DOTW(BITS_, NCH_, 128); break;                         \
    }
    if (bits == 8) {
      if (nch == 1) { DOTG(8, 1) } else if (nch == 2) { DOTG(8, 2) } else { DOTG(8, 4) }
    } else {
      if (nch == 1) { DOTG(4, 1) } else if (nch == 2) { DOTG(4, 2) } else { DOTG(4, 4) }
    }
#undef DOTG
#undef DOTW
  } else if (op == TANGO_SDDMM_ADD) {
    if (cols != heads) return TANGO_ERR_SHAPE;
    ProfScope ps(bits == 8 ? "sddmm_add_i8" : "sddmm_add_i4", stream);
    const uint8_t* S = static_cast<const uint8_t*>(Xsrc);
    const uint8_t* D = static_cast<const uint8_t*>(Xdst);
    const int grid = warp_grid((G->e_in + 32 * ADD_PER - 1) / (32 * ADD_PER));
    if (bits == 8)
      k_sddmm_add_e<8><<<grid, 256, 0, stream>>>(g, heads, S, ld_src, s_src, D, ld_dst, s_dst, slope, out0, out1);
    else
      k_sddmm_add_e<4><<<grid, 256, 0, stream>>>(g, heads, S, ld_src, s_src, D, ld_dst, s_dst, slope, out0, out1);
  } else {
    return TANGO_ERR_INVALID_ARG;
  }
  return cudaGetLastError() == cudaSuccess ? TANGO_OK : TANGO_ERR_CUDA;
}

}  // extern "C"
