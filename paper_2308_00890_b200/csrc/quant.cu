// quant.cu — dedicated quantization pass (§3.3: "a dedicated quantization kernel would
// read 32-bit input floating-point matrices sequentially once and write the 8-bit quantized
// matrices out, again, sequentially and once") with tensor-level dynamic symmetric scaling
// and Philox stochastic rounding (Eq.3; readings R1-R7).
//
// Two kernels: k_absmax (HBM-bound read, warp/block max + one atomicMax per block) and
// k_quantize (one Philox call per group of 8 consecutive elements, 16-B loads, 8-B stores).
#include "kernels.h"

namespace tango {

// amax over |x * rowscale[row]| (rowscale optional, reading R26 for GCN's Gs = dout*nd)
__global__ void __launch_bounds__(256) k_absmax(const float* __restrict__ x, int64_t rows, int64_t cols,
                                                const float* __restrict__ rowscale, unsigned* __restrict__ slot) {
  const int64_t count = rows * cols;
  float m = 0.0f;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  if (rowscale == nullptr && (reinterpret_cast<uintptr_t>(x) & 15) == 0) {
    const int64_t n4 = count >> 2;
    const float4* x4 = reinterpret_cast<const float4*>(x);
    for (int64_t i = tid; i < n4; i += nthr) {
      float4 v = __ldg(x4 + i);
      m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
      // NaN must dominate: fmaxf drops NaN, so fold it explicitly
      if (!(fabsf(v.x) <= 3.4e38f) || !(fabsf(v.y) <= 3.4e38f) || !(fabsf(v.z) <= 3.4e38f) ||
          !(fabsf(v.w) <= 3.4e38f))
        m = __uint_as_float(0x7FC00000u);
    }
    for (int64_t i = (n4 << 2) + tid; i < count; i += nthr) {
      float a = fabsf(x[i]);
      m = (a <= 3.4e38f) ? fmaxf(m, a) : __uint_as_float(0x7FC00000u);
    }
  } else {
    for (int64_t i = tid; i < count; i += nthr) {
      float v = x[i];
      if (rowscale) v = __fmul_rn(v, rowscale[i / cols]);
      float a = fabsf(v);
      m = (a <= 3.4e38f) ? fmaxf(m, a) : __uint_as_float(0x7FC00000u);
    }
  }
  // block reduce on bit patterns (non-negative floats and NaN order as unsigned)
  unsigned b = __float_as_uint(m);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) b = max(b, __shfl_xor_sync(0xffffffffu, b, o));
  __shared__ unsigned red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = b;
  __syncthreads();
  if (threadIdx.x < 32) {
    b = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) b = max(b, __shfl_xor_sync(0xffffffffu, b, o));
    if (threadIdx.x == 0) atomicMax(slot, b);
  }
}

// q[i][j] = SR(x[i][j] * rowscale[i] * r) for the logical tensor rows x cols whose element (i, j)
// has global index g = g0 + i*cols + j.  Out: q[i*ld + j] (and, if qt, the transpose qt[j*ldt + i]).
__global__ void __launch_bounds__(256) k_quantize(const float* __restrict__ x, int64_t rows, int64_t cols,
                                                  const float* __restrict__ rowscale, int64_t g0,
                                                  const unsigned* __restrict__ amax_slot, int bits, const PhiloxKey key,
                                                  uint32_t step, uint32_t tag, int8_t* __restrict__ q, int64_t ld,
                                                  int8_t* __restrict__ qt, int64_t ldt, float* __restrict__ scale_out,
                                                  int32_t* __restrict__ status, uint32_t code_xor) {
  const Scale sc = scale_from_amax(amax_load(amax_slot), bits);
  const int qmax = (1 << (bits - 1)) - 1;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (tid == 0) {
    if (scale_out) *scale_out = sc.s;
    if (sc.bad && status) atomicExch(status, ST_NONFINITE);
  }
  const int64_t count = rows * cols;
  const int64_t blk0 = g0 >> 3, blk1 = (g0 + count + 7) >> 3;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  const bool aligned = (rowscale == nullptr) && (qt == nullptr) && ((g0 & 7) == 0) && ((ld & 7) == 0) &&
                       ((reinterpret_cast<uintptr_t>(x) & 15) == 0) && ((reinterpret_cast<uintptr_t>(q) & 7) == 0);
  const bool fast = aligned && ((cols & 7) == 0);
  const bool dense = ld == cols;   // q[i*ld + j] = q[e]: no division in the fast loop
  const bool aligned_x = (rowscale == nullptr) && (qt == nullptr) && ((g0 & 7) == 0) &&
                         ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
  if (aligned_x && !dense && (cols & 7) != 0) {
    // padded output rows whose width is not a multiple of 8 (e.g. F = 602 -> ld 608): stream x as one flat
    // run of 8-element groups (the same Philox groups) and scatter each group's codes to (i, j); the row
    // coordinates of the thread's group advance by a fixed (si, sj) per grid stride, no division in the loop
    const int64_t full1 = blk0 + (count >> 3);
    const int64_t e0 = tid << 3, stride = nthr << 3;
    int64_t ci = e0 / cols, cj = e0 - ci * cols;
    const int64_t si = stride / cols, sj = stride - si * cols;
    for (int64_t blk = blk0 + tid; blk < full1; blk += nthr) {
      const int64_t e = (blk << 3) - g0;
      const float4* src = reinterpret_cast<const float4*>(x + e);
      const float4 a = __ldcs(src), b = __ldcs(src + 1);
      const SR8 rnd = sr_draw8((uint64_t)blk, tag, step, key);
      const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
      uint2 pk = sr_quant8(v, sc.r, rnd, qmax);
      pk.x ^= code_xor; pk.y ^= code_xor;
      const uint32_t w2[2] = {pk.x, pk.y};
      int64_t i = ci, j = cj;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (j == cols) { j = 0; ++i; }
        q[i * ld + j] = (int8_t)(w2[k >> 2] >> (8 * (k & 3)));
        ++j;
      }
      cj += sj; ci += si;
      if (cj >= cols) { cj -= cols; ++ci; }
    }
    if ((count & 7) && tid == nthr - 1) {   // the partial last group, element by element
      const SR8 rnd = sr_draw8((uint64_t)full1, tag, step, key);
      for (int k = 0; k < (int)(count & 7); ++k) {
        const int64_t e = ((full1 << 3) - g0) + k;
        const int64_t i = e / cols, j = e - i * cols;
        const int qq = sr_quant(x[e], sc.r, sr_half(rnd, k), qmax);
        q[i * ld + j] = (int8_t)(qq ^ (int)(code_xor & 0xFFu));
      }
    }
    return;
  }
  if (aligned && dense) {
    // streaming path over the whole groups (any cols: the tensor is one flat run of codes); the
    // next group's 32 bytes are loaded before this one is rounded.  A partial last group (count
    // not a multiple of 8) is rounded element by element by one thread.
    const int64_t full1 = blk0 + (count >> 3);
    if ((count & 7) && tid == nthr - 1) {
      const SR8 rnd = sr_draw8((uint64_t)full1, tag, step, key);
      for (int k = 0; k < (int)(count & 7); ++k) {
        const int64_t e = ((full1 << 3) - g0) + k;
        const int qq = sr_quant(x[e], sc.r, sr_half(rnd, k), qmax);
        q[e] = (int8_t)(qq ^ (int)(code_xor & 0xFFu));
      }
    }
    const int64_t blk1 = full1;
    int64_t blk = blk0 + tid;
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
    if (blk < blk1) {
      const float4* src = reinterpret_cast<const float4*>(x + ((blk << 3) - g0));
      a = __ldcs(src); b = __ldcs(src + 1);
    }
    for (; blk < blk1; blk += nthr) {
      const int64_t nb = blk + nthr;
      float4 na = a, nbv = b;
      if (nb < blk1) {
        const float4* src = reinterpret_cast<const float4*>(x + ((nb << 3) - g0));
        na = __ldcs(src); nbv = __ldcs(src + 1);
      }
      const SR8 rnd = sr_draw8((uint64_t)blk, tag, step, key);
      const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
      uint2 pk = sr_quant8(v, sc.r, rnd, qmax);
      pk.x ^= code_xor; pk.y ^= code_xor;
      *reinterpret_cast<uint2*>(q + ((blk << 3) - g0)) = pk;
      a = na; b = nbv;
    }
    return;
  }
  for (int64_t blk = blk0 + tid; blk < blk1; blk += nthr) {
    const SR8 rnd = sr_draw8((uint64_t)blk, tag, step, key);
    const int64_t gs = blk << 3;
    if (fast) {
      const int64_t e = gs - g0;  // first local element, multiple of 8, within one row
      int64_t i = 0, j = e;
      if (!dense) {
        i = e / cols;
        j = e - i * cols;
      }
      const float4* src = reinterpret_cast<const float4*>(x + e);
      const float4 a = __ldg(src), b = __ldg(src + 1);
      const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
      uint2 pk = sr_quant8(v, sc.r, rnd, qmax);
      pk.x ^= code_xor; pk.y ^= code_xor;
      *reinterpret_cast<uint2*>(q + i * ld + j) = pk;
    } else {
#pragma unroll 1
      for (int k = 0; k < 8; ++k) {
        const int64_t g = gs + k;
        if (g < g0 || g >= g0 + count) continue;
        const int64_t e = g - g0;
        const int64_t i = e / cols, j = e - i * cols;
        float v = x[e];
        if (rowscale) v = __fmul_rn(v, rowscale[i]);
        const int qq = sr_quant(v, sc.r, sr_half(rnd, k), qmax);
        if (q) q[i * ld + j] = (int8_t)(qq ^ (int)(code_xor & 0xFFu));
        if (qt) qt[j * ldt + i] = (int8_t)qq;
      }
    }
  }
}

// ------------------------------------------------------------------ launchers
static int grid_for(int64_t work, int threads, int per_sm = 8) {
  int64_t g = (work + threads - 1) / threads;
  const int64_t cap = (int64_t)num_sms() * per_sm;
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

cudaError_t launch_absmax(const float* x, int64_t rows, int64_t cols, const float* rowscale, unsigned* slot,
                          cudaStream_t st) {
  if (rows * cols == 0) return cudaSuccess;
  ProfScope ps("absmax", st);
  k_absmax<<<grid_for(rows * cols / 4 + 1, 256), 256, 0, st>>>(x, rows, cols, rowscale, slot);
  return cudaGetLastError();
}

cudaError_t launch_quantize(const float* x, int64_t rows, int64_t cols, const float* rowscale, int64_t g0,
                            const unsigned* amax_slot, int bits, uint64_t seed, uint32_t step, uint32_t tag,
                            int8_t* q, int64_t ld, int8_t* qt, int64_t ldt, float* scale_out, int32_t* status,
                            cudaStream_t st, uint32_t code_xor) {
  const int64_t count = rows * cols;
  if (count == 0) {
    if (scale_out) {
      // empty tensor: amax = 0 -> s = 1 (reading R7)
      const float one = 1.0f;
      return cudaMemcpyAsync(scale_out, &one, sizeof(float), cudaMemcpyHostToDevice, st);
    }
    return cudaSuccess;
  }
  if (q && ld > cols) {
    cudaError_t e = cudaMemset2DAsync(q + cols, (size_t)ld, 0, (size_t)(ld - cols), (size_t)rows, st);
    if (e != cudaSuccess) return e;
  }
  if (qt && ldt > rows) {
    cudaError_t e = cudaMemset2DAsync(qt + rows, (size_t)ldt, 0, (size_t)(ldt - rows), (size_t)cols, st);
    if (e != cudaSuccess) return e;
  }
  const int64_t groups = (count + 15) / 8;
  ProfScope ps("quantize", st);
  k_quantize<<<grid_for(groups, 256, 16), 256, 0, st>>>(x, rows, cols, rowscale, g0, amax_slot, bits, philox_key(seed), step, tag,
                                                       q, ld, qt, ldt, scale_out, status, code_xor);
  return cudaGetLastError();
}

// in place: the amax held (as float bits) in `slot` -> its scale s = amax/qmax (reading R1/R7); used when a
// caller of tango_quantize gives no amax slot, so the scale word doubles as the amax scratch
__global__ void k_amax_to_scale(float* slot, int bits) {
  *slot = scale_from_amax(amax_load(reinterpret_cast<const unsigned*>(slot)), bits).s;
}
cudaError_t launch_amax_to_scale(float* slot, int bits, cudaStream_t st) {
  ProfScope ps("amax_to_scale", st);
  k_amax_to_scale<<<1, 1, 0, st>>>(slot, bits);
  return cudaGetLastError();
}

}  // namespace tango

// ================================================================== Error_X and bit selection (NEXT-2)
namespace tango {
namespace {
// Eq.4 term with the reading-A24 denominator: |x − x̂| / (|x| + |x̂| + ε), ε = 0.0005, fp32 rn ops
__device__ __forceinline__ float error_term(float x, float xh) {
  return __fdiv_rn(fabsf(__fsub_rn(x, xh)), __fadd_rn(__fadd_rn(fabsf(x), fabsf(xh)), 0.0005f));
}
__device__ __forceinline__ double block_sum_d(double v) {
  __shared__ double red[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x < 32) {
    t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  }
  return t;   // valid in thread 0
}
}  // namespace

__global__ void __launch_bounds__(256) k_error_x(const float* __restrict__ x, int64_t rows, int64_t cols,
                                                 const int8_t* __restrict__ q, int64_t ld, const float* __restrict__ s,
                                                 double* __restrict__ sum) {
  const float sc = *s;
  const int64_t count = rows * cols;
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols, c = i - r * cols;
    acc += (double)error_term(x[i], __fmul_rn((float)q[r * ld + c], sc));
  }
  acc = block_sum_d(acc);
  if (threadIdx.x == 0) atomicAdd(sum, acc);
}
// nb bit widths at once (nearest rounding, reading R31): one pass over x
template <int NB>
__global__ void __launch_bounds__(256) k_select_bits_sweep(const float* __restrict__ x, int64_t count, int bmin,
                                                           const int32_t* __restrict__ amax_bits,
                                                           double* __restrict__ sums) {
  const float amax = __int_as_float(*amax_bits);
  float s[NB], r[NB], qm[NB];
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const Scale sc = scale_from_amax(amax, bmin + b);
    s[b] = sc.s; r[b] = sc.r; qm[b] = (float)((1 << (bmin + b - 1)) - 1);
  }
  double acc[NB];
#pragma unroll
  for (int b = 0; b < NB; ++b) acc[b] = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    const float v = x[i];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const float q = fminf(fmaxf(rintf(__fmul_rn(v, r[b])), -qm[b]), qm[b]);
      acc[b] += (double)error_term(v, __fmul_rn(q, s[b]));
    }
  }
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const double t = block_sum_d(acc[b]);
    if (threadIdx.x == 0) atomicAdd(sums + b, t);
  }
}
__global__ void k_select_bits_final(double* errs, int nb, int bmin, int64_t count, float threshold, int32_t* bits) {
  int chosen = -1;
  for (int b = 0; b < nb; ++b) {
    errs[b] = count > 0 ? errs[b] / (double)count : 0.0;
    if (chosen < 0 && errs[b] <= (double)threshold) chosen = bmin + b;
  }
  *bits = chosen < 0 ? -(bmin + nb - 1) : chosen;   // negative: no width met the threshold (|value| = bmax)
}
__global__ void k_div_count(double* v, int64_t count) { *v = count > 0 ? *v / (double)count : 0.0; }

cudaError_t launch_error_x(const float* x, int64_t rows, int64_t cols, const int8_t* q, int64_t ld, const float* s,
                           double* err, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(err, 0, sizeof(double), st);
  if (e != cudaSuccess) return e;
  if (rows * cols > 0) {
    ProfScope ps("error_x", st);
    k_error_x<<<grid_for(rows * cols, 256), 256, 0, st>>>(x, rows, cols, q, ld, s, err);
  }
  k_div_count<<<1, 1, 0, st>>>(err, rows * cols);
  return cudaGetLastError();
}
cudaError_t launch_select_bits(const float* x, int64_t count, float threshold, int bmin, int bmax, double* errs,
                               int32_t* bits, cudaStream_t st) {
  const int nb = bmax - bmin + 1;
  cudaError_t e = cudaMemsetAsync(errs, 0, sizeof(double) * nb, st);
  if (e != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(bits, 0, sizeof(int32_t), st)) != cudaSuccess) return e;
  if (count > 0) {
    // amax into *bits (float bit pattern, non-negative: unsigned max == float max), then the sweep
    if ((e = launch_absmax(x, count, 1, nullptr, reinterpret_cast<unsigned*>(bits), st)) != cudaSuccess) return e;
    ProfScope ps("select_bits", st);
    switch (nb) {
#define NB_CASE(K) case K: k_select_bits_sweep<K><<<grid_for(count, 256), 256, 0, st>>>(x, count, bmin, bits, errs); break;
      NB_CASE(1) NB_CASE(2) NB_CASE(3) NB_CASE(4) NB_CASE(5) NB_CASE(6) NB_CASE(7)
#undef NB_CASE
      default: return cudaErrorInvalidValue;
    }
  }
  k_select_bits_final<<<1, 1, 0, st>>>(errs, nb, bmin, count, threshold, bits);
  return cudaGetLastError();
}
}  // namespace tango
