// common.cuh — device helpers shared by the libtango kernels (sm_100a only).
//
// Independent of oracle/: the Philox stream, the stochastic-rounding step and
// the pinned exponential are written here from the paper / DESIGN.md readings,
// not from the oracle's source.  All fp32 arithmetic that feeds a value compared
// bit-for-bit with the oracle uses explicit round-to-nearest intrinsics
// (__fmul_rn, __fadd_rn, __fmaf_rn, __fdiv_rn, __int2float_rn) so that nvcc
// never contracts or reorders it.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda.h>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libtango is written for sm_100a only"
#endif

namespace tango {

constexpr int kWarp = 32;

// ------------------------------------------------------------------ status codes (mirror tango.h)
enum : int32_t { ST_OK = 0, ST_NONFINITE = 4 };

// ------------------------------------------------------------------ Philox4x32-10 (reading R5)
struct u32x4 { uint32_t x, y, z, w; };

// Round keys of Philox4x32-10 for a 64-bit seed (k0 = lo32, k1 = hi32, bumped by the Weyl constants
// after each round), precomputed on the host so kernels read them as constant-bank operands.
struct PhiloxKey { uint32_t k0[10], k1[10]; };
__host__ __device__ inline PhiloxKey philox_key(uint64_t seed) {
  PhiloxKey K;
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  for (int r = 0; r < 10; ++r) {
    K.k0[r] = k0; K.k1[r] = k1;
    k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
  }
  return K;
}
__device__ __forceinline__ u32x4 philox10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, const PhiloxKey& K) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    const uint32_t n0 = hi1 ^ c1 ^ K.k0[r], n2 = hi0 ^ c3 ^ K.k1[r];
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
  }
  return {c0, c1, c2, c3};
}

// The 8 16-bit uniforms of the group of 8 consecutive elements starting at global index g8 = 8*blk
// (reading R4): element j of the group takes half-word j: word j>>1, low half for even j.
struct SR8 { uint32_t w[4]; };
__device__ __forceinline__ SR8 sr_draw8(uint64_t blk, uint32_t tag, uint32_t step, const PhiloxKey& K) {
  u32x4 r = philox10((uint32_t)blk, (uint32_t)(blk >> 32), tag, step, K);
  SR8 s;
  s.w[0] = r.x; s.w[1] = r.y; s.w[2] = r.z; s.w[3] = r.w;
  return s;
}
__device__ __forceinline__ uint32_t sr_half(const SR8& s, int j) {
  const uint32_t word = s.w[j >> 1];
  return (j & 1) ? (word >> 16) : (word & 0xFFFFu);
}

// Stochastic rounding of x*r (reading R4/R6): q = floor(xs) + (u < xs - floor(xs)), clamped to ±qmax,
// u = hw16 * 2^-16.  Evaluated on the FMA/ALU pipes only (no XU conversions), bit-identical to the
// plain definition (all steps exact, |xs| < 2^22):
//   t  = fl_rd(xs + 1.5*2^23)  -> bits 0x4B400000 + floor(xs)
//   f  = t - 1.5*2^23, fr = fl(xs - f)                  (fr exactly as in the definition)
//   u < fr  <=>  hw16 < fr*2^16  <=>  2^23 + hw16 < fl_ru(fr*2^16 + 2^23)  (= 2^23 + ceil(fr*2^16))
// with kf = 2^23 + hw16 built by one PRMT; the sign bit of kf - rhs (exact) is the carry into q.
// Returns the bits 0x4B400000 + q (low byte = the int8 code).
__device__ __forceinline__ uint32_t sr_qbits(float x, float r, float kf /* 2^23 + hw16 */, int qmax) {
  const float xs = __fmul_rn(x, r);
  const float t = __fadd_rd(xs, 12582912.0f);
  const float f = __fsub_rn(t, 12582912.0f);
  const float fr = __fsub_rn(xs, f);
  const float rhs = __fmaf_ru(fr, 65536.0f, 8388608.0f);
  const uint32_t up = __float_as_uint(__fsub_rn(kf, rhs)) >> 31;
  int qb = (int)(__float_as_uint(t) + up);
  qb = min(max(qb, 0x4B400000 - qmax), 0x4B400000 + qmax);
  return (uint32_t)qb;
}
// 2^23 + (half-word j of the group's Philox output), as a float (one PRMT)
__device__ __forceinline__ float sr_kf(const SR8& s, int j) {
  return __uint_as_float(__byte_perm(s.w[j >> 1], 0x4B000000u, (j & 1) ? 0x7632u : 0x7610u));
}
__device__ __forceinline__ uint32_t pack4_low_bytes(uint32_t b0, uint32_t b1, uint32_t b2, uint32_t b3) {
  return __byte_perm(__byte_perm(b0, b1, 0x0040u), __byte_perm(b2, b3, 0x0040u), 0x5410u);
}
// Packed-pair form of sr_qbits on the f32x2 pipes (FMUL2 / FADD2 / FFMA2 with the same rounding
// modes, one instruction per two elements): identical results element by element.
__device__ __forceinline__ uint64_t pk2(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void sr_qbits2(float x0, float x1, float r, float kf0, float kf1, int qmax, uint32_t& q0,
                                          uint32_t& q1) {
  const uint64_t M = pk2(12582912.0f, 12582912.0f), R = pk2(r, r), K = pk2(kf0, kf1);
  const uint64_t S = pk2(65536.0f, 65536.0f), T23 = pk2(8388608.0f, 8388608.0f);
  uint64_t xs, t, f, fr, rhs, d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(xs) : "l"(pk2(x0, x1)), "l"(R));
  asm("add.rm.f32x2 %0, %1, %2;" : "=l"(t) : "l"(xs), "l"(M));
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(f) : "l"(t), "l"(M));
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(fr) : "l"(xs), "l"(f));
  asm("fma.rp.f32x2 %0, %1, %2, %3;" : "=l"(rhs) : "l"(fr), "l"(S), "l"(T23));
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(K), "l"(rhs));
  const uint32_t t0 = (uint32_t)t, t1 = (uint32_t)(t >> 32);
  const uint32_t u0 = (uint32_t)d >> 31, u1 = (uint32_t)(d >> 63);
  int a0 = (int)(t0 + u0), a1 = (int)(t1 + u1);
  a0 = min(max(a0, 0x4B400000 - qmax), 0x4B400000 + qmax);
  a1 = min(max(a1, 0x4B400000 - qmax), 0x4B400000 + qmax);
  q0 = (uint32_t)a0;
  q1 = (uint32_t)a1;
}
// SR of 8 consecutive elements sharing one Philox draw -> 8 codes packed little-endian
__device__ __forceinline__ uint2 sr_quant8(const float (&v)[8], float r, const SR8& rnd, int qmax) {
  uint32_t b[8];
#pragma unroll
  for (int k = 0; k < 8; k += 2) sr_qbits2(v[k], v[k + 1], r, sr_kf(rnd, k), sr_kf(rnd, k + 1), qmax, b[k], b[k + 1]);
  return make_uint2(pack4_low_bytes(b[0], b[1], b[2], b[3]), pack4_low_bytes(b[4], b[5], b[6], b[7]));
}
__device__ __forceinline__ int sr_quant(float x, float r, uint32_t hw16, int qmax) {
  return (int)sr_qbits(x, r, __uint_as_float(0x4B000000u | hw16), qmax) - 0x4B400000;
}

// Scale pair from amax (reading R1/R3/R7): s = amax/qmax, r = qmax/amax; amax = 0 -> s = r = 1.
struct Scale { float s, r; bool bad; };
__device__ __forceinline__ Scale scale_from_amax(float amax, int bits) {
  Scale sc;
  const float qmax = (float)((1 << (bits - 1)) - 1);
  sc.bad = !(amax <= 3.4028234663852886e38f);
  if (amax == 0.0f || sc.bad) { sc.s = 1.0f; sc.r = 1.0f; }
  else { sc.s = __fdiv_rn(amax, qmax); sc.r = __fdiv_rn(qmax, amax); }
  return sc;
}
__device__ __forceinline__ float amax_load(const unsigned* bits) { return __uint_as_float(*(volatile const unsigned*)bits); }

// Pinned exponential exp_p (reading R13), argument <= 0.
__device__ __forceinline__ float exp_p(float x) {
  const float t = __fmul_rn(x, 0x1.715476p+0f);
  if (t < -125.0f) return 0.0f;
  const float n = rintf(t);
  const float f = __fsub_rn(t, n);
  float p = 0x1.430912p-13f;
  p = __fmaf_rn(p, f, 0x1.5d87fep-10f);
  p = __fmaf_rn(p, f, 0x1.3b2ab6p-7f);
  p = __fmaf_rn(p, f, 0x1.c6b08ep-5f);
  p = __fmaf_rn(p, f, 0x1.ebfbep-3f);
  p = __fmaf_rn(p, f, 0x1.62e43p-1f);
  p = __fmaf_rn(p, f, 0x1p+0f);
  // ldexp(p, n): p in [0.70, 1.42] and n >= -125 keep the result normal -> add n to the exponent field
  return __int_as_float(__float_as_int(p) + ((int)n << 23));
}

// LeakyReLU of the SDDMM-add result (reading R11)
__device__ __forceinline__ float lrelu(float x, float slope) { return x > 0.0f ? x : __fmul_rn(x, slope); }

// ------------------------------------------------------------------ reductions
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
// atomicMax on the bit pattern of a non-negative float (NaN/Inf patterns order above finite ones)
__device__ __forceinline__ void atomic_max_abs(unsigned* slot, float v_abs) {
  atomicMax(slot, __float_as_uint(v_abs));
}

// int8 x16 -> exact fp32 via the magic-number trick: (b ^ 0x80) | 0x4B000000 = 2^23 + 128 + b
__device__ __forceinline__ float i8_to_f(uint32_t word, int byte) {
  const uint32_t b = (word >> (8 * byte)) & 0xFFu;
  return __fsub_rn(__uint_as_float(0x4B000000u | (b ^ 0x80u)), 8388736.0f);
}

// ------------------------------------------------------------------ PTX: mbarrier / TMA / tcgen05
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_async_shared() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  while (!mbar_try_wait(a, parity)) {
  }
}

__device__ __forceinline__ void mbar_wait_addr(uint32_t a, uint32_t parity) {
  while (!mbar_try_wait(a, parity)) {
  }
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[smem] · B[smem], int8 x int8 -> int32 (kind::i8), single CTA.
__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(
          d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// 32 lanes x 32 consecutive 32-bit columns: thread t of the warp gets row (lane_base + t), columns [col, col+32).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// UMMA shared-memory descriptor (sm_100 "version 1"): start, LBO, SBO (bytes), layout type (2 = SWIZZLE_128B).
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(layout & 7u) << 61;
  return d;
}
// Instruction descriptor for kind::i8: D = S32, A = B = signed int8, K- or MN-major, M x N.
__host__ __device__ constexpr uint32_t make_idesc_i8(int M, int N, bool a_mn, bool b_mn) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ int warp_id() { return __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0); }

}  // namespace tango
