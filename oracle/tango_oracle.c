/*
 * tango_oracle.c — CPU ORACLE for the quantized GAT / GCN layer of Tango
 * (arXiv 2308.00890, SC'23).  TEST INFRASTRUCTURE ONLY: it may be built and
 * called only by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg.  The product path (paper_2308_00890_b200) never links,
 * imports or executes anything under oracle/.  It shares no code, header,
 * table or constant generator with the CUDA path.
 *
 * Plain, slow, obviously correct.  Every floating-point operation is IEEE
 * binary32 round-to-nearest, in the order written below (build flags
 * -O2 -ffp-contract=off -fno-fast-math); fmaf() only where written.  Each
 * function cites the PAPER.md passage (P:line, section/equation) it follows
 * and the DESIGN.md reading (R#) that fixes what the paper leaves open.
 *
 * "bits == 0" is BYPASS mode: no quantization (codes are the fp32 values
 * themselves, scale 1, integer contractions become double-accumulated float
 * contractions).  It exists only so the oracle's backward formulas can be
 * pinned against fp64 autograd of the textbook layer (tests/test_oracle_*.py).
 *
 * Parity status: every function below is pinned by tests/test_oracle_*.py
 * except the value s_H' = 166.26 printed in Fig.4, which is not
 * reproducible from the text ("parity unpinned", R2).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>

/* chunk of the row/K-chunked FP32 sums of readings R33 and R39 (global rows) */
#define ORC_CK 1024
#endif

#define ORC_OK 0
#define ORC_ERR_NONFINITE 4
#define ORC_ERR_BITS 3
#define ORC_ERR_ALLOC 9

/* ------------------------------------------------------------------------- */
/* Philox4x32-10 (Salmon et al., SC'11 / Random123).  Replaces the paper's    */
/* xoshiro256++  per north_star: a counter-based stream keyed by   */
/* the global element index (reading R5).                                      */
/* ------------------------------------------------------------------------- */
void orc_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Uniform u in [0,1) with 16-bit resolution for global element index g
 * (reading R4): ctr = {lo32(g>>3), hi32(g>>3), tag, step}, key = seed;
 * element j = g&7 takes half-word j of the 128-bit Philox output. */
float orc_sr_uniform(uint64_t seed, uint32_t step, uint32_t tag, uint64_t g) {
  uint64_t blk = g >> 3;
  uint32_t ctr[4] = {(uint32_t)blk, (uint32_t)(blk >> 32), tag, step};
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t w[4];
  orc_philox4x32_10(ctr, key, w);
  uint32_t j = (uint32_t)(g & 7u);
  uint32_t word = w[j >> 1];
  uint32_t hw = (j & 1u) ? (word >> 16) : (word & 0xFFFFu);
  return (float)hw * 0x1p-16f;
}

/* ------------------------------------------------------------------------- */
/* Quantizer Q_B: symmetric, tensor-level, dynamic (§2.3, Eq.1 with */
/* Z=0), stochastic rounding (§3.2, Eq.3).  Readings R1,R3,R4,R6,R7: */
/*   s = amax/qmax, r = qmax/amax (IEEE divisions), x = X*r,                  */
/*   q = floor(x) + (u < x-floor(x)), clamped to [-qmax, qmax].              */
/* ------------------------------------------------------------------------- */
int orc_scale(float amax, int bits, float* s, float* r) {
  if (!(amax <= 3.4028234663852886e38f)) return ORC_ERR_NONFINITE; /* NaN or inf */
  float qmax = (float)((1 << (bits - 1)) - 1);
  if (amax == 0.0f) { *s = 1.0f; *r = 1.0f; return ORC_OK; }
  *s = amax / qmax;
  *r = qmax / amax;
  return ORC_OK;
}

float orc_absmax(const float* x, int64_t count, int* nonfinite) {
  float m = 0.0f;
  int bad = 0;
#pragma omp parallel for reduction(max : m) reduction(| : bad)
  for (int64_t i = 0; i < count; ++i) {
    float a = fabsf(x[i]);
    if (!(a <= 3.4028234663852886e38f)) bad = 1;
    else if (a > m) m = a;
  }
  *nonfinite = bad;
  return m;
}

/* Codes for a logical row-major tensor of `count` elements whose first element
 * has global index g0.  amax_in (nullable) overrides the tensor's own absmax
 * (used when the scale is global over partitions, reading R28). */
int orc_quantize(const float* x, int64_t count, int bits, uint64_t seed, uint32_t step, uint32_t tag,
                 int64_t g0, const float* amax_in, int8_t* q, float* s_out, float* amax_out) {
  if (bits < 2 || bits > 8) return ORC_ERR_BITS;
  int bad = 0;
  float amax = amax_in ? *amax_in : orc_absmax(x, count, &bad);
  if (bad) return ORC_ERR_NONFINITE;
  float s, r;
  int st = orc_scale(amax, bits, &s, &r);
  if (st) return st;
  int qmax = (1 << (bits - 1)) - 1;
#pragma omp parallel for
  for (int64_t i = 0; i < count; ++i) {
    float xs = x[i] * r;
    float f = floorf(xs);
    float fr = xs - f;
    float u = orc_sr_uniform(seed, step, tag, (uint64_t)(g0 + i));
    int qi = (int)f + (u < fr ? 1 : 0);
    if (qi > qmax) qi = qmax;
    if (qi < -qmax) qi = -qmax;
    q[i] = (int8_t)qi;
  }
  if (s_out) *s_out = s;
  if (amax_out) *amax_out = amax;
  return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* Error_X (§3.2 Eq.4) with the reading A24 denominator (SURVEY.md  */
/* §8(c.7)): Error_X = (1/N) Σ |X_i − X̂_i| / (|X_i| + |X̂_i| + ε), ε = 0.0005  */
/* ("Tango chooses ε = 0.0005"), X̂_i = i2f(q_i)·s.  Each term in fp32   */
/* (rn), the mean in fp64.  N = 0 -> 0.                                      */
/* ------------------------------------------------------------------------- */
float orc_error_term(float x, float xh) {
  float num = fabsf(x - xh);
  float den = (fabsf(x) + fabsf(xh)) + 0.0005f;
  return num / den;
}
double orc_error_x(const float* x, const int8_t* q, float s, int64_t count) {
  if (count <= 0) return 0.0;
  double acc = 0.0;
  for (int64_t i = 0; i < count; ++i) acc += (double)orc_error_term(x[i], (float)q[i] * s);
  return acc / (double)count;
}

/* select_bits (§3.2: "we compute Error_X of the output tensor of the first GNN layer",
 * "when Error_X < 0.3, Tango can maintain the accuracy ... we let Error_X = 0.3"): for every B in
 * [bmin, bmax] quantize X with NEAREST rounding (reading R31: the paper does not say which rounding
 * feeds Eq.4; nearest keeps the one-shot decision free of rounding noise), q = clamp(rintf(X*r_B)),
 * errs[B - bmin] = Error_X; returns the smallest B with Error_X <= threshold, or bmax if none
 * (*none = 1), in *bits.  Scales as orc_scale (amax over the whole tensor).  Returns a status. */
int orc_select_bits(const float* x, int64_t count, float threshold, int bmin, int bmax, double* errs, int* bits,
                    int* none) {
  int bad;
  float amax = orc_absmax(x, count, &bad);
  if (bad) return ORC_ERR_NONFINITE;
  if (bmin < 2 || bmax > 8 || bmin > bmax) return ORC_ERR_BITS;
  int chosen = -1;
  for (int B = bmin; B <= bmax; ++B) {
    float s, r;
    orc_scale(amax, B, &s, &r);
    const float qmax = (float)((1 << (B - 1)) - 1);
    double acc = 0.0;
    for (int64_t i = 0; i < count; ++i) {
      float q = rintf(x[i] * r);
      if (q > qmax) q = qmax;
      if (q < -qmax) q = -qmax;
      acc += (double)orc_error_term(x[i], q * s);
    }
    errs[B - bmin] = count > 0 ? acc / (double)count : 0.0;
    if (chosen < 0 && errs[B - bmin] <= (double)threshold) chosen = B;
  }
  *none = chosen < 0;
  *bits = chosen < 0 ? bmax : chosen;
  return ORC_OK;
}


/* ------------------------------------------------------------------------- */
/* Pinned exponential exp_p (reading R13): argument always <= 0.              */
/* t = x*log2(e); t < -125 -> 0; n = rint(t); f = t-n;                       */
/* p = Horner(c6..c0) with fmaf; result = ldexpf(p, n); c_k = (float)ln2^k/k! */
/* ------------------------------------------------------------------------- */
float orc_exp_p(float x) {
  const float c0 = 0x1p+0f, c1 = 0x1.62e43p-1f, c2 = 0x1.ebfbep-3f, c3 = 0x1.c6b08ep-5f;
  const float c4 = 0x1.3b2ab6p-7f, c5 = 0x1.5d87fep-10f, c6 = 0x1.430912p-13f;
  float t = x * 0x1.715476p+0f;
  if (t < -125.0f) return 0.0f;
  float n = rintf(t);
  float f = t - n;
  float p = c6;
  p = fmaf(p, f, c5);
  p = fmaf(p, f, c4);
  p = fmaf(p, f, c3);
  p = fmaf(p, f, c2);
  p = fmaf(p, f, c1);
  p = fmaf(p, f, c0);
  return ldexpf(p, (int)n);
}

/* ------------------------------------------------------------------------- */
/* Quantized-tensor view: codes (q != NULL) or, in bypass mode, fp32 values.  */
/* Dequantized element = QV(t,i) * t.s   (Eq.2, Z=0).              */
/* ------------------------------------------------------------------------- */
typedef struct { const int8_t* q; const float* v; float s; } orc_qref;
static inline float QV(orc_qref t, int64_t i) { return t.q ? (float)t.q[i] : t.v[i]; }

/* Graph view: in-CSR (rows = dst, src ascending), edge ids = in-CSR order.   */
typedef struct {
  int64_t n;
  int64_t e;
  const int64_t* in_ptr;
  const int32_t* in_src;
  int32_t chunk; /* C_E of the canonical chunked sum (reading R14) */
} orc_graph;

/* Out-edge view built here from the in-CSR (reading R14: source-major,
 * destinations ascending = stable counting sort of in-CSR positions by src). */
typedef struct { int64_t* ptr; int64_t* eid; int32_t* dst; } orc_rev;

static int orc_build_rev(const orc_graph* g, orc_rev* rv) {
  rv->ptr = (int64_t*)calloc((size_t)g->n + 1, sizeof(int64_t));
  rv->eid = (int64_t*)malloc(sizeof(int64_t) * (size_t)(g->e > 0 ? g->e : 1));
  rv->dst = (int32_t*)malloc(sizeof(int32_t) * (size_t)(g->e > 0 ? g->e : 1));
  if (!rv->ptr || !rv->eid || !rv->dst) return ORC_ERR_ALLOC;
  for (int64_t p = 0; p < g->e; ++p) rv->ptr[g->in_src[p] + 1]++;
  for (int64_t u = 0; u < g->n; ++u) rv->ptr[u + 1] += rv->ptr[u];
  int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)(g->n > 0 ? g->n : 1));
  if (!fill) return ORC_ERR_ALLOC;
  memcpy(fill, rv->ptr, sizeof(int64_t) * (size_t)g->n);
  for (int64_t v = 0; v < g->n; ++v)
    for (int64_t p = g->in_ptr[v]; p < g->in_ptr[v + 1]; ++p) {
      int64_t u = g->in_src[p];
      int64_t slot = fill[u]++;
      rv->eid[slot] = p;
      rv->dst[slot] = (int32_t)v;
    }
  free(fill);
  return ORC_OK;
}
static void orc_free_rev(orc_rev* rv) { free(rv->ptr); free(rv->eid); free(rv->dst); }

/* Canonical chunked sum Σᶜ (reading R14): consecutive chunks of C_E list
 * elements; within a chunk acc = 0 then acc += x (or fmaf); chunk partials are
 * combined left to right, total = partial_0, total = total + partial_c.
 * Implemented by the helpers below for a running list position `pos`. */
static inline void csum_fold(float* total, float* part, int64_t pos, int64_t chunk) {
  /* called before adding list element number `pos` */
  if (pos > 0 && pos % chunk == 0) {
    *total = (pos == chunk) ? *part : (*total + *part);
    *part = 0.0f;
  }
}
static inline float csum_finish(float total, float part, int64_t len, int64_t chunk) {
  if (len == 0) return 0.0f;
  return (len <= chunk) ? part : (total + part);
}

/* ------------------------------------------------------------------------- */
/* ③ SDDMM-add with on-the-fly dequantization (§2.1; P:864-873    */
/* §3.3) followed by LeakyReLU:                                  */
/*   e_pre[e,h] = QV(S,u,h)*s_S + QV(D,v,h)*s_D ;  el = e_pre>0 ? e_pre : e_pre*slope */
/* ------------------------------------------------------------------------- */
void orc_sddmm_add(const orc_graph* g, int heads, orc_qref S, orc_qref D, float slope,
                   float* e_pre, float* el) {
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t v = 0; v < g->n; ++v)
    for (int64_t p = g->in_ptr[v]; p < g->in_ptr[v + 1]; ++p) {
      int64_t u = g->in_src[p];
      for (int h = 0; h < heads; ++h) {
        float a = QV(S, u * heads + h) * S.s;
        float b = QV(D, v * heads + h) * D.s;
        float x = a + b;
        if (e_pre) e_pre[p * heads + h] = x;
        el[p * heads + h] = (x > 0.0f) ? x : x * slope;
      }
    }
}

/* ------------------------------------------------------------------------- */
/* ④ edge softmax in FP32 (§2.1; full precision per P:604-615,     */
/* reading R9), max-stabilised two-pass (reading R12):                        */
/*   m[v,h] = max el ; ex = exp_p(el-m) ; den = Σᶜ ex ; α = ex/den            */
/*   empty row: m = 0, den = 0.                                               */
/* ------------------------------------------------------------------------- */
void orc_edge_softmax(const orc_graph* g, int heads, const float* el, float* m_out, float* den_out,
                      float* alpha) {
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t v = 0; v < g->n; ++v) {
    int64_t b = g->in_ptr[v], len = g->in_ptr[v + 1] - b;
    for (int h = 0; h < heads; ++h) {
      float m = -INFINITY;
      for (int64_t i = 0; i < len; ++i) m = fmaxf(m, el[(b + i) * heads + h]);
      if (len == 0) m = 0.0f;
      float total = 0.0f, part = 0.0f;
      for (int64_t i = 0; i < len; ++i) {
        csum_fold(&total, &part, i, g->chunk);
        part = part + orc_exp_p(el[(b + i) * heads + h] - m);
      }
      float den = csum_finish(total, part, len, g->chunk);
      for (int64_t i = 0; i < len; ++i)
        alpha[(b + i) * heads + h] = orc_exp_p(el[(b + i) * heads + h] - m) / den;
      if (m_out) m_out[v * heads + h] = m;
      if (den_out) den_out[v * heads + h] = den;
    }
  }
}

/* ------------------------------------------------------------------------- */
/* ⑤ SPMM aggregation (§2.1) on quantized node features with fp32  */
/* accumulation (reading R8):                                     */
/*   out[v,j] = (Σᶜ_{e=(u→v)} fmaf(α[e,h(j)], QV(X,u,j), ·)) * s_X           */
/* dir = 0: in-edges of v (forward ⑤).  dir = 1: out-edges of v in the       */
/* reversed graph, (Gᵀ⊙α)·X — backward ⑤′.                      */
/* ------------------------------------------------------------------------- */
int orc_spmm_alpha(const orc_graph* g, int dir, int heads, int cols, const float* alpha, orc_qref X,
                   float* out) {
  orc_rev rv = {0};
  if (dir == 1 && orc_build_rev(g, &rv)) return ORC_ERR_ALLOC;
  int hd = cols / heads;
  int st = ORC_OK;
#pragma omp parallel
  {
    float* total = (float*)malloc(sizeof(float) * (size_t)cols);
    float* part = (float*)malloc(sizeof(float) * (size_t)cols);
#pragma omp for schedule(dynamic, 64)
    for (int64_t v = 0; v < g->n; ++v) {
      const int64_t* ptr = dir ? rv.ptr : g->in_ptr;
      int64_t b = ptr[v], len = ptr[v + 1] - b;
      for (int j = 0; j < cols; ++j) { total[j] = 0.0f; part[j] = 0.0f; }
      for (int64_t i = 0; i < len; ++i) {
        int64_t eid = dir ? rv.eid[b + i] : (b + i);
        int64_t w = dir ? rv.dst[b + i] : g->in_src[b + i];  /* the other endpoint */
        for (int j = 0; j < cols; ++j) {
          csum_fold(&total[j], &part[j], i, g->chunk);
          part[j] = fmaf(alpha[eid * heads + j / hd], QV(X, w * cols + j), part[j]);
        }
      }
      for (int j = 0; j < cols; ++j) out[v * cols + j] = csum_finish(total[j], part[j], len, g->chunk) * X.s;
    }
    free(total);
    free(part);
  }
  if (dir == 1) orc_free_rev(&rv);
  return st;
}

/* Unweighted fp32 row gather with the chunked order (R14), plain adds:
 *   out[v,j] = Σᶜ_{e} x[w,j]  over in-edges (dir 0, w = source) or out-edges
 *   (dir 1, w = destination) — the FP32 GCN aggregation (final layer, R35). */
int orc_spmm_alpha_unit(const orc_graph* g, int dir, int cols, const float* x, float* out) {
  orc_rev rv = {0};
  if (dir == 1 && orc_build_rev(g, &rv)) return ORC_ERR_ALLOC;
  for (int64_t v = 0; v < g->n; ++v) {
    const int64_t* ptr = dir ? rv.ptr : g->in_ptr;
    int64_t b = ptr[v], len = ptr[v + 1] - b;
    for (int j = 0; j < cols; ++j) {
      float total = 0.0f, part = 0.0f;
      for (int64_t i = 0; i < len; ++i) {
        int64_t w = dir ? rv.dst[b + i] : g->in_src[b + i];
        csum_fold(&total, &part, i, g->chunk);
        part = part + x[w * cols + j];
      }
      out[v * cols + j] = csum_finish(total, part, len, g->chunk);
    }
  }
  if (dir == 1) orc_free_rev(&rv);
  return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* ⑤″ SDDMM-dot directly on quantized values (§2.1):    */
/*   ∂α[e,h] = (float)(Σ_d QV(A,v,h,d)·QV(B,u,h,d)) * (s_A*s_B)              */
/* The integer dot is exact (int64 here; |acc| < 2^24 at D=128).  Bypass:    */
/* the dot is accumulated in double.  A rows are destinations, B rows sources.*/
/* ------------------------------------------------------------------------- */
void orc_sddmm_dot(const orc_graph* g, int heads, int cols, orc_qref A, orc_qref B, float* out) {
  int hd = cols / heads;
  float sAB = A.s * B.s;
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t v = 0; v < g->n; ++v)
    for (int64_t p = g->in_ptr[v]; p < g->in_ptr[v + 1]; ++p) {
      int64_t u = g->in_src[p];
      for (int h = 0; h < heads; ++h) {
        float dotf;
        if (A.q && B.q) {
          int64_t acc = 0;
          for (int d = 0; d < hd; ++d)
            acc += (int64_t)A.q[v * cols + h * hd + d] * (int64_t)B.q[u * cols + h * hd + d];
          dotf = (float)acc;
        } else {
          double acc = 0.0;
          for (int d = 0; d < hd; ++d)
            acc += (double)QV(A, v * cols + h * hd + d) * (double)QV(B, u * cols + h * hd + d);
          dotf = (float)acc;
        }
        out[p * heads + h] = dotf * sAB;
      }
    }
}

/* ------------------------------------------------------------------------- */
/* ④′ softmax backward (§2.1; FP32 per P:604-615):                 */
/*   P[v,h] = Σᶜ_{e→v} fmaf(∂α, α, ·) ; ∂E = α·(∂α − P[v]) (reading R22)    */
/*   then LeakyReLU backward (reading R11): ∂E_pre = e_pre>0 ? ∂E : ∂E·slope */
/* ------------------------------------------------------------------------- */
void orc_softmax_bwd(const orc_graph* g, int heads, const float* alpha, const float* dalpha,
                     const float* e_pre, float slope, float* P_out, float* dE_out, float* dEpre_out) {
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t v = 0; v < g->n; ++v) {
    int64_t b = g->in_ptr[v], len = g->in_ptr[v + 1] - b;
    for (int h = 0; h < heads; ++h) {
      float total = 0.0f, part = 0.0f;
      for (int64_t i = 0; i < len; ++i) {
        csum_fold(&total, &part, i, g->chunk);
        part = fmaf(dalpha[(b + i) * heads + h], alpha[(b + i) * heads + h], part);
      }
      float P = csum_finish(total, part, len, g->chunk);
      if (P_out) P_out[v * heads + h] = P;
      for (int64_t i = 0; i < len; ++i) {
        int64_t k = (b + i) * heads + h;
        float t = dalpha[k] - P;
        float dE = alpha[k] * t;
        if (dE_out) dE_out[k] = dE;
        dEpre_out[k] = (e_pre[k] > 0.0f) ? dE : dE * slope;
      }
    }
  }
}

/* ------------------------------------------------------------------------- */
/* ③′/③″ incidence-matrix SPMM (§2.1; §3.3, Fig.7):          */
/*   dir 0: ∂D[v,h] = Σᶜ over in-edges (in-CSR order) of x[e,h]              */
/*   dir 1: ∂S[u,h] = Σᶜ over out-edges (out order) of x[e,h]                */
/* ------------------------------------------------------------------------- */
int orc_edge_sum(const orc_graph* g, int dir, int heads, const float* x, float* out) {
  orc_rev rv = {0};
  if (dir == 1 && orc_build_rev(g, &rv)) return ORC_ERR_ALLOC;
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t v = 0; v < g->n; ++v) {
    const int64_t* ptr = dir ? rv.ptr : g->in_ptr;
    int64_t b = ptr[v], len = ptr[v + 1] - b;
    for (int h = 0; h < heads; ++h) {
      float total = 0.0f, part = 0.0f;
      for (int64_t i = 0; i < len; ++i) {
        int64_t eid = dir ? rv.eid[b + i] : (b + i);
        csum_fold(&total, &part, i, g->chunk);
        part = part + x[eid * heads + h];
      }
      out[v * heads + h] = csum_finish(total, part, len, g->chunk);
    }
  }
  if (dir == 1) orc_free_rev(&rv);
  return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* Unweighted SPMM with int32 accumulation (GCN, §2.2; north_star  */
/* "int32 accumulation"): out[v,j] = Σ_{e} q[w,j], exact and order-free.     */
/* dir 0: w = sources of in-edges of v;  dir 1: w = destinations of v's      */
/* out-edges.  Bypass: double accumulation.  Output as float (exact int).    */
/* ------------------------------------------------------------------------- */
/* NEXT-4 int8-α SPMM (the edge-feature quantization of P:900-902 applied to the attention
 * coefficients): with α quantized to int8 codes q_α [e][heads] (scale s_α, the same SR quantizer as every
 * other tensor), the aggregation is an exact integer sum, order-free:
 *   acc[v][j] = Σ_{e→v} q_α[e][h(j)] · q_X[w_e][j]   (int64 here; |acc| < 2^31 for deg < 133,144)
 *   out[v][j] = (float)acc · fl(s_α · s_X)            (one i2f, one rn multiply)
 * dir 0: in-edges of v (w_e = source, α in in-CSR order); dir 1: out-edges (w_e = destination, α of the
 * edge's in-CSR slot).  Pinned by the brute-force dense product in tests/test_oracle_dense.py. */
int orc_spmm_q8(const orc_graph* g, int dir, int heads, int cols, const int8_t* qa, float sa, const int8_t* qx,
                float sx, int32_t* out_i32, float* out_f) {
  orc_rev rv = {0};
  if (dir == 1 && orc_build_rev(g, &rv)) return ORC_ERR_ALLOC;
  const int hd = cols / heads;
  const float s = sa * sx;
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t v = 0; v < g->n; ++v) {
    const int64_t* ptr = dir ? rv.ptr : g->in_ptr;
    int64_t b = ptr[v], len = ptr[v + 1] - b;
    for (int j = 0; j < cols; ++j) {
      int64_t acc = 0;
      for (int64_t i = 0; i < len; ++i) {
        int64_t eid = dir ? rv.eid[b + i] : (b + i);
        int64_t w = dir ? rv.dst[b + i] : g->in_src[b + i];
        acc += (int64_t)qa[eid * heads + j / hd] * (int64_t)qx[w * cols + j];
      }
      if (out_i32) out_i32[v * cols + j] = (int32_t)acc;
      if (out_f) out_f[v * cols + j] = (float)acc * s;
    }
  }
  if (dir == 1) orc_free_rev(&rv);
  return ORC_OK;
}

int orc_spmm_sum(const orc_graph* g, int dir, int cols, orc_qref X, int32_t* out_i32, float* out_f) {
  orc_rev rv = {0};
  if (dir == 1 && orc_build_rev(g, &rv)) return ORC_ERR_ALLOC;
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t v = 0; v < g->n; ++v) {
    const int64_t* ptr = dir ? rv.ptr : g->in_ptr;
    int64_t b = ptr[v], len = ptr[v + 1] - b;
    for (int j = 0; j < cols; ++j) {
      if (X.q) {
        int64_t acc = 0;
        for (int64_t i = 0; i < len; ++i) {
          int64_t w = dir ? rv.dst[b + i] : g->in_src[b + i];
          acc += X.q[w * cols + j];
        }
        if (out_i32) out_i32[v * cols + j] = (int32_t)acc;
        if (out_f) out_f[v * cols + j] = (float)acc;
      } else {
        double acc = 0.0;
        for (int64_t i = 0; i < len; ++i) {
          int64_t w = dir ? rv.dst[b + i] : g->in_src[b + i];
          acc += (double)X.v[w * cols + j];
        }
        if (out_f) out_f[v * cols + j] = (float)acc;
      }
    }
  }
  if (dir == 1) orc_free_rev(&rv);
  return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* Integer GEMM (§3.2 Fig.4): int8 × int8 with 32-bit (or 64-bit)  */
/* exact accumulation.  C[m][n] = Σ_k A[m*lda + k] * B[k*ldb + n].           */
/* transA: A is stored [K][M] (A[k*lda + m]) — used for ∂W = Hᵀ·∂H′.        */
/* Bypass (A.q == NULL): double accumulation of the fp32 values.             */
/* Output: exact integer as int64 (acc64) and/or float = (float)acc.         */
/* ------------------------------------------------------------------------- */
void orc_gemm(int64_t M, int64_t N, int64_t K, orc_qref A, int64_t lda, int transA, orc_qref B,
              int64_t ldb, int transB, int64_t* acc64, float* accf) {
#pragma omp parallel
  {
    int64_t* ai = (int64_t*)malloc(sizeof(int64_t) * (size_t)N);
    double* ad = (double*)malloc(sizeof(double) * (size_t)N);
#pragma omp for schedule(static)
    for (int64_t m = 0; m < M; ++m) {
      for (int64_t n = 0; n < N; ++n) { ai[n] = 0; ad[n] = 0.0; }
      for (int64_t k = 0; k < K; ++k) {
        int64_t ia = transA ? (k * lda + m) : (m * lda + k);
        if (A.q && B.q) {
          int64_t a = A.q[ia];
          if (a == 0) continue;
          if (transB) for (int64_t n = 0; n < N; ++n) ai[n] += a * B.q[n * ldb + k];
          else        for (int64_t n = 0; n < N; ++n) ai[n] += a * B.q[k * ldb + n];
        } else {
          double a = (double)QV(A, ia);
          if (transB) for (int64_t n = 0; n < N; ++n) ad[n] += a * (double)QV(B, n * ldb + k);
          else        for (int64_t n = 0; n < N; ++n) ad[n] += a * (double)QV(B, k * ldb + n);
        }
      }
      for (int64_t n = 0; n < N; ++n) {
        if (A.q && B.q) {
          if (acc64) acc64[m * N + n] = ai[n];
          if (accf) accf[m * N + n] = (float)ai[n];
        } else {
          if (accf) accf[m * N + n] = (float)ad[n];
        }
      }
    }
    free(ai);
    free(ad);
  }
}

/* ========================================================================= */
/* GAT layer (§2.1 Fig.1, with the quantization rules of §3.2-3.3).*/
/* ========================================================================= */
typedef struct {
  int32_t F, H, D;
  float slope;
  int32_t bits;  /* 2..8, or 0 = bypass */
  uint64_t seed;
  uint32_t step;
  uint32_t layer_id;
} orc_gat_cfg;

/* Philox tag = (layer_id << 8) | role. */
enum { ROLE_H = 1, ROLE_W = 2, ROLE_HP = 3, ROLE_S = 4, ROLE_D = 5, ROLE_G = 6, ROLE_DHP = 7,
       ROLE_YS = 8, ROLE_GS = 9, ROLE_DY = 10 };
static inline uint32_t TAG(uint32_t layer, uint32_t role) { return (layer << 8) | role; }

typedef struct {
  /* quantized inputs cached for backward */
  int8_t* qH; float* sH;     /* [n][F] */
  int8_t* qW; float* sW;     /* [F][HD] */
  /* ① + ② */
  int32_t* maxacc;           /* scalar max |q_H·q_W| */
  float* Hp;                 /* [n][HD] H′ = (float)acc * (s_H*s_W), exact fp32 */
  float* S; float* Dd;       /* [n][H]  ② from exact H′ (reading R10) */
  int8_t* qHp; float* sHp;   /* [n][HD] */
  int8_t* qS; float* sS;     /* [n][H] */
  int8_t* qD; float* sD;     /* [n][H] */
  /* ③ ④ */
  float* e_pre; float* alpha; /* [e][H] */
  float* m; float* den;       /* [n][H] */
  /* ⑤ */
  float* Hout;                /* [n][HD] */
  float* amax_out;            /* scalar amax(H_out) (hint for the next layer) */
} orc_gat_fwd_out;

static int quant_or_bypass(const float* x, int64_t count, const orc_gat_cfg* c, uint32_t role, int8_t* q,
                           float* s, orc_qref* ref, const float* amax_in) {
  if (c->bits == 0) {
    *ref = (orc_qref){NULL, x, 1.0f};
    if (s) *s = 1.0f;
    return ORC_OK;
  }
  float sc;
  int st = orc_quantize(x, count, c->bits, c->seed, c->step, TAG(c->layer_id, role), 0, amax_in, q, &sc, NULL);
  if (st) return st;
  if (s) *s = sc;
  *ref = (orc_qref){q, NULL, sc};
  return ORC_OK;
}

int orc_gat_fwd(const orc_graph* g, const orc_gat_cfg* c, const float* H, const float* W, const float* a_src,
                const float* a_dst, orc_gat_fwd_out* o) {
  int64_t n = g->n, F = c->F, heads = c->H, hd = c->D, HD = heads * hd;
  int st;
  orc_qref rH, rW;
  /* F1/F2: quantize H and W */
  if ((st = quant_or_bypass(H, n * F, c, ROLE_H, o->qH, o->sH, &rH, NULL))) return st;
  if ((st = quant_or_bypass(W, F * HD, c, ROLE_W, o->qW, o->sW, &rW, NULL))) return st;
  /* F3 ①: acc = q_H·q_W (int32); H′ = (float)acc * (s_H*s_W) */
  float* accf = (float*)malloc(sizeof(float) * (size_t)(n * HD > 0 ? n * HD : 1));
  if (!accf) return ORC_ERR_ALLOC;
  int64_t* acc64 = NULL;
  if (c->bits) { acc64 = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n * HD > 0 ? n * HD : 1)); if (!acc64) return ORC_ERR_ALLOC; }
  orc_gemm(n, HD, F, rH, F, 0, rW, HD, 0, acc64, accf);
  float sHW = rH.s * rW.s;
  int64_t maxacc = 0;
  if (acc64) for (int64_t i = 0; i < n * HD; ++i) { int64_t a = acc64[i] < 0 ? -acc64[i] : acc64[i]; if (a > maxacc) maxacc = a; }
  if (o->maxacc) *o->maxacc = (int32_t)maxacc;
  float* Hp = o->Hp;
  for (int64_t i = 0; i < n * HD; ++i) Hp[i] = accf[i] * sHW;
  free(accf);
  free(acc64);
  /* ② S = (H′·a_src)ᵀ, D = (H′·a_dst)ᵀ per head, sequential fmaf over d */
  for (int64_t v = 0; v < n; ++v)
    for (int64_t h = 0; h < heads; ++h) {
      float s = 0.0f, d = 0.0f;
      for (int64_t k = 0; k < hd; ++k) {
        s = fmaf(Hp[v * HD + h * hd + k], a_src[h * hd + k], s);
        d = fmaf(Hp[v * HD + h * hd + k], a_dst[h * hd + k], d);
      }
      o->S[v * heads + h] = s;
      o->Dd[v * heads + h] = d;
    }
  /* F4: quantize H′, S, D (dedicated pass before sparse ops) */
  orc_qref rHp, rS, rD;
  if ((st = quant_or_bypass(Hp, n * HD, c, ROLE_HP, o->qHp, o->sHp, &rHp, NULL))) return st;
  if ((st = quant_or_bypass(o->S, n * heads, c, ROLE_S, o->qS, o->sS, &rS, NULL))) return st;
  if ((st = quant_or_bypass(o->Dd, n * heads, c, ROLE_D, o->qD, o->sD, &rD, NULL))) return st;
  /* F5 ③ + ④ */
  float* el = (float*)malloc(sizeof(float) * (size_t)(g->e * heads > 0 ? g->e * heads : 1));
  if (!el) return ORC_ERR_ALLOC;
  orc_sddmm_add(g, (int)heads, rS, rD, c->slope, o->e_pre, el);
  orc_edge_softmax(g, (int)heads, el, o->m, o->den, o->alpha);
  free(el);
  /* F6 ⑤ */
  if ((st = orc_spmm_alpha(g, 0, (int)heads, (int)HD, o->alpha, rHp, o->Hout))) return st;
  if (o->amax_out) { int bad; *o->amax_out = orc_absmax(o->Hout, n * HD, &bad); }
  return ORC_OK;
}

typedef struct {
  int8_t* qG; float* sG;      /* [n][HD] quantized ∂H_out, shared by ⑤′ and ⑤″ */
  float* dalpha;              /* [e][H] ⑤″ */
  float* P;                   /* [n][H] ④′ */
  float* dE; float* dE_pre;   /* [e][H] */
  float* dD; float* dS;       /* [n][H] ③″ / ③′ */
  float* dHp_agg;             /* [n][HD] ⑤′ */
  float* dHp;                 /* [n][HD] ②′ */
  float* da_src; float* da_dst;       /* [HD] */
  float* da_src_abs; float* da_dst_abs; /* [HD] Σ|terms| (tolerance bound for ∂a) */
  int8_t* qdHp; float* sdHp;  /* [n][HD] */
  float* dH;                  /* [n][F]  ①′ */
  float* dW;                  /* [F][HD] ①′ */
} orc_gat_bwd_out;

/* Backward (§2.1 Fig.1b; reuse of cached q_H, q_W, q_H′ P:886-889).
 * fwd: the forward's outputs (only the fields used below are read). */
int orc_gat_bwd(const orc_graph* g, const orc_gat_cfg* c, const float* W, const float* a_src, const float* a_dst,
                const orc_gat_fwd_out* f, const float* H, const float* dHout, orc_gat_bwd_out* o) {
  int64_t n = g->n, F = c->F, heads = c->H, hd = c->D, HD = heads * hd;
  int st;
  /* cached forward tensors (bypass: fp32 values with s = 1) */
  orc_qref rH = c->bits ? (orc_qref){f->qH, NULL, *f->sH} : (orc_qref){NULL, H, 1.0f};
  orc_qref rW = c->bits ? (orc_qref){f->qW, NULL, *f->sW} : (orc_qref){NULL, W, 1.0f};
  orc_qref rHp = c->bits ? (orc_qref){f->qHp, NULL, *f->sHp} : (orc_qref){NULL, f->Hp, 1.0f};
  /* B1: quantize ∂H_out once */
  orc_qref rG;
  if ((st = quant_or_bypass(dHout, n * HD, c, ROLE_G, o->qG, o->sG, &rG, NULL))) return st;
  /* B2 ⑤″ ∂α = G ⊙ (∂H_out · H′ᵀ) */
  orc_sddmm_dot(g, (int)heads, (int)HD, rG, rHp, o->dalpha);
  /* B3 ④′ */
  orc_softmax_bwd(g, (int)heads, f->alpha, o->dalpha, f->e_pre, c->slope, o->P, o->dE, o->dE_pre);
  /* B4 ③″ ∂D = (G ⊙ ∂E)·1 over in-edges; B6 ③′ ∂S = (Gᵀ ⊙ ∂E)·1 over out-edges */
  if ((st = orc_edge_sum(g, 0, (int)heads, o->dE_pre, o->dD))) return st;
  if ((st = orc_edge_sum(g, 1, (int)heads, o->dE_pre, o->dS))) return st;
  /* B5 ⑤′ ∂H′_agg = (Gᵀ ⊙ α)·∂H_out */
  if ((st = orc_spmm_alpha(g, 1, (int)heads, (int)HD, f->alpha, rG, o->dHp_agg))) return st;
  /* B7 ②′ chain rule through S = H′·a_src, D = H′·a_dst (reading R23):
   *   ∂H′ = (∂H′_agg + ∂S·a_src) + ∂D·a_dst
   *   ∂a_src[j] = Σ_u ∂S[u,h]·deq(q_H′)[u,j] (double accumulation), likewise ∂a_dst */
  for (int64_t u = 0; u < n; ++u)
    for (int64_t j = 0; j < HD; ++j) {
      int64_t h = j / hd;
      float t1 = o->dS[u * heads + h] * a_src[j];
      float t2 = o->dHp_agg[u * HD + j] + t1;
      float t3 = o->dD[u * heads + h] * a_dst[j];
      o->dHp[u * HD + j] = t2 + t3;
    }
  /* ∂a in the pinned order of reading R39 (= R33's row-chunked Σᶜ, chunk ORC_CK global rows):
   * ∂a_src[j] = Σᶜ_u fmaf(∂S[u,h], deq(q_H′)[u,j], ·), deq = i2f(q)·s_H′ (one rounding) */
  for (int64_t j = 0; j < HD; ++j) {
    int64_t h = j / hd;
    float as = 0.0f, ad = 0.0f, ps = 0.0f, pd = 0.0f;
    double as_abs = 0.0, ad_abs = 0.0;
    for (int64_t u = 0; u < n; ++u) {
      float hp = QV(rHp, u * HD + j) * rHp.s;
      ps = fmaf(o->dS[u * heads + h], hp, ps);
      pd = fmaf(o->dD[u * heads + h], hp, pd);
      as_abs += fabs((double)o->dS[u * heads + h] * (double)hp);
      ad_abs += fabs((double)o->dD[u * heads + h] * (double)hp);
      if ((u + 1) % ORC_CK == 0 || u + 1 == n) {   /* close the chunk, fold left to right */
        if (u < ORC_CK) { as = ps; ad = pd; } else { as = as + ps; ad = ad + pd; }
        ps = 0.0f; pd = 0.0f;
      }
    }
    o->da_src[j] = as;
    o->da_dst[j] = ad;
    if (o->da_src_abs) o->da_src_abs[j] = (float)as_abs;
    if (o->da_dst_abs) o->da_dst_abs[j] = (float)ad_abs;
  }
  /* B8: quantize ∂H′ */
  orc_qref rdHp;
  if ((st = quant_or_bypass(o->dHp, n * HD, c, ROLE_DHP, o->qdHp, o->sdHp, &rdHp, NULL))) return st;
  /* B9 ①′: ∂H = ∂H′·Wᵀ ; ∂W = Hᵀ·∂H′, int32 / int64 accumulation (reading R27) */
  float* tmp = (float*)malloc(sizeof(float) * (size_t)(n * F > F * HD ? (n * F > 0 ? n * F : 1) : F * HD));
  if (!tmp) return ORC_ERR_ALLOC;
  orc_gemm(n, F, HD, rdHp, HD, 0, rW, HD, 1, NULL, tmp);
  float s1 = rdHp.s * rW.s;
  for (int64_t i = 0; i < n * F; ++i) o->dH[i] = tmp[i] * s1;
  orc_gemm(F, HD, n, rH, F, 1, rdHp, HD, 0, NULL, tmp);
  float s2 = rH.s * rdHp.s;
  for (int64_t i = 0; i < F * HD; ++i) o->dW[i] = tmp[i] * s2;
  free(tmp);
  return ORC_OK;
}

/* ========================================================================= */
/* GCN layer: GEMM + SPMM (§2.2), DGL GraphConv(norm='both')       */
/* folded into node rows (reading R26): ns = out_deg^-1/2, nd = in_deg^-1/2. */
/* ========================================================================= */
typedef struct {
  int8_t* qX; float* sX;      /* [n][F] */
  int8_t* qW; float* sW;      /* [F][O] */
  float* Ys;                  /* [n][O]  (float)(q_X·q_W)*(s_X*s_W) * ns[u] */
  int8_t* qYs; float* sYs;    /* [n][O] */
  int32_t* ia;                /* [n][O]  Σ_{u→v} q_Ys[u]  (int32) */
  float* out;                 /* [n][O]  ((float)ia * s_Ys) * nd[v] */
} orc_gcn_fwd_out;

typedef struct {
  float* Gs; int8_t* qGs; float* sGs;  /* [n][O] ∂out·nd[v] */
  int32_t* ib;                          /* [n][O] Σ_{u→v} q_Gs[v] over out-edges of u */
  float* dY; int8_t* qdY; float* sdY;   /* [n][O] ((float)ib*s_Gs)*ns[u] */
  float* dX;                            /* [n][F] */
  float* dW;                            /* [F][O] */
} orc_gcn_bwd_out;

static void gcn_norms(const orc_graph* g, float* ns, float* nd) {
  int64_t n = g->n;
  int64_t* od = (int64_t*)calloc((size_t)(n > 0 ? n : 1), sizeof(int64_t));
  for (int64_t p = 0; p < g->e; ++p) od[g->in_src[p]]++;
  for (int64_t v = 0; v < n; ++v) {
    int64_t di = g->in_ptr[v + 1] - g->in_ptr[v];
    nd[v] = di > 0 ? 1.0f / sqrtf((float)di) : 0.0f;
    ns[v] = od[v] > 0 ? 1.0f / sqrtf((float)od[v]) : 0.0f;
  }
  free(od);
}

int orc_gcn_fwd(const orc_graph* g, const orc_gat_cfg* c /* F, D = out feats, H = 1 */, const float* X,
                const float* W, orc_gcn_fwd_out* o) {
  int64_t n = g->n, F = c->F, O = c->D;
  int st;
  float* ns = (float*)malloc(sizeof(float) * (size_t)(n > 0 ? n : 1));
  float* nd = (float*)malloc(sizeof(float) * (size_t)(n > 0 ? n : 1));
  gcn_norms(g, ns, nd);
  orc_qref rX, rW;
  if ((st = quant_or_bypass(X, n * F, c, ROLE_H, o->qX, o->sX, &rX, NULL))) return st;
  if ((st = quant_or_bypass(W, F * O, c, ROLE_W, o->qW, o->sW, &rW, NULL))) return st;
  float* accf = (float*)malloc(sizeof(float) * (size_t)(n * O > 0 ? n * O : 1));
  orc_gemm(n, O, F, rX, F, 0, rW, O, 0, NULL, accf);
  float sXW = rX.s * rW.s;
  for (int64_t u = 0; u < n; ++u)
    for (int64_t j = 0; j < O; ++j) o->Ys[u * O + j] = (accf[u * O + j] * sXW) * ns[u];
  free(accf);
  orc_qref rYs;
  if ((st = quant_or_bypass(o->Ys, n * O, c, ROLE_YS, o->qYs, o->sYs, &rYs, NULL))) return st;
  float* sumf = (float*)malloc(sizeof(float) * (size_t)(n * O > 0 ? n * O : 1));
  orc_spmm_sum(g, 0, (int)O, rYs, o->ia, sumf);
  for (int64_t v = 0; v < n; ++v)
    for (int64_t j = 0; j < O; ++j) o->out[v * O + j] = (sumf[v * O + j] * rYs.s) * nd[v];
  free(sumf); free(ns); free(nd);
  return ORC_OK;
}

int orc_gcn_bwd(const orc_graph* g, const orc_gat_cfg* c, const float* X, const float* W,
                const orc_gcn_fwd_out* f, const float* dout, orc_gcn_bwd_out* o) {
  int64_t n = g->n, F = c->F, O = c->D;
  int st;
  float* ns = (float*)malloc(sizeof(float) * (size_t)(n > 0 ? n : 1));
  float* nd = (float*)malloc(sizeof(float) * (size_t)(n > 0 ? n : 1));
  gcn_norms(g, ns, nd);
  orc_qref rX = c->bits ? (orc_qref){f->qX, NULL, *f->sX} : (orc_qref){NULL, X, 1.0f};
  orc_qref rW = c->bits ? (orc_qref){f->qW, NULL, *f->sW} : (orc_qref){NULL, W, 1.0f};
  for (int64_t v = 0; v < n; ++v)
    for (int64_t j = 0; j < O; ++j) o->Gs[v * O + j] = dout[v * O + j] * nd[v];
  orc_qref rGs;
  if ((st = quant_or_bypass(o->Gs, n * O, c, ROLE_GS, o->qGs, o->sGs, &rGs, NULL))) return st;
  float* sumf = (float*)malloc(sizeof(float) * (size_t)(n * O > 0 ? n * O : 1));
  orc_spmm_sum(g, 1, (int)O, rGs, o->ib, sumf);
  for (int64_t u = 0; u < n; ++u)
    for (int64_t j = 0; j < O; ++j) o->dY[u * O + j] = (sumf[u * O + j] * rGs.s) * ns[u];
  free(sumf);
  orc_qref rdY;
  if ((st = quant_or_bypass(o->dY, n * O, c, ROLE_DY, o->qdY, o->sdY, &rdY, NULL))) return st;
  float* tmp = (float*)malloc(sizeof(float) * (size_t)(n * F > F * O ? (n * F > 0 ? n * F : 1) : F * O));
  orc_gemm(n, F, O, rdY, O, 0, rW, O, 1, NULL, tmp);
  float s1 = rdY.s * rW.s;
  for (int64_t i = 0; i < n * F; ++i) o->dX[i] = tmp[i] * s1;
  orc_gemm(F, O, n, rX, F, 1, rdY, O, 0, NULL, tmp);
  float s2 = rX.s * rdY.s;
  for (int64_t i = 0; i < F * O; ++i) o->dW[i] = tmp[i] * s2;
  free(tmp); free(ns); free(nd);
  return ORC_OK;
}

int orc_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
void orc_set_threads(int t) {
#ifdef _OPENMP
  if (t > 0) omp_set_num_threads(t);
#else
  (void)t;
#endif
}

/* ========================================================================= */
/* NEXT-1: the training step around the quantized layer.   */
/* Full-precision final layer (§3.2 Eq.7-8), activation + bias,    */
/* cross-entropy, FP32 master-weight update (§3.2 Eq.5-6).         */
/* ========================================================================= */

/* Full-precision contraction order (reading R33): the K-chunked canonical sum
 * Σᶜ of R14 with chunk ORC_CK = 1024 and FMA terms:
 *   C[m][n] = Σᶜ_k fmaf(A(m,k), B(k,n), ·)
 * A(m,k) = transA ? A[k*lda + m] : A[m*lda + k];  B(k,n) = transB ? B[n*ldb + k] : B[k*ldb + n]. */
void orc_sgemm(int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, int transA, const float* B,
               int64_t ldb, int transB, float* C) {
#pragma omp parallel for schedule(static)
  for (int64_t m = 0; m < M; ++m)
    for (int64_t n = 0; n < N; ++n) {
      float total = 0.0f, part = 0.0f;
      for (int64_t k = 0; k < K; ++k) {
        csum_fold(&total, &part, k, ORC_CK);
        float a = transA ? A[k * lda + m] : A[m * lda + k];
        float b = transB ? B[n * ldb + k] : B[k * ldb + n];
        part = fmaf(a, b, part);
      }
      C[m * N + n] = csum_finish(total, part, K, ORC_CK);
    }
}

/* Column sum over rows with the same chunked order (reading R33): out[j] = Σᶜ_r x[r][j]. */
void orc_colsum(const float* x, int64_t rows, int64_t cols, float* out) {
  for (int64_t j = 0; j < cols; ++j) {
    float total = 0.0f, part = 0.0f;
    for (int64_t r = 0; r < rows; ++r) {
      csum_fold(&total, &part, r, ORC_CK);
      part = part + x[r * cols + j];
    }
    out[j] = csum_finish(total, part, rows, ORC_CK);
  }
}

/* Hidden-layer bias + activation (reading R34: ReLU after the concatenated
 * heads, bias per output column; the paper fixes neither):
 *   y = x + b[j] ; a = y > 0 ? y : 0 ;  amax = max |a| (the next layer's Q hint) */
void orc_bias_relu_fwd(const float* x, const float* b, int64_t rows, int64_t cols, float* a, float* amax) {
  float m = 0.0f;
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t j = 0; j < cols; ++j) {
      float y = x[r * cols + j] + b[j];
      float v = (y > 0.0f) ? y : 0.0f;
      a[r * cols + j] = v;
      m = fmaxf(m, v);
    }
  if (amax) *amax = m;
}

/* Backward: dx = a > 0 ? da : 0 (a > 0 <=> y > 0), db = Σᶜ_r dx (R33),
 * amax_dx = max |dx| (the quantized layer's ∂H_out hint). */
void orc_bias_relu_bwd(const float* a, const float* da, int64_t rows, int64_t cols, float* dx, float* db,
                       float* amax_dx) {
  float m = 0.0f;
  for (int64_t i = 0; i < rows * cols; ++i) {
    float d = (a[i] > 0.0f) ? da[i] : 0.0f;
    dx[i] = d;
    m = fmaxf(m, fabsf(d));
  }
  orc_colsum(dx, rows, cols, db);
  if (amax_dx) *amax_dx = m;
}

/* Full-precision final GAT layer ("use full precision to compute the
 * layer before the Softmax"; reading R35: heads averaged), FP32
 * end to end, the same steps ①-⑤ as orc_gat_fwd in bypass form:
 *   H′ = sgemm(H, W) [n][H·C] ; S, D = sequential fmaf over c (R10) ;
 *   ③ el (orc_sddmm_add, scale 1) ; ④ orc_edge_softmax ; ⑤ agg = orc_spmm_alpha ;
 *   logits[v,c] = ((Σ_h agg[v,h,c], left to right) / heads) + bias[c]. */
typedef struct { int32_t F, H, C; float slope; } orc_out_cfg;
typedef struct {
  float* Hp;                  /* [n][H*C] */
  float* S; float* Dd;        /* [n][H] */
  float* e_pre; float* alpha; /* [e][H] */
  float* m; float* den;       /* [n][H] */
  float* agg;                 /* [n][H*C] */
  float* logits;              /* [n][C] */
} orc_out_fwd_out;

int orc_gat_out_fwd(const orc_graph* g, const orc_out_cfg* c, const float* H, const float* W,
                    const float* a_src, const float* a_dst, const float* bias, orc_out_fwd_out* o) {
  int64_t n = g->n, F = c->F, heads = c->H, C = c->C, HC = heads * C;
  orc_sgemm(n, HC, F, H, F, 0, W, HC, 0, o->Hp);
  for (int64_t v = 0; v < n; ++v)
    for (int64_t h = 0; h < heads; ++h) {
      float s = 0.0f, d = 0.0f;
      for (int64_t k = 0; k < C; ++k) {
        s = fmaf(o->Hp[v * HC + h * C + k], a_src[h * C + k], s);
        d = fmaf(o->Hp[v * HC + h * C + k], a_dst[h * C + k], d);
      }
      o->S[v * heads + h] = s;
      o->Dd[v * heads + h] = d;
    }
  float* el = (float*)malloc(sizeof(float) * (size_t)(g->e * heads > 0 ? g->e * heads : 1));
  if (!el) return ORC_ERR_ALLOC;
  orc_sddmm_add(g, (int)heads, (orc_qref){NULL, o->S, 1.0f}, (orc_qref){NULL, o->Dd, 1.0f}, c->slope, o->e_pre, el);
  orc_edge_softmax(g, (int)heads, el, o->m, o->den, o->alpha);
  free(el);
  int st = orc_spmm_alpha(g, 0, (int)heads, (int)HC, o->alpha, (orc_qref){NULL, o->Hp, 1.0f}, o->agg);
  if (st) return st;
  for (int64_t v = 0; v < n; ++v)
    for (int64_t k = 0; k < C; ++k) {
      float t = o->agg[v * HC + k];
      for (int64_t h = 1; h < heads; ++h) t = t + o->agg[v * HC + h * C + k];
      t = t / (float)heads;
      o->logits[v * C + k] = t + bias[k];
    }
  return ORC_OK;
}

typedef struct {
  float* db;                  /* [C]  Σᶜ_v ∂logits */
  float* G;                   /* [n][C] ∂logits / heads = ∂agg of every head */
  float* dalpha;              /* [e][H] ⑤″ sequential fmaf over c */
  float* P; float* dE; float* dE_pre;
  float* dD; float* dS;
  float* dHp_agg; float* dHp; /* [n][H*C] */
  float* da_src; float* da_dst; float* da_src_abs; float* da_dst_abs;
  float* dH;                  /* [n][F] = sgemm(∂H′, Wᵀ) */
  float* dW;                  /* [F][H*C] = sgemm(Hᵀ, ∂H′) */
} orc_out_bwd_out;

int orc_gat_out_bwd(const orc_graph* g, const orc_out_cfg* c, const float* H, const float* W,
                    const float* a_src, const float* a_dst, const orc_out_fwd_out* f, const float* dlogits,
                    orc_out_bwd_out* o) {
  int64_t n = g->n, F = c->F, heads = c->H, C = c->C, HC = heads * C;
  int st;
  orc_colsum(dlogits, n, C, o->db);
  for (int64_t i = 0; i < n * C; ++i) o->G[i] = dlogits[i] / (float)heads;
  /* ∂agg[v,h,c] = G[v,c] for every head (mean), materialised for ⑤′ */
  float* dagg = (float*)malloc(sizeof(float) * (size_t)(n * HC > 0 ? n * HC : 1));
  if (!dagg) return ORC_ERR_ALLOC;
  for (int64_t v = 0; v < n; ++v)
    for (int64_t h = 0; h < heads; ++h)
      for (int64_t k = 0; k < C; ++k) dagg[v * HC + h * C + k] = o->G[v * C + k];
  /* ⑤″ ∂α[e,h] = Σ_c fmaf(G[v,c], H′[u,h,c]) sequential */
  for (int64_t v = 0; v < n; ++v)
    for (int64_t p = g->in_ptr[v]; p < g->in_ptr[v + 1]; ++p) {
      int64_t u = g->in_src[p];
      for (int64_t h = 0; h < heads; ++h) {
        float acc = 0.0f;
        for (int64_t k = 0; k < C; ++k) acc = fmaf(o->G[v * C + k], f->Hp[u * HC + h * C + k], acc);
        o->dalpha[p * heads + h] = acc;
      }
    }
  /* ④′, ③″, ③′, ⑤′ as in orc_gat_bwd */
  orc_softmax_bwd(g, (int)heads, f->alpha, o->dalpha, f->e_pre, c->slope, o->P, o->dE, o->dE_pre);
  if ((st = orc_edge_sum(g, 0, (int)heads, o->dE_pre, o->dD))) return st;
  if ((st = orc_edge_sum(g, 1, (int)heads, o->dE_pre, o->dS))) return st;
  if ((st = orc_spmm_alpha(g, 1, (int)heads, (int)HC, f->alpha, (orc_qref){NULL, dagg, 1.0f}, o->dHp_agg))) return st;
  free(dagg);
  /* ②′ (reading R23) */
  for (int64_t u = 0; u < n; ++u)
    for (int64_t j = 0; j < HC; ++j) {
      int64_t h = j / C;
      float t1 = o->dS[u * heads + h] * a_src[j];
      float t2 = o->dHp_agg[u * HC + j] + t1;
      float t3 = o->dD[u * heads + h] * a_dst[j];
      o->dHp[u * HC + j] = t2 + t3;
    }
  for (int64_t j = 0; j < HC; ++j) {   /* ∂a in the pinned order of reading R39 (row-chunked Σᶜ) */
    int64_t h = j / C;
    float as = 0.0f, ad = 0.0f, ps = 0.0f, pd = 0.0f;
    double as_abs = 0.0, ad_abs = 0.0;
    for (int64_t u = 0; u < n; ++u) {
      ps = fmaf(o->dS[u * heads + h], f->Hp[u * HC + j], ps);
      pd = fmaf(o->dD[u * heads + h], f->Hp[u * HC + j], pd);
      as_abs += fabs((double)o->dS[u * heads + h] * (double)f->Hp[u * HC + j]);
      ad_abs += fabs((double)o->dD[u * heads + h] * (double)f->Hp[u * HC + j]);
      if ((u + 1) % ORC_CK == 0 || u + 1 == n) {
        if (u < ORC_CK) { as = ps; ad = pd; } else { as = as + ps; ad = ad + pd; }
        ps = 0.0f; pd = 0.0f;
      }
    }
    o->da_src[j] = as;
    o->da_dst[j] = ad;
    if (o->da_src_abs) o->da_src_abs[j] = (float)as_abs;
    if (o->da_dst_abs) o->da_dst_abs[j] = (float)ad_abs;
  }
  /* ①′ */
  if (o->dH) orc_sgemm(n, F, HC, o->dHp, HC, 0, W, HC, 1, o->dH);
  orc_sgemm(F, HC, n, H, F, 1, o->dHp, HC, 0, o->dW);
  return ORC_OK;
}

/* Cross-entropy over labelled rows ("mean negative log-softmax";
 * reading R36): label < 0 = unlabelled (zero gradient).  Per labelled row v:
 *   m = max_c z ; ssum = Σ_c exp_p(z_c − m) (sequential) ; loss_v = (m + logf(ssum)) − z_y
 *   ∂z_c = (exp_p(z_c − m)/ssum − [c = y]) / n_lab
 * loss = (Σ_v loss_v in double) / n_lab.  Returns ORC_ERR_BITS+100 (=103) on a
 * label >= C (the caller's error).  logf is glibc's (not pinned: the loss is
 * compared within a tolerance, the gradient uses only exp_p and IEEE ops). */
int orc_cross_entropy(const float* z, const int32_t* labels, int64_t n, int32_t C, int64_t n_lab,
                      float* row_loss, double* loss, float* dz) {
  double acc = 0.0;
  float nl = (float)n_lab;
  for (int64_t v = 0; v < n; ++v) {
    int32_t y = labels[v];
    if (y >= C) return 103;
    if (y < 0) {
      for (int32_t k = 0; k < C; ++k) dz[v * C + k] = 0.0f;
      if (row_loss) row_loss[v] = 0.0f;
      continue;
    }
    float m = -INFINITY;
    for (int32_t k = 0; k < C; ++k) m = fmaxf(m, z[v * C + k]);
    float ssum = 0.0f;
    for (int32_t k = 0; k < C; ++k) ssum = ssum + orc_exp_p(z[v * C + k] - m);
    float lv = (m + logf(ssum)) - z[v * C + y];
    if (row_loss) row_loss[v] = lv;
    acc += (double)lv;
    for (int32_t k = 0; k < C; ++k) {
      float p = orc_exp_p(z[v * C + k] - m) / ssum;
      float t = p - (k == y ? 1.0f : 0.0f);
      dz[v * C + k] = t / nl;
    }
  }
  *loss = n_lab > 0 ? acc / (double)n_lab : 0.0;
  return ORC_OK;
}

/* FP32 master-weight update (§3.2 Eq.6, add-then-quantize): the
 * dequantized FP32 gradient is applied to the FP32 master, W ← W − lr·∂W (two
 * rn ops); the next iteration's Q(W) sees the updated master. */
void orc_sgd(float* w, const float* g, int64_t count, float lr) {
  for (int64_t i = 0; i < count; ++i) {
    float t = lr * g[i];
    w[i] = w[i] - t;
  }
}

/* Full-precision final GCN layer (P:604-615 FP32 rule; GCN P:347-348 with the
 * DGL norm='both' of reading R26, folded into rows; reading R35 for the bias):
 *   Y = sgemm(X, W) [n][C] (R33) ; Ys[u] = Y[u]·ns[u] ;
 *   agg[v] = Σᶜ over in-edges (in-CSR order) Ys[u] (plain adds, R14) ;
 *   logits[v] = agg[v]·nd[v] + b.                                             */
typedef struct { float* Y; float* Ys; float* agg; float* logits; } orc_gcn_out_fwd_out;
typedef struct { float* db; float* Gs; float* aggb; float* dY; float* dX; float* dW; } orc_gcn_out_bwd_out;

static int gcn_gather_sum(const orc_graph* g, int dir, int cols, const float* x, float* out) {
  return orc_spmm_alpha_unit(g, dir, cols, x, out);
}

int orc_gcn_out_fwd(const orc_graph* g, int F, int C, const float* X, const float* W, const float* bias,
                    orc_gcn_out_fwd_out* o) {
  int64_t n = g->n;
  float* ns = (float*)malloc(sizeof(float) * (size_t)(n > 0 ? n : 1));
  float* nd = (float*)malloc(sizeof(float) * (size_t)(n > 0 ? n : 1));
  gcn_norms(g, ns, nd);
  orc_sgemm(n, C, F, X, F, 0, W, C, 0, o->Y);
  for (int64_t u = 0; u < n; ++u)
    for (int j = 0; j < C; ++j) o->Ys[u * C + j] = o->Y[u * C + j] * ns[u];
  int st = gcn_gather_sum(g, 0, C, o->Ys, o->agg);
  for (int64_t v = 0; v < n; ++v)
    for (int j = 0; j < C; ++j) o->logits[v * C + j] = (o->agg[v * C + j] * nd[v]) + bias[j];
  free(ns); free(nd);
  return st;
}

/* Backward: db = Σᶜ_v ∂logits (R33); Gs[v] = ∂logits[v]·nd[v];
 * aggb[u] = Σᶜ over out-edges (out order) Gs[v]; dY[u] = aggb[u]·ns[u];
 * dX = sgemm(dY, Wᵀ) (nullable), dW = sgemm(Xᵀ, dY). */
int orc_gcn_out_bwd(const orc_graph* g, int F, int C, const float* X, const float* W, const float* dlogits,
                    orc_gcn_out_bwd_out* o) {
  int64_t n = g->n;
  float* ns = (float*)malloc(sizeof(float) * (size_t)(n > 0 ? n : 1));
  float* nd = (float*)malloc(sizeof(float) * (size_t)(n > 0 ? n : 1));
  gcn_norms(g, ns, nd);
  orc_colsum(dlogits, n, C, o->db);
  for (int64_t v = 0; v < n; ++v)
    for (int j = 0; j < C; ++j) o->Gs[v * C + j] = dlogits[v * C + j] * nd[v];
  int st = gcn_gather_sum(g, 1, C, o->Gs, o->aggb);
  for (int64_t u = 0; u < n; ++u)
    for (int j = 0; j < C; ++j) o->dY[u * C + j] = o->aggb[u * C + j] * ns[u];
  if (o->dX) orc_sgemm(n, F, C, o->dY, C, 0, W, C, 1, o->dX);
  orc_sgemm(F, C, n, X, F, 1, o->dY, C, 0, o->dW);
  free(ns); free(nd);
  return st;
}
