/*
 * tango.h — C ABI of libtango.so: the quantized GAT / GCN layer of Tango
 * (arXiv 2308.00890, SC'23) as hand-written CUDA for sm_100a (B200).
 *
 * Paper citations: P:n = PAPER.md line n (section / equation given beside it).
 * Readings of the paper (R#) are listed in DESIGN.md §2.
 *
 * CONVENTIONS (apply to every entry point)
 *  - Every tensor pointer is a DEVICE pointer, allocated and owned by the caller
 *    (e.g. by PyTorch).  The library never frees or retains a caller pointer
 *    beyond the call, except `ctx`, which holds the forward -> backward cache.
 *  - Every call is asynchronous on the given cudaStream_t (0 = legacy default
 *    stream).  Scales and maxima stay in device memory: no call synchronizes
 *    the host, except tango_status_poll and the optional launch-error check.
 *  - A call returns a tango_status after validating its arguments on the host
 *    (before any launch).  Errors that depend on tensor VALUES (a non-finite
 *    input) are written asynchronously into the caller-provided device word
 *    `dev_status` (int32, may be NULL); read it with tango_status_poll after
 *    the stream has run.  Output tensors of a call that saw a non-finite input
 *    are unspecified.
 *  - Layouts are row-major.  Node rows are head-major concatenations
 *    [h][d] (reading R15).  int8 matrices carry an explicit leading
 *    dimension `ld` (elements) which must be a multiple of 16 (TMA) and,
 *    for outputs written by the GEMM epilogue, of 32; bytes between the
 *    logical width and ld are zero padding.
 *  - Edge arrays are indexed by in-CSR position (destination-major, sources
 *    ascending: reading R14).
 *  - No C++ exception crosses this ABI.  All functions are reentrant; a
 *    tango_comm may be used by one stream at a time.
 */
#ifndef TANGO_H_
#define TANGO_H_

#include <stddef.h>
#include <stdint.h>
#include <cuda_runtime_api.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TANGO_ABI_VERSION 1

typedef enum {
  TANGO_OK = 0,
  TANGO_ERR_INVALID_ARG = 1,   /* NULL required pointer, bad enum, bad ctx size */
  TANGO_ERR_SHAPE = 2,         /* inconsistent sizes / heads / leading dimensions */
  TANGO_ERR_BITS = 3,          /* bit-width outside [2, 8] (reading R25) */
  TANGO_ERR_NONFINITE = 4,     /* (device status) NaN / Inf in a tensor being quantized */
  TANGO_ERR_OVERFLOW = 5,      /* a contraction length that could overflow int32 (reading R27) */
  TANGO_ERR_UNSUPPORTED = 6,   /* a shape this build does not implement (HD not in {64..512}, n_global*HD >= 2^32) */
  TANGO_ERR_CUDA = 7,          /* a CUDA launch / runtime error */
  TANGO_ERR_NCCL = 8           /* a NCCL error (multi-GPU) */
} tango_status;

const char* tango_status_string(tango_status s);
int tango_abi_version(void);

/* Reads a device status word written by earlier asynchronous work on `stream`.
 * SYNCHRONIZES the stream.  *out receives TANGO_OK or the first error seen. */
tango_status tango_status_poll(const int32_t* dev_status, cudaStream_t stream, tango_status* out);

/* ------------------------------------------------------------------------- */
/* Graph G ("sparse adjacency matrix G"; incidence rows P:831-832)  */
/* ------------------------------------------------------------------------- */
typedef struct {
  int64_t n_global;        /* N: number of nodes in the whole graph */
  int64_t row_begin;       /* owned node block [row_begin, row_end); one GPU: 0, N */
  int64_t row_end;
  /* in-CSR of the owned destination rows: in_ptr[n_local+1] (offsets from 0),
   * in_src[e_in] = GLOBAL source ids, ascending within a row. */
  const int64_t* in_ptr;
  const int32_t* in_src;
  int64_t e_in;
  /* out-CSR of the owned source rows: out_ptr[n_local+1], out_dst[e_out] =
   * GLOBAL destination ids ascending within a row; out_eid[e_out] = position
   * of that edge in the in-CSR (needed only by the standalone OUT-direction
   * primitives with explicit edge weights; may be NULL otherwise). */
  const int64_t* out_ptr;
  const int32_t* out_dst;
  const int32_t* out_eid;
  int64_t e_out;
  int32_t chunk_edges;     /* C_E of the canonical chunked sums (reading R14); 0 => 256 */
  /* Caller-chosen identity of this graph's CONTENTS for the static-plan cache (segment plans,
   * in-CSR -> out-CSR map) kept in a layer ctx: two calls with the same ctx and the same nonzero
   * graph_id reuse the plans built by the first; 0 rebuilds them on every call.  A caller that modifies
   * the graph arrays in place must give the new contents a new id. */
  uint64_t graph_id;
} tango_graph;

/* Quantized tensor (DS6): int8 codes [rows][ld] + DEVICE fp32 scale s,
 * dequantized value = code * s (Eq.2 with Z = 0, reading R1). */
typedef struct {
  int8_t* q;
  float* scale;            /* device scalar */
  int64_t rows, cols, ld;
  int32_t bits;            /* 2..8 */
} tango_qtensor;

/* Philox4x32-10 stream for stochastic rounding (Eq.3; reading R4/R5):
 * element g of a tensor draws half-word (g & 7) of
 * Philox(ctr = {lo32(g>>3), hi32(g>>3), tag, step}, key = seed). */
typedef struct {
  uint64_t seed;
  uint32_t step;           /* training iteration */
  uint32_t tag;            /* (layer_id << 8) | role, roles: H=1 W=2 H'=3 S=4 D=5 dHout=6 dH'=7 Ys=8 Gs=9 dY=10 */
} tango_rng;

/* ------------------------------------------------------------------------- */
/* Primitive 1 — quantize (§2.3 Eq.1; §3.2 Eq.3).         */
/* x: fp32 [rows][cols] (row stride cols).  amax = max|x| over the tensor      */
/* (or *amax_hint if non-NULL; a device scalar, e.g. produced by the previous  */
/* kernel), s = amax/qmax, r = qmax/amax (s = r = 1 if amax = 0),              */
/* q = clamp(floor(x*r) + (u < frac), ±qmax).  Element (i, j) uses the global  */
/* index g = (global_row0 + i) * cols + j.  out->q: [rows][out->ld], padding   */
/* columns are written as 0.  out->scale receives s.  amax_out (nullable):     */
/* device scalar receiving amax.  Non-finite x => *dev_status = NONFINITE.    */
/* ------------------------------------------------------------------------- */
tango_status tango_quantize(const float* x, int64_t rows, int64_t cols, int64_t global_row0,
                            const float* amax_hint, tango_rng rng, tango_qtensor* out, float* amax_out,
                            int32_t* dev_status, cudaStream_t stream);

/* ------------------------------------------------------------------------- */
/* Primitive 2 — quantization-aware GEMM (§3.2 Fig.4; P:736-739     */
/* §3.3): acc = A·B in exact integer arithmetic on the int8 tensor cores      */
/* (tcgen05.mma kind::i8), dequantized in the epilogue: C = (float)acc *      */
/* (s_A*s_B).  Logical A is M×K, logical B is K×N.                             */
/*   a_layout TANGO_K_MAJOR : A->q is [M][A->ld]  (row m holds K codes)        */
/*   a_layout TANGO_MN_MAJOR: A->q is [K][A->ld]  (row k holds M codes)        */
/*   b_layout TANGO_K_MAJOR : B->q is [N][B->ld]  (i.e. Bᵀ, row n holds K)     */
/*   b_layout TANGO_MN_MAJOR: B->q is [K][B->ld]  (row k holds N codes)        */
/* Outputs (each nullable, at least one non-NULL): C fp32 [M][N];             */
/* C_i32 int32 [M][N] raw accumulator (requires K <= 133,144, reading R27);    */
/* C_i64 int64 [M][N] raw accumulator for any K (split-K, int64 reduction;    */
/* C_i64 is OVERWRITTEN).  C requires K <= 133,144 or uses split-K as well.   */
/* ------------------------------------------------------------------------- */
enum { TANGO_K_MAJOR = 0, TANGO_MN_MAJOR = 1 };
tango_status tango_gemm_q(const tango_qtensor* A, int32_t a_layout, const tango_qtensor* B, int32_t b_layout,
                          int64_t M, int64_t N, int64_t K, float* C, int32_t* C_i32, int64_t* C_i64,
                          cudaStream_t stream);

/* ------------------------------------------------------------------------- */
/* Primitive 3 — SDDMM on quantized node features.                            */
/*  TANGO_SDDMM_ADD (③, §2.1; on-the-fly dequantization P:864-873): */
/*    e_pre[e,h] = q_S[u,h]*s_S + q_D[v,h]*s_D ; el = e_pre>0 ? e_pre : e_pre*slope */
/*    Xsrc = S [N][heads], Xdst = D [n_local][heads]; out0 = e_pre, out1 = el  */
/*  TANGO_SDDMM_DOT (⑤″; directly on codes P:875-876):             */
/*    out0[e,h] = (float)(Σ_d q_A[v,h,d] q_B[u,h,d]) * (s_A*s_B)               */
/*    Xdst = A (destination rows, e.g. ∂H_out), Xsrc = B (source rows, H′);    */
/*    acc_i32 (nullable): raw int32 dots [e][heads].  out1 unused.             */
/* Edge outputs are [e_in][heads] fp32 in in-CSR order.                       */
/* ------------------------------------------------------------------------- */
enum { TANGO_SDDMM_ADD = 0, TANGO_SDDMM_DOT = 1 };
tango_status tango_sddmm_q(const tango_graph* G, int32_t op, const tango_qtensor* Xsrc, const tango_qtensor* Xdst,
                           int32_t heads, float slope, float* out0, float* out1, int32_t* acc_i32,
                           cudaStream_t stream);

/* Edge softmax ④ in FP32 (full precision P:604-615, R9, R12, R13, */
/* R14): m = max el over in-edges, den = Σᶜ exp_p(el-m), α = exp_p(el-m)/den. */
/* el, alpha: [e_in][heads]; m, den: [n_local][heads] (m = den = 0 if empty). */
tango_status tango_edge_softmax(const tango_graph* G, int32_t heads, const float* el, float* m, float* den,
                                float* alpha, cudaStream_t stream);

/* Softmax backward ④′ + LeakyReLU backward (R11):               */
/* P[v,h] = Σᶜ fmaf(∂α, α); ∂E = α(∂α − P[v]); ∂E_pre = e_pre>0 ? ∂E : ∂E·slope */
tango_status tango_softmax_bwd(const tango_graph* G, int32_t heads, const float* alpha, const float* dalpha,
                               const float* e_pre, float slope, float* P, float* dE_pre, cudaStream_t stream);

/* ------------------------------------------------------------------------- */
/* Primitive 4 — SPMM on quantized node features (⑤ P:224-227; ⑤′ P:248-251; */
/* incidence SPMM ③′/③″ P:276; GCN P:347-348).                    */
/*  edge_w != NULL: out[v,j] = (Σᶜ fmaf(w[e,h(j)], q_X[w_e,j])) * s_X, fp32   */
/*     accumulation, dir TANGO_IN sums in-edges (w_e = source),               */
/*     dir TANGO_OUT sums out-edges (w_e = destination, weight w[out_eid[e]]).*/
/*  edge_w == NULL: out_i32[v,j] = Σ q_X[w_e,j] (exact int32, order-free);     */
/*     out (nullable) = (float)out_i32 * s_X.                                  */
/*  row_scale (nullable, device [n_local]): out[v,j] = out[v,j] * row_scale[v] */
/*     (one more rn multiply; the GCN normalisation nd / ns, reading R26).     */
/*  amax_out (nullable, device fp32 scalar, pre-set by the caller, e.g. 0):    */
/*     atomically raised to max |out| (the next layer's quantization scale,   */
/*     P:736-739), order-free.                                                 */
/* X: [n_global][X->ld] codes with X->cols = heads*D.  out [n_local][cols].    */
/* ------------------------------------------------------------------------- */
enum { TANGO_IN = 0, TANGO_OUT = 1 };
tango_status tango_spmm_q(const tango_graph* G, int32_t dir, const float* edge_w, const tango_qtensor* X,
                          int32_t heads, const float* row_scale, float* out, int32_t* out_i32, float* amax_out,
                          cudaStream_t stream);

/* NEXT-4 int8-α SPMM (edge-feature quantization P:900-902 applied to α): the edge weights
 * are int8 codes Aq (rows = e_in or e_out edges in in-CSR slot order, cols = heads, ld = heads, scale
 * Aq->scale, e.g. from tango_quantize of α), so the aggregation is an exact, order-free int32 sum:
 *   out_i32[v,j] = Σ_e Aq[e,h(j)]·q_X[w_e,j]   (dir TANGO_IN: in-edges, w_e = source, Aq in in-CSR order;
 *                                            dir TANGO_OUT: out-edges, w_e = destination, Aq[out_eid[e]])
 *   out[v,j] (nullable) = i2f(out_i32[v,j]) · fl(s_α·s_X)
 * out_i32 [n_local][cols] is required (it is also the accumulator; zeroed by the call), 16-B aligned.
 * Requires cols = heads·D with D % 4 == 0, X->ld % 4 == 0 and X->q 4-B aligned: TANGO_ERR_UNSUPPORTED
 * otherwise.  Exactness needs deg·127² < 2³¹ (deg < 133,144): TANGO_ERR_OVERFLOW is not checked per row. */
tango_status tango_spmm_q8(const tango_graph* G, int32_t dir, const tango_qtensor* Aq, const tango_qtensor* X,
                           int32_t heads, int32_t* out_i32, float* out, cudaStream_t stream);

/* Incidence-matrix SPMM for edge features (③″/③′):        */
/* out[v,h] = Σᶜ x[e,h] over the in-edges (dir IN) or out-edges (dir OUT).    */
tango_status tango_edge_sum(const tango_graph* G, int32_t dir, int32_t heads, const float* x, float* out,
                            cudaStream_t stream);

/* ------------------------------------------------------------------------- */
/* NEXT-4: 4-bit node features for the SDDMM primitives     */
/* (§4.4, Fig.18a).  Packed layout: element 2i of a row in the low */
/* nibble of byte i, element 2i+1 in the high nibble, 4-bit two's complement, */
/* codes in [−7, 7] (qmax = 2^(4−1) − 1).                                     */
/* ------------------------------------------------------------------------- */
/* SR quantization to packed 4-bit codes: the same scale rule, Philox stream and
 * element index g = (global_row0 + i)·cols + j as tango_quantize with bits = 4.
 * cols % 8 == 0; q: [rows][ld_bytes] (ld_bytes % 4 == 0, >= cols/2); x 16-B and q
 * 4-B aligned.  scale_out, amax_out: device scalars (amax_out doubles as the amax
 * slot; amax_hint, if given, is copied into it). */
tango_status tango_quantize_int4(const float* x, int64_t rows, int64_t cols, int64_t global_row0,
                                 const float* amax_hint, tango_rng rng, uint8_t* q, int64_t ld_bytes, float* scale_out,
                                 float* amax_out, int32_t* dev_status, cudaStream_t stream);
/* SDDMM on bits-bit codes (bits = 8: int8 bytes, bits = 4: packed nibbles), one warp per
 * destination row, the same values as tango_sddmm_q:
 *  TANGO_SDDMM_DOT: out0[e,h] = i2f(Σ_d qA[v,h,d]·qB[u,h,d])·(s_dst·s_src), Xdst = A (rows of the
 *    owned destinations, global row index), Xsrc = B (global rows); cols = heads·D codes per row,
 *    row words (32/bits codes per 32-bit word) <= 32, words per head a power of two, ld % 4 == 0.
 *  TANGO_SDDMM_ADD: cols == heads; e_pre = qS[u,h]·s_src + qD[v,h]·s_dst -> out0 (nullable),
 *    LeakyReLU -> out1 (nullable).
 * ld_src / ld_dst in bytes.  Edge outputs [e_in][heads] in in-CSR order. */
tango_status tango_sddmm_qn(const tango_graph* G, int32_t op, int32_t bits, const void* Xsrc, int64_t ld_src,
                            const float* s_src, const void* Xdst, int64_t ld_dst, const float* s_dst, int32_t heads,
                            int32_t cols, float slope, float* out0, float* out1, cudaStream_t stream);

/* ------------------------------------------------------------------------- */
/* Bit-width derivation (§3.2 Eq.4, Fig.5).  */
/* ------------------------------------------------------------------------- */
/* Error_X of codes q (with their scale) against x: the mean over the rows x cols
 * tensor of |X − X̂| / (|X| + |X̂| + ε), X̂ = i2f(q)·s, ε = 0.0005; the
 * denominator takes absolute values (reading A24: the printed X + X̂ + ε can be
 * <= 0 for small negative values, contradicting the stated [0, 1] range).  Terms
 * in fp32 (rn), the sum in fp64 (order not fixed).  err_out: device double. */
tango_status tango_quant_error(const float* x, int64_t rows, int64_t cols, const tango_qtensor* q, double* err_out,
                               cudaStream_t stream);
/* select_bits: for B in [bmin, bmax] (2 <= bmin <= bmax <= 8) the Error_X of x
 * quantized to B bits with NEAREST rounding (reading R31) -> errs_out[B − bmin]
 * (device doubles); bits_out (device int32) = the smallest B with Error_X <=
 * threshold ("we let Error_X = 0.3"), or −bmax if no width qualifies.
 * bits_out doubles as scratch for amax(x) during the call. */
tango_status tango_select_bits(const float* x, int64_t count, float threshold, int32_t bmin, int32_t bmax,
                               double* errs_out, int32_t* bits_out, cudaStream_t stream);

/* ------------------------------------------------------------------------- */
/* Fused GAT layer (§2.1 Fig.1 with §3.2-3.3 quantization rules).  */
/* Forward: F1 Q(H), F2 Q(W), F3 ①② tcgen05 GEMM + head dots, F4 Q(H′),Q(S),Q(D),
 * F5/F6 ③④⑤ one destination-row kernel.  Backward: B1 Q(∂H_out), B2-B4 one  */
/* destination-row kernel, B5-B7 one source-row kernel, B8 Q(∂H′), B9 ①′ GEMMs.*/
/* ------------------------------------------------------------------------- */
typedef struct {
  const float* W;          /* device [in_feats][heads*head_dim] fp32 master weights */
  const float* a_src;      /* device [heads*head_dim] */
  const float* a_dst;      /* device [heads*head_dim] */
  int32_t in_feats, heads, head_dim;
  float neg_slope;         /* LeakyReLU slope (R11) */
  int32_t bits;            /* quantization bits B (8 on the hot path, R25) */
} tango_gat_params;

/* Size of the caller-allocated ctx (device memory, 256-B aligned) holding the
 * forward->backward cache (q_H, q_W, q_H′, q_S, q_D, m, den, scales)
 * and all scratch of both passes.  0 on invalid arguments. */
size_t tango_gat_ctx_bytes(const tango_graph* G, const tango_gat_params* p);

/* H: [n_local][in_feats] fp32 (this rank's rows).  amax_H_hint (nullable): device
 * scalar max|H| over ALL ranks (e.g. the previous layer's amax_out) — skips the
 * amax pass.  H_out: [n_local][heads*head_dim] fp32.  amax_out (nullable): device
 * scalar receiving max|H_out| (hint for the next layer).  comm: NULL on one GPU. */
struct tango_comm;
tango_status tango_gat_layer_fwd(const tango_graph* G, const tango_gat_params* p, const float* H,
                                 const float* amax_H_hint, tango_rng rng, uint32_t layer_id, void* ctx,
                                 size_t ctx_bytes, float* H_out, float* amax_out, struct tango_comm* comm,
                                 int32_t* dev_status, cudaStream_t stream);

/* Must follow tango_gat_layer_fwd on the same graph, params and ctx (it reuses the
 * forward's cache, including the in-CSR segment plan).
 * dH_out: [n_local][heads*head_dim].  dH (nullable): [n_local][in_feats];
 * dW: [in_feats][heads*head_dim]; da_src, da_dst: [heads*head_dim]; all fp32,
 * all overwritten.  amax_dH (nullable): device scalar receiving max|dH|. */
tango_status tango_gat_layer_bwd(const tango_graph* G, const tango_gat_params* p, void* ctx, size_t ctx_bytes,
                                 const float* dH_out, const float* amax_dH_hint, tango_rng rng, uint32_t layer_id,
                                 float* dH, float* dW, float* da_src, float* da_dst, float* amax_dH,
                                 struct tango_comm* comm, int32_t* dev_status, cudaStream_t stream);

/* Debug views into a GAT ctx (device pointers inside ctx; for parity tests).  */
typedef struct {
  int8_t *qH, *qW, *qWt, *qHp, *qS, *qD, *qG, *qdHp;
  int64_t ldF, ldHD, ldFt;
  float *S, *D, *m, *den, *P, *dD, *dHp, *dalpha;   /* dalpha: [e_in][H] ∂α */
  float *alpha_pack;       /* dataflow 1: [e_in][2H] α (sign bit = LeakyReLU branch of e_pre) | ∂E_pre;
                              dataflow 2: [e_out][H] ∂α in out-CSR order (α, ∂E_pre are recomputed) */
  float *scalars;          /* see DESIGN.md §4 "ctx scalars" for the slot map */
  int32_t codes_biased;    /* 1: qHp and qG hold excess-128 codes (bit pattern q ^ 0x80) */
  float *dS;               /* [n_global][H] ∂S (③′) of the owned rows */
  int32_t dataflow;        /* 1: round-1 kernels (α stored); 2: v6 (single GPU, α recomputed, one
                              row-gather pass in the backward) */
} tango_gat_ctx_view;
tango_status tango_gat_ctx_get_view(const tango_graph* G, const tango_gat_params* p, void* ctx,
                                    tango_gat_ctx_view* view);

/* ------------------------------------------------------------------------- */
/* GCN layer: GEMM + SPMM (§2.2), DGL norm='both' folded into rows  */
/* (reading R26): out = diag(nd) · A · diag(ns) · (X·W), int32 aggregation.   */
/* ------------------------------------------------------------------------- */
typedef struct {
  const float* W;          /* device [in_feats][out_feats] */
  int32_t in_feats, out_feats;
  int32_t bits;
} tango_gcn_params;

size_t tango_gcn_ctx_bytes(const tango_graph* G, const tango_gcn_params* p);
tango_status tango_gcn_layer_fwd(const tango_graph* G, const tango_gcn_params* p, const float* X,
                                 const float* amax_X_hint, tango_rng rng, uint32_t layer_id, void* ctx,
                                 size_t ctx_bytes, float* out, float* amax_out, struct tango_comm* comm,
                                 int32_t* dev_status, cudaStream_t stream);
tango_status tango_gcn_layer_bwd(const tango_graph* G, const tango_gcn_params* p, void* ctx, size_t ctx_bytes,
                                 const float* dout, tango_rng rng, uint32_t layer_id, float* dX, float* dW,
                                 struct tango_comm* comm, int32_t* dev_status, cudaStream_t stream);

typedef struct {
  int8_t *qX, *qW, *qWt, *qYs, *qGs, *qdY;
  int64_t ldF, ldO, ldFt;
  int32_t *ia, *ib;
  float *scalars;
} tango_gcn_ctx_view;
tango_status tango_gcn_ctx_get_view(const tango_graph* G, const tango_gcn_params* p, void* ctx,
                                    tango_gcn_ctx_view* view);

/* ------------------------------------------------------------------------- */
/* NEXT-1: the training step around the quantized layer.     */
/* ------------------------------------------------------------------------- */
/* Full-precision GEMM (the FP32 final layer, §3.2 Eq.7-8) with the  */
/* pinned order of reading R33: C[m][n] = Σᶜ_k fmaf(A(m,k), B(k,n)), chunks of */
/* 1024 k folded left to right (a K <= 1024 contraction is one fmaf chain).    */
/* Layouts as tango_gemm_q: a_layout K_MAJOR: A is [M][lda]; MN_MAJOR: A is    */
/* [K][lda].  b_layout K_MAJOR: B is [N][ldb] (Bᵀ); MN_MAJOR: B is [K][ldb].   */
/* C: fp32 [M][N] (row stride N), overwritten.  workspace: device scratch of   */
/* tango_sgemm_workspace_bytes(M,N,K) bytes (0 when K <= 1024; may be NULL).  */
size_t tango_sgemm_workspace_bytes(int64_t M, int64_t N, int64_t K);
tango_status tango_sgemm(const float* A, int64_t lda, int32_t a_layout, const float* B, int64_t ldb, int32_t b_layout,
                         int64_t M, int64_t N, int64_t K, float* C, void* workspace, size_t ws_bytes,
                         cudaStream_t stream);

/* Column sums over rows with the same chunked order (R33): out[j] = Σᶜ_r x[r][j].
 * x: [rows][cols] fp32; out: [cols]; workspace as tango_colsum_workspace_bytes. */
size_t tango_colsum_workspace_bytes(int64_t rows, int64_t cols);
tango_status tango_colsum(const float* x, int64_t rows, int64_t cols, float* out, void* workspace, size_t ws_bytes,
                          cudaStream_t stream);

/* Hidden-layer bias + ReLU (reading R34; P:998-1001 does not fix them):
 * y = max(x + bias[j], 0) (one rn add), amax_out (nullable device scalar) = max y,
 * the amax hint of the next layer's Q(H).  x, y: [rows][cols] (may alias). */
tango_status tango_bias_act_fwd(const float* x, const float* bias, int64_t rows, int64_t cols, float* y,
                                float* amax_out, cudaStream_t stream);
/* Backward: dx = y > 0 ? dy : 0, dbias = Σᶜ_r dx (R33), amax_dx (nullable) = max|dx|,
 * the ∂H_out amax hint of the quantized layer below.  workspace: tango_colsum_workspace_bytes. */
tango_status tango_bias_act_bwd(const float* y, const float* dy, int64_t rows, int64_t cols, float* dx, float* dbias,
                                float* amax_dx, void* workspace, size_t ws_bytes, cudaStream_t stream);

/* Mean cross-entropy over labelled rows (reading R36; node classification P:987-990):
 * labels[v] in [0, classes) or −1 (unlabelled: zero gradient).  Per labelled row:
 * m = max z, Σ = Σ_c exp_p(z_c − m) in class order, loss_v = (m + logf Σ) − z_y,
 * dlogits_c = (exp_p(z_c − m)/Σ − [c = y]) / n_labeled.  loss_out: device double =
 * Σ_v loss_v / n_labeled (order-free double sum).  A label >= classes writes
 * TANGO_ERR_INVALID_ARG to *dev_status.  classes <= 1024. */
tango_status tango_cross_entropy(const float* logits, const int32_t* labels, int64_t rows, int32_t classes,
                                 int64_t n_labeled, float* dlogits, double* loss_out, int32_t* dev_status,
                                 cudaStream_t stream);

/* FP32 master-weight update (§3.2 Eq.6, add-then-quantize; reading R37):
 * w ← w − lr·g (two rn ops) for every listed tensor, in one launch (<= 32 tensors;
 * the host array is read during the call only).  The next step's Q(W) quantizes the
 * updated master. */
typedef struct { float* w; const float* g; int64_t count; } tango_sgd_tensor;
tango_status tango_sgd_update(const tango_sgd_tensor* tensors, int32_t count, float lr, cudaStream_t stream);

/* Full-precision final GAT layer ("use full precision to compute the layer
 * before the Softmax"; reading R35): FP32 ① H′ = H·W (tango_sgemm order), ② S, D
 * (sequential fmaf per head), ③ e_pre = S[u] + D[v] + LeakyReLU, ④ edge softmax
 * (exp_p, Σᶜ), ⑤ Σᶜ fmaf(α, H′[u]) per head, then logits = ((Σ_h, in head order)/heads)
 * + bias.  One GPU only (row_begin = 0, row_end = n_global; out_eid required):
 * TANGO_ERR_UNSUPPORTED otherwise.  heads*classes <= 1024. */
typedef struct {
  const float* W;          /* device [in_feats][heads*classes] */
  const float* a_src;      /* device [heads*classes] */
  const float* a_dst;
  const float* bias;       /* device [classes] */
  int32_t in_feats, heads, classes;
  float neg_slope;
} tango_gat_out_params;
size_t tango_gat_out_ctx_bytes(const tango_graph* G, const tango_gat_out_params* p);
/* H: [n][in_feats]; logits: [n][classes]. */
tango_status tango_gat_out_fwd(const tango_graph* G, const tango_gat_out_params* p, const float* H, void* ctx,
                               size_t ctx_bytes, float* logits, cudaStream_t stream);
/* Must follow tango_gat_out_fwd on the same H and ctx.  dlogits: [n][classes].
 * dH (nullable): [n][in_feats]; dW [in_feats][heads*classes]; da_src, da_dst
 * [heads*classes] (order-free atomics); dbias [classes]; all overwritten. */
tango_status tango_gat_out_bwd(const tango_graph* G, const tango_gat_out_params* p, void* ctx, size_t ctx_bytes,
                               const float* H, const float* dlogits, float* dH, float* dW, float* da_src,
                               float* da_dst, float* dbias, cudaStream_t stream);
typedef struct {
  float *Hp, *S, *D, *e_pre, *alpha, *m, *den;      /* forward: [n][HC], [n][H] x2, [e][H] x2, [n][H] x2 */
  float *G, *dalpha, *dE_pre, *P, *dD, *dS, *dHp;  /* backward: [n][C], [e][H] x2, [n][H] x3, [n][HC] */
  float *agg;                                      /* forward ⑤ before the head mean: [n][HC] */
} tango_gat_out_ctx_view;
tango_status tango_gat_out_ctx_get_view(const tango_graph* G, const tango_gat_out_params* p, void* ctx,
                                        tango_gat_out_ctx_view* view);

/* Full-precision final GCN layer (P:604-615 FP32 rule; GCN P:347-348 with the norm='both'
 * rows of reading R26; bias R35): Y = X·W (tango_sgemm order), Ys = Y·ns[u],
 * agg[v] = Σᶜ over in-edges Ys[u] (plain adds, R14), logits = agg·nd[v] + bias.
 * Backward: dbias = Σᶜ_v dlogits, Gs = dlogits·nd[v], aggb[u] = Σᶜ over out-edges Gs[v],
 * dY = aggb·ns[u], dX = dY·Wᵀ (nullable), dW = Xᵀ·dY.  One GPU only; classes <= 1024. */
typedef struct {
  const float* W;          /* device [in_feats][classes] */
  const float* bias;       /* device [classes] */
  int32_t in_feats, classes;
} tango_gcn_out_params;
size_t tango_gcn_out_ctx_bytes(const tango_graph* G, const tango_gcn_out_params* p);
tango_status tango_gcn_out_fwd(const tango_graph* G, const tango_gcn_out_params* p, const float* X, void* ctx,
                               size_t ctx_bytes, float* logits, cudaStream_t stream);
tango_status tango_gcn_out_bwd(const tango_graph* G, const tango_gcn_out_params* p, void* ctx, size_t ctx_bytes,
                               const float* X, const float* dlogits, float* dX, float* dW, float* dbias,
                               cudaStream_t stream);
typedef struct { float *Y, *Ys, *agg, *Gs, *aggb, *dY; } tango_gcn_out_ctx_view;   /* each [n][classes] */
tango_status tango_gcn_out_ctx_get_view(const tango_graph* G, const tango_gcn_out_params* p, void* ctx,
                                        tango_gcn_out_ctx_view* view);

/* ------------------------------------------------------------------------- */
/* Multi-GPU (destination-row partitioning): an NCCL          */
/* communicator built from a 128-byte ncclUniqueId that the caller broadcasts  */
/* (e.g. with torch.distributed).  Collectives are enqueued on the caller's    */
/* stream: AllReduce-MAX of amax scalars (R28), AllGather of int8 node rows,   */
/* AllReduce-SUM of int64 ∂W partials and fp32 ∂a.                            */
/* ------------------------------------------------------------------------- */
int32_t tango_comm_unique_id_bytes(void);
tango_status tango_comm_get_unique_id(void* id_out /* tango_comm_unique_id_bytes() bytes */);
tango_status tango_comm_init(struct tango_comm** out, const void* unique_id, int32_t nranks, int32_t rank);
tango_status tango_comm_destroy(struct tango_comm* comm);
/* In-process loopback group (validation of the partitioned path on ONE GPU): nranks
 * host threads, one tango_comm each (tango_comm_init_local), exchange through device
 * memory with host barriers; the collectives have the NCCL semantics above (fp32 sums
 * in rank order).  Every rank must enter every collective (blocking rendezvous).  Not
 * CUDA-graph capturable.  nranks <= 16. */
struct tango_local_group;
tango_status tango_local_group_create(struct tango_local_group** out, int32_t nranks);
tango_status tango_local_group_destroy(struct tango_local_group* group);
tango_status tango_comm_init_local(struct tango_comm** out, struct tango_local_group* group, int32_t rank);
/* Row partition of the node set: rank r owns [row_starts[r], row_starts[r+1]).
 * Must be called (identically on every rank) before a layer call with this comm. */
tango_status tango_comm_set_partition(struct tango_comm* comm, const int64_t* row_starts /* nranks+1, host */);
/* always != 0: a one-rank NCCL communicator still enqueues every collective (identities on one rank),
 * so the NCCL data plane executes on one GPU exactly as with N ranks (tests, bench --nccl-single). */
tango_status tango_comm_set_options(struct tango_comm* comm, int32_t always);
/* Allocates (outside any graph capture) the staging buffer of the padded all-gather: nranks x largest
 * row block x max_row_bytes device bytes, owned by the comm and freed by tango_comm_destroy.  Without
 * it, node-row all-gathers run as grouped in-place broadcasts.  Call after tango_comm_set_partition. */
tango_status tango_comm_reserve(struct tango_comm* comm, size_t max_row_bytes);
/* Number of NCCL collectives this comm has enqueued (an all-gather counts once, a broadcast group once
 * per broadcast); -1 for NULL. */
int64_t tango_comm_nccl_calls(const struct tango_comm* comm);

/* ------------------------------------------------------------------------- */
/* Tracing: every kernel launch increments a counter; with profiling enabled  */
/* each launch is bracketed by CUDA events on its stream and device time is   */
/* accumulated per kernel name (host-side state, process-wide, thread-safe).  */
/* ------------------------------------------------------------------------- */
void tango_profile_enable(int32_t on);
/* NVTX ranges (one per kernel launch, named after the kernel) for timeline tools; default from the
 * environment variable TANGO_NVTX (off). */
void tango_nvtx_enable(int32_t on);
int64_t tango_launch_count(void);
tango_status tango_profile_collect(void);          /* waits for the recorded events */
int32_t tango_profile_num_entries(void);
tango_status tango_profile_entry(int32_t i, char* name, int32_t name_cap, double* total_ms, int64_t* launches);
void tango_profile_reset(void);
/* on != 0: layer calls run their side-stream work (Q(W), graph plans, hub-row chains, the ∂a
 * reduction) in order on the caller's stream instead, so that per-launch event times measure each
 * kernel alone (bench.py's per-kernel pass).  Results are identical either way.  Process-wide. */
void tango_profile_serialize(int32_t on);

/* L2 fetch granularity for the calling thread's device (cudaLimitMaxL2FetchGranularity, bytes in
 * {0, 32, 64, 128}): the v6 passes gather 16-B per-edge records at random positions (∂α through the
 * in-CSR -> out-CSR map) and 4-B node codes, where a 128-B L2 fill multiplies the DRAM traffic.
 * Process-wide device setting, not a stream operation; *before (nullable) receives the previous value. */
tango_status tango_set_l2_fetch_granularity(int32_t bytes, int32_t* before);


#ifdef __cplusplus
}
#endif
#endif /* TANGO_H_ */
