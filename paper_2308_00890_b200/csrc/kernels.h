// kernels.h — internal launcher declarations of libtango (not part of the C ABI).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "common.cuh"

namespace tango {

int num_sms();


// Every kernel launch is wrapped in a ProfScope (prof.cu): launch counter + optional event timing.
class ProfScope {
 public:
  ProfScope(const char* name, cudaStream_t st);
  ~ProfScope();
 private:
  cudaStream_t st_;
  bool on_ = false;
  bool nvtx_ = false;
  int entry_ = -1;
  cudaEvent_t a_ = nullptr, b_ = nullptr;
};

// ---- quant.cu
cudaError_t launch_absmax(const float* x, int64_t rows, int64_t cols, const float* rowscale, unsigned* slot,
                          cudaStream_t st);
cudaError_t launch_quantize(const float* x, int64_t rows, int64_t cols, const float* rowscale, int64_t g0,
                            const unsigned* amax_slot, int bits, uint64_t seed, uint32_t step, uint32_t tag,
                            int8_t* q, int64_t ld, int8_t* qt, int64_t ldt, float* scale_out, int32_t* status,
                            cudaStream_t st, uint32_t code_xor = 0u);
cudaError_t launch_amax_to_scale(float* slot, int bits, cudaStream_t st);

cudaError_t launch_error_x(const float* x, int64_t rows, int64_t cols, const int8_t* q, int64_t ld, const float* s,
                           double* err, cudaStream_t st);
cudaError_t launch_select_bits(const float* x, int64_t count, float threshold, int bmin, int bmax, double* errs,
                               int32_t* bits, cudaStream_t st);

// ---- gemm_tc.cu : tcgen05 int8 GEMM with fused epilogues
enum EpiMode : int {
  EPI_AMAX = 0,     // v = i2f(acc)*sAB[*rowscale]; amax(|v|); optional per-head dots S = v·a_src, D = v·a_dst
  EPI_QUANT = 1,    // v as above -> SR quantize with the amax of a previous EPI_AMAX pass -> int8 out
  EPI_STORE = 2,    // v -> fp32 out [M][ldc]
  EPI_I32 = 3,      // raw int32 accumulator -> out [M][ldc]
  EPI_ATOMIC64 = 4  // raw accumulator atomically added into int64 out [M][ldc] (split-K)
};

struct GemmArgs {
  // operands
  const int8_t* A; int64_t lda; bool a_mn;  // K-major: A[M][lda]; MN-major: A[K][lda]
  const int8_t* B; int64_t ldb; bool b_mn;  // K-major: B[N][ldb]; MN-major: B[K][ldb]
  int64_t M, N, K;
  int splits;                               // split-K count (EPI_ATOMIC64 only)
  // scales: sAB = sA * sB (device scalars, may be null for raw modes)
  const float* sA; const float* sB;
  const float* rowscale;                    // optional per-row multiplier (GCN ns)
  int mode;
  // EPI_AMAX
  unsigned* amax_slot;                      // |v| max
  const float* a_src; const float* a_dst;   // optional head dots
  int head_dim;                             // D (columns per head)
  float* S; float* Dd; int heads;           // [M][heads] outputs of the head dots
  unsigned* amax_S; unsigned* amax_D;
  // EPI_QUANT
  const unsigned* amax_in; int bits; uint64_t seed; uint32_t step; uint32_t tag; int64_t g_row0;
  int8_t* q_out; int64_t ldq; float* scale_out; int32_t* status;
  uint32_t code_xor;                        // 0x80808080: store excess-128 codes (q + 128)
  // EPI_STORE / EPI_I32 / EPI_ATOMIC64
  void* C; int64_t ldc;
};
cudaError_t launch_gemm(const GemmArgs& a, cudaStream_t st);
bool make_row_gather_map(CUtensorMap* m, const void* base, uint64_t rows, uint64_t row_bytes, uint64_t ld_bytes);

// ---- gat.cu : fused GAT destination / source row kernels and standalone sparse primitives
struct GatDims { int heads, head_dim, hd; };
struct GraphDev {
  int64_t n_local, row_begin, n_global, e_in;
  const int64_t* in_ptr; const int32_t* in_src;
  const int64_t* out_ptr; const int32_t* out_dst; const int32_t* out_eid;
  int chunk;
};

// Segment plan of one CSR (gat.cu k_plan): rows with deg > C_E are "heavy" and split into
// ceil(deg/C_E) canonical chunks ("segments") with scratch slots [hbase[v], hbase[v] + nseg).
struct PlanDev {
  int32_t* hbase;      // [n_local] first slot of a heavy row, -1 for light rows
  int32_t* hseg_row;   // [cap] local row of each heavy segment slot
  int32_t* hrow;       // [n_local] heavy rows (first counts[1] entries)
  int32_t* counts;     // [0] = #heavy segments, [1] = #heavy rows, [2] = #light sub-tiles (zeroed first)
  int64_t cap;         // slot capacity: 2 * e / C_E + 1
  int32_t* tiles;      // [tcap] light-row sub-tiles (block, lo, hi) of k_plan_tiles
  int64_t tcap;        // n_local + n_local / 32 + 1
};
cudaError_t launch_plan(const int64_t* ptr, int64_t n, int chunk, const PlanDev& p, cudaStream_t st);
cudaError_t launch_plan_tiles(const int64_t* ptr, int64_t n, const PlanDev& p, cudaStream_t st);

struct GatFwdArgs {
  GraphDev g; GatDims d; float slope; int bits;
  const int8_t* qS; const unsigned* amax_S;   // [N][H]
  const int8_t* qD; const unsigned* amax_D;   // [N][H]
  const int8_t* qHp; int64_t ldHp; const unsigned* amax_Hp;   // [N][ldHp]
  float* Hout; float* m; float* den;          // Hout [n_local][HD]; m, den [N][H] (own rows written)
  unsigned* amax_out;
  PlanDev plan;                               // in-CSR plan
  float* hmax; float* hden;                   // [cap][H] heavy-segment softmax partials
  float* hagg;                                // [cap][HD] heavy-segment aggregation partials
  int32_t* work;                              // [8] work-queue counters (zeroed before the launch)
  float* alpha;                               // [e_in][2H]: α with the sign of e_pre (LeakyReLU branch) | ∂E_pre
  int part;                                   // work items: 0 all, 1 hub segments only, 2 light sub-tiles only
  int codes_biased;                           // q_H′ holds excess-128 codes (gat_codes_biased)
};
// aux (nullable): a second stream that runs the hub-row chain beside the light sub-tiles
// (fork/join with the two events); null -> everything in order on st.
struct SideStream { cudaStream_t s; cudaEvent_t fork, join; };
cudaError_t launch_gat_fwd(const GatFwdArgs& a, cudaStream_t st, const SideStream* aux = nullptr);
// true when the layer kernels for this shape take q_H′ and q_G as excess-128 codes (q + 128, stored
// as int8 bit patterns q ^ 0x80): the v4 gather engine then converts without the sign flip
bool gat_codes_biased(int heads, int hd);

struct GatBwdArgs {
  GraphDev g; GatDims d; float slope; int bits;
  const int8_t* qS; const unsigned* amax_S;
  const int8_t* qD; const unsigned* amax_D;
  const int8_t* qHp; int64_t ldHp; const unsigned* amax_Hp;
  const int8_t* qG; int64_t ldG; const unsigned* amax_G;   // [N][ldG]
  const float* m; const float* den;          // [N][H]
  float* dalpha;                             // scratch [e_in][H]
  float* P; float* dD;                       // [N][H] own rows written
  const float* a_src; const float* a_dst;
  float* dHp; unsigned* amax_dHp;            // [n_local][HD]
  float* da_src; float* da_dst;              // [HD], accumulated with atomics (pre-zeroed)
  float* dS;                                 // [N][H] ∂S of the owned rows (for the ∂a pass)
  PlanDev pin, pout;                         // in-CSR and out-CSR plans
  float* hP; float* hdD;                     // [pin.cap][H]
  float* hdS;                                // [pout.cap][H]
  float* hagg;                               // [pout.cap][HD]
  int32_t* work;                             // [8] work-queue counters (zeroed before the launch)
  const float* alpha;                        // [e_in][2H]: signed α from the forward | ∂E_pre (written here)
  float* alpha_dE;                           // same buffer, written by the destination passes
  int part;                                  // as GatFwdArgs::part
  int codes_biased;                          // q_H′ and q_G hold excess-128 codes (gat_codes_biased)
};
cudaError_t launch_gat_bwd_dst(const GatBwdArgs& a, cudaStream_t st, const SideStream* aux = nullptr);
cudaError_t launch_gat_bwd_src(const GatBwdArgs& a, cudaStream_t st, const SideStream* aux = nullptr);
cudaError_t launch_gat_attn_grad(const GatBwdArgs& a, cudaStream_t st);

// ---- gat2.cu : v6 single-GPU dataflow (α recomputed, one row-gather pass in the backward)
struct G2Args {
  GraphDev g; GatDims d; float slope; int bits;
  const int8_t* qS; const unsigned* amax_S;                  // [N][H]
  const int8_t* qD; const unsigned* amax_D;                  // [N][H]
  const int8_t* qHp; int64_t ldHp; const unsigned* amax_Hp;  // [N][ldHp] excess-128 codes
  const int8_t* qG; int64_t ldG; const unsigned* amax_G;     // [N][ldG] excess-128 codes
  float* m; float* den;                                      // [N][H]
  float* Hout; unsigned* amax_out;                           // forward output [n][HD]
  float* P; float* dD; float* dS;                            // [N][H]
  float* dal_out;                                            // [E][H] ∂α in out-CSR order
  float* dal_in;                                             // [E][H] ∂α of hub rows in in-CSR order (P2a -> P2b)
  const float* a_src; const float* a_dst;
  float* dHp; unsigned* amax_dHp;                            // [n][HD]: ∂H′_agg (P1) -> ∂H′ (P3)
  PlanDev pin, pout;
  float* hagg;                                               // [cap][HD] heavy-segment partials
  float* h1; float* h2;                                      // [pin.cap][H] segment partials (max, Σ, P, ∂D)
  float* hs;                                                 // [pout.cap][H] segment partials (∂S)
  int32_t* hcnt;                                             // [n] finished-segment counters (zeroed)
  int32_t* work;                                             // [8] work-queue counters (zeroed)
  float* da_part;                                            // [ceil(n/1024)][2 HD] ∂a chunk partials
  float* nrec; int nrs;                                      // [N][nrs] packed per-node record: m | den | P | q_D
  const int32_t* in2out;                                     // [E] out-CSR position of each in-CSR edge
  int scatter_in;                                            // P1 also writes ∂α at its in-CSR slot (dal_in)
  int hub_fs, hub_p2, hub_p3;                                // hub segments of F-stats / P2 / P3: 0 staged warp sums,
                                                             // 1 lane per (segment, head), 2 multi-segment staged
  float* alpha_st;                                           // [E][H] α from F-agg, sign = LeakyReLU branch (nullable)
  float* rec;                                                // [E][2H] P1's {∂α, signed α} at in-CSR slots (nullable)
  float* al_out;                                             // [E][H] P1's signed α in out-CSR order, for P3 (nullable)
  float* da_src; float* da_dst;                              // [HD]
  int codes_biased;
};
bool gat2_supported(const GraphDev& g, int heads, int hd);
constexpr int gat2_nrec_stride(int heads) { return heads <= 1 ? 4 : heads <= 2 ? 8 : heads <= 4 ? 16 : 32; }
cudaError_t launch_gat2_in2out(const int32_t* out_eid, int64_t e, int32_t* in2out, cudaStream_t st);
struct SideStream;
cudaError_t launch_gat2_fwd(const G2Args& a, cudaStream_t st, const SideStream* aux = nullptr);
cudaError_t launch_gat2_bwd(const G2Args& a, cudaStream_t st, const SideStream* aux = nullptr);
cudaError_t launch_gat2_attn_grad(const G2Args& a, cudaStream_t st);

// standalone primitives (unfused; used by the primitive C-ABI entry points)
cudaError_t launch_sddmm_add(const GraphDev& g, int heads, const int8_t* qS, const float* sS, const int8_t* qD,
                             const float* sD, float slope, float* e_pre, float* el, cudaStream_t st);
cudaError_t launch_sddmm_dot(const GraphDev& g, int heads, int hd_total, const int8_t* qA, int64_t lda,
                             const float* sA, const int8_t* qB, int64_t ldb, const float* sB, float* out,
                             int32_t* acc, cudaStream_t st);
cudaError_t launch_edge_softmax(const GraphDev& g, int heads, const float* el, float* m, float* den, float* alpha,
                                cudaStream_t st);
cudaError_t launch_softmax_bwd(const GraphDev& g, int heads, const float* alpha, const float* dalpha,
                               const float* e_pre, float slope, float* P, float* dEp, cudaStream_t st);
cudaError_t launch_edge_sum(const GraphDev& g, int dir, int heads, const float* x, float* out, int64_t e_list,
                            cudaStream_t st);
cudaError_t launch_spmm_w(const GraphDev& g, int dir, int heads, int cols, const float* w, const int8_t* qX,
                          int64_t ldx, const float* sX, const float* rowscale, float* out, unsigned* amax_out,
                          int64_t e_list, cudaStream_t st);
cudaError_t launch_spmm_q8(const GraphDev& g, int dir, int heads, int cols, const int8_t* qa, const float* sa,
                           const int8_t* qX, int64_t ldx, const float* sX, int32_t* out_i32, float* out,
                           int64_t e_list, cudaStream_t st);
cudaError_t launch_spmm_sum(const GraphDev& g, int dir, int cols, const int8_t* qX, int64_t ldx, const float* sX,
                            const float* rowscale, float* out, int32_t* out_i32, unsigned* amax_out,
                            cudaStream_t st);

// misc
cudaError_t launch_finalize_dw(const int64_t* acc, int64_t count, const float* sA, const float* sB, float* out,
                               cudaStream_t st);
cudaError_t launch_gcn_norms(const GraphDev& g, float* ns, float* nd, cudaStream_t st);

}  // namespace tango
