// api.cu — the C ABI of libtango.so (include/tango.h): argument validation, the ctx layout,
// orchestration of the fused kernels for one GAT / GCN layer (forward, backward) and the NCCL
// communicator for destination-row partitioning over several GPUs.
#include <nccl.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <algorithm>
#include <mutex>
#include <condition_variable>
#include <atomic>

#include "../../include/tango.h"
#include "kernels.h"

namespace tango {

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// tango_profile_serialize (see aux_stream)
static std::atomic<int> g_serialize{0};

static inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }
static inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// Philox tag = (layer_id << 8) | role (tango.h)
enum Role : uint32_t { R_H = 1, R_W = 2, R_HP = 3, R_S = 4, R_D = 5, R_G = 6, R_DHP = 7, R_YS = 8, R_GS = 9, R_DY = 10 };
static inline uint32_t tag_of(uint32_t layer, uint32_t role) { return (layer << 8) | role; }

// ctx scalar slots: amax bit patterns and scales, 64 x 4 B at the start of ctx.
enum Slot : int {
  SL_AMAX_H = 0, SL_AMAX_W = 1, SL_AMAX_HP = 2, SL_AMAX_S = 3, SL_AMAX_D = 4, SL_AMAX_G = 6, SL_AMAX_DHP = 7,
  SL_S_H = 8, SL_S_W = 9, SL_S_HP = 10, SL_S_S = 11, SL_S_D = 12, SL_S_G = 13, SL_S_DHP = 14,
  SL_NSLOTS = 64
};

}  // namespace tango

using namespace tango;

// In-process loopback group: nranks host threads on one device exchange through device memory
// (tests and one-GPU validation of the partitioned path; the NCCL communicator is the product path).
struct tango_local_group {
  int nranks = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<void*> ptr;             // per rank: buffer of the current collective
  std::vector<cudaEvent_t> ev_a, ev_b;
  std::vector<void*> tmp;             // per rank: reduction scratch (device)
  std::vector<size_t> tmp_bytes;
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t my = gen;
    if (++arrived == nranks) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != my; });
    }
  }
};

struct tango_comm {
  ncclComm_t nccl = nullptr;
  tango_local_group* local = nullptr;
  int nranks = 1, rank = 0;
  std::vector<int64_t> starts;  // nranks + 1
  int64_t max_rows = 0;         // largest row block
  bool always = false;          // run the NCCL collectives even with one rank (tango_comm_set_options)
  void* stage = nullptr;        // padded all-gather staging, nranks x max_rows x stage_row_bytes (tango_comm_reserve)
  size_t stage_row_bytes = 0;
  int64_t nccl_calls = 0;       // collectives enqueued (tango_comm_nccl_calls)
};

#define TRY_CUDA(x)                                  \
  do {                                               \
    cudaError_t e_ = (x);                            \
    if (e_ != cudaSuccess) {                         \
      fprintf(stderr, "[tango] CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return TANGO_ERR_CUDA;                         \
    }                                                \
  } while (0)
#define TRY_NCCL(x)                                  \
  do {                                               \
    ncclResult_t r_ = (x);                           \
    if (r_ != ncclSuccess) {                         \
      fprintf(stderr, "[tango] NCCL error %s at %s:%d\n", ncclGetErrorString(r_), __FILE__, __LINE__); \
      return TANGO_ERR_NCCL;                         \
    }                                                \
  } while (0)
#define TRY(x)                                       \
  do {                                               \
    tango_status s_ = (x);                           \
    if (s_ != TANGO_OK) return s_;                   \
  } while (0)

extern "C" {

const char* tango_status_string(tango_status s) {
  switch (s) {
    case TANGO_OK: return "ok";
    case TANGO_ERR_INVALID_ARG: return "invalid argument";
    case TANGO_ERR_SHAPE: return "shape mismatch";
    case TANGO_ERR_BITS: return "bit-width outside [2,8]";
    case TANGO_ERR_NONFINITE: return "non-finite value in a quantized tensor";
    case TANGO_ERR_OVERFLOW: return "contraction length may overflow int32";
    case TANGO_ERR_UNSUPPORTED: return "unsupported shape";
    case TANGO_ERR_CUDA: return "CUDA error";
    case TANGO_ERR_NCCL: return "NCCL error";
  }
  return "unknown";
}

int tango_abi_version(void) { return TANGO_ABI_VERSION; }

void tango_profile_serialize(int32_t on) { g_serialize.store(on ? 1 : 0, std::memory_order_relaxed); }

tango_status tango_set_l2_fetch_granularity(int32_t bytes, int32_t* before) {
  if (!(bytes == 0 || bytes == 32 || bytes == 64 || bytes == 128)) return TANGO_ERR_INVALID_ARG;
  size_t prev = 0;
  TRY_CUDA(cudaDeviceGetLimit(&prev, cudaLimitMaxL2FetchGranularity));
  if (before) *before = (int32_t)prev;
  TRY_CUDA(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)bytes));
  return TANGO_OK;
}


tango_status tango_status_poll(const int32_t* dev_status, cudaStream_t stream, tango_status* out) {
  if (!dev_status || !out) return TANGO_ERR_INVALID_ARG;
  int32_t v = 0;
  TRY_CUDA(cudaMemcpyAsync(&v, dev_status, sizeof(v), cudaMemcpyDeviceToHost, stream));
  TRY_CUDA(cudaStreamSynchronize(stream));
  *out = (tango_status)v;
  return TANGO_OK;
}

}  // extern "C"

// ------------------------------------------------------------------ validation helpers
static tango_status check_graph(const tango_graph* G, bool need_out) {
  if (!G || !G->in_ptr) return TANGO_ERR_INVALID_ARG;
  if (G->n_global < 0 || G->row_begin < 0 || G->row_end < G->row_begin || G->row_end > G->n_global)
    return TANGO_ERR_SHAPE;
  if (G->e_in > 0 && !G->in_src) return TANGO_ERR_INVALID_ARG;
  if (G->e_in >= (int64_t(1) << 31) || G->e_out >= (int64_t(1) << 31) || G->n_global >= (int64_t(1) << 31))
    return TANGO_ERR_UNSUPPORTED;
  if (need_out && (!G->out_ptr || (G->e_out > 0 && !G->out_dst))) return TANGO_ERR_INVALID_ARG;
  if (G->chunk_edges < 0) return TANGO_ERR_INVALID_ARG;
  return TANGO_OK;
}
static GraphDev dev_graph(const tango_graph* G) {
  GraphDev g;
  g.n_local = G->row_end - G->row_begin;
  g.n_global = G->n_global;
  g.row_begin = G->row_begin;
  g.e_in = G->e_in;
  g.in_ptr = G->in_ptr; g.in_src = G->in_src;
  g.out_ptr = G->out_ptr; g.out_dst = G->out_dst; g.out_eid = G->out_eid;
  g.chunk = G->chunk_edges > 0 ? G->chunk_edges : 256;
  return g;
}
// Auxiliary stream (per thread and device) for work that does not depend on the main chain (graph
// plans, Q(W), the ∂a reduction): forked from and joined back into the caller's stream with events,
// so the API stays asynchronous on `st` and CUDA-graph capture of `st` records the fork/join.
struct AuxStream {
  cudaStream_t s = nullptr;
  cudaEvent_t ev[10] = {};
  SideStream side(int k) const { return SideStream{s, ev[k], ev[k + 1]}; }
};
// tango_profile_serialize(1): the side-stream work runs in order on the caller's stream, so that
// per-launch event times (tango_profile_*) measure each kernel alone.
static AuxStream* aux_stream(cudaStream_t st) {
  thread_local AuxStream per_dev[16];
  thread_local AuxStream serial[16];
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= 16) return nullptr;
  if (g_serialize.load(std::memory_order_relaxed)) {
    AuxStream& a = serial[d];
    if (!a.ev[0])
      for (auto& e : a.ev)
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
    a.s = st;
    return &a;
  }
  AuxStream& a = per_dev[d];
  if (!a.s) {
    int lo = 0, hi = 0;   // highest priority: the latency-bound hub chain gets SM slots first
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if (cudaStreamCreateWithPriority(&a.s, cudaStreamNonBlocking, hi) != cudaSuccess) { a.s = nullptr; return nullptr; }
    for (auto& e : a.ev)
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
  }
  return &a;
}
// `to` waits for the work enqueued so far on `from` (event slot k)
static cudaError_t stream_after(cudaStream_t to, cudaStream_t from, cudaEvent_t ev) {
  cudaError_t e = cudaEventRecord(ev, from);
  return e == cudaSuccess ? cudaStreamWaitEvent(to, ev, 0) : e;
}

static tango_status check_q(const tango_qtensor* t) {
  if (!t || !t->q || !t->scale) return TANGO_ERR_INVALID_ARG;
  if (t->bits < 2 || t->bits > 8) return TANGO_ERR_BITS;
  if (t->rows < 0 || t->cols < 0 || t->ld < t->cols) return TANGO_ERR_SHAPE;
  return TANGO_OK;
}
static tango_status launch_status(cudaError_t e) {
  if (e != cudaSuccess) {
    fprintf(stderr, "[tango] launch failed: %s\n", cudaGetErrorString(e));
    return TANGO_ERR_CUDA;
  }
  return TANGO_OK;
}

// ------------------------------------------------------------------ loopback group (in-process)
namespace {
struct LocalPtrs { const void* p[16]; };
template <int OP>   // 0: max, 1: sum (rank order)
__global__ void k_local_reduce_f32(float* out, LocalPtrs in, int n, size_t count) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    float v = static_cast<const float*>(in.p[0])[i];
    for (int k = 1; k < n; ++k) {
      const float x = static_cast<const float*>(in.p[k])[i];
      v = OP == 0 ? fmaxf(v, x) : __fadd_rn(v, x);
    }
    out[i] = v;
  }
}
__global__ void k_local_reduce_i64(int64_t* out, LocalPtrs in, int n, size_t count) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    int64_t v = 0;
    for (int k = 0; k < n; ++k) v += static_cast<const int64_t*>(in.p[k])[i];
    out[i] = v;
  }
}
}  // namespace

// Every rank registers its buffer and the event of its producer, then waits for all peers'.
static tango_status local_begin(tango_comm* c, void* buf, cudaStream_t st) {
  tango_local_group* g = c->local;
  const int r = c->rank;
  g->ptr[r] = buf;
  TRY_CUDA(cudaEventRecord(g->ev_a[r], st));
  g->barrier();
  for (int k = 0; k < g->nranks; ++k)
    if (k != r) TRY_CUDA(cudaStreamWaitEvent(st, g->ev_a[k], 0));
  g->barrier();
  return TANGO_OK;
}
// No rank reuses its buffer before every peer has finished reading it.
static tango_status local_end(tango_comm* c, cudaStream_t st) {
  tango_local_group* g = c->local;
  const int r = c->rank;
  TRY_CUDA(cudaEventRecord(g->ev_b[r], st));
  g->barrier();
  for (int k = 0; k < g->nranks; ++k)
    if (k != r) TRY_CUDA(cudaStreamWaitEvent(st, g->ev_b[k], 0));
  g->barrier();
  return TANGO_OK;
}
static tango_status local_reduce(tango_comm* c, void* buf, size_t count, size_t esize, int op, cudaStream_t st) {
  tango_local_group* g = c->local;
  const int r = c->rank;
  if (g->tmp_bytes[r] < count * esize) {
    if (g->tmp[r]) cudaFree(g->tmp[r]);
    TRY_CUDA(cudaMalloc(&g->tmp[r], count * esize));
    g->tmp_bytes[r] = count * esize;
  }
  TRY(local_begin(c, buf, st));
  LocalPtrs lp{};
  for (int k = 0; k < g->nranks; ++k) lp.p[k] = g->ptr[k];
  const int grid = (int)((count + 255) / 256 < 1024 ? (count + 255) / 256 : 1024);
  if (esize == 8) k_local_reduce_i64<<<grid, 256, 0, st>>>(static_cast<int64_t*>(g->tmp[r]), lp, g->nranks, count);
  else if (op == 0) k_local_reduce_f32<0><<<grid, 256, 0, st>>>(static_cast<float*>(g->tmp[r]), lp, g->nranks, count);
  else k_local_reduce_f32<1><<<grid, 256, 0, st>>>(static_cast<float*>(g->tmp[r]), lp, g->nranks, count);
  TRY_CUDA(cudaGetLastError());
  TRY(local_end(c, st));
  TRY_CUDA(cudaMemcpyAsync(buf, g->tmp[r], count * esize, cudaMemcpyDeviceToDevice, st));
  return TANGO_OK;
}

// ------------------------------------------------------------------ collectives (caller stream)
// A one-rank communicator skips its collectives (identities) unless set to `always` (tests / bench
// --nccl-single: the NCCL calls then execute on the device with the same arguments as with N ranks).
static bool comm_skip(const tango_comm* c, size_t count) {
  return !c || count == 0 || (c->nranks == 1 && !(c->always && c->nccl));
}
static tango_status comm_max(tango_comm* c, void* buf, size_t count, cudaStream_t st) {
  if (comm_skip(c, count)) return TANGO_OK;
  if (c->local) return local_reduce(c, buf, count, 4, 0, st);
  TRY_NCCL(ncclAllReduce(buf, buf, count, ncclFloat32, ncclMax, c->nccl, st));
  ++c->nccl_calls;
  return TANGO_OK;
}
static tango_status comm_sum_f32(tango_comm* c, float* buf, size_t count, cudaStream_t st) {
  if (comm_skip(c, count)) return TANGO_OK;
  if (c->local) return local_reduce(c, buf, count, 4, 1, st);
  TRY_NCCL(ncclAllReduce(buf, buf, count, ncclFloat32, ncclSum, c->nccl, st));
  ++c->nccl_calls;
  return TANGO_OK;
}
static tango_status comm_sum_i64(tango_comm* c, int64_t* buf, size_t count, cudaStream_t st) {
  if (comm_skip(c, count)) return TANGO_OK;
  if (c->local) return local_reduce(c, buf, count, 8, 1, st);
  TRY_NCCL(ncclAllReduce(buf, buf, count, ncclInt64, ncclSum, c->nccl, st));
  ++c->nccl_calls;
  return TANGO_OK;
}
// All-gather of node-row blocks of `row_bytes` bytes (rank r owns rows [starts[r], starts[r+1])).  With a
// reserved staging buffer: one padded ncclAllGather (every block padded to max_rows rows; own block
// copied into its staging slot, in-place all-gather, the other blocks copied into place).  Without one:
// grouped in-place broadcasts of the blocks.
static tango_status comm_gather_rows(tango_comm* c, void* base, size_t row_bytes, cudaStream_t st) {
  if (comm_skip(c, 1)) return TANGO_OK;
  if (c->local) {
    TRY(local_begin(c, base, st));
    for (int k = 0; k < c->nranks; ++k) {
      const size_t off = (size_t)c->starts[k] * row_bytes;
      const size_t cnt = (size_t)(c->starts[k + 1] - c->starts[k]) * row_bytes;
      if (k == c->rank || cnt == 0) continue;
      TRY_CUDA(cudaMemcpyAsync(static_cast<char*>(base) + off, static_cast<const char*>(c->local->ptr[k]) + off, cnt,
                               cudaMemcpyDeviceToDevice, st));
    }
    return local_end(c, st);
  }
  if (c->stage && row_bytes <= c->stage_row_bytes && c->max_rows > 0) {
    const size_t slot = (size_t)c->max_rows * row_bytes;
    char* stg = static_cast<char*>(c->stage);
    char* b = static_cast<char*>(base);
    const size_t own = (size_t)(c->starts[c->rank + 1] - c->starts[c->rank]) * row_bytes;
    if (own) TRY_CUDA(cudaMemcpyAsync(stg + c->rank * slot, b + (size_t)c->starts[c->rank] * row_bytes, own,
                                      cudaMemcpyDeviceToDevice, st));
    TRY_NCCL(ncclAllGather(stg + c->rank * slot, stg, slot, ncclInt8, c->nccl, st));
    ++c->nccl_calls;
    for (int r = 0; r < c->nranks; ++r) {
      const size_t cnt = (size_t)(c->starts[r + 1] - c->starts[r]) * row_bytes;
      if (r == c->rank || cnt == 0) continue;
      TRY_CUDA(cudaMemcpyAsync(b + (size_t)c->starts[r] * row_bytes, stg + r * slot, cnt, cudaMemcpyDeviceToDevice, st));
    }
    return TANGO_OK;
  }
  TRY_NCCL(ncclGroupStart());
  for (int r = 0; r < c->nranks; ++r) {
    const size_t off = (size_t)c->starts[r] * row_bytes;
    const size_t cnt = (size_t)(c->starts[r + 1] - c->starts[r]) * row_bytes;
    if (cnt == 0) continue;
    char* p = static_cast<char*>(base) + off;
    TRY_NCCL(ncclBroadcast(p, p, cnt, ncclInt8, r, c->nccl, st));
    ++c->nccl_calls;
  }
  TRY_NCCL(ncclGroupEnd());
  return TANGO_OK;
}
static tango_status check_comm(const tango_graph* G, tango_comm* c) {
  if (!c) return (G->row_begin == 0 && G->row_end == G->n_global) ? TANGO_OK : TANGO_ERR_SHAPE;
  if ((int)c->starts.size() != c->nranks + 1) return TANGO_ERR_INVALID_ARG;
  if (c->starts[c->rank] != G->row_begin || c->starts[c->rank + 1] != G->row_end ||
      c->starts[c->nranks] != G->n_global)
    return TANGO_ERR_SHAPE;
  return TANGO_OK;
}

extern "C" {

// ================================================================== primitives
tango_status tango_quantize(const float* x, int64_t rows, int64_t cols, int64_t global_row0, const float* amax_hint,
                            tango_rng rng, tango_qtensor* out, float* amax_out, int32_t* dev_status,
                            cudaStream_t stream) {
  TRY(check_q(out));
  if (!x && rows * cols > 0) return TANGO_ERR_INVALID_ARG;
  if (out->rows != rows || out->cols != cols || global_row0 < 0) return TANGO_ERR_SHAPE;
  // the amax lives in amax_out if given; otherwise the scale word holds it until the codes are written and
  // is then converted in place (no allocation inside the call)
  float* slot = amax_out ? amax_out : out->scale;
  if (amax_hint) {
    TRY_CUDA(cudaMemcpyAsync(slot, amax_hint, sizeof(float), cudaMemcpyDeviceToDevice, stream));
  } else {
    TRY_CUDA(cudaMemsetAsync(slot, 0, sizeof(float), stream));
    TRY(launch_status(launch_absmax(x, rows, cols, nullptr, reinterpret_cast<unsigned*>(slot), stream)));
  }
  TRY(launch_status(launch_quantize(x, rows, cols, nullptr, global_row0 * cols, reinterpret_cast<unsigned*>(slot),
                                    out->bits, rng.seed, rng.step, rng.tag, out->q, out->ld, nullptr, 0,
                                    amax_out ? out->scale : nullptr, dev_status, stream)));
  if (!amax_out) TRY(launch_status(launch_amax_to_scale(out->scale, out->bits, stream)));
  return TANGO_OK;
}

tango_status tango_gemm_q(const tango_qtensor* A, int32_t a_layout, const tango_qtensor* B, int32_t b_layout,
                          int64_t M, int64_t N, int64_t K, float* C, int32_t* C_i32, int64_t* C_i64,
                          cudaStream_t stream) {
  TRY(check_q(A));
  TRY(check_q(B));
  if ((a_layout != TANGO_K_MAJOR && a_layout != TANGO_MN_MAJOR) ||
      (b_layout != TANGO_K_MAJOR && b_layout != TANGO_MN_MAJOR))
    return TANGO_ERR_INVALID_ARG;
  if (!C && !C_i32 && !C_i64) return TANGO_ERR_INVALID_ARG;
  if (M < 0 || N < 0 || K < 0) return TANGO_ERR_SHAPE;
  const bool amn = a_layout == TANGO_MN_MAJOR, bmn = b_layout == TANGO_MN_MAJOR;
  // logical extents vs stored tensors
  if (amn ? (A->rows != K || A->cols != M) : (A->rows != M || A->cols != K)) return TANGO_ERR_SHAPE;
  if (bmn ? (B->rows != K || B->cols != N) : (B->rows != N || B->cols != K)) return TANGO_ERR_SHAPE;
  if ((A->ld % 16) || (B->ld % 16)) return TANGO_ERR_SHAPE;
  const bool small_k = K <= 133144;
  if (C_i32 && !small_k) return TANGO_ERR_OVERFLOW;
  if (C && !small_k && !C_i64) return TANGO_ERR_OVERFLOW;
  if (M == 0 || N == 0) return TANGO_OK;
  GemmArgs g{};
  g.A = A->q; g.lda = A->ld; g.a_mn = amn;
  g.B = B->q; g.ldb = B->ld; g.b_mn = bmn;
  g.M = M; g.N = N; g.K = K; g.splits = 1;
  g.sA = A->scale; g.sB = B->scale;
  if (C_i32) {
    g.mode = EPI_I32; g.C = C_i32; g.ldc = N;
    TRY(launch_status(launch_gemm(g, stream)));
  }
  if (C_i64) {
    TRY_CUDA(cudaMemsetAsync(C_i64, 0, sizeof(int64_t) * M * N, stream));
    g.mode = EPI_ATOMIC64; g.C = C_i64; g.ldc = N;
    const int64_t tiles = ((M + 127) / 128) * ((N + 255) / 256);
    const int64_t kb = (K + 127) / 128;
    int64_t splits = (2 * num_sms() + tiles - 1) / tiles;
    const int64_t min_splits = (K + 131071) / 131072;   // int32-safe chunks (reading R27)
    if (splits < min_splits) splits = min_splits;
    if (splits > kb) splits = kb > 0 ? kb : 1;
    g.splits = (int)splits;
    TRY(launch_status(launch_gemm(g, stream)));
    g.splits = 1;
  }
  if (C) {
    if (small_k) {
      g.mode = EPI_STORE; g.C = C; g.ldc = N;
      TRY(launch_status(launch_gemm(g, stream)));
    } else {
      TRY(launch_status(launch_finalize_dw(C_i64, M * N, A->scale, B->scale, C, stream)));
    }
  }
  return TANGO_OK;
}

tango_status tango_sddmm_q(const tango_graph* G, int32_t op, const tango_qtensor* Xsrc, const tango_qtensor* Xdst,
                           int32_t heads, float slope, float* out0, float* out1, int32_t* acc_i32,
                           cudaStream_t stream) {
  TRY(check_graph(G, false));
  TRY(check_q(Xsrc));
  TRY(check_q(Xdst));
  if (heads <= 0) return TANGO_ERR_SHAPE;
  const GraphDev g = dev_graph(G);
  if (Xsrc->rows != G->n_global || Xdst->rows < G->row_end) return TANGO_ERR_SHAPE;
  // the warp-per-edge-run kernels of tango_sddmm_qn (int4.cu, bits = 8) compute the same values; the
  // thread-per-(row, head) kernels remain for the shapes they do not take and for the acc_i32 test hook
  if (op == TANGO_SDDMM_ADD) {
    if (Xsrc->cols != heads || Xdst->cols != heads || Xsrc->ld != heads || Xdst->ld != heads) return TANGO_ERR_SHAPE;
    if (!out0 && !out1) return TANGO_ERR_INVALID_ARG;
    if (out0 && Xsrc->bits == 8 && Xdst->bits == 8) {
      const tango_status st = tango_sddmm_qn(G, op, 8, Xsrc->q, Xsrc->ld, Xsrc->scale, Xdst->q, Xdst->ld, Xdst->scale,
                                             heads, heads, slope, out0, out1, stream);
      if (st != TANGO_ERR_UNSUPPORTED) return st;
    }
    return launch_status(launch_sddmm_add(g, heads, Xsrc->q, Xsrc->scale, Xdst->q, Xdst->scale, slope, out0, out1,
                                          stream));
  }
  if (op == TANGO_SDDMM_DOT) {
    if (Xsrc->cols != Xdst->cols || Xsrc->cols % heads) return TANGO_ERR_SHAPE;
    if (!out0 && !acc_i32) return TANGO_ERR_INVALID_ARG;
    if (out0 && !acc_i32) {
      const tango_status st = tango_sddmm_qn(G, op, 8, Xsrc->q, Xsrc->ld, Xsrc->scale, Xdst->q, Xdst->ld, Xdst->scale,
                                             heads, (int32_t)Xsrc->cols, slope, out0, nullptr, stream);
      if (st != TANGO_ERR_UNSUPPORTED) return st;
    }
    return launch_status(launch_sddmm_dot(g, heads, (int)Xsrc->cols, Xdst->q, Xdst->ld, Xdst->scale, Xsrc->q,
                                          Xsrc->ld, Xsrc->scale, out0, acc_i32, stream));
  }
  return TANGO_ERR_INVALID_ARG;
}

tango_status tango_edge_softmax(const tango_graph* G, int32_t heads, const float* el, float* m, float* den,
                                float* alpha, cudaStream_t stream) {
  TRY(check_graph(G, false));
  if (heads <= 0) return TANGO_ERR_SHAPE;
  if (!alpha || (!el && G->e_in > 0)) return TANGO_ERR_INVALID_ARG;
  return launch_status(launch_edge_softmax(dev_graph(G), heads, el, m, den, alpha, stream));
}

tango_status tango_softmax_bwd(const tango_graph* G, int32_t heads, const float* alpha, const float* dalpha,
                               const float* e_pre, float slope, float* P, float* dE_pre, cudaStream_t stream) {
  TRY(check_graph(G, false));
  if (heads <= 0) return TANGO_ERR_SHAPE;
  if (G->e_in > 0 && (!alpha || !dalpha || !e_pre || !dE_pre)) return TANGO_ERR_INVALID_ARG;
  return launch_status(launch_softmax_bwd(dev_graph(G), heads, alpha, dalpha, e_pre, slope, P, dE_pre, stream));
}

tango_status tango_spmm_q(const tango_graph* G, int32_t dir, const float* edge_w, const tango_qtensor* X,
                          int32_t heads, const float* row_scale, float* out, int32_t* out_i32, float* amax_out,
                          cudaStream_t stream) {
  TRY(check_graph(G, dir == TANGO_OUT));
  TRY(check_q(X));
  if (dir != TANGO_IN && dir != TANGO_OUT) return TANGO_ERR_INVALID_ARG;
  if (heads <= 0 || X->cols % heads || X->rows != G->n_global) return TANGO_ERR_SHAPE;
  if ((row_scale || amax_out) && !out) return TANGO_ERR_INVALID_ARG;
  const GraphDev g = dev_graph(G);
  unsigned* amax = reinterpret_cast<unsigned*>(amax_out);
  if (edge_w) {
    if (!out) return TANGO_ERR_INVALID_ARG;
    if (dir == TANGO_OUT && G->e_out > 0 && !G->out_eid) return TANGO_ERR_INVALID_ARG;
    return launch_status(launch_spmm_w(g, dir, heads, (int)X->cols, edge_w, X->q, X->ld, X->scale, row_scale, out,
                                       amax, dir == TANGO_OUT ? G->e_out : G->e_in, stream));
  }
  if (!out && !out_i32) return TANGO_ERR_INVALID_ARG;
  return launch_status(
      launch_spmm_sum(g, dir, (int)X->cols, X->q, X->ld, X->scale, row_scale, out, out_i32, amax, stream));
}

tango_status tango_spmm_q8(const tango_graph* G, int32_t dir, const tango_qtensor* Aq, const tango_qtensor* X,
                           int32_t heads, int32_t* out_i32, float* out, cudaStream_t stream) {
  TRY(check_graph(G, dir == TANGO_OUT));
  TRY(check_q(Aq));
  TRY(check_q(X));
  if (dir != TANGO_IN && dir != TANGO_OUT) return TANGO_ERR_INVALID_ARG;
  if (!out_i32) return TANGO_ERR_INVALID_ARG;
  if (dir == TANGO_OUT && G->e_out > 0 && !G->out_eid) return TANGO_ERR_INVALID_ARG;
  if (heads <= 0 || X->cols % heads || X->rows != G->n_global) return TANGO_ERR_SHAPE;
  if (Aq->cols != heads || Aq->ld != heads || Aq->rows != G->e_in) return TANGO_ERR_SHAPE;
  const int64_t D = X->cols / heads;
  if (D % 4 || X->ld % 4 || (reinterpret_cast<uintptr_t>(X->q) & 3) || (reinterpret_cast<uintptr_t>(out_i32) & 15))
    return TANGO_ERR_UNSUPPORTED;
  return launch_status(launch_spmm_q8(dev_graph(G), dir, heads, (int)X->cols, Aq->q, Aq->scale, X->q, X->ld,
                                      X->scale, out_i32, out, dir == TANGO_OUT ? G->e_out : G->e_in, stream));
}

tango_status tango_edge_sum(const tango_graph* G, int32_t dir, int32_t heads, const float* x, float* out,
                            cudaStream_t stream) {
  TRY(check_graph(G, dir == TANGO_OUT));
  if (dir != TANGO_IN && dir != TANGO_OUT) return TANGO_ERR_INVALID_ARG;
  if (dir == TANGO_OUT && G->e_out > 0 && !G->out_eid) return TANGO_ERR_INVALID_ARG;
  if (heads <= 0) return TANGO_ERR_SHAPE;
  if (!out) return TANGO_ERR_INVALID_ARG;
  return launch_status(launch_edge_sum(dev_graph(G), dir, heads, x, out, dir == TANGO_OUT ? G->e_out : G->e_in, stream));
}

}  // extern "C"

// ================================================================== GAT ctx layout
namespace {
struct GatLayout {
  int64_t n, N, E, Eo, F, H, Dh, HD, ldF, ldHD, ldFt, cap_in, cap_out;
  size_t off_scal, off_qH, off_qW, off_qWt, off_qHp, off_S, off_D, off_qS, off_qD, off_m, off_den, off_P, off_dD,
      off_qG, off_dal, off_dHp, off_qdHp, off_dW64, total;
  // segment plans (gat.cu) and heavy-segment scratch
  size_t off_pin_hbase, off_pin_hseg, off_pin_hrow, off_pin_cnt, off_pout_hbase, off_pout_hseg, off_pout_hrow,
      off_pout_cnt, off_h1, off_h2, off_hdS, off_hagg, off_work, off_dS, off_alpha, off_pin_tiles, off_pout_tiles;
  size_t off_hcnt, off_dapart;   // v6 dataflow: finished-segment counters [n], ∂a chunk partials
  size_t off_nrec;               // packed per-node record [N][nrs] (the v6 in-CSR -> out-CSR map reuses off_dal)
  size_t off_ast;                // v6: α stored by F-agg for P2 [E][H] (sign = LeakyReLU branch)
  int64_t tcap;
};
GatLayout gat_layout(const tango_graph* G, const tango_gat_params* p) {
  GatLayout L{};
  L.n = G->row_end - G->row_begin;
  L.N = G->n_global;
  L.E = G->e_in;
  L.F = p->in_feats; L.H = p->heads; L.Dh = p->head_dim; L.HD = L.H * L.Dh;
  L.ldF = round_up(L.F, 32);
  L.ldHD = round_up(L.HD, 32);
  L.ldFt = L.ldF;
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t at = o; o = align256(o + bytes); return at; };
  L.off_scal = take(SL_NSLOTS * 4);
  L.off_qH = take((size_t)L.n * L.ldF);
  L.off_qW = take((size_t)L.F * L.ldHD);
  L.off_qWt = take((size_t)L.HD * L.ldFt);
  L.off_qHp = take((size_t)L.N * L.ldHD);
  L.off_S = take((size_t)L.n * L.H * 4);
  L.off_D = take((size_t)L.n * L.H * 4);
  L.off_qS = take((size_t)L.N * L.H);
  L.off_qD = take((size_t)L.N * L.H);
  L.off_m = take((size_t)L.N * L.H * 4);
  L.off_den = take((size_t)L.N * L.H * 4);
  L.off_P = take((size_t)L.N * L.H * 4);
  L.off_dD = take((size_t)L.N * L.H * 4);
  L.off_qG = take((size_t)L.N * L.ldHD);
  L.off_dal = take((size_t)L.E * L.H * 4);
  L.off_dHp = take((size_t)L.n * L.HD * 4);
  L.off_qdHp = take((size_t)L.n * L.ldHD);
  L.off_dW64 = take((size_t)L.F * L.HD * 8);
  const int64_t C = G->chunk_edges > 0 ? G->chunk_edges : 256;
  L.Eo = G->e_out;
  L.cap_in = 2 * L.E / C + 1;
  L.cap_out = 2 * L.Eo / C + 1;
  L.off_pin_hbase = take((size_t)L.n * 4);
  L.off_pin_hseg = take((size_t)L.cap_in * 4);
  L.off_pin_hrow = take((size_t)L.n * 4);
  L.off_pin_cnt = take(16);
  L.off_pout_hbase = take((size_t)L.n * 4);
  L.off_pout_hseg = take((size_t)L.cap_out * 4);
  L.off_pout_hrow = take((size_t)L.n * 4);
  L.off_pout_cnt = take(16);
  L.off_h1 = take((size_t)L.cap_in * L.H * 4);     // fwd: hmax   bwd: hP
  L.off_h2 = take((size_t)L.cap_in * L.H * 4);     // fwd: hden   bwd: hdD
  L.off_hdS = take((size_t)L.cap_out * L.H * 4);
  L.off_hagg = take((size_t)(L.cap_in > L.cap_out ? L.cap_in : L.cap_out) * L.HD * 4);
  L.off_work = take(64);
  L.off_dS = take((size_t)L.N * L.H * 4);
  L.off_alpha = take((size_t)L.E * L.H * 8);     // [E][2H]: α | ∂E_pre
  L.tcap = L.n + L.n / 32 + 1;
  L.off_pin_tiles = take((size_t)L.tcap * 4);
  L.off_pout_tiles = take((size_t)L.tcap * 4);
  L.off_hcnt = take((size_t)L.n * 4);
  L.off_dapart = take((size_t)((L.n + 1023) / 1024 + 1) * 2 * L.HD * 4);
  L.off_nrec = take((size_t)L.N * gat2_nrec_stride((int)L.H) * 4);
  L.off_ast = take((size_t)L.E * L.H * 8);     // v6: F-agg's α [E][H], or P1's records [E][2H]
  L.total = o;
  return L;
}
PlanDev plan_of(char* c, size_t hb, size_t hs, size_t hr, size_t cn, int64_t cap, size_t tl, int64_t tcap) {
  PlanDev p;
  p.hbase = (int32_t*)(c + hb); p.hseg_row = (int32_t*)(c + hs); p.hrow = (int32_t*)(c + hr);
  p.counts = (int32_t*)(c + cn); p.cap = cap;
  p.tiles = (int32_t*)(c + tl); p.tcap = tcap;
  return p;
}
// Static-graph plan cache: the segment plans (k_plan / k_plan_tiles of the in- and out-CSR) and the v6
// in-CSR -> out-CSR map depend only on the graph, so a ctx keeps them across calls.  Keyed on the ctx,
// the caller's graph_id (0 disables the cache) and the graph's device arrays and sizes.
struct PlanKey {
  const void* ctx; const int64_t* in_ptr; const int64_t* out_ptr; const int32_t* out_eid;
  int64_t n, row_begin, e_in, e_out; int32_t chunk; uint64_t id;
  bool operator==(const PlanKey& o) const {
    return ctx == o.ctx && in_ptr == o.in_ptr && out_ptr == o.out_ptr && out_eid == o.out_eid && n == o.n &&
           row_begin == o.row_begin && e_in == o.e_in && e_out == o.e_out && chunk == o.chunk && id == o.id;
  }
};
struct PlanState { PlanKey key; bool in_done, out_done; };
std::mutex g_plan_mu;
std::vector<PlanState> g_plans;
PlanKey plan_key(const void* ctx, const tango_graph* G) {
  return PlanKey{ctx, G->in_ptr, G->out_ptr, G->out_eid, G->row_end - G->row_begin, G->row_begin, G->e_in, G->e_out,
                 G->chunk_edges, G->graph_id};
}
// returns true if the plan `which` (0 = in-CSR, 1 = out-CSR) of this ctx/graph still has to be built, and
// records it as built (the caller enqueues the build on the stream before any use)
bool plan_needed(const void* ctx, const tango_graph* G, int which) {
  if (G->graph_id == 0) return true;
  const PlanKey k = plan_key(ctx, G);
  std::lock_guard<std::mutex> lk(g_plan_mu);
  for (auto& p : g_plans)
    if (p.key.ctx == ctx) {
      if (!(p.key == k)) { p.key = k; p.in_done = p.out_done = false; }
      bool& done = which ? p.out_done : p.in_done;
      const bool need = !done;
      done = true;
      return need;
    }
  g_plans.push_back(PlanState{k, which == 0, which == 1});
  return true;
}

// v6 dataflow (gat2.cu) for single-GPU graphs with the edge-id map; TANGO_DATAFLOW=1 / 2 force the
// round-1 kernels (gat.cu) / v6 for A/B measurements.
bool use_gat2(const GraphDev& g, const tango_gat_params* p, tango_comm* comm) {
  static const int forced = [] {
    const char* e = getenv("TANGO_DATAFLOW");
    return e ? atoi(e) : 0;
  }();
  if (forced == 1 || comm) return false;
  const int HD = p->heads * p->head_dim;
  if (!(gat_codes_biased(p->heads, HD) && gat2_supported(g, p->heads, HD))) return false;
  if (forced == 2) return true;
  // v6 removes a whole row-gather pass but adds two edge-streaming passes: it pays off on dense graphs
  // (mean in-degree >= TANGO_V6_MIN_DEGREE, default 32: Reddit-shaped 489); sparse graphs (arxiv-shaped
  // 13) keep the round-1 kernels
  static const double min_deg = [] {
    const char* e = getenv("TANGO_V6_MIN_DEGREE");
    return e ? atof(e) : 32.0;
  }();
  return g.n_local > 0 && (double)g.e_in >= min_deg * (double)g.n_local;
}
G2Args g2_args(const GatLayout& L, char* c, const GraphDev& g, const tango_gat_params* p) {
  G2Args a{};
  unsigned* sc = reinterpret_cast<unsigned*>(c + L.off_scal);
  a.g = g; a.d = {p->heads, p->head_dim, (int)L.HD}; a.slope = p->neg_slope; a.bits = p->bits;
  a.qS = (int8_t*)(c + L.off_qS); a.amax_S = sc + SL_AMAX_S;
  a.qD = (int8_t*)(c + L.off_qD); a.amax_D = sc + SL_AMAX_D;
  a.qHp = (int8_t*)(c + L.off_qHp); a.ldHp = L.ldHD; a.amax_Hp = sc + SL_AMAX_HP;
  a.qG = (int8_t*)(c + L.off_qG); a.ldG = L.ldHD; a.amax_G = sc + SL_AMAX_G;
  a.m = (float*)(c + L.off_m); a.den = (float*)(c + L.off_den);
  a.P = (float*)(c + L.off_P); a.dD = (float*)(c + L.off_dD); a.dS = (float*)(c + L.off_dS);
  a.dal_out = (float*)(c + L.off_alpha);
  a.dal_in = (float*)(c + L.off_alpha) + L.E * L.H;
  a.a_src = p->a_src; a.a_dst = p->a_dst;
  a.dHp = (float*)(c + L.off_dHp); a.amax_dHp = sc + SL_AMAX_DHP;
  a.pin = plan_of(c, L.off_pin_hbase, L.off_pin_hseg, L.off_pin_hrow, L.off_pin_cnt, L.cap_in, L.off_pin_tiles, L.tcap);
  a.pout = plan_of(c, L.off_pout_hbase, L.off_pout_hseg, L.off_pout_hrow, L.off_pout_cnt, L.cap_out, L.off_pout_tiles,
                   L.tcap);
  a.hagg = (float*)(c + L.off_hagg);
  a.h1 = (float*)(c + L.off_h1); a.h2 = (float*)(c + L.off_h2); a.hs = (float*)(c + L.off_hdS);
  a.hcnt = (int32_t*)(c + L.off_hcnt);
  a.work = (int32_t*)(c + L.off_work);
  a.da_part = (float*)(c + L.off_dapart);
  a.nrec = (float*)(c + L.off_nrec); a.nrs = gat2_nrec_stride(p->heads);
  a.in2out = (const int32_t*)(c + L.off_dal);
  // P2's ∂α in in-CSR order: gathered by P2 through the in2out map (default) or scattered there by P1
  // (TANGO_P2_SCATTER=1: P2 reads coalesced, P1 pays the random 16-B stores — measured a wash on Reddit,
  // profiles/r2x_*); hub segments of F-stats / P2 / P3: staged warp sums (default) or lane-parallel chunk
  // sums (TANGO_HUB_LANE=1: latency-bound, no faster) — both variants stay parity-tested
  static const int scatter = [] {
    const char* e = getenv("TANGO_P2_SCATTER");
    return (e && atoi(e)) ? 1 : 0;
  }();
  a.scatter_in = scatter;
  static const int lane = [] {
    const char* e = getenv("TANGO_HUB_LANE");
    return e ? atoi(e) : 0;
  }();
  static const int lane_p2 = [] {   // per-pass override for P2 (TANGO_HUB_P2)
    const char* e = getenv("TANGO_HUB_P2");
    return e ? atoi(e) : -1;
  }();
  a.hub_fs = lane;   // 0: staged warp sums, 1: lane-pipelined, 2: multi-segment staged
  a.hub_p2 = lane_p2 >= 0 ? lane_p2 : lane;
  static const int lane_p3 = [] {   // per-pass override for P3 (TANGO_HUB_P3)
    const char* e = getenv("TANGO_HUB_P3");
    return e ? atoi(e) : -1;
  }();
  a.hub_p3 = lane_p3 >= 0 ? lane_p3 : lane;
  // α stored by F-agg and read by P2 (default), or recomputed by P2 (TANGO_ALPHA_RECOMPUTE=1)
  static const int recompute = [] {
    const char* e = getenv("TANGO_ALPHA_RECOMPUTE");
    return (e && atoi(e)) ? 1 : 0;
  }();
  a.alpha_st = recompute ? nullptr : (float*)(c + L.off_ast);
  // P1 writes a full-sector record {∂α, signed α} per edge at its in-CSR slot and P2 reads it coalesced
  // (default for H = 4 / 8: 2H floats = whole 32-B sectors; TANGO_P2_REC=0 keeps the gather of ∂α)
  static const int use_rec = [] {
    const char* e = getenv("TANGO_P2_REC");
    return e ? atoi(e) : 1;
  }();
  a.rec = nullptr;
  a.al_out = nullptr;
  if (use_rec && (p->heads == 4 || p->heads == 8) && !a.scatter_in) {
    a.rec = (float*)(c + L.off_ast);
    a.alpha_st = nullptr;
    a.al_out = a.dal_in;   // P1 also leaves its signed α in out-CSR order for P3 (dal_in is unused here)
    // P2 reading coalesced records: the multi-segment staged hub sums are the faster form (profiles/r3e_*)
    if (lane_p2 < 0 && lane == 0) a.hub_p2 = 2;
  }
  a.codes_biased = 1;
  return a;
}
tango_status check_gat(const tango_graph* G, const tango_gat_params* p) {
  TRY(check_graph(G, true));
  if (!p || !p->W || !p->a_src || !p->a_dst) return TANGO_ERR_INVALID_ARG;
  if (p->bits < 2 || p->bits > 8) return TANGO_ERR_BITS;
  if (p->in_feats <= 0 || p->heads <= 0 || p->head_dim <= 0) return TANGO_ERR_SHAPE;
  const int HD = p->heads * p->head_dim;
  if (HD % 32 || HD < 64 || HD > 512) return TANGO_ERR_UNSUPPORTED;
  const int vpl = HD / 32;
  if (!(vpl == 2 || vpl == 4 || vpl == 8 || vpl == 16)) return TANGO_ERR_UNSUPPORTED;
  if (!(p->heads == 1 || p->heads == 2 || p->heads == 4 || p->heads == 8)) return TANGO_ERR_UNSUPPORTED;
  if (!(p->head_dim == 8 || p->head_dim == 16 || p->head_dim % 32 == 0)) return TANGO_ERR_UNSUPPORTED;
  if (p->in_feats > 133144) return TANGO_ERR_OVERFLOW;
  if (256 % p->head_dim && HD > 256) return TANGO_ERR_UNSUPPORTED;
  // gathered rows are addressed by 32-bit byte offsets (row * ld) inside the gather kernels
  if ((uint64_t)G->n_global * (uint64_t)HD >= (1ull << 32)) return TANGO_ERR_UNSUPPORTED;
  return TANGO_OK;
}
}  // namespace

extern "C" {

size_t tango_gat_ctx_bytes(const tango_graph* G, const tango_gat_params* p) {
  if (check_gat(G, p) != TANGO_OK) return 0;
  return gat_layout(G, p).total;
}

tango_status tango_gat_ctx_get_view(const tango_graph* G, const tango_gat_params* p, void* ctx,
                                    tango_gat_ctx_view* v) {
  TRY(check_gat(G, p));
  if (!ctx || !v) return TANGO_ERR_INVALID_ARG;
  const GatLayout L = gat_layout(G, p);
  char* c = static_cast<char*>(ctx);
  v->qH = (int8_t*)(c + L.off_qH); v->qW = (int8_t*)(c + L.off_qW); v->qWt = (int8_t*)(c + L.off_qWt);
  v->qHp = (int8_t*)(c + L.off_qHp); v->qS = (int8_t*)(c + L.off_qS); v->qD = (int8_t*)(c + L.off_qD);
  v->qG = (int8_t*)(c + L.off_qG); v->qdHp = (int8_t*)(c + L.off_qdHp);
  v->ldF = L.ldF; v->ldHD = L.ldHD; v->ldFt = L.ldFt;
  v->S = (float*)(c + L.off_S); v->D = (float*)(c + L.off_D); v->m = (float*)(c + L.off_m);
  v->den = (float*)(c + L.off_den); v->P = (float*)(c + L.off_P); v->dD = (float*)(c + L.off_dD);
  v->dHp = (float*)(c + L.off_dHp); v->dalpha = (float*)(c + L.off_dal);
  v->alpha_pack = (float*)(c + L.off_alpha);
  v->dS = (float*)(c + L.off_dS);
  v->dataflow = use_gat2(dev_graph(G), p, nullptr) ? 2 : 1;
  v->scalars = (float*)(c + L.off_scal);
  v->codes_biased = gat_codes_biased(p->heads, (int)L.HD) ? 1 : 0;
  return TANGO_OK;
}

tango_status tango_gat_layer_fwd(const tango_graph* G, const tango_gat_params* p, const float* H,
                                 const float* amax_H_hint, tango_rng rng, uint32_t layer_id, void* ctx,
                                 size_t ctx_bytes, float* H_out, float* amax_out, tango_comm* comm,
                                 int32_t* dev_status, cudaStream_t st) {
  TRY(check_gat(G, p));
  TRY(check_comm(G, comm));
  const GatLayout L = gat_layout(G, p);
  if (!ctx || ctx_bytes < L.total) return TANGO_ERR_INVALID_ARG;
  if ((L.n > 0 && (!H || !H_out))) return TANGO_ERR_INVALID_ARG;
  char* c = static_cast<char*>(ctx);
  unsigned* sc = reinterpret_cast<unsigned*>(c + L.off_scal);
  float* scf = reinterpret_cast<float*>(sc);
  int8_t* qH = (int8_t*)(c + L.off_qH);
  int8_t* qW = (int8_t*)(c + L.off_qW);
  int8_t* qWt = (int8_t*)(c + L.off_qWt);
  int8_t* qHp = (int8_t*)(c + L.off_qHp);
  float* S = (float*)(c + L.off_S);
  float* D = (float*)(c + L.off_D);
  int8_t* qS = (int8_t*)(c + L.off_qS);
  int8_t* qD = (int8_t*)(c + L.off_qD);
  float* m = (float*)(c + L.off_m);
  float* den = (float*)(c + L.off_den);
  const int64_t r0 = G->row_begin;
  const GraphDev g = dev_graph(G);

  TRY_CUDA(cudaMemsetAsync(sc, 0, SL_NSLOTS * 4, st));
  // side stream: F2 Q(W) and the in-CSR segment plan (graph only) run beside F1
  AuxStream* aux = aux_stream(st);
  if (!aux) return TANGO_ERR_CUDA;
  const PlanDev pin = plan_of(c, L.off_pin_hbase, L.off_pin_hseg, L.off_pin_hrow, L.off_pin_cnt, L.cap_in, L.off_pin_tiles, L.tcap);
  TRY_CUDA(stream_after(aux->s, st, aux->ev[0]));
  // F2: Q(W) (replicated; identical on every rank), row-major and transposed copies
  TRY(launch_status(launch_absmax(p->W, L.F, L.HD, nullptr, sc + SL_AMAX_W, aux->s)));
  TRY(launch_status(launch_quantize(p->W, L.F, L.HD, nullptr, 0, sc + SL_AMAX_W, p->bits, rng.seed, rng.step,
                                    tag_of(layer_id, R_W), qW, L.ldHD, qWt, L.ldFt, scf + SL_S_W, dev_status, aux->s)));
  TRY_CUDA(cudaEventRecord(aux->ev[1], aux->s));
  if (plan_needed(ctx, G, 0)) {
    TRY_CUDA(cudaMemsetAsync(pin.counts, 0, 16, aux->s));
    TRY(launch_status(launch_plan(G->in_ptr, L.n, g.chunk, pin, aux->s)));
    TRY(launch_status(launch_plan_tiles(G->in_ptr, L.n, pin, aux->s)));
  }
  TRY_CUDA(cudaEventRecord(aux->ev[2], aux->s));
  // F1: amax(H) over all ranks (R28), Q(H)
  if (amax_H_hint) {
    TRY_CUDA(cudaMemcpyAsync(sc + SL_AMAX_H, amax_H_hint, 4, cudaMemcpyDeviceToDevice, st));
  } else {
    TRY(launch_status(launch_absmax(H, L.n, L.F, nullptr, sc + SL_AMAX_H, st)));
    TRY(comm_max(comm, sc + SL_AMAX_H, 1, st));
  }
  TRY(launch_status(launch_quantize(H, L.n, L.F, nullptr, r0 * L.F, sc + SL_AMAX_H, p->bits, rng.seed, rng.step,
                                    tag_of(layer_id, R_H), qH, L.ldF, nullptr, 0, scf + SL_S_H, dev_status, st)));
  TRY_CUDA(cudaStreamWaitEvent(st, aux->ev[1], 0));   // Q(W) done
  // F3 phase A: acc = q_H·q_W on tcgen05; H′ = i2f(acc)·s_H s_W; S, D head dots; amax(H′), amax(S), amax(D)
  GemmArgs ga{};
  ga.A = qH; ga.lda = L.ldF; ga.a_mn = false;
  ga.B = qWt; ga.ldb = L.ldFt; ga.b_mn = false;
  ga.M = L.n; ga.N = L.HD; ga.K = L.F; ga.splits = 1;
  ga.sA = scf + SL_S_H; ga.sB = scf + SL_S_W;
  ga.mode = EPI_AMAX;
  ga.amax_slot = sc + SL_AMAX_HP;
  ga.a_src = p->a_src; ga.a_dst = p->a_dst; ga.head_dim = p->head_dim; ga.heads = p->heads;
  ga.S = S; ga.Dd = D; ga.amax_S = sc + SL_AMAX_S; ga.amax_D = sc + SL_AMAX_D;
  TRY(launch_status(launch_gemm(ga, st)));
  TRY(comm_max(comm, sc + SL_AMAX_HP, 3, st));
  // F4: phase B recomputes the MMA and emits q_H′ with Philox SR in the epilogue; then Q(S), Q(D)
  GemmArgs gb = ga;
  gb.mode = EPI_QUANT;
  gb.a_src = nullptr; gb.a_dst = nullptr;
  gb.amax_in = sc + SL_AMAX_HP; gb.bits = p->bits; gb.seed = rng.seed; gb.step = rng.step;
  gb.tag = tag_of(layer_id, R_HP); gb.g_row0 = r0;
  gb.q_out = qHp + r0 * L.ldHD; gb.ldq = L.ldHD; gb.scale_out = scf + SL_S_HP; gb.status = dev_status;
  const bool biased = gat_codes_biased(p->heads, (int)L.HD);   // q_H′ / q_G as excess-128 codes
  gb.code_xor = biased ? 0x80808080u : 0u;
  // Q(S), Q(D) (tiny, latency-bound) on the side stream beside phase B
  TRY_CUDA(stream_after(aux->s, st, aux->ev[3]));
  TRY(launch_status(launch_quantize(S, L.n, L.H, nullptr, r0 * L.H, sc + SL_AMAX_S, p->bits, rng.seed, rng.step,
                                    tag_of(layer_id, R_S), qS + r0 * L.H, L.H, nullptr, 0, scf + SL_S_S, dev_status,
                                    aux->s)));
  TRY(launch_status(launch_quantize(D, L.n, L.H, nullptr, r0 * L.H, sc + SL_AMAX_D, p->bits, rng.seed, rng.step,
                                    tag_of(layer_id, R_D), qD + r0 * L.H, L.H, nullptr, 0, scf + SL_S_D, dev_status,
                                    aux->s)));
  TRY_CUDA(cudaEventRecord(aux->ev[6], aux->s));
  TRY(launch_status(launch_gemm(gb, st)));
  TRY(comm_gather_rows(comm, qHp, (size_t)L.ldHD, st));
  TRY_CUDA(cudaStreamWaitEvent(st, aux->ev[6], 0));   // Q(S), Q(D) done
  TRY(comm_gather_rows(comm, qS, (size_t)L.H, st));
  TRY(comm_gather_rows(comm, qD, (size_t)L.H, st));
  // F5 + F6: segment plan of the in-CSR, then softmax statistics, aggregation and heavy-row combine
  if (amax_out) TRY_CUDA(cudaMemsetAsync(amax_out, 0, 4, st));
  TRY_CUDA(cudaStreamWaitEvent(st, aux->ev[2], 0));   // in-CSR plan done
  GatFwdArgs fa{};
  fa.g = g; fa.d = {p->heads, p->head_dim, (int)L.HD}; fa.slope = p->neg_slope; fa.bits = p->bits;
  fa.qS = qS; fa.amax_S = sc + SL_AMAX_S; fa.qD = qD; fa.amax_D = sc + SL_AMAX_D;
  fa.qHp = qHp; fa.ldHp = L.ldHD; fa.amax_Hp = sc + SL_AMAX_HP;
  fa.Hout = H_out; fa.m = m; fa.den = den; fa.amax_out = reinterpret_cast<unsigned*>(amax_out);
  fa.plan = pin; fa.hmax = (float*)(c + L.off_h1); fa.hden = (float*)(c + L.off_h2); fa.hagg = (float*)(c + L.off_hagg);
  fa.work = (int32_t*)(c + L.off_work);
  fa.alpha = (float*)(c + L.off_alpha);
  fa.codes_biased = biased;
  TRY_CUDA(cudaMemsetAsync(fa.work, 0, 64, st));
  if (use_gat2(g, p, comm)) {
    G2Args a2 = g2_args(L, c, g, p);
    a2.Hout = H_out; a2.amax_out = reinterpret_cast<unsigned*>(amax_out);
    TRY_CUDA(cudaMemsetAsync(a2.hcnt, 0, (size_t)L.n * 4, st));
    TRY_CUDA(cudaMemsetAsync(a2.nrec, 0, (size_t)L.N * a2.nrs * 4, st));   // m keys of hub rows start below all
    const SideStream side = aux->side(4);
    TRY(launch_status(launch_gat2_fwd(a2, st, &side)));
  } else {
    const SideStream side = aux->side(4);
    TRY(launch_status(launch_gat_fwd(fa, st, &side)));
  }
  TRY(comm_max(comm, amax_out, amax_out ? 1 : 0, st));
  TRY(comm_gather_rows(comm, m, (size_t)L.H * 4, st));
  TRY(comm_gather_rows(comm, den, (size_t)L.H * 4, st));
  return TANGO_OK;
}

tango_status tango_gat_layer_bwd(const tango_graph* G, const tango_gat_params* p, void* ctx, size_t ctx_bytes,
                                 const float* dH_out, const float* amax_dH_hint, tango_rng rng, uint32_t layer_id,
                                 float* dH, float* dW, float* da_src, float* da_dst, float* amax_dH, tango_comm* comm,
                                 int32_t* dev_status, cudaStream_t st) {
  TRY(check_gat(G, p));
  TRY(check_comm(G, comm));
  const GatLayout L = gat_layout(G, p);
  if (!ctx || ctx_bytes < L.total) return TANGO_ERR_INVALID_ARG;
  if (!dW || !da_src || !da_dst || (L.n > 0 && !dH_out)) return TANGO_ERR_INVALID_ARG;
  char* c = static_cast<char*>(ctx);
  unsigned* sc = reinterpret_cast<unsigned*>(c + L.off_scal);
  float* scf = reinterpret_cast<float*>(sc);
  int8_t* qH = (int8_t*)(c + L.off_qH);
  int8_t* qW = (int8_t*)(c + L.off_qW);
  int8_t* qHp = (int8_t*)(c + L.off_qHp);
  int8_t* qS = (int8_t*)(c + L.off_qS);
  int8_t* qD = (int8_t*)(c + L.off_qD);
  float* m = (float*)(c + L.off_m);
  float* den = (float*)(c + L.off_den);
  float* P = (float*)(c + L.off_P);
  float* dD = (float*)(c + L.off_dD);
  int8_t* qG = (int8_t*)(c + L.off_qG);
  float* dal = (float*)(c + L.off_dal);
  float* dHp = (float*)(c + L.off_dHp);
  int8_t* qdHp = (int8_t*)(c + L.off_qdHp);
  int64_t* dW64 = (int64_t*)(c + L.off_dW64);
  const int64_t r0 = G->row_begin;
  const GraphDev g = dev_graph(G);

  TRY_CUDA(cudaMemsetAsync(sc + SL_AMAX_G, 0, 8, st));   // amax_G, amax_dH′
  TRY_CUDA(cudaMemsetAsync(da_src, 0, L.HD * 4, st));
  TRY_CUDA(cudaMemsetAsync(da_dst, 0, L.HD * 4, st));
  TRY_CUDA(cudaMemsetAsync(dW64, 0, L.F * L.HD * 8, st));
  AuxStream* aux = aux_stream(st);
  if (!aux) return TANGO_ERR_CUDA;
  {
    const PlanDev pout = plan_of(c, L.off_pout_hbase, L.off_pout_hseg, L.off_pout_hrow, L.off_pout_cnt, L.cap_out,
                                 L.off_pout_tiles, L.tcap);
    TRY_CUDA(stream_after(aux->s, st, aux->ev[0]));
    if (plan_needed(ctx, G, 1)) {
      TRY_CUDA(cudaMemsetAsync(pout.counts, 0, 16, aux->s));
      TRY(launch_status(launch_plan(G->out_ptr, L.n, g.chunk, pout, aux->s)));
      TRY(launch_status(launch_plan_tiles(G->out_ptr, L.n, pout, aux->s)));
      if (use_gat2(g, p, comm))
        TRY(launch_status(launch_gat2_in2out(G->out_eid, L.E, (int32_t*)(c + L.off_dal), aux->s)));
    }
    TRY_CUDA(cudaEventRecord(aux->ev[1], aux->s));
  }
  // B1: Q(∂H_out), shared by ⑤′ and ⑤″
  if (amax_dH_hint) {
    TRY_CUDA(cudaMemcpyAsync(sc + SL_AMAX_G, amax_dH_hint, 4, cudaMemcpyDeviceToDevice, st));
  } else {
    TRY(launch_status(launch_absmax(dH_out, L.n, L.HD, nullptr, sc + SL_AMAX_G, st)));
    TRY(comm_max(comm, sc + SL_AMAX_G, 1, st));
  }
  const bool biased = gat_codes_biased(p->heads, (int)L.HD);   // q_H′ / q_G as excess-128 codes
  TRY(launch_status(launch_quantize(dH_out, L.n, L.HD, nullptr, r0 * L.HD, sc + SL_AMAX_G, p->bits, rng.seed,
                                    rng.step, tag_of(layer_id, R_G), qG + r0 * L.ldHD, L.ldHD, nullptr, 0,
                                    scf + SL_S_G, dev_status, st, biased ? 0x80808080u : 0u)));
  TRY(comm_gather_rows(comm, qG, (size_t)L.ldHD, st));
  // B2-B4: destination rows (in-CSR plan from the forward call), B5-B7: source rows (out-CSR plan,
  // built on the side stream since the start of the call)
  const PlanDev pin = plan_of(c, L.off_pin_hbase, L.off_pin_hseg, L.off_pin_hrow, L.off_pin_cnt, L.cap_in, L.off_pin_tiles, L.tcap);
  const PlanDev pout = plan_of(c, L.off_pout_hbase, L.off_pout_hseg, L.off_pout_hrow, L.off_pout_cnt, L.cap_out, L.off_pout_tiles, L.tcap);
  GatBwdArgs ba{};
  ba.g = g; ba.d = {p->heads, p->head_dim, (int)L.HD}; ba.slope = p->neg_slope; ba.bits = p->bits;
  ba.qS = qS; ba.amax_S = sc + SL_AMAX_S; ba.qD = qD; ba.amax_D = sc + SL_AMAX_D;
  ba.qHp = qHp; ba.ldHp = L.ldHD; ba.amax_Hp = sc + SL_AMAX_HP;
  ba.qG = qG; ba.ldG = L.ldHD; ba.amax_G = sc + SL_AMAX_G;
  ba.m = m; ba.den = den; ba.dalpha = dal; ba.P = P; ba.dD = dD;
  ba.a_src = p->a_src; ba.a_dst = p->a_dst;
  ba.dHp = dHp; ba.amax_dHp = sc + SL_AMAX_DHP; ba.da_src = da_src; ba.da_dst = da_dst;
  ba.pin = pin; ba.pout = pout;
  ba.hP = (float*)(c + L.off_h1); ba.hdD = (float*)(c + L.off_h2); ba.hdS = (float*)(c + L.off_hdS);
  ba.hagg = (float*)(c + L.off_hagg);
  ba.work = (int32_t*)(c + L.off_work);
  ba.dS = (float*)(c + L.off_dS);
  ba.alpha = (const float*)(c + L.off_alpha);
  ba.alpha_dE = (float*)(c + L.off_alpha);
  ba.codes_biased = biased;
  TRY_CUDA(cudaMemsetAsync(ba.work, 0, 64, st));
  const bool v6 = use_gat2(g, p, comm);
  if (v6) {
    // P1 (⑤′ + ⑤″ on source rows), P2 (④′ + ③″ on destination rows), P3 (③′ + ②′ on source rows)
    G2Args a2 = g2_args(L, c, g, p);
    a2.da_src = da_src; a2.da_dst = da_dst;
    TRY_CUDA(cudaMemsetAsync(a2.hcnt, 0, (size_t)L.n * 4, st));
    TRY_CUDA(cudaStreamWaitEvent(st, aux->ev[1], 0));   // out-CSR plan and in-CSR -> out-CSR map done
    const SideStream side = aux->side(4);
    TRY(launch_status(launch_gat2_bwd(a2, st, &side)));
    // ∂a (needs ∂S, ∂D; deterministic chunk order, R39) on the side stream, beside B8/B9
    TRY_CUDA(stream_after(aux->s, st, aux->ev[2]));
    TRY(launch_status(launch_gat2_attn_grad(a2, aux->s)));
    TRY_CUDA(cudaEventRecord(aux->ev[3], aux->s));
  } else {
    const SideStream side_d = aux->side(4), side_s = aux->side(6);
    TRY(launch_status(launch_gat_bwd_dst(ba, st, &side_d)));
    TRY(comm_gather_rows(comm, P, (size_t)L.H * 4, st));
    TRY_CUDA(cudaStreamWaitEvent(st, aux->ev[1], 0));   // out-CSR plan done
    TRY(launch_status(launch_gat_bwd_src(ba, st, &side_s)));
    // ∂a (needs ∂S, ∂D) on the side stream, beside B8/B9: on one GPU in the pinned chunk order of R39
    // (deterministic, gat2.cu) when the shape allows, else fp32 atomics (summed over ranks by comm)
    TRY_CUDA(stream_after(aux->s, st, aux->ev[2]));
    if (!comm && g.row_begin == 0 && L.HD % 128 == 0 && gat_codes_biased(p->heads, (int)L.HD)) {
      G2Args a2 = g2_args(L, c, g, p);
      a2.da_src = da_src; a2.da_dst = da_dst;
      TRY(launch_status(launch_gat2_attn_grad(a2, aux->s)));
    } else {
      TRY(launch_status(launch_gat_attn_grad(ba, aux->s)));
    }
    TRY_CUDA(cudaEventRecord(aux->ev[3], aux->s));
  }
  TRY(comm_max(comm, sc + SL_AMAX_DHP, 1, st));
  // B8: Q(∂H′)
  TRY(launch_status(launch_quantize(dHp, L.n, L.HD, nullptr, r0 * L.HD, sc + SL_AMAX_DHP, p->bits, rng.seed,
                                    rng.step, tag_of(layer_id, R_DHP), qdHp, L.ldHD, nullptr, 0, scf + SL_S_DHP,
                                    dev_status, st)));
  // B9 ①′: ∂H = q_dH′·q_Wᵀ (K = HD) and ∂W = q_Hᵀ·q_dH′ (K = n, split-K int64)
  if (dH) {
    GemmArgs gh{};
    gh.A = qdHp; gh.lda = L.ldHD; gh.a_mn = false;
    gh.B = qW; gh.ldb = L.ldHD; gh.b_mn = false;
    gh.M = L.n; gh.N = L.F; gh.K = L.HD; gh.splits = 1;
    gh.sA = scf + SL_S_DHP; gh.sB = scf + SL_S_W;
    gh.mode = EPI_STORE; gh.C = dH; gh.ldc = L.F;
    TRY(launch_status(launch_gemm(gh, st)));
    if (amax_dH) {
      TRY_CUDA(cudaMemsetAsync(amax_dH, 0, 4, st));
      TRY(launch_status(launch_absmax(dH, L.n, L.F, nullptr, reinterpret_cast<unsigned*>(amax_dH), st)));
      TRY(comm_max(comm, amax_dH, 1, st));
    }
  }
  GemmArgs gw{};
  gw.A = qH; gw.lda = L.ldF; gw.a_mn = true;
  gw.B = qdHp; gw.ldb = L.ldHD; gw.b_mn = true;
  gw.M = L.F; gw.N = L.HD; gw.K = L.n;
  {
    const int64_t tiles = ((L.F + 127) / 128) * ((L.HD + 255) / 256);
    const int64_t kb = (L.n + 127) / 128;
    // CTAs per SM for the split-K ∂W GEMM: its cost is the int64 atomics of the split partials
    // (splits x F x HD), not the MMAs; measured on arxiv (splitk 62 / 50 / 58 / 82 us at 1 / 0.5 /
    // 0.25 / 0.125 CTAs per SM) -> default 0.5; TANGO_DW_CTAS_PER_SM overrides.
    static const double per_sm = [] {
      const char* e = getenv("TANGO_DW_CTAS_PER_SM");
      const double v = e ? atof(e) : 0.5;
      return v > 0 ? v : 0.5;
    }();
    int64_t splits = (int64_t)((num_sms() * per_sm + tiles - 1) / tiles);
    const int64_t min_splits = (L.n + 131071) / 131072;
    if (splits < min_splits) splits = min_splits;
    if (splits > kb) splits = kb > 0 ? kb : 1;
    if (splits < 1) splits = 1;
    gw.splits = (int)splits;
  }
  gw.mode = EPI_ATOMIC64; gw.C = dW64; gw.ldc = L.HD;
  TRY(launch_status(launch_gemm(gw, st)));
  TRY(comm_sum_i64(comm, dW64, (size_t)(L.F * L.HD), st));
  TRY(launch_status(launch_finalize_dw(dW64, L.F * L.HD, scf + SL_S_H, scf + SL_S_DHP, dW, st)));
  TRY_CUDA(cudaStreamWaitEvent(st, aux->ev[3], 0));   // ∂a done (join)
  TRY(comm_sum_f32(comm, da_src, (size_t)L.HD, st));
  TRY(comm_sum_f32(comm, da_dst, (size_t)L.HD, st));
  return TANGO_OK;
}

}  // extern "C"

// ================================================================== GCN
namespace {
struct GcnLayout {
  int64_t n, N, F, O, ldF, ldO;
  size_t off_scal, off_ns, off_nd, off_qX, off_qW, off_qWt, off_qYs, off_ia, off_qGs, off_ib, off_dY, off_qdY,
      off_dW64, total;
};
GcnLayout gcn_layout(const tango_graph* G, const tango_gcn_params* p) {
  GcnLayout L{};
  L.n = G->row_end - G->row_begin; L.N = G->n_global; L.F = p->in_feats; L.O = p->out_feats;
  L.ldF = round_up(L.F, 32); L.ldO = round_up(L.O, 32);
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t at = o; o = align256(o + bytes); return at; };
  L.off_scal = take(SL_NSLOTS * 4);
  L.off_ns = take((size_t)L.n * 4);
  L.off_nd = take((size_t)L.n * 4);
  L.off_qX = take((size_t)L.n * L.ldF);
  L.off_qW = take((size_t)L.F * L.ldO);
  L.off_qWt = take((size_t)L.O * L.ldF);
  L.off_qYs = take((size_t)L.N * L.ldO);
  L.off_ia = take((size_t)L.n * L.O * 4);
  L.off_qGs = take((size_t)L.N * L.ldO);
  L.off_ib = take((size_t)L.n * L.O * 4);
  L.off_dY = take((size_t)L.n * L.O * 4);
  L.off_qdY = take((size_t)L.n * L.ldO);
  L.off_dW64 = take((size_t)L.F * L.O * 8);
  L.total = o;
  return L;
}
tango_status check_gcn(const tango_graph* G, const tango_gcn_params* p) {
  TRY(check_graph(G, true));
  if (!p || !p->W) return TANGO_ERR_INVALID_ARG;
  if (p->bits < 2 || p->bits > 8) return TANGO_ERR_BITS;
  if (p->in_feats <= 0 || p->out_feats <= 0) return TANGO_ERR_SHAPE;
  if (p->in_feats > 133144 || p->out_feats > 133144) return TANGO_ERR_OVERFLOW;
  if (p->out_feats % 8) return TANGO_ERR_UNSUPPORTED;
  return TANGO_OK;
}
}  // namespace

extern "C" {

size_t tango_gcn_ctx_bytes(const tango_graph* G, const tango_gcn_params* p) {
  if (check_gcn(G, p) != TANGO_OK) return 0;
  return gcn_layout(G, p).total;
}

tango_status tango_gcn_ctx_get_view(const tango_graph* G, const tango_gcn_params* p, void* ctx,
                                    tango_gcn_ctx_view* v) {
  TRY(check_gcn(G, p));
  if (!ctx || !v) return TANGO_ERR_INVALID_ARG;
  const GcnLayout L = gcn_layout(G, p);
  char* c = static_cast<char*>(ctx);
  v->qX = (int8_t*)(c + L.off_qX); v->qW = (int8_t*)(c + L.off_qW); v->qWt = (int8_t*)(c + L.off_qWt);
  v->qYs = (int8_t*)(c + L.off_qYs); v->qGs = (int8_t*)(c + L.off_qGs); v->qdY = (int8_t*)(c + L.off_qdY);
  v->ldF = L.ldF; v->ldO = L.ldO; v->ldFt = L.ldF;
  v->ia = (int32_t*)(c + L.off_ia); v->ib = (int32_t*)(c + L.off_ib);
  v->scalars = (float*)(c + L.off_scal);
  return TANGO_OK;
}

tango_status tango_gcn_layer_fwd(const tango_graph* G, const tango_gcn_params* p, const float* X,
                                 const float* amax_X_hint, tango_rng rng, uint32_t layer_id, void* ctx,
                                 size_t ctx_bytes, float* out, float* amax_out, tango_comm* comm, int32_t* dev_status,
                                 cudaStream_t st) {
  TRY(check_gcn(G, p));
  TRY(check_comm(G, comm));
  const GcnLayout L = gcn_layout(G, p);
  if (!ctx || ctx_bytes < L.total) return TANGO_ERR_INVALID_ARG;
  if (L.n > 0 && (!X || !out)) return TANGO_ERR_INVALID_ARG;
  char* c = static_cast<char*>(ctx);
  unsigned* sc = reinterpret_cast<unsigned*>(c + L.off_scal);
  float* scf = reinterpret_cast<float*>(sc);
  float* ns = (float*)(c + L.off_ns);
  float* nd = (float*)(c + L.off_nd);
  int8_t* qX = (int8_t*)(c + L.off_qX);
  int8_t* qW = (int8_t*)(c + L.off_qW);
  int8_t* qWt = (int8_t*)(c + L.off_qWt);
  int8_t* qYs = (int8_t*)(c + L.off_qYs);
  int32_t* ia = (int32_t*)(c + L.off_ia);
  const int64_t r0 = G->row_begin;
  const GraphDev g = dev_graph(G);
  TRY_CUDA(cudaMemsetAsync(sc, 0, SL_NSLOTS * 4, st));
  TRY(launch_status(launch_gcn_norms(g, ns, nd, st)));
  if (amax_X_hint) {
    TRY_CUDA(cudaMemcpyAsync(sc + SL_AMAX_H, amax_X_hint, 4, cudaMemcpyDeviceToDevice, st));
  } else {
    TRY(launch_status(launch_absmax(X, L.n, L.F, nullptr, sc + SL_AMAX_H, st)));
    TRY(comm_max(comm, sc + SL_AMAX_H, 1, st));
  }
  TRY(launch_status(launch_quantize(X, L.n, L.F, nullptr, r0 * L.F, sc + SL_AMAX_H, p->bits, rng.seed, rng.step,
                                    tag_of(layer_id, R_H), qX, L.ldF, nullptr, 0, scf + SL_S_H, dev_status, st)));
  TRY(launch_status(launch_absmax(p->W, L.F, L.O, nullptr, sc + SL_AMAX_W, st)));
  TRY(launch_status(launch_quantize(p->W, L.F, L.O, nullptr, 0, sc + SL_AMAX_W, p->bits, rng.seed, rng.step,
                                    tag_of(layer_id, R_W), qW, L.ldO, qWt, L.ldF, scf + SL_S_W, dev_status, st)));
  // G2 phase A: Ys = (i2f(acc)·s_X s_W)·ns[u], amax(Ys); phase B: q_Ys
  GemmArgs ga{};
  ga.A = qX; ga.lda = L.ldF; ga.B = qWt; ga.ldb = L.ldF;
  ga.M = L.n; ga.N = L.O; ga.K = L.F; ga.splits = 1;
  ga.sA = scf + SL_S_H; ga.sB = scf + SL_S_W; ga.rowscale = ns;
  ga.mode = EPI_AMAX; ga.amax_slot = sc + SL_AMAX_HP;
  TRY(launch_status(launch_gemm(ga, st)));
  TRY(comm_max(comm, sc + SL_AMAX_HP, 1, st));
  GemmArgs gb = ga;
  gb.mode = EPI_QUANT; gb.amax_in = sc + SL_AMAX_HP; gb.bits = p->bits; gb.seed = rng.seed; gb.step = rng.step;
  gb.tag = tag_of(layer_id, R_YS); gb.g_row0 = r0; gb.q_out = qYs + r0 * L.ldO; gb.ldq = L.ldO;
  gb.scale_out = scf + SL_S_HP; gb.status = dev_status;
  TRY(launch_status(launch_gemm(gb, st)));
  TRY(comm_gather_rows(comm, qYs, (size_t)L.ldO, st));
  // G3: int32 SPMM; out = ((float)ia · s_Ys)·nd[v]
  if (amax_out) TRY_CUDA(cudaMemsetAsync(amax_out, 0, 4, st));
  TRY(launch_status(launch_spmm_sum(g, TANGO_IN, (int)L.O, qYs, L.ldO, scf + SL_S_HP, nd, out, ia,
                                    reinterpret_cast<unsigned*>(amax_out), st)));
  TRY(comm_max(comm, amax_out, amax_out ? 1 : 0, st));
  return TANGO_OK;
}

tango_status tango_gcn_layer_bwd(const tango_graph* G, const tango_gcn_params* p, void* ctx, size_t ctx_bytes,
                                 const float* dout, tango_rng rng, uint32_t layer_id, float* dX, float* dW,
                                 tango_comm* comm, int32_t* dev_status, cudaStream_t st) {
  TRY(check_gcn(G, p));
  TRY(check_comm(G, comm));
  const GcnLayout L = gcn_layout(G, p);
  if (!ctx || ctx_bytes < L.total) return TANGO_ERR_INVALID_ARG;
  if (!dW || (L.n > 0 && !dout)) return TANGO_ERR_INVALID_ARG;
  char* c = static_cast<char*>(ctx);
  unsigned* sc = reinterpret_cast<unsigned*>(c + L.off_scal);
  float* scf = reinterpret_cast<float*>(sc);
  float* ns = (float*)(c + L.off_ns);
  float* nd = (float*)(c + L.off_nd);
  int8_t* qX = (int8_t*)(c + L.off_qX);
  int8_t* qW = (int8_t*)(c + L.off_qW);
  int8_t* qGs = (int8_t*)(c + L.off_qGs);
  int32_t* ib = (int32_t*)(c + L.off_ib);
  float* dY = (float*)(c + L.off_dY);
  int8_t* qdY = (int8_t*)(c + L.off_qdY);
  int64_t* dW64 = (int64_t*)(c + L.off_dW64);
  const int64_t r0 = G->row_begin;
  const GraphDev g = dev_graph(G);
  TRY_CUDA(cudaMemsetAsync(sc + SL_AMAX_G, 0, 8, st));
  TRY_CUDA(cudaMemsetAsync(dW64, 0, L.F * L.O * 8, st));
  // Gs = ∂out·nd[v] -> q_Gs
  TRY(launch_status(launch_absmax(dout, L.n, L.O, nd, sc + SL_AMAX_G, st)));
  TRY(comm_max(comm, sc + SL_AMAX_G, 1, st));
  TRY(launch_status(launch_quantize(dout, L.n, L.O, nd, r0 * L.O, sc + SL_AMAX_G, p->bits, rng.seed, rng.step,
                                    tag_of(layer_id, R_GS), qGs + r0 * L.ldO, L.ldO, nullptr, 0, scf + SL_S_G,
                                    dev_status, st)));
  TRY(comm_gather_rows(comm, qGs, (size_t)L.ldO, st));
  // reverse int32 SPMM: ib[u] = Σ_{u→v} q_Gs[v]; ∂Y = ((float)ib·s_Gs)·ns[u]
  TRY(launch_status(launch_spmm_sum(g, TANGO_OUT, (int)L.O, qGs, L.ldO, scf + SL_S_G, ns, dY, ib,
                                    sc + SL_AMAX_DHP, st)));
  TRY(comm_max(comm, sc + SL_AMAX_DHP, 1, st));
  TRY(launch_status(launch_quantize(dY, L.n, L.O, nullptr, r0 * L.O, sc + SL_AMAX_DHP, p->bits, rng.seed, rng.step,
                                    tag_of(layer_id, R_DY), qdY, L.ldO, nullptr, 0, scf + SL_S_DHP, dev_status,
                                    st)));
  if (dX) {
    GemmArgs gh{};
    gh.A = qdY; gh.lda = L.ldO; gh.B = qW; gh.ldb = L.ldO;
    gh.M = L.n; gh.N = L.F; gh.K = L.O; gh.splits = 1;
    gh.sA = scf + SL_S_DHP; gh.sB = scf + SL_S_W;
    gh.mode = EPI_STORE; gh.C = dX; gh.ldc = L.F;
    TRY(launch_status(launch_gemm(gh, st)));
  }
  GemmArgs gw{};
  gw.A = qX; gw.lda = L.ldF; gw.a_mn = true;
  gw.B = qdY; gw.ldb = L.ldO; gw.b_mn = true;
  gw.M = L.F; gw.N = L.O; gw.K = L.n;
  {
    const int64_t tiles = ((L.F + 127) / 128) * ((L.O + 255) / 256);
    const int64_t kb = (L.n + 127) / 128;
    int64_t splits = (num_sms() + tiles - 1) / tiles;
    const int64_t min_splits = (L.n + 131071) / 131072;
    if (splits < min_splits) splits = min_splits;
    if (splits > kb) splits = kb > 0 ? kb : 1;
    gw.splits = (int)splits;
  }
  gw.mode = EPI_ATOMIC64; gw.C = dW64; gw.ldc = L.O;
  TRY(launch_status(launch_gemm(gw, st)));
  TRY(comm_sum_i64(comm, dW64, (size_t)(L.F * L.O), st));
  TRY(launch_status(launch_finalize_dw(dW64, L.F * L.O, scf + SL_S_H, scf + SL_S_DHP, dW, st)));
  return TANGO_OK;
}

// ================================================================== bit-width derivation (NEXT-2)
tango_status tango_quant_error(const float* x, int64_t rows, int64_t cols, const tango_qtensor* q, double* err_out,
                               cudaStream_t st) {
  if (!err_out || rows < 0 || cols < 0) return TANGO_ERR_INVALID_ARG;
  if (rows * cols > 0) {
    if (!x) return TANGO_ERR_INVALID_ARG;
    TRY(check_q(q));
    if (q->rows != rows || q->cols != cols) return TANGO_ERR_SHAPE;
  }
  return launch_status(launch_error_x(x, rows, cols, rows * cols > 0 ? q->q : nullptr, rows * cols > 0 ? q->ld : 0,
                                      rows * cols > 0 ? q->scale : nullptr, err_out, st));
}

tango_status tango_select_bits(const float* x, int64_t count, float threshold, int32_t bmin, int32_t bmax,
                               double* errs_out, int32_t* bits_out, cudaStream_t st) {
  if (!errs_out || !bits_out || count < 0 || (count > 0 && !x)) return TANGO_ERR_INVALID_ARG;
  if (bmin < 2 || bmax > 8 || bmin > bmax) return TANGO_ERR_BITS;
  return launch_status(launch_select_bits(x, count, threshold, bmin, bmax, errs_out, bits_out, st));
}

// ================================================================== communicator
int32_t tango_comm_unique_id_bytes(void) { return (int32_t)sizeof(ncclUniqueId); }

tango_status tango_comm_get_unique_id(void* id_out) {
  if (!id_out) return TANGO_ERR_INVALID_ARG;
  ncclUniqueId id;
  TRY_NCCL(ncclGetUniqueId(&id));
  memcpy(id_out, &id, sizeof(id));
  return TANGO_OK;
}

tango_status tango_comm_init(tango_comm** out, const void* unique_id, int32_t nranks, int32_t rank) {
  if (!out || !unique_id || nranks <= 0 || rank < 0 || rank >= nranks) return TANGO_ERR_INVALID_ARG;
  tango_comm* c = new (std::nothrow) tango_comm();
  if (!c) return TANGO_ERR_INVALID_ARG;
  c->nranks = nranks;
  c->rank = rank;
  ncclUniqueId id;
  memcpy(&id, unique_id, sizeof(id));
  ncclResult_t r = ncclCommInitRank(&c->nccl, nranks, id, rank);
  if (r != ncclSuccess) {
    fprintf(stderr, "[tango] ncclCommInitRank: %s\n", ncclGetErrorString(r));
    delete c;
    return TANGO_ERR_NCCL;
  }
  *out = c;
  return TANGO_OK;
}

tango_status tango_comm_set_partition(tango_comm* c, const int64_t* row_starts) {
  if (!c || !row_starts) return TANGO_ERR_INVALID_ARG;
  c->starts.assign(row_starts, row_starts + c->nranks + 1);
  c->max_rows = 0;
  for (int r = 0; r < c->nranks; ++r) {
    if (c->starts[r] > c->starts[r + 1]) return TANGO_ERR_SHAPE;
    c->max_rows = std::max<int64_t>(c->max_rows, c->starts[r + 1] - c->starts[r]);
  }
  return TANGO_OK;
}

tango_status tango_comm_set_options(tango_comm* c, int32_t always) {
  if (!c) return TANGO_ERR_INVALID_ARG;
  c->always = always != 0;
  return TANGO_OK;
}

tango_status tango_comm_reserve(tango_comm* c, size_t max_row_bytes) {
  if (!c || c->starts.empty()) return TANGO_ERR_INVALID_ARG;
  if (c->local || max_row_bytes <= c->stage_row_bytes) return TANGO_OK;
  if (c->stage) TRY_CUDA(cudaFree(c->stage));
  c->stage = nullptr;
  c->stage_row_bytes = 0;
  const size_t bytes = (size_t)c->nranks * (size_t)c->max_rows * max_row_bytes;
  if (bytes == 0) return TANGO_OK;
  TRY_CUDA(cudaMalloc(&c->stage, bytes));
  c->stage_row_bytes = max_row_bytes;
  return TANGO_OK;
}

int64_t tango_comm_nccl_calls(const tango_comm* c) { return c ? c->nccl_calls : -1; }

tango_status tango_comm_destroy(tango_comm* c) {
  if (!c) return TANGO_ERR_INVALID_ARG;
  if (c->nccl) ncclCommDestroy(c->nccl);
  if (c->stage) cudaFree(c->stage);
  delete c;
  return TANGO_OK;
}

tango_status tango_local_group_create(tango_local_group** out, int32_t nranks) {
  if (!out || nranks < 1 || nranks > 16) return TANGO_ERR_INVALID_ARG;
  tango_local_group* g = new (std::nothrow) tango_local_group();
  if (!g) return TANGO_ERR_INVALID_ARG;
  g->nranks = nranks;
  g->ptr.assign(nranks, nullptr);
  g->ev_a.assign(nranks, nullptr);
  g->ev_b.assign(nranks, nullptr);
  g->tmp.assign(nranks, nullptr);
  g->tmp_bytes.assign(nranks, 0);
  for (int r = 0; r < nranks; ++r) {
    if (cudaEventCreateWithFlags(&g->ev_a[r], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&g->ev_b[r], cudaEventDisableTiming) != cudaSuccess) {
      delete g;
      return TANGO_ERR_CUDA;
    }
  }
  *out = g;
  return TANGO_OK;
}

tango_status tango_local_group_destroy(tango_local_group* g) {
  if (!g) return TANGO_ERR_INVALID_ARG;
  for (int r = 0; r < g->nranks; ++r) {
    if (g->ev_a[r]) cudaEventDestroy(g->ev_a[r]);
    if (g->ev_b[r]) cudaEventDestroy(g->ev_b[r]);
    if (g->tmp[r]) cudaFree(g->tmp[r]);
  }
  delete g;
  return TANGO_OK;
}

tango_status tango_comm_init_local(tango_comm** out, tango_local_group* g, int32_t rank) {
  if (!out || !g || rank < 0 || rank >= g->nranks) return TANGO_ERR_INVALID_ARG;
  tango_comm* c = new (std::nothrow) tango_comm();
  if (!c) return TANGO_ERR_INVALID_ARG;
  c->local = g;
  c->nranks = g->nranks;
  c->rank = rank;
  *out = c;
  return TANGO_OK;
}

}  // extern "C"
