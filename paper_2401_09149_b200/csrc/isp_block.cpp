// The ISP block executor behind the C ABI (include/seqplan_isp.h).
//
// One context per rank. The block's forward and backward are written as a short
// list of phases separated by the exchange points of the ISP plan:
//
//   fwd  F1  norm1 -> QKV GEMM (+RoPE in the epilogue)          | AG(W) on the comm stream
//        --- barrier ---  A2A qkv tokens->heads
//        F2  causal attention on D/p heads
//        --- barrier ---  A2A o heads->tokens
//        F3  O GEMM(+x) -> norm2 -> gate|up GEMM(+SwiGLU) -> down GEMM(+h)
//   bwd  B1  down dgrad/wgrad -> SwiGLU bwd -> gate|up dgrad/wgrad -> norm2 bwd
//            -> O dgrad/wgrad                                  | re-AG(W), RS(dW) on comm
//        --- barrier ---  A2A dO tokens->heads
//        B2  attention backward
//        --- barrier ---  A2A dq|dk|dv heads->tokens (inverse RoPE in the attention-bwd epilogue)
//        B3  QKV dgrad/wgrad -> norm1 bwd
//        --- barrier ---  RS of every weight gradient (fused bf16->fp32 cast/scale)
//
// Multi-process mode (one process per GPU): phases run on the caller's stream,
// gathers and reduce-scatters on an internal comm stream fenced by events; the
// forward prefetches every weight of the block up front (inter-layer prefetch,
// overlap_sim.hpp:95-102) and the backward runs G-W before G-X so each RS overlaps
// the remaining compute (selective overlap, overlap_sim.hpp:141-150).
// Group mode (p contexts on one GPU, tests): the same phases run in lock-step on
// one stream with the collectives inline, which needs no cross-rank spinning.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include <unistd.h>

#include "../../include/seqplan_isp.h"
#include "device_pool.h"
#include "gemm.h"
#include "kernels.h"
#include "nvls.h"
#include "seqplan/mempool.hpp"
#include "seqplan/strategy.hpp"

using bf16 = __nv_bfloat16;

namespace isp {
namespace {

constexpr int kCommCtas = 32;     // SMs lent to a gather / reduce-scatter
constexpr int kA2ACtas = 148 * 4;  // the all-to-all is on the critical path: use the chip
constexpr size_t kFlagBytes = 4096;

struct Status {
  int code = SEQPLAN_ISP_OK;
  std::string msg;
};

#define ISP_CUDA(expr)                                                                   \
  do {                                                                                   \
    cudaError_t _e = (expr);                                                             \
    if (_e != cudaSuccess) {                                                             \
      throw IspError(SEQPLAN_ISP_ERR_RUNTIME,                                            \
                     std::string(#expr) + ": " + cudaGetErrorString(_e));                \
    }                                                                                    \
  } while (0)

struct IspError {
  int code;
  std::string msg;
  IspError(int c, std::string m) : code(c), msg(std::move(m)) {}
};

inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// Stream memory operations (executed by the GPU front end, no SM needed): used for the
// cross-GPU barrier so a comm-stream barrier never waits for SMs held by a persistent GEMM.
using PfnWriteValue32 = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using PfnWaitValue32 = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
struct MemOps {
  PfnWriteValue32 write = nullptr;
  PfnWaitValue32 wait = nullptr;
  bool ok() const { return write && wait; }
};
const MemOps& memops() {
  static MemOps m = [] {
    MemOps r;
    if (std::getenv("SEQPLAN_ISP_KERNEL_BARRIER")) return r;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      r.write = reinterpret_cast<PfnWriteValue32>(p);
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      r.wait = reinterpret_cast<PfnWaitValue32>(p);
    return r;
  }();
  return m;
}

}  // namespace
}  // namespace isp

using namespace isp;

struct seqplan_isp_ctx {
  // ---- configuration ----
  int world = 1, rank = 0, device = 0, num_sms = 148;
  bool group_mode = false;
  uint32_t flags = 0;
  int64_t H = 0, D = 0, S = 0, I = 0, d = 0, T = 0, Hl = 0, Dl = 0;
  float eps = 1e-5f;
  double rope_base = 10000.0;
  std::string last_error;

  // ---- symmetric heap (exchange buffers; identical offsets on every rank) ----
  char* heap = nullptr;
  size_t heap_bytes = 0;
  void* peer_heap[kMaxRanks] = {};
  bool peer_opened[kMaxRanks] = {};
  // ranks of one process on one device linked by seqplan_isp_link_local_peers: the multi-process
  // code path (own streams, production transports, memop barriers) with the peers' heaps on the
  // same GPU; TIMELINE / PROFILE collection is deferred to the query (no host sync in block_bwd)
  bool co_resident = false;
  // micro-batches per step (Strategy::micro_batch_num, cost.hpp:202-204): block_bwd calls
  // 2..n of a step add their weight gradients into the fp32 shards instead of overwriting
  int micro_batches = 1, mb_index = 0;
  bool accum = false;
  size_t off_flags = 0, off_wshard[SEQPLAN_W_COUNT] = {}, off_qkv_tok = 0, off_o_heads = 0,
         off_do_tok = 0, off_dqkv_heads = 0, off_part[SEQPLAN_W_COUNT] = {};
  // fused all-to-all (p > 1, d = 128): producers' epilogues push into these peer-writable buffers
  bool fused_a2a = false;
  size_t off_qkv_heads = 0, off_o_tok = 0, off_dO_heads = 0, off_dqkv_tok = 0;
  uint32_t epoch_compute = 0, epoch_comm = 0;
  // push-mode weight traffic (multi-process): every rank stores its shards into the peers'
  // pinned comm double buffer (set 0 = forward gather, set 1 = backward re-gather; the
  // reference's pinned comm pool, cost.hpp:147 / mempool.hpp pinned policy) and its gradient
  // partial slices into the owners' staging slots; per-(tensor, source) epoch flags order them
  size_t off_gath[2][SEQPLAN_W_COUNT] = {}, off_stage[SEQPLAN_W_COUNT] = {};
  uint32_t step_epoch = 0;
  int gather_set = 0;
  bool push_primed = false;  // SKIP_COMM: buffers filled by one real step, then reused
  bool defer_bwd_set = false;  // fwd_issue_gathers leaves the backward set to the caller (stacks)
  // gather tail: forward-set tensors (and the backward set) issued behind the Q|K|V all-to-all
  // (SEQPLAN_ISP_DEFER_GATHER=1; measured neutral at 7B-32K p = 2/4: the A2A shortens, the rank skew stays)
  bool defer_gathers = false;
  // stored-dS attention backward workspace cap, GiB (SEQPLAN_ISP_DS_WS_GB; 0 = two-role kernel);
  // default: a quarter of the device memory, at most 48 GiB (7B-32K p = 1: all 32 heads' dS, 34.6 GB)
  int64_t ds_ws_gb = -1;
  int64_t ds_ws_cached = 0;  // largest workspace the pool has served (its segment stays cached)
  int tail[SEQPLAN_W_COUNT] = {}, tail_n = 0;
  cudaEvent_t ev_tail = nullptr;
  bool owns_comm = true;       // false: the comm stream belongs to layer 0 of a stack
  int ag_ctas = 96, ag_kind = kPushBulk;  // all-gathers: bulk-copy push, one chunk stored to every rank
  // reduce-scatter staging: each chunk goes to one destination, so the bulk kernel (one load in
  // flight per CTA) is load-latency bound there; 16-B vector stores from 256-thread CTAs
  // (128 B in flight per thread, no shared memory: they co-reside with every compute kernel)
  int rs_ctas = 128;
  // NVLink SHARP reduce-scatter (push transport; seqplan_isp_nvls_*): the bf16 partials of Wqkv,
  // Wo, W_gate|up and W_down live in a device buffer bound to one multicast object across the
  // ranks, and each owner reduces its slices in the switch (multimem.ld_reduce) — no staging
  // copies, no reduction over p slots. Measured at p = 4: 7B-4K +7.5 %, 7B-32K +1.1 %.
  // The all-gather's pinned double buffer can live there too (SEQPLAN_ISP_NVLS bit 2): each rank
  // then stores its shard once, to the multicast address, and the switch writes every rank's copy
  // (measured slower than the bulk-copy push at 7B-4K p = 4, 1.456 vs 1.50 M tokens/s: off).
  Nvls nvls_buf;
  bool nvls = false, nvls_ag = false;
  int nvls_pref = 1;  // SEQPLAN_ISP_NVLS: 0 off, 1 reduce-scatter (default), 2 all-gather, 3 both
  size_t nvls_off[SEQPLAN_W_COUNT] = {}, nvls_gath_off[2][SEQPLAN_W_COUNT] = {}, nvls_bytes = 0;
  int red_ctas = 0;  // CTAs of the staged-slot reductions (SEQPLAN_ISP_RED_CTAS; default 4 per SM)
  int gemm_sm_budget = 0;  // > 0 when the all-gather holds SMs of its own (kPushBulkWide)
  uint32_t* error_flag = nullptr;  // device, in the heap flags page

  // ---- device pool (subsystem 5) and persistent buffers ----
  DevicePool own_pool;
  DevicePool* pool = &own_pool;  // a stack's layers share layer 0's pool
  bool owns_pool = true;
  bool recompute = false;        // a = 1: only the block input survives the forward
  bool fuse_swiglu_bwd = false;  // SEQPLAN_ISP_FUSE_SWIGLU_BWD=1 (development)
  bool no_bwd_prefetch = false;  // SEQPLAN_ISP_BWD_PREFETCH=0: copy-engine re-gather at backward start
  bool ce_a2a = false;           // Ulysses all-to-all on the copy engines (SEQPLAN_ISP_A2A_CE)
  bool rs_ce = false;            // push mode: reduce-scatter staged by the copy engines (SEQPLAN_ISP_RS_CE)
  bool early_reduce = true;      // RS reductions on their own stream as slices land (SEQPLAN_ISP_EARLY_REDUCE=0: at step end)
  cudaStream_t red = nullptr;    // reduction stream of the early reduce-scatter
  cudaEvent_t ev_rs_sent[SEQPLAN_W_COUNT] = {};
  cudaEvent_t ev_red_done = nullptr;
  // QKV GEMM reads the peers' working shards over NVLink with its own TMA loads (the weight
  // all-gather fused into its first consumer, no gather buffer); SEQPLAN_ISP_AG_GEMM=1
  bool ag_gemm = false;
  bool qkv_slice = true;         // QKV GEMM sliced by weight-shard source (SEQPLAN_ISP_QKV_SLICE=0 turns off; +1.1 % at 4K p = 2, neutral at p = 4)
  bool recomputing = false;      // inside the backward's forward recomputation
  bool acts_live = false;        // saved activations currently allocated
  bool scratch_live = false;     // backward scratch currently allocated
  float* master[SEQPLAN_W_COUNT] = {};
  float* grad[SEQPLAN_W_COUNT] = {};
  float* adam_m[SEQPLAN_W_COUNT] = {};  // optimizer moments (seqplan_isp_adamw_step), lazily created
  float* adam_v[SEQPLAN_W_COUNT] = {};
  bf16* wgu_local = nullptr;  // p = 1: interleaved gate|up working copy
  float* cos_t = nullptr;
  float* sin_t = nullptr;
  // saved activations
  bf16 *n1 = nullptr, *qkv_heads = nullptr, *o_tok = nullptr, *h = nullptr, *n2 = nullptr;
  float *rstd1 = nullptr, *rstd2 = nullptr, *lse = nullptr;
  bf16 *gu = nullptr, *a = nullptr;  // transient: fwd -> bwd
  // backward scratch
  bf16 *dh = nullptr, *dn = nullptr, *dO_heads = nullptr, *dqkv_tok = nullptr;
  float *delta = nullptr, *dq_acc = nullptr, *dg_scratch = nullptr;
  bf16* local_part[SEQPLAN_W_COUNT] = {};  // p = 1 not used

  // ---- streams / events ----
  cudaStream_t comm = nullptr;
  // one stream per peer: copy-engine transfers from different peers run concurrently
  cudaStream_t peer_st[kMaxRanks] = {};
  cudaEvent_t ev_fork = nullptr, ev_join[kMaxRanks] = {};
  // tensor t's shard from rank q has landed: [0] the forward set, [1] the backward re-gather
  cudaEvent_t ev_tq[2][SEQPLAN_W_COUNT][kMaxRanks] = {};
  bool pipelined_gather = false;                        // wait_gathered uses ev_tq (copy-engine path)
  int evset = 0;                                        // which ev_tq set the current pass waits on
  // copy-engine mode: the backward re-gather is issued at step start right behind the forward
  // set (the comm stream is idle during the forward), into its own CommBuffers
  bf16* pre_bwd[SEQPLAN_W_COUNT] = {};
  bool bwd_prefetched = false;
  cudaEvent_t ev_gathered[SEQPLAN_W_COUNT] = {};
  cudaEvent_t ev_wgrad[SEQPLAN_W_COUNT] = {};
  cudaEvent_t ev_comm_done = nullptr, ev_start = nullptr;
  cudaEvent_t ev_staged[SEQPLAN_W_COUNT] = {};
  void* stage[SEQPLAN_W_COUNT] = {};  // RS staging: this rank's slice of every rank's partial
  bool weights_dirty = true;
  bool fwd_done = false;
  const void* last_x = nullptr;

  // gathered weights of the current pass (pool CommBuffer allocations)
  bf16* gathered[SEQPLAN_W_COUNT] = {};
  // SEQPLAN_ISP_FLAG_SKIP_COMM: weights gathered once and kept (measurement of exposed comm)
  bf16* pregathered[SEQPLAN_W_COUNT] = {};
  bool skip_comm() const { return (flags & SEQPLAN_ISP_FLAG_SKIP_COMM) && world > 1; }
  // push (bulk-copy) weight traffic for p >= 4; at p = 2 the copy engines' pull is faster
  // (measured: 7B-4K/32K at p = 2, CE 2-7 % ahead; at p = 4 push +25 %). SEQPLAN_ISP_PUSH=0/1 forces.
  int push_pref = -1;
  bool push_mode() const { return world > 1 && !group_mode && (push_pref >= 0 ? push_pref == 1 : world >= 4); }
  bool push_skip() const { return skip_comm() && push_primed; }

  // timeline
  struct TEv {
    int stream, kind;
    int64_t layer;
    cudaEvent_t b, e;
  };
  std::vector<TEv> tl_pending;
  std::vector<seqplan_timeline_event> timeline;
  // per-kernel profile (SEQPLAN_ISP_FLAG_PROFILE) and launch counter
  struct KEv {
    int kind;
    double flops, bytes;
    cudaEvent_t b, e;
  };
  std::vector<KEv> kprof_pending;
  std::vector<seqplan_kernel_record> kprof;
  int64_t launches = 0;

  // ---- helpers ----
  template <typename T>
  T* hp(size_t off) { return reinterpret_cast<T*>(heap + off); }
  template <typename T>
  T* peer(int q, size_t off) { return reinterpret_cast<T*>(static_cast<char*>(peer_heap[q]) + off); }
  PeerPtrs peers_at(size_t off) {
    PeerPtrs p{};
    for (int q = 0; q < world; ++q) p.p[q] = static_cast<char*>(peer_heap[q]) + off;
    return p;
  }
  int64_t numel(int t) const {
    switch (t) {
      case SEQPLAN_W_NORM1: case SEQPLAN_W_NORM2: return H;
      case SEQPLAN_W_QKV: return 3 * H * H;
      case SEQPLAN_W_O: return H * H;
      default: return I * H;
    }
  }
  int64_t shard(int t) const { return numel(t) / world; }
  bf16* wshard(int t) { return hp<bf16>(off_wshard[t]); }
};

namespace {

using Ctx = seqplan_isp_ctx;

void* pool_alloc(Ctx* c, int64_t bytes, seqplan::AllocTag tag, cudaStream_t st) {
  void* p = c->pool->alloc(bytes, tag, st);
  if (!p) throw IspError(SEQPLAN_ISP_ERR_OOM, "device pool: " + c->pool->error());
  return p;
}

// ---- timeline -------------------------------------------------------------------
struct Span {
  Ctx* c;
  cudaStream_t st;
  int stream_kind, kind;
  int64_t layer;
  cudaEvent_t b = nullptr;
  Span(Ctx* cc, cudaStream_t s, int sk, int k, int64_t l) : c(cc), st(s), stream_kind(sk), kind(k), layer(l) {
    if (c->flags & SEQPLAN_ISP_FLAG_TIMELINE) {
      cudaEventCreate(&b);
      cudaEventRecord(b, st);
    }
  }
  ~Span() {
    if (!b) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    c->tl_pending.push_back({stream_kind, kind, layer, b, e});
  }
};

// Per-kernel CUDA events (SEQPLAN_ISP_FLAG_PROFILE): algorithmic flops/bytes per launch.
struct KTimer {
  Ctx* c;
  cudaStream_t st;
  int kind;
  double flops, bytes;
  cudaEvent_t b = nullptr;
  KTimer(Ctx* cc, cudaStream_t s, int k, double f, double by) : c(cc), st(s), kind(k), flops(f), bytes(by) {
    if (c->flags & SEQPLAN_ISP_FLAG_PROFILE) {
      cudaEventCreate(&b);
      cudaEventRecord(b, st);
    }
  }
  ~KTimer() {
    if (!b) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    c->kprof_pending.push_back({kind, flops, bytes, b, e});
  }
};

#define ISP_LAUNCH(n, expr) \
  do {                      \
    ISP_CUDA(expr);         \
    c->launches += (n);     \
  } while (0)

// HBM-bound elementwise kernels: timed under SEQPLAN_ISP_FLAG_PROFILE with their algorithmic bytes.
#define ISP_EW(n, bytes, expr)                                         \
  do {                                                                 \
    KTimer kt_ew_(c, st, SEQPLAN_K_ELEMENTWISE, 0, double(bytes));     \
    ISP_LAUNCH(n, expr);                                               \
  } while (0)

void gemm(Ctx* c, const GemmOperand& A, const GemmOperand& B, const GemmArgs& args, int epi, cudaStream_t st) {
  const double M = args.M, N = args.N, K = args.K;
  const double out_bytes = (epi == EPI_F32 ? 4.0 : 2.0) * M * N *
                           (epi == EPI_SWIGLU ? 1.5 : epi == EPI_SWIGLU_BWD ? 4.0 : 1.0);
  KTimer kt(c, st, SEQPLAN_K_GEMM, 2.0 * M * N * K, 2.0 * (M * K + N * K) + out_bytes);
  c->launches += 1;
  GemmArgs a = args;
  if (c->push_mode() && c->gemm_sm_budget > 0) a.sm_budget = c->gemm_sm_budget;
  // Wave pacing: off for co-resident ranks (their GEMMs run concurrently on one GPU: a paced grid
  // could wait for clusters that cannot become resident) and under the push transport, whose SM
  // copy / reduction kernels slow some clusters and then hold every cluster at the wave boundary
  // (7B-32K p = 4: 1.906 M tokens/s without, 1.867 M with; 7B-4K 1.60 vs 1.53 M)
  if (c->co_resident || c->push_mode()) a.wave_sync = 0;
  cudaError_t e = gemm_launch(A, B, a, epi, st);
  if (e == cudaErrorInvalidValue)
    throw IspError(SEQPLAN_ISP_ERR_UNSUPPORTED, "GEMM shape not tiled by the sm_100a kernel (M%128, N%128, K%64)");
  ISP_CUDA(e);
}

// ---- collectives (dispatch on mode) -----------------------------------------------
void barrier(Ctx* c, cudaStream_t st, bool comm_lane) {
  if (c->world == 1 || c->group_mode || c->skip_comm()) return;
  uint32_t& ep = comm_lane ? c->epoch_comm : c->epoch_compute;
  ++ep;
  const size_t off = c->off_flags + (comm_lane ? 64 * sizeof(uint32_t) : 0);
  const MemOps& mo = memops();
  if (mo.ok()) {  // publish epoch into every peer's slot for this rank, then wait for all peers
    for (int q = 0; q < c->world; ++q) {
      auto dst = reinterpret_cast<CUdeviceptr>(c->peer<uint32_t>(q, off) + c->rank);
      if (mo.write(reinterpret_cast<CUstream>(st), dst, ep, 0) != CUDA_SUCCESS)
        throw IspError(SEQPLAN_ISP_ERR_RUNTIME, "cuStreamWriteValue32 to a peer failed");
    }
    for (int q = 0; q < c->world; ++q) {
      auto mine = reinterpret_cast<CUdeviceptr>(c->hp<uint32_t>(off) + q);
      if (mo.wait(reinterpret_cast<CUstream>(st), mine, ep, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
        throw IspError(SEQPLAN_ISP_ERR_RUNTIME, "cuStreamWaitValue32 failed");
    }
    return;
  }
  ISP_LAUNCH(1, peer_barrier(c->peers_at(off), c->world, c->rank, ep, c->error_flag, st));
}

// Runs fn(q, stream) for every rank q: the local rank on `cs`, each peer on its own stream so
// copy-engine transfers from different peers proceed in parallel; joined back into `cs`.
template <typename F>
void fan_out(Ctx* c, cudaStream_t cs, F&& fn) {
  ISP_CUDA(cudaEventRecord(c->ev_fork, cs));
  for (int q = 0; q < c->world; ++q) {
    if (q == c->rank) continue;
    ISP_CUDA(cudaStreamWaitEvent(c->peer_st[q], c->ev_fork, 0));
    fn(q, c->peer_st[q]);
    ISP_CUDA(cudaEventRecord(c->ev_join[q], c->peer_st[q]));
  }
  fn(c->rank, cs);
  for (int q = 0; q < c->world; ++q)
    if (q != c->rank) ISP_CUDA(cudaStreamWaitEvent(cs, c->ev_join[q], 0));
}

// Gather tensor t into a pool CommBuffer (or return the local working copy at p = 1).
void gather_weight(Ctx* c, int t, cudaStream_t st) {
  if (c->world == 1) {
    c->gathered[t] = (t == SEQPLAN_W_GATE) ? c->wgu_local : c->wshard(t);
    return;
  }
  if (c->skip_comm() && c->pregathered[t]) {
    c->gathered[t] = c->pregathered[t];
    return;
  }
  Span sp(c, st, 1, SEQPLAN_EV_ALL_GATHER, t);
  const double frac = double(c->world - 1) / double(c->world);
  const bool ce = !c->group_mode;  // copy engines: no SM is taken from the compute stream
  if (t == SEQPLAN_W_GATE) {  // gate|up gathered together, interleaved in kGuBlock-row blocks
    const int64_t bytes = 2 * c->I * c->H * 2;
    KTimer kt(c, st, SEQPLAN_K_ALL_GATHER, 0, frac * double(bytes));
    bf16* dst = static_cast<bf16*>(pool_alloc(c, bytes, seqplan::AllocTag::CommBuffer, st));
    if (ce) {
      const int64_t B = kGuBlock, H = c->H, rpr = c->I / c->world;
      fan_out(c, st, [&](int q, cudaStream_t qs) {
        for (int which = 0; which < 2; ++which) {
          const bf16* src = c->peer<bf16>(q, c->off_wshard[which ? SEQPLAN_W_UP : SEQPLAN_W_GATE]);
          bf16* d0 = dst + ((q * rpr / B) * 2 * B + which * B) * H;
          ISP_CUDA(cudaMemcpy2DAsync(d0, size_t(2 * B * H * 2), src, size_t(B * H * 2), size_t(B * H * 2),
                                     size_t(rpr / B), cudaMemcpyDefault, qs));
        }
      });
    } else {
      ISP_LAUNCH(1, allgather_pull_interleave(c->peers_at(c->off_wshard[SEQPLAN_W_GATE]),
                                              c->peers_at(c->off_wshard[SEQPLAN_W_UP]), c->world, c->I, c->H,
                                              dst, st, kCommCtas));
    }
    c->gathered[t] = dst;
  } else {
    const int64_t bytes = c->numel(t) * 2;
    KTimer kt(c, st, SEQPLAN_K_ALL_GATHER, 0, frac * double(bytes));
    bf16* dst = static_cast<bf16*>(pool_alloc(c, bytes, seqplan::AllocTag::CommBuffer, st));
    if (ce) {
      const int64_t sh = c->shard(t);
      fan_out(c, st, [&](int q, cudaStream_t qs) {
        ISP_CUDA(cudaMemcpyAsync(dst + q * sh, c->peer<bf16>(q, c->off_wshard[t]), size_t(sh * 2),
                                 cudaMemcpyDefault, qs));
      });
    } else {
      ISP_LAUNCH(1, allgather_pull(c->peers_at(c->off_wshard[t]), c->world, c->shard(t), dst, st, c->num_sms,
                                   kCommCtas));
    }
    c->gathered[t] = dst;
  }
}

void release_weight(Ctx* c, int t, cudaStream_t st) {
  if (c->push_mode()) {  // pinned set buffers: nothing to free
    c->gathered[t] = nullptr;
    return;
  }
  if (c->skip_comm()) {
    c->pregathered[t] = c->gathered[t];
    c->gathered[t] = nullptr;
    return;
  }
  if (c->world > 1 && c->gathered[t]) c->pool->free(c->gathered[t], st);
  c->gathered[t] = nullptr;
}

// Reduce-scatter the weight gradient partial of tensor t into the fp32 grad shard.
bool nvls_tensor(int t) {
  return t == SEQPLAN_W_QKV || t == SEQPLAN_W_O || t == SEQPLAN_W_GATE || t == SEQPLAN_W_DOWN;
}
// bf16 weight-gradient partial of tensor t: the NVLS buffer (unicast mapping) or the heap
bf16* part_bf16(Ctx* c, int t) {
  if (c->nvls && nvls_tensor(t)) return reinterpret_cast<bf16*>(c->nvls_buf.uc + c->nvls_off[t]);
  return c->hp<bf16>(c->off_part[t]);
}

// This rank's slices of partial t reduced in the NVSwitch (every rank's partial complete).
void nvls_reduce(Ctx* c, int t, cudaStream_t st) {
  const bf16* mc = reinterpret_cast<const bf16*>(c->nvls_buf.mcva + c->nvls_off[t]);
  KTimer kt(c, st, SEQPLAN_K_REDUCE_SCATTER, 0, double(c->shard(t)) * 2 * (t == SEQPLAN_W_GATE ? 2 : 1));
  if (t == SEQPLAN_W_GATE)
    ISP_LAUNCH(1, nvls_reduce_scatter(mc, c->world, c->rank, 2 * (c->I / c->world) * c->H, c->I, c->H, 1.0f,
                                      c->accum ? 1 : 0, c->grad[SEQPLAN_W_GATE], c->grad[SEQPLAN_W_UP], st,
                                      c->red_ctas));
  else
    ISP_LAUNCH(1, nvls_reduce_scatter(mc, c->world, c->rank, c->shard(t), 0, c->H, 1.0f, c->accum ? 1 : 0,
                                      c->grad[t], nullptr, st, c->red_ctas));
}

void reduce_scatter_grad(Ctx* c, int t, cudaStream_t st) {
  if (c->skip_comm()) return;
  Span sp(c, st, 1, SEQPLAN_EV_REDUCE_SCATTER, t);
  const double frac = double(c->world - 1) / double(c->world);
  const bool norm = (t == SEQPLAN_W_NORM1 || t == SEQPLAN_W_NORM2);
  const double part_bytes = t == SEQPLAN_W_GATE ? 2.0 * c->I * c->H * 2 : double(c->numel(t)) * (norm ? 4 : 2);
  if (c->nvls && nvls_tensor(t)) {
    nvls_reduce(c, t, st);
    return;
  }
  KTimer kt(c, st, SEQPLAN_K_REDUCE_SCATTER, 0, frac * part_bytes);
  if (t == SEQPLAN_W_GATE) {
    ISP_LAUNCH(1, reduce_scatter_pull_interleave(c->peers_at(c->off_part[SEQPLAN_W_GATE]), c->world, c->rank,
                                            c->I, c->H, 1.0f, c->accum ? 1 : 0, c->grad[SEQPLAN_W_GATE],
                                            c->grad[SEQPLAN_W_UP], st, kCommCtas));
  } else {
    const bool f32 = (t == SEQPLAN_W_NORM1 || t == SEQPLAN_W_NORM2);
    ISP_LAUNCH(1, reduce_scatter_pull(c->peers_at(c->off_part[t]), c->world, c->rank, c->shard(t), f32, 1.0f,
                                 c->accum ? 1 : 0, c->grad[t], st, kCommCtas));
  }
}

// ---------------------------------------------------------------------------------
// forward phases
// ---------------------------------------------------------------------------------
bf16* qkv_tok_buf(Ctx* c) { return c->hp<bf16>(c->off_qkv_tok); }

void set_push(Ctx* c, GemmArgs& g, size_t heap_off, int parts) {
  for (int q = 0; q < c->world; ++q) g.push[q] = static_cast<char*>(c->peer_heap[q]) + heap_off;
  g.push_T = static_cast<int>(c->T);
  g.push_rank = c->rank;
  g.push_parts = parts;
  g.push_H = static_cast<int>(c->H);
  g.push_Hl = static_cast<int>(c->Hl);
  g.push_d = static_cast<int>(c->d);
}

AttnPush attn_push(Ctx* c, size_t heap_off, int64_t ld, int64_t col_o, int64_t col_q, int64_t col_k, int64_t col_v) {
  AttnPush p{};
  for (int q = 0; q < c->world; ++q) p.p[q] = static_cast<char*>(c->peer_heap[q]) + heap_off;
  p.T = static_cast<int>(c->T);
  p.ld = ld;
  p.col_o = col_o;
  p.col_q = col_q;
  p.col_k = col_k;
  p.col_v = col_v;
  return p;
}

// Ulysses all-to-all on the copy engines: one strided 2-D copy per source rank, each peer's on
// its own stream (no SM is used, the compute stream only waits). Rows are (token, part) pairs:
// token layout [T, parts*H] rows have pitch H, head layout [S, parts*Hl] rows pitch Hl.
// tokens -> heads: dst rows (q*T + t, part) <- rank q's (t, part) columns [rank*Hl, +Hl).
void a2a_ce_to_heads(Ctx* c, size_t src_off, int parts, bf16* dst, cudaStream_t st) {
  const int64_t T = c->T, H = c->H, Hl = c->Hl;
  fan_out(c, st, [&](int q, cudaStream_t qs) {
    const bf16* src = c->peer<bf16>(q, src_off) + c->rank * Hl;
    ISP_CUDA(cudaMemcpy2DAsync(dst + q * T * parts * Hl, size_t(Hl * 2), src, size_t(H * 2), size_t(Hl * 2),
                               size_t(T * parts), cudaMemcpyDefault, qs));
  });
}
// heads -> tokens: dst (t, part) columns [q*Hl, +Hl) <- rank q's rows (rank*T + t, part).
void a2a_ce_to_tokens(Ctx* c, size_t src_off, int parts, bf16* dst, cudaStream_t st) {
  const int64_t T = c->T, H = c->H, Hl = c->Hl;
  fan_out(c, st, [&](int q, cudaStream_t qs) {
    const bf16* src = c->peer<bf16>(q, src_off) + c->rank * T * parts * Hl;
    ISP_CUDA(cudaMemcpy2DAsync(dst + q * Hl, size_t(H * 2), src, size_t(Hl * 2), size_t(Hl * 2),
                               size_t(T * parts), cudaMemcpyDefault, qs));
  });
}

// Copy-engine all-gather of several tensors as one pipeline: every peer's stream pulls that
// peer's shards of all tensors back to back (no per-tensor join, so DMA setup of the next copy
// overlaps the current one and all peers stream concurrently); a consumer waits only on the
// per-(tensor, peer) events of the tensor it needs.
// set 0: into gathered[] (this pass); set 1: the backward re-gather prefetched into pre_bwd[].
void gather_pipelined(Ctx* c, const int* order, int n, cudaStream_t cs, int set = 0) {
  const int64_t B = kGuBlock, H = c->H, rpr = c->I / c->world;
  bf16** dsts = set ? c->pre_bwd : c->gathered;
  int todo[SEQPLAN_W_COUNT];
  int m = 0;
  for (int i = 0; i < n; ++i) {
    const int t = order[i];
    if (c->skip_comm() && c->pregathered[t]) {
      dsts[t] = c->pregathered[t];
      continue;
    }
    const int64_t bytes = (t == SEQPLAN_W_GATE ? 2 * c->I * c->H : c->numel(t)) * 2;
    dsts[t] = static_cast<bf16*>(pool_alloc(c, bytes, seqplan::AllocTag::CommBuffer, cs));
    todo[m++] = t;
  }
  if (m == 0) return;
  double remote = 0;
  for (int i = 0; i < m; ++i)
    remote += double(todo[i] == SEQPLAN_W_GATE ? 2 * c->I * c->H : c->numel(todo[i])) * 2 * (c->world - 1) / c->world;
  Span sp(c, cs, 1, SEQPLAN_EV_ALL_GATHER, todo[0]);
  KTimer kt(c, cs, SEQPLAN_K_ALL_GATHER, 0, remote);
  ISP_CUDA(cudaEventRecord(c->ev_fork, cs));
  auto copy = [&](int t, int q, cudaStream_t qs) {
    bf16* dst = dsts[t];
    if (t == SEQPLAN_W_GATE) {
      for (int which = 0; which < 2; ++which) {
        const bf16* src = c->peer<bf16>(q, c->off_wshard[which ? SEQPLAN_W_UP : SEQPLAN_W_GATE]);
        bf16* d0 = dst + ((q * rpr / B) * 2 * B + which * B) * H;
        ISP_CUDA(cudaMemcpy2DAsync(d0, size_t(2 * B * H * 2), src, size_t(B * H * 2), size_t(B * H * 2),
                                   size_t(rpr / B), cudaMemcpyDefault, qs));
      }
    } else {
      const int64_t sh = c->shard(t);
      ISP_CUDA(cudaMemcpyAsync(dst + q * sh, c->peer<bf16>(q, c->off_wshard[t]), size_t(sh * 2), cudaMemcpyDefault,
                               qs));
    }
    ISP_CUDA(cudaEventRecord(c->ev_tq[set][t][q], qs));
  };
  for (int q = 0; q < c->world; ++q) {
    if (q == c->rank) continue;
    ISP_CUDA(cudaStreamWaitEvent(c->peer_st[q], c->ev_fork, 0));
    for (int i = 0; i < m; ++i) copy(todo[i], q, c->peer_st[q]);
  }
  for (int i = 0; i < m; ++i) copy(todo[i], c->rank, cs);  // own shard: local copy
  for (int q = 0; q < c->world; ++q)  // the comm stream rejoins before later comm work
    if (q != c->rank) ISP_CUDA(cudaStreamWaitEvent(cs, c->ev_tq[set][todo[m - 1]][q], 0));
  c->pipelined_gather = true;
}

// ---- push-mode collectives (multi-process) -------------------------------------------
// Flag slots in the heap flags page (uint32 index): AG [512 + (set*8 + t)*8 + src],
// RS [640 + t*8 + src]; a slot holds the step epoch of the last completed transfer.
size_t ag_flag(const Ctx* c, int set, int t, int src) {
  return c->off_flags + sizeof(uint32_t) * (512 + (set * 8 + t) * 8 + src);
}
size_t rs_flag(const Ctx* c, int t, int src) { return c->off_flags + sizeof(uint32_t) * (640 + t * 8 + src); }

// After the push kernel on stream cs: publish this rank's epoch into every peer's slot
// (cuStreamWriteValue32 is preceded by a system-wide fence).
void signal_peers(Ctx* c, cudaStream_t cs, size_t slot_off) {
  const MemOps& mo = memops();
  for (int q = 0; q < c->world; ++q) {
    if (q == c->rank) continue;
    auto dst = reinterpret_cast<CUdeviceptr>(c->peer<uint32_t>(q, slot_off));
    if (!mo.ok() || mo.write(reinterpret_cast<CUstream>(cs), dst, c->step_epoch, 0) != CUDA_SUCCESS)
      throw IspError(SEQPLAN_ISP_ERR_RUNTIME, "cuStreamWriteValue32 to a peer failed");
  }
}
// Stream st waits until every peer q published the current epoch into slot_of(q).
template <typename F>
void wait_peers(Ctx* c, cudaStream_t st, F&& slot_of) {
  const MemOps& mo = memops();
  for (int q = 0; q < c->world; ++q) {
    if (q == c->rank) continue;
    auto mine = reinterpret_cast<CUdeviceptr>(c->hp<uint32_t>(slot_of(q)));
    if (!mo.ok() || mo.wait(reinterpret_cast<CUstream>(st), mine, c->step_epoch, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
      throw IspError(SEQPLAN_ISP_ERR_RUNTIME, "cuStreamWaitValue32 failed");
  }
}

// Gather-set buffer of tensor t: the NVLS buffer (unicast mapping) or the heap.
bf16* gath_ptr(Ctx* c, int set, int t) {
  if (c->nvls_ag) return reinterpret_cast<bf16*>(c->nvls_buf.uc + c->nvls_gath_off[set][t]);
  return c->hp<bf16>(c->off_gath[set][t]);
}

// All-gather of tensor t (gate|up together) by pushing this rank's shard into slot `rank` of
// every rank's set buffer (own slot: local copy). NVLS: one store of the shard to the multicast
// address writes every rank's slot.
void push_gather(Ctx* c, int set, int t, cudaStream_t cs) {
  PushJobs J{};
  const size_t gbase = c->nvls_ag ? c->nvls_gath_off[set][t] : c->off_gath[set][t];
  const int64_t r = c->rank;
  int64_t bytes = 0;
  if (t == SEQPLAN_W_GATE) {
    const int64_t B = kGuBlock, H = c->H, rpr = c->I / c->world;
    for (int which = 0; which < 2; ++which) {
      PushJob& j = J.j[which];
      j.src = reinterpret_cast<const char*>(c->wshard(which ? SEQPLAN_W_UP : SEQPLAN_W_GATE));
      j.src_q = 0;
      j.dst_off = int64_t(gbase) + ((r * rpr / B) * 2 * B + which * B) * H * 2;
      j.blk = B * H * 2;
      j.src_stride = B * H * 2;
      j.dst_stride = 2 * B * H * 2;
      j.nblk = rpr / B;
    }
    J.n = 2;
    bytes = 2 * rpr * H * 2;
  } else {
    const int64_t sh = c->shard(t);
    J.j[0] = PushJob{reinterpret_cast<const char*>(c->wshard(t)), 0, int64_t(gbase) + r * sh * 2, sh * 2, 0, 0, 1};
    J.n = 1;
    bytes = sh * 2;
  }
  KTimer kt(c, cs, SEQPLAN_K_ALL_GATHER, 0, double(c->world - 1) * double(bytes));
  if (c->nvls_ag)
    ISP_LAUNCH(1, nvls_push(J, reinterpret_cast<char*>(c->nvls_buf.mcva), cs, c->ag_ctas));
  else
    ISP_LAUNCH(1, push_copy(J, c->peers_at(0), c->world, c->rank, cs, c->ag_ctas, c->ag_kind));
  signal_peers(c, cs, ag_flag(c, set, t, c->rank));
}

// The set's buffers become this pass's gathered weights; with push == true the pushes of the
// given tensors are issued on the comm stream (in order).
void push_gather_set(Ctx* c, int set, const int* order, int n, bool push) {
  for (int i = 0; i < n; ++i) c->gathered[order[i]] = gath_ptr(c, set, order[i]);
  if (!push) return;
  Span sp(c, c->comm, 1, SEQPLAN_EV_ALL_GATHER, set);
  for (int i = 0; i < n; ++i) push_gather(c, set, order[i], c->comm);
}

// Reduce-scatter staging of tensor t's partial: slice q of this rank's partial -> slot `rank`
// of owner q's staging buffer, then the owner's flag. (Own slice: local copy.)
void push_rs(Ctx* c, int t, cudaStream_t cs) {
  if (c->nvls && nvls_tensor(t)) {  // nothing moves: publish that this rank's partial is complete
    Span sp(c, cs, 1, SEQPLAN_EV_REDUCE_SCATTER, t);
    signal_peers(c, cs, rs_flag(c, t, c->rank));
    return;
  }
  PushJobs J{};
  const int64_t r = c->rank, H = c->H, p = c->world;
  const char* part = c->hp<char>(c->off_part[t]);
  int64_t bytes = 0;
  if (t == SEQPLAN_W_GATE) {
    const int64_t B = kGuBlock, rpr = c->I / p, slot = 2 * rpr * H * 2;  // [gate rpr x H | up rpr x H]
    for (int which = 0; which < 2; ++which) {
      PushJob& j = J.j[which];
      j.src = part + which * B * H * 2;
      j.src_q = (rpr / B) * 2 * B * H * 2;
      j.dst_off = int64_t(c->off_stage[t]) + r * slot + which * rpr * H * 2;
      j.blk = B * H * 2;
      j.src_stride = 2 * B * H * 2;
      j.dst_stride = B * H * 2;
      j.nblk = rpr / B;
    }
    J.n = 2;
    bytes = slot;
  } else {
    const bool norm = (t == SEQPLAN_W_NORM1 || t == SEQPLAN_W_NORM2);
    const int64_t esz = norm ? 4 : 2, sh = c->shard(t);
    J.j[0] = PushJob{part, sh * esz, int64_t(c->off_stage[t]) + r * sh * esz, sh * esz, 0, 0, 1};
    J.n = 1;
    bytes = sh * esz;
  }
  Span sp(c, cs, 1, SEQPLAN_EV_REDUCE_SCATTER, t);
  KTimer kt(c, cs, SEQPLAN_K_REDUCE_SCATTER, 0, double(p - 1) * double(bytes));
  ISP_LAUNCH(1, push_copy(J, c->peers_at(0), c->world, c->rank, cs, c->rs_ctas, kPushLsu));
  signal_peers(c, cs, rs_flag(c, t, c->rank));
}

// Owner side: wait for every peer's slice, then the fp32 reduction + cast/scale (fixed rank order).
void reduce_pushed(Ctx* c, int t, cudaStream_t st) {
  wait_peers(c, st, [&](int q) { return rs_flag(c, t, q); });
  if (c->nvls && nvls_tensor(t)) {  // every rank's partial complete: reduce this rank's slices in the switch
    nvls_reduce(c, t, st);
    return;
  }
  PeerPtrs src{};
  const bool norm = (t == SEQPLAN_W_NORM1 || t == SEQPLAN_W_NORM2);
  if (t == SEQPLAN_W_GATE) {
    const int64_t half = (c->I / c->world) * c->H, slot = 2 * half;
    bf16* stg = c->hp<bf16>(c->off_stage[t]);
    for (int q = 0; q < c->world; ++q) src.p[q] = stg + q * slot;
    ISP_LAUNCH(1, reduce_scatter_pull(src, c->world, 0, half, false, 1.0f, c->accum ? 1 : 0, c->grad[SEQPLAN_W_GATE], st, c->red_ctas));
    for (int q = 0; q < c->world; ++q) src.p[q] = stg + q * slot + half;
    ISP_LAUNCH(1, reduce_scatter_pull(src, c->world, 0, half, false, 1.0f, c->accum ? 1 : 0, c->grad[SEQPLAN_W_UP], st, c->red_ctas));
  } else {
    const int64_t sh = c->shard(t), esz = norm ? 4 : 2;
    char* stg = c->hp<char>(c->off_stage[t]);
    for (int q = 0; q < c->world; ++q) src.p[q] = stg + q * sh * esz;
    ISP_LAUNCH(1, reduce_scatter_pull(src, c->world, 0, sh, norm, 1.0f, c->accum ? 1 : 0, c->grad[t], st, c->red_ctas));
  }
}

// Backward re-gather order: the backward's first consumer first; a = 1 re-runs the forward
// first, so forward order then.
const int* bwd_gather_order(const Ctx* c) {
  static const int bwd_order[] = {SEQPLAN_W_DOWN, SEQPLAN_W_GATE, SEQPLAN_W_NORM2, SEQPLAN_W_O, SEQPLAN_W_QKV, SEQPLAN_W_NORM1};
  static const int rec_order[] = {SEQPLAN_W_NORM1, SEQPLAN_W_QKV, SEQPLAN_W_O, SEQPLAN_W_NORM2, SEQPLAN_W_GATE, SEQPLAN_W_DOWN};
  return c->recompute ? rec_order : bwd_order;
}

// Copy-engine mode: queue the backward re-gather on the comm stream behind the forward set (no SM
// is used; the comm stream is otherwise idle until the first reduce-scatter).
void prefetch_bwd_set(Ctx* c) {
  if (c->world == 1 || c->group_mode || c->push_mode() || c->skip_comm() || c->bwd_prefetched || c->no_bwd_prefetch)
    return;
  gather_pipelined(c, bwd_gather_order(c), 6, c->comm, 1);
  c->bwd_prefetched = true;
}

// The QKV GEMM sliced by weight-shard source (fwd_phase1): own rows from the working shard first.
bool qkv_sliced(const Ctx* c) {
  return c->world > 1 && !c->group_mode && !c->fused_a2a && !c->ce_a2a && !c->skip_comm() && c->qkv_slice &&
         (3 * c->H / c->world) % 128 == 0;
}
// ... and its peer slices' B operands TMA-loaded from the peers' working shards over NVLink: the
// forward all-gather of Wqkv is fused into the GEMM (nothing is gathered for it).
bool qkv_ag_in_gemm(const Ctx* c) { return c->ag_gemm && qkv_sliced(c); }

// Only the tensors the first GEMM needs (norm1, Wqkv) are gathered at step start on the
// single-block transport paths; the rest of the forward set and the backward set follow the
// Q|K|V all-to-all (issue_gather_tail), which otherwise shares NVLink with them: 7B-32K p = 4,
// A2A L0 0.48 ms under the gathers vs 0.22 ms alone (profiles/r2/timeline_7b_s32k_p4.txt). The
// tail still has the whole attention forward to land before its first consumer (Wo).
bool defer_gather_tail(const Ctx* c) {
  return c->defer_gathers && c->world > 1 && !c->group_mode && !c->skip_comm() && !c->fused_a2a && !c->ce_a2a &&
         !c->defer_bwd_set && !c->recompute;
}

void fwd_issue_gathers(Ctx* c, cudaStream_t st) {
  c->tail_n = 0;
  if (c->world == 1) {
    for (int t : {SEQPLAN_W_NORM1, SEQPLAN_W_QKV, SEQPLAN_W_O, SEQPLAN_W_NORM2, SEQPLAN_W_GATE, SEQPLAN_W_DOWN})
      gather_weight(c, t, st);
    return;
  }
  cudaStream_t cs = c->group_mode ? st : c->comm;
  if (!c->group_mode) {  // comm stream starts after the caller's prior work
    ISP_CUDA(cudaEventRecord(c->ev_start, st));
    ISP_CUDA(cudaStreamWaitEvent(cs, c->ev_start, 0));
  }
  const int fo[] = {SEQPLAN_W_NORM1, SEQPLAN_W_QKV, SEQPLAN_W_O, SEQPLAN_W_NORM2, SEQPLAN_W_GATE, SEQPLAN_W_DOWN};
  const int fo_ag[] = {SEQPLAN_W_NORM1, SEQPLAN_W_O, SEQPLAN_W_NORM2, SEQPLAN_W_GATE, SEQPLAN_W_DOWN};
  const bool ag = qkv_ag_in_gemm(c);
  const int* f = ag ? fo_ag : fo;
  const int nf = ag ? 5 : 6;
  const bool defer = defer_gather_tail(c) && !(c->push_mode() && c->push_skip());
  const int head = defer ? (ag ? 1 : 2) : nf;
  for (int i = head; i < nf; ++i) c->tail[c->tail_n++] = f[i];
  if (c->push_mode()) {
    // forward set, then the backward re-gather into the second set (its buffers are free since
    // the step-start barrier), so the backward never waits for weights
    const int bo[] = {SEQPLAN_W_DOWN, SEQPLAN_W_GATE, SEQPLAN_W_NORM2, SEQPLAN_W_O, SEQPLAN_W_QKV, SEQPLAN_W_NORM1};
    c->gather_set = 0;
    push_gather_set(c, 0, f, head, !c->push_skip());
    if (!c->push_skip() && !c->defer_bwd_set && !defer) push_gather_set(c, 1, bo, 6, true);
    for (int t : fo) c->gathered[t] = gath_ptr(c, 0, t);
    return;
  }
  if (!c->group_mode) {
    c->evset = 0;
    gather_pipelined(c, f, head, cs);
    if (!c->defer_bwd_set && !defer) prefetch_bwd_set(c);
    return;
  }
  for (int t : {SEQPLAN_W_NORM1, SEQPLAN_W_QKV, SEQPLAN_W_O, SEQPLAN_W_NORM2, SEQPLAN_W_GATE, SEQPLAN_W_DOWN})
    gather_weight(c, t, cs);
}

// The deferred part of fwd_issue_gathers, behind the work already queued on st (the all-to-all).
void issue_gather_tail(Ctx* c, cudaStream_t st) {
  if (c->tail_n == 0) return;
  ISP_CUDA(cudaEventRecord(c->ev_tail, st));
  ISP_CUDA(cudaStreamWaitEvent(c->comm, c->ev_tail, 0));
  if (c->push_mode()) {
    const int bo[] = {SEQPLAN_W_DOWN, SEQPLAN_W_GATE, SEQPLAN_W_NORM2, SEQPLAN_W_O, SEQPLAN_W_QKV, SEQPLAN_W_NORM1};
    {
      Span sp(c, c->comm, 1, SEQPLAN_EV_ALL_GATHER, 0);
      for (int i = 0; i < c->tail_n; ++i) push_gather(c, 0, c->tail[i], c->comm);
    }
    Span sp(c, c->comm, 1, SEQPLAN_EV_ALL_GATHER, 1);
    for (int t : bo) push_gather(c, 1, t, c->comm);
  } else {
    gather_pipelined(c, c->tail, c->tail_n, c->comm);
    prefetch_bwd_set(c);
  }
  c->tail_n = 0;
}

void wait_gathered(Ctx* c, int t, cudaStream_t st) {
  if (c->world == 1 || c->group_mode) return;
  if (c->push_mode()) {
    if (!c->push_skip()) wait_peers(c, st, [&](int q) { return ag_flag(c, c->gather_set, t, q); });
    return;
  }
  if (c->skip_comm() && c->gathered[t] == c->pregathered[t] && c->pregathered[t]) return;
  for (int q = 0; q < c->world; ++q) ISP_CUDA(cudaStreamWaitEvent(st, c->ev_tq[c->evset][t][q], 0));
}

// QKV GEMM epilogue applies RoPE (rotate-half, position rank*T + row) to q and k before the bf16
// store, on the token layout [T, 3H] kept locally.
void set_rope_epilogue(Ctx* c, GemmArgs& g) {
  g.push_T = static_cast<int>(c->T);
  g.push_rank = c->rank;
  g.push_parts = 3;
  g.push_H = static_cast<int>(c->H);
  g.push_Hl = static_cast<int>(c->Hl);
  g.push_d = static_cast<int>(c->d);
  g.rope_cos = c->cos_t;
  g.rope_sin = c->sin_t;
  g.rope_parts = 2;
}

void fwd_phase1(Ctx* c, const bf16* x, cudaStream_t st) {
  Span sp(c, st, 0, SEQPLAN_EV_FORWARD, 0);
  const int T = static_cast<int>(c->T), H = static_cast<int>(c->H);
  wait_gathered(c, SEQPLAN_W_NORM1, st);
  ISP_EW(1, 4.0 * T * H, rmsnorm_fwd(x, c->gathered[SEQPLAN_W_NORM1], c->n1, c->rstd1, T, H, c->eps, st, c->num_sms));
  const int64_t n_own = 3 * c->H / c->world;  // rows of Wqkv in each rank's shard
  if (qkv_sliced(c)) {
    // The step's first gather consumer, sliced by weight-shard source: this rank's own rows of
    // Wqkv are multiplied straight from its working shard while the peers' rows are in flight,
    // the rest once they have landed (unsliced, the GEMM waits for every shard).
    const int64_t r0 = c->rank * n_own;
    bf16* out = qkv_tok_buf(c);
    auto slice = [&](const bf16* w, int64_t col0, int64_t ncols) {
      if (ncols <= 0) return;
      GemmArgs g;
      g.M = T; g.N = static_cast<int>(ncols); g.K = H;
      g.out = out + col0; g.ldo = 3 * H;
      set_rope_epilogue(c, g);  // RoPE on q, k from the fp32 accumulator (one bf16 rounding)
      g.rope_col0 = static_cast<int>(col0);
      gemm(c, {c->n1, H, false}, {w, H, false}, g, EPI_BF16, st);
    };
    slice(c->wshard(SEQPLAN_W_QKV), r0, n_own);
    if (qkv_ag_in_gemm(c)) {  // peers' rows straight from their working shards (TMA over NVLink)
      for (int k = 1; k < c->world; ++k) {
        const int q = (c->rank + k) % c->world;
        slice(c->peer<bf16>(q, c->off_wshard[SEQPLAN_W_QKV]), q * n_own, n_own);
      }
      return;
    }
    wait_gathered(c, SEQPLAN_W_QKV, st);
    const bf16* wq = c->gathered[SEQPLAN_W_QKV];
    slice(wq, 0, r0);
    slice(wq + (r0 + n_own) * H, r0 + n_own, 3 * H - r0 - n_own);
    return;
  }
  wait_gathered(c, SEQPLAN_W_QKV, st);
  GemmArgs g;
  g.M = T; g.N = 3 * H; g.K = H;
  g.out = c->world == 1 ? static_cast<void*>(c->qkv_heads) : static_cast<void*>(qkv_tok_buf(c));
  g.ldo = 3 * H;
  if (c->fused_a2a && !c->skip_comm()) {  // Ulysses all-to-all + RoPE fused into the epilogue (NVLink stores)
    set_push(c, g, c->off_qkv_heads, 3);
    g.rope_cos = c->cos_t;
    g.rope_sin = c->sin_t;
    g.rope_parts = 2;
  } else {  // RoPE in the epilogue, token layout kept locally (the all-to-all is a pure permutation)
    set_rope_epilogue(c, g);
  }
  gemm(c, {c->n1, H, false}, {c->gathered[SEQPLAN_W_QKV], H, false}, g, EPI_BF16, st);
}

AttnTensors attn_tensors(Ctx* c) {
  AttnTensors t{};
  const int64_t ldq = 3 * c->Hl;
  t.q = c->qkv_heads;
  t.k = c->qkv_heads + c->Hl;
  t.v = c->qkv_heads + 2 * c->Hl;
  t.ld_qkv = ldq;
  t.o = c->world == 1 ? c->o_tok : c->hp<bf16>(c->off_o_heads);
  t.ld_o = c->Hl;
  t.lse = c->lse;
  t.S = static_cast<int>(c->S);
  t.heads = static_cast<int>(c->Dl);
  t.d = static_cast<int>(c->d);
  return t;
}

void fwd_phase2(Ctx* c, cudaStream_t st) {
  if (c->world > 1 && !c->skip_comm() && c->ce_a2a) {
    Span sp(c, st, 0, SEQPLAN_EV_ALL_TO_ALL, 0);
    KTimer kt(c, st, SEQPLAN_K_ALL_TO_ALL, 0, double(c->world - 1) / double(c->world) * double(c->T) * 3 * double(c->H) * 2);
    a2a_ce_to_heads(c, c->off_qkv_tok, 3, c->qkv_heads, st);
  } else if (c->world > 1 && !c->skip_comm() && !c->fused_a2a) {
    Span sp(c, st, 0, SEQPLAN_EV_ALL_TO_ALL, 0);
    KTimer kt(c, st, SEQPLAN_K_ALL_TO_ALL, 0, double(c->world - 1) / double(c->world) * double(c->T) * 3 * double(c->H) * 2);
    ISP_LAUNCH(1, a2a_tokens_to_heads(c->peers_at(c->off_qkv_tok), c->world, c->rank, static_cast<int>(c->T),
                                 static_cast<int>(c->H), 3, c->qkv_heads, c->cos_t, c->sin_t,
                                 static_cast<int>(c->d), 0, st, kA2ACtas));
  }
  issue_gather_tail(c, st);
  Span sp(c, st, 0, SEQPLAN_EV_FORWARD, 1);
  KTimer kt(c, st, SEQPLAN_K_ATTN_FWD, 2.0 * double(c->S) * double(c->S) * double(c->Hl), 0);
  AttnTensors at = attn_tensors(c);
  if (c->fused_a2a && !c->skip_comm())  // O rows also stream to the owner of each token
    at.push = attn_push(c, c->off_o_tok, c->H, int64_t(c->rank) * c->Hl, 0, 0, 0);
  ISP_LAUNCH(1, attention_fwd(at, st, c->num_sms));
}

void fwd_phase3(Ctx* c, const bf16* x, bf16* y, cudaStream_t st) {
  issue_gather_tail(c, st);  // no-op after fwd_phase2
  const int T = static_cast<int>(c->T), H = static_cast<int>(c->H), I = static_cast<int>(c->I);
  if (c->world > 1 && !c->skip_comm() && c->ce_a2a) {
    Span sp(c, st, 0, SEQPLAN_EV_ALL_TO_ALL, 1);
    KTimer kt(c, st, SEQPLAN_K_ALL_TO_ALL, 0, double(c->world - 1) / double(c->world) * double(c->T) * 1 * double(c->H) * 2);
    a2a_ce_to_tokens(c, c->off_o_heads, 1, c->o_tok, st);
  } else if (c->world > 1 && !c->skip_comm() && !c->fused_a2a) {
    Span sp(c, st, 0, SEQPLAN_EV_ALL_TO_ALL, 1);
    KTimer kt(c, st, SEQPLAN_K_ALL_TO_ALL, 0, double(c->world - 1) / double(c->world) * double(c->T) * 1 * double(c->H) * 2);
    ISP_LAUNCH(1, a2a_heads_to_tokens(c->peers_at(c->off_o_heads), c->world, c->rank, T, H, 1, c->o_tok, c->cos_t,
                                 c->sin_t, static_cast<int>(c->d), 0, st, kA2ACtas));
  }
  Span sp(c, st, 0, SEQPLAN_EV_FORWARD, 2);
  wait_gathered(c, SEQPLAN_W_O, st);
  {
    GemmArgs g;
    g.M = T; g.N = H; g.K = H;
    g.out = c->h; g.ldo = H;
    g.resid = x; g.ldr = H;
    gemm(c, {c->o_tok, H, false}, {c->gathered[SEQPLAN_W_O], H, false}, g, EPI_BF16_RESID, st);
  }
  if (!c->recomputing) release_weight(c, SEQPLAN_W_O, st);
  wait_gathered(c, SEQPLAN_W_NORM2, st);
  ISP_EW(1, 4.0 * T * H, rmsnorm_fwd(c->h, c->gathered[SEQPLAN_W_NORM2], c->n2, c->rstd2, T, H, c->eps, st, c->num_sms));
  c->gu = static_cast<bf16*>(pool_alloc(c, int64_t(T) * 2 * I * 2, seqplan::AllocTag::MlpIntermediate, st));
  c->a = static_cast<bf16*>(pool_alloc(c, int64_t(T) * I * 2, seqplan::AllocTag::MlpIntermediate, st));
  wait_gathered(c, SEQPLAN_W_GATE, st);
  {
    GemmArgs g;
    g.M = T; g.N = 2 * I; g.K = H;
    g.out = c->gu; g.ldo = 2 * I;
    g.out2 = c->a; g.ldo2 = I;
    gemm(c, {c->n2, H, false}, {c->gathered[SEQPLAN_W_GATE], H, false}, g, EPI_SWIGLU, st);
  }
  // recomputation (a = 1) stops here: y is not needed again and the weights stay for the backward
  if (c->recomputing) return;
  release_weight(c, SEQPLAN_W_GATE, st);
  wait_gathered(c, SEQPLAN_W_DOWN, st);
  {
    GemmArgs g;
    g.M = T; g.N = H; g.K = I;
    g.out = y; g.ldo = H;
    g.resid = c->h; g.ldr = H;
    gemm(c, {c->a, I, false}, {c->gathered[SEQPLAN_W_DOWN], I, false}, g, EPI_BF16_RESID, st);
  }
  release_weight(c, SEQPLAN_W_DOWN, st);
  release_weight(c, SEQPLAN_W_QKV, st);
  release_weight(c, SEQPLAN_W_NORM1, st);
  release_weight(c, SEQPLAN_W_NORM2, st);
}

// ---------------------------------------------------------------------------------
// backward phases
// ---------------------------------------------------------------------------------
void bwd_issue_gathers(Ctx* c, cudaStream_t st) {
  // a = 1: the recomputed forward consumes the re-gathered weights first, in forward order
  const int* order = bwd_gather_order(c);
  if (c->bwd_prefetched) {  // copy-engine re-gather already queued at step start
    for (int i = 0; i < 6; ++i) {
      c->gathered[order[i]] = c->pre_bwd[order[i]];
      c->pre_bwd[order[i]] = nullptr;
    }
    c->evset = 1;
    c->bwd_prefetched = false;
    return;
  }
  c->evset = 0;
  if (c->world == 1) {
    for (int i = 0; i < 6; ++i) gather_weight(c, order[i], st);
    return;
  }
  if (c->push_mode()) {  // pushed at the start of the step (fwd_issue_gathers)
    c->gather_set = 1;
    for (int i = 0; i < 6; ++i) c->gathered[order[i]] = gath_ptr(c, 1, order[i]);
    return;
  }
  cudaStream_t cs = c->group_mode ? st : c->comm;
  if (!c->group_mode) {
    ISP_CUDA(cudaEventRecord(c->ev_start, st));
    ISP_CUDA(cudaStreamWaitEvent(cs, c->ev_start, 0));
  }
  if (!c->group_mode) {
    gather_pipelined(c, order, 6, cs);
    return;
  }
  for (int i = 0; i < 6; ++i) gather_weight(c, order[i], cs);
}

// Weight-gradient destination: fp32 grad shard directly at p = 1, bf16 partial in the heap otherwise.
void wgrad(Ctx* c, int t, const GemmOperand& A, const GemmOperand& B, int M, int N, int K, cudaStream_t st) {
  GemmArgs g;
  g.M = M; g.N = N; g.K = K;
  if (c->world == 1) {
    g.out = c->grad[t];
    g.ldo = N;
    g.accumulate = c->accum ? 1 : 0;
    if (t == SEQPLAN_W_GATE) {
      g.interleave64 = 1;
      g.out_b = c->grad[SEQPLAN_W_UP];
    }
    gemm(c, A, B, g, EPI_F32, st);
  } else {
    g.out = part_bf16(c, t);
    g.ldo = N;
    gemm(c, A, B, g, EPI_BF16, st);
  }
}

// After the G-W of tensor t: hand its partial to the comm stream for the reduce-scatter.
// Copy-engine staging of this rank's slice of every rank's partial (rank order) on the comm
// stream; the fp32 reduction + cast/scale runs on the reduction stream as soon as the slices land
// (schedule_rs, early_reduce) or at the end of the step on the compute stream (reduce_staged).
void stage_rs(Ctx* c, int t, cudaStream_t cs) {
  const bool norm = (t == SEQPLAN_W_NORM1 || t == SEQPLAN_W_NORM2);
  const int64_t esz = norm ? 4 : 2;
  const int64_t H = c->H, p = c->world;
  Span sp(c, cs, 1, SEQPLAN_EV_REDUCE_SCATTER, t);
  if (t == SEQPLAN_W_GATE) {
    const int64_t rpr = c->I / p, B = kGuBlock, slot = 2 * rpr * H;  // [gate rpr x H | up rpr x H]
    KTimer kt(c, cs, SEQPLAN_K_REDUCE_SCATTER, 0, double(p - 1) * double(slot) * 2);
    bf16* stg = static_cast<bf16*>(pool_alloc(c, p * slot * 2, seqplan::AllocTag::CommBuffer, cs));
    fan_out(c, cs, [&](int q, cudaStream_t qs) {
      for (int which = 0; which < 2; ++which) {
        const bf16* src = c->peer<bf16>(q, c->off_part[SEQPLAN_W_GATE]) + ((c->rank * rpr / B) * 2 * B + which * B) * H;
        ISP_CUDA(cudaMemcpy2DAsync(stg + q * slot + which * rpr * H, size_t(B * H * 2), src, size_t(2 * B * H * 2),
                                   size_t(B * H * 2), size_t(rpr / B), cudaMemcpyDefault, qs));
      }
    });
    c->stage[t] = stg;
  } else {
    const int64_t sh = c->shard(t);
    KTimer kt(c, cs, SEQPLAN_K_REDUCE_SCATTER, 0, double(p - 1) * double(sh) * double(esz));
    char* stg = static_cast<char*>(pool_alloc(c, p * sh * esz, seqplan::AllocTag::CommBuffer, cs));
    fan_out(c, cs, [&](int q, cudaStream_t qs) {
      ISP_CUDA(cudaMemcpyAsync(stg + q * sh * esz, c->peer<char>(q, c->off_part[t]) + c->rank * sh * esz,
                               size_t(sh * esz), cudaMemcpyDefault, qs));
    });
    c->stage[t] = stg;
  }
  ISP_CUDA(cudaEventRecord(c->ev_staged[t], cs));
}

void reduce_staged(Ctx* c, int t, cudaStream_t st) {
  if (!c->stage[t]) return;
  ISP_CUDA(cudaStreamWaitEvent(st, c->ev_staged[t], 0));
  const bool norm = (t == SEQPLAN_W_NORM1 || t == SEQPLAN_W_NORM2);
  PeerPtrs src{};
  if (t == SEQPLAN_W_GATE) {
    const int64_t slot = 2 * (c->I / c->world) * c->H, half = slot / 2;
    bf16* stg = static_cast<bf16*>(c->stage[t]);
    for (int q = 0; q < c->world; ++q) src.p[q] = stg + q * slot;
    ISP_LAUNCH(1, reduce_scatter_pull(src, c->world, 0, half, false, 1.0f, c->accum ? 1 : 0, c->grad[SEQPLAN_W_GATE], st, c->red_ctas));
    for (int q = 0; q < c->world; ++q) src.p[q] = stg + q * slot + half;
    ISP_LAUNCH(1, reduce_scatter_pull(src, c->world, 0, half, false, 1.0f, c->accum ? 1 : 0, c->grad[SEQPLAN_W_UP], st, c->red_ctas));
  } else {
    const int64_t sh = c->shard(t), esz = norm ? 4 : 2;
    char* stg = static_cast<char*>(c->stage[t]);
    for (int q = 0; q < c->world; ++q) src.p[q] = stg + q * sh * esz;
    ISP_LAUNCH(1, reduce_scatter_pull(src, c->world, 0, sh, norm, 1.0f, c->accum ? 1 : 0, c->grad[t], st, c->red_ctas));
  }
  c->pool->free(c->stage[t], st);
  c->stage[t] = nullptr;
}

void schedule_rs(Ctx* c, int t, cudaStream_t st) {
  if (c->world == 1 || c->group_mode || c->skip_comm()) return;
  ISP_CUDA(cudaEventRecord(c->ev_wgrad[t], st));
  ISP_CUDA(cudaStreamWaitEvent(c->comm, c->ev_wgrad[t], 0));
  if (c->push_mode() && !c->rs_ce) {
    push_rs(c, t, c->comm);
  } else {
    barrier(c, c->comm, true);
    stage_rs(c, t, c->comm);
  }
  if (c->early_reduce) {  // reduce this tensor as soon as its slices land, beside the compute stream
    ISP_CUDA(cudaEventRecord(c->ev_rs_sent[t], c->comm));
    ISP_CUDA(cudaStreamWaitEvent(c->red, c->ev_rs_sent[t], 0));
    if (c->push_mode() && !c->rs_ce) reduce_pushed(c, t, c->red);
    else reduce_staged(c, t, c->red);
  }
}

void bwd_phase1(Ctx* c, const bf16* dy, cudaStream_t st) {
  const int T = static_cast<int>(c->T), H = static_cast<int>(c->H), I = static_cast<int>(c->I);
  const bool selective = !(c->flags & SEQPLAN_ISP_FLAG_FUSED_BWD);
  // ---- down projection: G-W first (its RS overlaps the rest), then G-X ----
  wait_gathered(c, SEQPLAN_W_DOWN, st);
  {
    Span sp(c, st, 0, SEQPLAN_EV_GRAD_WEIGHT, 3);
    wgrad(c, SEQPLAN_W_DOWN, {dy, H, true}, {c->a, I, true}, H, I, T, st);
  }
  if (selective) schedule_rs(c, SEQPLAN_W_DOWN, st);
  // ---- down dgrad, then the SwiGLU backward. SEQPLAN_ISP_FUSE_SWIGLU_BWD=1 computes dgu in the
  // GEMM epilogue from da (never stored) and gu instead: measured no faster at 7B-4K (0.322 ms
  // fused vs 0.242 + 0.084 ms; the one-row-per-thread gu/dgu traffic slows the epilogue enough to
  // stall the MMAs), so the separate HBM-bound kernel stays the default ----
  bf16* dgu = static_cast<bf16*>(pool_alloc(c, int64_t(T) * 2 * I * 2, seqplan::AllocTag::MlpIntermediate, st));
  if (c->fuse_swiglu_bwd) {
    Span sp(c, st, 0, SEQPLAN_EV_GRAD_INPUT, 3);
    GemmArgs g;
    g.M = T; g.N = I; g.K = H;
    g.out = dgu; g.ldo = 2 * I;
    g.resid = c->gu; g.ldr = 2 * I;
    gemm(c, {dy, H, false}, {c->gathered[SEQPLAN_W_DOWN], I, true}, g, EPI_SWIGLU_BWD, st);
  } else {
    bf16* da = static_cast<bf16*>(pool_alloc(c, int64_t(T) * I * 2, seqplan::AllocTag::MlpIntermediate, st));
    {
      Span sp(c, st, 0, SEQPLAN_EV_GRAD_INPUT, 3);
      GemmArgs g;
      g.M = T; g.N = I; g.K = H;
      g.out = da; g.ldo = I;
      gemm(c, {dy, H, false}, {c->gathered[SEQPLAN_W_DOWN], I, true}, g, EPI_BF16, st);
    }
    ISP_EW(1, 10.0 * T * I, swiglu_bwd(da, c->gu, dgu, T, I, st, c->num_sms));
    c->pool->free(da, st);
  }
  release_weight(c, SEQPLAN_W_DOWN, st);
  c->pool->free(c->a, st);
  c->a = nullptr;
  c->pool->free(c->gu, st);
  c->gu = nullptr;
  // ---- gate|up ----
  wait_gathered(c, SEQPLAN_W_GATE, st);
  {
    Span sp(c, st, 0, SEQPLAN_EV_GRAD_WEIGHT, 2);
    wgrad(c, SEQPLAN_W_GATE, {dgu, 2 * I, true}, {c->n2, H, true}, 2 * I, H, T, st);
  }
  if (selective) schedule_rs(c, SEQPLAN_W_GATE, st);
  {
    Span sp(c, st, 0, SEQPLAN_EV_GRAD_INPUT, 2);
    GemmArgs g;
    g.M = T; g.N = H; g.K = 2 * I;
    g.out = c->dn; g.ldo = H;
    gemm(c, {dgu, 2 * I, false}, {c->gathered[SEQPLAN_W_GATE], H, true}, g, EPI_BF16, st);
  }
  release_weight(c, SEQPLAN_W_GATE, st);
  c->pool->free(dgu, st);
  // ---- norm2 backward: dh = dy + d(norm2) ----
  wait_gathered(c, SEQPLAN_W_NORM2, st);
  float* dg2 = c->world == 1 ? c->grad[SEQPLAN_W_NORM2] : c->hp<float>(c->off_part[SEQPLAN_W_NORM2]);
  if (c->world > 1 || !c->accum) ISP_CUDA(cudaMemsetAsync(dg2, 0, sizeof(float) * H, st));
  ISP_EW(2, 8.0 * T * H, rmsnorm_bwd(c->h, c->gathered[SEQPLAN_W_NORM2], c->rstd2, c->dn, dy, c->dh, dg2, T, H, st, c->num_sms, c->dg_scratch));
  release_weight(c, SEQPLAN_W_NORM2, st);
  if (selective) schedule_rs(c, SEQPLAN_W_NORM2, st);
  // ---- output projection ----
  wait_gathered(c, SEQPLAN_W_O, st);
  {
    Span sp(c, st, 0, SEQPLAN_EV_GRAD_WEIGHT, 1);
    wgrad(c, SEQPLAN_W_O, {c->dh, H, true}, {c->o_tok, H, true}, H, H, T, st);
  }
  if (selective) schedule_rs(c, SEQPLAN_W_O, st);
  {
    Span sp(c, st, 0, SEQPLAN_EV_GRAD_INPUT, 1);
    GemmArgs g;
    g.M = T; g.N = H; g.K = H;
    g.out = c->world == 1 ? c->dO_heads : c->hp<bf16>(c->off_do_tok);
    g.ldo = H;
    if (c->fused_a2a && !c->skip_comm()) set_push(c, g, c->off_dO_heads, 1);
    gemm(c, {c->dh, H, false}, {c->gathered[SEQPLAN_W_O], H, true}, g, EPI_BF16, st);
  }
  release_weight(c, SEQPLAN_W_O, st);
}

void bwd_phase2(Ctx* c, cudaStream_t st) {
  const int T = static_cast<int>(c->T), H = static_cast<int>(c->H);
  if (c->world > 1 && !c->skip_comm() && c->ce_a2a) {
    Span sp(c, st, 0, SEQPLAN_EV_ALL_TO_ALL, 2);
    KTimer kt(c, st, SEQPLAN_K_ALL_TO_ALL, 0, double(c->world - 1) / double(c->world) * double(c->T) * 1 * double(c->H) * 2);
    a2a_ce_to_heads(c, c->off_do_tok, 1, c->dO_heads, st);
  } else if (c->world > 1 && !c->skip_comm() && !c->fused_a2a) {
    Span sp(c, st, 0, SEQPLAN_EV_ALL_TO_ALL, 2);
    KTimer kt(c, st, SEQPLAN_K_ALL_TO_ALL, 0, double(c->world - 1) / double(c->world) * double(c->T) * 1 * double(c->H) * 2);
    ISP_LAUNCH(1, a2a_tokens_to_heads(c->peers_at(c->off_do_tok), c->world, c->rank, T, H, 1, c->dO_heads, c->cos_t,
                                 c->sin_t, static_cast<int>(c->d), 0, st, kA2ACtas));
  }
  Span sp(c, st, 0, SEQPLAN_EV_GRAD_INPUT, 0);
  AttnTensors t = attn_tensors(c);
  if (c->fused_a2a && !c->skip_comm())  // dq / dk / dv rows stream to the owner of each token
    t.push = attn_push(c, c->off_dqkv_tok, 3 * c->H, 0, int64_t(c->rank) * c->Hl, c->H + int64_t(c->rank) * c->Hl,
                       2 * c->H + int64_t(c->rank) * c->Hl);
  bf16* dqkv = c->world == 1 ? c->dqkv_tok : c->hp<bf16>(c->off_dqkv_heads);
  const int64_t ld = 3 * c->Hl;
  // the inverse RoPE of dq / dk is applied in the backward's epilogue, from fp32 (the all-to-all
  // back to tokens is then a pure permutation)
  t.rope_cos = c->cos_t;
  t.rope_sin = c->sin_t;
  // stored-dS backward: the causal dS tiles of up to ds_ws_gb GiB of heads (at least one head's,
  // up to twice the cap) per key-tile / dQ launch pair; 0 selects the two-role kernel
  void* ws = nullptr;
  if (c->d == 128 && c->ds_ws_gb > 0 && c->S % 128 == 0) {
    const int64_t per_head = attention_bwd_ds_head_bytes(static_cast<int>(c->S));
    const int64_t cap = std::max(c->ds_ws_gb << 30, per_head <= (c->ds_ws_gb << 30) * 2 ? per_head : int64_t(0));
    int64_t g = std::min<int64_t>(c->Dl, cap / per_head);
    if (g * per_head > c->ds_ws_cached) {  // a new segment: only what the device has free (1 GiB kept)
      size_t free_b = 0, total_b = 0;
      ISP_CUDA(cudaMemGetInfo(&free_b, &total_b));
      const int64_t room = std::max<int64_t>(int64_t(free_b) - (int64_t(1) << 30), 0);
      g = std::min<int64_t>(g, std::max(room, c->ds_ws_cached) / per_head);
    }
    if (g > 0) {
      t.ds_ws_bytes = g * per_head;
      ws = t.ds_ws = pool_alloc(c, t.ds_ws_bytes, seqplan::AllocTag::Other, st);
      c->ds_ws_cached = std::max(c->ds_ws_cached, t.ds_ws_bytes);  // the pool keeps the segment
    }
  }
  KTimer kt(c, st, SEQPLAN_K_ATTN_BWD, 4.0 * double(c->S) * double(c->S) * double(c->Hl), 0);
  ISP_LAUNCH(3, attention_bwd(t, c->dO_heads, dqkv, dqkv + c->Hl, dqkv + 2 * c->Hl, ld, c->delta, c->dq_acc, st,
                         c->num_sms));
  if (ws) c->pool->free(ws, st);
}

void bwd_phase3(Ctx* c, const bf16* x, bf16* dx, cudaStream_t st) {
  const int T = static_cast<int>(c->T), H = static_cast<int>(c->H);
  const bool selective = !(c->flags & SEQPLAN_ISP_FLAG_FUSED_BWD);
  if (c->world > 1 && !c->skip_comm() && c->ce_a2a) {
    Span sp(c, st, 0, SEQPLAN_EV_ALL_TO_ALL, 3);
    KTimer kt(c, st, SEQPLAN_K_ALL_TO_ALL, 0, double(c->world - 1) / double(c->world) * double(c->T) * 3 * double(c->H) * 2);
    a2a_ce_to_tokens(c, c->off_dqkv_heads, 3, c->dqkv_tok, st);
  } else if (c->world > 1 && !c->skip_comm() && !c->fused_a2a) {
    Span sp(c, st, 0, SEQPLAN_EV_ALL_TO_ALL, 3);
    KTimer kt(c, st, SEQPLAN_K_ALL_TO_ALL, 0, double(c->world - 1) / double(c->world) * double(c->T) * 3 * double(c->H) * 2);
    ISP_LAUNCH(1, a2a_heads_to_tokens(c->peers_at(c->off_dqkv_heads), c->world, c->rank, T, H, 3, c->dqkv_tok,
                                 c->cos_t, c->sin_t, static_cast<int>(c->d), 0, st, kA2ACtas));
  }
  wait_gathered(c, SEQPLAN_W_QKV, st);
  {
    Span sp(c, st, 0, SEQPLAN_EV_GRAD_WEIGHT, 0);
    wgrad(c, SEQPLAN_W_QKV, {c->dqkv_tok, 3 * H, true}, {c->n1, H, true}, 3 * H, H, T, st);
  }
  if (selective) schedule_rs(c, SEQPLAN_W_QKV, st);
  {
    Span sp(c, st, 0, SEQPLAN_EV_GRAD_INPUT, 0);
    GemmArgs g;
    g.M = T; g.N = H; g.K = 3 * H;
    g.out = c->dn; g.ldo = H;
    gemm(c, {c->dqkv_tok, 3 * H, false}, {c->gathered[SEQPLAN_W_QKV], H, true}, g, EPI_BF16, st);
  }
  release_weight(c, SEQPLAN_W_QKV, st);
  wait_gathered(c, SEQPLAN_W_NORM1, st);
  float* dg1 = c->world == 1 ? c->grad[SEQPLAN_W_NORM1] : c->hp<float>(c->off_part[SEQPLAN_W_NORM1]);
  if (c->world > 1 || !c->accum) ISP_CUDA(cudaMemsetAsync(dg1, 0, sizeof(float) * H, st));
  ISP_EW(2, 8.0 * T * H, rmsnorm_bwd(x, c->gathered[SEQPLAN_W_NORM1], c->rstd1, c->dn, c->dh, dx, dg1, T, H, st, c->num_sms, c->dg_scratch));
  release_weight(c, SEQPLAN_W_NORM1, st);
  if (selective) schedule_rs(c, SEQPLAN_W_NORM1, st);
}

// Fused backward (or group mode): every reduce-scatter after the last G-X.
void bwd_reduce_all(Ctx* c, cudaStream_t st) {
  if (c->world == 1) return;
  for (int t : {SEQPLAN_W_DOWN, SEQPLAN_W_GATE, SEQPLAN_W_NORM2, SEQPLAN_W_O, SEQPLAN_W_QKV, SEQPLAN_W_NORM1})
    reduce_scatter_grad(c, t, st);
}

// ---------------------------------------------------------------------------------
// context setup
// ---------------------------------------------------------------------------------
void layout_heap(Ctx* c) {
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off = align_up(off + bytes, 4096);
    return o;
  };
  c->off_flags = take(kFlagBytes);
  for (int t = 0; t < SEQPLAN_W_COUNT; ++t) c->off_wshard[t] = take(size_t(c->shard(t)) * 2);
  if (c->world > 1) {
    c->off_qkv_tok = take(size_t(c->T) * 3 * c->H * 2);
    c->off_o_heads = take(size_t(c->S) * c->Hl * 2);
    c->off_do_tok = take(size_t(c->T) * c->H * 2);
    c->off_dqkv_heads = take(size_t(c->S) * 3 * c->Hl * 2);
    if (c->fused_a2a) {
      c->off_qkv_heads = take(size_t(c->S) * 3 * c->Hl * 2);
      c->off_o_tok = take(size_t(c->T) * c->H * 2);
      c->off_dO_heads = take(size_t(c->S) * c->Hl * 2);
      c->off_dqkv_tok = take(size_t(c->T) * 3 * c->H * 2);
    }
    for (int t : {SEQPLAN_W_QKV, SEQPLAN_W_O, SEQPLAN_W_DOWN}) c->off_part[t] = take(size_t(c->numel(t)) * 2);
    c->off_part[SEQPLAN_W_GATE] = take(size_t(2 * c->I * c->H) * 2);
    c->off_part[SEQPLAN_W_NORM1] = take(size_t(c->H) * 4);
    c->off_part[SEQPLAN_W_NORM2] = take(size_t(c->H) * 4);
    // push transport only: the pinned gather double buffer and the RS staging slots the peers
    // write into (the copy-engine transport takes both from the device pool, per pass)
    if (c->push_mode()) {
      size_t o = 0;  // the NVLS partial buffer's layout (bound only if seqplan_isp_nvls_bind runs)
      for (int t : {SEQPLAN_W_QKV, SEQPLAN_W_O, SEQPLAN_W_GATE, SEQPLAN_W_DOWN}) {
        c->nvls_off[t] = o;
        o += (size_t(t == SEQPLAN_W_GATE ? 2 * c->I * c->H : c->numel(t)) * 2 + 4095) & ~size_t(4095);
      }
      if (c->nvls_pref & 2)
        for (int set = 0; set < 2; ++set)
          for (int t : {SEQPLAN_W_NORM1, SEQPLAN_W_QKV, SEQPLAN_W_O, SEQPLAN_W_NORM2, SEQPLAN_W_GATE, SEQPLAN_W_DOWN}) {
            c->nvls_gath_off[set][t] = o;
            o += (size_t(t == SEQPLAN_W_GATE ? 2 * c->I * c->H : c->numel(t)) * 2 + 4095) & ~size_t(4095);
          }
      c->nvls_bytes = o;
      for (int set = 0; set < 2; ++set)
        for (int t : {SEQPLAN_W_NORM1, SEQPLAN_W_QKV, SEQPLAN_W_O, SEQPLAN_W_NORM2, SEQPLAN_W_GATE, SEQPLAN_W_DOWN})
          c->off_gath[set][t] = take(size_t(t == SEQPLAN_W_GATE ? 2 * c->I * c->H : c->numel(t)) * 2);
      for (int t : {SEQPLAN_W_QKV, SEQPLAN_W_O, SEQPLAN_W_DOWN}) c->off_stage[t] = take(size_t(c->numel(t)) * 2);
      c->off_stage[SEQPLAN_W_GATE] = take(size_t(2 * c->I * c->H) * 2);
      c->off_stage[SEQPLAN_W_NORM1] = take(size_t(c->H) * 4);
      c->off_stage[SEQPLAN_W_NORM2] = take(size_t(c->H) * 4);
    }
  }
  c->heap_bytes = off;
}

// Saved activations of the forward (needed by the backward) and the backward's scratch.
// a = 0: allocated once at setup and kept. a = 1 (activation recomputation, SURVEY.md §8f
// item 3; cost.hpp:139 (34 - 32a)): allocated at the start of each pass and freed at its end, so
// between passes only the block input (the checkpoint) is live, and in a stack, whose layers
// share one pool, one layer's workspace is recycled by the next.
void alloc_acts(Ctx* c, cudaStream_t st) {
  if (c->acts_live) return;
  const int64_t T = c->T, H = c->H, S = c->S, Hl = c->Hl;
  auto A = [&](int64_t bytes) { return pool_alloc(c, bytes, seqplan::AllocTag::Other, st); };
  c->n1 = static_cast<bf16*>(A(T * H * 2));
  c->rstd1 = static_cast<float*>(A(T * 4));
  c->qkv_heads = c->fused_a2a ? c->hp<bf16>(c->off_qkv_heads) : static_cast<bf16*>(A(S * 3 * Hl * 2));
  c->o_tok = c->fused_a2a ? c->hp<bf16>(c->off_o_tok) : static_cast<bf16*>(A(T * H * 2));
  c->h = static_cast<bf16*>(A(T * H * 2));
  c->n2 = static_cast<bf16*>(A(T * H * 2));
  c->rstd2 = static_cast<float*>(A(T * 4));
  c->lse = static_cast<float*>(A(c->Dl * S * 4));
  c->acts_live = true;
}

void alloc_scratch(Ctx* c, cudaStream_t st) {
  if (c->scratch_live) return;
  const int64_t T = c->T, H = c->H, S = c->S, Hl = c->Hl;
  auto A = [&](int64_t bytes) { return pool_alloc(c, bytes, seqplan::AllocTag::Other, st); };
  c->dh = static_cast<bf16*>(A(T * H * 2));
  c->dn = static_cast<bf16*>(A(T * H * 2));
  c->dO_heads = c->fused_a2a ? c->hp<bf16>(c->off_dO_heads) : static_cast<bf16*>(A(S * Hl * 2));
  c->dqkv_tok = c->fused_a2a ? c->hp<bf16>(c->off_dqkv_tok) : static_cast<bf16*>(A(T * 3 * H * 2));
  c->delta = static_cast<float*>(A(c->Dl * S * 4));
  c->dq_acc = static_cast<float*>(A(c->Dl * S * c->d * 4));
  c->dg_scratch = static_cast<float*>(A(int64_t(rmsnorm_bwd_scratch_rows(c->num_sms)) * H * 4));
  c->scratch_live = true;
}

void free_acts(Ctx* c, cudaStream_t st) {
  if (!c->acts_live) return;
  for (void* p : {static_cast<void*>(c->n1), static_cast<void*>(c->rstd1), static_cast<void*>(c->h),
                  static_cast<void*>(c->n2), static_cast<void*>(c->rstd2), static_cast<void*>(c->lse)})
    c->pool->free(p, st);
  if (!c->fused_a2a) {
    c->pool->free(c->qkv_heads, st);
    c->pool->free(c->o_tok, st);
  }
  for (bf16* p : {c->gu, c->a})
    if (p) c->pool->free(p, st);
  c->gu = c->a = nullptr;
  c->acts_live = false;
}

void free_scratch(Ctx* c, cudaStream_t st) {
  if (!c->scratch_live) return;
  for (void* p : {static_cast<void*>(c->dh), static_cast<void*>(c->dn), static_cast<void*>(c->delta),
                  static_cast<void*>(c->dq_acc), static_cast<void*>(c->dg_scratch)})
    c->pool->free(p, st);
  if (!c->fused_a2a) {
    c->pool->free(c->dO_heads, st);
    c->pool->free(c->dqkv_tok, st);
  }
  c->scratch_live = false;
}

void setup(Ctx* c, const seqplan_isp_shape* shape, const seqplan_mempool_policy* policy, int premap_layers) {
  c->H = shape->hidden_dim;
  c->D = shape->heads;
  c->S = shape->seq_len;
  c->I = shape->ffn_dim > 0 ? shape->ffn_dim : seqplan::mlp_intermediate_dim(c->H);
  c->rope_base = shape->rope_base > 0 ? shape->rope_base : 10000.0;
  c->eps = shape->norm_eps > 0 ? static_cast<float>(shape->norm_eps) : 1e-5f;
  if (c->H <= 0 || c->D <= 0 || c->S <= 0 || c->H % c->D)
    throw IspError(SEQPLAN_ISP_ERR_INVALID, "invalid model config: hidden_dim must be divisible by heads");
  c->d = c->H / c->D;
  if (c->world < 1 || c->world > kMaxRanks || c->D % c->world || c->S % c->world)
    throw IspError(SEQPLAN_ISP_ERR_INVALID, "head count and sequence must be divisible by the ISP degree");
  c->T = c->S / c->world;
  c->Hl = c->H / c->world;
  c->Dl = c->D / c->world;
  if ((c->d != 64 && c->d != 128) || c->T % 128 || c->H % 256 || c->I % 256 || (c->I / c->world) % kGuBlock ||
      c->S % 128)
    throw IspError(SEQPLAN_ISP_ERR_UNSUPPORTED,
                   "shape not tiled by the sm_100a kernels (head dim 64/128, S/p % 128, H % 256, I % 256)");
  ISP_CUDA(cudaSetDevice(c->device));
  ISP_CUDA(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, c->device));
  seqplan::MempoolPolicy pol;
  if (policy) {
    pol.pinned_comm_pool = policy->pinned_comm_pool != 0;
    pol.consolidate_every_k_mlp = policy->consolidate_every_k_mlp;
    pol.grad_premap = policy->grad_premap != 0;
    pol.capacity = policy->capacity;
  } else {
    pol.pinned_comm_pool = true;
    pol.grad_premap = true;
  }
  if (c->owns_pool) c->pool->set_policy(pol);

  // Ulysses all-to-all: SM pull kernels after the producer (default), or fused into the producers'
  // epilogues as 16-B remote stores (SEQPLAN_ISP_FUSED_A2A=1). Measured at p = 2/4: the pull is
  // 3-7 % faster end to end (7B-4K/32K) — per-thread 16-B NVLink stores from 32 different rows
  // per warp instruction slow the QKV GEMM and attention epilogues more than the exchange costs.
  const char* fa = std::getenv("SEQPLAN_ISP_FUSED_A2A");
  c->fused_a2a = c->world > 1 && c->d == 128 && fa && std::atoi(fa) != 0;
  if (const char* e = std::getenv("SEQPLAN_ISP_PUSH")) c->push_pref = std::atoi(e) ? 1 : 0;
  if (const char* e = std::getenv("SEQPLAN_ISP_FUSE_SWIGLU_BWD")) c->fuse_swiglu_bwd = std::atoi(e) != 0;
  if (const char* e = std::getenv("SEQPLAN_ISP_BWD_PREFETCH")) c->no_bwd_prefetch = std::atoi(e) == 0;
  if (const char* e = std::getenv("SEQPLAN_ISP_RS_CE")) c->rs_ce = std::atoi(e) != 0;
  if (const char* e = std::getenv("SEQPLAN_ISP_QKV_SLICE")) c->qkv_slice = std::atoi(e) != 0;
  if (const char* e = std::getenv("SEQPLAN_ISP_AG_GEMM")) c->ag_gemm = std::atoi(e) != 0;
  if (const char* e = std::getenv("SEQPLAN_ISP_DS_WS_GB")) c->ds_ws_gb = std::max(0, std::atoi(e));
  if (c->ds_ws_gb < 0) {
    size_t free_b = 0, total_b = 0;
    ISP_CUDA(cudaMemGetInfo(&free_b, &total_b));
    c->ds_ws_gb = std::min<int64_t>(48, int64_t(total_b >> 30) / 4);
  }
  if (const char* e = std::getenv("SEQPLAN_ISP_DEFER_GATHER")) c->defer_gathers = std::atoi(e) != 0;
  if (const char* e = std::getenv("SEQPLAN_ISP_EARLY_REDUCE")) c->early_reduce = std::atoi(e) != 0;
  if (const char* e = std::getenv("SEQPLAN_ISP_A2A_CE")) c->ce_a2a = c->world > 1 && !c->fused_a2a && std::atoi(e) != 0;
  if (const char* e = std::getenv("SEQPLAN_ISP_RS_CTAS")) c->rs_ctas = std::atoi(e) ? std::atoi(e) : 128;
  if (const char* e = std::getenv("SEQPLAN_ISP_AG_CTAS")) c->ag_ctas = std::max(1, std::atoi(e));
  if (const char* e = std::getenv("SEQPLAN_ISP_AG_KIND")) c->ag_kind = std::atoi(e);
  c->red_ctas = c->num_sms * 4;
  if (const char* e = std::getenv("SEQPLAN_ISP_NVLS")) c->nvls_pref = std::atoi(e);
  if (const char* e = std::getenv("SEQPLAN_ISP_RED_CTAS")) c->red_ctas = std::max(1, std::atoi(e));
  if (c->ag_kind == kPushBulkWide) c->gemm_sm_budget = c->num_sms - c->ag_ctas;
  layout_heap(c);
  ISP_CUDA(cudaMalloc(&c->heap, c->heap_bytes));
  ISP_CUDA(cudaMemset(c->heap, 0, kFlagBytes));
  c->peer_heap[c->rank] = c->heap;
  c->peer_opened[c->rank] = false;
  c->error_flag = reinterpret_cast<uint32_t*>(c->heap + 1024);

  // persistent buffers through the pool
  const cudaStream_t s0 = nullptr;
  int64_t grad_bytes = 0;
  for (int t = 0; t < SEQPLAN_W_COUNT; ++t) grad_bytes += (c->shard(t) * 4 + 511) / 512 * 512;
  // a stack's pool owner pre-maps the gradient arena of every layer (grad_premap)
  if (c->owns_pool && !c->pool->premap_grads(grad_bytes * premap_layers))
    throw IspError(SEQPLAN_ISP_ERR_OOM, "grad arena");
  for (int t = 0; t < SEQPLAN_W_COUNT; ++t) {
    c->master[t] = static_cast<float*>(pool_alloc(c, c->shard(t) * 4, seqplan::AllocTag::Other, s0));
    c->grad[t] = static_cast<float*>(pool_alloc(c, c->shard(t) * 4, seqplan::AllocTag::Grad, s0));
  }
  if (c->world == 1)
    c->wgu_local = static_cast<bf16*>(pool_alloc(c, 2 * c->I * c->H * 2, seqplan::AllocTag::Other, s0));
  const int64_t T = c->T, H = c->H, S = c->S, Hl = c->Hl;
  auto A = [&](int64_t bytes, seqplan::AllocTag tag = seqplan::AllocTag::Other) {
    return pool_alloc(c, bytes, tag, s0);
  };
  c->cos_t = static_cast<float*>(A(S * (c->d / 2) * 4));
  c->sin_t = static_cast<float*>(A(S * (c->d / 2) * 4));
  (void)T; (void)H; (void)Hl;
  if (!c->recompute) {  // a = 0: the forward's saved tensors and the backward scratch live in the context
    alloc_acts(c, s0);
    alloc_scratch(c, s0);
  }

  ISP_CUDA(cudaStreamCreateWithFlags(&c->comm, cudaStreamNonBlocking));
  ISP_CUDA(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
  for (int q = 0; q < c->world; ++q) {
    ISP_CUDA(cudaStreamCreateWithFlags(&c->peer_st[q], cudaStreamNonBlocking));
    ISP_CUDA(cudaEventCreateWithFlags(&c->ev_join[q], cudaEventDisableTiming));
    for (int t = 0; t < SEQPLAN_W_COUNT; ++t)
      for (int set = 0; set < 2; ++set) ISP_CUDA(cudaEventCreateWithFlags(&c->ev_tq[set][t][q], cudaEventDisableTiming));
  }
  for (int t = 0; t < SEQPLAN_W_COUNT; ++t) {
    ISP_CUDA(cudaEventCreateWithFlags(&c->ev_gathered[t], cudaEventDisableTiming));
    ISP_CUDA(cudaEventCreateWithFlags(&c->ev_wgrad[t], cudaEventDisableTiming));
    ISP_CUDA(cudaEventCreateWithFlags(&c->ev_staged[t], cudaEventDisableTiming));
  }
  ISP_CUDA(cudaEventCreateWithFlags(&c->ev_comm_done, cudaEventDisableTiming));
  ISP_CUDA(cudaStreamCreateWithFlags(&c->red, cudaStreamNonBlocking));
  ISP_CUDA(cudaEventCreateWithFlags(&c->ev_red_done, cudaEventDisableTiming));
  for (int t = 0; t < SEQPLAN_W_COUNT; ++t) ISP_CUDA(cudaEventCreateWithFlags(&c->ev_rs_sent[t], cudaEventDisableTiming));
  ISP_CUDA(cudaEventCreateWithFlags(&c->ev_start, cudaEventDisableTiming));
  ISP_CUDA(cudaEventCreateWithFlags(&c->ev_tail, cudaEventDisableTiming));

  // RoPE table, computed like oracle/block_oracle.c:ob_rope_table (double -> fp32)
  {
    const int64_t half = c->d / 2;
    std::vector<float> cs(size_t(S * half)), sn(size_t(S * half));
    for (int64_t i = 0; i < half; ++i) {
      const double inv = std::pow(c->rope_base, -2.0 * double(i) / double(c->d));
      for (int64_t t = 0; t < S; ++t) {
        const double ang = double(t) * inv;
        cs[size_t(t * half + i)] = static_cast<float>(std::cos(ang));
        sn[size_t(t * half + i)] = static_cast<float>(std::sin(ang));
      }
    }
    ISP_CUDA(cudaMemcpy(c->cos_t, cs.data(), cs.size() * 4, cudaMemcpyHostToDevice));
    ISP_CUDA(cudaMemcpy(c->sin_t, sn.data(), sn.size() * 4, cudaMemcpyHostToDevice));
  }
  c->pool->step_boundary();
}

// Refresh the bf16 working shard(s) from the fp32 master of tensor t.
void refresh_working(Ctx* c, int t, cudaStream_t st) {
  ISP_CUDA(cast_f32_bf16(c->master[t], c->wshard(t), c->shard(t), st, c->num_sms));
  if (c->world == 1 && (t == SEQPLAN_W_GATE || t == SEQPLAN_W_UP)) {
    // p = 1: keep the gate|up working copy interleaved in kGuBlock-row blocks for the fused GEMM
    const int64_t rows = c->I, cols = c->H, B = kGuBlock;
    ISP_CUDA(cudaMemcpy2DAsync(c->wgu_local + (t == SEQPLAN_W_UP ? B : 0) * cols, size_t(2 * B * cols * 2),
                               c->wshard(t), size_t(B * cols * 2), size_t(B * cols * 2), size_t(rows / B),
                               cudaMemcpyDeviceToDevice, st));
  }
  c->weights_dirty = true;
}

int fail(Ctx* c, const IspError& e) {
  if (c) c->last_error = e.msg;
  return e.code;
}

void collect_timeline(Ctx* c) {
  if (c->tl_pending.empty()) return;
  cudaEvent_t t0 = c->tl_pending.front().b;
  for (auto& ev : c->tl_pending) {
    cudaEventSynchronize(ev.e);
    float s = 0, e = 0;
    cudaEventElapsedTime(&s, t0, ev.b);
    cudaEventElapsedTime(&e, t0, ev.e);
    c->timeline.push_back({ev.stream, ev.kind, ev.layer, s * 1e-3, e * 1e-3});
  }
  for (auto& ev : c->tl_pending) {
    if (ev.b != t0) cudaEventDestroy(ev.b);
    cudaEventDestroy(ev.e);
  }
  cudaEventDestroy(t0);
  c->tl_pending.clear();
}

void collect_kprof(Ctx* c) {
  for (auto& k : c->kprof_pending) {
    cudaEventSynchronize(k.e);
    float ms = 0;
    cudaEventElapsedTime(&ms, k.b, k.e);
    c->kprof.push_back({k.kind, k.flops, k.bytes, static_cast<double>(ms) * 1e-3});
    cudaEventDestroy(k.b);
    cudaEventDestroy(k.e);
  }
  c->kprof_pending.clear();
}

void check_device_error(Ctx* c) {
  if (c->world == 1 || c->group_mode) return;
  uint32_t flag = 0;
  cudaMemcpy(&flag, c->error_flag, 4, cudaMemcpyDeviceToHost);
  if (flag) throw IspError(SEQPLAN_ISP_ERR_RUNTIME, "peer barrier timed out (a rank stopped responding)");
}

}  // namespace

// =====================================================================================
// C ABI
// =====================================================================================
extern "C" {

static int create_ctx(int world, int rank, int device, const seqplan_isp_shape* shape,
                      const seqplan_strategy* strategy, const seqplan_mempool_policy* policy, uint32_t flags,
                      DevicePool* shared_pool, int premap_layers, seqplan_isp_ctx** out, int push_override = -1);

int seqplan_isp_ctx_create(int world, int rank, int device, const seqplan_isp_shape* shape,
                           const seqplan_strategy* strategy, const seqplan_mempool_policy* policy,
                           uint32_t flags, seqplan_isp_ctx** out) {
  return create_ctx(world, rank, device, shape, strategy, policy, flags, nullptr, 1, out);
}

static int create_ctx(int world, int rank, int device, const seqplan_isp_shape* shape,
                      const seqplan_strategy* strategy, const seqplan_mempool_policy* policy, uint32_t flags,
                      DevicePool* shared_pool, int premap_layers, seqplan_isp_ctx** out, int push_override) {
  if (!out || !shape) return SEQPLAN_ISP_ERR_INVALID;
  *out = nullptr;
  if (rank < 0 || rank >= world) return SEQPLAN_ISP_ERR_INVALID;
  if (strategy) {
    // The executor runs exactly the ISP plan: validate it with the reference's rules.
    seqplan::Strategy s;
    s.micro_batch = strategy->micro_batch; s.micro_batch_num = strategy->micro_batch_num;
    s.recompute = strategy->recompute; s.pp = strategy->pp; s.dp = strategy->dp; s.tp = strategy->tp;
    s.sp = strategy->sp; s.ps = strategy->ps; s.gs = strategy->gs; s.oss = strategy->oss;
    seqplan::ModelConfig m;
    m.hidden_dim = shape->hidden_dim; m.layers = 1; m.heads = shape->heads; m.vocab = 1;
    m.seq_len = shape->seq_len; m.global_batch_tokens = shape->seq_len * s.micro_batch * s.micro_batch_num * s.dp;
    seqplan::ClusterConfig cl{world, world, 0};
    if (!seqplan::validate(s, m, cl).ok() || s.sp != world || s.ps != world || s.tp != 1 || s.pp != 1 ||
        s.dp != 1 || (s.recompute != 0 && s.recompute != 1))
      return SEQPLAN_ISP_ERR_INVALID;
    // Legal plans this executor does not run: b > 1 sequences per micro-batch, gradient-sync (gs)
    // or optimizer-state-sharding (oss) groups. n > 1 micro-batches run as n fwd/bwd calls per
    // step whose weight gradients accumulate into the fp32 shards (reset by the first).
    if (s.micro_batch != 1 || s.gs != 1 || s.oss != 1) return SEQPLAN_ISP_ERR_UNSUPPORTED;
  }
  Ctx* c = new Ctx();
  c->world = world;
  c->rank = rank;
  c->device = device;
  c->flags = flags;
  c->recompute = (strategy && strategy->recompute == 1) || (flags & SEQPLAN_ISP_FLAG_RECOMPUTE);
  c->micro_batches = strategy ? static_cast<int>(strategy->micro_batch_num) : 1;
  c->push_pref = push_override;  // -1: by world size; SEQPLAN_ISP_PUSH overrides either (setup)
  if (shared_pool) {
    c->pool = shared_pool;
    c->owns_pool = false;
  }
  try {
    setup(c, shape, policy, premap_layers);
  } catch (const IspError& e) {
    const int code = e.code;
    std::fprintf(stderr, "seqplan_isp_ctx_create: %s\n", e.msg.c_str());
    seqplan_isp_ctx_destroy(c);
    return code;
  }
  *out = c;
  return SEQPLAN_ISP_OK;
}

void seqplan_isp_ctx_destroy(seqplan_isp_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  for (int q = 0; q < c->world; ++q)
    if (c->peer_opened[q]) cudaIpcCloseMemHandle(c->peer_heap[q]);
  if (c->owns_pool) c->pool->release_all();  // a stack's layers free their memory with layer 0's pool
  if (c->heap) cudaFree(c->heap);
  nvls_release(c->nvls_buf);
  if (c->comm && c->owns_comm) cudaStreamDestroy(c->comm);
  for (int q = 0; q < kMaxRanks; ++q) {
    if (c->peer_st[q]) cudaStreamDestroy(c->peer_st[q]);
    if (c->ev_join[q]) cudaEventDestroy(c->ev_join[q]);
    for (int t = 0; t < SEQPLAN_W_COUNT; ++t)
      for (int set = 0; set < 2; ++set)
        if (c->ev_tq[set][t][q]) cudaEventDestroy(c->ev_tq[set][t][q]);
  }
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  for (int t = 0; t < SEQPLAN_W_COUNT; ++t) {
    if (c->ev_gathered[t]) cudaEventDestroy(c->ev_gathered[t]);
    if (c->ev_wgrad[t]) cudaEventDestroy(c->ev_wgrad[t]);
    if (c->ev_staged[t]) cudaEventDestroy(c->ev_staged[t]);
  }
  if (c->ev_comm_done) cudaEventDestroy(c->ev_comm_done);
  if (c->red) cudaStreamDestroy(c->red);
  if (c->ev_red_done) cudaEventDestroy(c->ev_red_done);
  for (int t = 0; t < SEQPLAN_W_COUNT; ++t)
    if (c->ev_rs_sent[t]) cudaEventDestroy(c->ev_rs_sent[t]);
  if (c->ev_start) cudaEventDestroy(c->ev_start);
  if (c->ev_tail) cudaEventDestroy(c->ev_tail);
  delete c;
}

const char* seqplan_isp_last_error(const seqplan_isp_ctx* c) { return c ? c->last_error.c_str() : ""; }

size_t seqplan_isp_ipc_handle_size(void) { return sizeof(cudaIpcMemHandle_t); }

int seqplan_isp_ipc_handle(seqplan_isp_ctx* c, void* out) {
  if (!c || !out) return SEQPLAN_ISP_ERR_INVALID;
  try {
    ISP_CUDA(cudaSetDevice(c->device));
    cudaIpcMemHandle_t h;
    ISP_CUDA(cudaIpcGetMemHandle(&h, c->heap));
    std::memcpy(out, &h, sizeof(h));
  } catch (const IspError& e) {
    return fail(c, e);
  }
  return SEQPLAN_ISP_OK;
}

int seqplan_isp_open_peers(seqplan_isp_ctx* c, const void* handles) {
  if (!c || !handles) return SEQPLAN_ISP_ERR_INVALID;
  try {
    ISP_CUDA(cudaSetDevice(c->device));
    const auto* hs = static_cast<const cudaIpcMemHandle_t*>(handles);
    for (int q = 0; q < c->world; ++q) {
      if (q == c->rank) continue;
      void* p = nullptr;
      ISP_CUDA(cudaIpcOpenMemHandle(&p, hs[q], cudaIpcMemLazyEnablePeerAccess));
      c->peer_heap[q] = p;
      c->peer_opened[q] = true;
    }
  } catch (const IspError& e) {
    return fail(c, e);
  }
  return SEQPLAN_ISP_OK;
}

// ---- NVLink SHARP reduce-scatter setup (multi-process, push transport) ----
static bool nvls_applicable(const Ctx* c, std::string* why) {
  if ((c->nvls_pref & 3) == 0) return *why = "off (SEQPLAN_ISP_NVLS=0)", false;
  if (!c->push_mode() || c->group_mode || c->co_resident || c->rs_ce)
    return *why = "needs the multi-process push transport", false;
  if (c->world < 2 || c->nvls_bytes == 0) return *why = "nothing to reduce", false;
  return nvls_supported(c->device, why);
}

int seqplan_isp_nvls_export(seqplan_isp_ctx* c, int* pid, int* fd) {
  if (!c || !pid || !fd || c->rank != 0) return SEQPLAN_ISP_ERR_INVALID;
  std::string why;
  if (!nvls_applicable(c, &why)) {
    c->last_error = "nvls: " + why;
    return SEQPLAN_ISP_ERR_UNSUPPORTED;
  }
  try {
    ISP_CUDA(cudaSetDevice(c->device));
    if (!nvls_create(c->nvls_buf, c->device, c->world, c->nvls_bytes, &why))
      throw IspError(SEQPLAN_ISP_ERR_RUNTIME, "nvls: " + why);
    *pid = static_cast<int>(getpid());
    *fd = c->nvls_buf.export_fd;
  } catch (const IspError& e) {
    nvls_release(c->nvls_buf);
    return fail(c, e);
  }
  return SEQPLAN_ISP_OK;
}

int seqplan_isp_nvls_attach(seqplan_isp_ctx* c, int pid, int fd) {
  if (!c) return SEQPLAN_ISP_ERR_INVALID;
  std::string why;
  try {
    ISP_CUDA(cudaSetDevice(c->device));
    if (c->rank != 0) {
      if (!nvls_applicable(c, &why) ||
          !nvls_import(c->nvls_buf, c->device, c->world, c->nvls_bytes, pid, fd, &why))
        throw IspError(SEQPLAN_ISP_ERR_RUNTIME, "nvls: " + why);
    } else if (!c->nvls_buf.have_mc) {
      return SEQPLAN_ISP_ERR_INVALID;
    }
    if (!nvls_add_device(c->nvls_buf, &why)) throw IspError(SEQPLAN_ISP_ERR_RUNTIME, "nvls: " + why);
  } catch (const IspError& e) {
    nvls_release(c->nvls_buf);
    return fail(c, e);
  }
  return SEQPLAN_ISP_OK;
}

int seqplan_isp_nvls_bind(seqplan_isp_ctx* c) {
  if (!c || !c->nvls_buf.have_mc) return SEQPLAN_ISP_ERR_INVALID;
  std::string why;
  try {
    ISP_CUDA(cudaSetDevice(c->device));
    ISP_CUDA(cudaDeviceSynchronize());
    if (!nvls_bind(c->nvls_buf, &why)) throw IspError(SEQPLAN_ISP_ERR_RUNTIME, "nvls: " + why);
    c->nvls = (c->nvls_pref & 1) != 0;
    c->nvls_ag = (c->nvls_pref & 2) != 0;
  } catch (const IspError& e) {
    nvls_release(c->nvls_buf);
    return fail(c, e);
  }
  return SEQPLAN_ISP_OK;
}

int seqplan_isp_nvls_release(seqplan_isp_ctx* c) {
  if (!c) return SEQPLAN_ISP_ERR_INVALID;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  c->nvls = c->nvls_ag = false;
  nvls_release(c->nvls_buf);
  return SEQPLAN_ISP_OK;
}

int seqplan_isp_nvls_active(const seqplan_isp_ctx* c) { return c ? (c->nvls ? 1 : 0) | (c->nvls_ag ? 2 : 0) : 0; }

int seqplan_isp_link_local_peers(seqplan_isp_ctx** cs, int world) {
  if (!cs || world < 2 || world > kMaxRanks) return SEQPLAN_ISP_ERR_INVALID;
  for (int r = 0; r < world; ++r) {
    if (!cs[r] || cs[r]->world != world || cs[r]->rank != r || cs[r]->device != cs[0]->device || cs[r]->group_mode)
      return SEQPLAN_ISP_ERR_INVALID;
    for (int q = 0; q < world; ++q)
      if (cs[r]->peer_opened[q]) return SEQPLAN_ISP_ERR_INVALID;
  }
  for (int r = 0; r < world; ++r) {
    for (int q = 0; q < world; ++q) cs[r]->peer_heap[q] = cs[q]->heap;
    cs[r]->co_resident = true;
  }
  return SEQPLAN_ISP_OK;
}

int seqplan_isp_group_create(int world, int device, const seqplan_isp_shape* shape,
                             const seqplan_mempool_policy* policy, uint32_t flags, seqplan_isp_ctx** out_ctxs) {
  if (!out_ctxs || world < 1 || world > kMaxRanks) return SEQPLAN_ISP_ERR_INVALID;
  for (int r = 0; r < world; ++r) out_ctxs[r] = nullptr;
  for (int r = 0; r < world; ++r) {
    int st = seqplan_isp_ctx_create(world, r, device, shape, nullptr, policy, flags, &out_ctxs[r]);
    if (st != SEQPLAN_ISP_OK) {
      for (int q = 0; q < r; ++q) seqplan_isp_ctx_destroy(out_ctxs[q]);
      return st;
    }
    out_ctxs[r]->group_mode = true;
  }
  for (int r = 0; r < world; ++r)
    for (int q = 0; q < world; ++q) out_ctxs[r]->peer_heap[q] = out_ctxs[q]->heap;
  return SEQPLAN_ISP_OK;
}

int seqplan_isp_init_weights(seqplan_isp_ctx* c, uint64_t seed) {
  if (!c) return SEQPLAN_ISP_ERR_INVALID;
  try {
    ISP_CUDA(cudaSetDevice(c->device));
    // tensor ids 2..8: norms 1 + N(0, .02), linear N(0, .02)
    for (int t = 0; t < SEQPLAN_W_COUNT; ++t) {
      const bool norm = (t == SEQPLAN_W_NORM1 || t == SEQPLAN_W_NORM2);
      ISP_CUDA(keyed_fill(seed, t + 2, c->rank * c->shard(t), c->shard(t), norm ? 1.0 : 0.0, 0.02, c->master[t],
                          nullptr, nullptr, c->num_sms));
      refresh_working(c, t, nullptr);
    }
    ISP_CUDA(cudaDeviceSynchronize());
  } catch (const IspError& e) {
    return fail(c, e);
  }
  return SEQPLAN_ISP_OK;
}

int seqplan_isp_adamw_step(seqplan_isp_ctx* c, const seqplan_adamw_params* p, void* stream) {
  if (!c || !p || p->step < 1 || !(p->lr >= 0) || !(p->beta1 >= 0 && p->beta1 < 1) || !(p->beta2 >= 0 && p->beta2 < 1) ||
      !(p->eps > 0))
    return SEQPLAN_ISP_ERR_INVALID;
  try {
    ISP_CUDA(cudaSetDevice(c->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    AdamWArgs a;
    a.lr = static_cast<float>(p->lr);
    a.beta1 = static_cast<float>(p->beta1);
    a.beta2 = static_cast<float>(p->beta2);
    a.eps = static_cast<float>(p->eps);
    a.weight_decay = static_cast<float>(p->weight_decay);
    a.inv_bc1 = static_cast<float>(1.0 / (1.0 - std::pow(p->beta1, double(p->step))));
    a.inv_bc2 = static_cast<float>(1.0 / (1.0 - std::pow(p->beta2, double(p->step))));
    for (int t = 0; t < SEQPLAN_W_COUNT; ++t) {
      const int64_t n = c->shard(t);
      if (!c->adam_m[t]) {
        c->adam_m[t] = static_cast<float*>(pool_alloc(c, n * 4, seqplan::AllocTag::Other, st));
        c->adam_v[t] = static_cast<float*>(pool_alloc(c, n * 4, seqplan::AllocTag::Other, st));
        ISP_CUDA(cudaMemsetAsync(c->adam_m[t], 0, size_t(n) * 4, st));
        ISP_CUDA(cudaMemsetAsync(c->adam_v[t], 0, size_t(n) * 4, st));
      }
      ISP_LAUNCH(1, adamw_step(c->master[t], c->grad[t], c->adam_m[t], c->adam_v[t], c->wshard(t), n, a, st,
                               c->num_sms));
      if (c->world == 1 && (t == SEQPLAN_W_GATE || t == SEQPLAN_W_UP)) {  // interleaved gate|up working copy
        const int64_t rows = c->I, cols = c->H, B = kGuBlock;
        ISP_CUDA(cudaMemcpy2DAsync(c->wgu_local + (t == SEQPLAN_W_UP ? B : 0) * cols, size_t(2 * B * cols * 2),
                                   c->wshard(t), size_t(B * cols * 2), size_t(B * cols * 2), size_t(rows / B),
                                   cudaMemcpyDeviceToDevice, st));
      }
    }
    c->weights_dirty = true;  // peers gather the new working shards after the next barrier
  } catch (const IspError& e) {
    return fail(c, e);
  }
  return SEQPLAN_ISP_OK;
}

int64_t seqplan_isp_shard_numel(const seqplan_isp_ctx* c, int t) {
  if (!c || t < 0 || t >= SEQPLAN_W_COUNT) return -1;
  return c->shard(t);
}

int seqplan_isp_set_weight_shard(seqplan_isp_ctx* c, int t, const float* host, int64_t n) {
  if (!c || !host || t < 0 || t >= SEQPLAN_W_COUNT || n != c->shard(t)) return SEQPLAN_ISP_ERR_INVALID;
  try {
    ISP_CUDA(cudaSetDevice(c->device));
    ISP_CUDA(cudaMemcpy(c->master[t], host, size_t(n) * 4, cudaMemcpyHostToDevice));
    refresh_working(c, t, nullptr);
    ISP_CUDA(cudaDeviceSynchronize());
  } catch (const IspError& e) {
    return fail(c, e);
  }
  return SEQPLAN_ISP_OK;
}

int seqplan_isp_get_weight_shard(seqplan_isp_ctx* c, int t, float* host, int64_t n) {
  if (!c || !host || t < 0 || t >= SEQPLAN_W_COUNT || n != c->shard(t)) return SEQPLAN_ISP_ERR_INVALID;
  try {
    ISP_CUDA(cudaSetDevice(c->device));
    ISP_CUDA(cudaMemcpy(host, c->master[t], size_t(n) * 4, cudaMemcpyDeviceToHost));
  } catch (const IspError& e) {
    return fail(c, e);
  }
  return SEQPLAN_ISP_OK;
}

int seqplan_isp_get_grad_shard(seqplan_isp_ctx* c, int t, float* host, int64_t n) {
  if (!c || !host || t < 0 || t >= SEQPLAN_W_COUNT || n != c->shard(t)) return SEQPLAN_ISP_ERR_INVALID;
  try {
    ISP_CUDA(cudaSetDevice(c->device));
    ISP_CUDA(cudaDeviceSynchronize());
    ISP_CUDA(cudaMemcpy(host, c->grad[t], size_t(n) * 4, cudaMemcpyDeviceToHost));
  } catch (const IspError& e) {
    return fail(c, e);
  }
  return SEQPLAN_ISP_OK;
}

int seqplan_isp_grad_shard_ptr(seqplan_isp_ctx* c, int t, float** dev_ptr) {
  if (!c || !dev_ptr || t < 0 || t >= SEQPLAN_W_COUNT) return SEQPLAN_ISP_ERR_INVALID;
  *dev_ptr = c->grad[t];
  return SEQPLAN_ISP_OK;
}

int seqplan_isp_fill_activation(seqplan_isp_ctx* c, uint64_t seed, int tensor_id, void* dev_out, void* stream) {
  if (!c || !dev_out) return SEQPLAN_ISP_ERR_INVALID;
  try {
    ISP_CUDA(cudaSetDevice(c->device));
    ISP_CUDA(keyed_fill(seed, tensor_id, c->rank * c->T * c->H, c->T * c->H, 0.0, 1.0, nullptr,
                        static_cast<bf16*>(dev_out), static_cast<cudaStream_t>(stream), c->num_sms));
  } catch (const IspError& e) {
    return fail(c, e);
  }
  return SEQPLAN_ISP_OK;
}

// Step start: epoch, the write-after-read barrier (peers finished the previous step, refreshed
// working shards visible), and the weight gathers. defer_bwd_set (push mode): the backward
// re-gather set is left for the caller to issue (multi-layer stacks order it after every
// layer's forward set).
static void fwd_prologue(Ctx* c, cudaStream_t st, bool do_barrier, bool defer_bwd_set) {
  ++c->step_epoch;
  if (do_barrier && (c->weights_dirty || c->fused_a2a || c->push_mode())) {
    // peers must see refreshed working shards before gathering; with fused all-to-all, no
    // peer may push into this rank's exchange buffers before its previous backward finished
    barrier(c, st, false);
  }
  c->weights_dirty = false;
  c->timeline.clear();
  c->defer_bwd_set = defer_bwd_set;
  fwd_issue_gathers(c, st);
  c->defer_bwd_set = false;
}

// Backward re-gather of one layer of a stack on its comm stream, ordered after the compute
// stream's current point (the two-layer window of seqplan_isp_stack_*).
static void stack_prefetch_bwd(Ctx* c, cudaStream_t st) {
  if (c->bwd_prefetched) return;
  ISP_CUDA(cudaEventRecord(c->ev_start, st));
  ISP_CUDA(cudaStreamWaitEvent(c->comm, c->ev_start, 0));
  prefetch_bwd_set(c);
}

static void push_bwd_set(Ctx* c) {
  if (!c->push_mode()) {
    prefetch_bwd_set(c);
    return;
  }
  const int bo[] = {SEQPLAN_W_DOWN, SEQPLAN_W_GATE, SEQPLAN_W_NORM2, SEQPLAN_W_O, SEQPLAN_W_QKV, SEQPLAN_W_NORM1};
  push_gather_set(c, 1, bo, 6, !c->push_skip());
}

static void fwd_body(Ctx* c, const bf16* x, bf16* y, cudaStream_t st) {
  alloc_acts(c, st);
  fwd_phase1(c, x, st);
  barrier(c, st, false);
  fwd_phase2(c, st);
  barrier(c, st, false);
  fwd_phase3(c, x, y, st);
  if (c->recompute) free_acts(c, st);  // a = 1: only x (the checkpoint) outlives the forward
  c->fwd_done = true;
}

static void run_fwd(Ctx* c, const bf16* x, bf16* y, cudaStream_t st) {
  fwd_prologue(c, st, true, false);
  fwd_body(c, x, y, st);
}

// a = 1: the forward is re-run from the checkpoint x on the backward's re-gathered weights
// (the reference's passes = 3 + a, cost.hpp:227), minus the down projection whose output y
// the backward never reads.
static void recompute_fwd(Ctx* c, const bf16* x, cudaStream_t st) {
  alloc_acts(c, st);
  c->recomputing = true;
  fwd_phase1(c, x, st);
  barrier(c, st, false);
  fwd_phase2(c, st);
  barrier(c, st, false);
  fwd_phase3(c, x, nullptr, st);
  c->recomputing = false;
}

static void bwd_body(Ctx* c, const bf16* x, const bf16* dy, bf16* dx, cudaStream_t st) {
  bwd_issue_gathers(c, st);
  if (c->recompute) recompute_fwd(c, x, st);
  alloc_scratch(c, st);
  bwd_phase1(c, dy, st);
  barrier(c, st, false);
  bwd_phase2(c, st);
  barrier(c, st, false);
  bwd_phase3(c, x, dx, st);
  if (c->recompute) {
    free_acts(c, st);
    free_scratch(c, st);
  }
}

// Gradient reductions of the step and the join with the comm stream.
static void bwd_epilogue(Ctx* c, cudaStream_t st) {
  if (c->flags & SEQPLAN_ISP_FLAG_FUSED_BWD) {
    barrier(c, st, false);
    bwd_reduce_all(c, st);
  } else if (c->world > 1) {
    // reduce the staged slices (fp32 accumulate, cast/scale) and join the comm stream
    for (int t : {SEQPLAN_W_DOWN, SEQPLAN_W_GATE, SEQPLAN_W_NORM2, SEQPLAN_W_O, SEQPLAN_W_QKV, SEQPLAN_W_NORM1}) {
      if (c->early_reduce) break;  // already reduced on c->red (schedule_rs)
      if (c->push_mode() && !c->rs_ce) {
        if (!c->skip_comm()) reduce_pushed(c, t, st);
      } else {
        reduce_staged(c, t, st);
      }
    }
    ISP_CUDA(cudaEventRecord(c->ev_comm_done, c->comm));
    ISP_CUDA(cudaStreamWaitEvent(st, c->ev_comm_done, 0));
    if (c->early_reduce) {
      ISP_CUDA(cudaEventRecord(c->ev_red_done, c->red));
      ISP_CUDA(cudaStreamWaitEvent(st, c->ev_red_done, 0));
    }
  }
  if (c->owns_pool) c->pool->step_boundary();
  if (c->push_mode()) c->push_primed = true;
}

static void run_bwd(Ctx* c, const bf16* x, const bf16* dy, bf16* dx, cudaStream_t st) {
  c->accum = c->mb_index > 0;  // micro-batch 2..n of the step: accumulate the weight gradients
  bwd_body(c, x, dy, dx, st);
  bwd_epilogue(c, st);
  c->mb_index = (c->mb_index + 1) % std::max(1, c->micro_batches);
}

int seqplan_isp_block_fwd(seqplan_isp_ctx* c, const void* x, void* y, void* stream) {
  if (!c || !x || !y || c->group_mode) return SEQPLAN_ISP_ERR_INVALID;
  try {
    ISP_CUDA(cudaSetDevice(c->device));
    run_fwd(c, static_cast<const bf16*>(x), static_cast<bf16*>(y), static_cast<cudaStream_t>(stream));
    c->last_x = x;  // RMSNorm-1 input, needed again by block_bwd (caller keeps it alive)
  } catch (const IspError& e) {
    return fail(c, e);
  }
  return SEQPLAN_ISP_OK;
}

int seqplan_isp_block_bwd(seqplan_isp_ctx* c, const void* dy, void* dx, void* stream) {
  if (!c || !dy || !dx || c->group_mode) return SEQPLAN_ISP_ERR_INVALID;
  if (!c->fwd_done || !c->last_x) {
    c->last_error = "block_bwd without a preceding block_fwd";
    return SEQPLAN_ISP_ERR_INVALID;
  }
  try {
    ISP_CUDA(cudaSetDevice(c->device));
    run_bwd(c, static_cast<const bf16*>(c->last_x), static_cast<const bf16*>(dy), static_cast<bf16*>(dx),
            static_cast<cudaStream_t>(stream));
    c->fwd_done = false;
    if ((c->flags & (SEQPLAN_ISP_FLAG_TIMELINE | SEQPLAN_ISP_FLAG_PROFILE)) && !c->co_resident) {
      ISP_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
      check_device_error(c);
      collect_timeline(c);
      collect_kprof(c);
    }
  } catch (const IspError& e) {
    return fail(c, e);
  }
  return SEQPLAN_ISP_OK;
}

int seqplan_isp_group_fwd(seqplan_isp_ctx** cs, int world, const void* const* x, void* const* y, void* stream) {
  if (!cs || !x || !y || world < 1) return SEQPLAN_ISP_ERR_INVALID;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  try {
    ISP_CUDA(cudaSetDevice(cs[0]->device));
    for (int r = 0; r < world; ++r) {
      cs[r]->timeline.clear();
      cs[r]->weights_dirty = false;
      fwd_issue_gathers(cs[r], st);
    }
    for (int r = 0; r < world; ++r) alloc_acts(cs[r], st);
    for (int r = 0; r < world; ++r) fwd_phase1(cs[r], static_cast<const bf16*>(x[r]), st);
    for (int r = 0; r < world; ++r) fwd_phase2(cs[r], st);
    for (int r = 0; r < world; ++r) {
      fwd_phase3(cs[r], static_cast<const bf16*>(x[r]), static_cast<bf16*>(y[r]), st);
      if (cs[r]->recompute) free_acts(cs[r], st);
      cs[r]->fwd_done = true;
      cs[r]->last_x = x[r];
    }
  } catch (const IspError& e) {
    return fail(cs[0], e);
  }
  return SEQPLAN_ISP_OK;
}

int seqplan_isp_group_bwd(seqplan_isp_ctx** cs, int world, const void* const* dy, void* const* dx, void* stream) {
  if (!cs || !dy || !dx || world < 1) return SEQPLAN_ISP_ERR_INVALID;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  try {
    ISP_CUDA(cudaSetDevice(cs[0]->device));
    for (int r = 0; r < world; ++r)
      if (!cs[r]->fwd_done) throw IspError(SEQPLAN_ISP_ERR_INVALID, "group_bwd without group_fwd");
    for (int r = 0; r < world; ++r) bwd_issue_gathers(cs[r], st);
    if (cs[0]->recompute) {  // a = 1: every rank's forward again, in lock-step
      for (int r = 0; r < world; ++r) {
        alloc_acts(cs[r], st);
        cs[r]->recomputing = true;
      }
      for (int r = 0; r < world; ++r) fwd_phase1(cs[r], static_cast<const bf16*>(cs[r]->last_x), st);
      for (int r = 0; r < world; ++r) fwd_phase2(cs[r], st);
      for (int r = 0; r < world; ++r) {
        fwd_phase3(cs[r], static_cast<const bf16*>(cs[r]->last_x), nullptr, st);
        cs[r]->recomputing = false;
      }
    }
    for (int r = 0; r < world; ++r) alloc_scratch(cs[r], st);
    for (int r = 0; r < world; ++r) bwd_phase1(cs[r], static_cast<const bf16*>(dy[r]), st);
    for (int r = 0; r < world; ++r) bwd_phase2(cs[r], st);
    for (int r = 0; r < world; ++r)
      bwd_phase3(cs[r], static_cast<const bf16*>(cs[r]->last_x), static_cast<bf16*>(dx[r]), st);
    for (int r = 0; r < world; ++r) {
      bwd_reduce_all(cs[r], st);
      if (cs[r]->recompute) {
        free_acts(cs[r], st);
        free_scratch(cs[r], st);
      }
      cs[r]->pool->step_boundary();
      cs[r]->fwd_done = false;
    }
    if (cs[0]->flags & (SEQPLAN_ISP_FLAG_TIMELINE | SEQPLAN_ISP_FLAG_PROFILE)) {
      ISP_CUDA(cudaStreamSynchronize(st));
      for (int r = 0; r < world; ++r) {
        collect_timeline(cs[r]);
        collect_kprof(cs[r]);
      }
    }
  } catch (const IspError& e) {
    return fail(cs[0], e);
  }
  return SEQPLAN_ISP_OK;
}

int seqplan_isp_kernel_profile(seqplan_isp_ctx* c, seqplan_kernel_record* out, int64_t* n, int clear) {
  if (!c || !n) return SEQPLAN_ISP_ERR_INVALID;
  collect_kprof(c);  // deferred records (co-resident ranks); waits on their events
  const int64_t have = static_cast<int64_t>(c->kprof.size());
  if (out) {
    const int64_t k = std::min(*n, have);
    for (int64_t i = 0; i < k; ++i) out[i] = c->kprof[size_t(i)];
  }
  *n = have;
  if (clear) c->kprof.clear();
  return SEQPLAN_ISP_OK;
}

int64_t seqplan_isp_launch_count(const seqplan_isp_ctx* c) { return c ? c->launches : -1; }

// ---- multi-layer stacks ------------------------------------------
struct seqplan_isp_stack {
  std::vector<Ctx*> layers;
  bool window = true;  // two-layer prefetch window (copy-engine transport); SEQPLAN_ISP_STACK_WINDOW=0: all up front
  // layer boundaries, [T, H] bf16 from the shared pool: act[l] = input of layer l (l >= 1), the
  // checkpoint kept from the forward to layer l's backward (AllocTag::MlpOutput, packed k to a
  // region under consolidate_every_k_mlp, mempool.hpp:345-352); grad[l] = dx of layer l = dy of
  // layer l-1, live from layer l's backward to layer l-1's
  std::vector<bf16*> act;
  std::vector<bf16*> grad;
  const void* x0 = nullptr;
  bool fwd_done = false;
};

int seqplan_isp_stack_create(int layers, int world, int rank, int device, const seqplan_isp_shape* shape,
                             const seqplan_strategy* strategy, const seqplan_mempool_policy* policy, uint32_t flags,
                             seqplan_isp_stack** out) {
  if (!out || layers < 1) return SEQPLAN_ISP_ERR_INVALID;
  *out = nullptr;
  auto* s = new seqplan_isp_stack();
  if (const char* e = std::getenv("SEQPLAN_ISP_STACK_WINDOW")) s->window = std::atoi(e) != 0;
  // Transport: the push transport's pinned buffers (two gather sets + the RS staging, 3·e·Ψ_blk)
  // live in every layer's heap for the whole run; when the stack's share would exceed a quarter of
  // the device, the copy-engine transport with the two-layer gather window (pool buffers, at most
  // two layers' sets live; cost.hpp:147) is used instead (SEQPLAN_ISP_PUSH still forces either)
  int push_override = -1;
  if (shape && world >= 4) {
    const int64_t H = shape->hidden_dim, I = shape->ffn_dim > 0 ? shape->ffn_dim : seqplan::mlp_intermediate_dim(H);
    const int64_t psi = 4 * H * H + 3 * I * H + 2 * H;
    size_t free_b = 0, total_b = 0;
    if (cudaSetDevice(device) == cudaSuccess && cudaMemGetInfo(&free_b, &total_b) == cudaSuccess &&
        int64_t(layers) * 3 * psi * 2 > int64_t(total_b / 4))
      push_override = 0;
  }
  for (int l = 0; l < layers; ++l) {
    Ctx* c = nullptr;
    // one device pool for the stack (layer 0's): checkpoints, a = 1 workspaces and the gradient
    // arena of every layer (pre-mapped by the owner) share it, as in the reference's trace
    DevicePool* shared = l == 0 ? nullptr : s->layers[0]->pool;
    const int st =
        create_ctx(world, rank, device, shape, strategy, policy, flags, shared, l == 0 ? layers : 1, &c, push_override);
    if (st != SEQPLAN_ISP_OK) {
      seqplan_isp_stack_destroy(s);
      return st;
    }
    s->layers.push_back(c);
  }
  Ctx* c0 = s->layers[0];
  try {
    ISP_CUDA(cudaSetDevice(device));
    // one comm stream for the whole stack: gathers and reduce-scatters of all layers are one FIFO,
    // the reference's two-stream schedule (overlap_sim.hpp:55-74)
    for (int l = 1; l < layers; ++l) {
      Ctx* c = s->layers[l];
      ISP_CUDA(cudaStreamDestroy(c->comm));
      c->comm = c0->comm;
      c->owns_comm = false;
    }
    s->act.assign(size_t(layers), nullptr);
    s->grad.assign(size_t(layers), nullptr);
  } catch (const IspError& e) {
    std::fprintf(stderr, "seqplan_isp_stack_create: %s\n", e.msg.c_str());
    seqplan_isp_stack_destroy(s);
    return e.code;
  }
  *out = s;
  return SEQPLAN_ISP_OK;
}

void seqplan_isp_stack_destroy(seqplan_isp_stack* s) {
  if (!s) return;
  if (!s->layers.empty()) cudaSetDevice(s->layers[0]->device);
  cudaDeviceSynchronize();
  for (size_t l = s->layers.size(); l-- > 0;) seqplan_isp_ctx_destroy(s->layers[l]);  // layer 0 (comm owner) last
  delete s;
}

int seqplan_isp_stack_layers(const seqplan_isp_stack* s) { return s ? static_cast<int>(s->layers.size()) : 0; }

seqplan_isp_ctx* seqplan_isp_stack_layer(seqplan_isp_stack* s, int layer) {
  if (!s || layer < 0 || layer >= static_cast<int>(s->layers.size())) return nullptr;
  return s->layers[size_t(layer)];
}

// Forward of every layer. All forward gathers are issued up front in layer order, then every
// layer's backward re-gather in reverse layer order, on the one comm stream — the reference's
// InterLayerPrefetch forward (overlap_sim.hpp:80-105) and the reverse-order backward prefetch
// (overlap_sim.hpp:141-150); layer l's compute waits only on its own weights.
int seqplan_isp_stack_fwd(seqplan_isp_stack* s, const void* x, void* y, void* stream) {
  if (!s || !x || !y) return SEQPLAN_ISP_ERR_INVALID;
  const int L = static_cast<int>(s->layers.size());
  Ctx* cur = s->layers[0];
  try {
    ISP_CUDA(cudaSetDevice(cur->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    for (int l = 0; l < L; ++l)
      if (s->layers[size_t(l)]->group_mode) throw IspError(SEQPLAN_ISP_ERR_INVALID, "stacks run one process per GPU");
    // Copy-engine transport (gathers into pool buffers): a two-layer window — layer l+1's gathers
    // are issued as layer l starts (the comm stream follows the compute stream to that point, so
    // layer l-1's buffers are back in the pool) and the backward re-gathers one layer ahead —
    // the reference's double buffer (cost.hpp:147 other_buffers = 2 e Psi / tp). Push transport:
    // every layer's pinned sets are its own, so all sets are pushed up front.
    const bool window = !cur->push_mode() && cur->world > 1 && s->window;
    const int first = window ? 1 : L;
    for (int l = 0; l < first; ++l) fwd_prologue(s->layers[size_t(l)], st, l == 0, true);
    if (!window)
      for (int l = L; l-- > 0;) push_bwd_set(s->layers[size_t(l)]);
    const int64_t bytes = s->layers[0]->T * s->layers[0]->H * 2;
    for (int l = 0; l < L; ++l) {
      cur = s->layers[size_t(l)];
      if (window && l + 1 < L) fwd_prologue(s->layers[size_t(l + 1)], st, false, true);
      const bf16* in = l == 0 ? static_cast<const bf16*>(x) : s->act[size_t(l)];
      if (l < L - 1 && !s->act[size_t(l + 1)])
        s->act[size_t(l + 1)] = static_cast<bf16*>(pool_alloc(cur, bytes, seqplan::AllocTag::MlpOutput, st));
      bf16* outp = l == L - 1 ? static_cast<bf16*>(y) : s->act[size_t(l + 1)];
      fwd_body(cur, in, outp, st);
      cur->last_x = in;
    }
    if (window) stack_prefetch_bwd(s->layers[size_t(L - 1)], st);
    s->x0 = x;
    s->fwd_done = true;
  } catch (const IspError& e) {
    return fail(cur, e);
  }
  return SEQPLAN_ISP_OK;
}

// Backward in reverse layer order; the reduce-scatters of every layer overlap the backward of
// the layers below (selective, overlap_sim.hpp:114-153) and are reduced at the end of the step.
int seqplan_isp_stack_bwd(seqplan_isp_stack* s, const void* dy, void* dx, void* stream) {
  if (!s || !dy || !dx || !s->fwd_done) return SEQPLAN_ISP_ERR_INVALID;
  const int L = static_cast<int>(s->layers.size());
  Ctx* cur = s->layers[0];
  try {
    ISP_CUDA(cudaSetDevice(cur->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t bytes = s->layers[0]->T * s->layers[0]->H * 2;
    const bool window = !cur->push_mode() && cur->world > 1 && s->window;
    for (int l = L; l-- > 0;) {
      cur = s->layers[size_t(l)];
      if (window && l > 0) stack_prefetch_bwd(s->layers[size_t(l - 1)], st);  // one layer ahead
      const bf16* g_in = l == L - 1 ? static_cast<const bf16*>(dy) : s->grad[size_t(l + 1)];
      if (l > 0) s->grad[size_t(l)] = static_cast<bf16*>(pool_alloc(cur, bytes, seqplan::AllocTag::Other, st));
      bf16* g_out = l == 0 ? static_cast<bf16*>(dx) : s->grad[size_t(l)];
      cur->accum = cur->mb_index > 0;  // micro-batch 2..n of the step: accumulate
      bwd_body(cur, static_cast<const bf16*>(cur->last_x), g_in, g_out, st);
      cur->fwd_done = false;
      if (l > 0) {  // the checkpoint of layer l is consumed
        cur->pool->free(s->act[size_t(l)], st);
        s->act[size_t(l)] = nullptr;
      }
      if (l < L - 1) {
        cur->pool->free(s->grad[size_t(l + 1)], st);
        s->grad[size_t(l + 1)] = nullptr;
      }
    }
    for (int l = L; l-- > 0;) {
      cur = s->layers[size_t(l)];
      bwd_epilogue(cur, st);
      cur->mb_index = (cur->mb_index + 1) % std::max(1, cur->micro_batches);
      if (cur->flags & (SEQPLAN_ISP_FLAG_TIMELINE | SEQPLAN_ISP_FLAG_PROFILE)) {
        ISP_CUDA(cudaStreamSynchronize(st));
        check_device_error(cur);
        collect_timeline(cur);
        collect_kprof(cur);
      }
    }
    s->fwd_done = false;
  } catch (const IspError& e) {
    return fail(cur, e);
  }
  return SEQPLAN_ISP_OK;
}

// Development: `iters` rounds of (comm-lane barrier, push all-gather of the forward set [and the
// backward set], wait for every peer's flags) on the comm stream; *ms = time per round.
int seqplan_isp_debug_gather_bench(seqplan_isp_ctx* c, int iters, int both_sets, float* ms) {
  if (!c || !ms || !c->push_mode()) return SEQPLAN_ISP_ERR_INVALID;
  try {
    ISP_CUDA(cudaSetDevice(c->device));
    ISP_CUDA(cudaDeviceSynchronize());
    const int fo[] = {SEQPLAN_W_NORM1, SEQPLAN_W_QKV, SEQPLAN_W_O, SEQPLAN_W_NORM2, SEQPLAN_W_GATE, SEQPLAN_W_DOWN};
    cudaEvent_t e0, e1;
    ISP_CUDA(cudaEventCreate(&e0));
    ISP_CUDA(cudaEventCreate(&e1));
    for (int it = -1; it < iters; ++it) {
      if (it == 0) ISP_CUDA(cudaEventRecord(e0, c->comm));
      ++c->step_epoch;
      barrier(c, c->comm, true);
      for (int set = 0; set < (both_sets ? 2 : 1); ++set) {
        push_gather_set(c, set, fo, 6, true);
        for (int t : fo) wait_peers(c, c->comm, [&](int q) { return ag_flag(c, set, t, q); });
      }
    }
    ISP_CUDA(cudaEventRecord(e1, c->comm));
    ISP_CUDA(cudaEventSynchronize(e1));
    ISP_CUDA(cudaEventElapsedTime(ms, e0, e1));
    *ms /= iters;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  } catch (const IspError& e) {
    return fail(c, e);
  }
  return SEQPLAN_ISP_OK;
}

int seqplan_isp_pool_stats(seqplan_isp_ctx* c, seqplan_step_stats* out) {
  if (!c || !out) return SEQPLAN_ISP_ERR_INVALID;
  const auto s = c->pool->stats();
  out->reserved = s.reserved;
  out->allocated = s.allocated;
  out->free_cached = s.free_cached;
  out->fragmented = s.fragmented;
  out->peak_reserved = s.peak_reserved;
  out->peak_fragmented = s.peak_fragmented;
  out->peak_allocated = s.peak_allocated;
  return SEQPLAN_ISP_OK;
}

int seqplan_isp_pool_replay(seqplan_isp_ctx* c, seqplan_step_stats* out, int64_t* n_ops) {
  if (!c || !out) return SEQPLAN_ISP_ERR_INVALID;
  try {
    const seqplan::FragmentationReport r = c->pool->replay();
    const seqplan::StepStats last = r.per_step.empty() ? seqplan::StepStats{} : r.per_step.back();
    out->reserved = last.reserved;
    out->allocated = last.allocated;
    out->free_cached = last.free_cached;
    out->fragmented = last.fragmented;
    out->peak_reserved = r.peak_reserved;
    out->peak_fragmented = r.peak_fragmented;
    out->peak_allocated = 0;
    if (n_ops) *n_ops = static_cast<int64_t>(c->pool->trace().ops.size());
  } catch (const std::exception& e) {
    c->last_error = e.what();
    return SEQPLAN_ISP_ERR_INVALID;
  }
  return SEQPLAN_ISP_OK;
}

int seqplan_isp_timeline(seqplan_isp_ctx* c, seqplan_timeline_event* events, int64_t* n) {
  if (!c || !n) return SEQPLAN_ISP_ERR_INVALID;
  try {
    if (!c->tl_pending.empty()) {  // deferred (co-resident ranks): waits on the step's events
      ISP_CUDA(cudaSetDevice(c->device));
      collect_timeline(c);
      check_device_error(c);
    }
  } catch (const IspError& e) {
    return fail(c, e);
  }
  const int64_t have = static_cast<int64_t>(c->timeline.size());
  if (events) {
    const int64_t k = std::min(*n, have);
    for (int64_t i = 0; i < k; ++i) events[i] = c->timeline[size_t(i)];
  }
  *n = have;
  return SEQPLAN_ISP_OK;
}

}  // extern "C"
