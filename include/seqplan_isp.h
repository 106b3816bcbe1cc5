/*
 * seqplan_isp.h — C ABI of the B200-native ISP (hybrid-sharded) transformer block.
 *
 * The reference (InternEvo "seqplan", /root/reference/proj) has no executor: its
 * hot path exists only as prices and simulators —
 *   per-layer comm/compute   proj/include/seqplan/cost.hpp:160-241
 *   shard layout             proj/include/seqplan/strategy.hpp:52-62, placement.hpp:39-59
 *   overlap schedule         proj/include/seqplan/overlap_sim.hpp:80-153
 *   caching pool             proj/include/seqplan/mempool.hpp:168-387
 * These entry points are the executor those functions model. Every
 * struct below is a POD mirror of a seqplan:: value type so the C++ wrapper
 * (include/seqplan/isp_block.hpp) converts losslessly:
 *   seqplan_isp_shape     <- ModelConfig            (model.hpp:12-48)
 *   seqplan_strategy      <- Strategy               (strategy.hpp:16-48)
 *   seqplan_mempool_policy<- MempoolPolicy          (mempool.hpp:137-142)
 *   seqplan_step_stats    <- StepStats              (mempool.hpp:144-149)
 *   seqplan_timeline_event<- TimelineEvent          (overlap_sim.hpp:28-34)
 *
 * Error behaviour mirrors the reference's exception classes as status codes:
 *   SEQPLAN_ISP_ERR_INVALID  <-> std::invalid_argument (model.hpp:40-47, strategy.hpp:58-59)
 *   SEQPLAN_ISP_ERR_RUNTIME  <-> std::runtime_error (CUDA / peer-memory failure)
 *   SEQPLAN_ISP_ERR_OOM      <-> device allocation failure (pool capacity, mempool.hpp:331)
 *   SEQPLAN_ISP_ERR_UNSUPPORTED  shape the sm_100a kernels do not tile
 * A per-context message is available from seqplan_isp_last_error().
 *
 * All tensors are bf16 row-major on the device unless stated. Activations
 * x, y, dx, dy are caller-owned [S/p, H] slices (rank r owns tokens
 * [r*S/p, (r+1)*S/p)); weights, gathered-weight buffers, gradients and
 * collective scratch are owned by the context's device pool.
 */
#ifndef SEQPLAN_ISP_H_
#define SEQPLAN_ISP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  SEQPLAN_ISP_OK = 0,
  SEQPLAN_ISP_ERR_INVALID = 1,
  SEQPLAN_ISP_ERR_RUNTIME = 2,
  SEQPLAN_ISP_ERR_OOM = 3,
  SEQPLAN_ISP_ERR_UNSUPPORTED = 4,
};

/* Block weight tensors, in the order of SURVEY.md §8(d) tensor ids 2..8. */
enum {
  SEQPLAN_W_NORM1 = 0, /* [H]                 */
  SEQPLAN_W_QKV = 1,   /* [3H, H]  rows q|k|v */
  SEQPLAN_W_O = 2,     /* [H, H]              */
  SEQPLAN_W_NORM2 = 3, /* [H]                 */
  SEQPLAN_W_GATE = 4,  /* [I, H]              */
  SEQPLAN_W_UP = 5,    /* [I, H]              */
  SEQPLAN_W_DOWN = 6,  /* [H, I]              */
  SEQPLAN_W_COUNT = 7
};

/* Context flags. */
enum {
  SEQPLAN_ISP_FLAG_NO_OVERLAP = 1u << 0,   /* serialise gathers with compute (ForwardPolicy::Naive) */
  SEQPLAN_ISP_FLAG_FUSED_BWD = 1u << 1,    /* BackwardPolicy::Fused instead of Selective            */
  SEQPLAN_ISP_FLAG_TIMELINE = 1u << 2,     /* record CUDA-event timeline                            */
  SEQPLAN_ISP_FLAG_SKIP_COMM = 1u << 3,    /* measurement only: collectives become no-ops           */
  SEQPLAN_ISP_FLAG_PROFILE = 1u << 4,      /* per-kernel CUDA events (seqplan_isp_kernel_profile)    */
  SEQPLAN_ISP_FLAG_RECOMPUTE = 1u << 5,    /* a = 1 (Strategy::recompute) where no strategy is given */
};

/* Kernel classes of the per-kernel profile. */
enum {
  SEQPLAN_K_GEMM = 0,
  SEQPLAN_K_ATTN_FWD = 1,
  SEQPLAN_K_ATTN_BWD = 2,
  SEQPLAN_K_ALL_GATHER = 3,
  SEQPLAN_K_REDUCE_SCATTER = 4,
  SEQPLAN_K_ALL_TO_ALL = 5,
  SEQPLAN_K_ELEMENTWISE = 6, /* RMSNorm fwd/bwd, RoPE, SwiGLU bwd (HBM-bound) */
};

typedef struct {
  int32_t kind;   /* SEQPLAN_K_* */
  double flops;   /* algorithmic FLOPs of the launch */
  double bytes;   /* algorithmic bytes (NVLink bytes for collectives) */
  double seconds; /* CUDA-event duration on the launching stream */
} seqplan_kernel_record;

typedef struct seqplan_isp_ctx seqplan_isp_ctx;

typedef struct {
  int64_t hidden_dim; /* H */
  int64_t heads;      /* D */
  int64_t seq_len;    /* S (whole sequence; each rank holds S/p tokens) */
  int64_t ffn_dim;    /* I; 0 = mlp_intermediate_dim(H) (mempool.hpp:79-82) */
  double rope_base;   /* 10000 */
  double norm_eps;    /* 1e-5 */
} seqplan_isp_shape;

typedef struct {
  int64_t micro_batch, micro_batch_num, recompute, pp, dp, tp, sp, ps, gs, oss;
} seqplan_strategy;

typedef struct {
  int32_t pinned_comm_pool;
  int64_t consolidate_every_k_mlp;
  int32_t grad_premap;
  int64_t capacity;
} seqplan_mempool_policy;

typedef struct {
  int64_t reserved, allocated, free_cached, fragmented;
  int64_t peak_reserved, peak_fragmented, peak_allocated;
} seqplan_step_stats;

typedef struct {
  int32_t stream; /* 0 = compute, 1 = comm (StreamKind order) */
  int32_t kind;   /* SEQPLAN_EV_* */
  int64_t layer;
  double start_s, end_s; /* seconds since the first event of the call */
} seqplan_timeline_event;

enum {
  SEQPLAN_EV_FORWARD = 0,
  SEQPLAN_EV_GRAD_INPUT = 1,
  SEQPLAN_EV_GRAD_WEIGHT = 2,
  SEQPLAN_EV_ALL_GATHER = 3,
  SEQPLAN_EV_REDUCE_SCATTER = 4,
  SEQPLAN_EV_ALL_TO_ALL = 5,
};

/* ---- lifecycle ---------------------------------------------------------- */

/* Creates the context of rank `rank` of `world` on CUDA device `device`.
 * The strategy must be the ISP plan [b=1,n>=1,pp=1,dp=1,tp=1,sp=ps=world,gs=oss=1]
 * and must pass seqplan::validate (strategy.hpp:72-99): an illegal plan, or a non-ISP one, is
 * SEQPLAN_ISP_ERR_INVALID; a legal ISP plan with micro_batch != 1, gs != 1 or oss != 1 is
 * SEQPLAN_ISP_ERR_UNSUPPORTED. micro_batch_num = n > 1: the caller runs n block_fwd/block_bwd per
 * step and the weight gradients of calls 2..n accumulate into the fp32 shards (cost.hpp:202-204).
 * policy may be NULL. */
int seqplan_isp_ctx_create(int world, int rank, int device, const seqplan_isp_shape* shape,
                           const seqplan_strategy* strategy, const seqplan_mempool_policy* policy,
                           uint32_t flags, seqplan_isp_ctx** out);
void seqplan_isp_ctx_destroy(seqplan_isp_ctx* ctx);
const char* seqplan_isp_last_error(const seqplan_isp_ctx* ctx);

/* Peer-memory bootstrap (world > 1): every rank exports the IPC handle of its
 * symmetric heap, the caller exchanges the blobs (any transport), and every rank
 * opens all of them. handles = world blobs of seqplan_isp_ipc_handle_size() bytes
 * in rank order. */
size_t seqplan_isp_ipc_handle_size(void);
/* The same without IPC for world ranks created in ONE process on ONE device (ranks 0..world-1 in
 * order): each rank runs the multi-process code path (its own streams, the production weight /
 * gradient transports, stream-memop barriers) with the peers' heaps on the same GPU. The caller
 * issues every rank's block_fwd before any rank's block_bwd (the calls only enqueue work; ranks
 * wait for each other on the device); TIMELINE / PROFILE records are collected when queried.
 * The process must run with CUDA_MODULE_LOADING=EAGER (a lazily loaded kernel's first launch
 * waits for an idle device) and CUDA_DEVICE_MAX_CONNECTIONS >= the total stream count of all
 * ranks (a memop wait at the head of a shared hardware queue would block other ranks' streams). */
int seqplan_isp_link_local_peers(seqplan_isp_ctx** ctxs, int world);
int seqplan_isp_ipc_handle(seqplan_isp_ctx* ctx, void* out);
int seqplan_isp_open_peers(seqplan_isp_ctx* ctx, const void* handles);
/* NVLink SHARP reduce-scatter (multi-process push transport, p >= 4; default on where the
 * GPUs support multicast, SEQPLAN_ISP_NVLS=0 turns it off;
 * replaces the push-RS staging of the four weight matrices, the reference's RS(e*Psi) priced at
 * cost.hpp:184-188): after open_peers, rank 0 calls nvls_export (creates the multicast object,
 * returns its pid and an exported POSIX fd; SEQPLAN_ISP_ERR_UNSUPPORTED when not applicable: then
 * no rank calls the rest), every rank calls nvls_attach with rank 0's pid / fd (rank 0: 0, -1;
 * the others duplicate the fd out of rank 0's process with pidfd_getfd), then — after all ranks
 * attached — nvls_bind. nvls_release abandons it on this rank (the push RS is used again); a
 * failure on any rank must be followed by nvls_release on all. */
int seqplan_isp_nvls_export(seqplan_isp_ctx* ctx, int* pid, int* fd);
int seqplan_isp_nvls_attach(seqplan_isp_ctx* ctx, int pid, int fd);
int seqplan_isp_nvls_bind(seqplan_isp_ctx* ctx);
int seqplan_isp_nvls_release(seqplan_isp_ctx* ctx);
int seqplan_isp_nvls_active(const seqplan_isp_ctx* ctx);

/* Single-process multi-rank mode: p contexts on one device whose "peers" are
 * each other's heaps; collectives run as lock-step phases over all ranks. */
int seqplan_isp_group_create(int world, int device, const seqplan_isp_shape* shape,
                             const seqplan_mempool_policy* policy, uint32_t flags,
                             seqplan_isp_ctx** out_ctxs);
int seqplan_isp_group_fwd(seqplan_isp_ctx** ctxs, int world, const void* const* x,
                          void* const* y, void* stream);
int seqplan_isp_group_bwd(seqplan_isp_ctx** ctxs, int world, const void* const* dy,
                          void* const* dx, void* stream);

/* ---- weights and gradients ---------------------------------------------- */

/* Index-keyed synthetic init (splitmix64 -> Box-Muller): linear
 * weights N(0, 0.02), norm weights 1 + N(0, 0.02). Shard values are independent of p. */
int seqplan_isp_init_weights(seqplan_isp_ctx* ctx, uint64_t seed);
/* Number of elements of this rank's shard of tensor `tensor` (ShardingLayout E/F). */
int64_t seqplan_isp_shard_numel(const seqplan_isp_ctx* ctx, int tensor);
/* fp32 master shard in/out (host pointers). Setting refreshes the bf16 working shard. */
int seqplan_isp_set_weight_shard(seqplan_isp_ctx* ctx, int tensor, const float* host, int64_t n);
int seqplan_isp_get_weight_shard(seqplan_isp_ctx* ctx, int tensor, float* host, int64_t n);
/* fp32 gradient shard written by the last block_bwd (host pointer). */
int seqplan_isp_get_grad_shard(seqplan_isp_ctx* ctx, int tensor, float* host, int64_t n);
/* Device pointer of the fp32 gradient shard (stream-ordered after block_bwd). */
int seqplan_isp_grad_shard_ptr(seqplan_isp_ctx* ctx, int tensor, float** dev_ptr);

/* ---- multi-layer stacks ---------------------------
 * `layers` ISP blocks (one context each, independent weights) run as one step on one comm
 * stream: every layer's forward gathers are issued up front in layer order and every layer's
 * backward re-gather in reverse order (overlap_sim.hpp:80-105, 141-150); layer l's compute waits
 * only on its own weights, and the reduce-scatters of all layers overlap the backward of the
 * layers below. Each layer is a seqplan_isp_ctx (weights, grads, IPC bootstrap, timeline). */
typedef struct seqplan_isp_stack seqplan_isp_stack;
int seqplan_isp_stack_create(int layers, int world, int rank, int device, const seqplan_isp_shape* shape,
                             const seqplan_strategy* strategy, const seqplan_mempool_policy* policy,
                             uint32_t flags, seqplan_isp_stack** out);
void seqplan_isp_stack_destroy(seqplan_isp_stack* stack);
int seqplan_isp_stack_layers(const seqplan_isp_stack* stack);
seqplan_isp_ctx* seqplan_isp_stack_layer(seqplan_isp_stack* stack, int layer);
int seqplan_isp_stack_fwd(seqplan_isp_stack* stack, const void* x, void* y, void* stream);
int seqplan_isp_stack_bwd(seqplan_isp_stack* stack, const void* dy, void* dx, void* stream);

/* Optimizer step after the path (T_update of estimate_step, cost.hpp:292-294):
 * AdamW (torch.optim.AdamW rule: decoupled weight decay, bias-corrected moments) on every fp32
 * master shard with the gradient shard of the last block_bwd; the moment shards live in the device
 * pool (created zero on the first call); the bf16 working shards are refreshed in the same pass.
 * With ISP (dp = 1, oss = 1, gs = 1) there is no optimizer-state collective. step >= 1. */
typedef struct seqplan_adamw_params {
  double lr, beta1, beta2, eps, weight_decay;
  int64_t step;
} seqplan_adamw_params;
int seqplan_isp_adamw_step(seqplan_isp_ctx* ctx, const seqplan_adamw_params* params, void* stream);

/* Synthetic index-keyed bf16 activations for tokens [r*S/p, (r+1)*S/p) of tensor id. */
int seqplan_isp_fill_activation(seqplan_isp_ctx* ctx, uint64_t seed, int tensor_id, void* dev_out,
                                void* stream);

/* ---- the hot path --------------------------------------------------------- */

/* y = block(x) for this rank's S/p tokens; activations needed by backward are kept
 * in the context's pool. x, y: device bf16 [S/p, H]. stream: cudaStream_t.
 * x must stay valid until the matching block_bwd (it is the RMSNorm-1 input, saved by
 * reference rather than copied). */
int seqplan_isp_block_fwd(seqplan_isp_ctx* ctx, const void* x, void* y, void* stream);
/* dx = d block / dx . dy ; fp32 weight-gradient shards land in the pool
 * (gradient reduce-scatter fused with the bf16->fp32 cast and scale). */
int seqplan_isp_block_bwd(seqplan_isp_ctx* ctx, const void* dy, void* dx, void* stream);

/* ---- observability ------------------------------------------------------ */
int seqplan_isp_pool_stats(seqplan_isp_ctx* ctx, seqplan_step_stats* out);
/* The reference's model of this pool: run_mempool(trace, policy) (mempool.hpp:285-387) over the
 * alloc/free trace the device pool recorded (peak_* over the whole trace, the rest at its end);
 * *n_ops receives the trace length. A stack's layers share layer 0's pool. */
int seqplan_isp_pool_replay(seqplan_isp_ctx* ctx, seqplan_step_stats* out, int64_t* n_ops);
/* Copies up to *n events of the last fwd/bwd pair; *n receives the count. */
int seqplan_isp_timeline(seqplan_isp_ctx* ctx, seqplan_timeline_event* events, int64_t* n);

/* Per-kernel records of the calls made with SEQPLAN_ISP_FLAG_PROFILE (collected at the end
 * of each block_bwd). clear != 0 empties the buffer after copying. */
int seqplan_isp_kernel_profile(seqplan_isp_ctx* ctx, seqplan_kernel_record* out, int64_t* n, int clear);
/* Number of kernels this context has launched on the hot path (fwd/bwd). */
int64_t seqplan_isp_launch_count(const seqplan_isp_ctx* ctx);

/* ---- kernel-level entry points (tests) ------------------------------------ */
// Development: push all-gather rounds on the comm stream (multi-process); ms per round.
int seqplan_isp_debug_gather_bench(seqplan_isp_ctx* ctx, int iters, int both_sets, float* ms);
int seqplan_isp_debug_gemm(const void* a, int64_t lda, int a_mn, const void* b, int64_t ldb,
                           int b_mn, void* out, int64_t ldo, int M, int N, int K, int epi,
                           const void* resid, int64_t ldr, void* out2, int64_t ldo2, void* out_b,
                           float scale, int accumulate, int interleave64, void* stream);
/* Causal attention over S tokens (dout == NULL: forward; else backward into dq/dk/dv). */
int seqplan_isp_debug_attention(const void* q, const void* k, const void* v, int64_t ld_qkv, void* o,
                                int64_t ld_o, float* lse, int S, int heads, int d, const void* dout,
                                void* dq, void* dk, void* dv, int64_t ld_d, float* delta, float* dq_acc,
                                void* stream);
/* The same with the stored-dS backward's workspace (ws_bytes >= seqplan_isp_debug_attention_ds_bytes(S)
 * selects it for d = 128: key-tile launch storing the causal dS tiles, then the dQ launch). */
int seqplan_isp_debug_attention_ws(const void* q, const void* k, const void* v, int64_t ld_qkv, void* o,
                                   int64_t ld_o, float* lse, int S, int heads, int d, const void* dout,
                                   void* dq, void* dk, void* dv, int64_t ld_d, float* delta, float* dq_acc,
                                   void* ws, int64_t ws_bytes, void* stream);
/* Bytes of one head's causal dS tiles at sequence length S (the stored-dS backward). */
int64_t seqplan_isp_debug_attention_ds_bytes(int S);
/* RMSNorm forward (dn == NULL) or backward: dx = dres + d(norm), dg += sum dn*xhat. */
int seqplan_isp_debug_rmsnorm(const void* x, const void* g, void* y, float* rstd, const void* dn,
                              const void* dres, void* dx, float* dg, int T, int H, float eps, void* stream);
/* One rank's Ulysses all-to-all (priced at cost.hpp:179-183): dir = +1
 * token-sharded [T, parts*H] on every rank q (src[q]) -> this rank's head-sharded [S, parts*H/world];
 * dir = -1 the reverse. RoPE (+1 / inverse -1) on parts < rope_parts when cos_t != NULL. */
int seqplan_isp_debug_all_to_all(int world, int rank, int T, int H, int parts, int d, int dir,
                                 const void* const* src, void* dst, const float* cos_t, const float* sin_t,
                                 int rope_parts, void* stream);
/* One rank's gradient reduce-scatter fused with the fp32 cast / scale (cost.hpp:184-188):
 * out[i] (+)= scale * sum_{q=0..world-1, in order} part[q][rank*shard_elems + i]. */
int seqplan_isp_debug_reduce_scatter(int world, int rank, int64_t shard_elems, const void* const* part,
                                     int part_is_f32, float scale, int accumulate, float* out, void* stream);
/* One rank's push all-gather (the p >= 4 weight transport, cost.hpp:184-188): `bytes` at src go to
 * offset rank*bytes of every dst[q]; kind 0 = vector stores, 1 = cp.async.bulk driven. */
int seqplan_isp_debug_push_allgather(int world, int rank, void* const* dst, const void* src, int64_t bytes, int kind,
                                     int num_ctas, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SEQPLAN_ISP_H_ */
