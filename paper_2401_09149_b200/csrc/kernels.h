// Host launchers of the non-GEMM sm_100a kernels of the ISP block.
#pragma once

#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace isp {

// ---- elementwise.cu -------------------------------------------------------
uint64_t keyed_stream_base(uint64_t seed, int tensor_id);
cudaError_t keyed_fill(uint64_t seed, int tensor_id, int64_t offset, int64_t n, double mean,
                       double stdv, float* out_f32, __nv_bfloat16* out_bf16, cudaStream_t st,
                       int num_sms);
// AdamW (torch.optim.AdamW update rule) on an fp32 master shard with its fp32 gradient and moment
// shards, writing the refreshed bf16 working shard in the same pass.
struct AdamWArgs {
  float lr, beta1, beta2, eps, weight_decay, inv_bc1, inv_bc2;  // inv_bc = 1 / (1 - beta^step)
};
cudaError_t adamw_step(float* w, const float* g, float* m, float* v, __nv_bfloat16* wb, int64_t n, const AdamWArgs& a,
                       cudaStream_t st, int num_sms);
cudaError_t cast_f32_bf16(const float* in, __nv_bfloat16* out, int64_t n, cudaStream_t st,
                          int num_sms);
cudaError_t rmsnorm_fwd(const __nv_bfloat16* x, const __nv_bfloat16* g, __nv_bfloat16* y,
                        float* rstd, int T, int H, float eps, cudaStream_t st, int num_sms);
// dg += column sums; with dg_scratch (>= rmsnorm_bwd_scratch_rows(num_sms) x H fp32) the
// reduction is two-stage and deterministic, otherwise fp32 atomics.
cudaError_t rmsnorm_bwd(const __nv_bfloat16* x, const __nv_bfloat16* g, const float* rstd,
                        const __nv_bfloat16* dn, const __nv_bfloat16* dres, __nv_bfloat16* dx,
                        float* dg, int T, int H, cudaStream_t st, int num_sms,
                        float* dg_scratch = nullptr);
int rmsnorm_bwd_scratch_rows(int num_sms);
cudaError_t rope_inplace(__nv_bfloat16* qkv, int64_t ld, int T, int t0, int heads, int d,
                         const float* cos_t, const float* sin_t, int k_offset, int dir,
                         cudaStream_t st, int num_sms);
cudaError_t swiglu_bwd(const __nv_bfloat16* da, const __nv_bfloat16* gu, __nv_bfloat16* dgu, int T,
                       int I, cudaStream_t st, int num_sms);

// ---- attention.cu ---------------------------------------------------------
// Causal attention over S tokens for `heads` heads of width d (64 or 128).
// Q/K/V/O rows are `ld*` elements apart per token; head h starts at column h*d.
// lse: fp32 [heads, S] (natural log).
// Fused all-to-all of the attention outputs (d = 128 tcgen05 kernels): rows are global tokens
// s; row s belongs to rank s / T and lands in that rank's token-sharded buffer (row s % T,
// row stride ld) at column col_* (which already includes this rank's head offset).
struct AttnPush {
  void* p[8];
  int T;
  int64_t ld;
  int64_t col_o, col_q, col_k, col_v;
};

struct AttnTensors {
  const __nv_bfloat16* q;
  const __nv_bfloat16* k;
  const __nv_bfloat16* v;
  int64_t ld_qkv;
  __nv_bfloat16* o;
  int64_t ld_o;
  float* lse;
  int S, heads, d;
  AttnPush push;  // push.p[0] == nullptr: outputs stay local
  // backward only: inverse rotary embedding of dq / dk (rotate-half, position = token row) applied
  // before they are rounded to bf16; [S, d/2] fp32 tables, nullptr = none
  const float* rope_cos = nullptr;
  const float* rope_sin = nullptr;
  // backward only: workspace of the stored-dS backward (attention_bwd_ds_tc); too small for one
  // head's dS tiles (attention_bwd_ds_head_bytes) selects the two-role kernel
  void* ds_ws = nullptr;
  int64_t ds_ws_bytes = 0;
};
cudaError_t attention_fwd(const AttnTensors& t, cudaStream_t st, int num_sms);
// tcgen05/TMEM/TMA forward (attention_tc.cu); attention_fwd dispatches here.
cudaError_t attention_fwd_tc(const AttnTensors& t, cudaStream_t st);
// tcgen05/TMEM backward for d = 128 (dK, dV written; dq_acc += scale * dS K, fp32).
cudaError_t attention_bwd_tc(const AttnTensors& t, const __nv_bfloat16* dout, int64_t ld_dout, __nv_bfloat16* dk,
                             __nv_bfloat16* dv, int64_t ld_d, const float* delta, float* dq_acc, cudaStream_t st);
// Atomic-free tcgen05 backward (d = 128, S % 128 == 0): one launch of key-tile (dK/dV) and
// query-tile (dQ) CTAs, every gradient accumulated in TMEM and written once in bf16; delta must be
// computed before, with nlse2 = -lse*log2(e) [heads, S]; t.push routes dq/dk/dv rows to their owner ranks.
cudaError_t attention_bwd_nored_tc(const AttnTensors& t, const __nv_bfloat16* dout, int64_t ld_dout, __nv_bfloat16* dq,
                                   __nv_bfloat16* dk, __nv_bfloat16* dv, int64_t ld_d, const float* delta,
                                   const float* nlse2, cudaStream_t st);
// Stored-dS backward (d = 128, S % 128 == 0): a key-tile launch (dK, dV, and every causal dS tile
// stored in bf16 to ws) and a dQ launch (dQ = dS K from the stored tiles) per group of heads whose
// dS fits ws (attention_bwd_ds_head_bytes(S) per head); otherwise as attention_bwd_nored_tc.
int64_t attention_bwd_ds_head_bytes(int S);
cudaError_t attention_bwd_ds_tc(const AttnTensors& t, const __nv_bfloat16* dout, int64_t ld_dout, __nv_bfloat16* dq,
                                __nv_bfloat16* dk, __nv_bfloat16* dv, int64_t ld_d, const float* delta,
                                const float* nlse2, void* ws, int64_t ws_bytes, cudaStream_t st);
// dq/dk/dv written (bf16) with row stride ld_dqkv; scratch: fp32 [heads*S] (delta) and
// fp32 [heads*S*d] (dq accumulator).
cudaError_t attention_bwd(const AttnTensors& t, const __nv_bfloat16* dout, __nv_bfloat16* dq,
                          __nv_bfloat16* dk, __nv_bfloat16* dv, int64_t ld_dqkv, float* delta,
                          float* dq_acc, cudaStream_t st, int num_sms);

// ---- comm.cu --------------------------------------------------------------
constexpr int kMaxRanks = 8;
struct PeerPtrs {
  void* p[kMaxRanks];
};
// Weight all-gather (pull): dst[q*shard + i] = src_q[i] for every rank q; src_q is rank
// q's bf16 working shard at the same symmetric offset. row_map != 0 applies the 64-row
// gate|up interleave (two tensors of `rows` x `cols` gathered into one [2*rows, cols]).
cudaError_t allgather_pull(const PeerPtrs& src, int world, int64_t shard_elems, __nv_bfloat16* dst,
                           cudaStream_t st, int num_sms, int num_ctas);
cudaError_t allgather_pull_interleave(const PeerPtrs& src_gate, const PeerPtrs& src_up, int world,
                                      int64_t rows, int64_t cols, __nv_bfloat16* dst,
                                      cudaStream_t st, int num_ctas);
// Gradient reduce-scatter fused with the cast/scale: out[i] (+)= scale * sum_q part_q[off + i]
// (bf16 or fp32 partials, fp32 accumulate, fixed rank order).
// NVLink SHARP reduce-scatter: this rank's shard of a bf16 partial whose every rank's copy is
// bound to one multicast object (mc_part = its multicast address), reduced in the switch
// (multimem.ld_reduce, fp32 accumulation); interleave_rows > 0: the gate|up layout of
// reduce_scatter_pull_interleave (out = gate, out_up = up shard).
cudaError_t nvls_reduce_scatter(const __nv_bfloat16* mc_part, int world, int rank, int64_t shard_elems,
                                int64_t interleave_rows, int64_t cols, float scale, int accumulate, float* out,
                                float* out_up, cudaStream_t st, int num_ctas);
cudaError_t reduce_scatter_pull(const PeerPtrs& part, int world, int rank, int64_t shard_elems,
                                bool part_is_f32, float scale, int accumulate, float* out,
                                cudaStream_t st, int num_ctas);
// Same for the interleaved gate|up partial [2*rows, cols]: produces this rank's gate and up
// shards (each rows*cols/world elements).
cudaError_t reduce_scatter_pull_interleave(const PeerPtrs& part, int world, int rank, int64_t rows,
                                           int64_t cols, float scale, int accumulate,
                                           float* out_gate, float* out_up, cudaStream_t st,
                                           int num_ctas);
// Ulysses all-to-all (pull). Token-sharded [T, parts*H] on every rank -> head-sharded
// [S, parts*Hl] on this rank (Hl = H/world). Optional RoPE on parts 0,1 (dir=+1).
cudaError_t a2a_tokens_to_heads(const PeerPtrs& src, int world, int rank, int T, int H, int parts,
                                __nv_bfloat16* dst, const float* cos_t, const float* sin_t, int d,
                                int rope_parts, cudaStream_t st, int num_ctas);
// Head-sharded [S, parts*Hl] on every rank -> token-sharded [T, parts*H] on this rank;
// optional inverse RoPE on parts 0,1 (the dq/dk path).
cudaError_t a2a_heads_to_tokens(const PeerPtrs& src, int world, int rank, int T, int H, int parts,
                                __nv_bfloat16* dst, const float* cos_t, const float* sin_t, int d,
                                int rope_parts, cudaStream_t st, int num_ctas);
// Push copy over peer memory: for every rank q (this rank included, as a local copy) and job,
// nblk blocks of blk bytes: dst_q[dst_off + b*dst_stride] <- src[q*src_q + b*src_stride].
// All-gather: src_q = 0 (the same shard to everyone), dst_off = this rank's slot.
// Reduce-scatter staging: src_q = owner q's slice stride, dst_off = this rank's slot.
struct PushJob {
  const char* src;
  int64_t src_q, dst_off, blk, src_stride, dst_stride, nblk;
};
struct PushJobs {
  PushJob j[2];
  int n;
};
// kind: kPushLsu (16-B vector stores, 256-thread CTAs, no shared memory), kPushBulk (one thread
// driving cp.async.bulk through 2 x 16 KB slots: co-resident with compute CTAs), kPushBulkWide
// (4 x 32 KB slots: one SM per CTA).
enum PushKind : int { kPushLsu = 0, kPushBulk = 1, kPushBulkWide = 2 };
cudaError_t push_copy(const PushJobs& jobs, const PeerPtrs& dst, int world, int rank, cudaStream_t st, int num_ctas,
                      int kind);
// NVLink SHARP all-gather push: every job's blocks stored once to the multicast address mc +
// dst_off (multimem.st; the switch writes all ranks' copies); jobs must have src_q == 0.
cudaError_t nvls_push(const PushJobs& jobs, char* mc, cudaStream_t st, int num_ctas);
// Cross-GPU barrier over system-scope flags in every rank's heap. epoch increases by one per
// call; a rank spins (bounded, ~20 s) until all peers have published `epoch`.
cudaError_t peer_barrier(const PeerPtrs& flags, int world, int rank, uint32_t epoch,
                         uint32_t* error_flag, cudaStream_t st);

}  // namespace isp
