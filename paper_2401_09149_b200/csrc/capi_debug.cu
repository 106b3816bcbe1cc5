#include <cstdio>
// Kernel-level C-ABI entry points used by the unit/parity tests.
//
// These expose the individual sm_100a kernels (GEMM, norms, attention,
// collectives) with plain device pointers so that tests can check each one in
// isolation before the block-level entry points (capi.cpp) are exercised.
#include <cstdint>

#include "../../include/seqplan_isp.h"
#include "gemm.h"

extern "C" int seqplan_isp_debug_gemm(const void* a, int64_t lda, int a_mn, const void* b,
                                      int64_t ldb, int b_mn, void* out, int64_t ldo, int M,
                                      int N, int K, int epi, const void* resid, int64_t ldr,
                                      void* out2, int64_t ldo2, void* out_b, float scale,
                                      int accumulate, int interleave64, void* stream) {
  isp::GemmOperand A{a, lda, a_mn != 0};
  isp::GemmOperand B{b, ldb, b_mn != 0};
  isp::GemmArgs args;
  args.M = M;
  args.N = N;
  args.K = K;
  args.out = out;
  args.ldo = ldo;
  args.resid = static_cast<const __nv_bfloat16*>(resid);
  args.ldr = ldr;
  args.out2 = static_cast<__nv_bfloat16*>(out2);
  args.ldo2 = ldo2;
  args.out_b = static_cast<float*>(out_b);
  args.scale = scale;
  args.accumulate = accumulate;
  args.interleave64 = interleave64;
  cudaError_t e = isp::gemm_launch(A, B, args, epi, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SEQPLAN_ISP_OK : SEQPLAN_ISP_ERR_RUNTIME;
}

#include "kernels.h"

extern "C" int seqplan_isp_debug_attention_ws(const void* q, const void* k, const void* v, int64_t ld_qkv,
                                              void* o, int64_t ld_o, float* lse, int S, int heads, int d,
                                              const void* dout, void* dq, void* dk, void* dv, int64_t ld_d,
                                              float* delta, float* dq_acc, void* ws, int64_t ws_bytes,
                                              void* stream) {
  isp::AttnTensors t{};
  t.ds_ws = ws;
  t.ds_ws_bytes = ws_bytes;
  t.q = static_cast<const __nv_bfloat16*>(q);
  t.k = static_cast<const __nv_bfloat16*>(k);
  t.v = static_cast<const __nv_bfloat16*>(v);
  t.ld_qkv = ld_qkv;
  t.o = static_cast<__nv_bfloat16*>(o);
  t.ld_o = ld_o;
  t.lse = lse;
  t.S = S;
  t.heads = heads;
  t.d = d;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaError_t e;
  if (!dout) {
    e = isp::attention_fwd(t, st, sms);
  } else {
    e = isp::attention_bwd(t, static_cast<const __nv_bfloat16*>(dout), static_cast<__nv_bfloat16*>(dq),
                           static_cast<__nv_bfloat16*>(dk), static_cast<__nv_bfloat16*>(dv), ld_d, delta,
                           dq_acc, st, sms);
  }
  if (e != cudaSuccess) fprintf(stderr, "seqplan_isp_debug_attention: %s\n", cudaGetErrorString(e));
  return e == cudaSuccess ? SEQPLAN_ISP_OK : SEQPLAN_ISP_ERR_RUNTIME;
}

extern "C" int seqplan_isp_debug_attention(const void* q, const void* k, const void* v, int64_t ld_qkv,
                                           void* o, int64_t ld_o, float* lse, int S, int heads, int d,
                                           const void* dout, void* dq, void* dk, void* dv, int64_t ld_d,
                                           float* delta, float* dq_acc, void* stream) {
  return seqplan_isp_debug_attention_ws(q, k, v, ld_qkv, o, ld_o, lse, S, heads, d, dout, dq, dk, dv, ld_d, delta,
                                        dq_acc, nullptr, 0, stream);
}

extern "C" int64_t seqplan_isp_debug_attention_ds_bytes(int S) { return isp::attention_bwd_ds_head_bytes(S); }

extern "C" int seqplan_isp_debug_rmsnorm(const void* x, const void* g, void* y, float* rstd, const void* dn,
                                         const void* dres, void* dx, float* dg, int T, int H, float eps,
                                         void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  if (!dn)
    e = isp::rmsnorm_fwd(static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(g),
                         static_cast<__nv_bfloat16*>(y), rstd, T, H, eps, st, 148);
  else
    e = isp::rmsnorm_bwd(static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(g), rstd,
                         static_cast<const __nv_bfloat16*>(dn), static_cast<const __nv_bfloat16*>(dres),
                         static_cast<__nv_bfloat16*>(dx), dg, T, H, st, 148);
  return e == cudaSuccess ? SEQPLAN_ISP_OK : SEQPLAN_ISP_ERR_RUNTIME;
}

// Ulysses all-to-all of one rank (dir = +1: token-sharded [T, parts*H] on every rank -> this
// rank's head-sharded [S, parts*Hl]; dir = -1: the reverse), src[q] = rank q's buffer; no RoPE
// when cos_t == NULL. The kernels the block runs after the QKV GEMM / before the O projection.
extern "C" int seqplan_isp_debug_all_to_all(int world, int rank, int T, int H, int parts, int d, int dir,
                                            const void* const* src, void* dst, const float* cos_t,
                                            const float* sin_t, int rope_parts, void* stream) {
  if (world < 1 || world > isp::kMaxRanks || rank < 0 || rank >= world || !src || !dst)
    return SEQPLAN_ISP_ERR_INVALID;
  isp::PeerPtrs p{};
  for (int q = 0; q < world; ++q) p.p[q] = const_cast<void*>(src[q]);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int rp = cos_t ? rope_parts : 0;
  cudaError_t e = dir > 0 ? isp::a2a_tokens_to_heads(p, world, rank, T, H, parts, static_cast<__nv_bfloat16*>(dst),
                                                      cos_t, sin_t, d, rp, st, 592)
                          : isp::a2a_heads_to_tokens(p, world, rank, T, H, parts, static_cast<__nv_bfloat16*>(dst),
                                                     cos_t, sin_t, d, rp, st, 592);
  if (e == cudaErrorInvalidValue) return SEQPLAN_ISP_ERR_INVALID;
  return e == cudaSuccess ? SEQPLAN_ISP_OK : SEQPLAN_ISP_ERR_RUNTIME;
}

// Gradient reduce-scatter of one rank fused with the cast / scale: out[i] (+)= scale * sum over
// q = 0..world-1 (in that order, fp32) of part[q][rank * shard + i]; part bf16 or fp32.
extern "C" int seqplan_isp_debug_reduce_scatter(int world, int rank, int64_t shard_elems, const void* const* part,
                                                int part_is_f32, float scale, int accumulate, float* out,
                                                void* stream) {
  if (world < 1 || world > isp::kMaxRanks || rank < 0 || rank >= world || !part || !out)
    return SEQPLAN_ISP_ERR_INVALID;
  isp::PeerPtrs p{};
  for (int q = 0; q < world; ++q) p.p[q] = const_cast<void*>(part[q]);
  cudaError_t e = isp::reduce_scatter_pull(p, world, rank, shard_elems, part_is_f32 != 0, scale, accumulate, out,
                                           static_cast<cudaStream_t>(stream), 592);
  if (e == cudaErrorInvalidValue) return SEQPLAN_ISP_ERR_INVALID;
  return e == cudaSuccess ? SEQPLAN_ISP_OK : SEQPLAN_ISP_ERR_RUNTIME;
}

// One rank's push all-gather of a contiguous shard (the weight all-gather transport of p >= 4):
// this rank's `bytes` at src are stored into slot `rank` (offset rank*bytes) of every rank's
// buffer dst[q] (own slot: a local copy). kind: 0 = 16-B vector stores (push_copy_kernel),
// 1 = one thread per CTA driving cp.async.bulk through 2 x 16 KB slots (push_bulk_kernel).
extern "C" int seqplan_isp_debug_push_allgather(int world, int rank, void* const* dst, const void* src, int64_t bytes,
                                                int kind, int num_ctas, void* stream) {
  if (world < 1 || world > isp::kMaxRanks || rank < 0 || rank >= world || !dst || !src || bytes % 16 ||
      (kind != 0 && kind != 1) || num_ctas < 1)
    return SEQPLAN_ISP_ERR_INVALID;
  isp::PeerPtrs p{};
  for (int q = 0; q < world; ++q) p.p[q] = dst[q];
  isp::PushJobs J{};
  J.j[0] = isp::PushJob{static_cast<const char*>(src), 0, rank * bytes, bytes, 0, 0, 1};
  J.n = 1;
  cudaError_t e = isp::push_copy(J, p, world, rank, static_cast<cudaStream_t>(stream), num_ctas,
                                 kind == 1 ? isp::kPushBulk : isp::kPushLsu);
  if (e == cudaErrorInvalidValue) return SEQPLAN_ISP_ERR_INVALID;
  return e == cudaSuccess ? SEQPLAN_ISP_OK : SEQPLAN_ISP_ERR_RUNTIME;
}
