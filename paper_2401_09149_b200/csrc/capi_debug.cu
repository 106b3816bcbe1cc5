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

extern "C" int seqplan_isp_debug_attention(const void* q, const void* k, const void* v, int64_t ld_qkv,
                                           void* o, int64_t ld_o, float* lse, int S, int heads, int d,
                                           const void* dout, void* dq, void* dk, void* dv, int64_t ld_d,
                                           float* delta, float* dq_acc, void* stream) {
  isp::AttnTensors t{};
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
