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
