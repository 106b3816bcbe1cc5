// Host interface of the tcgen05 GEMM (see gemm.cu).
#pragma once

#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace isp {

// gate|up are interleaved in blocks of kGuBlock rows (weights) / columns (activations) so one
// GEMM produces both and its epilogue applies SwiGLU. 32 keeps every rank's I/p-row shard
// (I % 256 == 0, p <= 8) block-aligned, so gathers are strided copy-engine copies.
constexpr int kGuBlock = 32;

enum GemmEpilogue : int {
  EPI_BF16 = 0,        // out(bf16) = scale * acc
  EPI_BF16_RESID = 1,  // out(bf16) = scale * acc + resid(bf16)
  EPI_SWIGLU = 2,      // out(bf16) = acc (gate/up interleaved by kGuBlock cols); out2 = silu(g) * u
  EPI_F32 = 3,         // out(f32) (+)= scale * acc; optional kGuBlock-row gate/up de-interleave
  EPI_SWIGLU_BWD = 4,  // da = bf16(scale * acc) (N = I columns); out(bf16) = dgu, kGuBlock-col
                       // interleaved gate|up grads from da and the saved gu passed as resid [M, 2N]
};

// One GEMM operand. Logical shape is [rows, K] (A: rows = M, B: rows = N).
// K-major: stored row-major as [rows, K] with leading dimension ld.
// MN-major: stored row-major as [K, rows] with leading dimension ld.
struct GemmOperand {
  const void* ptr;
  int64_t ld;
  bool mn_major;
};

struct GemmArgs {
  int M = 0, N = 0, K = 0;
  void* out = nullptr;  // bf16 or f32
  int64_t ldo = 0;
  const __nv_bfloat16* resid = nullptr;
  int64_t ldr = 0;
  __nv_bfloat16* out2 = nullptr;  // SwiGLU activation [M, N/2]
  int64_t ldo2 = 0;
  float* out_b = nullptr;  // EPI_F32 + interleave64: destination of odd 64-row blocks
  float scale = 1.0f;
  int accumulate = 0;
  int interleave64 = 0;
  // Fused Ulysses all-to-all (EPI_BF16 only): when push[0] != nullptr the [T, parts*H] tile is
  // not stored locally; each head's columns go straight to the rank owning that head, into its
  // head-sharded buffer [S, parts*Hl] at row rank*T + row (NVLink stores from the epilogue).
  // RoPE (rotate-half, position = rank*T + row) is applied to parts < rope_parts on the way.
  void* push[8] = {};
  int push_T = 0, push_rank = 0, push_parts = 1, push_H = 0, push_Hl = 0, push_d = 128;
  const float* rope_cos = nullptr;
  const float* rope_sin = nullptr;
  int rope_parts = 0;
  // logical column of this GEMM's column 0 in the [parts*H] row (a GEMM over a column slice of
  // the QKV projection): selects the part / head for RoPE and the push target
  int rope_col0 = 0;
  // persistent-grid size limit (0 = every SM): SMs held by concurrent bulk-copy comm kernels
  // are left out so no CTA of the persistent grid waits for them
  int sm_budget = 0;
  // tile order: groups of group_m row-blocks walk the N dimension together (L2 reuse of A and B)
  int group_m = 16;
  // Split-K of the last partial wave (CTA-pair kernel; set by gemm_launch, not by callers): the
  // first split_base tiles run whole; each of the remaining split_L tiles is cut into split_s
  // K-ranges run concurrently in the last wave. Finishers but the last leave fp32 partials in
  // split_ws and raise their ready flag; the last adds them and runs the fused epilogue.
  int split_base = 0, split_L = 0, split_s = 1;
  float* split_ws = nullptr;
  uint32_t* split_cnt = nullptr;    // [L][2] arrivals per (tile, CTA of the pair); self-resetting
  uint32_t* split_ready = nullptr;  // [L][s-1][2] partial p of (tile, CTA) written; self-resetting
  // Wave pacing (CTA-pair kernel): a cluster starts
  // loading its tile of wave w only after every cluster has issued the loads of wave w-1, so the
  // tiles of one wave stream the same K-slices of the shared panels through L2 together instead of
  // drifting apart over the waves (7B-32K step: GEMM DRAM traffic 74.9 -> 46.1 GB, -7 % GEMM time
  // in ncu, +1 % end to end under the power cap). Needs every cluster of the grid resident at once:
  // callers whose GEMMs may run concurrently with another persistent grid clear wave_sync.
  int wave_sync = 1;  // SEQPLAN_GEMM_WAVE_SYNC=0 turns it off everywhere
  uint32_t* wave_cnt = nullptr;  // zeroed per launch by gemm_launch
};

int gemm_pick_bn(int N);
cudaError_t gemm_launch(const GemmOperand& A, const GemmOperand& B, GemmArgs args, int epi,
                        cudaStream_t stream);

}  // namespace isp
