// Causal flash attention, forward and backward, for the ISP block (sm_100a).
//
// Per rank this runs D/p heads over the full sequence after the Ulysses
// all-to-all (cost.hpp:217 prices it as
// 4*b*S*(S/sp)*H/tp, non-causal). The reference has no kernel; the algorithm is
// the standard online-softmax (FlashAttention).
//
// Version 1 uses the warp-level bf16 tensor-core path (mma.sync m16n8k16,
// ldmatrix from XOR-swizzled shared memory, cp.async double buffering). It is
// the correctness baseline; the tcgen05/TMEM version replaces it.
//
//   forward : CTA = 128 queries x 1 head, 8 warps x 16 rows, 64-key tiles.
//   backward: CTA = 128 keys x 1 head, 8 warps x 16 keys, 32-query tiles;
//             dK/dV in registers, dQ accumulated in fp32 with vector atomics.
#include <cuda_bf16.h>

#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace isp {

namespace {

constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void cp_async16(uint32_t smem, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// byte offset of 16-byte chunk `c` of row `r` in a swizzled tile with CH chunks per row
template <int CH>
__device__ __forceinline__ uint32_t swz(int r, int c) {
  return static_cast<uint32_t>(r * CH * 16 + ((c ^ (r & 7)) * 16));
}

// rows x (CH*8) bf16 tile from global (row stride ld elements) into swizzled smem
template <int CH, int NT>
__device__ __forceinline__ void load_tile(uint32_t smem, const __nv_bfloat16* g, int64_t ld,
                                          int rows) {
  for (int i = threadIdx.x; i < rows * CH; i += NT) {
    const int r = i / CH, c = i % CH;
    cp_async16(smem + swz<CH>(r, c), g + r * ld + c * 8);
  }
}

// ============================================================================
// forward
// ============================================================================
template <int D>
__global__ void __launch_bounds__(256, 1) attn_fwd_kernel(AttnTensors t, float scale_log2) {
  constexpr int BM = 128, BN = 64, CH = D / 8, NT = 256;
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t sQ = smem_u32(smem);
  const uint32_t sK = sQ + BM * D * 2;
  const uint32_t sV = sK + 2 * BN * D * 2;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int qt = gridDim.x - 1 - blockIdx.x;  // heavy (late) tiles first
  const int h = blockIdx.y;
  const int q0 = qt * BM;
  const int n_kv = (q0 + BM) / BN;
  const __nv_bfloat16* Qg = t.q + static_cast<int64_t>(q0) * t.ld_qkv + h * D;
  const __nv_bfloat16* Kg = t.k + h * D;
  const __nv_bfloat16* Vg = t.v + h * D;

  load_tile<CH, NT>(sQ, Qg, t.ld_qkv, BM);
  load_tile<CH, NT>(sK, Kg, t.ld_qkv, BN);
  load_tile<CH, NT>(sV, Vg, t.ld_qkv, BN);
  cp_commit();

  float o[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  uint32_t qf[D / 16][4];
  const int row_lo = q0 + warp * 16 + lane / 4;  // rows row_lo and row_lo + 8

  for (int j = 0; j < n_kv; ++j) {
    if (j + 1 < n_kv) {
      const int b = (j + 1) & 1;
      load_tile<CH, NT>(sK + b * BN * D * 2, Kg + static_cast<int64_t>(j + 1) * BN * t.ld_qkv,
                        t.ld_qkv, BN);
      load_tile<CH, NT>(sV + b * BN * D * 2, Vg + static_cast<int64_t>(j + 1) * BN * t.ld_qkv,
                        t.ld_qkv, BN);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    if (j == 0) {
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk)
        ldsm_x4(qf[kk], sQ + swz<CH>(warp * 16 + (lane % 16), kk * 2 + lane / 16));
    }
    const uint32_t kb = sK + (j & 1) * BN * D * 2;
    const uint32_t vb = sV + (j & 1) * BN * D * 2;

    float s[BN / 8][4];
#pragma unroll
    for (int i = 0; i < BN / 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
#pragma unroll
      for (int np = 0; np < BN / 16; ++np) {
        uint32_t b[4];
        ldsm_x4(b, kb + swz<CH>(np * 16 + (lane % 8) + (lane / 16) * 8, kk * 2 + ((lane / 8) & 1)));
        mma16816(s[2 * np], qf[kk], b[0], b[1]);
        mma16816(s[2 * np + 1], qf[kk], b[2], b[3]);
      }
    }
    // scale + causal mask
    const bool diag = (j * BN + BN - 1) > (q0 + warp * 16);
    float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
    for (int nt = 0; nt < BN / 8; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float v = s[nt][e] * scale_log2;
        if (diag) {
          const int key = j * BN + nt * 8 + (lane % 4) * 2 + (e & 1);
          const int row = row_lo + (e >> 1) * 8;
          if (key > row) v = -INFINITY;
        }
        s[nt][e] = v;
      }
      mx0 = fmaxf(mx0, fmaxf(s[nt][0], s[nt][1]));
      mx1 = fmaxf(mx1, fmaxf(s[nt][2], s[nt][3]));
    }
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
    const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
    const float a0 = exp2f(m0 - mn0), a1 = exp2f(m1 - mn1);
    m0 = mn0;
    m1 = mn1;
    l0 *= a0;
    l1 *= a1;
#pragma unroll
    for (int i = 0; i < D / 8; ++i) {
      o[i][0] *= a0; o[i][1] *= a0; o[i][2] *= a1; o[i][3] *= a1;
    }
#pragma unroll
    for (int nt = 0; nt < BN / 8; ++nt) {
      s[nt][0] = exp2f(s[nt][0] - mn0);
      s[nt][1] = exp2f(s[nt][1] - mn0);
      s[nt][2] = exp2f(s[nt][2] - mn1);
      s[nt][3] = exp2f(s[nt][3] - mn1);
      l0 += s[nt][0] + s[nt][1];
      l1 += s[nt][2] + s[nt][3];
    }
    // O += P V
#pragma unroll
    for (int kk = 0; kk < BN / 16; ++kk) {
      uint32_t pa[4];
      pa[0] = pack_bf16(s[2 * kk][0], s[2 * kk][1]);
      pa[1] = pack_bf16(s[2 * kk][2], s[2 * kk][3]);
      pa[2] = pack_bf16(s[2 * kk + 1][0], s[2 * kk + 1][1]);
      pa[3] = pack_bf16(s[2 * kk + 1][2], s[2 * kk + 1][3]);
#pragma unroll
      for (int dp = 0; dp < D / 16; ++dp) {
        uint32_t b[4];
        ldsm_x4_t(b, vb + swz<CH>(kk * 16 + (lane % 8) + ((lane / 8) & 1) * 8, dp * 2 + lane / 16));
        mma16816(o[2 * dp], pa, b[0], b[1]);
        mma16816(o[2 * dp + 1], pa, b[2], b[3]);
      }
    }
    __syncthreads();
  }
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  const float inv0 = 1.f / l0, inv1 = 1.f / l1;
  __nv_bfloat16* O0 = t.o + static_cast<int64_t>(row_lo) * t.ld_o + h * D + (lane % 4) * 2;
  __nv_bfloat16* O1 = O0 + 8 * t.ld_o;
#pragma unroll
  for (int i = 0; i < D / 8; ++i) {
    *reinterpret_cast<uint32_t*>(O0 + i * 8) = pack_bf16(o[i][0] * inv0, o[i][1] * inv0);
    *reinterpret_cast<uint32_t*>(O1 + i * 8) = pack_bf16(o[i][2] * inv1, o[i][3] * inv1);
  }
  if ((lane % 4) == 0) {
    const float ln2 = 0.6931471805599453f;
    t.lse[static_cast<int64_t>(h) * t.S + row_lo] = (m0 + log2f(l0)) * ln2;
    t.lse[static_cast<int64_t>(h) * t.S + row_lo + 8] = (m1 + log2f(l1)) * ln2;
  }
}

// ============================================================================
// backward
// ============================================================================
// delta[h, t] = sum_d dO[t, h*D + d] * O[t, h*D + d]
template <int D>
__global__ void attn_delta_kernel(const __nv_bfloat16* __restrict__ o, int64_t ld_o,
                                  const __nv_bfloat16* __restrict__ dout, float* __restrict__ delta,
                                  int S, int heads, const float* __restrict__ lse = nullptr,
                                  float* __restrict__ nlse2 = nullptr) {
  const int warps = blockDim.x / 32;
  const int64_t n = static_cast<int64_t>(S) * heads;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(warps) + threadIdx.x / 32; i < n;
       i += static_cast<int64_t>(gridDim.x) * warps) {
    const int tok = static_cast<int>(i / heads), h = static_cast<int>(i % heads);
    const int lane = threadIdx.x % 32;
    float acc = 0.f;
    for (int c = lane * 2; c < D; c += 64) {
      const int64_t off = static_cast<int64_t>(tok) * ld_o + h * D + c;
      const float2 a = unpack_bf16(*reinterpret_cast<const uint32_t*>(o + off));
      const float2 b = unpack_bf16(*reinterpret_cast<const uint32_t*>(dout + off));
      acc += a.x * b.x + a.y * b.y;
    }
    acc = warp_sum(acc);
    if (lane == 0) delta[static_cast<int64_t>(h) * S + tok] = acc;
    if (nlse2 && lane == 1) {  // -lse * log2(e): the exponent offset of the tcgen05 backward
      const int64_t k = static_cast<int64_t>(h) * S + tok;
      nlse2[k] = -lse[k] * kLog2e;
    }
  }
}

template <int D>
__global__ void __launch_bounds__(256, 1) attn_bwd_kernel(AttnTensors t,
                                                         const __nv_bfloat16* __restrict__ dout,
                                                         __nv_bfloat16* __restrict__ dk_out,
                                                         __nv_bfloat16* __restrict__ dv_out,
                                                         int64_t ld_d, const float* __restrict__ delta,
                                                         float* __restrict__ dq_acc, float scale) {
  constexpr int BN = 128, BM = 32, CH = D / 8, NT = 256, DS_LD = BM + 8;
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t sK = smem_u32(smem);
  const uint32_t sV = sK + BN * D * 2;
  const uint32_t sQ = sV + BN * D * 2;          // [2][BM][D]
  const uint32_t sdO = sQ + 2 * BM * D * 2;     // [2][BM][D]
  const uint32_t sdS = sdO + 2 * BM * D * 2;    // [BN][DS_LD] bf16, padded
  float* sL = reinterpret_cast<float*>(smem + (sdS - sK) + BN * DS_LD * 2);  // [2][BM] lse*log2e
  float* sD = sL + 2 * BM;                                                    // [2][BM] delta
  __nv_bfloat16* dS_ptr = reinterpret_cast<__nv_bfloat16*>(smem + (sdS - sK));

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int kt = blockIdx.x, h = blockIdx.y;
  const int k0 = kt * BN;
  const float scale_log2 = scale * kLog2e;
  const __nv_bfloat16* Qg = t.q + h * D;
  const __nv_bfloat16* dOg = dout + h * D;
  const float* lse_h = t.lse + static_cast<int64_t>(h) * t.S;
  const float* del_h = delta + static_cast<int64_t>(h) * t.S;

  load_tile<CH, NT>(sK, t.k + static_cast<int64_t>(k0) * t.ld_qkv + h * D, t.ld_qkv, BN);
  load_tile<CH, NT>(sV, t.v + static_cast<int64_t>(k0) * t.ld_qkv + h * D, t.ld_qkv, BN);
  const int qt0 = k0 / BM, nq = t.S / BM;
  auto load_q = [&](int qt, int b) {
    load_tile<CH, NT>(sQ + b * BM * D * 2, Qg + static_cast<int64_t>(qt) * BM * t.ld_qkv, t.ld_qkv, BM);
    load_tile<CH, NT>(sdO + b * BM * D * 2, dOg + static_cast<int64_t>(qt) * BM * t.ld_o, t.ld_o, BM);
    if (threadIdx.x < BM) {
      sL[b * BM + threadIdx.x] = lse_h[qt * BM + threadIdx.x] * kLog2e;
      sD[b * BM + threadIdx.x] = del_h[qt * BM + threadIdx.x];
    }
  };
  load_q(qt0, 0);
  cp_commit();

  float dk[D / 8][4], dv[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) dk[i][e] = dv[i][e] = 0.f;
  const int key_lo = k0 + warp * 16 + lane / 4;  // keys key_lo, key_lo + 8

  for (int qt = qt0; qt < nq; ++qt) {
    const int b = (qt - qt0) & 1;
    if (qt + 1 < nq) {
      load_q(qt + 1, b ^ 1);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const uint32_t qb = sQ + b * BM * D * 2, ob = sdO + b * BM * D * 2;
    const int q0 = qt * BM;

    // S^T = K_w Q^T and dP^T = V_w dO^T   (16 keys x 32 queries per warp)
    float st[BM / 8][4], dpt[BM / 8][4];
#pragma unroll
    for (int i = 0; i < BM / 8; ++i)
#pragma unroll
      for (int e = 0; e < 4; ++e) st[i][e] = dpt[i][e] = 0.f;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      uint32_t ka[4], va[4];
      ldsm_x4(ka, sK + swz<CH>(warp * 16 + (lane % 16), kk * 2 + lane / 16));
      ldsm_x4(va, sV + swz<CH>(warp * 16 + (lane % 16), kk * 2 + lane / 16));
#pragma unroll
      for (int np = 0; np < BM / 16; ++np) {
        uint32_t bq[4], bo[4];
        const int r = np * 16 + (lane % 8) + (lane / 16) * 8, c = kk * 2 + ((lane / 8) & 1);
        ldsm_x4(bq, qb + swz<CH>(r, c));
        ldsm_x4(bo, ob + swz<CH>(r, c));
        mma16816(st[2 * np], ka, bq[0], bq[1]);
        mma16816(st[2 * np + 1], ka, bq[2], bq[3]);
        mma16816(dpt[2 * np], va, bo[0], bo[1]);
        mma16816(dpt[2 * np + 1], va, bo[2], bo[3]);
      }
    }
    // P^T, dS^T
    const bool diag = q0 < k0 + warp * 16 + 16;
#pragma unroll
    for (int nt = 0; nt < BM / 8; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int ql = nt * 8 + (lane % 4) * 2 + (e & 1);
        const int key = key_lo + (e >> 1) * 8;
        float p = exp2f(st[nt][e] * scale_log2 - sL[b * BM + ql]);
        if (diag && key > q0 + ql) p = 0.f;
        st[nt][e] = p;
        dpt[nt][e] = p * (dpt[nt][e] - sD[b * BM + ql]);
      }
    }
    // dV += P^T dO ; dK += dS^T Q
#pragma unroll
    for (int kk = 0; kk < BM / 16; ++kk) {
      uint32_t pa[4], da[4];
      pa[0] = pack_bf16(st[2 * kk][0], st[2 * kk][1]);
      pa[1] = pack_bf16(st[2 * kk][2], st[2 * kk][3]);
      pa[2] = pack_bf16(st[2 * kk + 1][0], st[2 * kk + 1][1]);
      pa[3] = pack_bf16(st[2 * kk + 1][2], st[2 * kk + 1][3]);
      da[0] = pack_bf16(dpt[2 * kk][0], dpt[2 * kk][1]);
      da[1] = pack_bf16(dpt[2 * kk][2], dpt[2 * kk][3]);
      da[2] = pack_bf16(dpt[2 * kk + 1][0], dpt[2 * kk + 1][1]);
      da[3] = pack_bf16(dpt[2 * kk + 1][2], dpt[2 * kk + 1][3]);
#pragma unroll
      for (int dp = 0; dp < D / 16; ++dp) {
        uint32_t bo[4], bq[4];
        const int r = kk * 16 + (lane % 8) + ((lane / 8) & 1) * 8, c = dp * 2 + lane / 16;
        ldsm_x4_t(bo, ob + swz<CH>(r, c));
        ldsm_x4_t(bq, qb + swz<CH>(r, c));
        mma16816(dv[2 * dp], pa, bo[0], bo[1]);
        mma16816(dv[2 * dp + 1], pa, bo[2], bo[3]);
        mma16816(dk[2 * dp], da, bq[0], bq[1]);
        mma16816(dk[2 * dp + 1], da, bq[2], bq[3]);
      }
    }
    // dS^T -> smem (bf16), then dQ(32 x D) = dS (32 x 128) K (128 x D)
#pragma unroll
    for (int nt = 0; nt < BM / 8; ++nt) {
      const int ql = nt * 8 + (lane % 4) * 2;
      const int kr = warp * 16 + lane / 4;
      *reinterpret_cast<uint32_t*>(dS_ptr + kr * DS_LD + ql) = pack_bf16(dpt[nt][0], dpt[nt][1]);
      *reinterpret_cast<uint32_t*>(dS_ptr + (kr + 8) * DS_LD + ql) = pack_bf16(dpt[nt][2], dpt[nt][3]);
    }
    __syncthreads();
    {
      constexpr int DW = D / 4;  // d columns per warp (warps: 2 query halves x 4 d quarters)
      const int qh = warp & 1, dq4 = warp >> 1;
      float acc[DW / 8][4];
#pragma unroll
      for (int i = 0; i < DW / 8; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < BN / 16; ++kk) {
        uint32_t a[4];
        const int row = kk * 16 + (lane % 8) + (lane / 16) * 8;
        const int chunk = qh * 2 + ((lane / 8) & 1);
        ldsm_x4_t(a, sdS + static_cast<uint32_t>(row * DS_LD * 2 + chunk * 16));
#pragma unroll
        for (int dp = 0; dp < DW / 16; ++dp) {
          uint32_t bk[4];
          ldsm_x4_t(bk, sK + swz<CH>(kk * 16 + (lane % 8) + ((lane / 8) & 1) * 8,
                                     dq4 * (DW / 8) + dp * 2 + lane / 16));
          mma16816(acc[2 * dp], a, bk[0], bk[1]);
          mma16816(acc[2 * dp + 1], a, bk[2], bk[3]);
        }
      }
      float* dq_h = dq_acc + static_cast<int64_t>(h) * t.S * D;
      const int qr = q0 + qh * 16 + lane / 4;
#pragma unroll
      for (int nt = 0; nt < DW / 8; ++nt) {
        const int col = dq4 * DW + nt * 8 + (lane % 4) * 2;
        atomicAdd(reinterpret_cast<float2*>(dq_h + static_cast<int64_t>(qr) * D + col),
                  make_float2(acc[nt][0], acc[nt][1]));
        atomicAdd(reinterpret_cast<float2*>(dq_h + static_cast<int64_t>(qr + 8) * D + col),
                  make_float2(acc[nt][2], acc[nt][3]));
      }
    }
    __syncthreads();
  }
  // write dK (scaled) and dV
  __nv_bfloat16* DK0 = dk_out + static_cast<int64_t>(key_lo) * ld_d + h * D + (lane % 4) * 2;
  __nv_bfloat16* DV0 = dv_out + static_cast<int64_t>(key_lo) * ld_d + h * D + (lane % 4) * 2;
#pragma unroll
  for (int i = 0; i < D / 8; ++i) {
    *reinterpret_cast<uint32_t*>(DK0 + i * 8) = pack_bf16(dk[i][0] * scale, dk[i][1] * scale);
    *reinterpret_cast<uint32_t*>(DK0 + 8 * ld_d + i * 8) = pack_bf16(dk[i][2] * scale, dk[i][3] * scale);
    *reinterpret_cast<uint32_t*>(DV0 + i * 8) = pack_bf16(dv[i][0], dv[i][1]);
    *reinterpret_cast<uint32_t*>(DV0 + 8 * ld_d + i * 8) = pack_bf16(dv[i][2], dv[i][3]);
  }
}

// dq (bf16, row stride ld) = scale * dq_acc[h, t, :]
template <int D>
__global__ void attn_dq_convert_kernel(const float* __restrict__ dq_acc, __nv_bfloat16* __restrict__ dq,
                                       int64_t ld, int S, int heads, float scale, const __grid_constant__ AttnPush push) {
  const int64_t n = static_cast<int64_t>(heads) * S * (D / 4);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c4 = i % (D / 4);
    const int64_t row = i / (D / 4);  // h * S + t
    const int h = static_cast<int>(row / S), tok = static_cast<int>(row % S);
    const float4 v = *reinterpret_cast<const float4*>(dq_acc + row * D + c4 * 4);
    uint2 o;
    o.x = pack_bf16(v.x * scale, v.y * scale);
    o.y = pack_bf16(v.z * scale, v.w * scale);
    if (push.p[0]) {  // fused all-to-all: dq of token tok goes to its owner rank
      const int owner = tok / push.T;
      *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(push.p[owner]) +
                                static_cast<int64_t>(tok - owner * push.T) * push.ld + push.col_q + h * D + c4 * 4) = o;
    } else {
      *reinterpret_cast<uint2*>(dq + static_cast<int64_t>(tok) * ld + h * D + c4 * 4) = o;
    }
  }
  if (push.p[0]) __threadfence_system();  // pushed rows visible before the next barrier flag
}

template <int D>
cudaError_t fwd_impl(const AttnTensors& t, cudaStream_t st) {
  constexpr int smem = (128 * D + 4 * 64 * D) * 2;
  static bool set = false;
  if (!set) {
    cudaError_t e = cudaFuncSetAttribute(attn_fwd_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    set = true;
  }
  dim3 grid(t.S / 128, t.heads);
  const float scale_log2 = (1.0f / sqrtf(static_cast<float>(D))) * kLog2e;
  attn_fwd_kernel<D><<<grid, 256, smem, st>>>(t, scale_log2);
  return cudaGetLastError();
}

// Inverse RoPE of dq / dk for the backward variants that do not fuse it (the opt-in fused tcgen05
// kernel, the head-dim-64 mma.sync kernel): a separate pass over the head-sharded rows.
cudaError_t unrope_after(const AttnTensors& t, __nv_bfloat16* dq, __nv_bfloat16* dk, int64_t ld_d, cudaStream_t st,
                         int num_sms) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || !t.rope_cos) return e;
  if (t.push.p[0]) return cudaErrorInvalidValue;  // rows already pushed: only the fused-RoPE kernel may push
  return rope_inplace(dq, ld_d, t.S, 0, t.heads, t.d, t.rope_cos, t.rope_sin, static_cast<int>(dk - dq), -1, st,
                      num_sms);
}

template <int D>
cudaError_t bwd_impl(const AttnTensors& t, const __nv_bfloat16* dout, __nv_bfloat16* dq,
                     __nv_bfloat16* dk, __nv_bfloat16* dv, int64_t ld_d, float* delta,
                     float* dq_acc, cudaStream_t st, int num_sms) {
  constexpr int BN = 128, BM = 32;
  constexpr int smem = (2 * BN * D + 4 * BM * D + BN * (BM + 8)) * 2 + 4 * BM * 4;
  static bool set = false;
  if (!set) {
    cudaError_t e = cudaFuncSetAttribute(attn_bwd_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    set = true;
  }
  const float scale = 1.0f / sqrtf(static_cast<float>(D));
  if (D == 128 && !std::getenv("SEQPLAN_ISP_ATTN_MMA_SYNC") && !std::getenv("SEQPLAN_ISP_ATTN_FUSED_BWD")) {
    // production: atomic-free tcgen05 backward (attention_tc.cu attn_bwd_split_kernel)
    // dq_acc (unused by this path) holds -lse*log2e [heads, S]
    attn_delta_kernel<D><<<num_sms * 8, 256, 0, st>>>(t.o, t.ld_o, dout, delta, t.S, t.heads, t.lse, dq_acc);
    if (t.ds_ws && t.ds_ws_bytes >= attention_bwd_ds_head_bytes(t.S) && !std::getenv("SEQPLAN_ISP_ATTN_SPLIT_BWD"))
      return attention_bwd_ds_tc(t, dout, t.ld_o, dq, dk, dv, ld_d, delta, dq_acc, t.ds_ws, t.ds_ws_bytes, st);
    return attention_bwd_nored_tc(t, dout, t.ld_o, dq, dk, dv, ld_d, delta, dq_acc, st);
  }
  cudaError_t e = cudaMemsetAsync(dq_acc, 0, sizeof(float) * static_cast<size_t>(t.heads) * t.S * D, st);
  if (e != cudaSuccess) return e;
  attn_delta_kernel<D><<<num_sms * 8, 256, 0, st>>>(t.o, t.ld_o, dout, delta, t.S, t.heads);
  if (D == 128 && !std::getenv("SEQPLAN_ISP_ATTN_MMA_SYNC")) {
    // tcgen05/TMEM backward (attention_tc.cu); it applies the softmax scale to dq_acc itself
    e = attention_bwd_tc(t, dout, t.ld_o, dk, dv, ld_d, delta, dq_acc, st);
    if (e != cudaSuccess) return e;
    attn_dq_convert_kernel<D><<<num_sms * 8, 256, 0, st>>>(dq_acc, dq, ld_d, t.S, t.heads, 1.0f, t.push);
    return unrope_after(t, dq, dk, ld_d, st, num_sms);
  }
  attn_bwd_kernel<D><<<dim3(t.S / BN, t.heads), 256, smem, st>>>(t, dout, dk, dv, ld_d, delta, dq_acc, scale);
  if (t.push.p[0]) return cudaErrorInvalidValue;  // fused all-to-all needs the tcgen05 kernels
  attn_dq_convert_kernel<D><<<num_sms * 8, 256, 0, st>>>(dq_acc, dq, ld_d, t.S, t.heads, scale, t.push);
  return unrope_after(t, dq, dk, ld_d, st, num_sms);
}

}  // namespace

cudaError_t attention_fwd(const AttnTensors& t, cudaStream_t st, int num_sms) {
  (void)num_sms;
  if (t.S % 128) return cudaErrorInvalidValue;
  if (!std::getenv("SEQPLAN_ISP_ATTN_MMA_SYNC") || t.push.p[0]) return attention_fwd_tc(t, st);
  if (t.d == 128) return fwd_impl<128>(t, st);
  if (t.d == 64) return fwd_impl<64>(t, st);
  return cudaErrorInvalidValue;
}

cudaError_t attention_bwd(const AttnTensors& t, const __nv_bfloat16* dout, __nv_bfloat16* dq,
                          __nv_bfloat16* dk, __nv_bfloat16* dv, int64_t ld_dqkv, float* delta,
                          float* dq_acc, cudaStream_t st, int num_sms) {
  if (t.S % 128) return cudaErrorInvalidValue;
  if (t.d == 128) return bwd_impl<128>(t, dout, dq, dk, dv, ld_dqkv, delta, dq_acc, st, num_sms);
  if (t.d == 64) return bwd_impl<64>(t, dout, dq, dk, dv, ld_dqkv, delta, dq_acc, st, num_sms);
  return cudaErrorInvalidValue;
}

}  // namespace isp
