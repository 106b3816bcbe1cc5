// Causal flash-attention forward on tcgen05 / TMEM / TMA (sm_100a).
//
// Per rank this is the attention of D/p heads over the full sequence after the Ulysses
// all-to-all (priced at cost.hpp:217). CTA = 128 queries x 1 head.
//   warp 0      TMA producer: Q once, then K/V tiles of 64 keys into a 2-stage ring
//   warp 1      MMA issuer (one lane): S_j = Q K_j^T into a double-buffered TMEM S, then
//               O += P_{j-1} V_{j-1} with O resident in TMEM (software-pipelined by one tile)
//   warps 2..5  softmax, one thread per query row (= TMEM lane): S row from TMEM, online
//               softmax in exp2 with a stale-max rule (O rescaled in TMEM only when the row
//               max grows by > 2^8, warp-uniformly), P (bf16) into a double-buffered
//               SW128 smem tile that is the A operand of the PV MMA; epilogue O / l -> bf16.
// Shared memory (d = 128): Q 32 KB + K/V 2 x 32 KB + P 2 x 16 KB = 128 KB; TMEM 256 columns.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <type_traits>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace isp {

extern long long* g_attn_trace_fwd;  // development hook (seqplan_isp_debug_set_trace_fwd)

namespace {

constexpr int kBM = 128;      // queries per CTA
constexpr int kThreads = 320;  // warp 0 TMA, warp 1 MMA, warps 2..9 softmax
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kRescaleThreshold = 8.0f;  // log2 units

__device__ __forceinline__ void tmem_st_32x32b_x32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
      "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]),
      "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// CW consecutive TMEM columns of this thread's lane (CW = 32 or 64), one wait by the caller.
template <int CW>
__device__ __forceinline__ void tmem_ld_row(uint32_t taddr, uint32_t (&r)[CW]) {
  static_assert(CW == 32 || CW == 64, "row chunk");
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  if constexpr (CW == 64) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]),
          "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]),
          "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]),
          "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
        : "r"(taddr + 32));
  }
}

template <int N>
__device__ __forceinline__ void tmem_st_cols(uint32_t taddr, const uint32_t (&r)[N]) {
  static_assert(N == 16 || N == 32, "packed P row chunk");
  if constexpr (N == 16) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
  } else {
    tmem_st_32x32b_x32(taddr, r);
  }
}
// D[tmem] (+)= A[tmem] * B[smem] (kind::f16, A K-major: lane = row, 32-bit column = 2 K elements)
__device__ __forceinline__ void tc_mma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ float fast_exp2(float x) {  // MUFU.EX2, flush-to-zero
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void named_barrier(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

template <int D>
struct FwdCfg {
  static constexpr int BN = D == 128 ? 128 : 64;   // keys per tile
  static constexpr int NS = D == 128 ? 2 : 6;      // K/V ring depth
  static constexpr int NP = 2;                     // P lives in TMEM, aliasing the S buffer it came from
  static constexpr int CW = BN / 2;                // S columns per softmax warp (pair split)
  static constexpr int kQ = kBM * D * 2;           // D/64 chunks of [128 x 64]
  static constexpr int kKV = BN * D * 2;           // K (or V) tile: D/64 chunks of [BN x 64]
  static constexpr int kP = kBM * BN * 2;          // BN/64 chunks of [128 x 64]
  static constexpr int kOffQ = 0;
  static constexpr int kOffK = kOffQ + kQ;
  static constexpr int kOffV = kOffK + NS * kKV;
  static constexpr int kOffP = kOffV + NS * kKV;
  static constexpr int kOffBar = kOffP;           // (no shared-memory P: the PV MMA reads P from TMEM)
  static constexpr int kBarBytes = 256;
  static constexpr int kBytes = kOffBar + kBarBytes + 6 * kBM * 4 + 1024;  // barriers + max/sum exchange
  static constexpr int kTmemCols = D == 128 ? 512 : 256;  // S x2 at 0 / BN, O at 2 BN
  static_assert(kBytes <= 232448, "exceeds the 227 KB per-CTA shared memory");
};

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap mQ, const __grid_constant__ CUtensorMap mK,
                       const __grid_constant__ CUtensorMap mV, __nv_bfloat16* __restrict__ out,
                       int64_t ld_o, float* __restrict__ lse, int S, float scale_log2, const __grid_constant__ AttnPush push,
                       long long* trace, int dbg) {
  using L = FwdCfg<D>;
  constexpr int BN = L::BN, NS = L::NS, NP = L::NP, CW = L::CW;
  constexpr int NCH = D / 64;  // 64-wide chunks of the head dim
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::kOffBar);
  uint64_t* q_full = bar + 0;
  uint64_t* s_full = bar + 1;            // [2]
  uint64_t* s_free = bar + 3;            // [2]
  uint64_t* p_full = bar + 5;            // [NP]
  uint64_t* p_free = bar + 5 + NP;       // [NP]
  uint64_t* kv_full = bar + 5 + 2 * NP;  // [NS]
  uint64_t* kv_empty = kv_full + NS;     // [NS]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(kv_empty + NS);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // longest-first inside each L2-sized head group (grid: x tiles, y heads per group, z groups;
  // lpt_grid): the heavy late query tiles of every head of the group go first
  const int lin = static_cast<int>(blockIdx.y * gridDim.x + blockIdx.x);
  const int qt = static_cast<int>(gridDim.x) - 1 - lin / static_cast<int>(gridDim.y);
  const int h = static_cast<int>(blockIdx.z * gridDim.y) + lin % static_cast<int>(gridDim.y);
  const int q0 = qt * kBM;
  const int n_kv = (q0 + kBM + BN - 1) / BN;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&mQ);
    tma_prefetch(&mK);
    tma_prefetch(&mV);
    mbar_init(q_full, 1);
    for (int i = 0; i < NS; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 256);
    }
    for (int i = 0; i < NP; ++i) {
      mbar_init(&p_full[i], 256);
      mbar_init(&p_free[i], 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<L::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem;               // S buffers at columns 0 and BN
  const uint32_t tO = tmem + 2 * BN;      // O at columns 2 BN .. 2 BN + D

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      mbar_arrive_expect_tx(q_full, L::kQ);
      for (int c = 0; c < NCH; ++c)
        tma_load_2d(smem + L::kOffQ + c * kBM * 128, &mQ, q_full, h * D + c * 64, q0);
      for (int j = 0; j < n_kv; ++j) {
        const int s = j % NS;
        if (j >= NS) mbar_wait(&kv_empty[s], ((j / NS) - 1) & 1);
        mbar_arrive_expect_tx(&kv_full[s], 2 * L::kKV);
        for (int c = 0; c < NCH; ++c) {
          tma_load_2d(smem + L::kOffK + s * L::kKV + c * BN * 128, &mK, &kv_full[s], h * D + c * 64, j * BN);
          tma_load_2d(smem + L::kOffV + s * L::kKV + c * BN * 128, &mV, &kv_full[s], h * D + c * 64, j * BN);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer ----------------
      constexpr uint32_t idesc_s = make_idesc_bf16(kBM, BN, false, false);
      constexpr uint32_t idesc_o = make_idesc_bf16(kBM, D, false, true);
      const uint32_t sQ = smem_u32(smem + L::kOffQ);
      mbar_wait(q_full, 0);
      auto issue_pv = [&](int j) {
        const int pb = j % NP;  // == j & 1 == the S/P buffer of tile j
        mbar_wait(&p_full[pb], (j / NP) & 1);
        tc_fence_after();
        const uint32_t sV = smem_u32(smem + L::kOffV + (j % NS) * L::kKV);
#pragma unroll
        for (int k = 0; k < BN / 16; ++k) {  // A = P (bf16 pairs packed in TMEM columns), B = V (smem)
          const uint64_t bd = make_sw128_desc(sV + k * 2048, BN * 128, 1024);
          tc_mma_bf16_ts(tO, tS + pb * BN + k * 8, bd, idesc_o, (j > 0 || k > 0) ? 1u : 0u);
        }
        tc_commit(&kv_empty[j % NS]);
        tc_commit(&p_free[pb]);
      };
      for (int j = 0; j < n_kv; ++j) {
        const int b = j & 1;
        mbar_wait(&kv_full[j % NS], (j / NS) & 1);
        if (j >= 2) mbar_wait(&s_free[b], ((j >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t sK = smem_u32(smem + L::kOffK + (j % NS) * L::kKV);
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const int c = k / 4, kk = k % 4;
          const uint64_t ad = make_sw128_desc(sQ + c * kBM * 128 + kk * 32, 16, 1024);
          const uint64_t bd = make_sw128_desc(sK + c * BN * 128 + kk * 32, 16, 1024);
          tc_mma_bf16(tS + b * BN, ad, bd, idesc_s, k > 0 ? 1u : 0u);
        }
        tc_commit(&s_full[b]);
        const bool tr = trace && blockIdx.x == 0 && blockIdx.y == 0 && j < 64;
        if (tr) trace[j * 8 + 0] = clock64();
        if (j >= 1) issue_pv(j - 1);
        if (tr) trace[j * 8 + 1] = clock64();
      }
      issue_pv(n_kv - 1);
    }
  } else {
    // ---------------- softmax + epilogue (warps 2..9) ----------------
    // A warp pair per TMEM lane quadrant shares 32 query rows and splits the BN key columns
    // of S (and the D columns of O); the row max is exchanged through smem each tile.
    const int quad = warp & 3, half = (warp - 2) >> 2;
    const int r = quad * 32 + lane;  // query row within the tile == TMEM lane
    const int q = q0 + r;
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    float* xmax = reinterpret_cast<float*>(smem + L::kOffBar + L::kBarBytes);  // [2 slots][2 halves][128 rows]
    float m = -INFINITY, l = 0.f;
    int pf_seen0 = 0, pf_seen1 = 0;  // completed p_free phases consumed per buffer (registers)
    auto ensure_pfree = [&](int pb, int count) {
      int& seen = pb ? pf_seen1 : pf_seen0;
      while (seen < count) {
        mbar_wait(&p_free[pb], seen & 1);
        ++seen;
      }
    };
    for (int j = 0; j < n_kv; ++j) {
      const int b = j & 1;
      const bool tr = trace && blockIdx.x == 0 && blockIdx.y == 0 && j < 64 && warp == 2 && lane == 0;
      if (tr) trace[j * 8 + 2] = clock64();
      mbar_wait(&s_full[b], (j >> 1) & 1);
      if (tr) trace[j * 8 + 3] = clock64();
      tc_fence_after();
      if (dbg == 1) {  // development: pipeline bound without the softmax math
        ensure_pfree(j % NP, j / NP);
        tc_fence_before();
        mbar_arrive(&s_free[b]);
        mbar_arrive(&p_full[j % NP]);
        continue;
      }
      uint32_t sr[CW];
      tmem_ld_row<CW>(tS + lane_off + b * BN + half * CW, sr);
      tmem_ld_wait();
      const bool diag = (j + 1) * BN > q0;  // tile may contain keys > some query of the CTA
      if (diag) {
#pragma unroll
        for (int i = 0; i < CW; ++i)
          if (j * BN + half * CW + i > q) sr[i] = __float_as_uint(-INFINITY);
      }
      float mx0 = -INFINITY, mx1 = -INFINITY, mx2 = -INFINITY, mx3 = -INFINITY;
#pragma unroll
      for (int i = 0; i < CW; i += 4) {
        mx0 = fmaxf(mx0, __uint_as_float(sr[i]));
        mx1 = fmaxf(mx1, __uint_as_float(sr[i + 1]));
        mx2 = fmaxf(mx2, __uint_as_float(sr[i + 2]));
        mx3 = fmaxf(mx3, __uint_as_float(sr[i + 3]));
      }
      float mx = fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3));
      xmax[(b * 2 + half) * kBM + r] = mx;
      named_barrier(2 + quad, 64);
      if (tr) trace[j * 8 + 4] = clock64();
      mx = fmaxf(mx, xmax[(b * 2 + (half ^ 1)) * kBM + r]) * scale_log2;
      // stale-max online softmax: correct O only when the max grows by > 2^8 (uniform across
      // the pair: both warps hold the same rows and the same m)
      const float m_new = fmaxf(m, mx);
      if (j == 0) {
        m = m_new;
      } else if (__any_sync(0xffffffffu, m_new > m + kRescaleThreshold)) {
        ensure_pfree((j - 1) % NP, (j - 1) / NP + 1);  // PV_{j-1} has landed in O
        tc_fence_after();
        const float alpha = fast_exp2(m - m_new);
#pragma unroll 1
        for (int c = 0; c < D / 64; ++c) {
          uint32_t o[32];
          const uint32_t ta = tO + lane_off + half * (D / 2) + c * 32;
          tmem_ld_32x32b_x32(ta, o);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
          tmem_st_32x32b_x32(ta, o);
        }
        tmem_st_wait();
        l *= alpha;
        m = m_new;
      }
      // P = exp2(s * scale - m) into this warp's columns of the swizzled bf16 A tile
      uint32_t pk[CW / 2];
      float ps0 = 0.f, ps1 = 0.f;
#pragma unroll
      for (int i = 0; i < CW; i += 2) {
        const float p0 = fast_exp2(fmaf(__uint_as_float(sr[i]), scale_log2, -m));
        const float p1 = fast_exp2(fmaf(__uint_as_float(sr[i + 1]), scale_log2, -m));
        ps0 += p0;
        ps1 += p1;
        pk[i / 2] = pack_bf16(p0, p1);
      }
      l += ps0 + ps1;
      // P (bf16 pairs) overwrites the first half of this tile's S buffer: the PV MMA reads it as
      // its TMEM A operand; S_{j+2} is issued after PV_j, so in-order MMA execution protects it
      const int pb = j % NP;
      if (tr) trace[j * 8 + 5] = clock64();
      ensure_pfree(pb, j / NP);  // consume PV_{j-2}'s completion in order (mbarrier parity bookkeeping)
      tmem_st_cols<CW / 2>(tS + lane_off + b * BN + half * (CW / 2), pk);
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&s_free[b]);
      mbar_arrive(&p_full[pb]);
      if (tr) trace[j * 8 + 6] = clock64();
    }
    // epilogue: combine the pair's partial row sums, wait for the last PV, O / l -> bf16
    float* xsum = xmax + 4 * kBM;
    xsum[half * kBM + r] = l;
    named_barrier(2 + quad, 64);
    const float l_tot = l + xsum[(half ^ 1) * kBM + r];
    ensure_pfree((n_kv - 1) % NP, (n_kv - 1) / NP + 1);
    tc_fence_after();
    const float inv = 1.f / l_tot;
    __nv_bfloat16* orow = out + static_cast<int64_t>(q) * ld_o + h * D + half * (D / 2);
    __nv_bfloat16* prow_out = nullptr;  // fused all-to-all: the owner rank of token q
    if (push.p[0]) {
      const int owner = q / push.T;
      prow_out = static_cast<__nv_bfloat16*>(push.p[owner]) + static_cast<int64_t>(q - owner * push.T) * push.ld +
                 push.col_o + h * D + half * (D / 2);
    }
#pragma unroll 1
    for (int c = 0; c < D / 64; ++c) {
      uint32_t o[32];
      tmem_ld_32x32b_x32(tO + lane_off + half * (D / 2) + c * 32, o);
      tmem_ld_wait();
      uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        uint32_t pk[4];
#pragma unroll
        for (int e = 0; e < 4; ++e)
          pk[e] = pack_bf16(__uint_as_float(o[v * 8 + 2 * e]) * inv, __uint_as_float(o[v * 8 + 2 * e + 1]) * inv);
        const uint4 val = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        dst[v] = val;
        if (prow_out) reinterpret_cast<uint4*>(prow_out + c * 32)[v] = val;
      }
    }
    if (half == 0) lse[static_cast<int64_t>(h) * S + q] = (m + log2f(l_tot)) * 0.6931471805599453f;
    if (push.p[0]) __threadfence_system();  // pushed rows visible before the next barrier flag
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<L::kTmemCols>(tmem);
  }
}

// ---------------------------------------------------------------------------------
// CTA-pair, two-stream forward (d = 128): the production forward kernel.
//
// A cluster of 2 CTAs owns 4 query tiles of 128 of one head (512 queries); the leader CTA
// issues M = 256 tcgen05.mma.cta_group::2 for two independent streams:
//   stream A = tiles {4pp, 4pp+1} (CTA 0 / CTA 1 rows), stream B = tiles {4pp+2, 4pp+3}.
// Per stream: S_x = Q_x K^T (each CTA holds its own Q tile and half of the 128-key K tile),
// O_x += P_x V (P from each CTA's TMEM, each CTA holds half of V's head-dim columns).
// TMEM per CTA: S_A | S_B | O_A | O_B (4 x 128 columns); P_x overwrites S_x as bf16 pairs.
// The MMA order PV_A(j), S_A(j+1), PV_B(j), S_B(j+1) lets softmax A(j+1) run while the
// tensor pipe works on stream B and vice versa, so the softmax latency is hidden whenever
// it is below one stream's MMA time. Per 128-key tile each CTA streams 32 KB of K/V for 256
// queries (4x less L2->SM traffic than one 128-query tile per CTA).
// Softmax: warpgroup x (warps 4x..4x+3) owns stream x, one thread per query row with all
// 128 columns in registers (no cross-warp max exchange); 3 of every 8 exponentials run as a
// degree-3 polynomial on the FMA pipe, the rest on MUFU.EX2, since MUFU alone would need as
// many cycles per tile as the MMAs.
// Warps 0..7 softmax, warp 8 TMA, warp 9 MMA (leader only).
// ---------------------------------------------------------------------------------
struct Fa4Cfg {
  static constexpr int D = 128, BN = 128, NS = 4;
  static constexpr int kQ = kBM * D * 2;        // one Q tile: 2 chunks [128 q][64]
  static constexpr int kKh = (BN / 2) * D * 2;  // half K tile: 2 chunks [64 keys][64]
  static constexpr int kVh = BN * 64 * 2;       // half V tile: 1 chunk [128 keys][64 d]
  static constexpr int kStage = kKh + kVh;
  static constexpr int kOffQ = 0;               // Q_A, Q_B
  static constexpr int kOffKV = kOffQ + 2 * kQ;
  static constexpr int kOffBar = kOffKV + NS * kStage;
  static constexpr int kBytes = kOffBar + 256 + 1024;
  static_assert(kBytes <= 232448, "exceeds the 227 KB per-CTA shared memory");
};

__device__ __forceinline__ void tc_mma_bf16_ts_pair(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                                    uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void tmem_st_x8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
__device__ __forceinline__ void tmem_ld_x16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ float fmax3f(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
// 2^x on the FMA pipe for x <= ~8: round-to-nearest split x = j + f (f in [-1/2, 1/2]) via the
// 1.5*2^23 shifter, degree-3 polynomial for 2^f (|rel err| < 1e-3, below bf16's half ulp),
// then j added into the exponent field. x is clamped at -125 (masked -inf -> ~2^-125).
__device__ __forceinline__ float2 exp2_poly2(float2 x) {
  constexpr float kShift = 12582912.f;  // 1.5 * 2^23
  x.x = fmaxf(x.x, -125.f);
  x.y = fmaxf(x.y, -125.f);
  const float2 t = __fadd2_rn(x, make_float2(kShift, kShift));
  const float2 jf = __fadd2_rn(t, make_float2(-kShift, -kShift));
  const float2 f = __fadd2_rn(x, make_float2(-jf.x, -jf.y));
  float2 p = __ffma2_rn(make_float2(0.0555041f, 0.0555041f), f, make_float2(0.2402265f, 0.2402265f));
  p = __ffma2_rn(p, f, make_float2(0.6931472f, 0.6931472f));
  p = __ffma2_rn(p, f, make_float2(1.0f, 1.0f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

template <int kPolyPairs = 2>
__global__ void __launch_bounds__(kThreads, 1)
    attn_fwd_fa4_kernel(const __grid_constant__ CUtensorMap mQ, const __grid_constant__ CUtensorMap mK,
                        const __grid_constant__ CUtensorMap mV, __nv_bfloat16* __restrict__ out, int64_t ld_o,
                        float* __restrict__ lse, int S, float scale_log2, const __grid_constant__ AttnPush push,
                        long long* trace, int dbg) {
  using L = Fa4Cfg;
  constexpr int D = L::D, BN = L::BN, NS = L::NS;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::kOffBar);
  uint64_t* q_full = bar + 0;         // leader's: the pair's 4 Q tiles
  uint64_t* s_full = bar + 1;         // [2] local (multicast commit)
  uint64_t* p_full = bar + 3;         // [2] leader's: 4 warps x 2 CTAs per stream
  uint64_t* o_full = bar + 5;         // [2] local (multicast commit): last PV of the stream done
  uint64_t* kv_full = bar + 7;        // [NS] leader's
  uint64_t* kv_empty = kv_full + NS;  // [NS] local (multicast commit)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(kv_empty + NS);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t crank = cluster_rank();
  const bool leader = crank == 0;
  // longest-first over the whole grid: cluster (pair) lp in dispatch order takes the heaviest
  // remaining query group of head lp % heads
  const int lp = static_cast<int>((blockIdx.y * gridDim.x + blockIdx.x) / 2);
  const int pp = static_cast<int>(gridDim.x / 2) - 1 - lp / static_cast<int>(gridDim.y);
  const int h = static_cast<int>(blockIdx.z * gridDim.y) + lp % static_cast<int>(gridDim.y);
  const int q0A = (4 * pp + static_cast<int>(crank)) * kBM, q0B = q0A + 2 * kBM;
  const int nA = (4 * pp + 2) * kBM / BN, nB = nA + 2 * kBM / BN;  // key tiles per stream (its upper tile's)

  if (warp == 8 && lane == 0) {
    tma_prefetch(&mQ);
    tma_prefetch(&mK);
    tma_prefetch(&mV);
    mbar_init(q_full, 1);
    for (int i = 0; i < NS; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 8);
      mbar_init(&o_full[i], 1);
    }
    fence_barrier_init();
  }
  if (warp == 9) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;  // S_A 0, S_B 128, O_A 256, O_B 384

  if (warp == 8) {
    if (lane == 0) {
      // ---------------- TMA producer (both CTAs; completion on the leader's barriers) ----------------
      if (leader) mbar_arrive_expect_tx(q_full, 4 * L::kQ);
      for (int x = 0; x < 2; ++x)
        for (int c = 0; c < 2; ++c)
          tma_load_2d_pair(smem + L::kOffQ + x * L::kQ + c * kBM * 128, &mQ, q_full, h * D + c * 64, x ? q0B : q0A);
      for (int j = 0; j < nB; ++j) {
        const int s = j % NS;
        if (j >= NS) mbar_wait(&kv_empty[s], ((j / NS) - 1) & 1);
        if (leader) mbar_arrive_expect_tx(&kv_full[s], 2 * L::kStage);
        uint8_t* st = smem + L::kOffKV + s * L::kStage;
        for (int c = 0; c < 2; ++c)
          tma_load_2d_pair(st + c * (BN / 2) * 128, &mK, &kv_full[s], h * D + c * 64,
                           j * BN + static_cast<int>(crank) * (BN / 2));
        tma_load_2d_pair(st + L::kKh, &mV, &kv_full[s], h * D + static_cast<int>(crank) * 64, j * BN);
      }
    }
  } else if (warp == 9) {
    if (leader && lane == 0) {
      // ---------------- MMA issuer (leader only) ----------------
      constexpr uint32_t idS = make_idesc_bf16(2 * kBM, BN, false, false);
      constexpr uint32_t idO = make_idesc_bf16(2 * kBM, D, false, true);
      int waited = -1;
      auto wait_kv = [&](int j) {
        if (j > waited) {
          mbar_wait(&kv_full[j % NS], (j / NS) & 1);
          tc_fence_after();
          waited = j;
        }
      };
      auto issue_s = [&](int x, int j) {
        const uint32_t sQ = smem_u32(smem + L::kOffQ + x * L::kQ);
        const uint32_t sK = smem_u32(smem + L::kOffKV + (j % NS) * L::kStage);
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const int c = k / 4, kk = k % 4;
          tc_mma_bf16_pair(tmem + x * 128, make_sw128_desc(sQ + c * kBM * 128 + kk * 32, 16, 1024),
                           make_sw128_desc(sK + c * (BN / 2) * 128 + kk * 32, 16, 1024), idS, k > 0 ? 1u : 0u);
        }
        tc_commit_pair(&s_full[x]);
      };
      auto issue_pv = [&](int x, int j) {
        if (dbg != 2) mbar_wait(&p_full[x], j & 1);
        if (trace && blockIdx.x == 0 && blockIdx.y == 0 && j < 64) trace[j * 8 + 2 * x] = clock64();
        tc_fence_after();
        const uint32_t sV = smem_u32(smem + L::kOffKV + (j % NS) * L::kStage + L::kKh);
#pragma unroll
        for (int k = 0; k < BN / 16; ++k)  // A = P_x (TMEM), B = V half (MN-major)
          tc_mma_bf16_ts_pair(tmem + 256 + x * 128, tmem + x * 128 + k * 8,
                              make_sw128_desc(sV + k * 2048, BN * 128, 1024), idO, (j > 0 || k > 0) ? 1u : 0u);
        if (trace && blockIdx.x == 0 && blockIdx.y == 0 && j < 64) trace[j * 8 + 2 * x + 1] = clock64();
      };
      mbar_wait(q_full, 0);
      wait_kv(0);
      issue_s(0, 0);
      issue_s(1, 0);
      for (int j = 0; j < nB; ++j) {
        if (j < nA) {
          issue_pv(0, j);
          if (j == nA - 1) {
            tc_commit_pair(&o_full[0]);
          } else {
            wait_kv(j + 1);
            issue_s(0, j + 1);
          }
        }
        issue_pv(1, j);
        tc_commit_pair(&kv_empty[j % NS]);
        if (j == nB - 1) {
          tc_commit_pair(&o_full[1]);
        } else {
          wait_kv(j + 1);
          issue_s(1, j + 1);
        }
      }
    }
  } else {
    // ---------------- softmax + epilogue: warpgroup x = stream x ----------------
    const int x = warp >> 2, quad = warp & 3;
    const int r = quad * 32 + lane;
    const int q0 = x ? q0B : q0A, q = q0 + r, n = x ? nB : nA;
    const uint32_t lo = static_cast<uint32_t>(quad * 32) << 16;
    const uint32_t tSx = tmem + x * 128 + lo, tOx = tmem + 256 + x * 128 + lo;
    const bool tr = trace && blockIdx.x == 0 && blockIdx.y == 0 && x == 0 && lane == 0;
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < n; ++j) {
      mbar_wait(&s_full[x], j & 1);
      tc_fence_after();
      
      if (dbg == 0) {
        uint32_t sr[BN];
#pragma unroll
        for (int c = 0; c < BN / 32; ++c) {
          uint32_t (&chunk)[32] = *reinterpret_cast<uint32_t(*)[32]>(&sr[c * 32]);
          tmem_ld_32x32b_x32(tSx + c * 32, chunk);
        }
        tmem_ld_wait();
        if ((j + 1) * BN > q0) {  // tile reaches past some query of this tile: causal mask
#pragma unroll
          for (int i = 0; i < BN; ++i)
            if (j * BN + i > q) sr[i] = __float_as_uint(-INFINITY);
        }
        float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
        for (int i = 0; i < BN; i += 4) {
          mx0 = fmax3f(mx0, __uint_as_float(sr[i]), __uint_as_float(sr[i + 1]));
          mx1 = fmax3f(mx1, __uint_as_float(sr[i + 2]), __uint_as_float(sr[i + 3]));
        }
        const float m_new = fmaxf(m, fmaxf(mx0, mx1) * scale_log2);
        if (j == 0) {
          m = m_new;
        } else if (__any_sync(0xffffffffu, m_new > m + kRescaleThreshold)) {
          // stale-max rule: O is corrected only when the row max grows by > 2^8 (warp-uniform);
          // PV_x(j-1) has completed (it precedes S_x(j) in the tensor pipe)
          const float alpha = fast_exp2(m - m_new);
#pragma unroll 1
          for (int c = 0; c < D / 16; ++c) {  // 16-column chunks: S stays live in registers
            uint32_t o[16];
            tmem_ld_x16(tOx + c * 16, o);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st_cols<16>(tOx + c * 16, o);
          }
          l *= alpha;
          m = m_new;
        }
        const float2 sc = make_float2(scale_log2, scale_log2), nm = make_float2(-m, -m);
        float2 acc = make_float2(0.f, 0.f);
#pragma unroll
        for (int c = 0; c < BN / 16; ++c) {  // 16 columns -> 8 packed bf16 pairs per TMEM store
          uint32_t pk[8];
#pragma unroll
          for (int i = 0; i < 16; i += 2) {
            const float2 sv = make_float2(__uint_as_float(sr[c * 16 + i]), __uint_as_float(sr[c * 16 + i + 1]));
            const float2 xv = __ffma2_rn(sv, sc, nm);
            float2 pv;
            if (i >= 16 - 2 * kPolyPairs) {  // kPolyPairs of 8 pairs on the FMA pipe
              pv = exp2_poly2(xv);
            } else {
              pv.x = fast_exp2(xv.x);
              pv.y = fast_exp2(xv.y);
            }
            acc = __fadd2_rn(acc, pv);
            pk[i / 2] = pack_bf16(pv.x, pv.y);
          }
          tmem_st_x8(tSx + c * 8, pk);
        }
        l += acc.x + acc.y;
        tmem_st_wait();
      }
      tc_fence_before();
      __syncwarp();
      if (tr && j < 64) trace[j * 8 + 4 + quad] = clock64();
      if (lane == 0) {
        if (leader) mbar_arrive(&p_full[x]);
        else mbar_arrive_leader(&p_full[x]);
      }
    }
    // epilogue: O_x / l -> bf16 (+ push to the token owner), lse
    mbar_wait(&o_full[x], 0);
    tc_fence_after();
    const float inv = 1.f / l;
    __nv_bfloat16* orow = out + static_cast<int64_t>(q) * ld_o + h * D;
    __nv_bfloat16* prow_out = nullptr;
    if (push.p[0]) {
      const int owner = q / push.T;
      prow_out = static_cast<__nv_bfloat16*>(push.p[owner]) + static_cast<int64_t>(q - owner * push.T) * push.ld +
                 push.col_o + h * D;
    }
#pragma unroll 1
    for (int c = 0; c < D / 32; ++c) {
      uint32_t o[32];
      tmem_ld_32x32b_x32(tOx + c * 32, o);
      tmem_ld_wait();
      uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        uint32_t pk2[4];
#pragma unroll
        for (int e = 0; e < 4; ++e)
          pk2[e] = pack_bf16(__uint_as_float(o[v * 8 + 2 * e]) * inv, __uint_as_float(o[v * 8 + 2 * e + 1]) * inv);
        const uint4 val = make_uint4(pk2[0], pk2[1], pk2[2], pk2[3]);
        dst[v] = val;
        if (prow_out) reinterpret_cast<uint4*>(prow_out + c * 32)[v] = val;
      }
    }
    lse[static_cast<int64_t>(h) * S + q] = (m + log2f(l)) * 0.6931471805599453f;
    if (push.p[0]) __threadfence_system();  // pushed rows visible before the next barrier flag
  }

  tc_fence_before();
  cluster_sync_all();
  if (warp == 9) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// [rows, cols] bf16 with row stride ld elements; box {64 cols, box_rows}, 128-B swizzle.
bool map2d(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 2)};
  cuuint32_t box[2] = {64u, static_cast<cuuint32_t>(box_rows)};
  cuuint32_t es[2] = {1u, 1u};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Longest-first dispatch inside L2-sized head groups: grid (tiles, G, heads / G). Blocks
// dispatch in linear-index order, so within a group the heaviest causal tiles of all G heads go
// first (no heavy tile of the last head trails the grid), and the groups run one after another
// so the K/V (forward) or Q/dO (backward) streams in flight, G * S * d * 4 bytes, stay in L2.
dim3 lpt_grid(int tiles_x, int heads, int S, int d) {
  const int64_t per_head = int64_t(S) * d * 4;
  int g = 1;
  for (int c = 1; c <= heads; ++c)
    if (heads % c == 0 && c * per_head <= (int64_t(48) << 20)) g = c;
  return dim3(tiles_x, g, heads / g);
}

template <int D>
cudaError_t launch_fwd(const AttnTensors& t, cudaStream_t st) {
  using L = FwdCfg<D>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_fwd_tc_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kBytes);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  CUtensorMap mq, mk, mv;
  const int64_t cols = static_cast<int64_t>(t.heads) * D;
  if (!map2d(&mq, t.q, t.S, cols, t.ld_qkv, kBM) || !map2d(&mk, t.k, t.S, cols, t.ld_qkv, L::BN) ||
      !map2d(&mv, t.v, t.S, cols, t.ld_qkv, L::BN))
    return cudaErrorInvalidValue;
  const float scale_log2 = (1.0f / sqrtf(static_cast<float>(D))) * kLog2e;
  attn_fwd_tc_kernel<D><<<lpt_grid(t.S / kBM, t.heads, t.S, D), kThreads, L::kBytes, st>>>(mq, mk, mv, t.o, t.ld_o, t.lse, t.S,
                                                                               scale_log2, t.push, g_attn_trace_fwd,
      std::getenv("SEQPLAN_ISP_DBG") ? std::atoi(std::getenv("SEQPLAN_ISP_DBG")) : 0);
  return cudaGetLastError();
}

cudaError_t launch_fwd_pair(const AttnTensors& t, cudaStream_t st) {
  using L = Fa4Cfg;
  // exponential pairs of 8 on the FMA-pipe polynomial (development: SEQPLAN_ISP_FWD_POLY)
  const char* pe = std::getenv("SEQPLAN_ISP_FWD_POLY");
  // (32K x 32 heads, isolated: 0 -> 7.16 ms, 2 -> 6.98, 3 -> 7.17, 4 -> 7.36; in the power-capped
  // 7B-32K step all within noise, profiles/r2/attn_fwd_poly_sweep.txt)
  const int poly = pe ? std::atoi(pe) : 2;
  auto kern = attn_fwd_fa4_kernel<2>;
  switch (poly) {
    case 0: kern = attn_fwd_fa4_kernel<0>; break;
    case 1: kern = attn_fwd_fa4_kernel<1>; break;
    case 3: kern = attn_fwd_fa4_kernel<3>; break;
    case 4: kern = attn_fwd_fa4_kernel<4>; break;
    default: break;
  }
  static bool attr[8] = {};
  if (!attr[poly & 7]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kBytes);
    if (e != cudaSuccess) return e;
    attr[poly & 7] = true;
  }
  CUtensorMap mq, mk, mv;
  const int64_t cols = static_cast<int64_t>(t.heads) * 128;
  if (!map2d(&mq, t.q, t.S, cols, t.ld_qkv, kBM) || !map2d(&mk, t.k, t.S, cols, t.ld_qkv, L::BN / 2) ||
      !map2d(&mv, t.v, t.S, cols, t.ld_qkv, L::BN))
    return cudaErrorInvalidValue;
  const float scale_log2 = (1.0f / sqrtf(128.0f)) * kLog2e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = lpt_grid(t.S / (2 * kBM), t.heads, t.S, 128);  // 2 query tiles per CTA
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = L::kBytes;
  cfg.stream = st;
  cudaLaunchAttribute attr_[1];
  attr_[0].id = cudaLaunchAttributeClusterDimension;
  attr_[0].val.clusterDim.x = 2;
  attr_[0].val.clusterDim.y = 1;
  attr_[0].val.clusterDim.z = 1;
  cfg.attrs = attr_;
  cfg.numAttrs = 1;
  const int dbg = std::getenv("SEQPLAN_ISP_DBG") ? std::atoi(std::getenv("SEQPLAN_ISP_DBG")) : 0;
  return cudaLaunchKernelEx(&cfg, kern, mq, mk, mv, t.o, t.ld_o, t.lse, t.S, scale_log2, t.push,
                            g_attn_trace_fwd, dbg);
}

}  // namespace

cudaError_t attention_fwd_tc(const AttnTensors& t, cudaStream_t st) {
  if (t.S % kBM) return cudaErrorInvalidValue;
  if (t.d == 128) {
    if ((t.S / kBM) % 4 == 0 && !std::getenv("SEQPLAN_ISP_ATTN_SINGLE")) return launch_fwd_pair(t, st);
    return launch_fwd<128>(t, st);
  }
  if (t.d == 64) return launch_fwd<64>(t, st);
  return cudaErrorInvalidValue;
}


// =====================================================================================
// Causal flash-attention backward on tcgen05 / TMEM / TMA (d = 128).
//
// CTA = 128 keys x 1 head; iterates over 64-query tiles i >= k0 (causal). Per tile:
//   S^T  = K Q_i^T,  dP^T = V dO_i^T                (M=128 keys, N=64, K=d)   -> TMEM
//   P^T  = exp2(S^T*scale*log2e - lse_i*log2e),  dS^T = P^T (dP^T - delta_i)  (8 warps:
//          a warp pair per TMEM lane quadrant splits the 64 query columns; the math is
//          elementwise given lse/delta per column, so no cross-warp reduction)
//   dV  += P^T dO_i,  dK += dS^T Q_i               (M=128 keys, N=d, K=64)   TMEM-resident
//   dQ_i^T = K^T dS^T                              (M=d, N=64, K=128 keys)   -> TMEM
//          -> smem [64 q][d] fp32 -> one cp.reduce.async.bulk add.f32 into dq_acc (32 KB)
// The MMA warp software-pipelines S/dP of tile i with the gradient MMAs of tile i-1.
// Shared memory: K, V 64 KB + Q/dO 2-stage 64 KB + P^T, dS^T 32 KB + dQ staging 32 KB.
// TMEM 512 columns: S^T 0, dP^T 64, dK 128, dV 256, dQ^T 384.
// =====================================================================================
namespace {

constexpr int kBwdKeys = 128;
constexpr int kBwdQ = 64;
constexpr int kBwdThreads = 448;  // warp 0 TMA, warp 1 MMA, warps 2..9 P/dS, warps 10..13 dQ

struct BwdSmem {
  static constexpr int kStages = 4;                   // Q/dO ring depth (TMA latency lookahead)
  static constexpr int kKV = kBwdKeys * 128 * 2;      // [2 chunks][128 keys][64 d]
  static constexpr int kQ = kBwdQ * 128 * 2;          // [2 chunks][64 q][64 d]
  static constexpr int kStage = 2 * kQ;               // Q_i | dO_i
  static constexpr int kP = kBwdKeys * kBwdQ * 2;     // [128 keys][64 q]
  static constexpr int kOffK = 0;
  static constexpr int kOffV = kOffK + kKV;
  static constexpr int kOffQ = kOffV + kKV;           // stage s: Q at kOffQ + s*kStage, dO at +kQ
  static constexpr int kOffDS = kOffQ + kStages * kStage;  // dS^T (bf16, SW128): B operand of dQ^T
  static constexpr int kOffLD = kOffDS + kP;          // stage s: lse[64] | delta[64] (fp32), bulk-loaded
  static constexpr int kOffBar = kOffLD + kStages * 512;
  static constexpr int kBytes = kOffBar + 256 + 1024;
  static_assert(kBytes <= 232448, "exceeds the 227 KB per-CTA shared memory");
};

__device__ __forceinline__ void bulk_load(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(smem_dst)),
               "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_reduce_add_f32(float* gdst, const void* smem_src, uint32_t bytes) {
  asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(gdst),
               "r"(smem_u32(smem_src)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// Streamed once: L2 evict-first, so the stream does not push the reused operands out of L2.
__device__ __forceinline__ void bulk_store_stream(void* gdst, const void* smem_src, uint32_t bytes, uint64_t pol) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(gdst),
               "r"(smem_u32(smem_src)), "r"(bytes), "l"(pol)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_load_stream(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar,
                                                 uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// kDQ = false: a dK/dV-only variant (dQ from elsewhere):
// no dQ^T MMA / warps / atomics, and K lives in TMEM so S^T = K Q^T is a TS MMA.
// kKT (fused kernel): K also lives in TMEM (S^T as a TS MMA, 32 KB less shared-memory operand
// traffic per tile); P^T / dS^T then share the dQ^T columns, so the P/dS warps also wait for the
// dQ warps to have drained dQ^T of the previous tile before writing them.
template <bool kDQ, bool kKT = !kDQ>
__global__ void __launch_bounds__(kDQ ? kBwdThreads : 320, 1)
    attn_bwd_tc_kernel(const __grid_constant__ CUtensorMap mQ, const __grid_constant__ CUtensorMap mK,
                       const __grid_constant__ CUtensorMap mV, const __grid_constant__ CUtensorMap mDO,
                       const float* __restrict__ lse, const float* __restrict__ delta, float* __restrict__ dq_acc,
                       __nv_bfloat16* __restrict__ dk_out, __nv_bfloat16* __restrict__ dv_out, int64_t ld_d,
                       int S, float scale, int dbg, long long* trace, const __grid_constant__ AttnPush push,
                       const __nv_bfloat16* __restrict__ kg, int64_t ld_k) {
  using L = BwdSmem;
  constexpr int D = 128;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::kOffBar);
  constexpr int NS = L::kStages;
  uint64_t* kv_full = bar + 0;
  uint64_t* s_full = bar + 1;
  uint64_t* s_free = bar + 2;
  uint64_t* p_full = bar + 3;
  uint64_t* p_free = bar + 4;
  uint64_t* dq_full = bar + 5;
  uint64_t* dq_free = bar + 6;
  uint64_t* dkv_full = bar + 7;
  uint64_t* q_full = bar + 8;        // [NS]
  uint64_t* q_empty = bar + 8 + NS;  // [NS]
  uint64_t* k_tm = bar + 8 + 2 * NS;  // !kDQ: K rows written into TMEM by the P/dS warps
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 9 + 2 * NS);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // longest-first over the whole grid: key tile 0 (the most query tiles) of every head first
  const int lin = static_cast<int>(blockIdx.y * gridDim.x + blockIdx.x);
  const int kt = lin / static_cast<int>(gridDim.y);
  const int h = static_cast<int>(blockIdx.z * gridDim.y) + lin % static_cast<int>(gridDim.y);
  const int k0 = kt * kBwdKeys;
  const int qi0 = k0 / kBwdQ, nq = S / kBwdQ - qi0;
  const float scale_log2 = scale * kLog2e;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&mQ); tma_prefetch(&mK); tma_prefetch(&mV); tma_prefetch(&mDO);
    mbar_init(kv_full, 1);
    for (int i = 0; i < NS; ++i) { mbar_init(&q_full[i], 1); mbar_init(&q_empty[i], 1); }
    mbar_init(s_full, 1);
    mbar_init(s_free, 256);
    mbar_init(p_full, 256);
    mbar_init(p_free, 1);
    mbar_init(dq_full, 1);
    mbar_init(dq_free, 128);
    mbar_init(dkv_full, 1);
    mbar_init(k_tm, 256);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // TMEM, kDQ:  S^T 0 | dP^T 64 | dK 128 | dV 256 | dQ^T 384 (64) | P^T bf16 448 (32) | dS^T bf16 480 (32)
  //       !kDQ: S^T 0 | dP^T 64 | dK 128 | dV 256 | P^T bf16 384 (32) | dS^T bf16 416 (32) | K bf16 448 (64)
  //  kDQ && kKT: S^T 0 | dP^T 64 | dK 128 | dV 256 | dQ^T 384 (64) = P^T 384 | dS^T 416 | K bf16 448 (64)
  const uint32_t tS = tmem, tP = tmem + 64, tDK = tmem + 128, tDV = tmem + 256, tDQ = tmem + 384;
  const uint32_t tPT = tmem + (kDQ && !kKT ? 448 : 384), tDST = tmem + (kDQ && !kKT ? 480 : 416), tK = tmem + 448;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      mbar_arrive_expect_tx(kv_full, (kDQ ? 2 : 1) * L::kKV);
      for (int c = 0; c < 2; ++c) {
        if constexpr (kDQ) tma_load_2d(smem + L::kOffK + c * kBwdKeys * 128, &mK, kv_full, h * D + c * 64, k0);
        tma_load_2d(smem + L::kOffV + c * kBwdKeys * 128, &mV, kv_full, h * D + c * 64, k0);
      }
      for (int i = 0; i < nq; ++i) {
        const int s = i % NS, q0 = (qi0 + i) * kBwdQ;
        if (i >= NS) mbar_wait(&q_empty[s], ((i / NS) - 1) & 1);
        mbar_arrive_expect_tx(&q_full[s], 2 * L::kQ + 512);
        for (int c = 0; c < 2; ++c) {
          tma_load_2d(smem + L::kOffQ + s * L::kStage + c * kBwdQ * 128, &mQ, &q_full[s], h * D + c * 64, q0);
          tma_load_2d(smem + L::kOffQ + s * L::kStage + L::kQ + c * kBwdQ * 128, &mDO, &q_full[s], h * D + c * 64, q0);
        }
        bulk_load(smem + L::kOffLD + s * 512, lse + static_cast<int64_t>(h) * S + q0, 256, &q_full[s]);
        bulk_load(smem + L::kOffLD + s * 512 + 256, delta + static_cast<int64_t>(h) * S + q0, 256, &q_full[s]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer ----------------
      constexpr uint32_t id_s = make_idesc_bf16(kBwdKeys, kBwdQ, false, false);  // S^T, dP^T
      constexpr uint32_t id_g = make_idesc_bf16(kBwdKeys, D, false, true);       // dV, dK
      constexpr uint32_t id_q = make_idesc_bf16(D, kBwdQ, true, true);           // dQ^T
      const uint32_t sK = smem_u32(smem + L::kOffK), sV = smem_u32(smem + L::kOffV);
      const uint32_t sDS = smem_u32(smem + L::kOffDS);
      mbar_wait(kv_full, 0);
      if constexpr (kKT) mbar_wait(k_tm, 0);
      auto grads = [&](int j) {
        const int s = j % NS;
        mbar_wait(p_full, j & 1);
        if (kDQ && j >= 1) mbar_wait(dq_free, (j - 1) & 1);
        tc_fence_after();
        const uint32_t sQ = smem_u32(smem + L::kOffQ + s * L::kStage), sDO = sQ + L::kQ;
#pragma unroll
        for (int k = 0; k < kBwdQ / 16; ++k) {  // A = P^T / dS^T from TMEM (16 queries = 8 columns)
          tc_mma_bf16_ts(tDV, tPT + k * 8, make_sw128_desc(sDO + k * 2048, kBwdQ * 128, 1024), id_g,
                         (j > 0 || k > 0) ? 1u : 0u);
          tc_mma_bf16_ts(tDK, tDST + k * 8, make_sw128_desc(sQ + k * 2048, kBwdQ * 128, 1024), id_g,
                         (j > 0 || k > 0) ? 1u : 0u);
        }
        if constexpr (kDQ) {
#pragma unroll
          for (int k = 0; k < kBwdKeys / 16; ++k)
            tc_mma_bf16(tDQ, make_sw128_desc(sK + k * 2048, kBwdKeys * 128, 1024),
                        make_sw128_desc(sDS + k * 2048, kBwdQ * 128, 1024), id_q, k > 0 ? 1u : 0u);
        }
        tc_commit(&q_empty[s]);
        tc_commit(p_free);
        if constexpr (kDQ) tc_commit(dq_full);
      };
      for (int i = 0; i < nq; ++i) {
        const int s = i % NS;
        mbar_wait(&q_full[s], (i / NS) & 1);
        if (i >= 1) mbar_wait(s_free, (i - 1) & 1);
        tc_fence_after();
        const uint32_t sQ = smem_u32(smem + L::kOffQ + s * L::kStage), sDO = sQ + L::kQ;
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const int c = k / 4, kk = k % 4;
          if constexpr (!kKT)
            tc_mma_bf16(tS, make_sw128_desc(sK + c * kBwdKeys * 128 + kk * 32, 16, 1024),
                        make_sw128_desc(sQ + c * kBwdQ * 128 + kk * 32, 16, 1024), id_s, k > 0 ? 1u : 0u);
          else  // A = K from TMEM (16 head dims = 8 columns)
            tc_mma_bf16_ts(tS, tK + k * 8, make_sw128_desc(sQ + c * kBwdQ * 128 + kk * 32, 16, 1024), id_s,
                           k > 0 ? 1u : 0u);
          tc_mma_bf16(tP, make_sw128_desc(sV + c * kBwdKeys * 128 + kk * 32, 16, 1024),
                      make_sw128_desc(sDO + c * kBwdQ * 128 + kk * 32, 16, 1024), id_s, k > 0 ? 1u : 0u);
        }
        tc_commit(s_full);
        if (trace && blockIdx.x == 0 && blockIdx.y == 0 && i < 64) trace[i * 8 + 0] = clock64();
        if (i >= 1) grads(i - 1);
        if (trace && blockIdx.x == 0 && blockIdx.y == 0 && i < 64) trace[i * 8 + 1] = clock64();
      }
      grads(nq - 1);
      tc_commit(dkv_full);
    }
  } else if (kDQ && warp >= 10) {
    // ---------------- dQ warps 10..13: dQ^T (lane = head dim) -> fp32 reductions ----------------
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const uint32_t lo = static_cast<uint32_t>(quad * 32) << 16;
    for (int j = 0; j < nq; ++j) {
      mbar_wait(dq_full, j & 1);
      tc_fence_after();
      uint32_t v0[32], v1[32];
      if (dbg == 12) {  // development: pipeline bound without the dQ reductions
        tc_fence_before();
        mbar_arrive(dq_free);
        continue;
      }
      tmem_ld_32x32b_x32(tDQ + lo, v0);
      tmem_ld_32x32b_x32(tDQ + lo + 32, v1);
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(dq_free);
      // a warp instruction covers 32 consecutive floats (one query row, 32 head dims). 16-B vector
      // REDs after a 4 x 4 lane transpose (4 queries x 128 B per instruction) measured ~10 % slower
      // for the whole kernel (S = 16K: 3.54 vs 3.20 ms)
      float* dst = dq_acc + (static_cast<int64_t>(h) * S + (qi0 + j) * kBwdQ) * D + r;
#pragma unroll
      for (int c = 0; c < 32; ++c)
        asm volatile("red.global.add.f32 [%0], %1;" ::"l"(dst + c * D), "f"(__uint_as_float(v0[c]) * scale) : "memory");
#pragma unroll
      for (int c = 0; c < 32; ++c)
        asm volatile("red.global.add.f32 [%0], %1;" ::"l"(dst + (32 + c) * D), "f"(__uint_as_float(v1[c]) * scale)
                     : "memory");
    }
  } else {
    // ---------------- P^T / dS^T warps 2..9 ----------------
    // A warp pair per TMEM lane quadrant (key rows); each warp owns 32 of the 64 query
    // columns, processed in two 16-column chunks to bound register pressure.
    const int quad = warp & 3, half = (warp - 2) >> 2;
    const int r = quad * 32 + lane;  // key row
    const uint32_t lo = static_cast<uint32_t>(quad * 32) << 16;
    const int key = k0 + r;
    if constexpr (kKT) {  // K row of this key into TMEM (this warp's 64 head dims): the S^T A operand
      const uint4* src = reinterpret_cast<const uint4*>(kg + static_cast<int64_t>(key) * ld_k + h * D + half * 64);
      uint32_t kr[32];
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        const uint4 u = src[v];
        kr[4 * v] = u.x; kr[4 * v + 1] = u.y; kr[4 * v + 2] = u.z; kr[4 * v + 3] = u.w;
      }
      tmem_st_32x32b_x32(tK + lo + half * 32, kr);
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(k_tm);
    }
    for (int i = 0; i < nq; ++i) {
      const int q0 = (qi0 + i) * kBwdQ;
      const bool tr = trace && blockIdx.x == 0 && blockIdx.y == 0 && i < 64 && warp == 2 && lane == 0;
      if (tr) trace[i * 8 + 2] = clock64();
      mbar_wait(s_full, i & 1);
      mbar_wait(&q_full[i % NS], (i / NS) & 1);  // lse / delta of this tile are in shared memory
      if (tr) trace[i * 8 + 3] = clock64();
      tc_fence_after();
      if (dbg >= 11) {  // development: pipeline bound without the P / dS math
        tc_fence_before();
        mbar_arrive(s_free);
        if (i >= 1) mbar_wait(p_free, (i - 1) & 1);
        tc_fence_before();
        mbar_arrive(p_full);
        continue;
      }
      const bool diag = q0 < k0 + kBwdKeys;
      uint32_t pk[16], dk[16];
      // S^T and dP^T of this warp's 32 query columns into registers, then release the TMEM
      // buffers at once so the next tile's S^T / dP^T MMAs overlap this tile's math
      uint32_t sv[32], pv[32];
      tmem_ld_32x32b_x32(tS + lo + half * 32, sv);
      tmem_ld_32x32b_x32(tP + lo + half * 32, pv);
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(s_free);
      const float* lsm = reinterpret_cast<const float*>(smem + L::kOffLD + (i % NS) * 512) + half * 32;
#pragma unroll
      for (int hc = 0; hc < 2; ++hc) {
        float4 l4[4], d4[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {  // warp-uniform addresses: shared-memory broadcasts
          l4[k] = reinterpret_cast<const float4*>(lsm + hc * 16)[k];
          d4[k] = reinterpret_cast<const float4*>(lsm + 64 + hc * 16)[k];
        }
        const float* lr = reinterpret_cast<const float*>(l4);
        const float* dr = reinterpret_cast<const float*>(d4);
        // packed f32x2 math (FFMA2/FMUL2/FADD2), and 3 of 8 exponential pairs as a polynomial on
        // the FMA pipe (exp2_poly2, as in the forward): MUFU.EX2 alone needs 512 cycles per tile
#pragma unroll
        for (int c = 0; c < 16; c += 2) {
          const float2 s2 = make_float2(__uint_as_float(sv[hc * 16 + c]), __uint_as_float(sv[hc * 16 + c + 1]));
          const float2 nl = __fmul2_rn(make_float2(lr[c], lr[c + 1]), make_float2(-kLog2e, -kLog2e));
          const float2 x = __ffma2_rn(s2, make_float2(scale_log2, scale_log2), nl);
          float2 p;
          if (c >= 10) {
            p = exp2_poly2(x);
          } else {
            p.x = fast_exp2(x.x);
            p.y = fast_exp2(x.y);
          }
          if (diag) {
            const int qc = q0 + half * 32 + hc * 16 + c;
            if (key > qc) p.x = 0.f;
            if (key > qc + 1) p.y = 0.f;
          }
          const float2 dd = __fadd2_rn(make_float2(__uint_as_float(pv[hc * 16 + c]), __uint_as_float(pv[hc * 16 + c + 1])),
                                       make_float2(-dr[c], -dr[c + 1]));
          const float2 d = __fmul2_rn(p, dd);
          pk[hc * 8 + c / 2] = pack_bf16(p.x, p.y);
          dk[hc * 8 + c / 2] = pack_bf16(d.x, d.y);
        }
      }
      if (tr) trace[i * 8 + 4] = clock64();
      if (i >= 1) mbar_wait(p_free, (i - 1) & 1);  // gradient MMAs of tile i-1 released P^T / dS^T
      if (kDQ && kKT && i >= 1) mbar_wait(dq_free, (i - 1) & 1);  // dQ^T of tile i-1 drained (shared columns)
      if (tr) trace[i * 8 + 5] = clock64();
      // P^T, dS^T (bf16 pairs) into TMEM: the A operands of dV / dK; dS^T also into shared
      // memory (SW128) as the B operand of dQ^T
      tmem_st_cols<16>(tPT + lo + half * 16, pk);
      tmem_st_cols<16>(tDST + lo + half * 16, dk);
      if constexpr (kDQ) {
        uint8_t* drow = smem + L::kOffDS + r * 128;
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          const int chunk = (half * 4 + cc) ^ (r & 7);
          *reinterpret_cast<uint4*>(drow + chunk * 16) =
              make_uint4(dk[4 * cc], dk[4 * cc + 1], dk[4 * cc + 2], dk[4 * cc + 3]);
        }
      }
      tmem_st_wait();
      if constexpr (kDQ) fence_proxy_async();
      tc_fence_before();
      mbar_arrive(p_full);
      if (tr) trace[i * 8 + 6] = clock64();
    }
    // dK (scaled), dV -> bf16
    mbar_wait(dkv_full, 0);
    tc_fence_after();
#pragma unroll 1
    for (int c = 0; c < 2; ++c) {
      const int col = half * 64 + c * 32;
      uint32_t a[32], b[32];
      tmem_ld_32x32b_x32(tDK + lo + col, a);
      tmem_ld_32x32b_x32(tDV + lo + col, b);
      tmem_ld_wait();
      uint4* pk_out;
      uint4* pv_out;
      if (push.p[0]) {  // fused all-to-all: rows go to the owner of the key token
        const int owner = key / push.T;
        __nv_bfloat16* base = static_cast<__nv_bfloat16*>(push.p[owner]) +
                              static_cast<int64_t>(key - owner * push.T) * push.ld + h * D + col;
        pk_out = reinterpret_cast<uint4*>(base + push.col_k);
        pv_out = reinterpret_cast<uint4*>(base + push.col_v);
      } else {
        pk_out = reinterpret_cast<uint4*>(dk_out + static_cast<int64_t>(key) * ld_d + h * D + col);
        pv_out = reinterpret_cast<uint4*>(dv_out + static_cast<int64_t>(key) * ld_d + h * D + col);
      }
#pragma unroll
      for (int v4 = 0; v4 < 4; ++v4) {
        uint32_t x[4], y[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          x[e] = pack_bf16(__uint_as_float(a[v4 * 8 + 2 * e]) * scale, __uint_as_float(a[v4 * 8 + 2 * e + 1]) * scale);
          y[e] = pack_bf16(__uint_as_float(b[v4 * 8 + 2 * e]), __uint_as_float(b[v4 * 8 + 2 * e + 1]));
        }
        pk_out[v4] = make_uint4(x[0], x[1], x[2], x[3]);
        pv_out[v4] = make_uint4(y[0], y[1], y[2], y[3]);
      }
    }
    if (push.p[0]) __threadfence_system();  // pushed rows visible before the next barrier flag
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// =====================================================================================
// Causal flash-attention backward without atomics, one launch, two CTA roles (d = 128):
// the production backward.
//
// The fused backward (one CTA per 128 keys, dQ reduced into fp32 with L2 atomics) is capped by
// the L2 reduction rate: (S/128)·S·d·4 B per head of fp32 reductions ran at ~2.8 TB/s whatever the
// issuing path (scalar red.global or TMA cp.reduce), i.e. <= ~720 TF/s. Here every gradient is
// accumulated in TMEM and written once:
//   role KV (one CTA per 128 keys kt, walks query tiles i >= kt):   4 MMAs per tile
//     S^T = K Q_i^T (SS), dP^T = V dO_i^T (SS)                 -> TMEM S^T 0..127, dP^T 128..255
//     P^T = exp2(S^T*scale*log2e - lse*log2e) (registers), dS^T = P^T (dP^T - delta); both bf16
//     into the dP^T columns (per 64-query half: P^T 32 columns | dS^T 32 columns)
//     dV += P^T dO_i (TS), dK += dS^T Q_i (TS)                -> TMEM dK 256..383, dV 384..511
//     issue order S(i+1), dV(i), dK(i), dP(i+1): S^T is free as soon as it is in registers, so
//     P(i+1) is computed under dV(i)/dK(i)/dP(i+1) and only the dS store sits between dP(i) and
//     dV(i), under S(i+1).
//   role Q (one CTA per 128 queries qt, walks key tiles j <= qt):    3 MMAs per tile
//     S = Q K_j^T (SS), dP = dO V_j^T (SS)                     -> TMEM S 0..127, dP 128..255
//     P = exp2(S*scale*log2e - lse*log2e), dS = P (dP - delta)  bf16 over the dP columns
//     dQ += dS K_j (TS)                                        -> TMEM dQ 256..383
//     issue order S(j+1), dQ(j), dP(j+1): P(j+1) under dQ(j)/dP(j+1), dS(j) under S(j+1).
// Every MMA is M = 128, N = 128. 7 MMAs per (key tile, query tile) instead of the fused 5, but
// none waits on an L2 reduction; the dQ rows come out in bf16 (scaled), no fp32 accumulator.
// Dispatch: one grid over (role, tile) entries sorted by decreasing work (split_entry), inside
// L2-sized head groups (lpt_grid), so the heaviest CTAs of both roles start first.
// Shared memory: KV role K, V 64 KB + Q, dO 2 stages 128 KB; Q role Q, dO 64 KB + K 3 stages
// 96 KB + V 2 stages 64 KB.
// Warps: 0..7 math (a warp pair per TMEM lane quadrant, 64 columns each), 8 TMA, 9 MMA.
// =====================================================================================
struct BwdSCfg {
  static constexpr int kTile = 128 * 128 * 2;  // [2 chunks][128 rows][64 cols] bf16, SW128
  // role KV
  static constexpr int kOffK = 0, kOffV = kTile, kOffQ = 2 * kTile, kOffDO = 4 * kTile;  // Q, dO: 2 stages
  static constexpr int kOffLD = 6 * kTile;  // per stage lse[128] | delta[128] fp32 (bulk-loaded with Q / dO)
  // role Q
  static constexpr int kOffQq = 0, kOffDOq = kTile, kOffKq = 2 * kTile, kOffVq = 5 * kTile;  // K 3, V 2 stages
  static constexpr int kOffBar = 7 * kTile;
  static constexpr int kBytes = kOffBar + 256 + 1024;
  static_assert(kBytes <= 232448, "exceeds the 227 KB per-CTA shared memory");
  // key-tile variant staging dS for bulk stores (kDS = 1): a 32 KB staging tile after Q / dO, then
  // lse | delta, barriers; the alignment slack shrinks to 768 B (the dynamic window starts 1024-aligned)
  static constexpr int kOffStgD = 6 * kTile, kOffLDD = 7 * kTile, kOffBarD = 7 * kTile + 2048;
  static constexpr int kSlackD = 768;
  static constexpr int kBytesD = kOffBarD + 256 + kSlackD;
  static_assert(kBytesD <= 232448, "exceeds the 227 KB per-CTA shared memory");
};
constexpr int kBwdSThreads = 320;

__device__ __forceinline__ float4 lds_f4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
// exp2 of a packed pair: MUFU for most columns, the FMA-pipe polynomial for every 4th pair
template <bool kPoly>
__device__ __forceinline__ float2 exp2_pair(float2 x) {
  if constexpr (kPoly) return exp2_poly2(x);
  return make_float2(fast_exp2(x.x), fast_exp2(x.y));
}

// Entry e of the (role, tile) list sorted by decreasing work — KV key tile k: 4 (T - k) MMAs,
// Q query tile q: 3 (q + 1); ties put the KV tile first — without a table (no host copy, so the
// launch never synchronises the host): the work W at position e is the largest W with
// #{items of work >= W} > e (binary search), then the place inside the tie group picks the role.
// Returns k >= 0 for a KV tile, -(q + 1) for a Q tile.
__device__ __forceinline__ int split_entry(int e, int T) {
  auto count_ge = [&](int W) {  // items with work >= W
    const int a = T - (W + 3) / 4 + 1, b = T - (W + 2) / 3 + 1;
    return max(0, min(T, a)) + max(0, min(T, b));
  };
  int lo = 1, hi = 4 * T;  // count_ge(lo) = 2T > e; find the largest W with count_ge(W) > e
  while (lo < hi) {
    const int mid = (lo + hi + 1) / 2;
    if (count_ge(mid) > e) lo = mid;
    else hi = mid - 1;
  }
  const int W = lo;
  const int off = e - count_ge(W + 1);
  const bool has_kv = W % 4 == 0 && W / 4 <= T;
  if (off == 0 && has_kv) return T - W / 4;
  return -(W / 3 - 1) - 1;
}

// Causal dS tile store (kDS): tile (key tile k, query tile q >= k) of head h of a head group
// at slot k T - k (k - 1) / 2 + (q - k); each 32 KB tile is the shared-memory image of dS
// [128 queries x 128 keys] as a no-swizzle MN-major operand: byte (key / 32) * 8192 + (q / 8) * 512
// + (key % 32) * 16 + (q % 8) * 2 — core matrices of 8 keys x 8 queries (128 B), key groups 128 B
// apart inside a 32-key block, query groups 512 B apart — so the dQ kernel loads it with one bulk
// copy and each producing warp's 32 keys x 64 queries are 4 KB contiguous.
__host__ __device__ __forceinline__ int64_t ds_slot(int k, int q, int T) {
  return int64_t(k) * T - int64_t(k) * (k - 1) / 2 + (q - k);
}
__host__ __device__ __forceinline__ int64_t ds_tiles_per_head(int T) { return int64_t(T) * (T + 1) / 2; }

template <int kPolyKV, int kPolyQ, int kDS = 0>
__global__ void __launch_bounds__(kBwdSThreads, 1)
    attn_bwd_split_kernel(const __grid_constant__ CUtensorMap mQ, const __grid_constant__ CUtensorMap mK,
                          const __grid_constant__ CUtensorMap mV, const __grid_constant__ CUtensorMap mDO,
                          const float* __restrict__ nlse2,
                          const float* __restrict__ delta, __nv_bfloat16* __restrict__ dq_out,
                          __nv_bfloat16* __restrict__ dk_out, __nv_bfloat16* __restrict__ dv_out, int64_t ld_d, int S,
                          float scale, const __grid_constant__ AttnPush push, const float* __restrict__ rope_cos,
                          const float* __restrict__ rope_sin, int dbg, long long* trace,
                          uint8_t* __restrict__ ds_out, int h0) {
  using L = BwdSCfg;
  constexpr int D = 128;
  constexpr int kOffLD = kDS == 1 ? L::kOffLDD : L::kOffLD;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  if constexpr (kDS == 1) {
    if (smem - smem_raw > L::kSlackD) __trap();  // the layout assumes a (nearly) 1024-aligned window
  }
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + (kDS == 1 ? L::kOffBarD : L::kOffBar));
  uint64_t* fixed_full = bar + 0;  // KV: K, V   Q: Q, dO
  uint64_t* a_full = bar + 1;      // [3] KV: Q stages   Q: K stages
  uint64_t* a_empty = bar + 4;     // [3]
  uint64_t* b_full = bar + 7;      // [2] KV: dO stages  Q: V stages
  uint64_t* b_empty = bar + 9;     // [2]
  uint64_t* s_full = bar + 11;
  uint64_t* s_free = bar + 12;     // Q role: S read into registers
  uint64_t* p_full = bar + 13;     // KV role: P^T in TMEM
  uint64_t* dp_full = bar + 14;
  uint64_t* ds_full = bar + 15;
  uint64_t* acc_full = bar + 16;   // last gradient MMA done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 17);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int lin = static_cast<int>(blockIdx.y * gridDim.x + blockIdx.x);
  // kDS: key tiles only (k ascending = work descending), heads h0.. of the group
  const int entry = kDS ? lin / static_cast<int>(gridDim.y) : split_entry(lin / static_cast<int>(gridDim.y), S / 128);
  const int h = h0 + static_cast<int>(blockIdx.z * gridDim.y) + lin % static_cast<int>(gridDim.y);
  const bool role_q = entry < 0;
  const int tile = role_q ? -entry - 1 : entry;  // KV: key tile kt; Q: query tile qt
  const int T = S / 128;
  const int n = role_q ? tile + 1 : T - tile;    // KV: query tiles kt..T-1; Q: key tiles 0..qt
  const int t0 = role_q ? 0 : tile;              // first streamed tile index
  if (((dbg & 16) && role_q) || ((dbg & 32) && !role_q)) return;  // development: one role alone

  if (warp == 8 && lane == 0) {
    tma_prefetch(&mQ); tma_prefetch(&mK); tma_prefetch(&mV); tma_prefetch(&mDO);
    mbar_init(fixed_full, 1);
    for (int s = 0; s < 3; ++s) { mbar_init(&a_full[s], 1); mbar_init(&a_empty[s], 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(&b_full[s], 1); mbar_init(&b_empty[s], 1); }
    mbar_init(s_full, 1);
    mbar_init(s_free, 8);
    mbar_init(p_full, 8);
    mbar_init(dp_full, 1);
    mbar_init(ds_full, 8);
    mbar_init(acc_full, 1);
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem, tP = tmem + 128, tG0 = tmem + 256, tG1 = tmem + 384;  // KV: dK, dV; Q: dQ
  const int NA = role_q ? 3 : 2;  // stages of the A stream (KV: Q; Q: K)

  if (warp == 8) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      const int own = tile * 128;
      mbar_arrive_expect_tx(fixed_full, 2 * L::kTile);
      for (int c = 0; c < 2; ++c) {
        if (role_q) {
          tma_load_2d(smem + L::kOffQq + c * (L::kTile / 2), &mQ, fixed_full, h * D + c * 64, own);
          tma_load_2d(smem + L::kOffDOq + c * (L::kTile / 2), &mDO, fixed_full, h * D + c * 64, own);
        } else {
          tma_load_2d(smem + L::kOffK + c * (L::kTile / 2), &mK, fixed_full, h * D + c * 64, own);
          tma_load_2d(smem + L::kOffV + c * (L::kTile / 2), &mV, fixed_full, h * D + c * 64, own);
        }
      }
      for (int i = 0; i < n; ++i) {
        const int row = (t0 + i) * 128;
        const int sa = i % NA, sb = i & 1;
        if (i >= NA) mbar_wait(&a_empty[sa], ((i / NA) - 1) & 1);
        mbar_arrive_expect_tx(&a_full[sa], L::kTile + (role_q ? 0 : 512));
        if (!role_q) bulk_load(smem + kOffLD + sa * 1024, nlse2 + static_cast<int64_t>(h) * S + row, 512, &a_full[sa]);
        for (int c = 0; c < 2; ++c) {
          if (role_q)
            tma_load_2d(smem + L::kOffKq + sa * L::kTile + c * (L::kTile / 2), &mK, &a_full[sa], h * D + c * 64, row);
          else
            tma_load_2d(smem + L::kOffQ + sa * L::kTile + c * (L::kTile / 2), &mQ, &a_full[sa], h * D + c * 64, row);
        }
        if (i >= 2) mbar_wait(&b_empty[sb], ((i >> 1) - 1) & 1);
        mbar_arrive_expect_tx(&b_full[sb], L::kTile + (role_q ? 0 : 512));
        if (!role_q)
          bulk_load(smem + kOffLD + sb * 1024 + 512, delta + static_cast<int64_t>(h) * S + row, 512, &b_full[sb]);
        for (int c = 0; c < 2; ++c) {
          if (role_q)
            tma_load_2d(smem + L::kOffVq + sb * L::kTile + c * (L::kTile / 2), &mV, &b_full[sb], h * D + c * 64, row);
          else
            tma_load_2d(smem + L::kOffDO + sb * L::kTile + c * (L::kTile / 2), &mDO, &b_full[sb], h * D + c * 64, row);
        }
      }
    }
  } else if (warp == 9) {
    if (lane == 0) {
      // ---------------- MMA issuer ----------------
      constexpr uint32_t idSS = make_idesc_bf16(128, 128, false, false);  // S / S^T, dP / dP^T: K-major
      constexpr uint32_t idG = make_idesc_bf16(128, 128, false, true);    // A in TMEM, B MN-major
      auto mma_ss = [&](uint32_t d, uint32_t a, uint32_t b) {  // K = d: 8 steps of 16 head dims
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t off = (k >> 2) * (L::kTile / 2) + (k & 3) * 32;
          tc_mma_bf16(d, make_sw128_desc(a + off, 16, 1024), make_sw128_desc(b + off, 16, 1024), idSS, k > 0);
        }
      };
      // A from TMEM (packed bf16 pairs, 64 columns per 128-wide half at +64), B [128 x 128] MN-major
      auto mma_ts = [&](uint32_t d, uint32_t a_tm, uint32_t b, bool acc) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
          tc_mma_bf16_ts(d, a_tm + (k >> 2) * 64 + (k & 3) * 8, make_sw128_desc(b + k * 2048, L::kTile / 2, 1024),
                         idG, (acc || k > 0) ? 1u : 0u);
      };
      mbar_wait(fixed_full, 0);
      if (!role_q) {
        const uint32_t sK = smem_u32(smem + L::kOffK), sV = smem_u32(smem + L::kOffV);
        auto sQ = [&](int s) { return smem_u32(smem + L::kOffQ + s * L::kTile); };
        auto sDO = [&](int s) { return smem_u32(smem + L::kOffDO + s * L::kTile); };
        mbar_wait(&a_full[0], 0);
        tc_fence_after();
        mma_ss(tS, sK, sQ(0));
        tc_commit(s_full);
        mbar_wait(&b_full[0], 0);
        tc_fence_after();
        mma_ss(tP, sV, sDO(0));
        tc_commit(dp_full);
        const bool tr = trace && lin == 0;
        for (int i = 0; i < n; ++i) {
          const int s = i & 1, s1 = (i + 1) & 1;
          if (tr && i < 64) trace[i * 8 + 0] = clock64();
          if (i + 1 < n) {
            mbar_wait(s_free, i & 1);  // S^T(i) is in registers
            mbar_wait(&a_full[s1], ((i + 1) >> 1) & 1);
            tc_fence_after();
            mma_ss(tS, sK, sQ(s1));
            tc_commit(s_full);
          }
          if (tr && i < 64) trace[i * 8 + 1] = clock64();
          mbar_wait(ds_full, i & 1);  // P^T(i), dS^T(i) in the dP^T columns
          if (tr && i < 64) trace[i * 8 + 2] = clock64();
          tc_fence_after();
          mma_ts(tG1, tP, sDO(s), i > 0);       // dV += P^T dO(i)
          tc_commit(&b_empty[s]);
          mma_ts(tG0, tP + 32, sQ(s), i > 0);  // dK += dS^T Q(i)
          tc_commit(&a_empty[s]);
          if (i + 1 < n) {
            mbar_wait(&b_full[s1], ((i + 1) >> 1) & 1);
            tc_fence_after();
            mma_ss(tP, sV, sDO(s1));  // dP^T(i+1) over P^T / dS^T(i), consumed by dV(i) / dK(i) before it
            tc_commit(dp_full);
          }
          if (tr && i < 64) trace[i * 8 + 3] = clock64();
        }
      } else {
        const uint32_t sQ = smem_u32(smem + L::kOffQq), sDO = smem_u32(smem + L::kOffDOq);
        auto sK = [&](int s) { return smem_u32(smem + L::kOffKq + s * L::kTile); };
        auto sV = [&](int s) { return smem_u32(smem + L::kOffVq + s * L::kTile); };
        mbar_wait(&a_full[0], 0);
        tc_fence_after();
        mma_ss(tS, sQ, sK(0));
        tc_commit(s_full);
        mbar_wait(&b_full[0], 0);
        tc_fence_after();
        mma_ss(tP, sDO, sV(0));
        tc_commit(&b_empty[0]);
        tc_commit(dp_full);
        for (int j = 0; j < n; ++j) {
          if (j + 1 < n) {
            const int sa = (j + 1) % 3;
            mbar_wait(s_free, j & 1);  // S(j) is in registers
            mbar_wait(&a_full[sa], ((j + 1) / 3) & 1);
            tc_fence_after();
            mma_ss(tS, sQ, sK(sa));
            tc_commit(s_full);
          }
          mbar_wait(ds_full, j & 1);
          tc_fence_after();
          mma_ts(tG0, tP, sK(j % 3), j > 0);  // dQ += dS K(j)
          tc_commit(&a_empty[j % 3]);
          if (j + 1 < n) {
            const int sb = (j + 1) & 1;
            mbar_wait(&b_full[sb], ((j + 1) >> 1) & 1);
            tc_fence_after();
            mma_ss(tP, sDO, sV(sb));  // dP(j+1) over dS(j), consumed by dQ(j) before it
            tc_commit(&b_empty[sb]);
            tc_commit(dp_full);
          }
        }
      }
      tc_commit(acc_full);
    }
  } else {
    // ---------------- math warps 0..7 ----------------
    const int quad = warp & 3, half = warp >> 2;
    const int r = quad * 32 + lane;  // TMEM lane: KV key row / Q query row
    const uint32_t lo = static_cast<uint32_t>(quad * 32) << 16;
    const float scale_log2 = scale * kLog2e;
    // exponentials: MUFU.EX2 for all but kPoly of every 8 pairs (the math warps are issue-bound,
    // and the polynomial costs ~5 issue slots per element against 1 for MUFU)
    auto exp_pair = [&](int j4, int e2, float2 x, int kPoly) {
      return (2 * (j4 & 3) + e2 < kPoly) ? exp2_pair<true>(x) : exp2_pair<false>(x);
    };
    if (!role_q) {
      const int key = tile * 128 + r;
      // one query tile; kDiag (the first tile only) masks key > query
      auto kv_tile = [&](int i, auto diag_c) {
        constexpr bool kDiag = decltype(diag_c)::value;
        const int qb = (tile + i) * 128 + half * 64;  // this warp's 64 queries
        const bool tr = trace && lin == 0 && warp == 0 && lane == 0 && i < 64;
        float pf[64];
        uint32_t sv[64];
        mbar_wait(s_full, i & 1);
        if (tr) trace[i * 8 + 4] = clock64();
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld_x16(tS + lo + half * 64 + c * 16, *reinterpret_cast<uint32_t(*)[16]>(&sv[c * 16]));
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(s_free);  // S^T(i+1) may overwrite the S^T columns
        mbar_wait(&a_full[i & 1], (i >> 1) & 1);  // this tile's -lse*log2e (with Q(i)) is in shared memory
        const uint32_t l4 = smem_u32(smem + kOffLD + (i & 1) * 1024 + half * 256);
#pragma unroll
        for (int j4 = 0; j4 < 16; ++j4) {
          const float4 l = lds_f4(l4 + j4 * 16);  // warp-uniform: shared-memory broadcast
          const float2 x01 = __ffma2_rn(make_float2(__uint_as_float(sv[j4 * 4]), __uint_as_float(sv[j4 * 4 + 1])),
                                        make_float2(scale_log2, scale_log2), make_float2(l.x, l.y));
          const float2 x23 = __ffma2_rn(make_float2(__uint_as_float(sv[j4 * 4 + 2]), __uint_as_float(sv[j4 * 4 + 3])),
                                        make_float2(scale_log2, scale_log2), make_float2(l.z, l.w));
          const float2 p01 = exp_pair(j4, 0, x01, kPolyKV), p23 = exp_pair(j4, 1, x23, kPolyKV);
          pf[j4 * 4 + 0] = p01.x; pf[j4 * 4 + 1] = p01.y;
          pf[j4 * 4 + 2] = p23.x; pf[j4 * 4 + 3] = p23.y;
        }
        if constexpr (kDiag) {
#pragma unroll
          for (int j = 0; j < 64; ++j)
            if (key > qb + j) pf[j] = 0.f;
        }
        if (tr) trace[i * 8 + 5] = clock64();
        mbar_wait(dp_full, i & 1);
        if (tr) trace[i * 8 + 6] = clock64();
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld_x16(tP + lo + half * 64 + c * 16, *reinterpret_cast<uint32_t(*)[16]>(&sv[c * 16]));
        tmem_ld_wait();
        mbar_wait(&b_full[i & 1], (i >> 1) & 1);  // this tile's delta (with dO(i)) is in shared memory
        const uint32_t d4 = smem_u32(smem + kOffLD + (i & 1) * 1024 + 512 + half * 256);
        uint32_t pk[32], dk[32];
        // kDS: the tile image is the no-swizzle MN-major operand layout (8 keys x 8 queries core
        // matrices of 128 B, key groups 128 B apart, query groups 2 KB apart), so chunk c of the 32
        // key rows of this warp is 512 contiguous bytes: one fully coalesced store per chunk (a
        // swizzled row-per-thread image touches 32 lines per instruction and saturates the LSU;
        // staging it through shared memory competes with the SS MMAs for the shared-memory port)
#pragma unroll
        for (int j4 = 0; j4 < 16; ++j4) {
          const float4 dl = lds_f4(d4 + j4 * 16);
          const float2 a01 = __fadd2_rn(make_float2(__uint_as_float(sv[j4 * 4]), __uint_as_float(sv[j4 * 4 + 1])),
                                        make_float2(-dl.x, -dl.y));
          const float2 a23 = __fadd2_rn(make_float2(__uint_as_float(sv[j4 * 4 + 2]), __uint_as_float(sv[j4 * 4 + 3])),
                                        make_float2(-dl.z, -dl.w));
          const float2 d01 = __fmul2_rn(make_float2(pf[j4 * 4], pf[j4 * 4 + 1]), a01);
          const float2 d23 = __fmul2_rn(make_float2(pf[j4 * 4 + 2], pf[j4 * 4 + 3]), a23);
          dk[j4 * 2] = pack_bf16(d01.x, d01.y);
          dk[j4 * 2 + 1] = pack_bf16(d23.x, d23.y);
          pk[j4 * 2] = pack_bf16(pf[j4 * 4], pf[j4 * 4 + 1]);
          pk[j4 * 2 + 1] = pack_bf16(pf[j4 * 4 + 2], pf[j4 * 4 + 3]);
        }
        // P^T | dS^T over this warp's own 64 dP^T columns (all read above): A operands of dV / dK
        tmem_st_32x32b_x32(tP + lo + half * 64, pk);
        tmem_st_32x32b_x32(tP + lo + half * 64 + 32, dk);

        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(ds_full);
        if (tr) trace[i * 8 + 7] = clock64();
        // kDS: dS leaves after the MMA warp has it (off the tile's critical path). This warp's 32 keys
        // x 64 queries are 4 KB contiguous in the tile image (ds_slot): chunk c (queries 8c..8c+7)
        // of its keys is 512 contiguous bytes, one coalesced 16-B store per thread
        if (kDS != 0 && !(dbg & 512)) {  // dbg 512 / 256: development, no dS store / no bulk store
          const int64_t toff = ((int64_t(h - h0) * ds_tiles_per_head(T) + ds_slot(tile, tile + i, T)) << 15) +
                               quad * 8192 + half * 4096;
          if constexpr (kDS == 1) {  // staged in shared memory, one 4 KB bulk store per warp
            uint8_t* stg = smem + L::kOffStgD + quad * 8192 + half * 4096;
            if (lane == 0) bulk_wait_read();  // the previous tile's store has read these rows
            __syncwarp();
#pragma unroll
            for (int c = 0; c < 8; ++c)
              asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(smem_u32(stg + c * 512 + lane * 16)),
                           "r"(dk[c * 4]), "r"(dk[c * 4 + 1]), "r"(dk[c * 4 + 2]), "r"(dk[c * 4 + 3])
                           : "memory");
            fence_proxy_async();
            __syncwarp();
            if (lane == 0 && !(dbg & 256)) bulk_store_stream(ds_out + toff, stg, 4096, l2_evict_first_policy());
          } else {
            uint8_t* dst = ds_out + toff + lane * 16;
#pragma unroll
            for (int c = 0; c < 8; ++c)
              *reinterpret_cast<uint4*>(dst + c * 512) = make_uint4(dk[c * 4], dk[c * 4 + 1], dk[c * 4 + 2], dk[c * 4 + 3]);
          }
        }
      };
      for (int i = 0; i < n; ++i) {
        if (dbg & 8) {  // development: MMA pipeline bound (no P / dS math)
          mbar_wait(s_full, i & 1);
          if (lane == 0) mbar_arrive(s_free);
          mbar_wait(dp_full, i & 1);
          if (lane == 0) mbar_arrive(ds_full);
          continue;
        }
        if (i == 0) kv_tile(i, std::true_type{});
        else kv_tile(i, std::false_type{});
      }
    } else {
      const int q = tile * 128 + r;
      const float nl2 = nlse2[static_cast<int64_t>(h) * S + q];
      const float dl = delta[static_cast<int64_t>(h) * S + q];
      // one key tile; kDiag (the last tile only) masks key > query
      auto q_tile = [&](int j, auto diag_c) {
        constexpr bool kDiag = decltype(diag_c)::value;
        const int kb = j * 128 + half * 64;  // this warp's 64 keys
        float pf[64];
        uint32_t sv[64];
        mbar_wait(s_full, j & 1);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld_x16(tS + lo + half * 64 + c * 16, *reinterpret_cast<uint32_t(*)[16]>(&sv[c * 16]));
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(s_free);  // S(j+1) may overwrite the S columns
#pragma unroll
        for (int j4 = 0; j4 < 16; ++j4) {
          const float2 x01 = __ffma2_rn(make_float2(__uint_as_float(sv[j4 * 4]), __uint_as_float(sv[j4 * 4 + 1])),
                                        make_float2(scale_log2, scale_log2), make_float2(nl2, nl2));
          const float2 x23 = __ffma2_rn(make_float2(__uint_as_float(sv[j4 * 4 + 2]), __uint_as_float(sv[j4 * 4 + 3])),
                                        make_float2(scale_log2, scale_log2), make_float2(nl2, nl2));
          const float2 p01 = exp_pair(j4, 0, x01, kPolyQ), p23 = exp_pair(j4, 1, x23, kPolyQ);
          pf[j4 * 4 + 0] = p01.x; pf[j4 * 4 + 1] = p01.y;
          pf[j4 * 4 + 2] = p23.x; pf[j4 * 4 + 3] = p23.y;
        }
        if constexpr (kDiag) {
#pragma unroll
          for (int e = 0; e < 64; ++e)
            if (kb + e > q) pf[e] = 0.f;
        }
        mbar_wait(dp_full, j & 1);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld_x16(tP + lo + half * 64 + c * 16, *reinterpret_cast<uint32_t(*)[16]>(&sv[c * 16]));
        tmem_ld_wait();
        uint32_t dk[32];
#pragma unroll
        for (int j2 = 0; j2 < 32; ++j2) {
          const float2 a2 = __fadd2_rn(make_float2(__uint_as_float(sv[2 * j2]), __uint_as_float(sv[2 * j2 + 1])),
                                       make_float2(-dl, -dl));
          const float2 d2 = __fmul2_rn(make_float2(pf[2 * j2], pf[2 * j2 + 1]), a2);
          dk[j2] = pack_bf16(d2.x, d2.y);
        }
        tmem_st_32x32b_x32(tP + lo + half * 64, dk);  // dS over this warp's own, already read dP columns
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(ds_full);
      };
      for (int j = 0; j < n; ++j) {
        if (dbg & 8) {  // development: MMA pipeline bound (no P / dS math)
          mbar_wait(s_full, j & 1);
          if (lane == 0) mbar_arrive(s_free);
          mbar_wait(dp_full, j & 1);
          if (lane == 0) mbar_arrive(ds_full);
          continue;
        }
        if (j == n - 1) q_tile(j, std::true_type{});
        else q_tile(j, std::false_type{});
      }
    }
    if constexpr (kDS == 1) {
      if (lane == 0) bulk_wait_all();  // the last dS stores are complete
    }
    // epilogue: KV role dK (scaled) | dV; Q role dQ (scaled) -> bf16 rows (or pushed to the owner rank).
    // With rope_cos, dK / dQ leave through the inverse rotary embedding (d/dx of RoPE(x) is R^T)
    // from fp32, so the rotated q / k gradients are rounded to bf16 once.
    mbar_wait(acc_full, 0);
    tc_fence_after();
    const int tok = tile * 128 + r;
    int64_t off = static_cast<int64_t>(tok) * ld_d + h * D;
    __nv_bfloat16* base0 = role_q ? dq_out : dk_out;
    __nv_bfloat16* base1 = dv_out;
    if (push.p[0]) {  // fused all-to-all: rows go to the owner rank of the token
      const int owner = tok / push.T;
      __nv_bfloat16* pb = static_cast<__nv_bfloat16*>(push.p[owner]);
      off = static_cast<int64_t>(tok - owner * push.T) * push.ld + h * D;
      base0 = pb + (role_q ? push.col_q : push.col_k);
      base1 = pb + push.col_v;
    }
    auto store32 = [&](__nv_bfloat16* dst, const float (&v)[32]) {
      uint4* o4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
      for (int v4 = 0; v4 < 4; ++v4)
        o4[v4] = make_uint4(pack_bf16(v[v4 * 8], v[v4 * 8 + 1]), pack_bf16(v[v4 * 8 + 2], v[v4 * 8 + 3]),
                            pack_bf16(v[v4 * 8 + 4], v[v4 * 8 + 5]), pack_bf16(v[v4 * 8 + 6], v[v4 * 8 + 7]));
    };
    if (rope_cos) {  // this thread: rotation pairs (i, i + 64), i in [32 half, 32 half + 32)
      uint32_t a[32], b[32];
      tmem_ld_32x32b_x32(tG0 + lo + half * 32, a);
      tmem_ld_32x32b_x32(tG0 + lo + 64 + half * 32, b);
      tmem_ld_wait();
      const float* cs = rope_cos + static_cast<int64_t>(tok) * (D / 2) + half * 32;
      const float* sn = rope_sin + static_cast<int64_t>(tok) * (D / 2) + half * 32;
      float fl[32], fh[32];
#pragma unroll
      for (int i = 0; i < 32; i += 4) {
        const float4 c4 = *reinterpret_cast<const float4*>(cs + i), s4 = *reinterpret_cast<const float4*>(sn + i);
        const float cv[4] = {c4.x, c4.y, c4.z, c4.w}, sv4[4] = {s4.x, s4.y, s4.z, s4.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float x = __uint_as_float(a[i + e]) * scale, y = __uint_as_float(b[i + e]) * scale;
          fl[i + e] = x * cv[e] + y * sv4[e];
          fh[i + e] = y * cv[e] - x * sv4[e];
        }
      }
      store32(base0 + off + half * 32, fl);
      store32(base0 + off + 64 + half * 32, fh);
    } else {
#pragma unroll 1
      for (int c = 0; c < 2; ++c) {
        const int col = half * 64 + c * 32;
        uint32_t a[32];
        tmem_ld_32x32b_x32(tG0 + lo + col, a);
        tmem_ld_wait();
        float f[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) f[e] = __uint_as_float(a[e]) * scale;
        store32(base0 + off + col, f);
      }
    }
    if (!role_q) {
#pragma unroll 1
      for (int c = 0; c < 2; ++c) {
        const int col = half * 64 + c * 32;
        uint32_t a[32];
        tmem_ld_32x32b_x32(tG1 + lo + col, a);
        tmem_ld_wait();
        float f[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) f[e] = __uint_as_float(a[e]);
        store32(base1 + off + col, f);
      }
    }
    if (push.p[0]) __threadfence_system();  // pushed rows visible before the next barrier flag
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// dQ from the stored dS tiles (the kDS key-tile kernel): dQ(q) = scale * sum_{k <= q} dS(q, k) K(k),
// both operands MN-major from shared memory (dS tile: one 32 KB bulk copy; K: TMA), fp32 in TMEM,
// then the query-tile epilogue (inverse RoPE from fp32; bf16 rows or pushed to the owner rank).
// One MMA per tile pair; bound by the HBM stream of dS.
// ND dS stages and NK K stages: the dS stream comes from HBM, the K tiles mostly from L2, so the
// dS ring runs ND - NK tiles ahead of the K ring (more HBM bytes in flight per SM).
template <int ND, int NK>
struct BwdDqCfg {
  static constexpr int kTile = 128 * 128 * 2;
  static constexpr int kOffDS = 0, kOffK = ND * kTile;
  static constexpr int kOffBar = (ND + NK) * kTile;
  static constexpr int kBytes = kOffBar + 256 + 1024;
  static_assert(kBytes <= 232448, "exceeds the 227 KB per-CTA shared memory");
};
constexpr int kBwdDqThreads = 192;  // warps 0..3 epilogue (one TMEM lane quadrant each), 4 TMA, 5 MMA

template <int ND, int NK>
__global__ void __launch_bounds__(kBwdDqThreads, 1)
    attn_bwd_dq_kernel(const __grid_constant__ CUtensorMap mK, const uint8_t* __restrict__ ds,
                       __nv_bfloat16* __restrict__ dq_out, int64_t ld_d, int S, float scale,
                       const __grid_constant__ AttnPush push, const float* __restrict__ rope_cos,
                       const float* __restrict__ rope_sin, int h0) {
  using L = BwdDqCfg<ND, NK>;
  constexpr int D = 128;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::kOffBar);
  uint64_t* full_d = bar;              // [ND]
  uint64_t* empty_d = bar + ND;        // [ND]
  uint64_t* full_k = bar + 2 * ND;     // [NK]
  uint64_t* empty_k = full_k + NK;     // [NK]
  uint64_t* acc_full = empty_k + NK;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int lin = static_cast<int>(blockIdx.y * gridDim.x + blockIdx.x);
  const int T = S / 128;
  const int qt = T - 1 - lin / static_cast<int>(gridDim.y);  // heaviest (latest) query tiles first
  const int hg = static_cast<int>(blockIdx.z * gridDim.y) + lin % static_cast<int>(gridDim.y);
  const int h = h0 + hg;
  const int n = qt + 1;

  if (warp == 4 && lane == 0) {
    tma_prefetch(&mK);
    for (int s = 0; s < ND; ++s) { mbar_init(&full_d[s], 1); mbar_init(&empty_d[s], 1); }
    for (int s = 0; s < NK; ++s) { mbar_init(&full_k[s], 1); mbar_init(&empty_k[s], 1); }
    mbar_init(acc_full, 1);
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc<128>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 4) {
    if (lane == 0) {
      const uint8_t* dsh = ds + (int64_t(hg) * ds_tiles_per_head(T) << 15);
      const uint64_t pol = l2_evict_first_policy();
      constexpr int kLead = ND - NK;  // dS tiles issued ahead of the K tiles
      for (int i = 0; i < n + kLead; ++i) {
        if (i < n) {
          const int s = i % ND;
          if (i >= ND) mbar_wait(&empty_d[s], ((i / ND) - 1) & 1);
          mbar_arrive_expect_tx(&full_d[s], L::kTile);
          bulk_load_stream(smem + L::kOffDS + s * L::kTile, dsh + (ds_slot(i, qt, T) << 15), L::kTile, &full_d[s],
                           pol);
        }
        const int k = i - kLead;
        if (k >= 0 && k < n) {
          const int s = k % NK;
          if (k >= NK) mbar_wait(&empty_k[s], ((k / NK) - 1) & 1);
          mbar_arrive_expect_tx(&full_k[s], L::kTile);
          for (int c = 0; c < 2; ++c)
            tma_load_2d(smem + L::kOffK + s * L::kTile + c * (L::kTile / 2), &mK, &full_k[s], h * D + c * 64, k * 128);
        }
      }
    }
  } else if (warp == 5) {
    if (lane == 0) {
      constexpr uint32_t id = make_idesc_bf16(128, 128, true, true);  // A = dS, B = K: both MN-major
      // A: no-swizzle MN-major (ds_slot layout): for MN-major operands the leading byte offset is the
      // K-direction core-matrix stride (key groups, 128 B) and the stride byte offset the MN-direction
      // one (query groups, 512 B); the 16 keys of MMA kk start at (kk / 2) * 8192 + (kk % 2) * 256
      for (int k = 0; k < n; ++k) {
        const int sd = k % ND, sk = k % NK;
        mbar_wait(&full_d[sd], (k / ND) & 1);
        mbar_wait(&full_k[sk], (k / NK) & 1);
        tc_fence_after();
        const uint32_t a = smem_u32(smem + L::kOffDS + sd * L::kTile), b = smem_u32(smem + L::kOffK + sk * L::kTile);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)  // 16 keys per MMA
          tc_mma_bf16(tmem, make_nosw_desc(a + (kk >> 1) * 8192 + (kk & 1) * 256, 128, 512),
                      make_sw128_desc(b + kk * 2048, L::kTile / 2, 1024), id, (k > 0 || kk > 0) ? 1u : 0u);
        tc_commit(&empty_d[sd]);
        tc_commit(&empty_k[sk]);
      }
      tc_commit(acc_full);
    }
  } else {
    const int r = warp * 32 + lane;
    const uint32_t lo = static_cast<uint32_t>(warp * 32) << 16;
    mbar_wait(acc_full, 0);
    tc_fence_after();
    const int tok = qt * 128 + r;
    int64_t off = static_cast<int64_t>(tok) * ld_d + h * D;
    __nv_bfloat16* base = dq_out;
    if (push.p[0]) {  // fused all-to-all: the row goes to the owner rank of the token
      const int owner = tok / push.T;
      off = static_cast<int64_t>(tok - owner * push.T) * push.ld + h * D;
      base = static_cast<__nv_bfloat16*>(push.p[owner]) + push.col_q;
    }
    auto store32 = [&](__nv_bfloat16* dst, const float (&v)[32]) {
      uint4* o4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
      for (int v4 = 0; v4 < 4; ++v4)
        o4[v4] = make_uint4(pack_bf16(v[v4 * 8], v[v4 * 8 + 1]), pack_bf16(v[v4 * 8 + 2], v[v4 * 8 + 3]),
                            pack_bf16(v[v4 * 8 + 4], v[v4 * 8 + 5]), pack_bf16(v[v4 * 8 + 6], v[v4 * 8 + 7]));
    };
#pragma unroll 1
    for (int half = 0; half < 2; ++half) {
      if (rope_cos) {  // rotation pairs (i, i + 64), i in [32 half, 32 half + 32)
        uint32_t a[32], b[32];
        tmem_ld_32x32b_x32(tmem + lo + half * 32, a);
        tmem_ld_32x32b_x32(tmem + lo + 64 + half * 32, b);
        tmem_ld_wait();
        const float* cs = rope_cos + static_cast<int64_t>(tok) * (D / 2) + half * 32;
        const float* sn = rope_sin + static_cast<int64_t>(tok) * (D / 2) + half * 32;
        float fl[32], fh[32];
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          const float4 c4 = *reinterpret_cast<const float4*>(cs + i), s4 = *reinterpret_cast<const float4*>(sn + i);
          const float cv[4] = {c4.x, c4.y, c4.z, c4.w}, sv4[4] = {s4.x, s4.y, s4.z, s4.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float x = __uint_as_float(a[i + e]) * scale, y = __uint_as_float(b[i + e]) * scale;
            fl[i + e] = x * cv[e] + y * sv4[e];
            fh[i + e] = y * cv[e] - x * sv4[e];
          }
        }
        store32(base + off + half * 32, fl);
        store32(base + off + 64 + half * 32, fh);
      } else {
#pragma unroll 1
        for (int c = 0; c < 2; ++c) {
          const int col = half * 64 + c * 32;
          uint32_t a[32];
          tmem_ld_32x32b_x32(tmem + lo + col, a);
          tmem_ld_wait();
          float f[32];
#pragma unroll
          for (int e = 0; e < 32; ++e) f[e] = __uint_as_float(a[e]) * scale;
          store32(base + off + col, f);
        }
      }
    }
    if (push.p[0]) __threadfence_system();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc<128>(tmem);
  }
}

}  // namespace

long long* g_attn_trace = nullptr;  // development: clock64 trace of CTA (0,0)
long long* g_attn_trace_fwd = nullptr;
extern "C" void seqplan_isp_debug_set_trace(long long* dev_buf) { g_attn_trace = dev_buf; }
extern "C" void seqplan_isp_debug_set_trace_fwd(long long* dev_buf) { g_attn_trace_fwd = dev_buf; }

// Atomic-free backward (attn_bwd_split_kernel): (role, tile) entries in decreasing work
// (split_entry); delta and nlse2 = -lse*log2e computed before; dq/dk/dv bf16.
cudaError_t attention_bwd_nored_tc(const AttnTensors& t, const __nv_bfloat16* dout, int64_t ld_dout, __nv_bfloat16* dq,
                                   __nv_bfloat16* dk, __nv_bfloat16* dv, int64_t ld_d, const float* delta,
                                   const float* nlse2, cudaStream_t st) {
  if (t.d != 128 || t.S % 128) return cudaErrorInvalidValue;
  using L = BwdSCfg;
  const char* pe = std::getenv("SEQPLAN_ISP_BWD_POLY");  // development: exponential split (kv*10+q)
  const int poly = pe ? std::atoi(pe) : 0;
  auto kern = attn_bwd_split_kernel<0, 0>;
  switch (poly) {
    case 33: kern = attn_bwd_split_kernel<3, 3>; break;
    case 22: kern = attn_bwd_split_kernel<2, 2>; break;
    case 43: kern = attn_bwd_split_kernel<4, 3>; break;
    case 42: kern = attn_bwd_split_kernel<4, 2>; break;
    case 53: kern = attn_bwd_split_kernel<5, 3>; break;
    default: break;
  }
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kBytes) != cudaSuccess)
    return cudaErrorInvalidValue;
  const int T = t.S / 128;
  CUtensorMap mq, mk, mv, mdo;
  const int64_t cols = static_cast<int64_t>(t.heads) * 128;
  if (!map2d(&mq, t.q, t.S, cols, t.ld_qkv, 128) || !map2d(&mk, t.k, t.S, cols, t.ld_qkv, 128) ||
      !map2d(&mv, t.v, t.S, cols, t.ld_qkv, 128) || !map2d(&mdo, dout, t.S, cols, ld_dout, 128))
    return cudaErrorInvalidValue;
  const float scale = 1.0f / sqrtf(128.0f);
  const int dbg = std::getenv("SEQPLAN_ISP_DBG") ? std::atoi(std::getenv("SEQPLAN_ISP_DBG")) : 0;
  kern<<<lpt_grid(2 * T, t.heads, t.S, 128), kBwdSThreads, L::kBytes, st>>>(
      mq, mk, mv, mdo, nlse2, delta, dq, dk, dv, ld_d, t.S, scale, t.push, t.rope_cos, t.rope_sin, dbg,
      g_attn_trace, nullptr, 0);
  return cudaGetLastError();
}

int64_t attention_bwd_ds_head_bytes(int S) { return ds_tiles_per_head(S / 128) << 15; }

// Key-tile kernel storing dS (kDS) + the dQ kernel, per group of heads whose dS tiles fit ws.
cudaError_t attention_bwd_ds_tc(const AttnTensors& t, const __nv_bfloat16* dout, int64_t ld_dout, __nv_bfloat16* dq,
                                __nv_bfloat16* dk, __nv_bfloat16* dv, int64_t ld_d, const float* delta,
                                const float* nlse2, void* ws, int64_t ws_bytes, cudaStream_t st) {
  if (t.d != 128 || t.S % 128) return cudaErrorInvalidValue;
  const int64_t per_head = attention_bwd_ds_head_bytes(t.S);
  const int G = static_cast<int>(std::min<int64_t>(t.heads, ws_bytes / per_head));
  if (G < 1 || !ws) return cudaErrorInvalidValue;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(attn_bwd_split_kernel<0, 0, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             BwdSCfg::kBytesD) != cudaSuccess ||
        cudaFuncSetAttribute(attn_bwd_split_kernel<0, 0, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             BwdSCfg::kBytes) != cudaSuccess ||
        cudaFuncSetAttribute(attn_bwd_dq_kernel<3, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             BwdDqCfg<3, 3>::kBytes) != cudaSuccess ||
        cudaFuncSetAttribute(attn_bwd_dq_kernel<5, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             BwdDqCfg<5, 2>::kBytes) != cudaSuccess)
      return cudaErrorInvalidValue;
    attr = true;
  }
  const int T = t.S / 128;
  CUtensorMap mq, mk, mv, mdo;
  const int64_t cols = static_cast<int64_t>(t.heads) * 128;
  if (!map2d(&mq, t.q, t.S, cols, t.ld_qkv, 128) || !map2d(&mk, t.k, t.S, cols, t.ld_qkv, 128) ||
      !map2d(&mv, t.v, t.S, cols, t.ld_qkv, 128) || !map2d(&mdo, dout, t.S, cols, ld_dout, 128))
    return cudaErrorInvalidValue;
  const float scale = 1.0f / sqrtf(128.0f);
  const int dbg = std::getenv("SEQPLAN_ISP_DBG") ? std::atoi(std::getenv("SEQPLAN_ISP_DBG")) : 0;
  uint8_t* w = static_cast<uint8_t*>(ws);
  const bool direct = std::getenv("SEQPLAN_ISP_DS_DIRECT") != nullptr;  // development: st.global instead of bulk
  // dQ kernel rings: 3 dS + 3 K stages; SEQPLAN_ISP_DQ_STAGES=52 (5 dS ahead of 2 K) measured slower
  // (32K x 32 heads: dQ 6.0 vs 5.23 ms)
  static const bool deep = [] {
    const char* e = std::getenv("SEQPLAN_ISP_DQ_STAGES");
    return e && std::atoi(e) == 52;
  }();
  cudaEvent_t tev[3] = {};
  const bool timed = (dbg & 1024) != 0;  // development: per-kernel event times of the first group
  if (timed)
    for (auto& e : tev) cudaEventCreate(&e);
  for (int h0 = 0; h0 < t.heads; h0 += G) {
    const int g = std::min(G, t.heads - h0);
    const dim3 grid = lpt_grid(T, g, t.S, 128);
    if (timed && h0 == 0) cudaEventRecord(tev[0], st);
    if (!(dbg & 64)) {
      if (direct)
        attn_bwd_split_kernel<0, 0, 2><<<grid, kBwdSThreads, BwdSCfg::kBytes, st>>>(
            mq, mk, mv, mdo, nlse2, delta, dq, dk, dv, ld_d, t.S, scale, t.push, t.rope_cos, t.rope_sin, dbg,
            g_attn_trace, w, h0);
      else
        attn_bwd_split_kernel<0, 0, 1><<<grid, kBwdSThreads, BwdSCfg::kBytesD, st>>>(
            mq, mk, mv, mdo, nlse2, delta, dq, dk, dv, ld_d, t.S, scale, t.push, t.rope_cos, t.rope_sin, dbg,
            g_attn_trace, w, h0);
    }
    if (timed && h0 == 0) cudaEventRecord(tev[1], st);
    if (!(dbg & 128)) {
      if (deep)
        attn_bwd_dq_kernel<5, 2><<<grid, kBwdDqThreads, BwdDqCfg<5, 2>::kBytes, st>>>(
            mk, w, dq, ld_d, t.S, scale, t.push, t.rope_cos, t.rope_sin, h0);
      else
        attn_bwd_dq_kernel<3, 3><<<grid, kBwdDqThreads, BwdDqCfg<3, 3>::kBytes, st>>>(
            mk, w, dq, ld_d, t.S, scale, t.push, t.rope_cos, t.rope_sin, h0);
    }
    if (timed && h0 == 0) cudaEventRecord(tev[2], st);
  }
  if (timed) {
    float a = 0, b = 0;
    cudaEventSynchronize(tev[2]);
    cudaEventElapsedTime(&a, tev[0], tev[1]);
    cudaEventElapsedTime(&b, tev[1], tev[2]);
    fprintf(stderr, "attn_bwd_ds: key-tile %.3f ms, dq %.3f ms (group of %d heads)\n", a, b, std::min(G, t.heads));
    for (auto& e : tev) cudaEventDestroy(e);
  }
  return cudaGetLastError();
}

// dq_acc must be zeroed and delta = rowsum(dO * O) computed before this launch.
cudaError_t attention_bwd_tc(const AttnTensors& t, const __nv_bfloat16* dout, int64_t ld_dout, __nv_bfloat16* dk,
                             __nv_bfloat16* dv, int64_t ld_d, const float* delta, float* dq_acc, cudaStream_t st) {
  if (t.d != 128 || t.S % kBwdKeys) return cudaErrorInvalidValue;
  using L = BwdSmem;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_bwd_tc_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kBytes);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(attn_bwd_tc_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kBytes);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  CUtensorMap mq, mk, mv, mdo;
  const int64_t cols = static_cast<int64_t>(t.heads) * 128;
  if (!map2d(&mq, t.q, t.S, cols, t.ld_qkv, kBwdQ) || !map2d(&mk, t.k, t.S, cols, t.ld_qkv, kBwdKeys) ||
      !map2d(&mv, t.v, t.S, cols, t.ld_qkv, kBwdKeys) || !map2d(&mdo, dout, t.S, cols, ld_dout, kBwdQ))
    return cudaErrorInvalidValue;
  const float scale = 1.0f / sqrtf(128.0f);
  const char* kt_env = std::getenv("SEQPLAN_ISP_BWD_KTMEM");
  // K resident in TMEM (kKT) measured no faster (634 vs 639 TF/s at 32K): opt-in only
  auto kern = (kt_env && std::atoi(kt_env) != 0) ? attn_bwd_tc_kernel<true, true> : attn_bwd_tc_kernel<true, false>;
  kern<<<lpt_grid(t.S / kBwdKeys, t.heads, t.S, 128), kBwdThreads, L::kBytes, st>>>(
      mq, mk, mv, mdo, t.lse, delta, dq_acc, dk, dv, ld_d, t.S, scale,
      std::getenv("SEQPLAN_ISP_DBG") ? std::atoi(std::getenv("SEQPLAN_ISP_DBG")) : 0, g_attn_trace, t.push, t.k,
      t.ld_qkv);
  return cudaGetLastError();
}

}  // namespace isp
