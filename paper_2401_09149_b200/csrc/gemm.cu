// tcgen05 / TMEM / TMA GEMM for the ISP block (sm_100a).
//
// C[M,N] = A[M,K] * B[N,K]^T with bf16 operands and fp32 accumulation in TMEM.
// Each operand may be K-major (row-major [rows, K]) or MN-major (stored as
// [K, rows]), so one kernel family covers the three GEMM shapes of a linear
// layer:
//   forward  y  = x  * W^T   A=x  (K-major)      B=W  (K-major)
//   dgrad    dx = dy * W     A=dy (K-major)      B=W  (MN-major)
//   wgrad    dW = dy^T * x   A=dy (MN-major)     B=x  (MN-major)
// The reference prices these as the "Linear" term of layer_forward_flops
// (proj/include/seqplan/cost.hpp:212-219); it has no kernel of its own.
//
// Structure: persistent, warp-specialised. warp 0 = TMA producer, warp 1 =
// tcgen05.mma issuer (one lane), warps 2..5 = epilogue (TMEM -> registers ->
// global). A 4..6 stage smem ring feeds the tensor core; the accumulator is
// double-buffered in TMEM so the epilogue of tile i overlaps the mainloop of
// tile i+1. Fused epilogues: plain bf16 store, residual add, SwiGLU (gate/up
// interleaved in 32-column blocks), fp32 store with scale/accumulate and
// optional gate/up de-interleave (used for weight gradients).
#include <cstdio>
#include <cstdlib>
#include <cudaTypedefs.h>

#include <algorithm>
#include <unordered_map>

#include "common.cuh"
#include "gemm.h"

namespace isp {

namespace {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kNumThreads = 192;  // 6 warps

template <int BN>
struct GemmCfg {
  static constexpr int kStages = BN == 256 ? 4 : 6;
  static constexpr int kABytes = BM * BK * 2;
  static constexpr int kBBytes = BN * BK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kTmemCols = 2 * BN;  // double-buffered accumulator
  static constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 512 /*barriers*/;
};

struct TileSched {
  int num_m, num_n, num_tiles, kGroupM = 16;
  __device__ __forceinline__ void coords(int t, int& m_blk, int& n_blk) const {
    // Group kGroupM row-blocks together so the ~148 concurrently resident
    // tiles share A rows and B columns in L2 (GemmArgs::group_m; 16 by default).
    const int per_group = kGroupM * num_n;
    const int g = t / per_group;
    const int first_m = g * kGroupM;
    const int gm = min(num_m - first_m, kGroupM);
    const int r = t - g * per_group;
    m_blk = first_m + r % gm;
    n_blk = r / gm;
  }
};

__device__ __forceinline__ float silu(float x) { return x / (1.0f + __expf(-x)); }

// 32 accumulator columns of this thread's row from TMEM, plus the fp32 partials other K-ranges
// of a split tile left in the workspace (np of them, `pstride` floats apart).
__device__ __forceinline__ void ld_acc(uint32_t taddr, uint32_t (&r)[32], const float* part, int64_t pstride,
                                       int np) {
  tmem_ld_32x32b_x32(taddr, r);
  tmem_ld_wait();
  for (int q = 0; q < np; ++q) {
    const float4* pp = reinterpret_cast<const float4*>(part + q * pstride);
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const float4 a = __ldcg(pp + v);
      r[4 * v] = __float_as_uint(__uint_as_float(r[4 * v]) + a.x);
      r[4 * v + 1] = __float_as_uint(__uint_as_float(r[4 * v + 1]) + a.y);
      r[4 * v + 2] = __float_as_uint(__uint_as_float(r[4 * v + 2]) + a.z);
      r[4 * v + 3] = __float_as_uint(__uint_as_float(r[4 * v + 3]) + a.w);
    }
  }
}

// TMEM accumulator tile (this thread's row, BN columns) -> global, fused epilogue. part/np: the
// fp32 partial rows of a split tile to add (part + col addresses column col of the row).
template <int BN, int EPI>
__device__ __forceinline__ void epilogue_tile(const GemmArgs& args, uint32_t t_base, int row, int n0,
                                              const float* part = nullptr, int64_t pstride = 0, int np = 0) {
  if constexpr (EPI == EPI_SWIGLU) {
    // kGuBlock(=32)-column blocks alternate gate / up: pair chunk 2j (gate) with 2j+1 (up).
#pragma unroll 1
    for (int pr = 0; pr < BN / 64; ++pr) {
      const int cg = pr * 64;  // gate column within tile
      uint32_t g[32], u[32];
      ld_acc(t_base + cg, g, part + cg, pstride, np);
      ld_acc(t_base + cg + kGuBlock, u, part + cg + kGuBlock, pstride, np);
      __nv_bfloat16* gu_row = reinterpret_cast<__nv_bfloat16*>(args.out) +
                              static_cast<int64_t>(row) * args.ldo + n0;
      __nv_bfloat16* a_row = args.out2 + static_cast<int64_t>(row) * args.ldo2 + (n0 / 2 + pr * 32);
      uint4* gdst = reinterpret_cast<uint4*>(gu_row + cg);
      uint4* udst = reinterpret_cast<uint4*>(gu_row + cg + kGuBlock);
      uint4* adst = reinterpret_cast<uint4*>(a_row);
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        uint32_t pg[4], pu[4], pa[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int i = v * 8 + e * 2;
          const float g0 = __uint_as_float(g[i]), g1 = __uint_as_float(g[i + 1]);
          const float u0 = __uint_as_float(u[i]), u1 = __uint_as_float(u[i + 1]);
          pg[e] = pack_bf16(g0, g1);
          pu[e] = pack_bf16(u0, u1);
          // activation from the bf16-rounded values the backward will see
          const float2 gr = unpack_bf16(pg[e]);
          const float2 ur = unpack_bf16(pu[e]);
          pa[e] = pack_bf16(silu(gr.x) * ur.x, silu(gr.y) * ur.y);
        }
        gdst[v] = make_uint4(pg[0], pg[1], pg[2], pg[3]);
        udst[v] = make_uint4(pu[0], pu[1], pu[2], pu[3]);
        adst[v] = make_uint4(pa[0], pa[1], pa[2], pa[3]);
      }
    }
  } else if constexpr (EPI == EPI_SWIGLU_BWD) {
    // SwiGLU backward fused into the down-projection dgrad: this 32-column chunk of da covers one
    // kGuBlock of I, i.e. gate columns [64 b, 64 b + 32) and up columns [64 b + 32, 64 b + 64) of gu
    // gu rows are read from HBM by one thread per row: the next chunk's 128 B are loaded while
    // this chunk is computed (8 x 16-B loads in flight per thread), or the epilogue, not the MMA,
    // bounds the tile
    const __nv_bfloat16* gu_row = args.resid + static_cast<int64_t>(row) * args.ldr;
    uint4 nxt[8];
    {
      const uint4* src = reinterpret_cast<const uint4*>(gu_row + static_cast<int64_t>(n0 / kGuBlock) * 2 * kGuBlock);
#pragma unroll
      for (int v = 0; v < 8; ++v) nxt[v] = __ldcs(src + v);
    }
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
      uint4 cur[8];
#pragma unroll
      for (int v = 0; v < 8; ++v) cur[v] = nxt[v];
      const int64_t gcol = static_cast<int64_t>((n0 + c * 32) / kGuBlock) * 2 * kGuBlock;
      if (c + 1 < BN / 32) {
        const uint4* src = reinterpret_cast<const uint4*>(gu_row + gcol + 2 * kGuBlock);
#pragma unroll
        for (int v = 0; v < 8; ++v) nxt[v] = __ldcs(src + v);
      }
      uint32_t r[32];
      ld_acc(t_base + c * 32, r, part + c * 32, pstride, np);
      uint4* gdst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(args.out) +
                                             static_cast<int64_t>(row) * args.ldo + gcol);
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const uint4 g4 = cur[v], u4 = cur[v + 4];
        const uint32_t gw[4] = {g4.x, g4.y, g4.z, g4.w}, uw[4] = {u4.x, u4.y, u4.z, u4.w};
        uint32_t pg[4], pu[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 g = unpack_bf16(gw[e]), u = unpack_bf16(uw[e]);
          // da rounded to bf16 exactly as the unfused path stored it
          const float2 da = unpack_bf16(pack_bf16(__uint_as_float(r[v * 8 + 2 * e]) * args.scale,
                                                  __uint_as_float(r[v * 8 + 2 * e + 1]) * args.scale));
          const float s0 = 1.f / (1.f + __expf(-g.x)), s1 = 1.f / (1.f + __expf(-g.y));
          pg[e] = pack_bf16(da.x * u.x * s0 * (1.f + g.x * (1.f - s0)), da.y * u.y * s1 * (1.f + g.y * (1.f - s1)));
          pu[e] = pack_bf16(da.x * g.x * s0, da.y * g.y * s1);
        }
        __stcs(gdst + v, make_uint4(pg[0], pg[1], pg[2], pg[3]));
        __stcs(gdst + v + 4, make_uint4(pu[0], pu[1], pu[2], pu[3]));
      }
    }
  } else if (EPI == EPI_BF16 && (args.push[0] != nullptr || args.rope_parts > 0)) {
    // head-aligned chunk pairs (i, i + d/2), RoPE on parts < rope_parts at position
    // push_rank * push_T + row; stored locally (out, token layout), or with push[] set pushed to
    // the rank owning the head (fused all-to-all)
    const int d = args.push_d, hd = d / 2;
    const int64_t pos = static_cast<int64_t>(args.push_rank) * args.push_T + row;
#pragma unroll 1
    for (int hb = 0; hb < BN; hb += d) {
#pragma unroll 1
      for (int c = 0; c < hd; c += 32) {
        uint32_t lo[32], hi[32];
        ld_acc(t_base + hb + c, lo, part + hb + c, pstride, np);
        ld_acc(t_base + hb + c + hd, hi, part + hb + c + hd, pstride, np);
        const int col = n0 + hb + c;  // output column of the low half (storage)
        const int lcol = args.rope_col0 + col;  // logical column in the [parts*H] row
        const int part = lcol / args.push_H, hcol = lcol - part * args.push_H;
        const int q = hcol / args.push_Hl, lc = hcol - q * args.push_Hl;
        float fl[32], fh[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          fl[i] = __uint_as_float(lo[i]) * args.scale;
          fh[i] = __uint_as_float(hi[i]) * args.scale;
        }
        if (part < args.rope_parts) {
          const float* cp = args.rope_cos + pos * hd + c;
          const float* sp = args.rope_sin + pos * hd + c;
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            const float4 cv = *reinterpret_cast<const float4*>(cp + i);
            const float4 sv = *reinterpret_cast<const float4*>(sp + i);
            const float cs[4] = {cv.x, cv.y, cv.z, cv.w}, sn[4] = {sv.x, sv.y, sv.z, sv.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float a = fl[i + e], b = fh[i + e];
              fl[i + e] = a * cs[e] - b * sn[e];
              fh[i + e] = b * cs[e] + a * sn[e];
            }
          }
        }
        __nv_bfloat16* dst = args.push[0] != nullptr
                                 ? static_cast<__nv_bfloat16*>(args.push[q]) + (pos * args.push_parts + part) * args.push_Hl + lc
                                 : reinterpret_cast<__nv_bfloat16*>(args.out) + static_cast<int64_t>(row) * args.ldo + col;
        uint4* d_lo = reinterpret_cast<uint4*>(dst);
        uint4* d_hi = reinterpret_cast<uint4*>(dst + hd);
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          uint32_t pl[4], ph[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            pl[e] = pack_bf16(fl[v * 8 + 2 * e], fl[v * 8 + 2 * e + 1]);
            ph[e] = pack_bf16(fh[v * 8 + 2 * e], fh[v * 8 + 2 * e + 1]);
          }
          d_lo[v] = make_uint4(pl[0], pl[1], pl[2], pl[3]);
          d_hi[v] = make_uint4(ph[0], ph[1], ph[2], ph[3]);
        }
      }
    }
  } else {
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
      uint32_t r[32];
      ld_acc(t_base + c * 32, r, part + c * 32, pstride, np);
      const int col = n0 + c * 32;
      if constexpr (EPI == EPI_F32) {
        float* dst;
        int64_t orow = row;
        if (args.interleave64) {  // gate|up rows interleaved in kGuBlock-row blocks
          const int blk = row / kGuBlock;
          orow = static_cast<int64_t>(blk >> 1) * kGuBlock + (row % kGuBlock);
          dst = (blk & 1) ? args.out_b : reinterpret_cast<float*>(args.out);
        } else {
          dst = reinterpret_cast<float*>(args.out);
        }
        float4* p = reinterpret_cast<float4*>(dst + orow * args.ldo + col);
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          float4 o = make_float4(__uint_as_float(r[4 * v]) * args.scale,
                                 __uint_as_float(r[4 * v + 1]) * args.scale,
                                 __uint_as_float(r[4 * v + 2]) * args.scale,
                                 __uint_as_float(r[4 * v + 3]) * args.scale);
          if (args.accumulate) {
            const float4 prev = p[v];
            o.x += prev.x; o.y += prev.y; o.z += prev.z; o.w += prev.w;
          }
          p[v] = o;
        }
      } else {
        __nv_bfloat16* dst_row = reinterpret_cast<__nv_bfloat16*>(args.out) +
                                 static_cast<int64_t>(row) * args.ldo + col;
        float add[32];
        if constexpr (EPI == EPI_BF16_RESID) {
          const uint4* rs = reinterpret_cast<const uint4*>(
              args.resid + static_cast<int64_t>(row) * args.ldr + col);
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const uint4 q = rs[v];
            const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 f = unpack_bf16(w[e]);
              add[v * 8 + e * 2] = f.x;
              add[v * 8 + e * 2 + 1] = f.y;
            }
          }
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) add[i] = 0.f;
        }
        uint4* d4 = reinterpret_cast<uint4*>(dst_row);
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          uint32_t pk[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int i = v * 8 + e * 2;
            pk[e] = pack_bf16(__uint_as_float(r[i]) * args.scale + add[i],
                              __uint_as_float(r[i + 1]) * args.scale + add[i + 1]);
          }
          d4[v] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        }
      }
    }
  }
}

template <bool A_MN, bool B_MN, int BN, int EPI>
__global__ void __launch_bounds__(kNumThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap mapA,
                   const __grid_constant__ CUtensorMap mapB, const __grid_constant__ GemmArgs args) {
  using Cfg = GemmCfg<BN>;
  constexpr int S = Cfg::kStages;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + S * Cfg::kStageBytes);
  uint64_t* empty_bar = full_bar + S;
  uint64_t* tfull_bar = empty_bar + S;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;

  TileSched sched{args.M / BM, args.N / BN, (args.M / BM) * (args.N / BN), args.group_m};
  const int num_kb = args.K / BK;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&mapA);
    tma_prefetch(&mapB);
    for (int i = 0; i < S; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull_bar[i], 1);
      mbar_init(&tempty_bar[i], 128);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int t = blockIdx.x; t < sched.num_tiles; t += gridDim.x) {
        int mb, nb;
        sched.coords(t, mb, nb);
        const int m0 = mb * BM, n0 = nb * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&empty_bar[s], ph ^ 1);
          uint8_t* sa = smem + s * Cfg::kStageBytes;
          uint8_t* sb = sa + Cfg::kABytes;
          mbar_arrive_expect_tx(&full_bar[s], Cfg::kStageBytes);
          if constexpr (!A_MN) {
            tma_load_2d(sa, &mapA, &full_bar[s], kb * BK, m0);
          } else {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j)
              tma_load_2d(sa + j * 8192, &mapA, &full_bar[s], m0 + j * 64, kb * BK);
          }
          if constexpr (!B_MN) {
            tma_load_2d(sb, &mapB, &full_bar[s], kb * BK, n0);
          } else {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j)
              tma_load_2d(sb + j * 8192, &mapB, &full_bar[s], n0 + j * 64, kb * BK);
          }
          if (++s == S) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    constexpr uint32_t idesc = make_idesc_bf16(BM, BN, A_MN, B_MN);
    int s = 0;
    uint32_t ph = 0;
    int acc = 0;
    uint32_t acc_ph = 0;
    for (int t = blockIdx.x; t < sched.num_tiles; t += gridDim.x) {
      mbar_wait(&tempty_bar[acc], acc_ph ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int kb = 0; kb < num_kb; ++kb) {
        mbar_wait(&full_bar[s], ph);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t sa = smem_u32(smem + s * Cfg::kStageBytes);
          const uint32_t sb = sa + Cfg::kABytes;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = A_MN ? make_sw128_desc(sa + k * 2048, 8192, 1024)
                                     : make_sw128_desc(sa + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? make_sw128_desc(sb + k * 2048, 8192, 1024)
                                     : make_sw128_desc(sb + k * 32, 16, 1024);
            tc_mma_bf16(d_tmem, ad, bd, idesc, (kb | k) != 0 ? 1u : 0u);
          }
          tc_commit(&empty_bar[s]);
        }
        __syncwarp();
        if (++s == S) { s = 0; ph ^= 1; }
      }
      if (lane == 0) tc_commit(&tfull_bar[acc]);
      __syncwarp();
      if (++acc == 2) { acc = 0; acc_ph ^= 1; }
    }
  } else {
    // ---------------- epilogue (warps 2..5) ----------------
    const int lane_grp = warp & 3;  // TMEM lane quadrant this warp may access
    int acc = 0;
    uint32_t acc_ph = 0;
    for (int t = blockIdx.x; t < sched.num_tiles; t += gridDim.x) {
      int mb, nb;
      sched.coords(t, mb, nb);
      const int row = mb * BM + lane_grp * 32 + lane;
      const int n0 = nb * BN;
      mbar_wait(&tfull_bar[acc], acc_ph);
      tc_fence_after();
      const uint32_t t_base = tmem_base + (static_cast<uint32_t>(lane_grp * 32) << 16) + acc * BN;

      epilogue_tile<BN, EPI>(args, t_base, row, n0);
      tc_fence_before();
      mbar_arrive(&tempty_bar[acc]);
      if (++acc == 2) { acc = 0; acc_ph ^= 1; }
    }
    // remote (NVLink) stores of the fused all-to-all must be performed before the stream's
    // next barrier flag can be observed by the peer
    if (args.push[0]) __threadfence_system();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<Cfg::kTmemCols>(tmem_base);
  }
}

// ---------------------------------------------------------------------------
// CTA-pair variant (tcgen05.mma.cta_group::2): a cluster of 2 CTAs computes a 256 x BN tile.
// CTA r loads A rows [m0 + 128 r, +128) and B rows [n0 + BN/2 r, +BN/2) into its own smem
// (TMA completes on the leader's barrier); the leader issues M=256 MMAs that read both CTAs'
// smem and accumulate into each CTA's own TMEM (128 lanes x BN). Per-SM smem traffic per MMA
// halves vs the single-CTA kernel, which is what lets the tensor pipe run near peak.
// ---------------------------------------------------------------------------
// BN = 256 (production) or 128 (SEQPLAN_GEMM_PAIR_BN=128, development; see gemm_launch).
template <int BN>
struct PairCfg {
  static constexpr int BNH = BN / 2, S = BN == 256 ? 6 : 8;
  static constexpr int kSmem = S * (BM * BK * 2 + BNH * BK * 2) + 1024 + 512;
};

template <bool A_MN, bool B_MN, int EPI, int BN>
__global__ void __launch_bounds__(kNumThreads, 1)
    gemm_tc2_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                    const __grid_constant__ GemmArgs args) {
  constexpr int BNH = PairCfg<BN>::BNH, S = PairCfg<BN>::S;
  constexpr int kABytes = BM * BK * 2, kBBytes = BNH * BK * 2, kStageBytes = kABytes + kBBytes;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + S * kStageBytes);
  uint64_t* empty_bar = full_bar + S;
  uint64_t* tfull_bar = empty_bar + S;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t crank = cluster_rank();
  const bool leader = crank == 0;
  const int cid = blockIdx.x / 2, ncl = gridDim.x / 2;
  TileSched sched{args.M / (2 * BM), args.N / BN, (args.M / (2 * BM)) * (args.N / BN), args.group_m};
  const int num_kb = args.K / BK;
  // work units: split_base whole tiles, then split_L tiles x split_s K-ranges (the last wave)
  const int n_units = args.split_L > 0 ? args.split_base + args.split_L * args.split_s : sched.num_tiles;
  auto unit = [&](int u, int& tile, int& kb0, int& kb1, int& j, int& p) {
    if (u < args.split_base || args.split_L == 0) {
      tile = u; kb0 = 0; kb1 = num_kb; j = -1; p = 0;
    } else {
      const int v = u - args.split_base;
      j = v / args.split_s; p = v % args.split_s;
      tile = args.split_base + j;
      kb0 = num_kb * p / args.split_s;
      kb1 = num_kb * (p + 1) / args.split_s;
    }
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch(&mapA);
    tma_prefetch(&mapB);
    for (int i = 0; i < S; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull_bar[i], 1);
      mbar_init(&tempty_bar[i], 2 * 128);  // both CTAs' epilogue threads (leader's copy is used)
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int u = cid; u < n_units; u += ncl) {
        int t, kb0, kb1, j, p;
        unit(u, t, kb0, kb1, j, p);
        int mb, nb;
        sched.coords(t, mb, nb);
        const int m0 = mb * 2 * BM + static_cast<int>(crank) * BM, n0 = nb * BN + static_cast<int>(crank) * BNH;
        const int wave = (u - cid) / ncl;
        if (args.wave_cnt && wave > 0) {  // every cluster has issued wave - 1
          const uint32_t want = static_cast<uint32_t>(min(ncl, n_units - (wave - 1) * ncl));
          uint32_t got;
          do {
            asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(got) : "l"(args.wave_cnt + wave - 1) : "memory");
          } while (got < want && (__nanosleep(64), true));
        }
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty_bar[s], ph ^ 1);
          uint8_t* sa = smem + s * kStageBytes;
          uint8_t* sb = sa + kABytes;
          if (leader) mbar_arrive_expect_tx(&full_bar[s], 2 * kStageBytes);
          if constexpr (!A_MN) {
            tma_load_2d_pair(sa, &mapA, &full_bar[s], kb * BK, m0);
          } else {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j) tma_load_2d_pair(sa + j * 8192, &mapA, &full_bar[s], m0 + j * 64, kb * BK);
          }
          if constexpr (!B_MN) {
            tma_load_2d_pair(sb, &mapB, &full_bar[s], kb * BK, n0);
          } else {
#pragma unroll
            for (int j = 0; j < BNH / 64; ++j) tma_load_2d_pair(sb + j * 8192, &mapB, &full_bar[s], n0 + j * 64, kb * BK);
          }
          if (++s == S) { s = 0; ph ^= 1; }
        }
        if (args.wave_cnt && leader) atomicAdd(args.wave_cnt + wave, 1u);
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      constexpr uint32_t idesc = make_idesc_bf16(2 * BM, BN, A_MN, B_MN);
      int s = 0;
      uint32_t ph = 0;
      int acc = 0;
      uint32_t acc_ph = 0;
      for (int u = cid; u < n_units; u += ncl) {
        int t, kb0, kb1, j, p;
        unit(u, t, kb0, kb1, j, p);
        mbar_wait(&tempty_bar[acc], acc_ph ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full_bar[s], ph);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + s * kStageBytes);
          const uint32_t sb = sa + kABytes;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = A_MN ? make_sw128_desc(sa + k * 2048, 8192, 1024) : make_sw128_desc(sa + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? make_sw128_desc(sb + k * 2048, 8192, 1024) : make_sw128_desc(sb + k * 32, 16, 1024);
            tc_mma_bf16_pair(d_tmem, ad, bd, idesc, (kb != kb0 || k != 0) ? 1u : 0u);
          }
          tc_commit_pair(&empty_bar[s]);
          if (++s == S) { s = 0; ph ^= 1; }
        }
        tc_commit_pair(&tfull_bar[acc]);
        if (++acc == 2) { acc = 0; acc_ph ^= 1; }
      }
    }
  } else {
    const int lane_grp = warp & 3;
    int acc = 0;
    uint32_t acc_ph = 0;
    __shared__ uint32_t split_order;
    const int lrow = lane_grp * 32 + lane;  // this thread's row within the CTA's 128
    for (int u = cid; u < n_units; u += ncl) {
      int t, kb0, kb1, j, p;
      unit(u, t, kb0, kb1, j, p);
      int mb, nb;
      sched.coords(t, mb, nb);
      const int row = mb * 2 * BM + static_cast<int>(crank) * BM + lrow;
      const int n0 = nb * BN;
      mbar_wait(&tfull_bar[acc], acc_ph);
      tc_fence_after();
      const uint32_t t_base = tmem_base + (static_cast<uint32_t>(lane_grp * 32) << 16) + acc * BN;
      if (j < 0) {
        epilogue_tile<BN, EPI>(args, t_base, row, n0);
      } else {
        // split tile: arrival order decides who finishes it (no unit ever waits for one that has
        // not arrived, so the partial wave cannot deadlock on unscheduled clusters)
        const int sm1 = args.split_s - 1;
        const int64_t slot_f = int64_t(2) * 128 * BN;  // floats per (slot, both CTAs)
        uint32_t* cnt = args.split_cnt + j * 2 + crank;
        uint32_t* rdy = args.split_ready + (int64_t(j) * sm1) * 2 + crank;
        float* ws = args.split_ws + (int64_t(j) * sm1) * slot_f + (int64_t(crank) * 128 + lrow) * BN;
        if (threadIdx.x == 64) split_order = atomicAdd(cnt, 1u);
        asm volatile("bar.sync 1, 128;" ::: "memory");
        const uint32_t order = split_order;
        if (static_cast<int>(order) < sm1) {  // not last: leave the fp32 partial in slot `order`
          float* dst = ws + int64_t(order) * slot_f;
#pragma unroll 1
          for (int c = 0; c < BN / 32; ++c) {
            uint32_t r[32];
            tmem_ld_32x32b_x32(t_base + c * 32, r);
            tmem_ld_wait();
            float4* d4 = reinterpret_cast<float4*>(dst + c * 32);
#pragma unroll
            for (int v = 0; v < 8; ++v)
              __stcg(d4 + v, make_float4(__uint_as_float(r[4 * v]), __uint_as_float(r[4 * v + 1]),
                                         __uint_as_float(r[4 * v + 2]), __uint_as_float(r[4 * v + 3])));
          }
          __threadfence();
          asm volatile("bar.sync 1, 128;" ::: "memory");
          if (threadIdx.x == 64) st_release_sys(rdy + int64_t(order) * 2, 1u);
        } else {  // last: wait for the others' partials, reset the flags, fused epilogue on the sum
          if (threadIdx.x == 64) {
            for (int q = 0; q < sm1; ++q)
              while (ld_acquire_sys(rdy + int64_t(q) * 2) == 0u) {
              }
            for (int q = 0; q < sm1; ++q) rdy[int64_t(q) * 2] = 0u;
            *cnt = 0u;
            __threadfence();
          }
          asm volatile("bar.sync 1, 128;" ::: "memory");
          epilogue_tile<BN, EPI>(args, t_base, row, n0, ws, slot_f, sm1);
        }
      }
      tc_fence_before();
      if (leader) mbar_arrive(&tempty_bar[acc]);
      else mbar_arrive_leader(&tempty_bar[acc]);
      if (++acc == 2) { acc = 0; acc_ph ^= 1; }
    }
    if (args.push[0]) __threadfence_system();  // remote stores visible before the next barrier flag
  }

  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2-D bf16 map over a row-major [rows, cols] matrix with leading dimension ld
// (elements), 128-byte swizzle, box = {64 cols, box_rows}.
bool make_map(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int64_t ld,
              int box_rows) {
  auto fn = get_encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 2)};
  cuuint32_t box[2] = {64u, static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int g_num_sms = 0;

template <bool A_MN, bool B_MN, int BN, int EPI>
cudaError_t launch_t(const CUtensorMap& ma, const CUtensorMap& mb, const GemmArgs& args,
                     cudaStream_t stream) {
  using Cfg = GemmCfg<BN>;
  auto kern = gemm_tc_kernel<A_MN, B_MN, BN, EPI>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int tiles = (args.M / BM) * (args.N / BN);
  const int sms = args.sm_budget > 0 && args.sm_budget < g_num_sms ? args.sm_budget : g_num_sms;
  const int grid = tiles < sms ? tiles : sms;
  kern<<<grid, kNumThreads, Cfg::kSmemBytes, stream>>>(ma, mb, args);
  return cudaGetLastError();
}

// Split-K of the last partial wave. With `tiles` = w * clusters + L (0 < L <= clusters / 2), the
// L trailing tiles would leave most CTA pairs idle for a whole tile time; cut each into
// s = min(4, clusters / L) K-ranges instead (>= 8 K-blocks each), so the last wave takes ~1/s
// of a tile time. 4096 x 4096 outputs: 256 tiles = 3 waves + 34 -> 3 + 1/2 waves.
// Workspace (fp32 partials, arrival counters, ready flags) per stream, allocated once.
struct SplitWs {
  float* ws = nullptr;
  uint32_t* flags = nullptr;
};
void split_last_wave(GemmArgs& a, int tiles, int clusters, int num_kb, cudaStream_t st) {
  a.split_base = 0; a.split_L = 0; a.split_s = 1;
  // opt-in (SEQPLAN_GEMM_SPLIT=1): measured neutral on the 7B block (4.327 vs 4.327 ms/step at
  // S = 4K; per GEMM -6 % .. +3.5 %): the partial last wave runs faster per tile than a full one
  // (fewer clusters share L2 bandwidth), so the idle-slot loss is smaller than the tile count says
  const char* on = std::getenv("SEQPLAN_GEMM_SPLIT");
  if (!on || std::atoi(on) == 0 || tiles <= clusters) return;
  const int L = tiles % clusters;
  if (L == 0 || 2 * L > clusters) return;
  int sp = std::min(4, clusters / L);
  while (sp > 1 && num_kb / sp < 8) --sp;
  if (sp < 2) return;
  constexpr int kMaxSlots = 74;                 // L * (s - 1) <= clusters - L < 74
  constexpr size_t kSlotBytes = 2 * 128 * 256 * 4;  // one (tile, K-range) partial, both CTAs
  static std::unordered_map<cudaStream_t, SplitWs> per_stream;
  SplitWs& w = per_stream[st];
  if (!w.ws) {
    if (cudaMalloc(&w.ws, kMaxSlots * kSlotBytes) != cudaSuccess) { w.ws = nullptr; return; }
    if (cudaMalloc(&w.flags, 4 * 1024 * sizeof(uint32_t)) != cudaSuccess) { cudaFree(w.ws); w.ws = nullptr; return; }
    cudaMemsetAsync(w.flags, 0, 4 * 1024 * sizeof(uint32_t), st);
  }
  if (L * (sp - 1) > kMaxSlots) return;
  a.split_base = tiles - L;
  a.split_L = L;
  a.split_s = sp;
  a.split_ws = w.ws;
  a.split_cnt = w.flags;            // [L][2]
  a.split_ready = w.flags + 2048;   // [L][s-1][2]
}

template <bool A_MN, bool B_MN, int EPI, int BN>
cudaError_t launch_pair(const CUtensorMap& ma, const CUtensorMap& mb, const GemmArgs& args, cudaStream_t stream) {
  constexpr int kSmem = PairCfg<BN>::kSmem;
  auto kern = gemm_tc2_kernel<A_MN, B_MN, EPI, BN>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int tiles = (args.M / 256) * (args.N / BN);
  const int sms = args.sm_budget > 0 && args.sm_budget < g_num_sms ? args.sm_budget : g_num_sms;
  const int clusters = tiles < sms / 2 ? tiles : sms / 2;
  GemmArgs a2 = args;
  split_last_wave(a2, tiles, clusters, args.K / BK, stream);
  static const bool wave_sync_env = [] {
    const char* e = std::getenv("SEQPLAN_GEMM_WAVE_SYNC");
    return !e || std::atoi(e) != 0;
  }();
  a2.wave_cnt = nullptr;
  if (wave_sync_env && args.wave_sync && tiles > clusters) {
    static std::unordered_map<cudaStream_t, uint32_t*> per_stream;
    uint32_t*& w = per_stream[stream];
    if (!w && cudaMalloc(&w, 4096 * sizeof(uint32_t)) != cudaSuccess) w = nullptr;
    const int units = a2.split_L > 0 ? a2.split_base + a2.split_L * a2.split_s : tiles;
    if (w && units / clusters + 1 <= 4096) {
      cudaMemsetAsync(w, 0, size_t(units / clusters + 1) * sizeof(uint32_t), stream);
      a2.wave_cnt = w;
    }
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * clusters);
  cfg.blockDim = dim3(kNumThreads);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, ma, mb, a2);
}

template <bool A_MN, bool B_MN, int BN>
cudaError_t dispatch_pair(const CUtensorMap& ma, const CUtensorMap& mb, const GemmArgs& a, int epi, cudaStream_t st) {
  switch (epi) {
    case EPI_BF16: return launch_pair<A_MN, B_MN, EPI_BF16, BN>(ma, mb, a, st);
    case EPI_BF16_RESID: return launch_pair<A_MN, B_MN, EPI_BF16_RESID, BN>(ma, mb, a, st);
    case EPI_SWIGLU: return launch_pair<A_MN, B_MN, EPI_SWIGLU, BN>(ma, mb, a, st);
    case EPI_F32: return launch_pair<A_MN, B_MN, EPI_F32, BN>(ma, mb, a, st);
    case EPI_SWIGLU_BWD: return launch_pair<A_MN, B_MN, EPI_SWIGLU_BWD, BN>(ma, mb, a, st);
  }
  return cudaErrorInvalidValue;
}


template <bool A_MN, bool B_MN, int BN>
cudaError_t dispatch_epi(const CUtensorMap& ma, const CUtensorMap& mb, const GemmArgs& a,
                         int epi, cudaStream_t st) {
  switch (epi) {
    case EPI_BF16: return launch_t<A_MN, B_MN, BN, EPI_BF16>(ma, mb, a, st);
    case EPI_BF16_RESID: return launch_t<A_MN, B_MN, BN, EPI_BF16_RESID>(ma, mb, a, st);
    case EPI_SWIGLU: return launch_t<A_MN, B_MN, BN, EPI_SWIGLU>(ma, mb, a, st);
    case EPI_F32: return launch_t<A_MN, B_MN, BN, EPI_F32>(ma, mb, a, st);
    case EPI_SWIGLU_BWD: return launch_t<A_MN, B_MN, BN, EPI_SWIGLU_BWD>(ma, mb, a, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

int gemm_pick_bn(int N) { return (N % 256 == 0) ? 256 : ((N % 128 == 0) ? 128 : 0); }

cudaError_t gemm_launch(const GemmOperand& A, const GemmOperand& B, GemmArgs args, int epi,
                        cudaStream_t stream) {
  if (args.M % BM || args.K % BK || args.M <= 0 || args.N <= 0 || args.K <= 0)
    return cudaErrorInvalidValue;
  if (const char* f = std::getenv("SEQPLAN_GEMM_GROUP_M")) args.group_m = std::max(1, std::atoi(f));  // development
  int bn = gemm_pick_bn(args.N);
  if (const char* f = std::getenv("SEQPLAN_GEMM_BN")) {  // development override
    const int want = std::atoi(f);
    if ((want == 128 || want == 256) && args.N % want == 0) bn = want;
  }
  if (epi == EPI_SWIGLU) bn = (args.N % 256 == 0) ? 256 : (args.N % 128 == 0 ? 128 : 0);
  if (bn == 0) return cudaErrorInvalidValue;
  if ((args.push[0] || args.rope_parts > 0) &&
      (epi != EPI_BF16 || bn % args.push_d || args.push_H % 32 || args.push_Hl % 32))
    return cudaErrorInvalidValue;
  const bool pair = bn == 256 && args.M % 256 == 0 && !std::getenv("SEQPLAN_GEMM_NO_PAIR");
  // pair tile width: 256 x 256. 256 x 128 tiles (SEQPLAN_GEMM_PAIR_BN=128, development) fill the
  // last wave better (4096 x 4096: 512 tiles = 6.9 waves of 74 pairs instead of 3.46) but
  // measured ~30 % slower per FLOP on B200 (1000-1070 vs 1410-1550 TF/s, 7B shapes): twice the
  // operand bytes per MMA cycle, which L2 cannot feed to all 148 SMs.
  int pbn = 256;
  if (pair) {
    if (const char* f = std::getenv("SEQPLAN_GEMM_PAIR_BN")) pbn = std::atoi(f) == 128 ? 128 : 256;
    if ((args.push[0] || args.rope_parts > 0) && pbn % args.push_d) pbn = 256;
  }
  CUtensorMap ma, mb;
  // A: logical [M, K]; K-major storage is [M, K], MN-major storage is [K, M].
  bool ok = A.mn_major ? make_map(&ma, A.ptr, args.K, args.M, A.ld, 64)
                       : make_map(&ma, A.ptr, args.M, args.K, A.ld, BM);
  ok = ok && (B.mn_major ? make_map(&mb, B.ptr, args.K, args.N, B.ld, 64)
                         : make_map(&mb, B.ptr, args.N, args.K, B.ld, pair ? pbn / 2 : bn));
  if (!ok) return cudaErrorInvalidValue;
  const int code = (A.mn_major ? 2 : 0) | (B.mn_major ? 1 : 0);
  if (pair && pbn == 128) {
    switch (code) {
      case 0: return dispatch_pair<false, false, 128>(ma, mb, args, epi, stream);
      case 1: return dispatch_pair<false, true, 128>(ma, mb, args, epi, stream);
      case 2: return dispatch_pair<true, false, 128>(ma, mb, args, epi, stream);
      case 3: return dispatch_pair<true, true, 128>(ma, mb, args, epi, stream);
    }
  }
  if (pair) {
    switch (code) {
      case 0: return dispatch_pair<false, false, 256>(ma, mb, args, epi, stream);
      case 1: return dispatch_pair<false, true, 256>(ma, mb, args, epi, stream);
      case 2: return dispatch_pair<true, false, 256>(ma, mb, args, epi, stream);
      case 3: return dispatch_pair<true, true, 256>(ma, mb, args, epi, stream);
    }
  }
  if (bn == 256) {
    switch (code) {
      case 0: return dispatch_epi<false, false, 256>(ma, mb, args, epi, stream);
      case 1: return dispatch_epi<false, true, 256>(ma, mb, args, epi, stream);
      case 2: return dispatch_epi<true, false, 256>(ma, mb, args, epi, stream);
      case 3: return dispatch_epi<true, true, 256>(ma, mb, args, epi, stream);
    }
  } else {
    switch (code) {
      case 0: return dispatch_epi<false, false, 128>(ma, mb, args, epi, stream);
      case 1: return dispatch_epi<false, true, 128>(ma, mb, args, epi, stream);
      case 2: return dispatch_epi<true, false, 128>(ma, mb, args, epi, stream);
      case 3: return dispatch_epi<true, true, 128>(ma, mb, args, epi, stream);
    }
  }
  return cudaErrorInvalidValue;
}

}  // namespace isp
