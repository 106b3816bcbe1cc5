// Peer-memory collectives of the ISP block over NVLink / NVSwitch (sm_100a).
//
// Every rank owns a symmetric heap; peers' heaps are mapped into this process
// (CUDA IPC in multi-process mode, plain device pointers in single-process
// group mode), so collectives are ordinary kernels issuing 16-byte loads to
// peer addresses — no NCCL on the data path. They are the executor-side
// counterparts of the prices in proj/include/seqplan/cost.hpp:
//   parameter all-gather (ps)            cost.hpp:184-188 (2n x AG of e*Psi/tp)
//   gradient reduce-scatter (ps)         cost.hpp:187     (n x RS), fused with cast/scale
//   Ulysses all-to-all (sp)              cost.hpp:179-183 (QKV and attention output)
// All are "pull" kernels: rank r reads what it needs from every peer, so each
// byte crosses NVLink exactly once and no remote writes need ordering. A small
// system-scope flag barrier separates producer and consumer phases.
#include <cuda_bf16.h>

#include <cstdlib>

#include "common.cuh"
#include "gemm.h"
#include "kernels.h"

namespace isp {

namespace {

__device__ __forceinline__ uint4 ld_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// dst[q*shard + i] = src_q[i]; 16-byte vectors, 4 in flight per thread.
__global__ void allgather_pull_kernel(PeerPtrs src, int world, int64_t shard_vec, uint4* dst) {
  const int64_t total = shard_vec * world;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  for (; i + 3 * stride < total; i += 4 * stride) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t j = i + u * stride;
      const int q = static_cast<int>(j / shard_vec);
      v[u] = ld_v4(static_cast<const uint4*>(src.p[q]) + (j - q * shard_vec));
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) dst[i + u * stride] = v[u];
  }
  for (; i < total; i += stride) {
    const int q = static_cast<int>(i / shard_vec);
    dst[i] = ld_v4(static_cast<const uint4*>(src.p[q]) + (i - q * shard_vec));
  }
}

// gate|up gathered into one [2*rows, cols] buffer interleaved in kGuBlock-row blocks.
__global__ void allgather_interleave_kernel(PeerPtrs sg, PeerPtrs su, int world, int64_t rows,
                                            int64_t cols, uint4* dst) {
  const int64_t cvec = cols / 8;
  const int64_t total = 2 * rows * cvec;
  const int64_t rows_per_rank = rows / world;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t drow = i / cvec, c = i % cvec;
    const int64_t blk = drow / kGuBlock, within = drow % kGuBlock;
    const bool up = blk & 1;
    const int64_t srow = (blk >> 1) * kGuBlock + within;
    const int q = static_cast<int>(srow / rows_per_rank);
    const int64_t off = (srow - q * rows_per_rank) * cvec + c;
    const uint4* s = static_cast<const uint4*>(up ? su.p[q] : sg.p[q]);
    dst[i] = ld_v4(s + off);
  }
}

__device__ __forceinline__ void add8(float (&acc)[8], const uint4& v) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 f = unpack_bf16(w[e]);
    acc[2 * e] += f.x;
    acc[2 * e + 1] += f.y;
  }
}

// out[i] (+)= scale * sum_q part_q[base + i]; 8 elements per thread, fixed rank order.
template <bool F32>
__global__ void reduce_scatter_kernel(PeerPtrs part, int world, int64_t base, int64_t n8,
                                      float scale, int accumulate, float* __restrict__ out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n8;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int q = 0; q < world; ++q) {
      if constexpr (F32) {
        const float* p = static_cast<const float*>(part.p[q]) + base + i * 8;
        const uint4 a = ld_v4(p), b = ld_v4(p + 4);
        acc[0] += __uint_as_float(a.x); acc[1] += __uint_as_float(a.y);
        acc[2] += __uint_as_float(a.z); acc[3] += __uint_as_float(a.w);
        acc[4] += __uint_as_float(b.x); acc[5] += __uint_as_float(b.y);
        acc[6] += __uint_as_float(b.z); acc[7] += __uint_as_float(b.w);
      } else {
        add8(acc, ld_v4(static_cast<const __nv_bfloat16*>(part.p[q]) + base + i * 8));
      }
    }
    float4* o = reinterpret_cast<float4*>(out + i * 8);
    float4 r0 = make_float4(acc[0] * scale, acc[1] * scale, acc[2] * scale, acc[3] * scale);
    float4 r1 = make_float4(acc[4] * scale, acc[5] * scale, acc[6] * scale, acc[7] * scale);
    if (accumulate) {
      const float4 p0 = o[0], p1 = o[1];
      r0.x += p0.x; r0.y += p0.y; r0.z += p0.z; r0.w += p0.w;
      r1.x += p1.x; r1.y += p1.y; r1.z += p1.z; r1.w += p1.w;
    }
    o[0] = r0;
    o[1] = r1;
  }
}

// gate/up shards of rank `rank` from interleaved bf16 partials [2*rows, cols].
__global__ void reduce_scatter_interleave_kernel(PeerPtrs part, int world, int rank, int64_t rows,
                                                 int64_t cols, float scale, int accumulate,
                                                 float* __restrict__ og, float* __restrict__ ou) {
  const int64_t rpr = rows / world;
  const int64_t c8 = cols / 8;
  const int64_t total = 2 * rpr * c8;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const bool up = i >= rpr * c8;
    const int64_t li = up ? i - rpr * c8 : i;
    const int64_t lrow = li / c8, c = li % c8;
    const int64_t srow = rank * rpr + lrow;
    const int64_t irow = (srow / kGuBlock) * 2 * kGuBlock + (up ? kGuBlock : 0) + srow % kGuBlock;
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int q = 0; q < world; ++q)
      add8(acc, ld_v4(static_cast<const __nv_bfloat16*>(part.p[q]) + irow * cols + c * 8));
    float* dst = (up ? ou : og) + lrow * cols + c * 8;
    float4* o = reinterpret_cast<float4*>(dst);
    float4 r0 = make_float4(acc[0] * scale, acc[1] * scale, acc[2] * scale, acc[3] * scale);
    float4 r1 = make_float4(acc[4] * scale, acc[5] * scale, acc[6] * scale, acc[7] * scale);
    if (accumulate) {
      const float4 p0 = o[0], p1 = o[1];
      r0.x += p0.x; r0.y += p0.y; r0.z += p0.z; r0.w += p0.w;
      r1.x += p1.x; r1.y += p1.y; r1.z += p1.z; r1.w += p1.w;
    }
    o[0] = r0;
    o[1] = r1;
  }
}

// NVLink SHARP reduce-scatter of a bf16 weight-gradient partial: `mc` is the partial at its
// multicast address (every rank's copy bound at the same offset), so one 16-B multimem.ld_reduce
// returns the sum over all ranks of 8 elements, accumulated in fp32 inside the NVSwitch (and
// rounded to bf16); this rank reads only its own shard. rows > 0: the gate|up 64-row interleave
// (as reduce_scatter_interleave_kernel); the fp32 shard gets scale * sum (or += with accumulate).
__global__ void nvls_reduce_kernel(const __nv_bfloat16* __restrict__ mc, int world, int rank, int64_t shard8,
                                   int64_t rows, int64_t cols, float scale, int accumulate,
                                   float* __restrict__ og, float* __restrict__ ou) {
  const int64_t rpr = rows / world, c8 = cols / 8;
  const int64_t total = rows > 0 ? 2 * rpr * c8 : shard8;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const __nv_bfloat16* src;
    float* dst;
    if (rows > 0) {
      const bool up = i >= rpr * c8;
      const int64_t li = up ? i - rpr * c8 : i;
      const int64_t lrow = li / c8, c = li % c8;
      const int64_t srow = rank * rpr + lrow;
      const int64_t irow = (srow / kGuBlock) * 2 * kGuBlock + (up ? kGuBlock : 0) + srow % kGuBlock;
      src = mc + irow * cols + c * 8;
      dst = (up ? ou : og) + lrow * cols + c * 8;
    } else {
      src = mc + (rank * shard8 + i) * 8;
      dst = og + i * 8;
    }
    uint32_t w[4];
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0, %1, %2, %3}, [%4];"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3])
                 : "l"(src)
                 : "memory");
    float acc[8];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[e]));
      acc[2 * e] = f.x * scale;
      acc[2 * e + 1] = f.y * scale;
    }
    float4* o = reinterpret_cast<float4*>(dst);
    float4 r0 = make_float4(acc[0], acc[1], acc[2], acc[3]), r1 = make_float4(acc[4], acc[5], acc[6], acc[7]);
    if (accumulate) {
      const float4 p0 = o[0], p1 = o[1];
      r0.x += p0.x; r0.y += p0.y; r0.z += p0.z; r0.w += p0.w;
      r1.x += p1.x; r1.y += p1.y; r1.z += p1.z; r1.w += p1.w;
    }
    o[0] = r0;
    o[1] = r1;
  }
}

__device__ __forceinline__ void rotate8(uint4& lo, uint4& hi, const float* c, const float* s,
                                        float sign) {
  uint32_t* a = reinterpret_cast<uint32_t*>(&lo);
  uint32_t* b = reinterpret_cast<uint32_t*>(&hi);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 x = unpack_bf16(a[e]), y = unpack_bf16(b[e]);
    const float c0 = c[2 * e], c1 = c[2 * e + 1];
    const float s0 = sign * s[2 * e], s1 = sign * s[2 * e + 1];
    a[e] = pack_bf16(x.x * c0 - y.x * s0, x.y * c1 - y.y * s1);
    b[e] = pack_bf16(y.x * c0 + x.x * s0, y.y * c1 + x.y * s1);
  }
}

// Token-sharded [T, parts*H] on every rank -> head-sharded [S, parts*Hl] on this rank.
// Work unit: (global token s, part, local head, 8-element group j of the low half); optional
// RoPE on parts < rope_parts at global position s. 32-bit index math (units < 2^31).
template <int kU>
__global__ void __launch_bounds__(256) a2a_to_heads_kernel(PeerPtrs src, int world, int rank, int T, int H,
                                                           int parts, int d, __nv_bfloat16* __restrict__ dst,
                                                           const float* __restrict__ cos_t,
                                                           const float* __restrict__ sin_t, int rope_parts) {
  const int Hl = H / world, heads_l = Hl / d, half = d / 2, g8 = half / 8;
  const int per_part = heads_l * g8;
  const int per_row = parts * per_part;
  const int total = T * world * per_row;
  const int stride = gridDim.x * blockDim.x;
  // kU units per thread per round, all 2*kU remote loads issued before any store (NVLink latency
  // needs bytes in flight; one unit at a time leaves the exchange latency-bound)
  for (int i0 = blockIdx.x * blockDim.x + threadIdx.x; i0 < total; i0 += kU * stride) {
    uint4 lo[kU], hi[kU];
    __nv_bfloat16* dp[kU];
    int spos[kU], part_u[kU], j_u[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int i = i0 + u * stride;
      dp[u] = nullptr;
      if (i >= total) continue;
      const int s = i / per_row;
      int rem = i - s * per_row;
      const int part = rem / per_part;
      rem -= part * per_part;
      const int hl = rem / g8, j = (rem - hl * g8) * 8;
      const int q = s / T, t = s - q * T;
      const __nv_bfloat16* sp = static_cast<const __nv_bfloat16*>(src.p[q]) +
                                (static_cast<int64_t>(t) * parts + part) * H + rank * Hl + hl * d + j;
      dp[u] = dst + (static_cast<int64_t>(s) * parts + part) * Hl + hl * d + j;
      spos[u] = s; part_u[u] = part; j_u[u] = j;
      lo[u] = ld_v4(sp);
      hi[u] = ld_v4(sp + half);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (!dp[u]) continue;
      if (part_u[u] < rope_parts) {
        const int64_t cs = static_cast<int64_t>(spos[u]) * half + j_u[u];
        rotate8(lo[u], hi[u], cos_t + cs, sin_t + cs, 1.f);
      }
      *reinterpret_cast<uint4*>(dp[u]) = lo[u];
      *reinterpret_cast<uint4*>(dp[u] + half) = hi[u];
    }
  }
}

// Head-sharded [S, parts*Hl] on every rank -> token-sharded [T, parts*H] on this rank.
template <int kU>
__global__ void __launch_bounds__(256) a2a_to_tokens_kernel(PeerPtrs src, int world, int rank, int T, int H,
                                                            int parts, int d, __nv_bfloat16* __restrict__ dst,
                                                            const float* __restrict__ cos_t,
                                                            const float* __restrict__ sin_t, int rope_parts) {
  const int Hl = H / world, heads = H / d, heads_l = Hl / d, half = d / 2, g8 = half / 8;
  const int per_part = heads * g8;
  const int per_row = parts * per_part;
  const int total = T * per_row;
  const int stride = gridDim.x * blockDim.x;
  // kU units per round as in a2a_to_heads_kernel
  for (int i0 = blockIdx.x * blockDim.x + threadIdx.x; i0 < total; i0 += kU * stride) {
    uint4 lo[kU], hi[kU];
    __nv_bfloat16* dp[kU];
    int spos[kU], part_u[kU], j_u[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int i = i0 + u * stride;
      dp[u] = nullptr;
      if (i >= total) continue;
      const int t = i / per_row;
      int rem = i - t * per_row;
      const int part = rem / per_part;
      rem -= part * per_part;
      const int hg = rem / g8, j = (rem - hg * g8) * 8;  // hg = global head
      const int q = hg / heads_l;                        // owner rank of that head
      const int hl = hg - q * heads_l;
      const int s = rank * T + t;                        // global position
      const __nv_bfloat16* sp = static_cast<const __nv_bfloat16*>(src.p[q]) +
                                (static_cast<int64_t>(s) * parts + part) * Hl + hl * d + j;
      dp[u] = dst + (static_cast<int64_t>(t) * parts + part) * H + hg * d + j;
      spos[u] = s; part_u[u] = part; j_u[u] = j;
      lo[u] = ld_v4(sp);
      hi[u] = ld_v4(sp + half);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (!dp[u]) continue;
      if (part_u[u] < rope_parts) {
        const int64_t cs = static_cast<int64_t>(spos[u]) * half + j_u[u];
        rotate8(lo[u], hi[u], cos_t + cs, sin_t + cs, -1.f);
      }
      *reinterpret_cast<uint4*>(dp[u]) = lo[u];
      *reinterpret_cast<uint4*>(dp[u] + half) = hi[u];
    }
  }
}

__global__ void peer_barrier_kernel(PeerPtrs flags, int world, int rank, uint32_t epoch,
                                    uint32_t* error_flag) {
  const int q = threadIdx.x;
  if (q >= world) return;
  __threadfence_system();
  // publish: flags_q[rank] = epoch on every peer (including self)
  st_release_sys(static_cast<uint32_t*>(flags.p[q]) + rank, epoch);
  // wait: own flags[q] >= epoch
  const uint32_t* mine = static_cast<const uint32_t*>(flags.p[rank]) + q;
  const long long start = clock64();
  const long long limit = 40000000000LL;  // ~20 s at 2 GHz
  while (static_cast<int32_t>(ld_acquire_sys(mine) - epoch) < 0) {
    if (clock64() - start > limit) {  // a dead or hung peer: fail loudly instead of reading stale data
      atomicExch(error_flag, 1u);
      __threadfence_system();
      __trap();
    }
    __nanosleep(64);
  }
  __threadfence_system();
}

// Push copy (all-gather of weight shards, reduce-scatter staging of gradient partials): for
// every destination rank q (starting at rank+1 so that at any moment each GPU receives from one
// peer) and every job, blocks of `blk` bytes are read from this rank's memory at
// src + q*src_q + b*src_stride and stored into q's symmetric heap at dst_q + dst_off + b*dst_stride.
// Posted NVLink writes run at link speed with few CTAs, which stay co-resident with the
// persistent tcgen05 kernels (no shared memory, 32 registers).
__global__ void __launch_bounds__(256) push_copy_kernel(PushJobs jobs, PeerPtrs dst, int world, int rank) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int k = 0; k < world; ++k) {
    const int q = (rank + 1 + k) % world;
    for (int jb = 0; jb < jobs.n; ++jb) {
      const PushJob& J = jobs.j[jb];
      const char* src = J.src + q * J.src_q;
      char* dbase = static_cast<char*>(dst.p[q]) + J.dst_off;
      const int64_t bv = J.blk / 16, total = bv * J.nblk;
      int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
      if (J.nblk == 1) {
        const uint4* s4 = reinterpret_cast<const uint4*>(src);
        uint4* d4 = reinterpret_cast<uint4*>(dbase);
        for (; i + 7 * stride < total; i += 8 * stride) {  // 128 B in flight per thread
          uint4 v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = ld_v4(s4 + i + u * stride);
#pragma unroll
          for (int u = 0; u < 8; ++u) d4[i + u * stride] = v[u];
        }
        for (; i < total; i += stride) d4[i] = ld_v4(s4 + i);
      } else {
        for (; i < total; i += stride) {
          const int64_t b = i / bv, e = i - b * bv;
          const uint4 v = ld_v4(src + b * J.src_stride + e * 16);
          *reinterpret_cast<uint4*>(dbase + b * J.dst_stride + e * 16) = v;
        }
      }
    }
  }
  __threadfence_system();  // remote stores performed before the stream's flag write
}

// NVLink SHARP all-gather: this rank's shard blocks (jobs with src_q == 0) stored once, 16 B per
// thread, to the multicast address `mc` + dst_off — the switch writes every rank's copy, this
// rank's included — then a system-scope fence so the stores are performed before the stream's flag.
__global__ void __launch_bounds__(256) nvls_push_kernel(PushJobs jobs, char* mc) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int jb = 0; jb < jobs.n; ++jb) {
    const PushJob& J = jobs.j[jb];
    const uint32_t bv = static_cast<uint32_t>(J.blk / 16);  // 16-B units per block (< 2^32)
    const int64_t total = int64_t(bv) * J.nblk;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total; i += stride) {
      int64_t b = 0, e = i;
      if (J.nblk > 1) {  // one job stays below 2^32 units: 32-bit division
        const uint32_t i32 = static_cast<uint32_t>(i);
        b = i32 / bv;
        e = i32 - static_cast<uint32_t>(b) * bv;
      }
      const uint4 v = ld_v4(J.src + b * J.src_stride + e * 16);
      char* d = mc + J.dst_off + b * J.dst_stride + e * 16;
      asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(d), "r"(v.x), "r"(v.y),
                   "r"(v.z), "r"(v.w)
                   : "memory");
    }
  }
  asm volatile("fence.sc.sys;" ::: "memory");
}

// Bulk-copy push (the production weight all-gather / reduce-scatter staging in multi-process
// mode): one thread per CTA drives the TMA unit — cp.async.bulk global -> shared (mbarrier
// completion), then cp.async.bulk shared -> peer global for every destination. Tens of such
// CTAs keep ~1 MB in flight over NVLink with no per-byte SM instructions.
// bcast (every job has src_q == 0): each chunk is read once and stored to all ranks.
// 2 x 16 KB slots: the CTA fits beside a GEMM / attention-forward CTA (~198 KB) on one SM, so
// the copy needs no SMs of its own and the persistent grids stay whole.
template <int CH, int NS>
constexpr int bulk_smem() { return CH * NS + 64 + 128; }

__device__ __forceinline__ void bulk_g2s(uint32_t smem, const void* g, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem),
               "l"(g), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* g, uint32_t smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(smem), "r"(bytes) : "memory");
}

struct ChunkRef {
  const char* src;
  char* dst_rel;  // offset within the destination heap (added to dst.p[q])
  uint32_t bytes;
};

template <int kBulkChunk, int kBulkSlots>
__global__ void __launch_bounds__(32) push_bulk_kernel(PushJobs jobs, PeerPtrs dst, int world, int rank, int bcast) {
  extern __shared__ __align__(128) uint8_t sm_raw[];
  if (threadIdx.x != 0) return;
  uint8_t* buf = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 127) & ~uintptr_t(127));
  uint64_t* bars = reinterpret_cast<uint64_t*>(buf + kBulkChunk * kBulkSlots);
  for (int i = 0; i < kBulkSlots; ++i) mbar_init(&bars[i], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  // item space: per job, nblk x ceil(blk / chunk) chunks; per destination unless bcast
  int64_t cpb[2], njob_items[2], per_dest = 0;
  for (int j = 0; j < jobs.n; ++j) {
    cpb[j] = (jobs.j[j].blk + kBulkChunk - 1) / kBulkChunk;
    njob_items[j] = cpb[j] * jobs.j[j].nblk;
    per_dest += njob_items[j];
  }
  const int ndest = bcast ? 1 : world;
  const int64_t total = per_dest * ndest;
  auto item = [&](int64_t it, int& qsel) {
    const int k = static_cast<int>(it / per_dest);
    int64_t r = it - k * per_dest;
    qsel = bcast ? -1 : (rank + 1 + k) % world;
    int j = 0;
    if (jobs.n > 1 && r >= njob_items[0]) {
      r -= njob_items[0];
      j = 1;
    }
    const PushJob& J = jobs.j[j];
    const int64_t b = r / cpb[j], c = r - b * cpb[j];
    const int64_t off = c * kBulkChunk;
    ChunkRef ref;
    ref.src = J.src + (qsel < 0 ? 0 : qsel * J.src_q) + b * J.src_stride + off;
    ref.dst_rel = reinterpret_cast<char*>(J.dst_off + b * J.dst_stride + off);
    ref.bytes = static_cast<uint32_t>(J.blk - off < kBulkChunk ? J.blk - off : kBulkChunk);
    return ref;
  };
  // this CTA's items: it = blockIdx.x + n * gridDim.x
  const int64_t mine = total > blockIdx.x ? (total - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const uint32_t sbase = smem_u32(buf), bbase = smem_u32(bars);
  auto issue_load = [&](int64_t n) {
    int qs;
    const ChunkRef r = item(blockIdx.x + n * gridDim.x, qs);
    const int slot = static_cast<int>(n % kBulkSlots);
    mbar_arrive_expect_tx(&bars[slot], r.bytes);
    bulk_g2s(sbase + slot * kBulkChunk, r.src, r.bytes, bbase + slot * 8);
  };
  for (int64_t n = 0; n < mine && n < kBulkSlots - 1; ++n) issue_load(n);
  for (int64_t n = 0; n < mine; ++n) {
    const int slot = static_cast<int>(n % kBulkSlots);
    mbar_wait(&bars[slot], static_cast<uint32_t>((n / kBulkSlots) & 1));
    int qs;
    const ChunkRef r = item(blockIdx.x + n * gridDim.x, qs);
    if (qs < 0) {
      for (int k = 0; k < world; ++k) {
        const int q = (rank + 1 + k) % world;
        bulk_s2g(static_cast<char*>(dst.p[q]) + reinterpret_cast<uintptr_t>(r.dst_rel), sbase + slot * kBulkChunk, r.bytes);
      }
    } else {
      bulk_s2g(static_cast<char*>(dst.p[qs]) + reinterpret_cast<uintptr_t>(r.dst_rel), sbase + slot * kBulkChunk, r.bytes);
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    // refill: the slot of item n+kBulkSlots-1 was last used by item n-1, whose stores must have
    // finished reading it (at most the current group still reading)
    if (n + kBulkSlots - 1 < mine) {
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      issue_load(n + kBulkSlots - 1);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // stores complete
  __threadfence_system();
}

int ctas(int64_t work, int threads, int cap) {
  const int64_t b = (work + threads - 1) / threads;
  return static_cast<int>(b < cap ? (b > 0 ? b : 1) : cap);
}

}  // namespace

cudaError_t allgather_pull(const PeerPtrs& src, int world, int64_t shard_elems, __nv_bfloat16* dst,
                           cudaStream_t st, int num_sms, int num_ctas) {
  (void)num_sms;
  if (shard_elems % 8) return cudaErrorInvalidValue;
  const int64_t sv = shard_elems / 8;
  allgather_pull_kernel<<<ctas(sv * world, 256, num_ctas), 256, 0, st>>>(src, world, sv,
                                                                        reinterpret_cast<uint4*>(dst));
  return cudaGetLastError();
}

cudaError_t allgather_pull_interleave(const PeerPtrs& sg, const PeerPtrs& su, int world,
                                      int64_t rows, int64_t cols, __nv_bfloat16* dst,
                                      cudaStream_t st, int num_ctas) {
  if (cols % 8 || rows % kGuBlock || rows % world) return cudaErrorInvalidValue;
  allgather_interleave_kernel<<<ctas(2 * rows * cols / 8, 256, num_ctas), 256, 0, st>>>(
      sg, su, world, rows, cols, reinterpret_cast<uint4*>(dst));
  return cudaGetLastError();
}

cudaError_t reduce_scatter_pull(const PeerPtrs& part, int world, int rank, int64_t shard_elems,
                                bool part_is_f32, float scale, int accumulate, float* out,
                                cudaStream_t st, int num_ctas) {
  if (shard_elems % 8) return cudaErrorInvalidValue;
  const int64_t n8 = shard_elems / 8;
  const int64_t base = static_cast<int64_t>(rank) * shard_elems;
  if (part_is_f32)
    reduce_scatter_kernel<true><<<ctas(n8, 256, num_ctas), 256, 0, st>>>(part, world, base, n8, scale,
                                                                       accumulate, out);
  else
    reduce_scatter_kernel<false><<<ctas(n8, 256, num_ctas), 256, 0, st>>>(part, world, base, n8, scale,
                                                                        accumulate, out);
  return cudaGetLastError();
}

cudaError_t reduce_scatter_pull_interleave(const PeerPtrs& part, int world, int rank, int64_t rows,
                                           int64_t cols, float scale, int accumulate,
                                           float* out_gate, float* out_up, cudaStream_t st,
                                           int num_ctas) {
  if (cols % 8 || rows % world || rows % kGuBlock) return cudaErrorInvalidValue;
  reduce_scatter_interleave_kernel<<<ctas(2 * rows / world * cols / 8, 256, num_ctas), 256, 0, st>>>(
      part, world, rank, rows, cols, scale, accumulate, out_gate, out_up);
  return cudaGetLastError();
}

cudaError_t nvls_reduce_scatter(const __nv_bfloat16* mc_part, int world, int rank, int64_t shard_elems,
                                int64_t interleave_rows, int64_t cols, float scale, int accumulate, float* out,
                                float* out_up, cudaStream_t st, int num_ctas) {
  if (shard_elems % 8 || cols % 8) return cudaErrorInvalidValue;
  const int64_t units = interleave_rows > 0 ? 2 * interleave_rows / world * cols / 8 : shard_elems / 8;
  nvls_reduce_kernel<<<ctas(units, 256, num_ctas), 256, 0, st>>>(mc_part, world, rank, shard_elems / 8,
                                                                 interleave_rows, cols, scale, accumulate, out,
                                                                 out_up);
  return cudaGetLastError();
}

// Units per thread per round of the all-to-all kernels (SEQPLAN_ISP_A2A_UNROLL=1 for A/B).
int a2a_unroll() {
  static const int u = [] {
    const char* e = std::getenv("SEQPLAN_ISP_A2A_UNROLL");
    return e && std::atoi(e) == 1 ? 1 : 4;
  }();
  return u;
}

cudaError_t a2a_tokens_to_heads(const PeerPtrs& src, int world, int rank, int T, int H, int parts,
                                __nv_bfloat16* dst, const float* cos_t, const float* sin_t, int d,
                                int rope_parts, cudaStream_t st, int num_ctas) {
  if ((H / world) % d || d % 16) return cudaErrorInvalidValue;
  const int64_t work = static_cast<int64_t>(T) * world * parts * (H / world / d) * (d / 16);
  auto kern = a2a_unroll() == 1 ? a2a_to_heads_kernel<1> : a2a_to_heads_kernel<4>;
  kern<<<ctas(work, 256, num_ctas), 256, 0, st>>>(src, world, rank, T, H, parts, d,
                                                                  dst, cos_t, sin_t, rope_parts);
  return cudaGetLastError();
}

cudaError_t a2a_heads_to_tokens(const PeerPtrs& src, int world, int rank, int T, int H, int parts,
                                __nv_bfloat16* dst, const float* cos_t, const float* sin_t, int d,
                                int rope_parts, cudaStream_t st, int num_ctas) {
  if ((H / world) % d || d % 16) return cudaErrorInvalidValue;
  const int64_t work = static_cast<int64_t>(T) * parts * (H / d) * (d / 16);
  auto kern = a2a_unroll() == 1 ? a2a_to_tokens_kernel<1> : a2a_to_tokens_kernel<4>;
  kern<<<ctas(work, 256, num_ctas), 256, 0, st>>>(src, world, rank, T, H, parts, d,
                                                                   dst, cos_t, sin_t, rope_parts);
  return cudaGetLastError();
}

cudaError_t nvls_push(const PushJobs& jobs, char* mc, cudaStream_t st, int num_ctas) {
  for (int j = 0; j < jobs.n; ++j) {
    const PushJob& J = jobs.j[j];
    if (J.blk / 16 * J.nblk >= (int64_t(1) << 32)) return cudaErrorInvalidValue;
    if (J.blk % 16 || J.src_stride % 16 || J.dst_stride % 16 || J.dst_off % 16 || J.src_q != 0 ||
        reinterpret_cast<uintptr_t>(J.src) % 16)
      return cudaErrorInvalidValue;
  }
  nvls_push_kernel<<<num_ctas, 256, 0, st>>>(jobs, mc);
  return cudaGetLastError();
}

cudaError_t push_copy(const PushJobs& jobs, const PeerPtrs& dst, int world, int rank, cudaStream_t st, int num_ctas,
                      int kind) {
  for (int j = 0; j < jobs.n; ++j) {
    const PushJob& J = jobs.j[j];
    if (J.blk % 16 || J.src_stride % 16 || J.dst_stride % 16 || J.dst_off % 16 || J.src_q % 16 ||
        reinterpret_cast<uintptr_t>(J.src) % 16)
      return cudaErrorInvalidValue;
  }
  int bcast = 1;
  for (int j = 0; j < jobs.n; ++j) bcast &= jobs.j[j].src_q == 0;
  if (kind == kPushBulk) {  // 2 x 16 KB slots: co-resides with a ~198 KB GEMM / attention CTA
    constexpr int sm = bulk_smem<16384, 2>();
    static bool attr = false;
    if (!attr) {
      cudaError_t e = cudaFuncSetAttribute(push_bulk_kernel<16384, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
      if (e != cudaSuccess) return e;
      attr = true;
    }
    push_bulk_kernel<16384, 2><<<num_ctas, 32, sm, st>>>(jobs, dst, world, rank, bcast);
    return cudaGetLastError();
  }
  if (kind == kPushBulkWide) {  // 4 x 32 KB slots: an SM of its own per CTA
    constexpr int sm = bulk_smem<32768, 4>();
    static bool attr = false;
    if (!attr) {
      cudaError_t e = cudaFuncSetAttribute(push_bulk_kernel<32768, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
      if (e != cudaSuccess) return e;
      attr = true;
    }
    push_bulk_kernel<32768, 4><<<num_ctas, 32, sm, st>>>(jobs, dst, world, rank, bcast);
    return cudaGetLastError();
  }
  push_copy_kernel<<<num_ctas, 256, 0, st>>>(jobs, dst, world, rank);
  return cudaGetLastError();
}

cudaError_t peer_barrier(const PeerPtrs& flags, int world, int rank, uint32_t epoch,
                         uint32_t* error_flag, cudaStream_t st) {
  peer_barrier_kernel<<<1, 32, 0, st>>>(flags, world, rank, epoch, error_flag);
  return cudaGetLastError();
}

}  // namespace isp
