// HBM-bound kernels of the ISP block: RMSNorm fwd/bwd, RoPE, SwiGLU backward,
// casts and the index-keyed synthetic initialiser (sm_100a).
//
// These carry no reference counterpart (the reference's FLOP model prices
// matmuls only, proj/include/seqplan/cost.hpp:209-219); their algorithm follows
// the block definition of oracle/block_oracle.c. All loads/stores are 16-byte
// vectors over rows; grids are sized in multiples of the SM count.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "gemm.h"
#include "kernels.h"

namespace isp {

namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// Same construction as oracle/block_oracle.c:ob_keyed_normal (double precision).
__device__ __forceinline__ double keyed_normal(uint64_t base, int64_t idx) {
  const uint64_t r1 = splitmix64(base ^ static_cast<uint64_t>(2 * idx));
  const uint64_t r2 = splitmix64(base ^ static_cast<uint64_t>(2 * idx + 1));
  const double u1 = static_cast<double>((r1 >> 11) + 1) * 0x1.0p-53;
  const double u2 = static_cast<double>(r2 >> 11) * 0x1.0p-53;
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

__global__ void keyed_fill_kernel(uint64_t base, int64_t offset, int64_t n, double mean,
                                  double stdv, float* __restrict__ out_f32,
                                  __nv_bfloat16* __restrict__ out_bf16) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float v = static_cast<float>(mean + stdv * keyed_normal(base, offset + i));
    if (out_f32) out_f32[i] = v;
    if (out_bf16) out_bf16[i] = __float2bfloat16_rn(v);
  }
}

// fp32 -> bf16, 8 elements per thread (two 16-B loads, one 16-B store) when both pointers are
// 16-B aligned; the scalar loop takes the tail (and misaligned calls).
__global__ void cast_f32_bf16_kernel(const float* __restrict__ in, __nv_bfloat16* __restrict__ out,
                                     int64_t n) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t tid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  int64_t done = 0;
  if ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) % 16 == 0) {
    const int64_t n8 = n / 8;
    const float4* in4 = reinterpret_cast<const float4*>(in);
    uint4* out8 = reinterpret_cast<uint4*>(out);
    for (int64_t i = tid; i < n8; i += stride) {
      const float4 a = in4[2 * i], b = in4[2 * i + 1];
      out8[i] = make_uint4(pack_bf16(a.x, a.y), pack_bf16(a.z, a.w), pack_bf16(b.x, b.y), pack_bf16(b.z, b.w));
    }
    done = n8 * 8;
  }
  for (int64_t i = done + tid; i < n; i += stride) out[i] = __float2bfloat16_rn(in[i]);
}

// One CTA of 128 threads per row; row held in registers (H <= 8192).
constexpr int kNormThreads = 128;
constexpr int kNormVecCap = 8;  // up to 8 x 8 bf16 per thread (H <= 8192)

__device__ __forceinline__ float block_sum_128(float v, float* red) {
  v = warp_sum(v);
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  return red[0] + red[1] + red[2] + red[3];
}

__device__ __forceinline__ void load8(const __nv_bfloat16* p, float (&f)[8]) {
  const uint4 q = *reinterpret_cast<const uint4*>(p);
  const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 t = unpack_bf16(w[e]);
    f[2 * e] = t.x;
    f[2 * e + 1] = t.y;
  }
}
__device__ __forceinline__ void store8(__nv_bfloat16* p, const float (&f)[8]) {
  *reinterpret_cast<uint4*>(p) = make_uint4(pack_bf16(f[0], f[1]), pack_bf16(f[2], f[3]),
                                            pack_bf16(f[4], f[5]), pack_bf16(f[6], f[7]));
}

template <int kNormMaxVec>
__global__ void __launch_bounds__(kNormThreads) rmsnorm_fwd_kernel(
    const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ g,
    __nv_bfloat16* __restrict__ y, float* __restrict__ rstd, int T, int H, float eps) {
  __shared__ float red[4];
  const int nvec = H / 8;
  for (int t = blockIdx.x; t < T; t += gridDim.x) {
    const __nv_bfloat16* xr = x + static_cast<int64_t>(t) * H;
    float v[kNormMaxVec][8];
    float ss = 0.f;
#pragma unroll
    for (int c = 0; c < kNormMaxVec; ++c) {
      const int vi = threadIdx.x + c * kNormThreads;
      if (vi < nvec) {
        load8(xr + vi * 8, v[c]);
#pragma unroll
        for (int e = 0; e < 8; ++e) ss += v[c][e] * v[c][e];
      }
    }
    ss = block_sum_128(ss, red);
    const float r = rsqrtf(ss / static_cast<float>(H) + eps);
    if (threadIdx.x == 0) rstd[t] = r;
#pragma unroll
    for (int c = 0; c < kNormMaxVec; ++c) {
      const int vi = threadIdx.x + c * kNormThreads;
      if (vi < nvec) {
        float gw[8], o[8];
        load8(g + vi * 8, gw);
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = v[c][e] * r * gw[e];
        store8(y + static_cast<int64_t>(t) * H + vi * 8, o);
      }
    }
  }
}

// dx = dres + rstd * (dn*g - xhat * mean(dn*g*xhat)); dg[j] += sum_t dn*xhat.
template <int kNormMaxVec>
__global__ void __launch_bounds__(kNormThreads) rmsnorm_bwd_kernel(
    const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ g,
    const float* __restrict__ rstd, const __nv_bfloat16* __restrict__ dn,
    const __nv_bfloat16* __restrict__ dres, __nv_bfloat16* __restrict__ dx,
    float* __restrict__ dg, float* __restrict__ dg_part, int T, int H) {
  __shared__ float red[4];
  const int nvec = H / 8;
  float dgacc[kNormMaxVec][8];
#pragma unroll
  for (int c = 0; c < kNormMaxVec; ++c)
#pragma unroll
    for (int e = 0; e < 8; ++e) dgacc[c][e] = 0.f;
  for (int t = blockIdx.x; t < T; t += gridDim.x) {
    const int64_t row = static_cast<int64_t>(t) * H;
    const float r = rstd[t];
    float xh[kNormMaxVec][8], dng[kNormMaxVec][8];
    float dot = 0.f;
#pragma unroll
    for (int c = 0; c < kNormMaxVec; ++c) {
      const int vi = threadIdx.x + c * kNormThreads;
      if (vi < nvec) {
        float xv[8], dv[8], gw[8];
        load8(x + row + vi * 8, xv);
        load8(dn + row + vi * 8, dv);
        load8(g + vi * 8, gw);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          xh[c][e] = xv[e] * r;
          dng[c][e] = dv[e] * gw[e];
          dot += dng[c][e] * xh[c][e];
          dgacc[c][e] += dv[e] * xh[c][e];
        }
      }
    }
    dot = block_sum_128(dot, red);
    const float m = dot / static_cast<float>(H);
#pragma unroll
    for (int c = 0; c < kNormMaxVec; ++c) {
      const int vi = threadIdx.x + c * kNormThreads;
      if (vi < nvec) {
        float rv[8], o[8];
        load8(dres + row + vi * 8, rv);
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = rv[e] + r * (dng[c][e] - xh[c][e] * m);
        store8(dx + row + vi * 8, o);
      }
    }
  }
#pragma unroll
  for (int c = 0; c < kNormMaxVec; ++c) {
    const int vi = threadIdx.x + c * kNormThreads;
    if (vi < nvec) {
      if (dg_part) {  // stage 1 of a deterministic two-stage column reduction
        float4* o = reinterpret_cast<float4*>(dg_part + static_cast<int64_t>(blockIdx.x) * H + vi * 8);
        o[0] = make_float4(dgacc[c][0], dgacc[c][1], dgacc[c][2], dgacc[c][3]);
        o[1] = make_float4(dgacc[c][4], dgacc[c][5], dgacc[c][6], dgacc[c][7]);
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) atomicAdd(dg + vi * 8 + e, dgacc[c][e]);
      }
    }
  }
}

// dg[j] += sum_b part[b, j]: one CTA per 32 columns, 32 row groups (warp w sums rows w, w+32, ...
// with its lanes on consecutive columns: 128-B coalesced rows), then the 32 group sums are added
// in fixed order through shared memory — deterministic, and 128 CTAs instead of H/128 long loops.
__global__ void __launch_bounds__(1024) column_sum_kernel(const float* __restrict__ part, int rows, int H,
                                                          float* __restrict__ dg) {
  __shared__ float red[32][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int j = blockIdx.x * 32 + lane;
  float s0 = 0.f, s1 = 0.f;
  if (j < H) {
    int b = w;
    for (; b + 32 < rows; b += 64) {
      s0 += part[static_cast<int64_t>(b) * H + j];
      s1 += part[static_cast<int64_t>(b + 32) * H + j];
    }
    if (b < rows) s0 += part[static_cast<int64_t>(b) * H + j];
  }
  red[w][lane] = s0 + s1;
  __syncthreads();
  if (w == 0 && j < H) {
    float t = 0.f;
#pragma unroll 8
    for (int g = 0; g < 32; ++g) t += red[g][lane];
    dg[j] += t;
  }
}

// In-place rotate-half RoPE on the q and k parts of token rows (ld elements apart).
// dir = +1 forward rotation, -1 its transpose (backward). One thread = 8 pairs (16-B vectors).
__global__ void rope_kernel(__nv_bfloat16* __restrict__ qkv, int64_t ld, int T, int t0,
                            int heads, int d, const float* __restrict__ cos_t,
                            const float* __restrict__ sin_t, int k_offset, int dir) {
  const int half = d / 2, g8 = half / 8;
  const int per_row = 2 * heads * g8;  // q and k
  const int64_t total = static_cast<int64_t>(T) * per_row;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int t = static_cast<int>(i / per_row);
    int rem = static_cast<int>(i % per_row);
    const int part = rem / (heads * g8);
    rem %= heads * g8;
    const int h = rem / g8, j = (rem % g8) * 8;
    __nv_bfloat16* base = qkv + static_cast<int64_t>(t) * ld + (part ? k_offset : 0) + h * d;
    const float* cp = cos_t + static_cast<int64_t>(t0 + t) * half + j;
    const float* sp = sin_t + static_cast<int64_t>(t0 + t) * half + j;
    const float4 c0 = *reinterpret_cast<const float4*>(cp), c1 = *reinterpret_cast<const float4*>(cp + 4);
    const float4 s0 = *reinterpret_cast<const float4*>(sp), s1 = *reinterpret_cast<const float4*>(sp + 4);
    const float cs[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
    const float sg = dir < 0 ? -1.f : 1.f;
    const float sn[8] = {sg * s0.x, sg * s0.y, sg * s0.z, sg * s0.w, sg * s1.x, sg * s1.y, sg * s1.z, sg * s1.w};
    float a[8], b[8], oa[8], ob[8];
    load8(base + j, a);
    load8(base + j + half, b);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      oa[e] = a[e] * cs[e] - b[e] * sn[e];
      ob[e] = b[e] * cs[e] + a[e] * sn[e];
    }
    store8(base + j, oa);
    store8(base + j + half, ob);
  }
}

// dgu (kGuBlock-col interleaved gate|up) from da and saved gu.
__global__ void swiglu_bwd_kernel(const __nv_bfloat16* __restrict__ da,
                                  const __nv_bfloat16* __restrict__ gu,
                                  __nv_bfloat16* __restrict__ dgu, int T, int I) {
  const int64_t total = static_cast<int64_t>(T) * I / 8;  // 8 activation columns per thread
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t col8 = (i % (I / 8)) * 8;
    const int64_t t = i / (I / 8);
    const int64_t blk = col8 / kGuBlock, within = col8 % kGuBlock;
    const int64_t gcol = blk * 2 * kGuBlock + within, ucol = gcol + kGuBlock;
    float dav[8], gv[8], uv[8], dg[8], du[8];
    load8(da + t * I + col8, dav);
    load8(gu + t * 2 * I + gcol, gv);
    load8(gu + t * 2 * I + ucol, uv);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float sg = 1.f / (1.f + __expf(-gv[e]));
      dg[e] = dav[e] * uv[e] * sg * (1.f + gv[e] * (1.f - sg));
      du[e] = dav[e] * gv[e] * sg;
    }
    store8(dgu + t * 2 * I + gcol, dg);
    store8(dgu + t * 2 * I + ucol, du);
  }
}

int grid_for(int64_t work, int threads, int num_sms) {
  const int64_t blocks = (work + threads - 1) / threads;
  const int64_t cap = static_cast<int64_t>(num_sms) * 16;
  return static_cast<int>(blocks < cap ? (blocks > 0 ? blocks : 1) : cap);
}

}  // namespace

int rmsnorm_bwd_scratch_rows(int num_sms) { return 4 * num_sms; }  // 4 CTAs per SM (measured: 8 -> 4 is 62 -> 54 us at 7B-4K; fewer rows of dg partials)

uint64_t keyed_stream_base(uint64_t seed, int tensor_id) {
  uint64_t z = seed * 0x9E3779B97F4A7C15ULL + static_cast<uint64_t>(tensor_id);
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

cudaError_t keyed_fill(uint64_t seed, int tensor_id, int64_t offset, int64_t n, double mean,
                       double stdv, float* out_f32, __nv_bfloat16* out_bf16, cudaStream_t st,
                       int num_sms) {
  if (n <= 0) return cudaSuccess;
  keyed_fill_kernel<<<grid_for(n, 256, num_sms), 256, 0, st>>>(keyed_stream_base(seed, tensor_id),
                                                                offset, n, mean, stdv, out_f32,
                                                                out_bf16);
  return cudaGetLastError();
}

// AdamW on one fp32 master shard (decoupled weight decay, bias-corrected moments, the update
// rule of torch.optim.AdamW), fused with the refresh of the bf16 working shard. 4 elements per
// thread (16-B vectors); n % 4 == 0 (every shard is a multiple of 8 elements).
__global__ void adamw_kernel(float* __restrict__ w, const float* __restrict__ g, float* __restrict__ m,
                             float* __restrict__ v, __nv_bfloat16* __restrict__ wb, int64_t n4, AdamWArgs a) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float4 W = reinterpret_cast<float4*>(w)[i];
    const float4 G = reinterpret_cast<const float4*>(g)[i];
    float4 M = reinterpret_cast<float4*>(m)[i], V = reinterpret_cast<float4*>(v)[i];
    float* pw = &W.x;
    const float* pg = &G.x;
    float* pm = &M.x;
    float* pv = &V.x;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      pw[e] -= a.lr * a.weight_decay * pw[e];
      pm[e] = a.beta1 * pm[e] + (1.f - a.beta1) * pg[e];
      pv[e] = a.beta2 * pv[e] + (1.f - a.beta2) * pg[e] * pg[e];
      const float mh = pm[e] * a.inv_bc1, vh = pv[e] * a.inv_bc2;
      pw[e] -= a.lr * mh / (sqrtf(vh) + a.eps);
    }
    reinterpret_cast<float4*>(w)[i] = W;
    reinterpret_cast<float4*>(m)[i] = M;
    reinterpret_cast<float4*>(v)[i] = V;
    uint2 b;
    b.x = pack_bf16(W.x, W.y);
    b.y = pack_bf16(W.z, W.w);
    reinterpret_cast<uint2*>(wb)[i] = b;
  }
}

cudaError_t adamw_step(float* w, const float* g, float* m, float* v, __nv_bfloat16* wb, int64_t n, const AdamWArgs& a,
                       cudaStream_t st, int num_sms) {
  if (n % 4) return cudaErrorInvalidValue;
  if (n == 0) return cudaSuccess;
  adamw_kernel<<<grid_for(n / 4, 256, num_sms), 256, 0, st>>>(w, g, m, v, wb, n / 4, a);
  return cudaGetLastError();
}

cudaError_t cast_f32_bf16(const float* in, __nv_bfloat16* out, int64_t n, cudaStream_t st,
                          int num_sms) {
  if (n <= 0) return cudaSuccess;
  cast_f32_bf16_kernel<<<grid_for(n, 256, num_sms), 256, 0, st>>>(in, out, n);
  return cudaGetLastError();
}

cudaError_t rmsnorm_fwd(const __nv_bfloat16* x, const __nv_bfloat16* g, __nv_bfloat16* y,
                        float* rstd, int T, int H, float eps, cudaStream_t st, int num_sms) {
  if (H % 8 || H > kNormThreads * kNormVecCap * 8) return cudaErrorInvalidValue;
  const int grid = T < num_sms * 8 ? T : num_sms * 8;
  const int nv = (H / 8 + kNormThreads - 1) / kNormThreads;
  switch (nv) {
#define ISP_NORM_CASE(N) case N: rmsnorm_fwd_kernel<N><<<grid, kNormThreads, 0, st>>>(x, g, y, rstd, T, H, eps); break;
    ISP_NORM_CASE(1) ISP_NORM_CASE(2) ISP_NORM_CASE(3) ISP_NORM_CASE(4)
    ISP_NORM_CASE(5) ISP_NORM_CASE(6) ISP_NORM_CASE(7) ISP_NORM_CASE(8)
#undef ISP_NORM_CASE
  }
  return cudaGetLastError();
}

cudaError_t rmsnorm_bwd(const __nv_bfloat16* x, const __nv_bfloat16* g, const float* rstd,
                        const __nv_bfloat16* dn, const __nv_bfloat16* dres, __nv_bfloat16* dx,
                        float* dg, int T, int H, cudaStream_t st, int num_sms, float* dg_scratch) {
  if (H % 8 || H > kNormThreads * kNormVecCap * 8) return cudaErrorInvalidValue;
  int cap = dg_scratch ? rmsnorm_bwd_scratch_rows(num_sms) : num_sms * 4;
  if (const char* e = std::getenv("SEQPLAN_NORM_BWD_CTAS"))  // development: CTAs per SM
    cap = std::min(cap, std::max(1, std::atoi(e)) * num_sms);
  const int grid = T < cap ? T : cap;
  const int nv = (H / 8 + kNormThreads - 1) / kNormThreads;
  switch (nv) {
#define ISP_NORM_CASE(N) case N: rmsnorm_bwd_kernel<N><<<grid, kNormThreads, 0, st>>>(x, g, rstd, dn, dres, dx, dg, dg_scratch, T, H); break;
    ISP_NORM_CASE(1) ISP_NORM_CASE(2) ISP_NORM_CASE(3) ISP_NORM_CASE(4)
    ISP_NORM_CASE(5) ISP_NORM_CASE(6) ISP_NORM_CASE(7) ISP_NORM_CASE(8)
#undef ISP_NORM_CASE
  }
  if (dg_scratch) column_sum_kernel<<<(H + 31) / 32, 1024, 0, st>>>(dg_scratch, grid, H, dg);
  return cudaGetLastError();
}

cudaError_t rope_inplace(__nv_bfloat16* qkv, int64_t ld, int T, int t0, int heads, int d,
                         const float* cos_t, const float* sin_t, int k_offset, int dir,
                         cudaStream_t st, int num_sms) {
  if (d % 16) return cudaErrorInvalidValue;
  const int64_t work = static_cast<int64_t>(T) * 2 * heads * (d / 16);
  rope_kernel<<<grid_for(work, 256, num_sms), 256, 0, st>>>(qkv, ld, T, t0, heads, d, cos_t, sin_t,
                                                            k_offset, dir);
  return cudaGetLastError();
}

cudaError_t swiglu_bwd(const __nv_bfloat16* da, const __nv_bfloat16* gu, __nv_bfloat16* dgu, int T,
                       int I, cudaStream_t st, int num_sms) {
  if (I % kGuBlock) return cudaErrorInvalidValue;
  const int64_t work = static_cast<int64_t>(T) * I / 8;
  swiglu_bwd_kernel<<<grid_for(work, 256, num_sms), 256, 0, st>>>(da, gu, dgu, T, I);
  return cudaGetLastError();
}

}  // namespace isp
