// NVLink all-gather pattern microbenchmark (one process, N GPUs with peer access):
// every GPU receives a `size`-byte shard from every peer at the same time, by
//   ce_pull  copy engine, destination GPU's stream per peer (cudaMemcpyAsync peer -> local)
//   ce_push  copy engine, source GPU's stream per peer (local -> peer)
//   sm_pull  kernel on the destination GPU loading peer memory (16-B vectors)
//   sm_push  kernel on the source GPU storing into peer memory
// Prints per-GPU incoming GB/s = (N-1) * size / time. Development tool.
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

__global__ void copy_kernel(const int4* __restrict__ src, int4* __restrict__ dst, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    int4 a = src[i], b = src[i + stride], c = src[i + 2 * stride], d = src[i + 3 * stride];
    dst[i] = a; dst[i + stride] = b; dst[i + 2 * stride] = c; dst[i + 3 * stride] = d;
  }
  for (; i < n; i += stride) dst[i] = src[i];
}

struct Dst { char* p[8]; };
// one kernel per GPU pushing its shard to every peer: seq = peers one after another (all CTAs on
// one destination), split = CTAs partitioned across destinations
__global__ void push_all_kernel(const int4* __restrict__ src, Dst dst, int N, int g, size_t n, size_t slot, int split) {
  const size_t stride0 = (size_t)gridDim.x * blockDim.x;
  if (!split) {
    for (int k = 1; k < N; ++k) {
      const int q = (g + k) % N;
      int4* d = (int4*)(dst.p[q] + g * slot);
      size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
      for (; i + 3 * stride0 < n; i += 4 * stride0) {
        int4 a = src[i], b = src[i + stride0], c = src[i + 2 * stride0], e = src[i + 3 * stride0];
        d[i] = a; d[i + stride0] = b; d[i + 2 * stride0] = c; d[i + 3 * stride0] = e;
      }
      for (; i < n; i += stride0) d[i] = src[i];
    }
  } else {
    const int per = gridDim.x / (N - 1);
    const int k = 1 + blockIdx.x / per;
    if (k >= N) return;
    const int q = (g + k) % N;
    int4* d = (int4*)(dst.p[q] + g * slot);
    const size_t stride = (size_t)per * blockDim.x;
    size_t i = (blockIdx.x % per) * (size_t)blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n; i += 4 * stride) {
      int4 a = src[i], b = src[i + stride], c = src[i + 2 * stride], e = src[i + 3 * stride];
      d[i] = a; d[i + stride] = b; d[i + 2 * stride] = c; d[i + 3 * stride] = e;
    }
    for (; i < n; i += stride) d[i] = src[i];
  }
}

template <int CH, int NS>
__global__ void push_bulk(const char* src, Dst dst, int N, int g, size_t bytes, size_t slot_bytes) {
  extern __shared__ __align__(128) unsigned char sm[];
  if (threadIdx.x) return;
  unsigned long long* bars = (unsigned long long*)(sm + CH * NS);
  for (int i = 0; i < NS; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&bars[i])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const long long nch = (bytes + CH - 1) / CH;
  const long long mine = nch > blockIdx.x ? (nch - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const unsigned sb = (unsigned)__cvta_generic_to_shared(sm);
  auto load = [&](long long n) {
    const long long c = blockIdx.x + n * gridDim.x;
    const unsigned b = (unsigned)((bytes - c * CH) < CH ? (bytes - c * CH) : CH);
    const int slot = n % NS;
    const unsigned bar = (unsigned)__cvta_generic_to_shared(&bars[slot]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(b) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sb + slot * CH), "l"(src + c * CH), "r"(b), "r"(bar) : "memory");
  };
  for (long long n = 0; n < mine && n < NS - 1; ++n) load(n);
  for (long long n = 0; n < mine; ++n) {
    const int slot = n % NS;
    const unsigned bar = (unsigned)__cvta_generic_to_shared(&bars[slot]);
    const unsigned par = (n / NS) & 1;
    asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W;\n}" ::"r"(bar), "r"(par) : "memory");
    const long long c = blockIdx.x + n * gridDim.x;
    const unsigned b = (unsigned)((bytes - c * CH) < CH ? (bytes - c * CH) : CH);
    for (int k = 1; k < N; ++k) {
      const int q = (g + k) % N;
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst.p[q] + g * slot_bytes + c * CH), "r"(sb + slot * CH), "r"(b) : "memory");
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (n + NS - 1 < mine) { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); load(n + NS - 1); }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
  int N = 0;
  CK(cudaGetDeviceCount(&N));
  if (argc > 1) N = atoi(argv[1]);
  std::vector<size_t> sizes = {8u << 20, 25u << 20, 64u << 20};
  for (int g = 0; g < N; ++g) {
    CK(cudaSetDevice(g));
    for (int q = 0; q < N; ++q) if (q != g) CK(cudaDeviceEnablePeerAccess(q, 0));
  }
  for (size_t size : sizes) {
    std::vector<char*> src(N), dst(N);
    std::vector<std::vector<cudaStream_t>> st(N, std::vector<cudaStream_t>(N));
    for (int g = 0; g < N; ++g) {
      CK(cudaSetDevice(g));
      CK(cudaMalloc(&src[g], size));
      CK(cudaMalloc(&dst[g], size * N));
      CK(cudaMemset(src[g], g, size));
      for (int q = 0; q < N; ++q) CK(cudaStreamCreateWithFlags(&st[g][q], cudaStreamNonBlocking));
    }
    const char* names[] = {"ce_pull", "ce_push", "sm_pull", "sm_push", "push_seq", "push_split", "bulk12x2", "bulk32x4"};
    CK(cudaFuncSetAttribute(push_bulk<12288, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 12288 * 2 + 256));
    CK(cudaFuncSetAttribute(push_bulk<32768, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768 * 4 + 256));
    Dst D{};
    for (int g = 0; g < N; ++g) D.p[g] = dst[g];
    for (int mode = 4; mode < 8; ++mode) {
      for (int ctas : {16, 48, 96, 148}) {
        if (mode < 2 && ctas != 16) continue;
        auto run = [&]() {
          for (int g = 0; g < N; ++g) {
            CK(cudaSetDevice(g));
            if (mode == 6) { push_bulk<12288, 2><<<ctas, 32, 12288 * 2 + 256, st[g][0]>>>(src[g], D, N, g, size, size); continue; }
            if (mode == 7) { push_bulk<32768, 4><<<ctas, 32, 32768 * 4 + 256, st[g][0]>>>(src[g], D, N, g, size, size); continue; }
            if (mode >= 4) {
              push_all_kernel<<<ctas, 256, 0, st[g][0]>>>((const int4*)src[g], D, N, g, size / 16, size, mode == 5);
              continue;
            }
            for (int q = 0; q < N; ++q) {
              if (q == g) continue;
              if (mode == 0) CK(cudaMemcpyAsync(dst[g] + q * size, src[q], size, cudaMemcpyDefault, st[g][q]));
              if (mode == 1) CK(cudaMemcpyAsync(dst[q] + g * size, src[g], size, cudaMemcpyDefault, st[g][q]));
              const int per = ctas / (N - 1) > 0 ? ctas / (N - 1) : 1;
              if (mode == 2) copy_kernel<<<per, 512, 0, st[g][q]>>>((const int4*)src[q], (int4*)(dst[g] + q * size), size / 16);
              if (mode == 3) copy_kernel<<<per, 512, 0, st[g][q]>>>((const int4*)src[g], (int4*)(dst[q] + g * size), size / 16);
            }
          }
          for (int g = 0; g < N; ++g) { CK(cudaSetDevice(g)); CK(cudaDeviceSynchronize()); }
        };
        run(); run();
        const int it = 10;
        auto t0 = std::chrono::high_resolution_clock::now();
        for (int k = 0; k < it; ++k) run();
        auto t1 = std::chrono::high_resolution_clock::now();
        const double s = std::chrono::duration<double>(t1 - t0).count() / it;
        printf("N=%d shard=%4zu MB %s ctas=%3d: %6.0f GB/s incoming per GPU (%.3f ms)\n", N, size >> 20, names[mode],
               mode < 2 ? 0 : ctas, (N - 1) * (double)size / s / 1e9, s * 1e3);
        fflush(stdout);
      }
    }
    for (int g = 0; g < N; ++g) {
      CK(cudaSetDevice(g));
      CK(cudaFree(src[g]));
      CK(cudaFree(dst[g]));
      for (int q = 0; q < N; ++q) CK(cudaStreamDestroy(st[g][q]));
    }
  }
  return 0;
}
