// NVLink SHARP probe (development): p processes (one per GPU, rank from argv) build one multicast
// object (POSIX-fd handle: rank 0 exports, the others take the fd with pidfd_getfd or over a Unix
// socket with SCM_RIGHTS), bind a device buffer each, fill it with bf16 (rank + 1), and reduce it
// through the switch with multimem.ld_reduce; prints correctness and the reduce bandwidth.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o nvls_probe nvls_probe.cu -lcuda
//   for r in 0 1; do ./nvls_probe $r 2 /tmp/nvls & done; wait
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <sys/socket.h>
#include <sys/stat.h>
#include <sys/syscall.h>
#include <sys/un.h>
#include <unistd.h>

#include <cerrno>
#include <cstring>
#include <thread>

#include <cstdio>
#include <cstdlib>
#include <string>

#define CK(x)                                                                       \
  do {                                                                              \
    CUresult r_ = (x);                                                              \
    if (r_ != CUDA_SUCCESS) {                                                       \
      const char* s_ = nullptr;                                                     \
      cuGetErrorString(r_, &s_);                                                    \
      std::fprintf(stderr, "rank %d: %s failed: %s\n", g_rank, #x, s_ ? s_ : "?");  \
      std::exit(1);                                                                 \
    }                                                                               \
  } while (0)

static int g_rank = 0;

static void touch(const std::string& p) {
  FILE* f = std::fopen(p.c_str(), "w");
  if (f) std::fclose(f);
}
static void wait_file(const std::string& p) {
  struct stat st;
  for (int i = 0; i < 600000 && stat(p.c_str(), &st) != 0; ++i) usleep(100);
}
static void barrier(const std::string& dir, const char* tag, int rank, int world) {
  touch(dir + "/" + tag + "_" + std::to_string(rank));
  for (int q = 0; q < world; ++q) wait_file(dir + "/" + tag + "_" + std::to_string(q));
}

__global__ void fill_kernel(__nv_bfloat16* p, size_t n, float v) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    p[i] = __float2bfloat16(v);
}

// out[i] = sum over ranks of mc[i] (8 bf16 per thread per iteration, fp32 accumulation in the switch)
__global__ void reduce_kernel(const __nv_bfloat16* mc, float* out, size_t n8) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n8; i += size_t(gridDim.x) * blockDim.x) {
    uint32_t a, b, c, d;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0, %1, %2, %3}, [%4];"
                 : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
                 : "l"(mc + i * 8)
                 : "memory");
    const uint32_t w[4] = {a, b, c, d};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const __nv_bfloat162 h = *reinterpret_cast<const __nv_bfloat162*>(&w[e]);
      out[i * 8 + 2 * e] = __bfloat162float(h.x);
      out[i * 8 + 2 * e + 1] = __bfloat162float(h.y);
    }
  }
}

int main(int argc, char** argv) {
  if (argc < 4) return 2;
  const int rank = std::atoi(argv[1]), world = std::atoi(argv[2]);
  const std::string dir = argv[3];
  g_rank = rank;
  CK(cuInit(0));
  CUdevice dev;
  CK(cuDeviceGet(&dev, rank));
  CUcontext ctx;
  CK(cuDevicePrimaryCtxRetain(&ctx, dev));
  CK(cuCtxSetCurrent(ctx));
  size_t size = size_t(256) << 20;
  CUmulticastObjectProp mp = {};
  mp.numDevices = world;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  mp.size = size;
  size_t gran = 0;
  CK(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  size = (size + gran - 1) / gran * gran;
  mp.size = size;
  CUmemGenericAllocationHandle mc;
  const std::string hfile = dir + "/handle";
  const std::string sock_name = "nvls_probe_" + std::to_string(getppid());
  auto sock_addr = [&](sockaddr_un& a) {
    std::memset(&a, 0, sizeof(a));
    a.sun_family = AF_UNIX;
    std::memcpy(a.sun_path + 1, sock_name.data(), sock_name.size());  // abstract namespace
    return socklen_t(offsetof(sockaddr_un, sun_path) + 1 + sock_name.size());
  };
  std::thread server;
  if (rank == 0) {
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    CK(cuMulticastCreate(&mc, &mp));
    int fd = -1;
    CK(cuMemExportToShareableHandle(&fd, mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
    int ls = socket(AF_UNIX, SOCK_STREAM, 0);
    sockaddr_un a;
    const socklen_t al = sock_addr(a);
    if (bind(ls, reinterpret_cast<sockaddr*>(&a), al) != 0 || listen(ls, 16) != 0)
      std::fprintf(stderr, "rank 0: socket bind/listen failed: %s\n", std::strerror(errno));
    server = std::thread([=] {
      for (int q = 1; q < world; ++q) {
        int cs = accept(ls, nullptr, nullptr);
        char byte = 0;
        iovec io{&byte, 1};
        char cbuf[CMSG_SPACE(sizeof(int))] = {};
        msghdr m{};
        m.msg_iov = &io;
        m.msg_iovlen = 1;
        m.msg_control = cbuf;
        m.msg_controllen = sizeof(cbuf);
        cmsghdr* c = CMSG_FIRSTHDR(&m);
        c->cmsg_level = SOL_SOCKET;
        c->cmsg_type = SCM_RIGHTS;
        c->cmsg_len = CMSG_LEN(sizeof(int));
        std::memcpy(CMSG_DATA(c), &fd, sizeof(int));
        sendmsg(cs, &m, 0);
        close(cs);
      }
      close(ls);
    });
    FILE* f = std::fopen((hfile + ".tmp").c_str(), "w");
    std::fprintf(f, "%d %d\n", int(getpid()), fd);
    std::fclose(f);
    std::rename((hfile + ".tmp").c_str(), hfile.c_str());
  } else {
    wait_file(hfile);
    int pid = 0, rfd = -1;
    FILE* f = std::fopen(hfile.c_str(), "r");
    if (std::fscanf(f, "%d %d", &pid, &rfd) != 2) return 3;
    std::fclose(f);
    int fd = -1;
    const long pfd = syscall(SYS_pidfd_open, pid, 0);
    if (pfd >= 0) fd = int(syscall(SYS_pidfd_getfd, pfd, rfd, 0));
    std::printf("rank %d: pidfd_open %ld pidfd_getfd %d (%s)\n", rank, pfd, fd, fd < 0 ? std::strerror(errno) : "ok");
    if (fd < 0) {  // Unix socket with SCM_RIGHTS
      int cs = socket(AF_UNIX, SOCK_STREAM, 0);
      sockaddr_un a;
      const socklen_t al = sock_addr(a);
      for (int i = 0; i < 1000 && connect(cs, reinterpret_cast<sockaddr*>(&a), al) != 0; ++i) usleep(1000);
      char byte = 0;
      iovec io{&byte, 1};
      char cbuf[CMSG_SPACE(sizeof(int))] = {};
      msghdr m{};
      m.msg_iov = &io;
      m.msg_iovlen = 1;
      m.msg_control = cbuf;
      m.msg_controllen = sizeof(cbuf);
      if (recvmsg(cs, &m, 0) >= 0) {
        cmsghdr* c = CMSG_FIRSTHDR(&m);
        if (c && c->cmsg_type == SCM_RIGHTS) std::memcpy(&fd, CMSG_DATA(c), sizeof(int));
      }
      close(cs);
      std::printf("rank %d: SCM_RIGHTS fd %d\n", rank, fd);
    }
    CK(cuMemImportFromShareableHandle(&mc, reinterpret_cast<void*>(static_cast<uintptr_t>(fd)),
                                      CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR));
  }
  CK(cuMulticastAddDevice(mc, dev));
  barrier(dir, "added", rank, world);
  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = rank;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t agran = 0;
  CK(cuMemGetAllocationGranularity(&agran, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  CUmemGenericAllocationHandle phys;
  std::printf("rank %d: multicast granularity %zu, allocation granularity %zu, size %zu\n", rank, gran, agran, size);
  CK(cuMemCreate(&phys, size, &ap, 0));
  CK(cuMulticastBindMem(mc, 0, phys, 0, size, 0));
  CUdeviceptr uc = 0, mcva = 0;
  CUmemAccessDesc acc = {};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = rank;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemAddressReserve(&uc, size, gran, 0, 0));
  CK(cuMemMap(uc, size, 0, phys, 0));
  CK(cuMemSetAccess(uc, size, &acc, 1));
  CK(cuMemAddressReserve(&mcva, size, gran, 0, 0));
  CK(cuMemMap(mcva, size, 0, mc, 0));
  CK(cuMemSetAccess(mcva, size, &acc, 1));
  const size_t n = size / 2;
  fill_kernel<<<592, 256>>>(reinterpret_cast<__nv_bfloat16*>(uc), n, float(rank + 1));
  cudaDeviceSynchronize();
  barrier(dir, "filled", rank, world);
  float* out = nullptr;
  cudaMalloc(&out, n / world * sizeof(float));
  const size_t n8 = n / world / 8;  // this rank's slice
  const __nv_bfloat16* slice = reinterpret_cast<const __nv_bfloat16*>(mcva) + size_t(rank) * (n / world);
  reduce_kernel<<<592, 256>>>(slice, out, n8);
  cudaError_t e = cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int it = 0; it < 10; ++it) reduce_kernel<<<592, 256>>>(slice, out, n8);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  float h[4];
  cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
  const float want = world * (world + 1) / 2.0f;
  std::printf("rank %d: %s, out[0..3] = %g %g %g %g (want %g), slice %zu MB reduced in %.3f ms = %.1f GB/s of slice\n",
              rank, cudaGetErrorString(e), h[0], h[1], h[2], h[3], want, n / world * 2 >> 20, ms / 10,
              double(n / world * 2) / (ms / 10 * 1e-3) / 1e9);
  barrier(dir, "done", rank, world);
  if (server.joinable()) server.join();
  return h[0] == want ? 0 : 4;
}
