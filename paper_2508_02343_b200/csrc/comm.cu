// comm.cu -- N-sharding support: layout of the all-gathered BF16 shards and the
// NCCL binding (loaded at run time; the torch-bundled libnccl.so.2 is reused
// when torch already loaded it).  DESIGN.md "Multi-GPU".
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstdint>
#include <cstdio>
#include <mutex>

#include "internal.h"

namespace mmx {
namespace {

// stage [G][M][Ns] (BF16) -> y [M][ldy], 16-byte vectors (Ns % 8 == 0).
__global__ void gather_layout_kernel(const uint4* __restrict__ stage, int G, int64_t M, int64_t Ns8,
                                     uint16_t* __restrict__ y, int64_t ldy) {
  const int64_t total = (int64_t)G * M * Ns8;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c8 = i % Ns8;
    const int64_t m = (i / Ns8) % M;
    const int64_t g = i / (Ns8 * M);
    *reinterpret_cast<uint4*>(y + m * ldy + (g * Ns8 + c8) * 8) = __ldcs(stage + i);
  }
}

// Flag barrier of a peer window (NEXT F1): thread j signals "rank `rank` is done" in
// rank j's flag array (system-scope release, after a system fence so the preceding
// GEMM's peer stores are performed first), then waits until rank j's flag in this
// rank's array reaches `epoch` (system-scope acquire).  timeout_ns == 0 waits forever
// (NCCL's behaviour: a legitimately slow rank must not kill the job); otherwise a
// peer that never arrives makes the waiting thread record (missing rank + 1) in this
// rank's error word (flag slot kPeerErrSlot, read by mm_peer_window_error) and return
// -- no trap, so the context stays usable.
__global__ void peer_barrier_kernel(PeerFlags fl, int rank, int world, uint32_t epoch, uint64_t timeout_ns) {
  const int j = threadIdx.x;
  if (j >= world) return;
  __threadfence_system();
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(fl.f[j] + rank), "r"(epoch) : "memory");
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(fl.f[rank] + j) : "memory");
    if ((int32_t)(v - epoch) >= 0) break;
    if (timeout_ns) {
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > timeout_ns) {
        atomicCAS(fl.f[rank] + kPeerErrSlot, 0u, (uint32_t)(j + 1));
        return;
      }
    }
    __nanosleep(100);
  }
}

// NVLS barrier (NEXT F1 over NVLink SHARP): one system-scope release-add through the
// multicast view increments word 0 of EVERY rank's flag array; each rank then waits for
// its own copy to reach world * epoch.  The preceding GEMM's multimem stores are
// performed first (kernel boundary + system fence + release).
__global__ void mc_barrier_kernel(uint32_t* flags_mc, uint32_t* flags_local, int world, uint32_t epoch,
                                  uint64_t timeout_ns) {
  if (threadIdx.x != 0) return;
  __threadfence_system();
  asm volatile("multimem.red.release.sys.global.add.u32 [%0], %1;" ::"l"(flags_mc), "r"(1u) : "memory");
  const uint32_t target = (uint32_t)world * epoch;
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags_local) : "memory");
    if ((int32_t)(v - target) >= 0) break;
    if (timeout_ns) {
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > timeout_ns) {
        atomicCAS(flags_local + kPeerErrSlot, 0u, 0xFFFFu);   // some rank(s) missing
        return;
      }
    }
    __nanosleep(100);
  }
}

}  // namespace

cudaError_t launch_mc_barrier(uint32_t* flags_mc, uint32_t* flags_local, int world, uint32_t epoch,
                              uint64_t timeout_ns, cudaStream_t s, int64_t* launches) {
  mc_barrier_kernel<<<1, 32, 0, s>>>(flags_mc, flags_local, world, epoch, timeout_ns);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_peer_barrier(const PeerFlags& fl, int rank, int world, uint32_t epoch, uint64_t timeout_ns,
                                cudaStream_t s, int64_t* launches) {
  peer_barrier_kernel<<<1, 32, 0, s>>>(fl, rank, world, epoch, timeout_ns);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_gather_layout(const uint16_t* stage, int G, int64_t M, int64_t Ns, uint16_t* y,
                                 int64_t ldy, cudaStream_t s, int64_t* launches) {
  const int64_t total = (int64_t)G * M * (Ns / 8);
  if (total == 0) return cudaSuccess;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 8 * sm_count()) blocks = 8 * sm_count();
  gather_layout_kernel<<<(unsigned)blocks, 256, 0, s>>>(reinterpret_cast<const uint4*>(stage), G, M, Ns / 8, y,
                                                        ldy);
  if (launches) ++*launches;
  return cudaGetLastError();
}

// ---- NCCL, resolved with dlopen ------------------------------------------------
const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, []() {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.getUniqueId = reinterpret_cast<decltype(&ncclGetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    api.commInitRank = reinterpret_cast<decltype(&ncclCommInitRank)>(dlsym(h, "ncclCommInitRank"));
    api.commDestroy = reinterpret_cast<decltype(&ncclCommDestroy)>(dlsym(h, "ncclCommDestroy"));
    api.allGather = reinterpret_cast<decltype(&ncclAllGather)>(dlsym(h, "ncclAllGather"));
    api.errStr = reinterpret_cast<decltype(&ncclGetErrorString)>(dlsym(h, "ncclGetErrorString"));
    api.ok = api.getUniqueId && api.commInitRank && api.commDestroy && api.allGather && api.errStr;
  });
  return api;
}

}  // namespace mmx
