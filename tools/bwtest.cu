// bwtest.cu -- read-bandwidth microbenchmark for the reorder-quantize load phase
// (tuning aid, not part of the library).  Reads a 2048 x 4096 BF16 matrix
// (16.8 MB) with different load strategies; each kernel XOR-reduces what it
// read into one word per CTA so the loads cannot be elided.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bwtest tools/bwtest.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// (1) all threads, LDG.128 evict-first, U loads in flight per thread
template <int U>
__global__ void k_ldg(const uint4* __restrict__ x, size_t n16, uint32_t* out) {
  uint32_t acc = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += stride * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = (i + u * stride < n16) ? __ldcs(x + i + u * stride) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678u) out[blockIdx.x] = acc;
}

// (2) one thread per CTA issues 1-D bulk copies (cp.async.bulk) of `chunk` bytes
// into a ring of `stages` buffers; consumers touch one word per 16 B.
__global__ void k_bulk(const uint8_t* __restrict__ x, size_t bytes, int chunk, int stages, uint32_t* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)stages * chunk);
  uint64_t* empty = full + stages;
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&empty[i])), "r"((int)(blockDim.x / 32 - 1)));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const size_t nchunks = bytes / chunk;
  const int64_t mine = (nchunks - blockIdx.x + gridDim.x - 1) / gridDim.x;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) {
    if (lane == 0) {
      for (int64_t i = 0; i < mine; ++i) {
        const int s = int(i % stages);
        const uint32_t ph = uint32_t(i / stages) & 1;
        uint32_t ok = 0;
        while (!ok)
          asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                       : "=r"(ok) : "r"(smem_u32(&empty[s])), "r"(ph ^ 1));
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(chunk));
        const uint8_t* src = x + (blockIdx.x + i * gridDim.x) * (size_t)chunk;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(smem_u32(sm + (size_t)s * chunk)), "l"(src), "r"(chunk), "r"(smem_u32(&full[s])) : "memory");
      }
    }
    return;
  }
  uint32_t acc = 0;
  for (int64_t i = 0; i < mine; ++i) {
    const int s = int(i % stages);
    const uint32_t ph = uint32_t(i / stages) & 1;
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                   : "=r"(ok) : "r"(smem_u32(&full[s])), "r"(ph));
    const uint32_t* b = reinterpret_cast<const uint32_t*>(sm + (size_t)s * chunk);
    for (int j = threadIdx.x - 32; j < chunk / 16; j += blockDim.x - 32) acc ^= b[4 * j];
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])));
  }
  if (acc == 0x12345678u) out[blockIdx.x] = acc;
}

int main() {
  const size_t bytes = 2048ull * 4096 * 2;
  const int NB = 12;  // rotate 12 buffers (> L2)
  std::vector<uint8_t*> xs(NB);
  for (auto& p : xs) { CK(cudaMalloc(&p, bytes)); CK(cudaMemset(p, 1, bytes)); }
  uint32_t* out;
  CK(cudaMalloc(&out, 1 << 20));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, auto launch) {
    for (int i = 0; i < 5; ++i) launch(xs[i % NB]);
    cudaDeviceSynchronize();
    const int reps = 60;
    cudaEventRecord(e0);
    for (int i = 0; i < reps; ++i) launch(xs[i % NB]);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double us = ms * 1e3 / reps;
    printf("%-40s %7.2f us  %6.0f GB/s  err=%s\n", name, us, bytes / us / 1e3, cudaGetErrorString(cudaGetLastError()));
  };
  for (int bpsm : {1, 2, 4, 8}) {
    for (int thr : {256, 512}) {
      char nm[64];
      snprintf(nm, 64, "ldg U=4 grid=%dx%d thr=%d", sms, bpsm, thr);
      run(nm, [&](uint8_t* x) { k_ldg<4><<<sms * bpsm, thr>>>((const uint4*)x, bytes / 16, out); });
    }
  }
  for (int chunk : {8192, 16384, 32768}) {
    for (int stages : {4, 6}) {
      const size_t smem = (size_t)stages * chunk + 2 * stages * 8;
      if (smem > 220 * 1024) continue;
      cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      char nm[64];
      snprintf(nm, 64, "bulk chunk=%d stages=%d", chunk, stages);
      run(nm, [&](uint8_t* x) { k_bulk<<<sms, 256, smem>>>(x, bytes, chunk, stages, out); });
    }
  }
  return 0;
}
