// wstream.cu -- does the decode GEMM's W access pattern, not the kernel, bound its
// W stream?  (tuning aid, not part of the library.)
// Streams one quantized-weight-sized matrix (4096 rows x 9120 B = 37 MB, the decode
// down_proj W) once through shared memory with 128 CTAs x an 8-stage ring, like the
// small-M kernel (32 row tiles x 4 K splits), two ways:
//   (a) row-major: 2-D TMA boxes of 128 rows x 128 B (128 pieces one pitch apart),
//   (b) tile-contiguous: the same bytes as 16 KB 1-D bulk copies.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o wstream tools/wstream.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)
constexpr int kRows = 4096, kPitch = 9120, kStages = 8, kBox = 16384, kSplits = 4;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint32_t bar, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                 : "=r"(ok) : "r"(bar), "r"(ph));
}

// CTA b: row tile b / kSplits, K-block range split b % kSplits.  tiled = 0: TMA boxes of
// the row-major matrix; 1: 16 KB contiguous blocks of a [tile][kblock][128 x 128 B] copy.
__global__ void k_stream(const __grid_constant__ CUtensorMap tm, const uint8_t* __restrict__ tiled_src, int tiled,
                         uint32_t* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + kStages * kBox);
  uint64_t* empty = full + kStages;
  const int nkb = kPitch / 128;                        // 71 K-blocks of 128 B (9088 B; tail ignored)
  const int tile = blockIdx.x / kSplits, split = blockIdx.x % kSplits;
  const int kb0 = split * nkb / kSplits, kb1 = (split + 1) * nkb / kSplits;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&empty[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int kb = kb0; kb < kb1; ++kb) {
      const int i = kb - kb0, s = i % kStages;
      wait(smem_u32(&empty[s]), ((i / kStages) & 1) ^ 1);
      const uint32_t fb = smem_u32(&full[s]), dst = smem_u32(sm + s * kBox);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(kBox));
      if (tiled) {
        const uint8_t* src = tiled_src + ((size_t)tile * nkb + kb) * kBox;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(dst), "l"(src), "r"(kBox), "r"(fb) : "memory");
      } else {
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                     " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst), "l"(reinterpret_cast<uint64_t>(&tm)),
                     "r"(kb * 128), "r"(tile * 128), "r"(fb) : "memory");
      }
    }
  } else if (threadIdx.x == 32) {
    uint32_t acc = 0;
    for (int kb = kb0; kb < kb1; ++kb) {
      const int i = kb - kb0, s = i % kStages;
      wait(smem_u32(&full[s]), (i / kStages) & 1);
      acc ^= *reinterpret_cast<const uint32_t*>(sm + s * kBox);
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])));
    }
    if (acc == 0x12345678u) out[blockIdx.x] = acc;
  }
}

int main() {
  const size_t bytes = (size_t)kRows * kPitch;
  const int NB = 6;   // rotate 6 buffers of each kind (> L2)
  std::vector<uint8_t*> rm(NB), tl(NB);
  std::vector<CUtensorMap> maps(NB);
  for (int b = 0; b < NB; ++b) {
    CK(cudaMalloc(&rm[b], bytes)); CK(cudaMemset(rm[b], 1, bytes));
    CK(cudaMalloc(&tl[b], bytes)); CK(cudaMemset(tl[b], 1, bytes));
    cuuint64_t dims[2] = {(cuuint64_t)kPitch, (cuuint64_t)kRows};
    cuuint64_t strides[1] = {(cuuint64_t)kPitch};
    cuuint32_t box[2] = {128, 128}, estr[2] = {1, 1};
    if (cuTensorMapEncodeTiled(&maps[b], CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, rm[b], dims, strides, box, estr,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      printf("tensor map encode failed\n");
      return 1;
    }
  }
  uint32_t* out;
  CK(cudaMalloc(&out, 1 << 16));
  const size_t smem = kStages * kBox + 2 * kStages * 8 + 1024;
  CK(cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int grid = (kRows / 128) * kSplits;
  const double moved = (double)kRows * (kPitch / 128) * 128;
  for (int tiled : {0, 1, 0, 1}) {
    for (int i = 0; i < 4; ++i) k_stream<<<grid, 64, smem>>>(maps[i % NB], tl[i % NB], tiled, out);
    CK(cudaDeviceSynchronize());
    const int reps = 30;
    cudaEventRecord(e0);
    for (int i = 0; i < reps; ++i) k_stream<<<grid, 64, smem>>>(maps[i % NB], tl[i % NB], tiled, out);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double us = ms * 1e3 / reps;
    printf("%-48s %7.2f us  %6.0f GB/s\n", tiled ? "tile-contiguous 16 KB bulk copies" : "row-major 128 x 128 B TMA boxes",
           us, moved / us / 1e3);
  }
  return 0;
}
