// calib.cu -- per-channel calibration statistics for mm_calibrate_thresholds
// (§3.1: Eq. 6 needs max|P_n| per channel group, Eq. 7 the channel-
// wise absolute mean M_k = (1/L) sum_i |X_ik|; §4.1: 32 x 2048 tokens).
//
// One streaming pass over X[L, K] (HBM-bound, offline):
//   * exact per-channel max|x| as an integer max over the BF16 magnitude bits;
//   * per-channel sum of |x| accumulated in double-double (TwoSum), per
//     row-split partials combined in a fixed order, then one compensated
//     division by L -- the correctly rounded fp64 mean in all but
//     astronomically rare cases (reading R26).
#include <cuda_runtime.h>
#include <cmath>
#include <cstdint>
#include <cstring>

#include "internal.h"

namespace mmx {
namespace {

constexpr int kColsPerThread = 2;   // bf16x2 loads
constexpr int kThreadsX = 64;       // 128 channels per block
constexpr int kRowGroups = 4;       // warps-of-rows per block (blockDim.y)

struct DD { double hi, lo; };

__device__ __forceinline__ void dd_add(DD& a, double v) {
  double s = a.hi + v;
  double bb = s - a.hi;
  double err = (a.hi - (s - bb)) + (v - bb);
  a.hi = s;
  a.lo += err;
}
__device__ __forceinline__ DD dd_add_dd(DD a, DD b) {
  double s = a.hi + b.hi;
  double bb = s - a.hi;
  double err = (a.hi - (s - bb)) + (b.hi - bb);
  err += a.lo + b.lo;
  double hi = s + err;
  double lo = err - (hi - s);
  return {hi, lo};
}

struct Partial { double hi, lo; uint32_t mx; uint32_t pad; };

__global__ void calib_pass(const uint16_t* __restrict__ x, int64_t L, int64_t ldx, int K,
                           int splits, Partial* __restrict__ part) {
  const int col = (blockIdx.x * kThreadsX + threadIdx.x) * kColsPerThread;
  const int split = blockIdx.y;
  const int64_t rows_per = (L + splits - 1) / splits;
  const int64_t rbeg = split * rows_per;
  const int64_t rend = min(L, rbeg + rows_per);
  DD s0{0, 0}, s1{0, 0};
  uint32_t m0 = 0, m1 = 0;
  if (col < K) {
    for (int64_t r = rbeg + threadIdx.y; r < rend; r += kRowGroups) {
      uint32_t v = __ldcs(reinterpret_cast<const uint32_t*>(x + r * ldx + col));
      uint32_t a0 = v & 0x7FFFu, a1 = (v >> 16) & 0x7FFFu;
      m0 = max(m0, a0);
      m1 = max(m1, a1);
      dd_add(s0, (double)__uint_as_float(a0 << 16));
      dd_add(s1, (double)__uint_as_float(a1 << 16));
    }
  }
  __shared__ Partial sh[kRowGroups][kThreadsX][2];
  sh[threadIdx.y][threadIdx.x][0] = {s0.hi, s0.lo, m0, 0};
  sh[threadIdx.y][threadIdx.x][1] = {s1.hi, s1.lo, m1, 0};
  __syncthreads();
  if (threadIdx.y == 0 && col < K) {
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      DD acc{sh[0][threadIdx.x][c].hi, sh[0][threadIdx.x][c].lo};
      uint32_t m = sh[0][threadIdx.x][c].mx;
      for (int g = 1; g < kRowGroups; ++g) {
        acc = dd_add_dd(acc, DD{sh[g][threadIdx.x][c].hi, sh[g][threadIdx.x][c].lo});
        m = max(m, sh[g][threadIdx.x][c].mx);
      }
      part[(int64_t)split * K + col + c] = {acc.hi, acc.lo, m, 0};
    }
  }
}

__global__ void calib_finalize(const Partial* __restrict__ part, int splits, int K, int64_t L,
                               double* __restrict__ chmax, double* __restrict__ chmean) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  DD acc{0, 0};
  uint32_t m = 0;
  for (int s = 0; s < splits; ++s) {
    Partial p = part[(int64_t)s * K + k];
    acc = dd_add_dd(acc, DD{p.hi, p.lo});
    m = max(m, p.mx);
  }
  chmax[k] = (double)__uint_as_float(m << 16);
  // (hi + lo) / L with one compensated step: q1 = hi/L, r = (hi - q1 L) + lo.
  const double dl = (double)L;
  double q1 = acc.hi / dl;
  double r = fma(-q1, dl, acc.hi) + acc.lo;
  chmean[k] = q1 + r / dl;
}

// Streaming calibration: add one batch's split partials into the running state
// (per channel: double-double |x| sum and max |x| bits; header: total rows).
__global__ void calib_merge(const Partial* __restrict__ part, int splits, int K, int64_t L,
                            Partial* __restrict__ state, int64_t* __restrict__ rows) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k == 0) *rows += L;
  if (k >= K) return;
  DD acc{state[k].hi, state[k].lo};
  uint32_t m = state[k].mx;
  for (int s = 0; s < splits; ++s) {
    Partial p = part[(int64_t)s * K + k];
    acc = dd_add_dd(acc, DD{p.hi, p.lo});
    m = max(m, p.mx);
  }
  state[k] = {acc.hi, acc.lo, m, 0};
}

int calib_splits(int64_t L, int K) {
  const int colblocks = (K + kThreadsX * kColsPerThread - 1) / (kThreadsX * kColsPerThread);
  int want = (4 * sm_count() + colblocks - 1) / colblocks;
  int64_t max_splits = (L + 63) / 64;  // at least 64 rows per split
  if (want > max_splits) want = (int)max_splits;
  if (want < 1) want = 1;
  return want;
}

}  // namespace

size_t calib_workspace_bytes(int64_t L, int K) {
  return (size_t)calib_splits(L, K) * (size_t)K * sizeof(Partial);
}

cudaError_t launch_calib_stats(const uint16_t* x, int64_t L, int64_t ldx, int K, void* ws,
                               double* d_chmax, double* d_chmean, cudaStream_t s,
                               int64_t* launches) {
  const int splits = calib_splits(L, K);
  dim3 grid((K + kThreadsX * kColsPerThread - 1) / (kThreadsX * kColsPerThread), splits);
  dim3 block(kThreadsX, kRowGroups);
  calib_pass<<<grid, block, 0, s>>>(x, L, ldx, K, splits, reinterpret_cast<Partial*>(ws));
  if (launches) ++*launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  calib_finalize<<<(K + 255) / 256, 256, 0, s>>>(reinterpret_cast<const Partial*>(ws), splits, K,
                                                 L, d_chmax, d_chmean);
  if (launches) ++*launches;
  return cudaGetLastError();
}

size_t calib_state_bytes(int K) { return 256 + (size_t)K * sizeof(Partial); }

cudaError_t launch_calib_accumulate(const uint16_t* x, int64_t L, int64_t ldx, int K, void* ws, void* state,
                                    cudaStream_t s, int64_t* launches) {
  const int splits = calib_splits(L, K);
  dim3 grid((K + kThreadsX * kColsPerThread - 1) / (kThreadsX * kColsPerThread), splits);
  dim3 block(kThreadsX, kRowGroups);
  calib_pass<<<grid, block, 0, s>>>(x, L, ldx, K, splits, reinterpret_cast<Partial*>(ws));
  if (launches) ++*launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  uint8_t* st = static_cast<uint8_t*>(state);
  calib_merge<<<(K + 255) / 256, 256, 0, s>>>(reinterpret_cast<const Partial*>(ws), splits, K, L,
                                              reinterpret_cast<Partial*>(st + 256), reinterpret_cast<int64_t*>(st));
  if (launches) ++*launches;
  return cudaGetLastError();
}

void calib_state_to_stats(const void* h_state, int K, double* chmax, double* chmean, int64_t* rows) {
  const uint8_t* st = static_cast<const uint8_t*>(h_state);
  const int64_t L = *reinterpret_cast<const int64_t*>(st);
  const Partial* p = reinterpret_cast<const Partial*>(st + 256);
  const double dl = (double)L;
  for (int k = 0; k < K; ++k) {
    uint32_t b = p[k].mx << 16;
    float f;
    memcpy(&f, &b, 4);
    chmax[k] = (double)f;
    // the same compensated division as calib_finalize (fma is exact-rounded on host too)
    const double q1 = p[k].hi / dl;
    const double r = std::fma(-q1, dl, p[k].hi) + p[k].lo;
    chmean[k] = L > 0 ? q1 + r / dl : 0.0;
  }
  *rows = L;
}

}  // namespace mmx
