// rq.cu -- fused reorder-and-quantize of BF16 rows into MXFP4 / MXFP6 / MXFP8
// channel segments (§3.2 "Quantization Kernel", line 151; Fig. 6
// caption line 148; Eq. 1 lines 40-45), sm_100a.
//
// HBM-bound streaming kernel.  Persistent CTAs, warp-specialised:
//   * 4 producer warps stream R rows at a time from HBM with 128-bit loads and
//     write them into shared memory "row-interleaved": smem slot p holds the R
//     BF16 values of channel p (R = 4: 8-byte slots), XOR-swizzled so the
//     128-bit -> slot transposition stores are bank-conflict free.  Two slots
//     (double buffer) overlap the next tile's loads with this tile's work.
//   * 4 consumer warps own one 32-channel block of the reordered row each:
//     the gather x_r[j] = X[perm[j]] is a single 64-bit shared load per channel
//     that fetches all R rows at once (R-fold fewer random smem accesses than a
//     per-row gather); block amax is an integer max over |bf16| bits; the E8M0
//     exponent is integer arithmetic on the BF16 exponent field (no log2f); the
//     scaled value x * 2^-e is exact (power of two, no FTZ); the element code is
//     produced by the hardware cvt.rn.satfinite.{e2m1x2,e3m2x2,e2m3x2,e4m3x2,
//     e5m2x2}.f32 (round-to-nearest-even, saturating, sign-preserving); codes are
//     packed (FP4 two per byte, FP6 a tight LSB-first bit stream, FP8 bytes) and
//     written with 64/128-bit stores; the scale byte goes straight into the
//     128x4 scale-factor atom the GEMM's tcgen05.cp consumes.
//   Segment padding columns (up to a multiple of 128) and scale rows up to a
//   multiple of 128 are written as zero on every call.
#include <cuda_runtime.h>
#include <cstdint>

#include "internal.h"

namespace mmx {
namespace {

constexpr int kProdThreads = 128;
constexpr int kConsThreads = 128;
constexpr int kThreads = kProdThreads + kConsThreads;

__device__ __forceinline__ void named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// Slot swizzle: slot(p) = p ^ ((p >> S) & (W - 1)) with W slots per 128-byte line.
template <int R> struct SlotT;
template <> struct SlotT<1> { using T = uint16_t; static constexpr int W = 1, S = 0; };
template <> struct SlotT<2> { using T = uint32_t; static constexpr int W = 32, S = 5; };
template <> struct SlotT<4> { using T = uint2; static constexpr int W = 16, S = 4; };

template <int R>
__device__ __forceinline__ uint32_t swz(uint32_t p) {
  if constexpr (R == 1) return p;
  else return p ^ ((p >> SlotT<R>::S) & (SlotT<R>::W - 1));
}

template <int R>
__device__ __forceinline__ uint32_t row_bits(const typename SlotT<R>::T& v, int rho) {
  if constexpr (R == 1) return v;
  else if constexpr (R == 2) return (v >> (16 * rho)) & 0xFFFFu;
  else return ((rho < 2 ? v.x : v.y) >> (16 * (rho & 1))) & 0xFFFFu;
}

// ---- element conversions (hardware RNE + satfinite) -------------------------
// cvt.*x2.f32 d, a, b puts a in the upper half of d and b in the lower half.
__device__ __forceinline__ uint32_t cvt_fp8x2(float lo, float hi, int fmt) {
  uint16_t r;
  if (fmt == F_E4M3)
    asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
  else
    asm("cvt.rn.satfinite.e5m2x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ uint32_t cvt_fp6x2(float lo, float hi, int fmt) {
  uint16_t r;
  if (fmt == F_E3M2)
    asm("cvt.rn.satfinite.e3m2x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
  else
    asm("cvt.rn.satfinite.e2m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
  return r;  // byte0 = code(lo) (6 bits), byte1 = code(hi)
}
// Four E2M1 codes -> one 16-bit value, element 0 in the lowest nibble.
__device__ __forceinline__ uint32_t cvt_fp4x4(float a0, float a1, float a2, float a3) {
  uint32_t r;
  asm("{\n\t.reg .b8 b0, b1;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b0, %2, %1;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b1, %4, %3;\n\t"
      "mov.b32 %0, {b0, b1, 0, 0};\n\t}"
      : "=r"(r) : "f"(a0), "f"(a1), "f"(a2), "f"(a3));
  return r;
}

__device__ __forceinline__ float bf16_to_f32(uint32_t b) { return __uint_as_float(b << 16); }

// Byte offset of scale (r, kb) inside the 128x4-atom layout of a segment with
// kp128 = Kp/128 atoms per 128-row group.
__device__ __forceinline__ int64_t sf_offset(int64_t r, int kb, int kp128) {
  return ((r >> 7) * kp128 + (kb >> 2)) * 512 + (r & 31) * 16 + ((r >> 5) & 3) * 4 + (kb & 3);
}

// Quantize one row's 32-element block `v` (BF16 bits) and store codes+scale.
__device__ __forceinline__ void quantize_store_block(const uint32_t (&v)[32], int g, int fmt,
                                                     int off, uint8_t* codes_row, int kb,
                                                     bool store_codes, uint8_t* sf, int64_t r,
                                                     int kp128) {
  uint32_t amax = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) amax = max(amax, v[i] & 0x7FFFu);
  // e = floor(log2 amax) - off, clamped at -127 (zero / subnormal blocks -> -127).
  int sb = max(int(amax >> 7) - off, 0);          // E8M0 byte = e + 127
  float inv = __uint_as_float(uint32_t(254 - sb) << 23);  // 2^-e exactly
  sf[sf_offset(r, kb, kp128)] = uint8_t(sb);
  if (!store_codes) return;
  if (g == 0) {  // MXFP4: 16 bytes
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t lo = cvt_fp4x4(bf16_to_f32(v[8 * q + 0]) * inv, bf16_to_f32(v[8 * q + 1]) * inv,
                              bf16_to_f32(v[8 * q + 2]) * inv, bf16_to_f32(v[8 * q + 3]) * inv);
      uint32_t hi = cvt_fp4x4(bf16_to_f32(v[8 * q + 4]) * inv, bf16_to_f32(v[8 * q + 5]) * inv,
                              bf16_to_f32(v[8 * q + 6]) * inv, bf16_to_f32(v[8 * q + 7]) * inv);
      w[q] = lo | (hi << 16);
    }
    *reinterpret_cast<uint4*>(codes_row + 16 * kb) = make_uint4(w[0], w[1], w[2], w[3]);
  } else if (g == 1) {  // MXFP6: 24 bytes, LSB-first 6-bit stream
    uint32_t q24[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      uint32_t h0 = cvt_fp6x2(bf16_to_f32(v[4 * q + 0]) * inv, bf16_to_f32(v[4 * q + 1]) * inv, fmt);
      uint32_t h1 = cvt_fp6x2(bf16_to_f32(v[4 * q + 2]) * inv, bf16_to_f32(v[4 * q + 3]) * inv, fmt);
      q24[q] = (h0 & 0x3Fu) | (((h0 >> 8) & 0x3Fu) << 6) | ((h1 & 0x3Fu) << 12) |
               (((h1 >> 8) & 0x3Fu) << 18);
    }
    uint2* dst = reinterpret_cast<uint2*>(codes_row + 24 * kb);
    dst[0] = make_uint2(q24[0] | (q24[1] << 24), (q24[1] >> 8) | (q24[2] << 16));
    dst[1] = make_uint2((q24[2] >> 16) | (q24[3] << 8), q24[4] | (q24[5] << 24));
    dst[2] = make_uint2((q24[5] >> 8) | (q24[6] << 16), (q24[6] >> 16) | (q24[7] << 8));
  } else {  // MXFP8: 32 bytes
    uint32_t w[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      uint32_t lo = cvt_fp8x2(bf16_to_f32(v[4 * q + 0]) * inv, bf16_to_f32(v[4 * q + 1]) * inv, fmt);
      uint32_t hi = cvt_fp8x2(bf16_to_f32(v[4 * q + 2]) * inv, bf16_to_f32(v[4 * q + 3]) * inv, fmt);
      w[q] = lo | (hi << 16);
    }
    uint4* dst = reinterpret_cast<uint4*>(codes_row + 32 * kb);
    dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
    dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
  }
}

template <int R>
__global__ void __launch_bounds__(kThreads, 1)
rq_kernel(const RqArgs a, int64_t rows_pad, int64_t n_tiles) {
  using ST = typename SlotT<R>::T;
  extern __shared__ __align__(128) uint8_t smem[];
  const int K = a.K;
  const int nblk = K / 32;                       // real blocks of the reordered row
  // [gidx: u32 pairs, (K/2) words laid out [i/2][blk]] [slot0][slot1]
  uint32_t* gidx2 = reinterpret_cast<uint32_t*>(smem);
  const size_t gbytes = ((size_t)K * 2 + 127) / 128 * 128;
  ST* buf0 = reinterpret_cast<ST*>(smem + gbytes);
  ST* buf1 = buf0 + K;

  // Gather indices (swizzled smem slots) of reordered position j = 32*blk + i,
  // stored transposed so that lanes (consecutive blk) read consecutive words.
  for (int w = threadIdx.x; w < K / 2; w += blockDim.x) {
    int i2 = w / nblk, blk = w % nblk;
    int j = 32 * blk + 2 * i2;
    uint32_t p0 = swz<R>(uint32_t(__ldg(a.perm + j)));
    uint32_t p1 = swz<R>(uint32_t(__ldg(a.perm + j + 1)));
    gidx2[w] = p0 | (p1 << 16);
  }
  __syncthreads();

  const int64_t my_tiles = (n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
  if (threadIdx.x < kProdThreads) {
    // ---------------- producers: HBM -> row-interleaved smem ----------------
    const int pt = threadIdx.x;
    const int nchunk = K / 8;                      // 8 channels = 16 bytes per row
    constexpr int U = 16 / R;                      // chunks in flight per thread
    for (int64_t i = 0; i < my_tiles; ++i) {
      const int slot = int(i & 1);
      if (i >= 2) named_bar_sync(1 + 2 + slot, kThreads);      // EMPTY[slot]
      ST* buf = slot ? buf1 : buf0;
      const int64_t r0 = (blockIdx.x + i * gridDim.x) * R;
      for (int c0 = pt; c0 < nchunk; c0 += kProdThreads * U) {
        uint4 d[U][R];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int c = c0 + u * kProdThreads;
#pragma unroll
          for (int rho = 0; rho < R; ++rho) {
            const int64_t r = r0 + rho;
            if (c < nchunk && r < a.rows)
              d[u][rho] = __ldcs(reinterpret_cast<const uint4*>(a.x + r * a.ldx) + c);
            else
              d[u][rho] = make_uint4(0, 0, 0, 0);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int c = c0 + u * kProdThreads;
          if (c >= nchunk) break;
          if constexpr (R == 1) {
            *reinterpret_cast<uint4*>(buf + 8 * c) = d[u][0];
          } else {
            const uint32_t* w0 = reinterpret_cast<const uint32_t*>(&d[u][0]);
            const uint32_t* w1 = reinterpret_cast<const uint32_t*>(&d[u][1]);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint32_t p = 8 * c + 2 * k;
              if constexpr (R == 2) {
                buf[swz<R>(p)] = __byte_perm(w0[k], w1[k], 0x5410);
                buf[swz<R>(p + 1)] = __byte_perm(w0[k], w1[k], 0x7632);
              } else {
                const uint32_t* w2 = reinterpret_cast<const uint32_t*>(&d[u][2]);
                const uint32_t* w3 = reinterpret_cast<const uint32_t*>(&d[u][3]);
                buf[swz<R>(p)] = make_uint2(__byte_perm(w0[k], w1[k], 0x5410),
                                            __byte_perm(w2[k], w3[k], 0x5410));
                buf[swz<R>(p + 1)] = make_uint2(__byte_perm(w0[k], w1[k], 0x7632),
                                                __byte_perm(w2[k], w3[k], 0x7632));
              }
            }
          }
        }
      }
      named_bar_arrive(1 + slot, kThreads);                  // FULL[slot]
    }
  } else {
    // ---------------- consumers: gather + quantize + pack + store ------------
    const int ct = threadIdx.x - kProdThreads;
    const SegGeom& G = a.geom;
    const int nvb0 = G.kp[0] / 32, nvb1 = G.kp[1] / 32, nvb2 = G.kp[2] / 32;
    const int nvb = nvb0 + nvb1 + nvb2;
    for (int64_t i = 0; i < my_tiles; ++i) {
      const int slot = int(i & 1);
      named_bar_sync(1 + slot, kThreads);                    // FULL[slot]
      const ST* buf = slot ? buf1 : buf0;
      const int64_t r0 = (blockIdx.x + i * gridDim.x) * R;
      for (int vb = ct; vb < nvb; vb += kConsThreads) {
        int g, kb;
        if (vb < nvb0) { g = 0; kb = vb; }
        else if (vb < nvb0 + nvb1) { g = 1; kb = vb - nvb0; }
        else { g = 2; kb = vb - nvb0 - nvb1; }
        const int kp128 = G.kp[g] / 128;
        const int bytes_per_blk = g == 0 ? 16 : (g == 1 ? 24 : 32);
        if (kb * 32 >= G.n[g]) {
          // padding block: zero codes and zero scale bytes
#pragma unroll
          for (int rho = 0; rho < R; ++rho) {
            const int64_t r = r0 + rho;
            if (r >= rows_pad) break;
            a.sf[g][sf_offset(r, kb, kp128)] = 0;
            if (r < a.rows) {
              uint8_t* dst = a.codes[g] + r * G.pitch[g] + (int64_t)kb * bytes_per_blk;
              for (int q = 0; q < bytes_per_blk; q += 8)
                *reinterpret_cast<uint2*>(dst + q) = make_uint2(0, 0);
            }
          }
          continue;
        }
        const int blk = (G.off[g] + 32 * kb) / 32;   // real block index in the reordered row
        ST vals[32];
#pragma unroll
        for (int i2 = 0; i2 < 16; ++i2) {
          const uint32_t pr = gidx2[i2 * nblk + blk];
          vals[2 * i2] = buf[pr & 0xFFFFu];
          vals[2 * i2 + 1] = buf[pr >> 16];
        }
#pragma unroll
        for (int rho = 0; rho < R; ++rho) {
          const int64_t r = r0 + rho;
          if (r >= rows_pad) break;
          uint32_t v[32];
#pragma unroll
          for (int k = 0; k < 32; ++k) v[k] = row_bits<R>(vals[k], rho);
          uint8_t* crow = a.codes[g] + r * G.pitch[g];
          quantize_store_block(v, g, G.fmt[g], G.sc_off[g], crow, kb, r < a.rows, a.sf[g], r,
                               kp128);
        }
      }
      if (i + 2 < my_tiles) named_bar_arrive(1 + 2 + slot, kThreads);  // EMPTY[slot]
    }
  }
}

__global__ void reorder_bf16_kernel(const uint16_t* __restrict__ x, int64_t rows, int64_t ldx,
                                    int K, const int32_t* __restrict__ perm,
                                    uint16_t* __restrict__ xr, int64_t ldxr) {
  const int64_t r = blockIdx.y;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < K; j += gridDim.x * blockDim.x)
    xr[r * ldxr + j] = x[r * ldx + perm[j]];
}

template <int R>
cudaError_t launch_rq_t(const RqArgs& a, cudaStream_t s, int64_t* launches) {
  const size_t gbytes = ((size_t)a.K * 2 + 127) / 128 * 128;
  const size_t smem = gbytes + 2 * (size_t)a.K * sizeof(typename SlotT<R>::T);
  cudaError_t e = cudaFuncSetAttribute(rq_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t rows_pad = (a.rows + 127) / 128 * 128;
  const int64_t n_tiles = (rows_pad + R - 1) / R;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rq_kernel<R>, kThreads, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  int64_t grid = (int64_t)sm_count() * per_sm;
  if (grid > n_tiles) grid = n_tiles;
  rq_kernel<R><<<(unsigned)grid, kThreads, smem, s>>>(a, rows_pad, n_tiles);
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_reorder_quantize(const RqArgs& a, cudaStream_t s, int64_t* launches) {
  // Rows per tile: as many as keep two tiles of smem within ~100 KB (R = 4 for
  // Llama/Qwen hidden sizes, R = 2 / 1 for the wide down_proj inputs).
  const size_t row_bytes = (size_t)a.K * 2;
  if (4 * row_bytes * 2 <= 100 * 1024) return launch_rq_t<4>(a, s, launches);
  if (2 * row_bytes * 2 <= 150 * 1024) return launch_rq_t<2>(a, s, launches);
  return launch_rq_t<1>(a, s, launches);
}

cudaError_t launch_reorder_bf16(const uint16_t* x, int64_t rows, int64_t ldx, int K,
                                const int32_t* perm, uint16_t* xr, int64_t ldxr,
                                cudaStream_t s, int64_t* launches) {
  if (rows == 0) return cudaSuccess;
  dim3 grid((K + 255) / 256, (unsigned)rows);
  reorder_bf16_kernel<<<grid, 256, 0, s>>>(x, rows, ldx, K, perm, xr, ldxr);
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace mmx
