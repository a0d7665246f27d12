// rq.cu -- fused reorder-and-quantize of BF16 rows into MXFP4 / MXFP6 / MXFP8
// channel segments (§3.2 "Quantization Kernel", line 151; Fig. 6
// caption line 148; Eq. 1 lines 40-45), sm_100a.
//
// HBM-bound streaming kernel (see rq_kernel below for the tile structure):
//   * tiles of R rows are streamed from HBM by TMA into a shared-memory ring and
//     transposed in place into "row-interleaved" slots: slot p holds the R BF16
//     values of channel p (R = 2: 4-byte slots); the transpose's 16-byte chunk
//     stores are ordered to be bank-conflict free, and an optional plan-time gather
//     layout (layout.cpp) permutes the 4-channel chunks inside each 128-byte line;
//   * a lane pair owns one 32-channel block of the reordered row: the gather
//     x_r[j] = X[perm[j]] is a single shared load per channel that fetches all R
//     rows at once (R-fold fewer random smem accesses than a per-row gather), its
//     slot offsets read from a per-plan table built once per CTA;
//     block amax is an integer max over |bf16| bits; the E8M0
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
#include <cstdlib>

#include "internal.h"
#include "ptx.cuh"

// Timing experiments and the timeline trace (env MM_RQ_DEBUG) are compiled in only
// with -DMM_RQ_EXPERIMENTS=1; the product build folds every check away.
#ifndef MM_RQ_EXPERIMENTS
#define MM_RQ_EXPERIMENTS 0
#endif

namespace mmx {
namespace {


// ---- element conversions (hardware RNE + satfinite, sign-preserving) --------
// cvt.*x2.f32 d, a, b puts a in the upper half of d and b in the lower half.
template <int FMT> struct Cvt;
template <> struct Cvt<F_E4M3> {
  static __device__ __forceinline__ uint32_t x4(float a0, float a1, float a2, float a3) {
    uint32_t r;
    asm("{\n\t.reg .b16 h0, h1;\n\t"
        "cvt.rn.satfinite.e4m3x2.f32 h0, %2, %1;\n\t"
        "cvt.rn.satfinite.e4m3x2.f32 h1, %4, %3;\n\t"
        "mov.b32 %0, {h0, h1};\n\t}" : "=r"(r) : "f"(a0), "f"(a1), "f"(a2), "f"(a3));
    return r;
  }
};
template <> struct Cvt<F_E5M2> {
  static __device__ __forceinline__ uint32_t x4(float a0, float a1, float a2, float a3) {
    uint32_t r;
    asm("{\n\t.reg .b16 h0, h1;\n\t"
        "cvt.rn.satfinite.e5m2x2.f32 h0, %2, %1;\n\t"
        "cvt.rn.satfinite.e5m2x2.f32 h1, %4, %3;\n\t"
        "mov.b32 %0, {h0, h1};\n\t}" : "=r"(r) : "f"(a0), "f"(a1), "f"(a2), "f"(a3));
    return r;
  }
};
// FP6: four codes -> 24-bit LSB-first stream c0 | c1<<6 | c2<<12 | c3<<18, from
// t = c0 | c1<<8 | c2<<16 | c3<<24 (each code 6 bits): close the byte gaps pairwise.
// The cvt leaves the top two bits of every code byte zero, so each step is one shift and
// one bitwise select with complementary masks (a single LOP3): the bits the select takes
// from the shifted word outside the wanted fields are zero or are dropped by the next step
// (w bits 14-15 hold c2's low bits; the second select takes w bits 0-11 and 16-27 only).
template <uint32_t M>
__device__ __forceinline__ uint32_t sel_bits(uint32_t a, uint32_t b) {   // (a & M) | (b & ~M), one LOP3
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(r) : "r"(a), "r"(b), "n"(M));
  return r;
}
__device__ __forceinline__ uint32_t pack6(uint32_t t) {
  const uint32_t w = sel_bits<0x003F003Fu>(t, t >> 2);   // c0|c1<<6 , c2|c3<<6 at bit 16
  return sel_bits<0xFFFu>(w, w >> 4);
}
template <> struct Cvt<F_E3M2> {
  static __device__ __forceinline__ uint32_t x4(float a0, float a1, float a2, float a3) {
    uint32_t t;
    asm("{\n\t.reg .b16 h0, h1;\n\t"
        "cvt.rn.satfinite.e3m2x2.f32 h0, %2, %1;\n\t"
        "cvt.rn.satfinite.e3m2x2.f32 h1, %4, %3;\n\t"
        "mov.b32 %0, {h0, h1};\n\t}" : "=r"(t) : "f"(a0), "f"(a1), "f"(a2), "f"(a3));
    return pack6(t);
  }
};
template <> struct Cvt<F_E2M3> {
  static __device__ __forceinline__ uint32_t x4(float a0, float a1, float a2, float a3) {
    uint32_t t;
    asm("{\n\t.reg .b16 h0, h1;\n\t"
        "cvt.rn.satfinite.e2m3x2.f32 h0, %2, %1;\n\t"
        "cvt.rn.satfinite.e2m3x2.f32 h1, %4, %3;\n\t"
        "mov.b32 %0, {h0, h1};\n\t}" : "=r"(t) : "f"(a0), "f"(a1), "f"(a2), "f"(a3));
    return pack6(t);
  }
};
// FP4: eight codes -> one 32-bit word, element 0 in the lowest nibble.
__device__ __forceinline__ uint32_t cvt_e2m1_x8(const float (&f)[8]) {
  uint32_t r;
  asm("{\n\t.reg .b8 b0, b1, b2, b3;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b0, %2, %1;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b1, %4, %3;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b2, %6, %5;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b3, %8, %7;\n\t"
      "mov.b32 %0, {b0, b1, b2, b3};\n\t}"
      : "=r"(r)
      : "f"(f[0]), "f"(f[1]), "f"(f[2]), "f"(f[3]), "f"(f[4]), "f"(f[5]), "f"(f[6]), "f"(f[7]));
  return r;
}

// Byte offset of scale (r, kb) inside the 128x4-atom layout of a segment with
// kp128 = Kp/128 atoms per 128-row group.
__device__ __forceinline__ int64_t sf_offset(int64_t r, int kb, int kp128) {
  return ((r >> 7) * kp128 + (kb >> 2)) * 512 + (r & 31) * 16 + ((r >> 5) & 3) * 4 + (kb & 3);
}

// Slot types: the R BF16 values of one channel, rows interleaved (even rows in
// the low halves): R = 1 -> uint16_t, 2 -> uint32_t, 4 -> uint2 {rows 0|1, 2|3}.
template <int R> struct Slot;
template <> struct Slot<1> { using T = uint16_t; };
template <> struct Slot<2> { using T = uint32_t; };
template <> struct Slot<4> { using T = uint2; };

// Row RHO of a slot as an fp32 value (BF16 = the top half of an fp32).
template <int RHO>
__device__ __forceinline__ float slot_f32(const uint16_t& s) { return __uint_as_float(uint32_t(s) << 16); }
template <int RHO>
__device__ __forceinline__ float slot_f32(const uint32_t& s) {
  return (RHO & 1) == 0 ? __uint_as_float(s << 16) : __uint_as_float(s & 0xFFFF0000u);
}
template <int RHO>
__device__ __forceinline__ float slot_f32(const uint2& s) {
  const uint32_t w = (RHO < 2) ? s.x : s.y;
  return (RHO & 1) == 0 ? __uint_as_float(w << 16) : __uint_as_float(w & 0xFFFF0000u);
}

// Scale 8 consecutive elements of row RHO by 2^-e (exact; packed fp32x2 multiply).
template <int RHO, typename ST>
__device__ __forceinline__ void scaled8(const ST* v, float inv, float (&f)[8]) {
#pragma unroll
  for (int i = 0; i < 8; i += 2) {
    const float2 p = __fmul2_rn(make_float2(slot_f32<RHO>(v[i]), slot_f32<RHO>(v[i + 1])), make_float2(inv, inv));
    f[i] = p.x;
    f[i + 1] = p.y;
  }
}

// Encode + store row RHO of NV consecutive channels of one 32-element block (NV =
// 32: the whole block; NV = 16: one half, the lane pair splits the block) for
// segment kind G (0 FP4, 1 FP6, 2 FP8) in element format FMT.
template <int G, int FMT, int RHO, int NV, typename ST>
__device__ __forceinline__ void encode_store(const ST (&v)[NV], float inv, uint8_t* dst) {
  if constexpr (G == 0) {  // MXFP4: NV/2 bytes
    uint32_t w[NV / 8];
#pragma unroll
    for (int q = 0; q < NV / 8; ++q) {
      float f[8];
      scaled8<RHO>(v + 8 * q, inv, f);
      w[q] = cvt_e2m1_x8(f);
    }
    if constexpr (NV == 32) *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
    else *reinterpret_cast<uint2*>(dst) = make_uint2(w[0], w[1]);
  } else if constexpr (G == 1) {  // MXFP6: 3 NV / 4 bytes, LSB-first 6-bit stream
    uint32_t q24[NV / 4];
#pragma unroll
    for (int q = 0; q < NV / 8; ++q) {
      float f[8];
      scaled8<RHO>(v + 8 * q, inv, f);
      q24[2 * q] = Cvt<FMT>::x4(f[0], f[1], f[2], f[3]);
      q24[2 * q + 1] = Cvt<FMT>::x4(f[4], f[5], f[6], f[7]);
    }
    // (the 24-bit groups do not overlap: shift-and-add, one IMAD / LEA each)
    if constexpr (NV == 32) {
      uint2* d2 = reinterpret_cast<uint2*>(dst);
      d2[0] = make_uint2(q24[1] * 0x1000000u + q24[0], q24[2] * 0x10000u + (q24[1] >> 8));
      d2[1] = make_uint2(q24[3] * 0x100u + (q24[2] >> 16), q24[5] * 0x1000000u + q24[4]);
      d2[2] = make_uint2(q24[6] * 0x10000u + (q24[5] >> 8), q24[7] * 0x100u + (q24[6] >> 16));
    } else {  // 12 bytes, 4-byte aligned
      uint32_t* d1 = reinterpret_cast<uint32_t*>(dst);
      d1[0] = q24[1] * 0x1000000u + q24[0];
      d1[1] = q24[2] * 0x10000u + (q24[1] >> 8);
      d1[2] = q24[3] * 0x100u + (q24[2] >> 16);
    }
  } else {  // MXFP8: NV bytes
    uint32_t w[NV / 4];
#pragma unroll
    for (int q = 0; q < NV / 8; ++q) {
      float f[8];
      scaled8<RHO>(v + 8 * q, inv, f);
      w[2 * q] = Cvt<FMT>::x4(f[0], f[1], f[2], f[3]);
      w[2 * q + 1] = Cvt<FMT>::x4(f[4], f[5], f[6], f[7]);
    }
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    d4[0] = make_uint4(w[0], w[1], w[2], w[3]);
    if constexpr (NV == 32) d4[1] = make_uint4(w[4], w[5], w[6], w[7]);
  }
}

// ---- fused RMSNorm (reading R27) ----------------------
template <int RHO> __device__ __forceinline__ uint32_t slot_bits(const uint16_t& s) { return s; }
template <int RHO> __device__ __forceinline__ uint32_t slot_bits(const uint32_t& s) { return (s >> (16 * RHO)) & 0xFFFFu; }
template <int RHO> __device__ __forceinline__ uint32_t slot_bits(const uint2& s) {
  return ((RHO < 2 ? s.x : s.y) >> (16 * (RHO & 1))) & 0xFFFFu;
}
__device__ __forceinline__ void slot_pack(uint16_t& s, const uint32_t (&b)[4]) { s = (uint16_t)b[0]; }
__device__ __forceinline__ void slot_pack(uint32_t& s, const uint32_t (&b)[4]) { s = b[0] | (b[1] << 16); }
__device__ __forceinline__ void slot_pack(uint2& s, const uint32_t (&b)[4]) {
  s = make_uint2(b[0] | (b[1] << 16), b[2] | (b[3] << 16));
}
__device__ __forceinline__ double bf16_f64(uint32_t b) { return (double)__uint_as_float(b << 16); }
// double-double accumulation (TwoSum): exact sums of squares of BF16 values
__device__ __forceinline__ void dd_add(double& hi, double& lo, double v) {
  const double s = hi + v, bb = s - hi;
  lo += (hi - (s - bb)) + (v - bb);
  hi = s;
}
__device__ __forceinline__ void dd_add_dd(double& hi, double& lo, double bhi, double blo) {
  const double s = hi + bhi, bb = s - hi;
  double err = (hi - (s - bb)) + (bhi - bb);
  err += lo + blo;
  hi = s + err;
  lo = err - (hi - s);
}
// t = bf16_rne(fp32(x * r)), y = bf16_rne(fp32(gamma * t)) for every row of a slot
// (reading R27: the HF LlamaRMSNorm data flow), packed fp32x2 multiplies
// and bf16x2 conversions (RNE, no flush of subnormals).
__device__ __forceinline__ uint32_t bf16x2_rne(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ uint32_t norm_pair(uint32_t w, float g, float r0, float r1) {
  const float2 p = __fmul2_rn(make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xFFFF0000u)),
                              make_float2(r0, r1));
  const uint32_t t = bf16x2_rne(p.x, p.y);
  const float2 q = __fmul2_rn(make_float2(__uint_as_float(t << 16), __uint_as_float(t & 0xFFFF0000u)),
                              make_float2(g, g));
  return bf16x2_rne(q.x, q.y);
}
template <int R>
__device__ __forceinline__ void norm_slot(uint16_t& v, uint32_t gbits, const float (&r)[4]) {
  const float g = __uint_as_float(gbits << 16);
  v = (uint16_t)norm_pair(v, g, r[0], r[0]);
}
template <int R>
__device__ __forceinline__ void norm_slot(uint32_t& v, uint32_t gbits, const float (&r)[4]) {
  v = norm_pair(v, __uint_as_float(gbits << 16), r[0], r[1]);
}
template <int R>
__device__ __forceinline__ void norm_slot(uint2& v, uint32_t gbits, const float (&r)[4]) {
  const float g = __uint_as_float(gbits << 16);
  v = make_uint2(norm_pair(v.x, g, r[0], r[1]), norm_pair(v.y, g, r[2], r[3]));
}

// Block amax of each of the R rows over |bf16| bits (packed 16x2 maxima).  With
// NV = 16 each lane holds half a block; the lane pair combines with one shuffle.
template <int NV, typename F>
__device__ __forceinline__ uint32_t tree_reduce(const uint32_t (&w)[NV], F f);
__device__ __forceinline__ uint32_t absmax_bf16x2(uint32_t a, uint32_t b);
template <int NV>
__device__ __forceinline__ void block_amax(const uint16_t (&v)[NV], uint32_t (&am)[4]) {
  // single-row slots: pack channel pairs into bf16x2 words (one PRMT per pair) and
  // reduce them with the packed |max| -- half the operations of a per-value max
  uint32_t w[NV / 2];
#pragma unroll
  for (int i = 0; i < NV / 2; ++i) w[i] = __byte_perm(uint32_t(v[2 * i]), uint32_t(v[2 * i + 1]), 0x5410);
  uint32_t m = tree_reduce<NV / 2>(w, absmax_bf16x2);
  if constexpr (NV == 16) m = absmax_bf16x2(m, __shfl_xor_sync(0xffffffffu, m, 1));
  am[0] = max(m & 0x7FFFu, (m >> 16) & 0x7FFFu);
}
// max(|a|, |b|) per BF16 half (sign = xor of the signs; masked off by the caller):
// one instruction per word instead of an abs-mask and an integer max.  Inputs are
// finite (NaN/Inf are outside the contract, R8); subnormals are ordered
// exactly like their bit patterns.
__device__ __forceinline__ uint32_t absmax_bf16x2(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("max.xorsign.abs.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
// Pairwise tree over NV (a power of two) words: log2(NV) dependent steps, not NV.
template <int NV, typename F>
__device__ __forceinline__ uint32_t tree_reduce(const uint32_t (&w)[NV], F f) {
  uint32_t t[NV / 2];
#pragma unroll
  for (int i = 0; i < NV / 2; ++i) t[i] = f(w[2 * i], w[2 * i + 1]);
#pragma unroll
  for (int n = NV / 4; n >= 1; n /= 2)
#pragma unroll
    for (int i = 0; i < n; ++i) t[i] = f(t[2 * i], t[2 * i + 1]);
  return t[0];
}
template <int NV>
__device__ __forceinline__ void block_amax(const uint32_t (&v)[NV], uint32_t (&am)[4]) {
  uint32_t m = tree_reduce<NV>(v, absmax_bf16x2);
  if constexpr (NV == 16) m = absmax_bf16x2(m, __shfl_xor_sync(0xffffffffu, m, 1));
  am[0] = m & 0x7FFFu;
  am[1] = (m >> 16) & 0x7FFFu;
}
template <int NV>
__device__ __forceinline__ void block_amax(const uint2 (&v)[NV], uint32_t (&am)[4]) {
  uint32_t x[NV], y[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) { x[i] = v[i].x; y[i] = v[i].y; }
  uint32_t m01 = tree_reduce<NV>(x, absmax_bf16x2), m23 = tree_reduce<NV>(y, absmax_bf16x2);
  if constexpr (NV == 16) {
    m01 = absmax_bf16x2(m01, __shfl_xor_sync(0xffffffffu, m01, 1));
    m23 = absmax_bf16x2(m23, __shfl_xor_sync(0xffffffffu, m23, 1));
  }
  am[0] = m01 & 0x7FFFu;
  am[1] = (m01 >> 16) & 0x7FFFu;
  am[2] = m23 & 0x7FFFu;
  am[3] = (m23 >> 16) & 0x7FFFu;
}

// One row of one block: E8M0 exponent by integer arithmetic on the BF16 exponent
// field (e = floor(log2 amax) - off, clamped at -127; zero and subnormal amax give
// -127), the scale byte into its 128x4 atom (rows of a tile are consecutive rows of
// one 32-row group: +16 bytes per row; written by the even lane of a pair), codes
// packed and stored.
template <int RHO, int G, int FMT, int NV, typename ST>
__device__ __forceinline__ void quantize_row(const ST (&v)[NV], uint32_t amax, int off, uint8_t* crow,
                                             uint8_t* sfp, bool store_codes, bool store_sf, bool zero) {
  const int sb = max(int(amax >> 7) - off, 0);                  // E8M0 byte = e + 127
  const float inv = __uint_as_float(uint32_t(254 - sb) << 23);  // 2^-e exactly
  if (store_sf) sfp[16 * RHO] = zero ? uint8_t(0) : uint8_t(sb);
  if (store_codes) {
    if (zero) {   // padding block: zero codes
      constexpr int hb = G == 0 ? NV / 2 : (G == 1 ? 3 * NV / 4 : NV);
#pragma unroll
      for (int b = 0; b < hb; b += 4) *reinterpret_cast<uint32_t*>(crow + b) = 0u;
    } else {
      encode_store<G, FMT, RHO, NV>(v, inv, crow);
    }
  }
}

// Rows of one block after its amax is known (no warp-collective operations, so it
// may run under divergence: a chunk that straddles two segments runs two formats).
template <int R, int G, int FMT, int NV>
__device__ __forceinline__ void quantize_rows(const typename Slot<R>::T (&v)[NV], const uint32_t (&am)[4], int off,
                                              uint8_t* crow0, uint32_t pitch, uint8_t* sfp, int nvalid, bool live,
                                              bool store_sf) {
  quantize_row<0, G, FMT, NV>(v, am[0], off, crow0, sfp, live && nvalid > 0, store_sf, false);
  if constexpr (R >= 2) quantize_row<1, G, FMT, NV>(v, am[1], off, crow0 + pitch, sfp, live && nvalid > 1, store_sf, false);
  if constexpr (R >= 4) {
    quantize_row<2, G, FMT, NV>(v, am[2], off, crow0 + 2 * pitch, sfp, live && nvalid > 2, store_sf, false);
    quantize_row<3, G, FMT, NV>(v, am[3], off, crow0 + 3 * pitch, sfp, live && nvalid > 3, store_sf, false);
  }
}

// Shared-memory loads by 32-bit shared address: with a warp-uniform base the gather
// becomes one LDS [R + UR] per slot (no generic-to-shared window arithmetic per load).
__device__ __forceinline__ void lds_slot(uint32_t a, uint16_t& v) {
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
}
__device__ __forceinline__ void lds_slot(uint32_t a, uint32_t& v) {
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a));
}
__device__ __forceinline__ void lds_slot(uint32_t a, uint2& v) {
  asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
}
__device__ __forceinline__ uint4 lds_u4(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}

// Per-tile context of a consumer warp (everything tile_chunks needs besides the plan).
template <int R> struct ChunkCtx {
  const uint8_t* st;        // stage: 256-channel boxes of row-interleaved slots
  const uint8_t* smem0;     // shared-memory base (the stage's offset from it is made warp-uniform)
  const uint32_t* gidx;     // gather table: tab == 3: one u32 slot byte offset per reordered position;
                            // tab == 1, 2: u16 offsets, two per word [block][16 words]; 0: none (L1 perm)
  const uint16_t* gamma_r;  // RMSNorm weight in reordered order (NORM only)
  int r0;                   // first row of the tile
  int nvalid;               // rows of the tile inside the matrix
  int group_warps, lane, dbg;
  int tab;
};

__device__ __forceinline__ int sel3(int g, int x0, int x1, int x2) { return g == 0 ? x0 : (g == 1 ? x1 : x2); }

// Encode + stores of one block row set for a chunk whose blocks all lie in segment G
// (first block of the segment: bseg; fmt_a: E3M2 for G = 1, E4M3 for G = 2).
template <int R, int G>
__device__ __forceinline__ void encode_uniform(const RqArgs& a, const typename Slot<R>::T (&v)[16],
                                               const uint32_t (&am)[4], int b, int h, unsigned r0, unsigned sf_row,
                                               int bseg, int nvalid, bool live, bool store_sf, bool fmt_a) {
  constexpr int hb = G == 0 ? 8 : (G == 1 ? 12 : 16);
  const int kb = b - bseg;
  const uint32_t pitch = (uint32_t)a.geom.pitch[G];
  uint8_t* crow0 = a.codes[G] + (uint64_t)r0 * pitch + (unsigned)(h * hb) + (unsigned)kb * (2 * hb);
  uint8_t* sfp = a.sf[G] + (size_t)((r0 >> 7) * ((unsigned)a.geom.kp[G] >> 7) + ((unsigned)kb >> 2)) * 512 + sf_row +
                 (kb & 3);
  const int off = a.geom.sc_off[G];
  if constexpr (G == 0) {
    quantize_rows<R, 0, F_E2M1, 16>(v, am, off, crow0, pitch, sfp, nvalid, live, store_sf);
  } else if constexpr (G == 1) {
    if (fmt_a) quantize_rows<R, 1, F_E3M2, 16>(v, am, off, crow0, pitch, sfp, nvalid, live, store_sf);
    else quantize_rows<R, 1, F_E2M3, 16>(v, am, off, crow0, pitch, sfp, nvalid, live, store_sf);
  } else {
    if (fmt_a) quantize_rows<R, 2, F_E4M3, 16>(v, am, off, crow0, pitch, sfp, nvalid, live, store_sf);
    else quantize_rows<R, 2, F_E5M2, 16>(v, am, off, crow0, pitch, sfp, nvalid, live, store_sf);
  }
}

// The chunks of one tile owned by this warp (chunk c_first, c_first + group_warps, ...).
// A chunk is 16 consecutive 32-channel blocks of the REORDERED row -- the segments are
// contiguous there (FP4 blocks, then FP6, then FP8) -- so a K = 4096 row is 8 chunks
// whatever the mix (per-segment chunks would need 10 at the q_proj mix, two of them
// two-thirds idle).  The lane pair (2 l, 2 l + 1) owns block 16 c + l: gather, (norm),
// block amax and the E8M0 exponent run on every lane; the encode + stores branch on the
// block's segment, which is warp-uniform except in the (at most two) chunks that
// straddle a segment boundary.  Storage padding blocks (n_g .. kp_g) are written by
// tile_padding.
template <int R, bool NORM, bool U16>
__device__ __forceinline__ void tile_chunks(const RqArgs& a, const ChunkCtx<R>& cx, int c_first, bool e3m2,
                                            bool e4m3, const float (&rn)[4]) {
  using ST = typename Slot<R>::T;
  const int nbt = (unsigned)a.K >> 5;                           // real blocks of the row
  const int nch = (unsigned)(nbt + 15) >> 4;
  if (c_first >= nch) return;
  const int b1 = (unsigned)a.geom.off[1] >> 5, b2 = (unsigned)a.geom.off[2] >> 5;   // first block of FP6 / FP8
  const int h = cx.lane & 1;                                    // which half of the block
  const unsigned r0 = (unsigned)cx.r0;
  const uint32_t st_off = __reduce_max_sync(0xffffffffu, (uint32_t)(cx.st - cx.smem0));
  const uint8_t* const st_u = cx.smem0 + st_off;
  const uint32_t st_s = __reduce_max_sync(0xffffffffu, ptx::smem_u32(cx.st));   // stage, shared address
  // u16 table: the lane's two 16-byte table vectors of block b sit at 64 b + 32 h + 16 rot
  // and 64 b + 32 h + 16 (rot ^ 1) (rot: the table build's per-lane swap)
  // (opaque moves: keep the two per-lane bases in registers instead of recomputing them
  // from the thread index in every chunk)
  const uint32_t trot = (uint32_t)((cx.lane >> 2) & 1);
  uint32_t tb0, tb1;
  asm("mov.b32 %0, %1;" : "=r"(tb0) : "r"(ptx::smem_u32(cx.gidx) + 32u * (uint32_t)h + 16u * trot));
  asm("mov.b32 %0, %1;" : "=r"(tb1) : "r"(ptx::smem_u32(cx.gidx) + 32u * (uint32_t)h + 16u * (trot ^ 1u)));
  // per-tile row bases of the three segments' code rows and scale atoms
  const unsigned sf_row = (r0 & 31) * 16 + ((r0 >> 5) & 3) * 4;
  for (int c = c_first; c < nch; c += cx.group_warps) {
    const int b_raw = c * 16 + (cx.lane >> 1);
    const bool live = b_raw < nbt;                              // pair-uniform
    const int b = live ? b_raw : nbt - 1;                       // dead lanes compute on the last block
    if (MM_RQ_EXPERIMENTS && (cx.dbg & 16)) continue;           // timing experiment: no stores at all
    const int bg = (MM_RQ_EXPERIMENTS && (cx.dbg & 64)) ? 0 : b;   // experiment 64: broadcast gather
    ST v[16];
    if (!U16 && cx.tab == 3) {   // u32 offsets: 4 x 128-bit table loads, slot address = stage base + offset
      const uint4* gp = reinterpret_cast<const uint4*>(cx.gidx + 32 * bg + 16 * h);
      const int rot = (cx.lane >> 1) & 3;          // the table build's per-lane rotation
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) {
        const uint4 e = gp[(q4 + rot) & 3];
        v[4 * q4 + 0] = *reinterpret_cast<const ST*>(st_u + e.x);
        v[4 * q4 + 1] = *reinterpret_cast<const ST*>(st_u + e.y);
        v[4 * q4 + 2] = *reinterpret_cast<const ST*>(st_u + e.z);
        v[4 * q4 + 3] = *reinterpret_cast<const ST*>(st_u + e.w);
      }
    } else if (U16 || cx.tab) {
      const uint4 p0 = lds_u4(tb0 + 64u * (uint32_t)bg), p1 = lds_u4(tb1 + 64u * (uint32_t)bg);
      const uint32_t pr[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        lds_slot(st_s + (pr[q] & 0xFFFFu), v[2 * q + 0]);
        lds_slot(st_s + (pr[q] >> 16), v[2 * q + 1]);
      }
    } else {
      const ST* slots = reinterpret_cast<const ST*>(cx.st);
      const int4* pp = reinterpret_cast<const int4*>(a.perm + 32 * bg + 16 * h);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int4 pv = __ldg(pp + q);
        v[4 * q + 0] = slots[pv.x];
        v[4 * q + 1] = slots[pv.y];
        v[4 * q + 2] = slots[pv.z];
        v[4 * q + 3] = slots[pv.w];
      }
    }
    if constexpr (NORM) {
      const uint4* gp4 = reinterpret_cast<const uint4*>(cx.gamma_r + 32 * bg + 16 * h);
      const uint4 ga = gp4[0], gb = gp4[1];
      const uint32_t gw8[8] = {ga.x, ga.y, ga.z, ga.w, gb.x, gb.y, gb.z, gb.w};
#pragma unroll
      for (int i = 0; i < 16; ++i) norm_slot<R>(v[i], (gw8[i >> 1] >> (16 * (i & 1))) & 0xFFFFu, rn);
    }
    uint32_t am[4];
    block_amax<16>(v, am);   // every lane of the warp (full-warp shuffle), before any divergence
    const bool store_sf = live && h == 0;
    if (MM_RQ_EXPERIMENTS && (cx.dbg & 8)) continue;            // experiment: no encode, no stores
    // Encode + stores: a per-lane branch on the block's segment (warp-uniform except in the
    // at most two chunks that straddle a segment boundary); each branch addresses its
    // segment with compile-time geometry (no per-lane selects of pitch / base / offsets).
    if (b < b1) encode_uniform<R, 0>(a, v, am, b, h, r0, sf_row, 0, cx.nvalid, live, store_sf, true);
    else if (b < b2) encode_uniform<R, 1>(a, v, am, b, h, r0, sf_row, b1, cx.nvalid, live, store_sf, e3m2);
    else encode_uniform<R, 2>(a, v, am, b, h, r0, sf_row, b2, cx.nvalid, live, store_sf, e4m3);
  }
}

// Storage padding of one tile: the blocks n_g .. kp_g of every segment (at most three
// per segment) get zero codes (rows inside the matrix) and zero scale bytes (all R rows
// of the tile).  One lane per (padding block, row).
template <int R>
__device__ __forceinline__ void tile_padding(const RqArgs& a, int r0, int nvalid, int lane) {
  const int np0 = (a.geom.kp[0] - a.geom.n[0]) >> 5, np1 = (a.geom.kp[1] - a.geom.n[1]) >> 5;
  const int tot = np0 + np1 + ((a.geom.kp[2] - a.geom.n[2]) >> 5);
  for (int t = lane; t < tot * R; t += 32) {
    const int rho = t % R, p = t / R;
    const int g = p < np0 ? 0 : (p < np0 + np1 ? 1 : 2);
    const int kb = (sel3(g, a.geom.n[0], a.geom.n[1], a.geom.n[2]) >> 5) + p - sel3(g, 0, np0, np0 + np1);
    const int64_t r = (int64_t)r0 + rho;
    const int hb2 = sel3(g, 16, 24, 32);   // code bytes per block
    uint8_t* const codes = g == 0 ? a.codes[0] : (g == 1 ? a.codes[1] : a.codes[2]);
    uint8_t* const sf = g == 0 ? a.sf[0] : (g == 1 ? a.sf[1] : a.sf[2]);
    if (rho < nvalid) {
      uint32_t* c = reinterpret_cast<uint32_t*>(codes + r * sel3(g, (int)a.geom.pitch[0], (int)a.geom.pitch[1],
                                                               (int)a.geom.pitch[2]) + (int64_t)kb * hb2);
      for (int w = 0; w < hb2 / 4; ++w) c[w] = 0u;
    }
    sf[sf_offset(r, kb, sel3(g, a.geom.kp[0], a.geom.kp[1], a.geom.kp[2]) >> 7)] = 0;
  }
}

// Timeline trace (env MM_RQ_DEBUG & 32; read with mm_debug_rq_trace): per CTA
// [start, table ready, tile0 data ready, tile0 done, tile1 ready, tile1 done, ..., last TMA issued].
__device__ unsigned long long g_rq_trace[160][16];

struct RqDev {
  RqArgs a;
  int64_t n_tiles;      // tiles of R rows covering roundup(rows, 128)
  int nbox;             // TMA boxes of 256 channels per row
  int stages, groups, group_warps;
  int perm_smem;        // gather table: 3 = perm bulk-copied and turned IN PLACE into u32 slot offsets;
                        // 1 = perm bulk-copied + u16 table; 2 = u16 table built from global; 0 = none (L1)
  int box3d;            // 1: one 3-D TMA per tile ({256, R, nbox} box), 0: nbox 2-D boxes
  int lay_copy;         // 1: the gather layout's words are bulk-copied with the permutation
  int dbg;              // timing experiments only (env MM_RQ_DEBUG): 1 = skip gather/quantize, 2 = skip transpose too
};

// Fused reorder-and-quantize, warp-specialised and TMA-fed:
//  * warp 0 (one thread) streams tiles of R rows into a ring of `stages` shared
//    memory buffers with 2-D TMA loads (boxes of 256 channels x R rows, one
//    mbarrier per stage) -- HBM latency is hidden by the ring depth, not by
//    registers;
//  * `groups` consumer groups of `group_warps` warps take tiles round-robin.  For
//    each tile a group first transposes the stage in place, warp w owning whole
//    256-channel boxes, into "row-interleaved" slots (slot p = the R BF16 values
//    of channel p at byte p * 2R); then thread t owns 32-channel blocks of the
//    reordered rows: the gather x_r[j] = X[perm[j]] is one shared load per
//    channel that returns all R rows (the permutation is read through L1 as
//    16-byte vectors), block amax, scale and encode as above; finally the stage
//    is released to the producer.
#ifndef RQ_T4
#define RQ_T4 640
#endif
#ifndef RQ_T2
#define RQ_T2 768
#endif
// Thread budget per variant (register file / threads = registers per lane).
constexpr int rq_max_threads(int R, bool NORM) { return (R == 4 || NORM) ? RQ_T4 : (R == 2 ? RQ_T2 : 1024); }

// U16: the instantiation for the default u16 gather table (table modes 1 and 2); the
// u32 (mode 3, opt-in) and table-less (mode 0) paths compiled out -- a smaller kernel.
template <int R, bool NORM, bool U16>
__global__ void __launch_bounds__(rq_max_threads(R, NORM), 1)
rq_kernel(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ RqDev d) {
  using ST = typename Slot<R>::T;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment by pointer arithmetic on the shared pointer (keeps the
  // shared state space: a uintptr_t round trip would turn every access generic).
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  const RqArgs& a = d.a;
  const int stage_bytes = d.nbox * 512 * R;
  // [ring of stages][perm copy: K x int32][gather table: K x u16][barriers]
  const int K = a.K;
  const size_t perm_copy = (d.perm_smem == 1 || d.perm_smem == 3) ? (size_t)K * 4 : 0;
  // (+ the gather layout's per-line words for the transpose, R = 2 only)
  const size_t tab_core = perm_copy + ((d.perm_smem == 1 || d.perm_smem == 2) ? ((size_t)K * 2 + 15) / 16 * 16 : 0);
  const uint32_t* layout = R == 2 ? a.layout : nullptr;
  // R = 2 without the norm: the transpose reads per-(box, lane) store offsets (lay_x,
  // 32 words per box, built below); R = 2 with the norm: one layout word per 32-channel line
  constexpr bool LX = R == 2 && !NORM;
  const size_t lay_bytes = LX ? (size_t)d.nbox * 128 : (layout ? (size_t)d.nbox * 32 : 0);
  const size_t tab_bytes = tab_core + lay_bytes + (d.lay_copy ? (size_t)K / 8 : 0);
  uint32_t* lay_s = reinterpret_cast<uint32_t*>(smem + (size_t)d.stages * stage_bytes + tab_core);
  // the layout's per-line words: a shared copy that arrives with the permutation, or global
  const uint32_t* lay_w = d.lay_copy ? reinterpret_cast<const uint32_t*>(smem + (size_t)d.stages * stage_bytes +
                                                                         tab_core + lay_bytes)
                                     : layout;
  const int32_t* perm_s = reinterpret_cast<const int32_t*>(smem + (size_t)d.stages * stage_bytes);
  uint32_t* gidx = d.perm_smem == 3 ? reinterpret_cast<uint32_t*>(smem + (size_t)d.stages * stage_bytes)   // K words
                                    : reinterpret_cast<uint32_t*>(smem + (size_t)d.stages * stage_bytes + perm_copy);  // K/2
  // optional RMSNorm region: gamma in reordered order (K x u16) + reduction scratch
  constexpr bool norm = NORM;   // RMSNorm fused ahead of the quantization (a.gamma != nullptr)
  const size_t norm_bytes = norm ? ((size_t)K * 2 + 255) / 256 * 256 + 4096 : 0;
  uint16_t* gamma_r = reinterpret_cast<uint16_t*>(smem + (size_t)d.stages * stage_bytes + tab_bytes);
  double* nred = reinterpret_cast<double*>(smem + (size_t)d.stages * stage_bytes + tab_bytes +
                                           ((size_t)K * 2 + 255) / 256 * 256);   // [3 grp][..]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)d.stages * stage_bytes + tab_bytes + norm_bytes);
  uint64_t* empty = full + d.stages;
  uint64_t* permbar = empty + d.stages;
  // warp index through a warp reduction: the compiler then knows it is warp-uniform, so
  // the role / group / ring-slot values derived from it live in uniform registers and
  // the gather's shared loads take the stage base as a uniform operand ([R + UR]).
  const int warp = (int)__reduce_max_sync(0xffffffffu, threadIdx.x / 32), lane = threadIdx.x % 32;
  const uint64_t t_start = ptx::globaltimer_ns();
  if (threadIdx.x == 0 && (MM_RQ_EXPERIMENTS && (d.dbg & 32))) g_rq_trace[blockIdx.x][0] = t_start;
  if (threadIdx.x == 0) {
    for (int i = 0; i < d.stages; ++i) {
      ptx::mbar_init(ptx::smem_u32(&full[i]), 1);
      ptx::mbar_init(ptx::smem_u32(&empty[i]), d.group_warps);
    }
    ptx::mbar_init(ptx::smem_u32(permbar), 1);
    ptx::fence_barrier_init();
    ptx::tma_prefetch_desc(&tmx);
    if (d.perm_smem == 1 || d.perm_smem == 3) {  // the permutation arrives asynchronously, alongside the first tiles
      ptx::mbar_arrive_expect_tx(ptx::smem_u32(permbar), (uint32_t)K * 4 + (d.lay_copy ? (uint32_t)K / 8 : 0u));
      ptx::bulk_load(ptx::smem_u32(perm_s), a.perm, (uint32_t)K * 4, ptx::smem_u32(permbar));
      if (d.lay_copy) ptx::bulk_load(ptx::smem_u32(lay_w), layout, (uint32_t)K / 8, ptx::smem_u32(permbar));
    }
  }
  __syncthreads();
  const int64_t my_tiles = (d.n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x;

  ptx::grid_dep_launch();
  if (warp == 0) {
    // ============================ TMA producer ============================
    ptx::grid_dep_wait();   // X may be produced by the preceding kernel
    if (lane == 0) {
      const uint32_t tx = (uint32_t)stage_bytes;
      for (int64_t i = 0; i < my_tiles; ++i) {
        const int s = int(i % d.stages);
        const uint32_t ph = uint32_t(i / d.stages) & 1u;
        ptx::mbar_wait_sleep(ptx::smem_u32(&empty[s]), ph ^ 1u, 11, s, (int)i);
        const uint32_t fb = ptx::smem_u32(&full[s]);
        if (MM_RQ_EXPERIMENTS && (d.dbg & 4)) { ptx::mbar_arrive(fb); continue; }   // timing experiment: no loads
        ptx::mbar_arrive_expect_tx(fb, tx);
        const int row0 = (int)((blockIdx.x + i * gridDim.x) * R);
        const uint32_t dst = ptx::smem_u32(smem + (size_t)s * stage_bytes);
        if (d.box3d) ptx::tma_load_3d(dst, &tmx, fb, 0, row0, 0);   // all boxes of the tile at once
        else
          for (int b = 0; b < d.nbox; ++b) ptx::tma_load_2d(dst + b * 512 * R, &tmx, fb, 256 * b, row0);
        if ((MM_RQ_EXPERIMENTS && (d.dbg & 32)) && i == my_tiles - 1) g_rq_trace[blockIdx.x][14] = ptx::globaltimer_ns();
      }
    }
    return;
  }
  // ============================ consumer groups ============================
  const int cw = warp - 1;
  const int grp = cw / d.group_warps, gw = cw % d.group_warps;
  if (grp >= d.groups) return;
  const int gthreads = d.group_warps * 32;
  // Kernel parameters are copied into (uniform) registers once: indexing the
  // parameter block inside the loop would go through generic/local memory.
  const int stages = d.stages, groups = d.groups, group_warps = d.group_warps, nbox = d.nbox;
  const int dbg = MM_RQ_EXPERIMENTS ? d.dbg : 0;
  const int64_t rows = a.rows;
  const int fm1 = a.geom.fmt[1], fm2 = a.geom.fmt[2];
  // Gather table: u16 slot byte offsets, two per word, [block][16 words]: the lane
  // holding half h of block b reads words 16 b + 8 h .. + 7 with two 128-bit loads
  // (the warp reads 1 KB contiguously: conflict free).
  const int tab = U16 ? (d.perm_smem == 1 ? 1 : 2) : d.perm_smem;
  if (tab) {
    if (tab == 1 || tab == 3) ptx::mbar_wait(ptx::smem_u32(permbar), 0, 13, 0, 0);
    const int ct = threadIdx.x - 32, cn = groups * group_warps * 32;
    // Table layouts are swizzled per lane so that the warp-wide 128-bit table loads of
    // the gather are bank-conflict free: lane l of a chunk reads its vector q at
    // "rotated" slot (q + rot(l)) of its own group (see tile_chunks).
    const uint32_t sz = (uint32_t)sizeof(ST);
    // slot of channel p: the layout moves 4-channel chunks inside each 32-channel line
    auto slot = [layout, lay_w](uint32_t p) -> uint32_t {
      if (!layout) return p;
      return (p & ~31u) | (((lay_w[p >> 5] >> (4 * ((p >> 2) & 7))) & 7u) << 2) | (p & 3u);
    };
    if (layout && !LX)   // one word per 32-channel line of every box; lines past K keep the natural order
      for (int t = ct; t < 8 * nbox; t += cn) lay_s[t] = t < K / 32 ? __ldg(layout + t) : 0x76543210u;
    if (tab == 3) {   // in place, one 16-position group per thread: perm[j] -> slot byte offset
      for (int t = ct; t < K / 16; t += cn) {
        const int r = (t >> 1) & 3;
        uint4* g = reinterpret_cast<uint4*>(gidx) + 4 * t;
        uint4 w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          w[q] = g[q];
          w[q].x = slot(w[q].x) * sz; w[q].y = slot(w[q].y) * sz; w[q].z = slot(w[q].z) * sz; w[q].w = slot(w[q].w) * sz;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) g[(q + r) & 3] = w[q];
      }
    } else {          // u16 pairs, one 16-position group (8 words) per thread
      for (int t = ct; t < K / 16; t += cn) {
        const int r = (t >> 2) & 1;
        uint4 pv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          pv[q] = tab == 1 ? reinterpret_cast<const uint4*>(perm_s)[4 * t + q]
                           : __ldg(reinterpret_cast<const uint4*>(a.perm) + 4 * t + q);
        uint4* g = reinterpret_cast<uint4*>(gidx) + 2 * t;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          pv[q].x = slot(pv[q].x) * sz; pv[q].y = slot(pv[q].y) * sz;
          pv[q].z = slot(pv[q].z) * sz; pv[q].w = slot(pv[q].w) * sz;
        }
        g[r] = make_uint4(pv[0].x | pv[0].y << 16, pv[0].z | pv[0].w << 16, pv[1].x | pv[1].y << 16,
                          pv[1].z | pv[1].w << 16);
        g[r ^ 1] = make_uint4(pv[2].x | pv[2].y << 16, pv[2].z | pv[2].w << 16, pv[3].x | pv[3].y << 16,
                              pv[3].z | pv[3].w << 16);
      }
    }
  }
  if constexpr (LX) {
    // Transpose store offsets: for lane l of box b, the byte offsets inside the box of its two
    // 16-byte chunks, the one stored first in the low half.  Lane l owns chunks 2 (l & 3) and
    // 2 (l & 3) + 1 of 32-channel line l / 4; lanes 4..7 of every 8 store their odd chunk
    // first (8 bank groups per store instruction); the chunk positions come from the plan's
    // parity-preserving gather layout (natural order without one and past K).
    const int ct = threadIdx.x - 32, cn = groups * group_warps * 32;
    for (int t = ct; t < 32 * nbox; t += cn) {
      const int l = t & 31, li = 8 * (t >> 5) + (l >> 2);
      const uint32_t qf = 2u * (uint32_t)(l & 3) + (uint32_t)((l >> 2) & 1);
      uint32_t pf = qf, ps = qf ^ 1u;
      if (layout && li < K / 32) {
        const uint32_t lw = lay_w[li];
        pf = (lw >> (4 * qf)) & 7u;
        ps = (lw >> (4 * (qf ^ 1u))) & 7u;
      }
      const uint32_t base = (uint32_t)(l >> 2) * 128u;
      lay_s[t] = (base + 16u * pf) | ((base + 16u * ps) << 16);
    }
  }
  if (tab || LX) {
    ptx::named_bar_sync(15, groups * group_warps * 32);
    if ((MM_RQ_EXPERIMENTS && (d.dbg & 32)) && threadIdx.x == 32) g_rq_trace[blockIdx.x][1] = ptx::globaltimer_ns();
  }
  ptx::grid_dep_wait();   // the outputs may still be read by the preceding kernel
  if constexpr (NORM) {   // gamma in reordered channel order
    const int ct = threadIdx.x - 32, cn = groups * group_warps * 32;
    for (int j = ct; j < K; j += cn) {
      const int pj = d.perm_smem == 1 ? perm_s[j] : __ldg(a.perm + j);   // (tab 3: perm_s already rewritten)
      gamma_r[j] = __ldg(a.gamma + pj);
    }
    ptx::named_bar_sync(15, cn);
  }
  const double eps = a.eps;
  // Work is split into chunks of 16 consecutive 32-channel blocks of the reordered
  // row (tile_chunks; the two lanes of a pair share a block, 16 channels each).  Warp
  // gw of a group owns the chunks ch = gw (mod group_warps), the same in every tile;
  // its last warp also zeroes the storage padding blocks (tile_padding).
  const bool e3m2 = fm1 == F_E3M2, e4m3 = fm2 == F_E4M3;
  const bool has_pad = a.geom.kp[0] != a.geom.n[0] || a.geom.kp[1] != a.geom.n[1] || a.geom.kp[2] != a.geom.n[2];
  int s = grp;           // ring slot and phase of tile i, advanced incrementally
  uint32_t ph = 0;       // (groups < stages: at most one wrap per step)
  for (int64_t i = grp; i < my_tiles; i += groups) {
    uint8_t* st = smem + (size_t)s * stage_bytes;
    ptx::mbar_wait(ptx::smem_u32(&full[s]), ph, 12, s, (int)i);
    if ((MM_RQ_EXPERIMENTS && (d.dbg & 32)) && gw == 0 && lane == 0 && i < 6) g_rq_trace[blockIdx.x][2 + 2 * i] = ptx::globaltimer_ns();
    // ---- in-place transpose: box [R rows][256] -> 256 slots of R values ----
    // (NORM: the exact per-row sums of squares are accumulated from the same
    // registers, so the norm needs no second pass over the stage.)
    double nhi[4] = {0, 0, 0, 0}, nlo[4] = {0, 0, 0, 0};
    if constexpr (R > 1) {
      if constexpr (LX) {
        // Lane l owns channels 8 l .. 8 l + 7 of each box; it reads its row words as two
        // 8-byte halves in store order (no register selects) and stores the two transposed
        // 16-byte chunks at the offsets lay_s holds for (box, lane).  Shared addresses are
        // 32-bit with a warp-uniform box base.
        const uint32_t f8 = 8u * (uint32_t)((lane >> 2) & 1);
        const uint32_t rf = (uint32_t)lane * 16u + f8, rs = (uint32_t)lane * 16u + (f8 ^ 8u);
        const uint32_t st_b = __reduce_max_sync(0xffffffffu, ptx::smem_u32(st));
        const uint32_t lx = ptx::smem_u32(lay_s) + 4u * (uint32_t)lane;
        for (int b = gw; b < nbox && !(dbg & 2); b += group_warps) {
          const uint32_t box = st_b + (uint32_t)b * 1024u;
          uint2 a0, a1, b0, b1;
          asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(a0.x), "=r"(a0.y) : "r"(box + rf));
          asm volatile("ld.shared.v2.b32 {%0, %1}, [%2+512];" : "=r"(a1.x), "=r"(a1.y) : "r"(box + rf));
          asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(b0.x), "=r"(b0.y) : "r"(box + rs));
          asm volatile("ld.shared.v2.b32 {%0, %1}, [%2+512];" : "=r"(b1.x), "=r"(b1.y) : "r"(box + rs));
          uint32_t w;
          asm volatile("ld.shared.b32 %0, [%1];" : "=r"(w) : "r"(lx + (uint32_t)b * 128u));
          __syncwarp();
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(box + (w & 0xFFFFu)),
                       "r"(__byte_perm(a0.x, a1.x, 0x5410)), "r"(__byte_perm(a0.x, a1.x, 0x7632)),
                       "r"(__byte_perm(a0.y, a1.y, 0x5410)), "r"(__byte_perm(a0.y, a1.y, 0x7632)) : "memory");
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(box + (w >> 16)),
                       "r"(__byte_perm(b0.x, b1.x, 0x5410)), "r"(__byte_perm(b0.x, b1.x, 0x7632)),
                       "r"(__byte_perm(b0.y, b1.y, 0x5410)), "r"(__byte_perm(b0.y, b1.y, 0x7632)) : "memory");
        }
      } else
      for (int b = gw; b < nbox && !(dbg & 2); b += group_warps) {
        uint8_t* box = st + b * 512 * R;
        uint4 w[R];
#pragma unroll
        for (int rho = 0; rho < R; ++rho) w[rho] = *reinterpret_cast<const uint4*>(box + rho * 512 + lane * 16);
        __syncwarp();
        if constexpr (NORM) {
#pragma unroll
          for (int rho = 0; rho < R; ++rho) {
            const uint32_t* u = reinterpret_cast<const uint32_t*>(&w[rho]);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const double x0 = bf16_f64(u[k] & 0xFFFFu), x1 = bf16_f64(u[k] >> 16);
              dd_add(nhi[rho], nlo[rho], x0 * x0);
              dd_add(nhi[rho], nlo[rho], x1 * x1);
            }
          }
        }
        const uint32_t* u0 = reinterpret_cast<const uint32_t*>(&w[0]);
        const uint32_t* u1 = reinterpret_cast<const uint32_t*>(&w[1]);
        if constexpr (R == 2) {
          // lane l writes 16-byte chunks 2l and 2l+1; lanes 4..7 of every 8 write their odd
          // chunk first, so the 8 chunks of each store instruction fill 8 different bank
          // groups (4 wavefronts per 512 B instead of 8)
          const uint4 c0 = make_uint4(__byte_perm(u0[0], u1[0], 0x5410), __byte_perm(u0[0], u1[0], 0x7632),
                                      __byte_perm(u0[1], u1[1], 0x5410), __byte_perm(u0[1], u1[1], 0x7632));
          const uint4 c1 = make_uint4(__byte_perm(u0[2], u1[2], 0x5410), __byte_perm(u0[2], u1[2], 0x7632),
                                      __byte_perm(u0[3], u1[3], 0x5410), __byte_perm(u0[3], u1[3], 0x7632));
          const bool f = (lane & 4) != 0;
          // chunk positions inside this lane's 128-byte line: natural, or the plan's
          // parity-preserving gather layout (an odd chunk stays odd: still 8 bank groups
          // per store instruction)
          int p0 = 2 * (lane & 3), p1 = p0 + 1;
          const int li = 8 * b + (lane >> 2);   // 32-channel line of this lane's chunks
          if (layout && li < K / 32) {          // lines past K (the last box's OOB tail) stay natural
            const uint32_t lw = lay_s[li];
            p0 = (lw >> (4 * p0)) & 7;
            p1 = (lw >> (4 * p1)) & 7;
          }
          uint4* line = reinterpret_cast<uint4*>(box + (lane >> 2) * 128);
          line[f ? p1 : p0] = f ? c1 : c0;
          line[f ? p0 : p1] = f ? c0 : c1;
        } else {
          const uint32_t* u2 = reinterpret_cast<const uint32_t*>(&w[2]);
          const uint32_t* u3 = reinterpret_cast<const uint32_t*>(&w[3]);
          // lane l writes its 4 chunks in the order k = (j + l / 2) % 4: the 8 lanes of
          // each 128-byte bank window then hit 8 different bank groups (4 wavefronts per
          // 512 B store instruction instead of 16)
          uint4* o = reinterpret_cast<uint4*>(box + lane * 64);
          uint4 c[4];
#pragma unroll
          for (int k = 0; k < 4; ++k)
            c[k] = make_uint4(__byte_perm(u0[k], u1[k], 0x5410), __byte_perm(u2[k], u3[k], 0x5410),
                              __byte_perm(u0[k], u1[k], 0x7632), __byte_perm(u2[k], u3[k], 0x7632));
          const int rot = (lane >> 1) & 3;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int k = (j + rot) & 3;
            o[k] = k == 0 ? c[0] : (k == 1 ? c[1] : (k == 2 ? c[2] : c[3]));
          }
        }
      }
      ptx::named_bar_sync(1 + grp, gthreads);
    }
    // ---- gather + quantize + pack + store ----
    if (dbg & 3) {
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(ptx::smem_u32(&empty[s]));
    } else {
      float rn[4] = {0.f, 0.f, 0.f, 0.f};
      if constexpr (NORM) {
        const ST* slots = reinterpret_cast<const ST*>(st);
        // exact per-row sums of squares (double-double), group reduction in a fixed order
        double hi[4] = {nhi[0], nhi[1], nhi[2], nhi[3]}, lo[4] = {nlo[0], nlo[1], nlo[2], nlo[3]};
        for (int pc = gw * 32 + lane; R == 1 && pc < K; pc += gthreads) {   // R > 1: summed in the transpose
          const ST v = slots[pc];
          { const double x = bf16_f64(slot_bits<0>(v)); dd_add(hi[0], lo[0], x * x); }
          if constexpr (R >= 2) { const double x = bf16_f64(slot_bits<1>(v)); dd_add(hi[1], lo[1], x * x); }
          if constexpr (R >= 4) {
            { const double x = bf16_f64(slot_bits<2>(v)); dd_add(hi[2], lo[2], x * x); }
            { const double x = bf16_f64(slot_bits<3>(v)); dd_add(hi[3], lo[3], x * x); }
          }
        }
#pragma unroll
        for (int rho = 0; rho < R; ++rho)
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const double oh = __shfl_xor_sync(0xffffffffu, hi[rho], o), ol = __shfl_xor_sync(0xffffffffu, lo[rho], o);
            dd_add_dd(hi[rho], lo[rho], oh, ol);
          }
        // scratch: [consumer warp (<= 31)][rho][hi, lo] doubles, then [group][rho] norms
        double* red = nred + (grp * group_warps) * 8;
        if (lane == 0)
#pragma unroll
          for (int rho = 0; rho < R; ++rho) { red[gw * 8 + 2 * rho] = hi[rho]; red[gw * 8 + 2 * rho + 1] = lo[rho]; }
        ptx::named_bar_sync(1 + grp, gthreads);
        if (gw == 0 && lane < R) {
          double h2 = 0.0, l2 = 0.0;
          for (int ww = 0; ww < group_warps; ++ww) dd_add_dd(h2, l2, red[ww * 8 + 2 * lane], red[ww * 8 + 2 * lane + 1]);
          const double ss = h2 + l2;
          nred[32 * 8 + grp * 4 + lane] = (double)(float)(1.0 / sqrt(ss / (double)K + eps));   // fp32 row scale
        }
        ptx::named_bar_sync(1 + grp, gthreads);
#pragma unroll
        for (int rho = 0; rho < R; ++rho) rn[rho] = (float)nred[32 * 8 + grp * 4 + rho];
      }
      // (through a warp reduction: a uniform register, so the per-tile row bases of the
      // code / scale stores stay uniform instead of being rematerialised per store)
      const int64_t r0 = (int64_t)__reduce_max_sync(0xffffffffu, (unsigned)((blockIdx.x + i * gridDim.x) * R));
      const int64_t left = rows - r0;
      const int nvalid = left >= R ? R : (left > 0 ? (int)left : 0);
      const ChunkCtx<R> cx{st, smem, gidx, gamma_r, (int)r0, nvalid, group_warps, lane, dbg, tab};
      tile_chunks<R, NORM, U16>(a, cx, gw, e3m2, e4m3, rn);
      if (gw == group_warps - 1 && has_pad && !(dbg & 16)) tile_padding<R>(a, (int)r0, nvalid, lane);
      if ((MM_RQ_EXPERIMENTS && (d.dbg & 32)) && gw == 0 && lane == 0 && i < 6) g_rq_trace[blockIdx.x][3 + 2 * i] = ptx::globaltimer_ns();
      if ((MM_RQ_EXPERIMENTS && (d.dbg & 32)) && gw == 0 && lane == 0) g_rq_trace[blockIdx.x][15] = ptx::globaltimer_ns();
      // ---- release the stage (every warp of the group arrives once) ----
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(ptx::smem_u32(&empty[s]));
    }
    s += groups;
    if (s >= stages) { s -= stages; ph ^= 1u; }
  }
}

__global__ void reorder_bf16_kernel(const uint16_t* __restrict__ x, int64_t rows, int64_t ldx,
                                    int K, const int32_t* __restrict__ perm,
                                    uint16_t* __restrict__ xr, int64_t ldxr) {
  const int64_t r = blockIdx.y;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < K; j += gridDim.x * blockDim.x)
    xr[r * ldxr + j] = x[r * ldx + perm[j]];
}

template <int R, bool NORM>
cudaError_t launch_rq_t(const RqArgs& a, cudaStream_t s, int64_t* launches) {
  EncodeTiledFn enc = tensor_map_encoder();
  if (!enc) return cudaErrorNotSupported;
  RqDev d{};
  d.a = a;
  const int64_t rows_pad = (a.rows + 127) / 128 * 128;
  d.n_tiles = rows_pad / R;
  d.nbox = (a.K + 255) / 256;
  const size_t stage_bytes = (size_t)d.nbox * 512 * R;
  // Stage the permutation in smem (gather table) when that still leaves >= 3 stages.
  // Gather table in smem: with an asynchronous copy of the permutation when that still
  // leaves >= 3 stages (mode 1), else built straight from global memory (mode 2: large K,
  // where the one-time prologue is amortised over many tiles), else none (L1 reads).
  // Gather table: u32 slot offsets made in place from the bulk-copied permutation
  // (mode 3: no offset unpacking in the gather, opt-in) when that leaves >= 3 stages; else u16
  // offsets two per word, from a bulk copy (mode 1, >= 3 stages) or built straight from
  // global memory (mode 2, >= 2 stages: large K, one-time prologue amortised over many
  // tiles); else none (L1 reads of the permutation).
  const size_t norm_need = a.gamma ? ((size_t)a.K * 2 + 255) / 256 * 256 + 4096 : 0;
  const size_t budget = kRqSmemBudget - norm_need;
  const size_t gtab = ((size_t)a.K * 2 + 15) / 16 * 16;
  const size_t tab_need = (size_t)a.K * 4 + gtab;
  // Mode 3 is opt-in (MM_RQ_TAB32=1): measured 3 % slower than mode 1 at M = 16384,
  // K = 4096 (the two extra table loads per lane cost more than the offset unpacking).
  static const int tab32 = [] { const char* e = getenv("MM_RQ_TAB32"); return e ? atoi(e) : 0; }();
  if (tab32 && a.K % 4 == 0 && (budget - (size_t)a.K * 4) / stage_bytes >= 3) d.perm_smem = 3;
  else d.perm_smem = (budget - tab_need) / stage_bytes >= 3 ? 1 : ((budget - gtab) / stage_bytes >= 2 ? 2 : 0);
  { const char* e = getenv("MM_RQ_TABMODE"); if (e && atoi(e) >= 0 && atoi(e) <= 3) d.perm_smem = atoi(e); }   // tuning
  if (d.perm_smem != 3 && (size_t)a.K * 2 * R > 65536) d.perm_smem = 0;   // u16 table holds byte offsets
  size_t tab_bytes = d.perm_smem == 3 ? (size_t)a.K * 4 : (d.perm_smem == 1 ? tab_need : (d.perm_smem == 2 ? gtab : 0));
  // gather layout (R = 2 with a table only): per-line words for the transpose
  static const int no_layout = [] { const char* e = getenv("MM_RQ_NO_LAYOUT"); return e ? atoi(e) : 0; }();  // A/B
  if (R != 2 || d.perm_smem == 0 || no_layout) d.a.layout = nullptr;
  // transpose offsets (R = 2 without the norm: one word per box and lane) or layout words
  // (R = 2 with the norm: one per 32-channel line of every box)
  if (R == 2 && !NORM) tab_bytes += (size_t)d.nbox * 128;
  else if (d.a.layout) tab_bytes += (size_t)d.nbox * 32;
  // the layout words travel with the permutation's bulk copy (mode 1; whole 16-byte units):
  // the table build then reads them from shared memory, not through an L2 round trip
  static const int no_lay_copy = [] { const char* e = getenv("MM_RQ_NO_LAYCOPY"); return e ? atoi(e) : 0; }();  // A/B
  d.lay_copy = (d.a.layout && d.perm_smem == 1 && a.K % 128 == 0 && !no_lay_copy) ? 1 : 0;
  if (d.lay_copy) tab_bytes += (size_t)a.K / 8;
  int stages = (int)((budget - tab_bytes) / stage_bytes);
  if (stages > 32) stages = 32;
  { const char* e = getenv("MM_RQ_STAGES"); if (e && atoi(e) >= 2 && atoi(e) < stages) stages = atoi(e); }
  if (stages < 2) return cudaErrorInvalidConfiguration;
  d.stages = stages;
  // Consumer layout: W warps (register budget) in `groups` groups of gw warps; a group
  // works on one tile, warp gw of it on chunks gw, gw + group_warps, ... .  Per-tile
  // overhead (ring wait, transpose barrier, row bases) is paid per warp, so each warp
  // should own several chunks (~5 measured best); more groups need more stages.
  const int nch = (a.K / 32 + 15) / 16;   // chunks per tile (tile_chunks)
  const int W = rq_max_threads(R, NORM) / 32 - 1;
  int gw = (nch + 4) / 5;
  if (gw < 1) gw = 1;
  if (gw > W) gw = W;
  int groups = W / gw;
  // Ring lookahead: each group holds its stage while it works on the tile, so only
  // stages - groups tiles can be in flight from HBM ahead of the groups.
  // Two tiles of lookahead where the ring is deep (K = 4096, 12 stages: 10 groups instead
  // of 11, 16384 x 4096 41.2 -> 39.0 us); one where stages are scarce (K = 14336: 3
  // stages, 2 groups -- one group of 23 warps is 28 % slower).  MM_RQ_LOOKAHEAD: tuning.
  static const int look_env = [] { const char* e = getenv("MM_RQ_LOOKAHEAD"); return e ? atoi(e) : 0; }();
  const int look = look_env >= 1 ? look_env : (stages >= 8 ? 2 : 1);
  const int max_groups = stages - look > 1 ? stages - look : 1;
  if (groups > max_groups) {   // stage-limited: fewer, larger groups that still use every warp
    groups = max_groups;
    gw = W / groups;
    if (gw > nch) gw = nch;
  }
  // Few tiles per CTA (small M): no more groups than tiles, each with more warps, so
  // every warp has work in the first round and a tile's latency shrinks.
  const int64_t grid_est = d.n_tiles < (int64_t)sm_count() ? d.n_tiles : (int64_t)sm_count();
  const int64_t tpc = (d.n_tiles + grid_est - 1) / grid_est;
  if (groups > tpc) {
    groups = (int)tpc;
    gw = W / groups;
    if (gw > nch) gw = nch;
  } else if (tpc <= 32 && groups > 7) {
    // A few rounds of tiles per CTA (M up to ~8192 at K = 4096): the last round's latency
    // matters more than the lookahead -- 7 groups of 3 warps instead of 10 of 2 (M = 4096:
    // 13.43 -> 12.86 us, M = 8192: 22.21 -> 21.77 us; M = 16384, 55 tiles per CTA, keeps 10)
    groups = 7;
    gw = W / groups;
    if (gw > nch) gw = nch;
  }
  const char* gw_env = getenv("MM_RQ_GW");   // tuning
  if (gw_env && atoi(gw_env) >= 1 && atoi(gw_env) <= W) { gw = atoi(gw_env); groups = W / gw; } else gw_env = nullptr;
  { const char* e = getenv("MM_RQ_GROUPS"); if (e && atoi(e) >= 1 && atoi(e) <= W) { groups = atoi(e); gw = W / groups; if (gw > nch) gw = nch; } }
  if (groups > max_groups) groups = max_groups;
  if (groups < 1) groups = 1;
  if (!gw_env) {
    // Group width: the fewest warps that still give the fewest chunk rounds per tile
    // (ceil(nch / gw)), within the register budget -- K = 28672: 14 warps, 4 rounds
    // (was 12 warps, 5 rounds: 142.4 -> 140.7 us); K = 27648: 141.6 -> 135.3 us.
    const int gmax = W / groups > 0 ? W / groups : 1;
    const int best_rounds = (nch + gmax - 1) / gmax;
    gw = gmax;
    while (gw > 1 && (nch + gw - 2) / (gw - 1) == best_rounds) --gw;
  }
  d.group_warps = gw;
  d.groups = groups;
  { const char* e = getenv("MM_RQ_DEBUG"); d.dbg = e ? atoi(e) : 0; }
  // TMA map over X.  Preferred: a 3-D view {256 channels, rows, K/256 boxes} with
  // strides {ldx*2, 512 B}, so ONE load per tile lands box-major ([box][R][256]);
  // else (K % 256 != 0, or the driver rejects the view) 2-D boxes of 256 x R.
  CUtensorMap m;
  d.box3d = 0;
  const char* no3d = getenv("MM_RQ_NO3D");   // timing experiments only
  if (a.K % 256 == 0 && d.nbox <= 256 && !(no3d && atoi(no3d))) {
    cuuint64_t dims[3] = {256, (cuuint64_t)a.rows, (cuuint64_t)d.nbox};
    cuuint64_t strides[2] = {(cuuint64_t)a.ldx * 2, 512};
    cuuint32_t box[3] = {256, (cuuint32_t)R, (cuuint32_t)d.nbox};
    cuuint32_t estr[3] = {1, 1, 1};
    if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, const_cast<uint16_t*>(a.x), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
      d.box3d = 1;
  }
  if (!d.box3d) {
    cuuint64_t dims[2] = {(cuuint64_t)a.K, (cuuint64_t)a.rows};
    cuuint64_t strides[1] = {(cuuint64_t)a.ldx * 2};
    cuuint32_t box[2] = {256, (cuuint32_t)R};
    cuuint32_t estr[2] = {1, 1};
    if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, const_cast<uint16_t*>(a.x), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  const size_t norm_bytes = a.gamma ? ((size_t)a.K * 2 + 255) / 256 * 256 + 4096 : 0;
  const size_t smem = 1024 + (size_t)stages * stage_bytes + tab_bytes + norm_bytes + (2 * stages + 1) * 8;
  const bool u16 = d.perm_smem == 1 || d.perm_smem == 2;
  auto kern = u16 ? rq_kernel<R, NORM, true> : rq_kernel<R, NORM, false>;
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), smem);
  if (e != cudaSuccess) return e;
  const int threads = 32 * (1 + groups * gw);
  int64_t grid = sm_count();
  if (grid > d.n_tiles) grid = d.n_tiles;
  e = launch_pdl(kern, dim3((unsigned)grid), dim3(threads), smem, s, m, d);
  if (launches) ++*launches;
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace

cudaError_t launch_reorder_quantize(const RqArgs& a, cudaStream_t s, int64_t* launches) {
  if (a.rows == 0) return cudaSuccess;
  const size_t row_bytes = (size_t)((a.K + 255) / 256) * 512;
  static const int force_r = [] { const char* e = getenv("MM_RQ_ROWS"); return e ? atoi(e) : 0; }();  // tuning
  if (force_r == 2) return (a.gamma ? launch_rq_t<2, true>(a, s, launches) : launch_rq_t<2, false>(a, s, launches));
  if (force_r == 1) return (a.gamma ? launch_rq_t<1, true>(a, s, launches) : launch_rq_t<1, false>(a, s, launches));
  if (force_r == 4) return (a.gamma ? launch_rq_t<4, true>(a, s, launches) : launch_rq_t<4, false>(a, s, launches));
  // Two-row tiles while >= 3 stages fit (measured faster than four-row tiles at
  // q_proj: twice the tiles balance the persistent grid, fewer registers per lane
  // allow more consumer warps), single rows beyond.
  if (2 * row_bytes * 3 <= kRqSmemBudget && a.K * 4 <= 65536) return (a.gamma ? launch_rq_t<2, true>(a, s, launches) : launch_rq_t<2, false>(a, s, launches));
  return (a.gamma ? launch_rq_t<1, true>(a, s, launches) : launch_rq_t<1, false>(a, s, launches));
}

}  // namespace mmx
extern "C" int mm_debug_rq_trace(unsigned long long* h, int n) {
  return (int)cudaMemcpyFromSymbol(h, mmx::g_rq_trace, sizeof(unsigned long long) * (size_t)(n < 2560 ? n : 2560));
}
namespace mmx {

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
