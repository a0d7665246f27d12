// gemm.cu -- the MicroMix mixed-precision block-scaled GEMM on sm_100a
// (§3.2 "GEMM Kernel", line 143; Fig. 5 caption line 137; Eq. 2,
// lines 47-51): Y[M, N] (BF16) = sum over the MXFP4, MXFP6 and MXFP8 K-segments
// of A_g W_g^T with E8M0 block scales, one FP32 accumulator.
//
// B200-native design: instead of the paper's three
// decoupled CUTLASS GEMMs, ONE persistent warp-specialised kernel walks all
// three segments in a single K loop and accumulates into a single TMEM tile:
//   * every pipeline stage holds 128-byte smem rows for A (128 rows) and W
//     (BN rows): FP4 stage = 256 K (packed, 4 x tcgen05.mma kind::mxf4, K=64),
//     FP6 stage = 128 K (TMA 16U6_ALIGN16B unpacks 16 x 6 bit into 16 bytes,
//     4 x kind::mxf8f6f4 e3m2/e2m3, K=32), FP8 stage = 128 K (4 x
//     kind::mxf8f6f4 e4m3/e5m2) -- identical smem footprint and MMA count, only
//     the tensor map, the instruction descriptor and the number of scale atoms
//     change per segment;
//   * warp 0: TMA producer (128B-swizzled operand tiles + 512-byte scale atoms
//     via cp.async.bulk, all completing on one mbarrier per stage);
//   * warp 1: single-thread MMA issuer: tcgen05.cp scale atoms smem -> TMEM,
//     4 block-scaled tcgen05.mma per stage (only ceil(tail/K_mma) in a
//     segment's last stage), tcgen05.commit frees the stage;
//   * warps 4-7: epilogue, tcgen05.ld FP32 -> cvt.rn.bf16x2 -> global;
//   * warp 2 owns the TMEM allocation (512 columns; accumulators double
//     buffered when they fit next to the scale columns).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "internal.h"
#include "ptx.cuh"

namespace mmx {
namespace {

constexpr int BM = 128;
constexpr int ROW_BYTES = 128;     // smem bytes per operand row per stage
constexpr int kThreads = 256;

struct GemmDev {
  int64_t M, N;
  int num_m, num_n, num_tiles;
  int nst[3];            // stages per segment
  int n[3], kp[3];
  const uint8_t* sfa[3];
  const uint8_t* sfb[3];
  int64_t sfb_rows_pad;  // roundup(N, 128)
  uint32_t idesc[3];     // instruction descriptors (sf ids = 0)
  uint16_t* y;
  int64_t ldy;
  int dbg;               // timing experiments only (env MM_GEMM_DEBUG): 1 = SF copy once per tile, 2 = no MMA
};

template <int BN, int STAGES>
struct Cfg {
  static constexpr int A_BYTES = BM * ROW_BYTES;
  static constexpr int B_BYTES = BN * ROW_BYTES;
  static constexpr int RG = BN / 128;               // 128-row scale groups of W per tile
  static constexpr int SFA_BYTES = 2 * 512;
  static constexpr int SFB_BYTES = 2 * RG * 512;
  // TMEM columns: [accumulator(s) | one scale-factor slot per smem stage].  A slot
  // holds up to 2 atoms of SFA (4 columns each) and 2 x RG atoms of SFB.  Giving
  // every pipeline stage its own slot removes the write-after-read hazard between
  // stage i's MMAs and stage i+1's tcgen05.cp, so the tensor pipe never drains.
  static constexpr int SF_STRIDE = 8 + 8 * RG;
  static constexpr int NUM_ACC = (2 * BN + STAGES * SF_STRIDE <= 512) ? 2 : 1;
  static constexpr int SF_BASE = NUM_ACC * BN;
  static_assert(NUM_ACC * BN + STAGES * SF_STRIDE <= 512, "TMEM budget");
};

struct StageInfo {
  int g;        // segment
  int kcoord;   // TMA inner coordinate (bytes for FP4/FP8, elements for FP6)
  int nmma;     // MMAs to issue
  int atoms;    // scale atoms (512 B per 128 rows)
  int atom0;    // first atom index inside the segment
};

__device__ __forceinline__ StageInfo stage_info(const GemmDev& p, int s) {
  StageInfo si;
  if (s < p.nst[0]) {
    const int j = s;
    const int real = min(p.n[0] - 256 * j, 256);
    si.g = 0;
    si.kcoord = 128 * j;                     // bytes (2 E2M1 per byte)
    si.nmma = (real + 63) / 64;
    si.atoms = min(p.kp[0] - 256 * j, 256) / 128;
    si.atom0 = 2 * j;
  } else {
    const int g = (s < p.nst[0] + p.nst[1]) ? 1 : 2;
    const int j = s - p.nst[0] - (g == 2 ? p.nst[1] : 0);
    const int real = min(p.n[g] - 128 * j, 128);
    si.g = g;
    si.kcoord = 128 * j;                     // elements (FP6 map) == bytes (FP8 map)
    si.nmma = (real + 31) / 32;
    si.atoms = 1;
    si.atom0 = j;
  }
  return si;
}

template <int BN, int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
mixgemm_kernel(const __grid_constant__ CUtensorMap ta0, const __grid_constant__ CUtensorMap ta1,
               const __grid_constant__ CUtensorMap ta2, const __grid_constant__ CUtensorMap tb0,
               const __grid_constant__ CUtensorMap tb1, const __grid_constant__ CUtensorMap tb2,
               const GemmDev p) {
  using C = Cfg<BN, STAGES>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = sA + STAGES * C::A_BYTES;
  uint8_t* sSFA = sB + STAGES * C::B_BYTES;
  uint8_t* sSFB = sSFA + STAGES * C::SFA_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sSFB + STAGES * C::SFB_BYTES);
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  uint64_t* tfull = bars + 2 * STAGES;
  uint64_t* tempty = tfull + C::NUM_ACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + C::NUM_ACC);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&ta0); ptx::tma_prefetch_desc(&ta1); ptx::tma_prefetch_desc(&ta2);
    ptx::tma_prefetch_desc(&tb0); ptx::tma_prefetch_desc(&tb1); ptx::tma_prefetch_desc(&tb2);
  }
  if (warp == 1 && lane == 0) {
    for (int i = 0; i < STAGES; ++i) {
      ptx::mbar_init(ptx::smem_u32(&full[i]), 1);
      ptx::mbar_init(ptx::smem_u32(&empty[i]), 1);
    }
    for (int i = 0; i < C::NUM_ACC; ++i) {
      ptx::mbar_init(ptx::smem_u32(&tfull[i]), 1);
      ptx::mbar_init(ptx::smem_u32(&tempty[i]), 128);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc(ptx::smem_u32(tmem_slot), 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int nstages = p.nst[0] + p.nst[1] + p.nst[2];

  if (warp == 0 || warp == 3) {
    // ============================ TMA producers ============================
    // warp 0: transaction count + A and W tiles; warp 3: the scale atoms (two issuing
    // threads, as in the CTA-pair kernel).
    const bool ops = warp == 0;
    if (lane == 0) {
      const CUtensorMap* ta[3] = {&ta0, &ta1, &ta2};
      const CUtensorMap* tb[3] = {&tb0, &tb1, &tb2};
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
        const int mb = t % p.num_m, nb = t / p.num_m;
        const int m0 = mb * BM, n0 = nb * BN;
        for (int s = 0; s < nstages; ++s) {
          const StageInfo si = stage_info(p, s);
          ptx::mbar_wait(ptx::smem_u32(&empty[stage]), phase ^ 1, 1, s, t);
          const uint32_t fb = ptx::smem_u32(&full[stage]);
          const int kp128 = p.kp[si.g] / 128;
          // TMA counts transaction bytes in GLOBAL element bits: a 16U6 (FP6) box of
          // 128 elements x rows lands as 128 B per smem row but completes 96 B per row.
          uint32_t bytes = (si.g == 1 ? (C::A_BYTES + C::B_BYTES) / 4 * 3 : C::A_BYTES + C::B_BYTES) +
                           si.atoms * 512;
          int nrg = 0;
#pragma unroll
          for (int rg = 0; rg < C::RG; ++rg)
            if ((int64_t)(n0 / 128 + rg) * 128 < p.sfb_rows_pad) ++nrg;
          bytes += nrg * si.atoms * 512;
          if (ops) {
            ptx::mbar_arrive_expect_tx(fb, bytes);
            ptx::tma_load_2d(ptx::smem_u32(sA + stage * C::A_BYTES), ta[si.g], fb, si.kcoord, m0);
            ptx::tma_load_2d(ptx::smem_u32(sB + stage * C::B_BYTES), tb[si.g], fb, si.kcoord, n0);
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
            continue;
          }
          const uint8_t* a_src = p.sfa[si.g] + ((int64_t)mb * kp128 + si.atom0) * 512;
          ptx::bulk_load(ptx::smem_u32(sSFA + stage * C::SFA_BYTES), a_src, si.atoms * 512, fb);
          for (int rg = 0; rg < nrg; ++rg) {
            const uint8_t* b_src = p.sfb[si.g] + ((int64_t)(n0 / 128 + rg) * kp128 + si.atom0) * 512;
            for (int at = 0; at < si.atoms; ++at)
              ptx::bulk_load(ptx::smem_u32(sSFB + stage * C::SFB_BYTES + (at * C::RG + rg) * 512),
                             b_src + at * 512, 512, fb);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer ============================
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x, ++it) {
      const int acc = it % C::NUM_ACC;
      const uint32_t acc_phase = (it / C::NUM_ACC) & 1;
      ptx::mbar_wait(ptx::smem_u32(&tempty[acc]), acc_phase ^ 1, 2, it, t);
      ptx::tc_fence_after();
      const uint32_t d_t = tmem_base + acc * BN;
      for (int s = 0; s < nstages; ++s) {
        const StageInfo si = stage_info(p, s);
        ptx::mbar_wait(ptx::smem_u32(&full[stage]), phase, 3, s, t);
        ptx::tc_fence_after();
        const uint32_t sfa_t = tmem_base + C::SF_BASE + stage * C::SF_STRIDE;
        const uint32_t sfb_t = sfa_t + 8;
        const uint32_t a_base = ptx::smem_u32(sA + stage * C::A_BYTES);
        const uint32_t b_base = ptx::smem_u32(sB + stage * C::B_BYTES);
        if (si.nmma == 4 && !p.dbg) {
          // full stage: one issue block (elect.sync, scale copies, 4 MMAs, commit)
          const uint64_t ad = ptx::smem_desc(a_base, 16, 1024, 2), bd = ptx::smem_desc(b_base, 16, 1024, 2);
          const uint64_t sda = ptx::smem_desc(ptx::smem_u32(sSFA + stage * C::SFA_BYTES), 0, 128, 0);
          const uint64_t sdb = ptx::smem_desc(ptx::smem_u32(sSFB + stage * C::SFB_BYTES), 0, 128, 0);
          const uint32_t accum = s > 0 ? 1u : 0u;
          const uint32_t eb = ptx::smem_u32(&empty[stage]);
          if constexpr (C::RG == 1) {
            if (si.g == 0) ptx::stage_f4_cg1(d_t, ad, bd, p.idesc[0], sfa_t, sfb_t, sda, sdb, accum, eb);
            else ptx::stage_f8f6_cg1(d_t, ad, bd, p.idesc[si.g], sfa_t, sfb_t, sda, sdb, accum, eb);
          } else {
            if (si.g == 0) ptx::stage_f4_cg1_rg2(d_t, ad, bd, p.idesc[0], sfa_t, sfb_t, sda, sdb, accum, eb);
            else ptx::stage_f8f6_cg1_rg2(d_t, ad, bd, p.idesc[si.g], sfa_t, sfb_t, sda, sdb, accum, eb);
          }
        } else if (lane == 0) {
          // scale atoms -> TMEM (32 rows x 16 B each, replicated to 4 lane quadrants)
          for (int at = 0; at < si.atoms && !((p.dbg & 1) && s > 0); ++at) {
            ptx::tc_cp_32x128b_x4(sfa_t + 4 * at,
                                  ptx::smem_desc(ptx::smem_u32(sSFA + stage * C::SFA_BYTES + at * 512), 0, 128, 0));
#pragma unroll
            for (int rg = 0; rg < C::RG; ++rg)
              ptx::tc_cp_32x128b_x4(
                  sfb_t + at * 4 * C::RG + 4 * rg,
                  ptx::smem_desc(ptx::smem_u32(sSFB + stage * C::SFB_BYTES + (at * C::RG + rg) * 512), 0, 128, 0));
          }
          for (int k = 0; k < ((p.dbg & 2) ? 0 : si.nmma); ++k) {
            const uint64_t ad = ptx::smem_desc(a_base + 32 * k, 16, 1024, 2);
            const uint64_t bd = ptx::smem_desc(b_base + 32 * k, 16, 1024, 2);
            const uint32_t accum = (s > 0 || k > 0) ? 1u : 0u;
            if (si.g == 0) {
              const uint32_t id = p.idesc[0] | ((uint32_t)(2 * (k & 1)) << 29) | ((uint32_t)(2 * (k & 1)) << 4);
              ptx::tc_mma_mxf4(d_t, ad, bd, id, sfa_t + 4 * (k >> 1), sfb_t + (k >> 1) * 4 * C::RG, accum);
            } else {
              const uint32_t id = p.idesc[si.g] | ((uint32_t)k << 29) | ((uint32_t)k << 4);
              ptx::tc_mma_mxf8f6f4(d_t, ad, bd, id, sfa_t, sfb_t, accum);
            }
          }
          ptx::tc_commit(ptx::smem_u32(&empty[stage]));
        }
        __syncwarp();
        if (s == nstages - 1 && lane == 0) ptx::tc_commit(ptx::smem_u32(&tfull[acc]));
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp >= 4) {
    // ============================ epilogue ============================
    const int q = warp & 3;                       // TMEM lane quadrant
    int it = 0;
    for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x, ++it) {
      const int mb = t % p.num_m, nb = t / p.num_m;
      const int acc = it % C::NUM_ACC;
      const uint32_t acc_phase = (it / C::NUM_ACC) & 1;
      ptx::mbar_wait(ptx::smem_u32(&tfull[acc]), acc_phase, 4, it, t);
      ptx::tc_fence_after();
      const int64_t row = (int64_t)mb * BM + q * 32 + lane;
      const int64_t n0 = (int64_t)nb * BN;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r[32];
        ptx::tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + 32 * c, r);
        ptx::tc_wait_ld();
        if (row < p.M) {
          uint16_t* yrow = p.y + row * p.ldy + n0 + 32 * c;
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            if (n0 + 32 * c + 8 * v < p.N) {
              uint4 o;
              o.x = ptx::pack_bf16x2(__uint_as_float(r[8 * v + 0]), __uint_as_float(r[8 * v + 1]));
              o.y = ptx::pack_bf16x2(__uint_as_float(r[8 * v + 2]), __uint_as_float(r[8 * v + 3]));
              o.z = ptx::pack_bf16x2(__uint_as_float(r[8 * v + 4]), __uint_as_float(r[8 * v + 5]));
              o.w = ptx::pack_bf16x2(__uint_as_float(r[8 * v + 6]), __uint_as_float(r[8 * v + 7]));
              *reinterpret_cast<uint4*>(yrow + 8 * v) = o;
            }
          }
        }
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(ptx::smem_u32(&tempty[acc]));
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 2) ptx::tmem_dealloc(tmem_base, 512);
}

template <int BN, int STAGES>
size_t smem_bytes() {
  using C = Cfg<BN, STAGES>;
  return 1024 + (size_t)STAGES * (C::A_BYTES + C::B_BYTES + C::SFA_BYTES + C::SFB_BYTES) +
         (2 * STAGES + 2 * C::NUM_ACC) * 8 + 16;
}

template <int BN, int STAGES>
cudaError_t run(const GemmArgs& a, const GemmConfig& cfg, cudaStream_t s, int64_t* launches,
                const char** err) {
  CUtensorMap maps[6];
  int first = -1;
  for (int g = 0; g < 3; ++g) {
    if (a.geom.n[g] == 0) continue;
    if (!make_operand_map(&maps[g], a.a_codes[g], g, a.geom.kp[g], a.M, a.geom.pitch[g], BM) ||
        !make_operand_map(&maps[3 + g], a.w_codes[g], g, a.geom.kp[g], a.N, a.geom.pitch[g], BN)) {
      *err = "cuTensorMapEncodeTiled failed";
      return cudaErrorInvalidValue;
    }
    if (first < 0) first = g;
  }
  if (first < 0) { *err = "empty plan"; return cudaErrorInvalidValue; }
  for (int g = 0; g < 3; ++g)
    if (a.geom.n[g] == 0) {  // unused segment: a valid (never used) map
      maps[g] = maps[first];
      maps[3 + g] = maps[3 + first];
    }
  GemmDev p{};
  p.M = a.M;
  p.N = a.N;
  p.num_m = (int)((a.M + BM - 1) / BM);
  p.num_n = (int)((a.N + BN - 1) / BN);
  p.num_tiles = p.num_m * p.num_n;
  for (int g = 0; g < 3; ++g) {
    p.n[g] = a.geom.n[g];
    p.kp[g] = a.geom.kp[g];
    p.nst[g] = g == 0 ? (a.geom.kp[0] + 255) / 256 : a.geom.kp[g] / 128;
    p.sfa[g] = a.a_sf[g];
    p.sfb[g] = a.w_sf[g];
    p.idesc[g] = make_idesc_mn(a.geom.fmt[g], g, BM, BN);
  }
  p.sfb_rows_pad = (a.N + 127) / 128 * 128;
  p.y = a.y;
  p.ldy = a.ldy;
  { const char* d = getenv("MM_GEMM_DEBUG"); p.dbg = d ? atoi(d) : 0; }
  if (p.num_tiles == 0) return cudaSuccess;
  const size_t smem = smem_bytes<BN, STAGES>();
  auto kern = mixgemm_kernel<BN, STAGES>;
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), smem);
  if (e != cudaSuccess) { *err = "cudaFuncSetAttribute(smem) failed"; return e; }
  int grid = sm_count();
  if (cfg.max_ctas > 0 && cfg.max_ctas < grid) grid = cfg.max_ctas;
  if (grid > p.num_tiles) grid = p.num_tiles;
  kern<<<grid, kThreads, smem, s>>>(maps[0], maps[1], maps[2], maps[3], maps[4], maps[5], p);
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace

// 2-D K-major operand map: inner dim = K coordinate (bytes, or FP6 elements),
// outer = rows; box = 128 x box_rows; 128-byte swizzle.
static CUtensorMapL2promotion operand_l2_promotion() {
  static const int v = [] { const char* e = getenv("MM_GEMM_L2PROMO"); return e ? atoi(e) : 3; }();
  return v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                : v == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                         : v == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
}

bool make_operand_map(CUtensorMap* m, const void* base, int g, int kp, int64_t rows, int64_t pitch,
                      int box_rows) {
  EncodeTiledFn enc = tensor_map_encoder();
  if (!enc) return false;
  CUtensorMapDataType dt = CU_TENSOR_MAP_DATA_TYPE_UINT8;
  cuuint64_t inner;
  if (g == 0) inner = kp / 2;
  else if (g == 1) { dt = CU_TENSOR_MAP_DATA_TYPE_16U6_ALIGN16B; inner = kp; }
  else inner = kp;
  cuuint64_t dims[2] = {inner, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)pitch};
  cuuint32_t box[2] = {128, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, dt, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, operand_l2_promotion(),
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

uint32_t make_idesc_mn(int fmt, int g, int m, int n) {
  uint32_t code;
  if (g == 0) code = 1;  // kind::mxf4 E2M1
  else {
    switch (fmt) {
      case F_E4M3: code = 0; break;
      case F_E5M2: code = 1; break;
      case F_E2M3: code = 3; break;
      case F_E3M2: code = 4; break;
      default: code = 5; break;
    }
  }
  return (code << 7) | (code << 10) | ((uint32_t)(n >> 3) << 17) | (1u << 23) | ((uint32_t)(m >> 4) << 24);
}


EncodeTiledFn tensor_map_encoder() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, []() {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  });
  return fn;
}

// Kernel choice of the dispatcher (shared by the launch and the workspace query).
enum GemmPath { PATH_SMALLM, PATH_PAIR, PATH_TILE128, PATH_TILE256 };
static GemmPath choose_path(const GemmArgs& a, const GemmConfig& cfg) {
  int bn = cfg.block_n;
  // auto: CTA-pair 256 x 256 tiles once M fills a pair tile's rows, else single-CTA 128 x 256
  if (bn == 0) bn = a.M > 128 ? 512 : 256;
  if (a.n_dst > 0 || a.y_mc) return PATH_PAIR;   // the fused all-gather epilogues live in the CTA-pair kernel
  // small M (decode-like): swap-AB + split-K kernel (gemm_sm.cu), unless a tile
  // configuration is forced, MM_GEMM_SMALLM=0, or the caller's path must not use a
  // workspace (N-shard entry points).
  // Auto (measured, q_proj N = 4096: M = 1 / 32 / 64 / 128 -> 10 / 13 / 18 / 26 us vs
  // 25-27 us with 128 x 256 tiles): every M <= 128 when few enough 128-row W tiles
  // exist for each to get >= 2 K splits; otherwise the tile kernel.
  // MM_GEMM_SMALLM=1 forces it for any M <= 128, =0 disables it.
  static const int smallm_env = [] { const char* e = getenv("MM_GEMM_SMALLM"); return e ? atoi(e) : -1; }();
  const bool smallm_auto = a.M <= 128 && 2 * ((a.N + 127) / 128) <= sm_count();
  if (!cfg.no_workspace && a.M <= 128 &&
      (cfg.block_n == 1 || (cfg.block_n == 0 && smallm_env != 0 && (smallm_env == 1 || smallm_auto))))
    return PATH_SMALLM;
  if (bn == 1) bn = a.M > 128 ? 512 : 256;   // small-M kernel requested but M > 128
  if (bn == 512) return PATH_PAIR;
  return bn == 128 ? PATH_TILE128 : PATH_TILE256;
}

size_t gemm_workspace_bytes(const GemmArgs& a, const GemmConfig& cfg) {
  if (a.M <= 0 || a.N <= 0) return 0;
  switch (choose_path(a, cfg)) {
    case PATH_SMALLM: return smallm_workspace_bytes(a, cfg);
    case PATH_PAIR: return pair_workspace_bytes(a, cfg);
    default: return 0;
  }
}

cudaError_t launch_mixed_gemm(const GemmArgs& a, const GemmConfig& cfg, cudaStream_t s, int64_t* launches,
                              const char** err) {
  switch (choose_path(a, cfg)) {
    case PATH_SMALLM: return launch_mixed_gemm_smallm(a, cfg, s, launches, err);
    case PATH_PAIR: return launch_mixed_gemm_2cta(a, cfg, s, launches, err);
    case PATH_TILE128:
      if (cfg.num_stages == 4) return run<128, 4>(a, cfg, s, launches, err);
      return run<128, 6>(a, cfg, s, launches, err);
    default:
      if (cfg.num_stages == 3) return run<256, 3>(a, cfg, s, launches, err);
      return run<256, 4>(a, cfg, s, launches, err);
  }
}

}  // namespace mmx
