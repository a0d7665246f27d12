// gemm_sm.cu -- the mixed block-scaled GEMM for SMALL M (decode-like batches,
// M <= 128), sm_100a.  Same mathematics as gemm.cu /
// gemm2.cu (§3.2 "GEMM Kernel" line 143, Eq. 2 lines 47-51: one FP32
// accumulator over the MXFP4, MXFP6 and MXFP8 K-segments, BF16 output), with the
// operand roles SWAPPED and the K loop SPLIT:
//   * swap-AB: the 128-row MMA dimension takes 128 rows of W (output channels) and
//     the MMA N dimension the M activation rows (BNM = 32 / 64 / 128), so a decode
//     batch of 16 rows wastes no 128-row MMA; the accumulator is Y^T [n][m];
//   * split-K: at small M the layer is bound by reading W once from HBM, so the
//     work is cut into (128-row W tile) x (K range) units, one CTA each, sized to
//     fill the 148 SMs; each unit's FP32 partial goes to a workspace and the LAST
//     unit of a W tile (atomic arrival count) sums the partials in split order
//     (deterministic) and writes BF16 Y;
//   * warp roles as in gemm.cu: warp 0 TMA producer, warp 1 MMA issuer, warp 2
//     TMEM allocator, warps 4-7 epilogue (transposed: lane = output channel).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>

#include "internal.h"
#include "ptx.cuh"

namespace mmx {
namespace {

constexpr int kThreadsSm = 256;
constexpr int W_BYTES = 128 * 128;   // 128 W rows x 128 B per stage
constexpr int kMaxSplits = 4;
// Timeline trace (env MM_GEMM_DEBUG & 32; mm_debug_gemm_sm_trace): per CTA
// [start, setup done, first stage full, last stage full, MMAs done (tfull), partial written, end].
__device__ unsigned long long g_sm_trace[1024][10];

struct SmDev {
  int64_t M, N;
  int num_nt;            // 128-row W tiles
  int splits;            // K ranges per W tile
  int nst[3];            // stages per segment
  int n[3], kp[3];
  const uint8_t* sfw[3];
  const uint8_t* sfa[3];
  uint32_t idesc[3];
  uint16_t* y;
  int64_t ldy;
  int interleave;        // 1: units take every splits-th stage, 0: contiguous K ranges (default; measured equal)
  int dbg;
};

template <int BNM, int STAGES>
struct SmCfg {
  static constexpr int A_BYTES = BNM * 128;
  static constexpr int SF_BYTES = 2 * 512;          // up to 2 atoms (FP4 stage), per operand
  static constexpr int STAGE_BYTES = W_BYTES + A_BYTES + 2 * SF_BYTES;
  static constexpr int SF_STRIDE = 16;              // TMEM columns per stage: SFW 2 x 4, SFA 2 x 4
  static constexpr int TMEM_COLS = (BNM + STAGES * SF_STRIDE <= 256) ? 256 : 512;
  static_assert(BNM + STAGES * SF_STRIDE <= 512, "TMEM budget");
};

struct SmStage {
  int g, kcoord, nmma, atoms, atom0;
};

__device__ __forceinline__ SmStage sm_stage(const SmDev& p, int s) {
  SmStage si;
  if (s < p.nst[0]) {
    const int j = s;
    si.g = 0;
    si.kcoord = 128 * j;
    si.nmma = (min(p.n[0] - 256 * j, 256) + 63) / 64;
    si.atoms = min(p.kp[0] - 256 * j, 256) / 128;
    si.atom0 = 2 * j;
  } else {
    const int g = (s < p.nst[0] + p.nst[1]) ? 1 : 2;
    const int j = s - p.nst[0] - (g == 2 ? p.nst[1] : 0);
    si.g = g;
    si.kcoord = 128 * j;
    si.nmma = (min(p.n[g] - 128 * j, 128) + 31) / 32;
    si.atoms = 1;
    si.atom0 = j;
  }
  return si;
}

// TRACE: the timeline-trace instantiation (MM_GEMM_DEBUG & 32); the default one compiles
// the trace stores out.
template <int BNM, int STAGES, bool TRACE>
__global__ void __launch_bounds__(kThreadsSm, 1)
mixgemm_sm_kernel(const __grid_constant__ CUtensorMap tw0, const __grid_constant__ CUtensorMap tw1,
                  const __grid_constant__ CUtensorMap tw2, const __grid_constant__ CUtensorMap ta0,
                  const __grid_constant__ CUtensorMap ta1, const __grid_constant__ CUtensorMap ta2,
                  const __grid_constant__ SmDev p) {
  using C = SmCfg<BNM, STAGES>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sW = smem;
  uint8_t* sA = sW + STAGES * W_BYTES;
  uint8_t* sSF = sA + STAGES * C::A_BYTES;           // [STAGES][SFW | SFA]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sSF + STAGES * 2 * C::SF_BYTES);
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  uint64_t* tfull = bars + 2 * STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const bool trace = TRACE && blockIdx.x < 1024;
  if (trace && threadIdx.x == 0) g_sm_trace[blockIdx.x][0] = ptx::globaltimer_ns();
  const int nt = blockIdx.x / p.splits, ks = blockIdx.x % p.splits;
  const int S = p.nst[0] + p.nst[1] + p.nst[2];
  // Stages of this unit: interleaved (ks, ks + splits, ...) so that the splits of one
  // W tile read neighbouring 128-byte pieces of the same rows at the same time (DRAM
  // page locality), or one contiguous K range (p.interleave = 0).
  const int s_step = p.interleave ? p.splits : 1;
  const int s_lo = p.interleave ? ks : (int)((int64_t)ks * S / p.splits);
  const int s_end = p.interleave ? S : (int)((int64_t)(ks + 1) * S / p.splits);
  const int s_fin = s_end > s_lo ? s_lo + (s_end - 1 - s_lo) / s_step * s_step : s_lo - 1;   // last stage

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&tw0); ptx::tma_prefetch_desc(&tw1); ptx::tma_prefetch_desc(&tw2);
    ptx::tma_prefetch_desc(&ta0); ptx::tma_prefetch_desc(&ta1); ptx::tma_prefetch_desc(&ta2);
  }
  if (warp == 1 && lane == 0) {
    for (int i = 0; i < STAGES; ++i) {
      ptx::mbar_init(ptx::smem_u32(&full[i]), 1);
      ptx::mbar_init(ptx::smem_u32(&empty[i]), 1);
    }
    ptx::mbar_init(ptx::smem_u32(tfull), 1);
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc(ptx::smem_u32(tmem_slot), C::TMEM_COLS);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  ptx::grid_dep_launch();
  ptx::grid_dep_wait();   // A and its scales may come from the preceding kernel
  if (trace && threadIdx.x == 0) g_sm_trace[blockIdx.x][1] = ptx::globaltimer_ns();

  if (warp == 0 || warp == 3) {
    // ============================ TMA producers ============================
    // warp 0: transaction count + W and A tiles; warp 3: the scale atoms (two issuing
    // threads, as in the CTA-pair kernel).
    const bool ops_w = warp == 0;
    if (lane == 0) {
      const CUtensorMap* tw[3] = {&tw0, &tw1, &tw2};
      const CUtensorMap* ta[3] = {&ta0, &ta1, &ta2};
      int stage = 0;
      uint32_t phase = 0;
      for (int s = s_lo; s < s_end; s += s_step) {
        const SmStage si = sm_stage(p, s);
        ptx::mbar_wait(ptx::smem_u32(&empty[stage]), phase ^ 1, 31, s, nt);
        const uint32_t fb = ptx::smem_u32(&full[stage]);
        const int kp128 = p.kp[si.g] / 128;
        const uint32_t ops = si.g == 1 ? (W_BYTES + C::A_BYTES) / 4 * 3 : (W_BYTES + C::A_BYTES);
        if (ops_w) {
          ptx::mbar_arrive_expect_tx(fb, ops + 2u * si.atoms * 512u);
          ptx::tma_load_2d(ptx::smem_u32(sW + stage * W_BYTES), tw[si.g], fb, si.kcoord, nt * 128);
          ptx::tma_load_2d(ptx::smem_u32(sA + stage * C::A_BYTES), ta[si.g], fb, si.kcoord, 0);
        } else {
          uint8_t* sf = sSF + stage * 2 * C::SF_BYTES;
          ptx::bulk_load(ptx::smem_u32(sf), p.sfw[si.g] + ((int64_t)nt * kp128 + si.atom0) * 512, si.atoms * 512, fb);
          ptx::bulk_load(ptx::smem_u32(sf + C::SF_BYTES), p.sfa[si.g] + (int64_t)si.atom0 * 512, si.atoms * 512, fb);
        }
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer ============================
    int stage = 0;
    uint32_t phase = 0;
    for (int s = s_lo; s < s_end; s += s_step) {
      const SmStage si = sm_stage(p, s);
      ptx::mbar_wait(ptx::smem_u32(&full[stage]), phase, 32, s, nt);
      if (trace && lane == 0 && (s == s_lo || s == s_fin)) g_sm_trace[blockIdx.x][s == s_lo ? 2 : 3] = ptx::globaltimer_ns();
      ptx::tc_fence_after();
      const uint32_t sfw_t = tmem_base + BNM + stage * C::SF_STRIDE;
      const uint32_t sfa_t = sfw_t + 8;
      const uint32_t sf = ptx::smem_u32(sSF + stage * 2 * C::SF_BYTES);
      const uint32_t w_base = ptx::smem_u32(sW + stage * W_BYTES);
      const uint32_t a_base = ptx::smem_u32(sA + stage * C::A_BYTES);
      if (si.nmma == 4) {
        // full stage: one issue block (elect.sync, scale copies, 4 MMAs, commit)
        const uint64_t wd = ptx::smem_desc(w_base, 16, 1024, 2), ad = ptx::smem_desc(a_base, 16, 1024, 2);
        const uint64_t sdw = ptx::smem_desc(sf, 0, 128, 0), sda = ptx::smem_desc(sf + C::SF_BYTES, 0, 128, 0);
        const uint32_t accum = s > s_lo ? 1u : 0u;
        if (si.g == 0) ptx::stage_f4_cg1(tmem_base, wd, ad, p.idesc[0], sfw_t, sfa_t, sdw, sda, accum, ptx::smem_u32(&empty[stage]));
        else ptx::stage_f8f6_cg1(tmem_base, wd, ad, p.idesc[si.g], sfw_t, sfa_t, sdw, sda, accum, ptx::smem_u32(&empty[stage]));
      } else if (lane == 0) {
        // a segment's partial last stage: the atoms it uses, then nmma MMAs
        for (int at = 0; at < si.atoms; ++at) {
          ptx::tc_cp_32x128b_x4(sfw_t + 4 * at, ptx::smem_desc(sf + at * 512, 0, 128, 0));
          ptx::tc_cp_32x128b_x4(sfa_t + 4 * at, ptx::smem_desc(sf + C::SF_BYTES + at * 512, 0, 128, 0));
        }
        for (int k = 0; k < si.nmma; ++k) {
          const uint64_t wd = ptx::smem_desc(w_base + 32 * k, 16, 1024, 2);
          const uint64_t ad = ptx::smem_desc(a_base + 32 * k, 16, 1024, 2);
          const uint32_t accum = (s > s_lo || k > 0) ? 1u : 0u;
          if (si.g == 0) {
            const uint32_t id = p.idesc[0] | ((uint32_t)(2 * (k & 1)) << 29) | ((uint32_t)(2 * (k & 1)) << 4);
            ptx::tc_mma_mxf4(tmem_base, wd, ad, id, sfw_t + 4 * (k >> 1), sfa_t + 4 * (k >> 1), accum);
          } else {
            const uint32_t id = p.idesc[si.g] | ((uint32_t)k << 29) | ((uint32_t)k << 4);
            ptx::tc_mma_mxf8f6f4(tmem_base, wd, ad, id, sfw_t, sfa_t, accum);
          }
        }
        ptx::tc_commit(ptx::smem_u32(&empty[stage]));
      }
      __syncwarp();
      if (s == s_fin && lane == 0) ptx::tc_commit(ptx::smem_u32(tfull));
      __syncwarp();
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
    }
  } else if (warp >= 4) {
    // ============================ epilogue (lane = output channel) ============================
    const int q = warp & 3;
    const int nl = q * 32 + lane;                       // row of the W tile
    const int64_t n = (int64_t)nt * 128 + nl;
    const bool empty_range = s_fin < s_lo;             // (splits <= stages / 2, never true)
    if (!empty_range) ptx::mbar_wait(ptx::smem_u32(tfull), 0, 33, nt, ks);
    if (trace && q == 0 && lane == 0) g_sm_trace[blockIdx.x][4] = ptx::globaltimer_ns();
    ptx::tc_fence_after();
    const int M = (int)p.M;
    if (p.splits == 1) {
#pragma unroll 1
      for (int c = 0; c < BNM / 32; ++c) {
        uint32_t r[32];
        ptx::tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + 32 * c, r);
        ptx::tc_wait_ld();
        if (n < p.N) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int m = 32 * c + j;
            if (m < M) {
              const uint32_t b = ptx::pack_bf16x2(__uint_as_float(r[j]), 0.f);
              p.y[(int64_t)m * p.ldy + n] = (uint16_t)(b & 0xFFFFu);
            }
          }
        }
      }
    } else {
      // this unit's FP32 partial -> its own shared memory [m][128] (the operand ring is
      // idle once tfull completed: every MMA has read its stages)
      float* part = reinterpret_cast<float*>(sW);
#pragma unroll 1
      for (int c = 0; c < BNM / 32; ++c) {
        if (32 * c >= M) break;
        uint32_t r[32];
        ptx::tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + 32 * c, r);
        ptx::tc_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (32 * c + j < M) part[(32 * c + j) * 128 + nl] = __uint_as_float(r[j]);
      }
      if (trace && q == 0 && lane == 0) g_sm_trace[blockIdx.x][5] = ptx::globaltimer_ns();
    }
  }

  if (p.splits > 1) {
    // Split-K reduction inside the thread-block cluster of this W tile (cluster rank =
    // split index): after a cluster barrier, the epilogue warps of every split read the
    // partials of their share of the rows from all splits' shared memory (DSMEM), add
    // them in split order (the deterministic order of DESIGN.md R28) and round once to
    // BF16.  A second barrier keeps every CTA's shared memory alive until all reads are
    // done.  No global workspace and no arrival counters.
    ptx::cluster_sync();
    if (trace && threadIdx.x == 128) g_sm_trace[blockIdx.x][7] = ptx::globaltimer_ns();
    if (warp >= 4) {
      // every CTA of the cluster reduces the rows m = ks, ks + splits, ...: 8 rows x
      // up to kMaxSplits remote loads in flight per thread, summed in split order
      const int nl = (warp & 3) * 32 + lane;
      const int64_t n = (int64_t)nt * 128 + nl;
      const int M = (int)p.M;
      if (n < p.N) {
        const uint32_t base = ptx::smem_u32(sW) + 4u * (uint32_t)nl;
#pragma unroll 1
        for (int m0 = ks; m0 < M; m0 += 8 * p.splits) {
          float v[8][kMaxSplits];
#pragma unroll
          for (int mm = 0; mm < 8; ++mm)
#pragma unroll
            for (int k2 = 0; k2 < kMaxSplits; ++k2) {
              const int m = m0 + mm * p.splits;
              v[mm][k2] = 0.f;
              if (m < M && k2 < p.splits) {
                const uint32_t ra = ptx::mapa(base + 512u * (uint32_t)m, (uint32_t)k2);
                asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v[mm][k2]) : "r"(ra) : "memory");
              }
            }
#pragma unroll
          for (int mm = 0; mm < 8; ++mm) {
            const int m = m0 + mm * p.splits;
            float acc = v[mm][0];
#pragma unroll
            for (int k2 = 1; k2 < kMaxSplits; ++k2)
              if (k2 < p.splits) acc += v[mm][k2];
            if (m < M) p.y[(int64_t)m * p.ldy + n] = (uint16_t)(ptx::pack_bf16x2(acc, 0.f) & 0xFFFFu);
          }
        }
      }
    }
    if (trace && threadIdx.x == 128) g_sm_trace[blockIdx.x][8] = ptx::globaltimer_ns();
    ptx::cluster_sync();
  }

  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (trace && threadIdx.x == 0) g_sm_trace[blockIdx.x][6] = ptx::globaltimer_ns();
  if (warp == 2) ptx::tmem_dealloc(tmem_base, C::TMEM_COLS);
}

// Split count of the small-M kernel: fill the SMs once (one CTA per SM), at least 2
// stages per unit, at most kMaxSplits (the splits of a tile form one cluster; split 0
// reads splits x M x 512 B of partials from its peers' shared memory).
int sm_splits(const GemmArgs& a, const GemmConfig& cfg) {
  const int num_nt = (int)((a.N + 127) / 128);
  int S = (a.geom.kp[0] + 255) / 256 + a.geom.kp[1] / 128 + a.geom.kp[2] / 128;
  const int sms = cfg.max_ctas > 0 ? cfg.max_ctas : sm_count();
  int splits = num_nt > 0 ? sms / num_nt : 1;
  static const int env_splits = [] { const char* e = getenv("MM_GEMM_SPLITS"); return e ? atoi(e) : 0; }();
  if (env_splits > 0) splits = env_splits;
  if (splits > S / 2) splits = S / 2;
  if (splits > kMaxSplits) splits = kMaxSplits;
  if (splits < 1) splits = 1;
  return splits;
}
int sm_bnm(int64_t M) { return M <= 32 ? 32 : (M <= 64 ? 64 : 128); }

}  // namespace

// The small-M kernel needs no workspace: its split-K partials are reduced inside a
// thread-block cluster through distributed shared memory.
size_t smallm_workspace_bytes(const GemmArgs&, const GemmConfig&) { return 0; }

namespace {

template <int BNM, int STAGES>
cudaError_t run_sm(const GemmArgs& a, const GemmConfig& cfg, cudaStream_t s, int64_t* launches, const char** err) {
  using C = SmCfg<BNM, STAGES>;
  CUtensorMap maps[6];
  int first = -1;
  for (int g = 0; g < 3; ++g) {
    if (a.geom.n[g] == 0) continue;
    if (!make_operand_map(&maps[g], a.w_codes[g], g, a.geom.kp[g], a.N, a.geom.pitch[g], 128) ||
        !make_operand_map(&maps[3 + g], a.a_codes[g], g, a.geom.kp[g], a.M, a.geom.pitch[g], BNM)) {
      *err = "cuTensorMapEncodeTiled failed";
      return cudaErrorInvalidValue;
    }
    if (first < 0) first = g;
  }
  if (first < 0) { *err = "empty plan"; return cudaErrorInvalidValue; }
  for (int g = 0; g < 3; ++g)
    if (a.geom.n[g] == 0) { maps[g] = maps[first]; maps[3 + g] = maps[3 + first]; }
  SmDev p{};
  p.M = a.M;
  p.N = a.N;
  p.num_nt = (int)((a.N + 127) / 128);
  int S = 0;
  for (int g = 0; g < 3; ++g) {
    p.n[g] = a.geom.n[g];
    p.kp[g] = a.geom.kp[g];
    p.nst[g] = g == 0 ? (a.geom.kp[0] + 255) / 256 : a.geom.kp[g] / 128;
    S += p.nst[g];
    p.sfw[g] = a.w_sf[g];
    p.sfa[g] = a.a_sf[g];
    p.idesc[g] = make_idesc_mn(a.geom.fmt[g], g, 128, BNM);
  }
  p.y = a.y;
  p.ldy = a.ldy;
  { const char* d = getenv("MM_GEMM_DEBUG"); p.dbg = d ? atoi(d) : 0; }
  { const char* e = getenv("MM_GEMM_SPLIT_INTERLEAVE"); p.interleave = e ? atoi(e) : 0; }
  if (p.num_nt == 0 || a.M == 0) return cudaSuccess;
  (void)S;
  const int splits = sm_splits(a, cfg);
  p.splits = splits;

  const size_t smem = 1024 + (size_t)STAGES * C::STAGE_BYTES + (2 * STAGES + 1) * 8 + 16;
  auto kern = (p.dbg & 32) ? mixgemm_sm_kernel<BNM, STAGES, true> : mixgemm_sm_kernel<BNM, STAGES, false>;
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), smem);
  if (e != cudaSuccess) { *err = "cudaFuncSetAttribute(smem) failed"; return e; }
  // the splits of one W tile form a thread-block cluster (cluster rank = split index)
  if (splits > 1)
    e = launch_pdl_cluster(kern, dim3(p.num_nt * splits), dim3(kThreadsSm), smem, s, splits, maps[0], maps[1],
                           maps[2], maps[3], maps[4], maps[5], p);
  else
    e = launch_pdl(kern, dim3(p.num_nt * splits), dim3(kThreadsSm), smem, s, maps[0], maps[1], maps[2], maps[3],
                   maps[4], maps[5], p);
  if (launches) ++*launches;
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace

cudaError_t launch_mixed_gemm_smallm(const GemmArgs& a, const GemmConfig& cfg, cudaStream_t s, int64_t* launches,
                                     const char** err) {
  // (BNM as in sm_bnm)
  if (a.M <= 32) return run_sm<32, 8>(a, cfg, s, launches, err);
  if (a.M <= 64) return run_sm<64, 8>(a, cfg, s, launches, err);
  return run_sm<128, 6>(a, cfg, s, launches, err);
}

}  // namespace mmx

// Debug hook (not part of include/mm.h): copy the small-M GEMM trace to the host.
extern "C" int mm_debug_gemm_sm_trace(unsigned long long* h, int n) {
  return (int)cudaMemcpyFromSymbol(h, mmx::g_sm_trace, sizeof(unsigned long long) * (size_t)(n < 10240 ? n : 10240));
}
