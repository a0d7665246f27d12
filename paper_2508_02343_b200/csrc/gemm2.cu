// gemm2.cu -- the MicroMix mixed block-scaled GEMM on CTA PAIRS (tcgen05
// cta_group::2), sm_100a.  PAPER.md §3.2 "GEMM Kernel" (line 143), Fig. 5 (line
// 137), Eq. 2 (lines 47-51): Y[M, N] (BF16) = sum over the MXFP4 / MXFP6 / MXFP8
// K-segments of A_g W_g^T with E8M0 block scales, one FP32 accumulator.
//
// Same stage structure as gemm.cu (every stage = 128-byte smem rows: an FP4
// stage covers 256 K with 4 x kind::mxf4 K=64, an FP6 or FP8 stage 128 K with
// 4 x kind::mxf8f6f4 K=32; one persistent K loop over the three segments into one
// TMEM accumulator), but the output tile is 256 x 256 per CTA PAIR: each CTA of
// the pair loads its 128 rows of A and its 128 rows of W (half of N) per stage,
// the even CTA issues tcgen05.mma.cta_group::2 (M = 256, N = 256) which reads both
// CTAs' shared memory, and each CTA's TMEM holds its 128 rows x 256 columns.  Per
// CTA and stage that is 32 KB of operand traffic for a 128 x 256 x K_stage slab
// (the single-CTA 128 x 256 tile needs 48 KB): the L2 -> SM traffic, which bounds
// the single-CTA kernel, drops by a third.
//
// Roles (per CTA, 256 threads): warp 0 = TMA producer of the operand tiles (posts the
// stage's transaction count on the even CTA's full barrier), warp 3 = TMA producer of
// the scale atoms (own SFA rows; one W scale row group, multicast to the pair), warp 1 =
// MMA issuer (even CTA only: tcgen05.cp of the scale atoms + the MMAs, commits multicast
// to both CTAs), warp 2 = TMEM allocator, warps 4-7 = epilogue (tcgen05.ld -> BF16 ->
// TMA store); warps 0-3 help drain the last item.
//
// Schedules: whole 256 x 256 tiles round-robin over the pairs in an 8-row-block raster
// (data-parallel); for a ragged last wave with few waves, the balanced schedule
// (build_sched: q whole tiles + at most one narrow item per pair); opt-in stream-K.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>
#include <vector>
#include <tuple>
#include <algorithm>

#include "internal.h"
#include "ptx.cuh"

namespace mmx {
namespace {

constexpr int kThreads2 = 256;
constexpr int kMaxPairs = 80;   // >= SMs / 2 (148 SMs on B200)
// Timeline trace (env MM_GEMM_DEBUG & 32; read with mm_debug_gemm_trace): per CTA
// [start, setup, first stage ready, tile0 start, tile0 issued, tile1 start, tile1
// issued, tile2 start, tile2 issued, epi0 ready, epi1 ready, epi2 ready, epi done].
__device__ unsigned long long g_trace[160][24];
constexpr int A_BYTES = 128 * 128;       // this CTA's 128 rows x 128 B
constexpr int B_BYTES = 128 * 128;       // this CTA's 128 W rows x 128 B
constexpr int SFA_BYTES = 2 * 512;       // up to 2 atoms (FP4 stage)
constexpr int SFB_BYTES = 2 * 2 * 512;   // 2 row groups (N = 256) x up to 2 atoms
constexpr int STAGE_BYTES = A_BYTES + B_BYTES + SFA_BYTES + SFB_BYTES;
constexpr int SF_STRIDE = 24;            // TMEM columns per scale slot: SFA 2x4, SFB 2x2x4
// TMEM (512 columns): two 256-column accumulators that OVERLAP by 48 columns,
// acc0 = [0, 256), acc1 = [208, 464), and two scale slots in [464, 512).  The
// epilogue drains the overlapping columns of an accumulator first and releases them
// early, so the next tile's MMAs (into the other accumulator) start after ~1/4 of
// the epilogue instead of after all of it.
constexpr int ACC1_COL = 208;
// An item of <= 208 columns in the odd accumulator sits at column 256 instead: it does not
// overlap the even accumulator at all, so its MMAs need not wait for the previous item's
// overlap columns to drain (that wait idles the tensor pipe for the previous item's MMA
// completion + first TMEM loads, ~1 us between the whole tile and the narrow item of the balanced schedule).
__host__ __device__ constexpr uint32_t acc_col(int acc, int w) { return acc == 0 ? 0u : (w <= 208 ? 256u : (uint32_t)ACC1_COL); }
constexpr int SF_COL = 464;
// epilogue staging: 4 warps x NB buffers x (32 x 32 BF16); one buffer per warp when
// 6 operand stages take the shared memory
template <int STAGES> __host__ __device__ constexpr int epi_nbuf() { return STAGES >= 6 ? 1 : 2; }
template <int STAGES> __host__ __device__ constexpr int epi_bytes() { return 4 * epi_nbuf<STAGES>() * 32 * 64; }

// Output tensor maps.  NP = 1: Y.  NP = kMaxPeers (NEXT F1, fused all-gather
// epilogue): one map per rank of the peer window, each viewing THIS rank's column
// slice [rank * Ns, (rank + 1) * Ns) of that rank's full Y, so every output tile is
// stored straight into every rank's Y over NVLink and no separate all-gather runs.
template <int NP>
struct YMaps {
  CUtensorMap m[NP];
};

struct Gemm2Dev {
  int64_t M, N;
  int num_m2, num_n, num_tiles;   // pair tiles of 256 x 256
  int nst0, nst1, nst2;           // stages per segment
  int n0, n1, n2;                 // real channels per segment
  int kp0, kp1, kp2;              // stored channels per segment
  uint32_t idesc0, idesc1, idesc2;
  uint16_t* y;
  int64_t ldy;
  int stream_k;                   // 1: stream-K split of the K loop over pairs (see work_item)
  float* ws;                      // stream-K partial tiles: [npairs][256 rows][256 cols] fp32
  int* ws_flag;                   // [npairs][8 epilogue warps]: 1 = that warp's 32 partial rows are
                                  // published; the one reader warp resets it to 0 after consuming
  int ndst;  // output maps used (1, or the peer window's world size)
  int raster;  // pair-row blocks per raster group (8, or 16 for >= 64 column tiles; MM_GEMM_RASTER for tuning)
  int helpers; // 1: warps 0-3 drain half of the LAST tile's accumulator (data-parallel schedule)
  uint16_t* y_mc;        // NVLS: multicast view of all ranks' Y (nullptr: TMA stores)
  int64_t mc_col_off;    // this rank's column offset in the full Y
  int dbg;   // timing experiments only (env MM_GEMM_DEBUG): 2 = no MMA, 4 = no epilogue stores
  int sfb_mc;  // 1: W scale row groups multicast across the pair (one TMA per CTA instead of two)
  int sched2;  // 1: balanced schedule (build_sched): sq whole tiles per pair + at most one narrow item
  int sq;      // whole tiles per pair
  int npairs;  // pairs of the grid
  uint16_t a_pref[65];            // whole tiles enumerated row-block-major: first index of row block b
  uint32_t narrow[kMaxPairs];     // [pair]: bit 31 valid | mb2 | (n0 / 64) << 10 | (w / 64) << 24
};

// Tile raster: groups of up to 8 pair-row blocks (2048 rows of A) sweep all of N
// before moving on, so a wave of tiles reuses the same A rows from L2 (for large M
// the whole A does not fit in L2, W of one layer does).
__device__ __forceinline__ void tile_coords(int t, int num_m2, int num_n, int raster, int& mb2, int& nb) {
  const int G = num_m2 < raster ? num_m2 : raster;
  const int per_group = G * num_n;
  const int grp = t / per_group, r = t - grp * per_group;
  const int rows = min(G, num_m2 - grp * G);
  mb2 = grp * G + r % rows;
  nb = r / rows;
}

// Work items of pair `pair`.  Data-parallel: whole tiles pair, pair + npairs, ...
// Stream-K (opt-in, when the tile count leaves a ragged last wave): the T x S stage
// iterations (S = stages per tile) are cut into npairs contiguous ranges; a range
// covers the tail of one tile (this pair finishes it: adds the partial the
// previous pair left in the workspace), whole tiles, and the head of another
// (this pair leaves a partial for the next pair).  Items run in DESCENDING tile
// order, so every pair writes its partial head first and the finisher of that
// tile -- the next pair, at the end of its own range -- finds it ready.
template <bool LEAN = false>
__device__ __forceinline__ int num_items(const Gemm2Dev& p, int pair, int npairs, int S) {
  if (p.sched2) return p.sq + (int)(p.narrow[pair] >> 31);
  if (LEAN || !p.stream_k) return (p.num_tiles - pair + npairs - 1) / npairs;
  const int64_t W = (int64_t)p.num_tiles * S;
  const int64_t lo = pair * W / npairs, hi = (pair + 1) * W / npairs;
  return hi > lo ? (int)((hi - 1) / S - lo / S + 1) : 0;
}
template <bool LEAN = false>
__device__ __forceinline__ void work_item(const Gemm2Dev& p, int pair, int npairs, int S, int i, int& t, int& s0,
                                          int& s1) {
  if (LEAN || !p.stream_k) { t = pair + i * npairs; s0 = 0; s1 = S; return; }
  const int64_t W = (int64_t)p.num_tiles * S;
  const int64_t lo = pair * W / npairs, hi = (pair + 1) * W / npairs;
  t = (int)((hi - 1) / S) - i;
  const int64_t base = (int64_t)t * S;
  s0 = (int)(lo > base ? lo - base : 0);
  s1 = (int)(hi - base < S ? hi - base : S);
}

// Output block of item i of a pair: rows [256 mb2, +256), columns [n0, n0 + w).  Whole
// tiles (w = 256) in the data-parallel / stream-K schedules; in the balanced schedule
// (p.sched2) a pair's items are sq whole tiles and then at most one narrow item of 64 /
// 128 / 192 columns that may start 64 rows into a W scale atom (its MMAs then read SFB
// two TMEM words in; see build_sched).
__device__ __forceinline__ void item_coords(const Gemm2Dev& p, int pair, int i, int t, int& mb2, int& n0, int& w) {
  if (p.sched2) {
    if (i < p.sq) {   // whole tile pair + i * npairs of the row-block-major enumeration
      const int tw = pair + i * p.npairs;
      int lo = 0, hi = p.num_m2;   // last row block b with a_pref[b] <= tw
      while (hi - lo > 1) { const int mid = (lo + hi) >> 1; if (p.a_pref[mid] <= tw) lo = mid; else hi = mid; }
      mb2 = lo;
      n0 = (tw - p.a_pref[lo]) * 256;
      w = 256;
      return;
    }
    const uint32_t e = p.narrow[pair];
    mb2 = (int)(e & 1023u);
    n0 = (int)((e >> 10) & 4095u) * 64;
    w = (int)((e >> 24) & 7u) * 64;
    return;
  }
  int nb;
  tile_coords(t, p.num_m2, p.num_n, p.raster, mb2, nb);
  n0 = nb * 256;
  w = 256;
}

template <int G>
__device__ __forceinline__ void seg_stage(const Gemm2Dev& p, int j, int& kcoord, int& nmma, int& atoms, int& atom0) {
  const int n = G == 0 ? p.n0 : (G == 1 ? p.n1 : p.n2);
  const int kp = G == 0 ? p.kp0 : (G == 1 ? p.kp1 : p.kp2);
  if constexpr (G == 0) {
    kcoord = 128 * j;                               // bytes (2 E2M1 per byte)
    nmma = (min(n - 256 * j, 256) + 63) / 64;
    atoms = min(kp - 256 * j, 256) / 128;
    atom0 = 2 * j;
  } else {
    kcoord = 128 * j;                               // FP6: elements, FP8: bytes
    nmma = (min(n - 128 * j, 128) + 31) / 32;
    atoms = 1;
    atom0 = j;
  }
}

// Drain of accumulator columns [32 c_lo, 32 c_hi) of this CTA's 128 x 256 tile slab by
// one warp (TMEM lane quadrant q): tcgen05.ld -> BF16 RNE -> 64B-swizzled staging
// (one private 2 KB buffer per chunk) -> TMA store of each 32 x 32 box.
template <int NP>
__device__ __forceinline__ void drain_chunks(const YMaps<NP>& tys, int ndst, uint32_t trow, uint8_t* stg, int c_lo,
                                             int c_hi, int n0, int row0, int lane) {
  for (int c = c_lo; c < c_hi; ++c) {
    uint32_t r[32];
    ptx::tmem_ld_32x32b_x32(trow + 32 * c, r);
    ptx::tc_wait_ld();
    uint32_t w[16];
#pragma unroll
    for (int v = 0; v < 16; ++v) w[v] = ptx::pack_bf16x2(__uint_as_float(r[2 * v]), __uint_as_float(r[2 * v + 1]));
    uint8_t* buf = stg + (c - c_lo) * 2048;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      *reinterpret_cast<uint4*>(buf + lane * 64 + ((k ^ ((lane >> 1) & 3)) << 4)) =
          make_uint4(w[4 * k], w[4 * k + 1], w[4 * k + 2], w[4 * k + 3]);
    ptx::fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      for (int dst = 0; dst < (NP == 1 ? 1 : ndst); ++dst) ptx::tma_store_2d(&tys.m[dst], ptx::smem_u32(buf), n0 + 32 * c, row0);
      ptx::bulk_commit_group();
    }
  }
}

// LEAN: the default path's instantiation -- stream-K, the NVLS multicast epilogue, the
// timeline trace and the timing-experiment switches compiled out (a smaller kernel).
template <int STAGES, int NP, bool LEAN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads2, 1)
mixgemm2_kernel(const __grid_constant__ CUtensorMap ta0, const __grid_constant__ CUtensorMap ta1,
                const __grid_constant__ CUtensorMap ta2, const __grid_constant__ CUtensorMap tb0,
                const __grid_constant__ CUtensorMap tb1, const __grid_constant__ CUtensorMap tb2,
                const __grid_constant__ CUtensorMap tsa0, const __grid_constant__ CUtensorMap tsa1,
                const __grid_constant__ CUtensorMap tsa2, const __grid_constant__ CUtensorMap tsb0,
                const __grid_constant__ CUtensorMap tsb1, const __grid_constant__ CUtensorMap tsb2,
                const __grid_constant__ YMaps<NP> tys, const __grid_constant__ Gemm2Dev p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = sA + STAGES * A_BYTES;
  uint8_t* sSFA = sB + STAGES * B_BYTES;
  uint8_t* sSFB = sSFA + STAGES * SFA_BYTES;
  uint8_t* sEpi = sSFB + STAGES * SFB_BYTES;      // [4 warps][2][32 rows x 64 B] BF16 staging
  uint64_t* bars = reinterpret_cast<uint64_t*>(sEpi + epi_bytes<STAGES>());
  uint64_t* full = bars;                  // [STAGES]  (used in the even CTA)
  uint64_t* empty = bars + STAGES;        // [STAGES]  (each CTA)
  uint64_t* tfull = bars + 2 * STAGES;    // [2] per accumulator (each CTA)
  uint64_t* tempty = tfull + 2;           // [2] accumulator fully drained (even CTA)
  uint64_t* tovl = tempty + 2;            // [2] overlap columns drained (even CTA)
  uint64_t* pbar = tovl + 2;              // [4] stream-K: a warp's partial rows landed in smem
  uint64_t* hgo = pbar + 4;               // [1] helpers: the 4 epilogue warps reached the last tile
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(hgo + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = ptx::cluster_ctarank();    // 0 = MMA leader
  const uint64_t t_start = ptx::globaltimer_ns();
  const int dbg = LEAN ? 0 : p.dbg;
  const bool streamk = !LEAN && p.stream_k;
  uint16_t* const y_mc = LEAN ? nullptr : p.y_mc;
  const bool trace = (dbg & 32) && lane == 0;
  const int pair = blockIdx.x / 2, npairs = gridDim.x / 2;

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&ta0); ptx::tma_prefetch_desc(&ta1); ptx::tma_prefetch_desc(&ta2);
    ptx::tma_prefetch_desc(&tb0); ptx::tma_prefetch_desc(&tb1); ptx::tma_prefetch_desc(&tb2);
    ptx::tma_prefetch_desc(&tsa0); ptx::tma_prefetch_desc(&tsa1); ptx::tma_prefetch_desc(&tsa2);
    ptx::tma_prefetch_desc(&tsb0); ptx::tma_prefetch_desc(&tsb1); ptx::tma_prefetch_desc(&tsb2);
  }
  if (warp == 1 && lane == 0) {
    for (int i = 0; i < STAGES; ++i) {
      ptx::mbar_init(ptx::smem_u32(&full[i]), 1);
      ptx::mbar_init(ptx::smem_u32(&empty[i]), 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(ptx::smem_u32(&tfull[i]), 1);
      ptx::mbar_init(ptx::smem_u32(&tempty[i]), 8);   // 4 epilogue warps x 2 CTAs
      ptx::mbar_init(ptx::smem_u32(&tovl[i]), 8);
    }
    for (int i = 0; i < 4; ++i) {
      ptx::mbar_init(ptx::smem_u32(&pbar[i]), 1);
    }
    ptx::mbar_init(ptx::smem_u32(hgo), 4);
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc_cg2(ptx::smem_u32(tmem_slot), 512);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  ptx::grid_dep_launch();
  ptx::grid_dep_wait();   // A, W, scales may come from the preceding kernel; Y may still be read by it
  if (trace && warp == 1) { g_trace[blockIdx.x][0] = t_start; g_trace[blockIdx.x][1] = ptx::globaltimer_ns(); }
  const int64_t M = p.M, N = p.N;
  const int S = p.nst0 + p.nst1 + p.nst2;
  const int n_items = num_items<LEAN>(p, pair, npairs, S);

  if (warp == 0 || warp == 3) {
    // ============================ TMA producers (both CTAs) ============================
    // Two issuing threads follow the same stage sequence and wait on the same empty
    // barriers: warp 0 posts the stage's transaction count and loads the A and W
    // tiles, warp 3 loads the scale atoms.  One thread issuing all five TMAs of a
    // stage limited the stage rate (measured: -7 % per tile at b8, -11 % at q_proj).
    const bool ops = warp == 0;
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t full0 = ptx::smem_u32(&full[0]);
      for (int it = 0; it < n_items; ++it) {
        int t, s0, s1;
        work_item<LEAN>(p, pair, npairs, S, it, t, s0, s1);
        int mb2, nt0, w;
        item_coords(p, pair, it, t, mb2, nt0, w);
        const int m0 = mb2 * 256 + 128 * (int)rank;      // this CTA's A rows
        const int n0 = nt0 + (w / 2) * (int)rank;        // this CTA's W rows (its half of the item's N)
        const int mgrp = mb2 * 2 + (int)rank;           // 128-row scale group of A
        const int rgb = nt0 >> 7;                       // first 128-row scale group of W
#pragma unroll
        for (int g = 0; g < 3; ++g) {
          const int nst = g == 0 ? p.nst0 : (g == 1 ? p.nst1 : p.nst2);
          const int kp128 = (g == 0 ? p.kp0 : (g == 1 ? p.kp1 : p.kp2)) / 128;
          const CUtensorMap* ta = g == 0 ? &ta0 : (g == 1 ? &ta1 : &ta2);
          const CUtensorMap* tb = g == 0 ? &tb0 : (g == 1 ? &tb1 : &tb2);
          const CUtensorMap* tsa = g == 0 ? &tsa0 : (g == 1 ? &tsa1 : &tsa2);
          const CUtensorMap* tsb = g == 0 ? &tsb0 : (g == 1 ? &tsb1 : &tsb2);
          const int box_atoms = g == 0 ? 2 : 1;
          // TMA counts GLOBAL element bits: a 16U6 (FP6) box of 128 elements lands
          // as 128 B per smem row but completes 96 B per row.
          const uint32_t ab = g == 1 ? (A_BYTES + B_BYTES) / 4 * 3 : (A_BYTES + B_BYTES);
          const uint32_t cta_bytes = ab + 3u * box_atoms * 512u;
          const int sbase = g == 0 ? 0 : (g == 1 ? p.nst0 : p.nst0 + p.nst1);
          const int j_lo = max(s0 - sbase, 0), j_hi = min(s1 - sbase, nst);
          for (int j = j_lo; j < j_hi; ++j) {
            int kcoord, nmma, atoms, atom0;
            if (g == 0) seg_stage<0>(p, j, kcoord, nmma, atoms, atom0);
            else if (g == 1) seg_stage<1>(p, j, kcoord, nmma, atoms, atom0);
            else seg_stage<2>(p, j, kcoord, nmma, atoms, atom0);
            ptx::mbar_wait(ptx::smem_u32(&empty[stage]), phase ^ 1, 21, stage, t);
            const uint32_t fb = full0 + 8 * stage;     // the even CTA's barrier (peer bit cleared)
            const bool no_sf = (dbg & 8) != 0;   // timing experiment only
            if (dbg & 16) {                      // timing experiment: no loads at all
              if (rank == 0 && ops) ptx::mbar_arrive(fb);
              if (++stage == STAGES) { stage = 0; phase ^= 1; }
              continue;
            }
            if (ops) {
              if (rank == 0) ptx::mbar_arrive_expect_tx(fb, 2 * (no_sf ? ab : cta_bytes));
              ptx::tma_load_2d_cg2(ptx::smem_u32(sA + stage * A_BYTES), ta, fb, kcoord, m0);
              ptx::tma_load_2d_cg2(ptx::smem_u32(sB + stage * B_BYTES), tb, fb, kcoord, n0);
            } else if (!no_sf) {
              ptx::tma_load_2d_cg2(ptx::smem_u32(sSFA + stage * SFA_BYTES), tsa, fb, 0, mgrp * kp128 + atom0);
              if (p.sfb_mc) {
                // both CTAs need all 256 W rows' scales: each loads its own row group ONCE and
                // multicasts it to the pair (both deliveries complete on the leader's barrier)
                ptx::tma_load_2d_cg2_mc(ptx::smem_u32(sSFB + stage * SFB_BYTES + (int)rank * 1024), tsb, fb, 0,
                                        (rgb + (int)rank) * kp128 + atom0, (uint16_t)0x3);
              } else {
                for (int rg = 0; rg < 2; ++rg)
                  ptx::tma_load_2d_cg2(ptx::smem_u32(sSFB + stage * SFB_BYTES + rg * 1024), tsb, fb, 0,
                                       (rgb + rg) * kp128 + atom0);
              }
            }
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer (even CTA) ============================
    // The whole warp runs this loop converged; elect.sync inside the issue blocks
    // picks the one lane that issues (operands stay warp-uniform).  Full stages go
    // through one asm block each (scale copies + 4 MMAs + commit); only a segment's
    // last stage may issue fewer MMAs and takes the per-MMA path.
    if (rank == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      const uint32_t sA0 = ptx::smem_u32(sA), sB0 = ptx::smem_u32(sB);
      const uint32_t sSFA0 = ptx::smem_u32(sSFA), sSFB0 = ptx::smem_u32(sSFB);
      const uint32_t empty0 = ptx::smem_u32(&empty[0]), full0 = ptx::smem_u32(&full[0]);
      const bool no_mma = (dbg & 2) != 0;
      for (; it < n_items; ++it) {
        int t, s0, s1;
        work_item<LEAN>(p, pair, npairs, S, it, t, s0, s1);
        const int acc = it & 1;
        int mb2_, nt0, w;
        item_coords(p, pair, it, t, mb2_, nt0, w);
        const uint32_t d_t = tmem_base + acc_col(acc, w);
        bool ovl = false;   // does this item's accumulator overlap the previous item's?
        if (it > 0) {
          int tp, s0p, s1p, mbp, np0, wp;
          work_item<LEAN>(p, pair, npairs, S, it - 1, tp, s0p, s1p);
          item_coords(p, pair, it - 1, tp, mbp, np0, wp);
          const int c0 = (int)acc_col(acc ^ 1, wp), c1 = (int)acc_col(acc, w);
          ovl = max(c0, c1) < min(c0 + wp, c1 + w);
        }
        // the item's N in the instruction descriptor (bits 17-22: N >> 3); an item that
        // starts 64 rows into a W scale atom reads SFB two TMEM words in
        const uint32_t nfield = ~(0x3Fu << 17), nbits = (uint32_t)(w >> 3) << 17;
        const uint32_t sfb_off = (nt0 & 127) ? 2u : 0u;
        ptx::mbar_wait(ptx::smem_u32(&tempty[acc]), ((it >> 1) & 1) ^ 1, 22, it, t);   // tile it-2 drained acc
        if (trace && it == 1) g_trace[blockIdx.x][16] = ptx::globaltimer_ns();
        if (ovl) ptx::mbar_wait(ptx::smem_u32(&tovl[acc ^ 1]), ((it - 1) >> 1) & 1, 25, it, t);  // overlap of it-1
        if (trace && it < 3) g_trace[blockIdx.x][3 + 2 * it] = ptx::globaltimer_ns();
        if (trace && it == 0) g_trace[blockIdx.x][13] = clock64();
        if (trace && it == 1) g_trace[blockIdx.x][22] = clock64();
        ptx::tc_fence_after();
        uint32_t accum = 0;
#pragma unroll
        for (int g = 0; g < 3; ++g) {
          const int nst = g == 0 ? p.nst0 : (g == 1 ? p.nst1 : p.nst2);
          const int n_g = g == 0 ? p.n0 : (g == 1 ? p.n1 : p.n2);
          const uint32_t idesc = ((g == 0 ? p.idesc0 : (g == 1 ? p.idesc1 : p.idesc2)) & nfield) | nbits;
          const int kstage = g == 0 ? 256 : 128;                    // K per stage
          const int kmma = g == 0 ? 64 : 32;                        // K per MMA
          const int sbase = g == 0 ? 0 : (g == 1 ? p.nst0 : p.nst0 + p.nst1);
          const int j_lo = max(s0 - sbase, 0), j_hi = min(s1 - sbase, nst);
          for (int j = j_lo; j < j_hi; ++j) {
            const int nmma = min((n_g - kstage * j + kmma - 1) / kmma, 4);
            ptx::mbar_wait(full0 + 8 * stage, phase, 23, stage, t);
            if (trace && it == 0 && j == j_lo && g == 0) g_trace[blockIdx.x][2] = ptx::globaltimer_ns();
            ptx::tc_fence_after();
            const uint32_t sfa_t = tmem_base + SF_COL + (stage & 1) * SF_STRIDE;
            const uint32_t sfb_t = sfa_t + 8;
            const uint64_t ad = ptx::smem_desc(sA0 + stage * A_BYTES, 16, 1024, 2);
            const uint64_t bd = ptx::smem_desc(sB0 + stage * B_BYTES, 16, 1024, 2);
            const uint64_t sda = ptx::smem_desc(sSFA0 + stage * SFA_BYTES, 0, 128, 0);
            const uint64_t sdb0 = ptx::smem_desc(sSFB0 + stage * SFB_BYTES, 0, 128, 0);
            const uint64_t sdb1 = ptx::smem_desc(sSFB0 + stage * SFB_BYTES + 1024, 0, 128, 0);
            if (nmma == 4 && !no_mma) {
              if (g == 0) ptx::stage_f4_cg2(d_t, ad, bd, idesc, sfa_t, sfb_t, sda, sdb0, sdb1, accum, empty0 + 8 * stage,
                                            sfb_t + sfb_off);
              else ptx::stage_f8f6_cg2(d_t, ad, bd, idesc, sfa_t, sfb_t, sda, sdb0, sdb1, accum, empty0 + 8 * stage,
                                       (dbg & 64) ? 0u : 1u, sfb_t + sfb_off);
              accum = 1;
            } else {
              // partial stage: scale copies for the atoms it uses, then nmma MMAs
              if (lane == 0) {
                const int atoms = g == 0 ? (nmma + 1) / 2 : 1;
                for (int at = 0; at < atoms; ++at) {
                  ptx::tc_cp_32x128b_x4_cg2(sfa_t + 4 * at, sda + 32 * at);
                  ptx::tc_cp_32x128b_x4_cg2(sfb_t + 8 * at, sdb0 + 32 * at);
                  ptx::tc_cp_32x128b_x4_cg2(sfb_t + 8 * at + 4, sdb1 + 32 * at);
                }
                for (int k = 0; k < (no_mma ? 0 : nmma); ++k) {
                  if (g == 0) {
                    const uint32_t sid = 2u * (k & 1);
                    ptx::tc_mma_mxf4_cg2(d_t, ad + 2 * k, bd + 2 * k, idesc | (sid << 29) | (sid << 4),
                                         sfa_t + 4 * (k >> 1), sfb_t + sfb_off + (k >> 1) * 8, accum);
                  } else {
                    ptx::tc_mma_mxf8f6f4_cg2(d_t, ad + 2 * k, bd + 2 * k, idesc | ((uint32_t)k << 29) | ((uint32_t)k << 4),
                                             sfa_t, sfb_t + sfb_off, accum);
                  }
                  accum = 1;
                }
                ptx::tc_commit_cg2_mc(empty0 + 8 * stage, 0x3);
              }
              accum = __shfl_sync(0xffffffffu, accum, 0);
              __syncwarp();
            }
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
        }
        ptx::commit_cg2_mc_elect(ptx::smem_u32(&tfull[acc]));
        if (trace && it < 3) g_trace[blockIdx.x][4 + 2 * it] = ptx::globaltimer_ns();
        if (trace && it == 0) g_trace[blockIdx.x][14] = clock64();
        __syncwarp();
      }
    }
  } else if (warp >= 4) {
    // ============================ epilogue (both CTAs) ============================
    // Per 32-column chunk: tcgen05.ld (32 lanes x 32 columns) -> BF16 RNE -> this
    // warp's smem staging buffer -> one TMA store of the 32 x 32 box (the TMA clips
    // rows >= M and columns >= N).  Two staging buffers per warp let the next
    // chunk's conversion overlap the previous store; the accumulator is released to
    // the MMA warp as soon as its last chunk is in registers.
    const int q = warp & 3;                           // TMEM lane quadrant
    const uint32_t tempty_leader = ptx::mapa(ptx::smem_u32(&tempty[0]), 0);
    const uint32_t tovl_leader = ptx::mapa(ptx::smem_u32(&tovl[0]), 0);
    constexpr int NB = epi_nbuf<STAGES>();
    uint8_t* stg = sEpi + q * NB * 2048;
    int nstore = 0;
    for (int it = 0; it < n_items; ++it) {
      int t, s0, s1;
      work_item<LEAN>(p, pair, npairs, S, it, t, s0, s1);
      int mb2, n0, w;
      item_coords(p, pair, it, t, mb2, n0, w);
      const int nch = w / 32;   // 32-column chunks of this item (8 for a whole tile)
      // stream-K roles of this item: leave a partial (head of a tile) / add one (tail)
      const bool to_ws = s1 < S, from_ws = s0 > 0;
      const int wrow = 128 * (int)rank + q * 32 + lane;   // row inside the 256-row pair tile
      // Stream-K hand-off, one flag per writer warp: warp (rank, q) of pair `pair - 1`
      // wrote exactly the 32 partial rows warp (rank, q) of this pair reads, so each
      // reader waits on its own writer only and resets that flag after consuming it
      // (one writer, one reader per flag per launch; the next launch is stream-ordered).
      int* const my_flag = p.ws_flag + (pair - 1) * 8 + (int)rank * 4 + q;
      if (from_ws) {
        if (lane == 0) {
          const uint64_t t0 = ptx::globaltimer_ns();
          for (uint32_t n = 1;; ++n) {
            int v;
            asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(my_flag) : "memory");
            if (v != 0) break;
            __nanosleep(64);
            if ((n & 1023u) == 0 && ptx::globaltimer_ns() - t0 > (uint64_t)MM_WATCHDOG_NS)
              ptx::watchdog_fire(29, 0u, 0u, it, t);
          }
          // the partial was written through the generic proxy; the bulk copy below
          // reads it through the async proxy
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        __syncwarp();
      }
      const int acc = it & 1;
      ptx::mbar_wait(ptx::smem_u32(&tfull[acc]), (it >> 1) & 1, 24, it, t);
      // Stream-K tail: this is the pair's last item, so once its MMAs are done the
      // operand ring is idle.  The warp's 32 partial rows (contiguous 32 KB in the
      // workspace) are staged there with ONE bulk copy, instead of eight dependent
      // rounds of global loads (one per 32-column chunk) in the drain loop.
      const uint8_t* pst = nullptr;
      if (from_ws) {
        uint8_t* dstp = sA + q * 32768;   // sA and sB are contiguous: >= 128 KB for >= 4 stages
        const uint32_t pb = ptx::smem_u32(&pbar[q]);
        if (lane == 0) {
          ptx::mbar_arrive_expect_tx(pb, 32768);
          ptx::bulk_load(ptx::smem_u32(dstp), p.ws + ((size_t)(pair - 1) * 256 + 128 * (int)rank + q * 32) * 256, 32768, pb);
        }
        ptx::mbar_wait(pb, 0, 28, it, t);
        pst = dstp;
        if (lane == 0) *reinterpret_cast<volatile int*>(my_flag) = 0;   // consumed: re-arm for the next launch
      }
      if (trace && q == 0 && it < 3) g_trace[blockIdx.x][9 + it] = ptx::globaltimer_ns();
      if (trace && q == 0 && it == 0 && rank == 0) g_trace[blockIdx.x][21] = clock64();
      ptx::tc_fence_after();
      const int row0 = mb2 * 256 + 128 * (int)rank + q * 32;
      const uint32_t acc_c = acc_col(acc, w);
      uint32_t rn[32];   // chunk 1 of the drain order, loaded together with chunk 0
      const uint32_t trow = tmem_base + ((uint32_t)(q * 32) << 16) + acc_c;
      if (p.helpers && it == n_items - 1 && !(dbg & 4)) {
        // last tile: warps 0-3 drain chunks 4-7 (drain_chunks below); these warps drain
        // 0-3 into private staging buffers in the (now idle) operand ring.  The helpers
        // are released through their own barrier, not tfull: a phase-parity wait on tfull
        // from a warp that did not follow every earlier phase could alias an older one.
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(ptx::smem_u32(hgo));
        if (lane == 0) ptx::bulk_wait_group_read<0>();   // this warp's earlier stores have read `stg`
        __syncwarp();
        drain_chunks<NP>(tys, p.ndst, trow, sA + (4 + q) * 8192, 0, min(4, nch), n0, row0, lane);
        continue;
      }
      // acc0 of a whole tile: its overlap with acc1 (columns 208..255) lives in chunks 6,
      // 7 -> drain those first (a narrower item does not reach the overlap); acc1: its
      // overlap is its own columns 0..47 -> chunks 0, 1 come first anyway.  The first two
      // chunks are loaded back to back and the overlap released before any conversion,
      // so the next tile's MMAs wait for two TMEM loads only.
      const int rot = (acc == 0 && nch == 8) ? 6 : 0;
#pragma unroll 1
      for (int i = 0; i < nch; ++i) {
        const int c = (i + rot) & 7;
        uint32_t r[32];
        if (i == 0) {
          if (trace && q == 0 && it == 0 && rank == 0) g_trace[blockIdx.x][19] = clock64();
          ptx::tmem_ld_32x32b_x32(trow + 32 * c, r);
          ptx::tmem_ld_32x32b_x32(trow + 32 * ((1 + rot) & 7), rn);
          ptx::tc_wait_ld();
          if (trace && q == 0 && it == 0 && rank == 0) g_trace[blockIdx.x][20] = clock64();
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive_cluster(tovl_leader + 8 * acc);   // overlap drained
          if (nch == 2 && lane == 0) ptx::mbar_arrive_cluster(tempty_leader + 8 * acc);   // all drained
          if (trace && q == 0 && it == 0) g_trace[blockIdx.x][17 + (int)rank] = ptx::globaltimer_ns();
        } else if (i == 1) {
#pragma unroll
          for (int v = 0; v < 32; ++v) r[v] = rn[v];
        } else {
          ptx::tmem_ld_32x32b_x32(trow + 32 * c, r);
          ptx::tc_wait_ld();
          if (i == nch - 1) {   // whole accumulator drained
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive_cluster(tempty_leader + 8 * acc);
          }
        }
        if (dbg & 4) continue;
        if (to_ws) {   // fp32 partial -> workspace row (128 B per chunk per thread)
          float4* dst = reinterpret_cast<float4*>(p.ws + ((size_t)pair * 256 + wrow) * 256 + 32 * c);
#pragma unroll
          for (int v = 0; v < 8; ++v)
            dst[v] = make_float4(__uint_as_float(r[4 * v]), __uint_as_float(r[4 * v + 1]),
                                 __uint_as_float(r[4 * v + 2]), __uint_as_float(r[4 * v + 3]));
          continue;
        }
        if (from_ws) {   // add the previous pair's partial (fixed order: partial + own)
          const float4* src = reinterpret_cast<const float4*>(pst + lane * 1024 + 128 * c);
#pragma unroll
          for (int v = 0; v < 8; ++v) {
            const float4 o = src[v];
            r[4 * v] = __float_as_uint(o.x + __uint_as_float(r[4 * v]));
            r[4 * v + 1] = __float_as_uint(o.y + __uint_as_float(r[4 * v + 1]));
            r[4 * v + 2] = __float_as_uint(o.z + __uint_as_float(r[4 * v + 2]));
            r[4 * v + 3] = __float_as_uint(o.w + __uint_as_float(r[4 * v + 3]));
          }
        }
        uint32_t w[16];
#pragma unroll
        for (int v = 0; v < 16; ++v) w[v] = ptx::pack_bf16x2(__uint_as_float(r[2 * v]), __uint_as_float(r[2 * v + 1]));
        if (y_mc) {
          // NVLS: row row0 + lane, 32 columns as four 16-byte multimem stores (one write
          // per element reaches every rank's Y); rows >= M and columns >= N (the shard)
          // are clipped like the TMA boxes clip them.
          const int64_t rr = row0 + lane;
          const int col = n0 + 32 * c;
          if (rr < M) {
            uint16_t* dst = y_mc + rr * p.ldy + p.mc_col_off + col;
#pragma unroll
            for (int k = 0; k < 4; ++k)
              if (col + 8 * k < N)
                asm volatile("multimem.st.relaxed.sys.global.v4.bf16x2 [%0], {%1, %2, %3, %4};" ::"l"(dst + 8 * k),
                             "r"(w[4 * k]), "r"(w[4 * k + 1]), "r"(w[4 * k + 2]), "r"(w[4 * k + 3])
                             : "memory");
          }
          continue;
        }
        uint8_t* buf = stg + (nstore % NB) * 2048;
        if (lane == 0) ptx::bulk_wait_group_read<NB - 1>();   // the store that last used `buf` has read it
        __syncwarp();
        // row `lane` = 64 B in the TMA 64-byte swizzle layout (16-byte chunk k of row
        // r at chunk k ^ ((r >> 1) & 3)): conflict-free, and w[] is indexed statically
#pragma unroll
        for (int k = 0; k < 4; ++k)
          *reinterpret_cast<uint4*>(buf + lane * 64 + ((k ^ ((lane >> 1) & 3)) << 4)) =
              make_uint4(w[4 * k], w[4 * k + 1], w[4 * k + 2], w[4 * k + 3]);
        ptx::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          if constexpr (NP == 1) {
            ptx::tma_store_2d(&tys.m[0], ptx::smem_u32(buf), n0 + 32 * c, row0);
          } else {
            for (int dst = 0; dst < p.ndst; ++dst) ptx::tma_store_2d(&tys.m[dst], ptx::smem_u32(buf), n0 + 32 * c, row0);
          }
          ptx::bulk_commit_group();
        }
        ++nstore;
      }
      if (to_ws) {   // publish: this warp's rows of the partial are in global memory
        __syncwarp();   // orders the other lanes' stores before lane 0's release
        if (lane == 0) {
          __threadfence();
          asm volatile("st.release.gpu.global.s32 [%0], 1;" ::"l"(p.ws_flag + pair * 8 + (int)rank * 4 + q) : "memory");
        }
      }
    }
    if (lane == 0) {
      if constexpr (NP == 1) ptx::bulk_wait_group_read<0>();
      else ptx::bulk_wait_group<0>();   // peer stores fully performed before the CTA retires
    }
    if (trace && q == 0) g_trace[blockIdx.x][12] = ptx::globaltimer_ns();
  }

  if (warp < 4 && p.helpers && n_items > 0 && !(dbg & 4)) {
    // ==================== helpers: drain of the last tile ====================
    // The producer, MMA and allocator warps are idle once the last tile is issued; they
    // drain columns 128..255 of its accumulator (their TMEM lane quadrant = warp % 4)
    // while the epilogue warps drain columns 0..127, halving the exposed final drain.
    __syncwarp();
    const int it = n_items - 1;
    int t, s0, s1;
    work_item<LEAN>(p, pair, npairs, S, it, t, s0, s1);
    int mb2, n0, w;
    item_coords(p, pair, it, t, mb2, n0, w);
    const int acc = it & 1;
    // single phase: the epilogue warps saw tfull.  A suspended wait: warps 1 (odd CTA)
    // and 2 have no role and would otherwise spin for the whole kernel, stealing issue
    // slots from the epilogue.
    ptx::mbar_wait_sleep(ptx::smem_u32(hgo), 0, 26, it, t);
    ptx::tc_fence_after();
    const int q = warp & 3;
    const uint32_t trow = tmem_base + ((uint32_t)(q * 32) << 16) + acc_col(acc, w);
    drain_chunks<NP>(tys, p.ndst, trow, sA + q * 8192, 4, w / 32, n0, mb2 * 256 + 128 * (int)rank + q * 32, lane);
    if (lane == 0) {
      if constexpr (NP == 1) ptx::bulk_wait_group_read<0>();
      else ptx::bulk_wait_group<0>();
    }
  }

  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  if (warp == 2) ptx::tmem_dealloc_cg2(tmem_base, 512);
}

// Scale-factor map: the atoms of one operand segment viewed as a 2-D array of
// [n_atoms][128 x u32] (512-byte atoms, see include/mm.h), box = box_atoms atoms.
bool make_sf_map(CUtensorMap* m, const void* base, int64_t rows, int kp, int box_atoms) {
  EncodeTiledFn enc = tensor_map_encoder();
  if (!enc) return false;
  const int64_t n_atoms = (rows + 127) / 128 * (kp / 128);
  cuuint64_t dims[2] = {128, (cuuint64_t)n_atoms};
  cuuint64_t strides[1] = {512};
  cuuint32_t box[2] = {128, (cuuint32_t)box_atoms};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Stream-K schedule: opt-in (MM_GEMM_STREAMK=1) when the last wave of tiles would be
// ragged and there are only a few waves (each pair then finishes at most one tile
// left by its neighbour).  Measured on q_proj it LOSES (39 vs 26.7 us): each extra
// work item costs a full TMEM drain plus a 256 KB fp32 partial round trip, more than
// the ragged wave it removes.  Kept as a tested alternative schedule.
int pair_grid(const GemmArgs& a, const GemmConfig& cfg) {
  const int num_tiles = (int)(((a.M + 255) / 256) * ((a.N + 255) / 256));
  int grid = sm_count() & ~1;
  if (cfg.max_ctas > 0 && cfg.max_ctas < grid) grid = cfg.max_ctas & ~1;
  if (grid > 2 * num_tiles) grid = 2 * num_tiles;
  return grid;
}
bool use_stream_k(const GemmArgs& a, const GemmConfig& cfg) {
  const char* sk_env = getenv("MM_GEMM_STREAMK");   // read per call (tests switch it)
  const bool sk_env_on = sk_env && atoi(sk_env) == 1;
  const int num_tiles = (int)(((a.M + 255) / 256) * ((a.N + 255) / 256));
  const int npairs = pair_grid(a, cfg) / 2;
  return sk_env_on && !cfg.no_stream_k && !cfg.no_workspace && a.n_dst == 0 && npairs > 0 &&
         num_tiles > npairs && num_tiles % npairs != 0 && num_tiles < 4 * npairs;
}

// Balanced schedule for a ragged last wave (T whole tiles = q P + r with 0 < r < P, q >= 1;
// e.g. q_proj: 128 tiles on 74 pairs, qkv at M = 2048: 192 tiles).  Every pair takes q
// whole 256 x 256 tiles; what is left of each 256-row block (its columns past the whole
// tiles) is cut into narrow items of wn 64-column units (wn <= 3: 192 columns, so an item
// that starts 64 rows into a W scale atom still spans two row groups), at most one per
// pair, instead of r pairs computing a (q+1)-th whole tile while the others idle.  The
// whole tiles per row block a_b (summing to q P) come from a small DP that minimises the
// item count; q_proj ends with 74 whole tiles + 72 items of 192 columns (no pair above
// 448 columns instead of two whole tiles).  A narrow item still reads the whole 128-row
// A slab per stage, so it costs more than its share of columns (~81 % of a tile for 75 %
// of its columns at 192).  Results are cached per (row blocks, N, pairs).
struct Sched {
  bool ok = false;
  int q = 0;
  std::vector<uint16_t> a_pref;
  std::vector<uint32_t> narrow;
};
Sched build_sched_uncached(int num_m2, int64_t N, int P) {
  Sched r;
  const int U = (int)((N + 63) / 64);   // 64-column units per row block
  const int A = U / 4;                  // whole tiles per row block
  const int64_t T = (int64_t)num_m2 * ((N + 255) / 256);
  if (P < 1 || P > kMaxPairs || num_m2 > 64 || T <= P || T % P == 0) return r;
  const int q = (int)(T / P), QP = q * P;
  // Whole tiles are enumerated row-block-major here, not in the 8-row-block raster of the
  // data-parallel schedule; with many waves that costs more L2 reuse than the balanced
  // last wave gains (gate_up at M = 2048, q = 12: 142.5 -> 157.9 us), so few waves only.
  if (q > 3) return r;
  // (bounded host work: the DP runs once per shape, on the first call)
  if ((int64_t)num_m2 * A < QP || (int64_t)num_m2 * (QP + 1) * (A + 1) > 4000000) return r;
  for (int wn = 1; wn <= 3; ++wn) {
    // dp[b + 1][s]: fewest items over row blocks 0..b using s whole tiles; ch[b][s] = a_b
    const int INF = 1 << 29;
    std::vector<std::vector<int>> dp(num_m2 + 1, std::vector<int>(QP + 1, INF)), ch(num_m2, std::vector<int>(QP + 1, -1));
    dp[0][0] = 0;
    for (int b = 0; b < num_m2; ++b)
      for (int s0 = 0; s0 <= QP; ++s0) {
        if (dp[b][s0] >= INF) continue;
        for (int a = 0; a <= A && s0 + a <= QP; ++a) {
          const int v = dp[b][s0] + (U - 4 * a + wn - 1) / wn;
          if (v < dp[b + 1][s0 + a]) { dp[b + 1][s0 + a] = v; ch[b][s0 + a] = a; }
        }
      }
    if (dp[num_m2][QP] > P) continue;
    std::vector<int> a_b(num_m2);
    for (int b = num_m2 - 1, s1 = QP; b >= 0; --b) { a_b[b] = ch[b][s1]; s1 -= a_b[b]; }
    r.a_pref.assign(num_m2 + 1, 0);
    for (int b = 0; b < num_m2; ++b) r.a_pref[b + 1] = (uint16_t)(r.a_pref[b] + a_b[b]);
    r.narrow.assign(P, 0u);
    int k = 0;
    for (int b = 0; b < num_m2; ++b)
      for (int u = 4 * a_b[b]; u < U; u += wn)
        r.narrow[k++] = 0x80000000u | (uint32_t)b | (uint32_t)u << 10 | (uint32_t)std::min(wn, U - u) << 24;
    r.q = q;
    r.ok = true;
    return r;
  }
  return r;
}
const Sched& build_sched(int num_m2, int64_t N, int P) {
  static std::mutex mu;
  static std::map<std::tuple<int, int64_t, int>, Sched> cache;
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_tuple(num_m2, N, P);
  auto it = cache.find(key);
  if (it == cache.end()) it = cache.emplace(key, build_sched_uncached(num_m2, N, P)).first;
  return it->second;
}

template <int STAGES, int NP>
cudaError_t run2(const GemmArgs& a, const GemmConfig& cfg, cudaStream_t s, int64_t* launches, const char** err) {
  CUtensorMap maps[12];
  YMaps<NP> ym;
  int first = -1;
  for (int g = 0; g < 3; ++g) {
    if (a.geom.n[g] == 0) continue;
    const int box_atoms = g == 0 ? 2 : 1;
    if (!make_operand_map(&maps[g], a.a_codes[g], g, a.geom.kp[g], a.M, a.geom.pitch[g], 128) ||
        !make_operand_map(&maps[3 + g], a.w_codes[g], g, a.geom.kp[g], a.N, a.geom.pitch[g], 128) ||
        !make_sf_map(&maps[6 + g], a.a_sf[g], a.M, a.geom.kp[g], box_atoms) ||
        !make_sf_map(&maps[9 + g], a.w_sf[g], a.N, a.geom.kp[g], box_atoms)) {
      *err = "cuTensorMapEncodeTiled failed";
      return cudaErrorInvalidValue;
    }
    if (first < 0) first = g;
  }
  if (first < 0) { *err = "empty plan"; return cudaErrorInvalidValue; }
  for (int g = 0; g < 3; ++g)
    if (a.geom.n[g] == 0)
      for (int k = 0; k < 4; ++k) maps[3 * k + g] = maps[3 * k + first];   // valid, never used
  // Y [M, N] BF16 row-major (ld = ldy): TMA store boxes of 32 rows x 32 columns; in
  // peer mode one map per destination rank (its Y + this rank's column offset).
  const int ndst = NP == 1 ? 1 : a.n_dst;
  for (int dst = 0; dst < ndst; ++dst) {
    EncodeTiledFn enc = tensor_map_encoder();
    cuuint64_t dims[2] = {(cuuint64_t)a.N, (cuuint64_t)a.M};
    cuuint64_t strides[1] = {(cuuint64_t)a.ldy * 2};
    cuuint32_t box[2] = {32, 32};
    cuuint32_t estr[2] = {1, 1};
    uint16_t* base = NP == 1 ? a.y : a.y_dst[dst] + a.y_col_off;
    if (!enc || enc(&ym.m[dst], CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, base, dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      *err = "cuTensorMapEncodeTiled(Y) failed";
      return cudaErrorInvalidValue;
    }
  }
  for (int dst = ndst; dst < NP; ++dst) ym.m[dst] = ym.m[0];   // valid, never used
  Gemm2Dev p{};
  p.M = a.M;
  p.N = a.N;
  p.num_m2 = (int)((a.M + 255) / 256);
  p.num_n = (int)((a.N + 255) / 256);
  p.num_tiles = p.num_m2 * p.num_n;
  p.nst0 = (a.geom.kp[0] + 255) / 256;
  p.nst1 = a.geom.kp[1] / 128;
  p.nst2 = a.geom.kp[2] / 128;
  p.n0 = a.geom.n[0]; p.n1 = a.geom.n[1]; p.n2 = a.geom.n[2];
  p.kp0 = a.geom.kp[0]; p.kp1 = a.geom.kp[1]; p.kp2 = a.geom.kp[2];
  p.idesc0 = make_idesc_mn(a.geom.fmt[0], 0, 256, 256);
  p.idesc1 = make_idesc_mn(a.geom.fmt[1], 1, 256, 256);
  p.idesc2 = make_idesc_mn(a.geom.fmt[2], 2, 256, 256);
  p.y = a.y;
  p.ldy = a.ldy;
  p.ndst = ndst;
  p.y_mc = a.y_mc;
  p.mc_col_off = a.y_col_off;
  { const char* d = getenv("MM_GEMM_DEBUG"); p.dbg = d ? atoi(d) : 0; }
  {
    // raster groups of 8 pair-row blocks; 16 for very wide layers (>= 64 column tiles:
    // gate_up at M = 16384 1088 -> 1065 us, Qwen gate_up N = 55296 1263 -> 1232 us; the
    // N <= 8192 layers measured 0.2-1.8 % slower with 16, so they keep 8)
    const char* r = getenv("MM_GEMM_RASTER");
    p.raster = (r && atoi(r) > 0) ? atoi(r) : (p.num_n >= 64 ? 16 : 8);
  }
  if (p.num_tiles == 0) return cudaSuccess;
  const int grid = pair_grid(a, cfg);
  const int npairs = grid / 2;
  p.stream_k = use_stream_k(a, cfg) ? 1 : 0;
  { const char* e = getenv("MM_GEMM_SFBMC"); p.sfb_mc = e ? atoi(e) : 1; }
  {
    // balanced schedule (build_sched) for a ragged last wave; MM_GEMM_SPLIT2=0 turns it off
    const char* e = getenv("MM_GEMM_SPLIT2");
    const bool want = e ? atoi(e) == 1 : true;
    p.sched2 = 0;
    if (!p.stream_k && want) {
      const Sched& sc = build_sched(p.num_m2, a.N, npairs);
      if (sc.ok) {
        p.sched2 = 1;
        p.sq = sc.q;
        p.npairs = npairs;
        for (int b = 0; b <= p.num_m2; ++b) p.a_pref[b] = sc.a_pref[b];
        for (int q = 0; q < npairs; ++q) p.narrow[q] = sc.narrow[q];
      }
    }
  }
  // Helper drain of the last tile: for few tiles per pair (<= 4), where the exposed final
  // drain is a visible share of the kernel (q_proj: 27 -> 25 us); measured ~1 % slower
  // with ~14 tiles per pair (70B down_proj), so off there.  MM_GEMM_HELPERS=0/1 forces it.
  {
    const char* h = getenv("MM_GEMM_HELPERS");
    const bool want = h ? atoi(h) == 1 : p.num_tiles <= 4 * npairs;
    p.helpers = (!p.stream_k && !p.y_mc && want) ? 1 : 0;
  }
  if (p.stream_k) {   // caller workspace: [flags npairs x 8 ints, 256-B padded][partials]
    if (!a.ws || a.ws_bytes < pair_workspace_bytes(a, cfg)) {
      *err = "stream-K workspace missing or too small";
      return cudaErrorInvalidValue;
    }
    p.ws_flag = static_cast<int*>(a.ws);
    p.ws = reinterpret_cast<float*>(static_cast<uint8_t*>(a.ws) + ws_align((size_t)npairs * 8 * sizeof(int)));
  }
  const size_t smem = 1024 + (size_t)STAGES * STAGE_BYTES + epi_bytes<STAGES>() + (2 * STAGES + 11) * 8 + 16;
  auto kern = (NP == 1 && !p.stream_k && !p.y_mc && p.dbg == 0) ? mixgemm2_kernel<STAGES, NP, true>
                                                                : mixgemm2_kernel<STAGES, NP, false>;
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), smem);
  if (e != cudaSuccess) { *err = "cudaFuncSetAttribute(smem) failed"; return e; }
  e = launch_pdl(kern, dim3(grid), dim3(kThreads2), smem, s, maps[0], maps[1], maps[2], maps[3], maps[4], maps[5],
                 maps[6], maps[7], maps[8], maps[9], maps[10], maps[11], ym, p);
  if (launches) ++*launches;
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace
}  // namespace mmx

// Debug hook (not part of include/mm.h): copy the GEMM timeline trace to the host.
extern "C" int mm_debug_gemm_trace(unsigned long long* h, int n) {
  return (int)cudaMemcpyFromSymbol(h, mmx::g_trace, sizeof(unsigned long long) * (size_t)(n < 3840 ? n : 3840));
}

namespace mmx {

size_t pair_workspace_bytes(const GemmArgs& a, const GemmConfig& cfg) {
  if (!use_stream_k(a, cfg)) return 0;
  const size_t npairs = (size_t)(pair_grid(a, cfg) / 2);
  return ws_align(npairs * 8 * sizeof(int)) + npairs * 256 * 256 * sizeof(float);
}

cudaError_t launch_mixed_gemm_2cta(const GemmArgs& a, const GemmConfig& cfg, cudaStream_t s, int64_t* launches,
                                   const char** err) {
  if (a.n_dst > 0) return run2<5, kMaxPeers>(a, cfg, s, launches, err);   // fused all-gather epilogue
  // default 6 stages (one epilogue staging buffer per warp makes room): +0.6-1 %
  // over 5 with the two-producer pipeline, bit-identical results
  if (cfg.num_stages == 4) return run2<4, 1>(a, cfg, s, launches, err);
  if (cfg.num_stages == 5) return run2<5, 1>(a, cfg, s, launches, err);
  return run2<6, 1>(a, cfg, s, launches, err);
}

}  // namespace mmx
