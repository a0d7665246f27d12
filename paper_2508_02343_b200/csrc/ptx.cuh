// ptx.cuh -- thin inline-PTX wrappers for sm_100a (mbarrier, TMA, tcgen05).
#pragma once
#include <cstdint>
#include <cstdio>

namespace mmx {
namespace ptx {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- mbarrier ----------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// Wait for the phase with parity `parity` to complete.  Watchdog: a wait that
// lasts longer than MM_WATCHDOG_NS (default 4 s; 0 disables) prints the site
// and traps, so a pipeline bug surfaces as a launch error instead of a hang.
#ifndef MM_WATCHDOG_NS
#define MM_WATCHDOG_NS 4000000000ull
#endif
static __device__ __noinline__ void watchdog_fire(int tag, uint32_t bar, uint32_t parity, int a, int b) {
  printf("[mm watchdog] block %d thread %d: mbarrier wait tag=%d bar=0x%x parity=%u info=(%d,%d) timed out\n",
         blockIdx.x, threadIdx.x, tag, bar, parity, a, b);
  __trap();
}
// try_wait with a suspend-time hint (ns): the waiting thread sleeps until the phase
// completes or the hint expires, instead of re-polling (for warps that wait long).
__device__ __forceinline__ bool mbar_try_wait_hint(uint32_t bar, uint32_t parity, uint32_t ns) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity), "r"(ns)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t parity, int tag = 0, int a = 0, int b = 0) {
#if MM_WATCHDOG_NS
  uint64_t t0 = 0;
  for (uint32_t n = 0; !mbar_try_wait_hint(bar, parity, 20000u); ++n) {
    if (n == 0) t0 = globaltimer_ns();
    else if (globaltimer_ns() - t0 > (uint64_t)MM_WATCHDOG_NS) watchdog_fire(tag, bar, parity, a, b);
  }
#else
  while (!mbar_try_wait_hint(bar, parity, 20000u)) {
  }
#endif
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity, int tag = 0, int a = 0, int b = 0) {
  if (mbar_try_wait(bar, parity)) return;
#if MM_WATCHDOG_NS
  // the timer is read once per 1024 polls (an inner loop without it), so the spin
  // costs two instructions per poll
  const uint64_t t0 = globaltimer_ns();
  for (;;) {
#pragma unroll 1
    for (int n = 0; n < 1024; ++n)
      if (mbar_try_wait(bar, parity)) return;
    if (globaltimer_ns() - t0 > (uint64_t)MM_WATCHDOG_NS) watchdog_fire(tag, bar, parity, a, b);
  }
#else
  while (!mbar_try_wait(bar, parity)) {
  }
#endif
}

__device__ __forceinline__ void named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// ---- TMA / bulk copies ---------------------------------------------------------
__device__ __forceinline__ void tma_prefetch_desc(const void* desc) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(desc)) : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const void* desc, uint32_t bar, int32_t c0,
                                            int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const void* desc, uint32_t bar, int32_t c0,
                                            int32_t c1, int32_t c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(bar)
      : "memory");
}

// ---- tcgen05 -------------------------------------------------------------------
__device__ __forceinline__ void tmem_alloc(uint32_t dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(dst_smem),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}
// smem (32 rows x 128 bit, one 512-byte scale atom) -> TMEM, replicated to the
// four 32-lane quadrants.
__device__ __forceinline__ void tc_cp_32x128b_x4(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}
__device__ __forceinline__ void tc_mma_mxf8f6f4(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                uint32_t sfa, uint32_t sfb, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::mxf8f6f4.block_scale [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum), "r"(sfa), "r"(sfb)
      : "memory");
}
__device__ __forceinline__ void tc_mma_mxf4(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t sfa, uint32_t sfb, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum), "r"(sfa), "r"(sfb)
      : "memory");
}
// ---- whole-stage issue blocks for single-CTA kernels (the small-M kernel) -----------
// Executed by a full, converged warp: elect.sync picks the issuing lane.  One FP8/FP6
// stage: 2 scale copies (operand A atom, operand B atom) + 4 MMAs (K = 32, scale ids
// 0..3) + a commit to `bar`.
__device__ __forceinline__ void stage_f8f6_cg1(uint32_t d, uint64_t ad, uint64_t bd, uint32_t id0, uint32_t sfa,
                                               uint32_t sfb, uint64_t sda, uint64_t sdb, uint32_t accum,
                                               uint32_t bar) {
  const uint32_t id1 = id0 | (1u << 29) | (1u << 4), id2 = id0 | (2u << 29) | (2u << 4), id3 = id0 | (3u << 29) | (3u << 4);
  asm volatile(
      "{\n\t.reg .pred p, acc, one;\n\t.reg .b64 a1, a2, a3, b1, b2, b3;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "setp.ne.b32 acc, %8, 0;\n\t"
      "setp.eq.b32 one, 0, 0;\n\t"
      "add.s64 a1, %1, 2;\n\tadd.s64 a2, %1, 4;\n\tadd.s64 a3, %1, 6;\n\t"
      "add.s64 b1, %2, 2;\n\tadd.s64 b2, %2, 4;\n\tadd.s64 b3, %2, 6;\n\t"
      "@p tcgen05.cp.cta_group::1.32x128b.warpx4 [%4], %6;\n\t"
      "@p tcgen05.cp.cta_group::1.32x128b.warpx4 [%5], %7;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::mxf8f6f4.block_scale [%0], %1, %2, %3, [%4], [%5], acc;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::mxf8f6f4.block_scale [%0], a1, b1, %9, [%4], [%5], one;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::mxf8f6f4.block_scale [%0], a2, b2, %10, [%4], [%5], one;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::mxf8f6f4.block_scale [%0], a3, b3, %11, [%4], [%5], one;\n\t"
      "@p tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%12];\n\t}"
      ::"r"(d), "l"(ad), "l"(bd), "r"(id0), "r"(sfa), "r"(sfb), "l"(sda), "l"(sdb), "r"(accum), "r"(id1), "r"(id2),
        "r"(id3), "r"(bar)
      : "memory");
}
// One full FP4 stage: 2 atoms each of the A and B scales + 4 kind::mxf4 MMAs (K = 64;
// MMA k uses atom k/2, scale ids 0/2) + commit.
__device__ __forceinline__ void stage_f4_cg1(uint32_t d, uint64_t ad, uint64_t bd, uint32_t id0, uint32_t sfa,
                                             uint32_t sfb, uint64_t sda, uint64_t sdb, uint32_t accum, uint32_t bar) {
  const uint32_t id2 = id0 | (2u << 29) | (2u << 4);
  const uint32_t sfa4 = sfa + 4, sfb4 = sfb + 4;
  asm volatile(
      "{\n\t.reg .pred p, acc, one;\n\t.reg .b64 a1, a2, a3, b1, b2, b3, sa1, sb1;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "setp.ne.b32 acc, %8, 0;\n\t"
      "setp.eq.b32 one, 0, 0;\n\t"
      "add.s64 a1, %1, 2;\n\tadd.s64 a2, %1, 4;\n\tadd.s64 a3, %1, 6;\n\t"
      "add.s64 b1, %2, 2;\n\tadd.s64 b2, %2, 4;\n\tadd.s64 b3, %2, 6;\n\t"
      "add.s64 sa1, %6, 32;\n\tadd.s64 sb1, %7, 32;\n\t"
      "@p tcgen05.cp.cta_group::1.32x128b.warpx4 [%4], %6;\n\t"
      "@p tcgen05.cp.cta_group::1.32x128b.warpx4 [%10], sa1;\n\t"
      "@p tcgen05.cp.cta_group::1.32x128b.warpx4 [%5], %7;\n\t"
      "@p tcgen05.cp.cta_group::1.32x128b.warpx4 [%11], sb1;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%4], [%5], acc;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], a1, b1, %9, [%4], [%5], one;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], a2, b2, %3, [%10], [%11], one;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], a3, b3, %9, [%10], [%11], one;\n\t"
      "@p tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%12];\n\t}"
      ::"r"(d), "l"(ad), "l"(bd), "r"(id0), "r"(sfa), "r"(sfb), "l"(sda), "l"(sdb), "r"(accum), "r"(id2), "r"(sfa4),
        "r"(sfb4), "r"(bar)
      : "memory");
}
// Single-CTA stages whose W scales span two 128-row groups (N = 256 tiles): SFB row
// group r of atom a at TMEM column sfb + 4 (2a + r); in shared memory the atoms are laid
// out [atom][row group] (512 B each), so atom 1 is 1 KB (64 descriptor units) further.
__device__ __forceinline__ void stage_f8f6_cg1_rg2(uint32_t d, uint64_t ad, uint64_t bd, uint32_t id0, uint32_t sfa,
                                                   uint32_t sfb, uint64_t sda, uint64_t sdb0, uint32_t accum,
                                                   uint32_t bar) {
  const uint32_t id1 = id0 | (1u << 29) | (1u << 4), id2 = id0 | (2u << 29) | (2u << 4), id3 = id0 | (3u << 29) | (3u << 4);
  const uint32_t sfb4 = sfb + 4;
  asm volatile(
      "{\n\t.reg .pred p, acc, one;\n\t.reg .b64 a1, a2, a3, b1, b2, b3, s1;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "setp.ne.b32 acc, %8, 0;\n\t"
      "setp.eq.b32 one, 0, 0;\n\t"
      "add.s64 a1, %1, 2;\n\tadd.s64 a2, %1, 4;\n\tadd.s64 a3, %1, 6;\n\t"
      "add.s64 b1, %2, 2;\n\tadd.s64 b2, %2, 4;\n\tadd.s64 b3, %2, 6;\n\t"
      "add.s64 s1, %7, 32;\n\t"
      "@p tcgen05.cp.cta_group::1.32x128b.warpx4 [%4], %6;\n\t"
      "@p tcgen05.cp.cta_group::1.32x128b.warpx4 [%5], %7;\n\t"
      "@p tcgen05.cp.cta_group::1.32x128b.warpx4 [%12], s1;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::mxf8f6f4.block_scale [%0], %1, %2, %3, [%4], [%5], acc;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::mxf8f6f4.block_scale [%0], a1, b1, %9, [%4], [%5], one;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::mxf8f6f4.block_scale [%0], a2, b2, %10, [%4], [%5], one;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::mxf8f6f4.block_scale [%0], a3, b3, %11, [%4], [%5], one;\n\t"
      "@p tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%13];\n\t}"
      ::"r"(d), "l"(ad), "l"(bd), "r"(id0), "r"(sfa), "r"(sfb), "l"(sda), "l"(sdb0), "r"(accum), "r"(id1), "r"(id2),
        "r"(id3), "r"(sfb4), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void stage_f4_cg1_rg2(uint32_t d, uint64_t ad, uint64_t bd, uint32_t id0, uint32_t sfa,
                                                 uint32_t sfb, uint64_t sda, uint64_t sdb0, uint32_t accum,
                                                 uint32_t bar) {
  const uint32_t id2 = id0 | (2u << 29) | (2u << 4);
  const uint32_t sfa4 = sfa + 4, sfb4 = sfb + 4, sfb8 = sfb + 8, sfb12 = sfb + 12;
  asm volatile(
      "{\n\t.reg .pred p, acc, one;\n\t.reg .b64 a1, a2, a3, b1, b2, b3, sa1, s01, s10, s11;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "setp.ne.b32 acc, %8, 0;\n\t"
      "setp.eq.b32 one, 0, 0;\n\t"
      "add.s64 a1, %1, 2;\n\tadd.s64 a2, %1, 4;\n\tadd.s64 a3, %1, 6;\n\t"
      "add.s64 b1, %2, 2;\n\tadd.s64 b2, %2, 4;\n\tadd.s64 b3, %2, 6;\n\t"
      "add.s64 sa1, %6, 32;\n\tadd.s64 s01, %7, 32;\n\tadd.s64 s10, %7, 64;\n\tadd.s64 s11, %7, 96;\n\t"
      "@p tcgen05.cp.cta_group::1.32x128b.warpx4 [%4], %6;\n\t"
      "@p tcgen05.cp.cta_group::1.32x128b.warpx4 [%10], sa1;\n\t"
      "@p tcgen05.cp.cta_group::1.32x128b.warpx4 [%5], %7;\n\t"
      "@p tcgen05.cp.cta_group::1.32x128b.warpx4 [%11], s01;\n\t"
      "@p tcgen05.cp.cta_group::1.32x128b.warpx4 [%12], s10;\n\t"
      "@p tcgen05.cp.cta_group::1.32x128b.warpx4 [%13], s11;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%4], [%5], acc;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], a1, b1, %9, [%4], [%5], one;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], a2, b2, %3, [%10], [%12], one;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], a3, b3, %9, [%10], [%12], one;\n\t"
      "@p tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%14];\n\t}"
      ::"r"(d), "l"(ad), "l"(bd), "r"(id0), "r"(sfa), "r"(sfb), "l"(sda), "l"(sdb0), "r"(accum), "r"(id2), "r"(sfa4),
        "r"(sfb4), "r"(sfb8), "r"(sfb12), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// 32 lanes x 32 consecutive 32-bit columns -> 32 registers per thread.
__device__ __forceinline__ void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
        "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
        "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
}

// Shared-memory matrix descriptor (tcgen05 "matrix descriptor"): start >> 4 in
// [0,14), LBO >> 4 in [16,30), SBO >> 4 in [32,46), version 1 at bit 46,
// base offset 0, layout type in [61,64) (2 = 128-byte swizzle, 0 = none).
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(layout & 7) << 61;
  return d;
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

// ---- programmatic dependent launch ----------------------------------------------
// wait: block until the preceding grid in the stream has completed and its memory
// is visible (call before touching anything it may produce or still read);
// launch_dependents: allow the next grid to be scheduled as SMs free up.
__device__ __forceinline__ void grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void grid_dep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---- clusters / CTA pairs ------------------------------------------------------
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cta address of this CTA -> shared::cluster address of the same offset in CTA `rank`.
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// 2-SM TMA: data lands in this CTA's smem, the transaction bytes complete on the
// barrier of the pair's even CTA (peer bit cleared, as CUTLASS SM100_TMA_2SM_LOAD).
__device__ __forceinline__ void tma_load_2d_cg2(uint32_t dst, const void* desc, uint32_t bar, int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(c0), "r"(c1), "r"(bar & 0xFEFFFFFFu)
      : "memory");
}
// Same, multicast: the box lands at `dst` in every CTA of `mask`; each destination's
// bytes complete on the barrier of that CTA's pair leader (CUTLASS SM100_TMA_2SM_LOAD_MULTICAST).
__device__ __forceinline__ void tma_load_2d_cg2_mc(uint32_t dst, const void* desc, uint32_t bar, int32_t c0, int32_t c1,
                                                   uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(c0), "r"(c1), "r"(bar & 0xFEFFFFFFu), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void tmem_alloc_cg2(uint32_t dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(dst_smem), "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_cg2(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
// commit all prior tcgen05 ops of this thread; arrive on the barrier at the same
// offset in every CTA of `mask` (both CTAs of the pair: 0b11).
__device__ __forceinline__ void tc_commit_cg2_mc(uint32_t bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
      "h"(mask)
      : "memory");
}
__device__ __forceinline__ void tc_cp_32x128b_x4_cg2(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::2.32x128b.warpx4 [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}
__device__ __forceinline__ void tc_mma_mxf8f6f4_cg2(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                    uint32_t sfa, uint32_t sfb, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::mxf8f6f4.block_scale [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum), "r"(sfa), "r"(sfb)
      : "memory");
}
__device__ __forceinline__ void tc_mma_mxf4_cg2(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                uint32_t sfa, uint32_t sfb, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum), "r"(sfa), "r"(sfb)
      : "memory");
}

// ---- whole-stage issue blocks for the CTA-pair GEMM ---------------------------------
// Executed by a full, converged warp: elect.sync picks the single issuing lane, so
// all operands stay warp-uniform (no per-instruction lane loops).  One FP8/FP6
// stage: 3 scale-atom copies (SFA, SFB row groups 0/1) + 4 MMAs (K = 32 each,
// scale-factor ids 0..3) + a commit that frees the smem stage in both CTAs.
__device__ __forceinline__ void stage_f8f6_cg2(uint32_t d, uint64_t ad, uint64_t bd, uint32_t id0, uint32_t sfa,
                                               uint32_t sfb, uint64_t sda, uint64_t sdb0, uint64_t sdb1,
                                               uint32_t accum, uint32_t empty_bar, uint32_t do_cp = 1,
                                               uint32_t sfbm = 0xFFFFFFFFu, uint16_t mask = 3) {
  // sfbm: the SFB address the MMAs read (default sfb).  An item whose first output
  // column sits 64 rows into a scale atom reads from sfb + 2 (two 32-row TMEM words).
  if (sfbm == 0xFFFFFFFFu) sfbm = sfb;
  const uint32_t sfb4 = sfb + 4;
  const uint32_t id1 = id0 | (1u << 29) | (1u << 4), id2 = id0 | (2u << 29) | (2u << 4), id3 = id0 | (3u << 29) | (3u << 4);
  asm volatile(
      "{\n\t.reg .pred p, acc, one, c;\n\t.reg .b64 a1, a2, a3, b1, b2, b3;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "setp.ne.b32 acc, %9, 0;\n\t"
      "setp.eq.b32 one, 0, 0;\n\t"
      "setp.ne.and.b32 c, %16, 0, p;\n\t"
      "add.s64 a1, %1, 2;\n\tadd.s64 a2, %1, 4;\n\tadd.s64 a3, %1, 6;\n\t"
      "add.s64 b1, %2, 2;\n\tadd.s64 b2, %2, 4;\n\tadd.s64 b3, %2, 6;\n\t"
      "@c tcgen05.cp.cta_group::2.32x128b.warpx4 [%4], %6;\n\t"
      "@c tcgen05.cp.cta_group::2.32x128b.warpx4 [%5], %7;\n\t"
      "@c tcgen05.cp.cta_group::2.32x128b.warpx4 [%13], %8;\n\t"
      "@p tcgen05.mma.cta_group::2.kind::mxf8f6f4.block_scale [%0], %1, %2, %3, [%4], [%17], acc;\n\t"
      "@p tcgen05.mma.cta_group::2.kind::mxf8f6f4.block_scale [%0], a1, b1, %10, [%4], [%17], one;\n\t"
      "@p tcgen05.mma.cta_group::2.kind::mxf8f6f4.block_scale [%0], a2, b2, %11, [%4], [%17], one;\n\t"
      "@p tcgen05.mma.cta_group::2.kind::mxf8f6f4.block_scale [%0], a3, b3, %12, [%4], [%17], one;\n\t"
      "@p tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%14], %15;\n\t}"
      ::"r"(d), "l"(ad), "l"(bd), "r"(id0), "r"(sfa), "r"(sfb), "l"(sda), "l"(sdb0), "l"(sdb1), "r"(accum),
        "r"(id1), "r"(id2), "r"(id3), "r"(sfb4), "r"(empty_bar), "h"(mask), "r"(do_cp), "r"(sfbm)
      : "memory");
}
// One full FP4 stage: 2 atoms each of SFA and of SFB row groups 0/1 + 4
// kind::mxf4 MMAs (K = 64; MMA k uses atom k/2, scale-factor ids 0/2) + commit.
__device__ __forceinline__ void stage_f4_cg2(uint32_t d, uint64_t ad, uint64_t bd, uint32_t id0, uint32_t sfa,
                                             uint32_t sfb, uint64_t sda, uint64_t sdb0, uint64_t sdb1,
                                             uint32_t accum, uint32_t empty_bar, uint32_t sfbm = 0xFFFFFFFFu,
                                             uint16_t mask = 3) {
  // SFA atoms at columns sfa, sfa+4; SFB (atom a, row group r) at sfb + (2a + r) * 4;
  // the MMAs read SFB from sfbm (default sfb; +2 for an item starting 64 rows into an atom)
  if (sfbm == 0xFFFFFFFFu) sfbm = sfb;
  const uint32_t sfa4 = sfa + 4, sfb4 = sfb + 4, sfb8 = sfb + 8, sfb12 = sfb + 12, sfbm8 = sfbm + 8;
  const uint32_t id2 = id0 | (2u << 29) | (2u << 4);
  asm volatile(
      "{\n\t.reg .pred p, acc, one;\n\t.reg .b64 a1, a2, a3, b1, b2, b3, sa1, s01, s11;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "setp.ne.b32 acc, %9, 0;\n\t"
      "setp.eq.b32 one, 0, 0;\n\t"
      "add.s64 a1, %1, 2;\n\tadd.s64 a2, %1, 4;\n\tadd.s64 a3, %1, 6;\n\t"
      "add.s64 b1, %2, 2;\n\tadd.s64 b2, %2, 4;\n\tadd.s64 b3, %2, 6;\n\t"
      "add.s64 sa1, %6, 32;\n\tadd.s64 s01, %7, 32;\n\tadd.s64 s11, %8, 32;\n\t"
      "@p tcgen05.cp.cta_group::2.32x128b.warpx4 [%4], %6;\n\t"
      "@p tcgen05.cp.cta_group::2.32x128b.warpx4 [%11], sa1;\n\t"
      "@p tcgen05.cp.cta_group::2.32x128b.warpx4 [%5], %7;\n\t"
      "@p tcgen05.cp.cta_group::2.32x128b.warpx4 [%12], %8;\n\t"
      "@p tcgen05.cp.cta_group::2.32x128b.warpx4 [%13], s01;\n\t"
      "@p tcgen05.cp.cta_group::2.32x128b.warpx4 [%14], s11;\n\t"
      "@p tcgen05.mma.cta_group::2.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%4], [%17], acc;\n\t"
      "@p tcgen05.mma.cta_group::2.kind::mxf4.block_scale.scale_vec::2X [%0], a1, b1, %10, [%4], [%17], one;\n\t"
      "@p tcgen05.mma.cta_group::2.kind::mxf4.block_scale.scale_vec::2X [%0], a2, b2, %3, [%11], [%18], one;\n\t"
      "@p tcgen05.mma.cta_group::2.kind::mxf4.block_scale.scale_vec::2X [%0], a3, b3, %10, [%11], [%18], one;\n\t"
      "@p tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%15], %16;\n\t}"
      ::"r"(d), "l"(ad), "l"(bd), "r"(id0), "r"(sfa), "r"(sfb), "l"(sda), "l"(sdb0), "l"(sdb1), "r"(accum),
        "r"(id2), "r"(sfa4), "r"(sfb4), "r"(sfb8), "r"(sfb12), "r"(empty_bar), "h"(mask), "r"(sfbm), "r"(sfbm8)
      : "memory");
}
__device__ __forceinline__ void commit_cg2_mc_elect(uint32_t bar, uint16_t mask = 3) {
  asm volatile(
      "{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\t"
      "@p tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}"
      ::"r"(bar), "h"(mask)
      : "memory");
}

// ---- TMA stores -----------------------------------------------------------------
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tma_store_2d(const void* desc, uint32_t src, int32_t c0, int32_t c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(desc)),
               "r"(c0), "r"(c1), "r"(src)
               : "memory");
}
__device__ __forceinline__ void bulk_commit_group() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_group() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_group_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

}  // namespace ptx
}  // namespace mmx
