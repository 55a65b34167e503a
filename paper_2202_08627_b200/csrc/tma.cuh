// tma.cuh — thin inline-PTX helpers for the sm_100a async-copy pipeline used by K1/K3:
// 1-D bulk copies global -> shared (cp.async.bulk, the TMA engine's non-tensor mode) completing
// on an mbarrier transaction count, and the mbarrier init / arrive / wait primitives.
#pragma once
#include <stdint.h>

namespace ei {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

// make mbarrier inits visible to the async proxy (TMA) and the other threads
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// The same wait with a suspend-time hint: the warp sleeps in the barrier unit (SASS
// NANOSLEEP.SYNCS, woken when the phase completes) instead of re-issuing try_wait.  Used by K1's
// producer warp waiting for a free stage (C4 K1 8.84 -> 8.80 ms); K2's and K3's producers and all
// consumers keep spinning (sleeping there measured 0-1 % slower, tools/dbg/ab_defs.sh)
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *bar, uint32_t parity) {
#ifdef EI_SPIN_WAIT   // A/B switch: the plain spinning wait
  mbar_wait(bar, parity);
  return;
#endif
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(1000000u)
      : "memory");
}

// consumers waiting for a filled stage: spin (default) or sleep (A/B switch EI_CONSUMER_SLEEP)
__device__ __forceinline__ void mbar_wait_full(uint64_t *bar, uint32_t parity) {
#ifdef EI_CONSUMER_SLEEP
  mbar_wait_sleep(bar, parity);
#else
  mbar_wait(bar, parity);
#endif
}

// bytes must be a multiple of 16; src and dst 16-B aligned
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Programmatic dependent launch (PDL): a kernel launched with launch_pdl() may start while its
// stream predecessor is still running; every thread that reads the predecessor's output first
// executes pdl_wait() (returns once the predecessor grid has completed and its writes are
// visible).  pdl_trigger() lets the dependent grid's CTAs be scheduled before this grid exits.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
// K0 triggers K1 at its start: K1's CTAs are scheduled once all of K0's CTAs have started and
// run their prologue while K0 works (whatever they read of K0's output they read after
// pdl_wait(), which waits for K0's completion): C1 28.8 -> 26.7 us.  The later kernels trigger
// at the end of their work: an early trigger there let the next single-wave grid (K3 after K2)
// land on whichever SMs happened to be free while the imbalanced predecessor still ran, and C2
// lost 3 us (tools/dbg/step_trace.py).
#ifdef EI_NO_K0_TRIGGER
#define PDL_TRIGGER_K0()
#else
#define PDL_TRIGGER_K0() pdl_trigger()
#endif

}  // namespace ei
