// vxb_ptx.cuh — thin inline-PTX wrappers for the sm_100a features the
// convolution kernels use: mbarriers, TMA (cp.async.bulk[.tensor]), and the
// tcgen05 family (TMEM alloc, UMMA issue/commit, TMEM loads).
#pragma once
#include <cstdint>
#include <cuda.h>

namespace vxb {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ bool mbar_test(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// try_wait with a suspend-time hint: the thread is parked until the phase
// completes (woken by the barrier, not by a timer), so idle waiters neither
// spin nor oversleep past the phase flip.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAITS_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAITS_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(10000000u)
      : "memory");
}

// ---------------------------------------------------------------- TMA
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap *m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(m) : "memory");
}
__device__ __forceinline__ void tma_load_4d(void *dst, const CUtensorMap *m, uint64_t *bar,
                                            int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_5d(void *dst, const CUtensorMap *m, uint64_t *bar,
                                            int c0, int c1, int c2, int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar))
      : "memory");
}
// plain bulk copy global -> shared, completes on the mbarrier
__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes,
                                          uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// multicast bulk copy: the same bytes land at the same smem offset of every
// CTA in cta_mask, each CTA's mbarrier (same offset) gets the complete_tx
__device__ __forceinline__ void bulk_load_mc(void *dst, const void *src, uint32_t bytes,
                                             uint64_t *bar, uint16_t cta_mask) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "h"(cta_mask)
      : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

// CTA-pair (cta_group::2) forms.  A shared::cta address has the pair-rank bit
// at bit 24; clearing it names the same offset in the leader CTA (rank 0).
constexpr uint32_t PEER_BIT_MASK = 0xFEFFFFFFu;
// shared::cluster address of the same smem offset in the pair leader (rank 0)
__device__ __forceinline__ uint32_t leader_addr(const void *p) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(smem_u32(p)));
  return r;
}
__device__ __forceinline__ void tma_load_4d_pair(void *dst, const CUtensorMap *m, uint64_t *bar,
                                                 int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(leader_addr(bar))
      : "memory");
}
// arrive on the mbarrier at the same offset in CTA `cta` of the cluster
// arrive on CTA `cta`'s barrier at the same smem offset, releasing this
// thread's prior shared-memory writes at cluster scope
__device__ __forceinline__ void mbar_arrive_cta_release(uint64_t *bar, uint32_t cta) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\t"
      "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
      "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n}" ::"r"(smem_u32(bar)),
      "r"(cta)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_cta(uint64_t *bar, uint32_t cta) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\t"
      "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
      "mbarrier.arrive.shared::cluster.b64 _, [ra];\n}" ::"r"(smem_u32(bar)),
      "r"(cta)
      : "memory");
}

// ---------------------------------------------------------------- tcgen05
__device__ __forceinline__ void tmem_alloc(uint32_t *dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tmem_alloc_pair(uint32_t *dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tmem_relinquish_pair() {
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tmem_relinquish() {
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
// D[tmem] (+)= A[smem] * B[smem]^T, bf16 inputs, fp32 accumulate
__device__ __forceinline__ void umma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// warp-collective forms: every lane executes, one elected lane issues
__device__ __forceinline__ void umma_bf16_elect(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                                uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit_elect(uint64_t *bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(
          smem_u32(bar))
      : "memory");
}
// M = 256 across the CTA pair: A rows 0-127 / 128-255 and B rows [0, N/2) /
// [N/2, N) come from the two CTAs' smem at the same offsets; issued by the
// leader only
__device__ __forceinline__ void umma_bf16_pair_elect(uint32_t d_tmem, uint64_t a_desc,
                                                     uint64_t b_desc, uint32_t idesc,
                                                     uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit_pair_elect(uint64_t *bar, uint16_t cta_mask) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;\n}" ::"r"(smem_u32(bar)),
      "h"(cta_mask)
      : "memory");
}
__device__ __forceinline__ void umma_commit_mc_elect(uint64_t *bar, uint16_t cta_mask) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;\n}" ::"r"(smem_u32(bar)),
      "h"(cta_mask)
      : "memory");
}
// arrive on the mbarrier once all previously issued tcgen05 ops of this thread finish
__device__ __forceinline__ void umma_commit(uint64_t *bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}
// 32 lanes x 32 bit, 16 consecutive columns: thread t gets row (lane base + t)
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// 32 lanes x 32 bit, 32 consecutive columns
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// split TMEM load: issue now, wait later (the wait names the registers so
// the compiler cannot read them before the data has arrived)
__device__ __forceinline__ void tmem_ld16_issue(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_wait_ld16(uint32_t (&r)[16]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15]) : : "memory");
}

// zero 16 consecutive accumulator columns of this warp's 32 TMEM lanes
__device__ __forceinline__ void tmem_st16_zero(uint32_t taddr) {
  const uint32_t z = 0u;
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr),
      "r"(z)
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// descriptor split into a low word (start address | LBO) and a high word
// (SBO | version | layout) so loops only add to the low word
__device__ __forceinline__ uint32_t desc_lo(uint32_t saddr, uint32_t lbo) {
  return ((saddr >> 4) & 0x3FFFu) | (((lbo >> 4) & 0x3FFFu) << 16);
}
__host__ __device__ inline uint32_t desc_hi(uint32_t sbo) {
  return ((sbo >> 4) & 0x3FFFu) | (1u << 14);   // version bit 46 -> bit 14 of the high word
}
__device__ __forceinline__ void umma_bf16_lohi(uint32_t d, uint32_t a_lo, uint32_t a_hi,
                                               uint32_t b_lo, uint32_t b_hi, uint32_t idesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b64 ad, bd;\n\t"
      "mov.b64 ad, {%1, %2};\n\tmov.b64 bd, {%3, %4};\n\t"
      "setp.ne.b32 p, %6, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], ad, bd, %5, p;\n}" ::"r"(d),
      "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_bf16_pair_lohi(uint32_t d, uint32_t a_lo, uint32_t a_hi,
                                                    uint32_t b_lo, uint32_t b_hi, uint32_t idesc,
                                                    uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b64 ad, bd;\n\t"
      "mov.b64 ad, {%1, %2};\n\tmov.b64 bd, {%3, %4};\n\t"
      "setp.ne.b32 p, %6, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], ad, bd, %5, p;\n}" ::"r"(d),
      "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(accumulate)
      : "memory");
}
// warp-collective lo/hi forms (convergent warp, one elected lane issues)
__device__ __forceinline__ void umma_bf16_lohi_elect(uint32_t d, uint32_t a_lo, uint32_t a_hi,
                                                     uint32_t b_lo, uint32_t b_hi, uint32_t idesc,
                                                     uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\t.reg .b64 ad, bd;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "mov.b64 ad, {%1, %2};\n\tmov.b64 bd, {%3, %4};\n\t"
      "setp.ne.b32 p, %6, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ad, bd, %5, p;\n}" ::"r"(d),
      "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_bf16_pair_lohi_elect(uint32_t d, uint32_t a_lo,
                                                          uint32_t a_hi, uint32_t b_lo,
                                                          uint32_t b_hi, uint32_t idesc,
                                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\t.reg .b64 ad, bd;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "mov.b64 ad, {%1, %2};\n\tmov.b64 bd, {%3, %4};\n\t"
      "setp.ne.b32 p, %6, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], ad, bd, %5, p;\n}" ::"r"(d),
      "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(accumulate)
      : "memory");
}
// One K step of BX slices in a single asm block: one elect, then BX MMAs
// whose A start (lo word) and D column advance by constant strides.  Keeping
// the whole step in one block avoids re-electing and re-broadcasting the
// loop-invariant descriptor words for every MMA (the issue loop, not the
// tensor pipe, bounded the N = 128 convs).
#define VXB_UMMA_HEAD                                                        \
  "{\n\t.reg .pred e, p;\n\t.reg .b64 ad, bd;\n\t.reg .b32 al, dd;\n\t"     \
  "elect.sync _|e, 0xffffffff;\n\t"                                          \
  "setp.ne.b32 p, %6, 0;\n\t"                                                \
  "mov.b32 al, %1;\n\tmov.b32 dd, %0;\n\t"                                   \
  "mov.b64 ad, {al, %2};\n\tmov.b64 bd, {%3, %4};\n\t"
#define VXB_UMMA_NEXT "add.u32 al, al, %8;\n\tadd.u32 dd, dd, %7;\n\tmov.b64 ad, {al, %2};\n\t"
#define VXB_UMMA_1 "@e tcgen05.mma.cta_group::1.kind::f16 [dd], ad, bd, %5, p;\n\t"
#define VXB_UMMA_2 "@e tcgen05.mma.cta_group::2.kind::f16 [dd], ad, bd, %5, p;\n\t"
#define VXB_UMMA_OPS                                                                      \
  ::"r"(d), "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(accumulate), "r"(d_inc), \
      "r"(a_inc)                                                                          \
      : "memory"

// Folded K step (slice-axis taps stacked in N, see mma_group_fold) as ONE asm
// block: a single elect, every descriptor derived in-block from the step's
// base words.  Operands: %0 d_base, %1 a_lo, %2 a_hi, %3 b_lo, %4 b_hi,
// %5..%7 idesc for N = nt / 2nt / 3nt, %8 nt (TMEM columns), %9 slice_inc
// (A lo-word step between input slices), %10 blk_inc (B lo-word step between
// the stacked tap blocks).  BX >= 2.
//
// Input slice j writes accumulator slices [j - min(j,2), j - max(j-BX+1,0)],
// so MMAs of neighbouring j overlap in TMEM.  Issued in j order they form a
// read-after-write chain through the accumulator and the tensor pipe
// serialises them (~64 instead of ~46 cycles per MMA); the orders below
// (found by search, tools/fold_order.py) keep MMAs that touch the same
// slices at least two issues apart.  VXB_FM(D, A, B, ID, P): accumulator
// slice D, input slice A, B tap block B, instruction descriptor ID,
// accumulate predicate P (q = overwrite, for the tile's first step).
#define VXB_FM(D, A, B, ID, P)                                                               \
  "mad.lo.u32 dd, %8, " #D ", %0;\n\tmad.lo.u32 al, %9, " #A ", %1;\n\t"                    \
  "mad.lo.u32 bl, %10, " #B ", %3;\n\tmov.b64 ad, {al, %2};\n\tmov.b64 bd, {bl, %4};\n\t"  \
  "@e tcgen05.mma.cta_group::1.kind::f16 [dd], ad, bd, " ID ", " P ";\n\t"
#define VXB_FOLD_ASM(SEQ)                                                                   \
  "{\n\t.reg .pred e, p, q;\n\t.reg .b64 ad, bd;\n\t.reg .b32 al, dd, bl;\n\t"           \
  "elect.sync _|e, 0xffffffff;\n\tsetp.eq.u32 p, %8, %8;\n\tsetp.ne.u32 q, %8, %8;\n\t" SEQ "}"
#define VXB_FOLD_OPS                                                                        \
  ::"r"(d), "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(id1), "r"(id2), "r"(id3), "r"(nt), \
      "r"(slice_inc), "r"(blk_inc)                                                          \
      : "memory"
#define VXB_FOLD_STEADY_2 VXB_FM(1, 3, 0, "%5", "p") VXB_FM(0, 0, 2, "%5", "p") VXB_FM(0, 2, 0, "%6", "p") VXB_FM(0, 1, 1, "%6", "p")
#define VXB_FOLD_FIRST_2 VXB_FM(0, 0, 2, "%5", "q") VXB_FM(1, 1, 2, "%5", "q") VXB_FM(0, 1, 1, "%5", "p") VXB_FM(1, 3, 0, "%5", "p") VXB_FM(0, 2, 0, "%6", "p")
#define VXB_FOLD_STEADY_3 VXB_FM(0, 1, 1, "%6", "p") VXB_FM(0, 2, 0, "%7", "p") VXB_FM(1, 3, 0, "%6", "p") VXB_FM(0, 0, 2, "%5", "p") VXB_FM(2, 4, 0, "%5", "p")
#define VXB_FOLD_FIRST_3 VXB_FM(2, 2, 2, "%5", "q") VXB_FM(1, 1, 2, "%5", "q") VXB_FM(0, 0, 2, "%5", "q") VXB_FM(1, 3, 0, "%6", "p") VXB_FM(0, 1, 1, "%5", "p") VXB_FM(2, 4, 0, "%5", "p") VXB_FM(0, 2, 0, "%6", "p")
#define VXB_FOLD_STEADY_4 VXB_FM(3, 5, 0, "%5", "p") VXB_FM(0, 2, 0, "%7", "p") VXB_FM(1, 3, 0, "%7", "p") VXB_FM(0, 0, 2, "%5", "p") VXB_FM(2, 4, 0, "%6", "p") VXB_FM(0, 1, 1, "%6", "p")
#define VXB_FOLD_FIRST_4 VXB_FM(3, 3, 2, "%5", "q") VXB_FM(1, 1, 2, "%5", "q") VXB_FM(2, 2, 2, "%5", "q") VXB_FM(0, 0, 2, "%5", "q") VXB_FM(3, 5, 0, "%5", "p") VXB_FM(1, 3, 0, "%6", "p") VXB_FM(0, 1, 1, "%5", "p") VXB_FM(2, 4, 0, "%6", "p") VXB_FM(0, 2, 0, "%6", "p")
#define VXB_FOLD_STEADY_6 VXB_FM(0, 0, 2, "%5", "p") VXB_FM(1, 3, 0, "%7", "p") VXB_FM(4, 6, 0, "%6", "p") VXB_FM(0, 2, 0, "%7", "p") VXB_FM(3, 5, 0, "%7", "p") VXB_FM(0, 1, 1, "%6", "p") VXB_FM(2, 4, 0, "%7", "p") VXB_FM(5, 7, 0, "%5", "p")
#define VXB_FOLD_FIRST_6 VXB_FM(3, 3, 2, "%5", "q") VXB_FM(0, 0, 2, "%5", "q") VXB_FM(1, 1, 2, "%5", "q") VXB_FM(4, 4, 2, "%5", "q") VXB_FM(2, 2, 2, "%5", "q") VXB_FM(0, 1, 1, "%5", "p") VXB_FM(5, 5, 2, "%5", "q") VXB_FM(1, 3, 0, "%6", "p") VXB_FM(3, 5, 0, "%6", "p") VXB_FM(5, 7, 0, "%5", "p") VXB_FM(0, 2, 0, "%6", "p") VXB_FM(2, 4, 0, "%6", "p") VXB_FM(4, 6, 0, "%6", "p")
#define VXB_FOLD_STEADY_8 VXB_FM(1, 3, 0, "%7", "p") VXB_FM(4, 6, 0, "%7", "p") VXB_FM(7, 9, 0, "%5", "p") VXB_FM(0, 2, 0, "%7", "p") VXB_FM(3, 5, 0, "%7", "p") VXB_FM(6, 8, 0, "%6", "p") VXB_FM(0, 1, 1, "%6", "p") VXB_FM(2, 4, 0, "%7", "p") VXB_FM(5, 7, 0, "%7", "p") VXB_FM(0, 0, 2, "%5", "p")
#define VXB_FOLD_FIRST_8 VXB_FM(4, 4, 2, "%5", "q") VXB_FM(0, 0, 2, "%5", "q") VXB_FM(5, 5, 2, "%5", "q") VXB_FM(6, 6, 2, "%5", "q") VXB_FM(2, 2, 2, "%5", "q") VXB_FM(7, 7, 2, "%5", "q") VXB_FM(5, 7, 0, "%6", "p") VXB_FM(0, 1, 1, "%5", "p") VXB_FM(1, 1, 2, "%5", "q") VXB_FM(3, 3, 2, "%5", "q") VXB_FM(6, 8, 0, "%6", "p") VXB_FM(1, 3, 0, "%6", "p") VXB_FM(7, 9, 0, "%5", "p") VXB_FM(3, 5, 0, "%6", "p") VXB_FM(0, 2, 0, "%6", "p") VXB_FM(2, 4, 0, "%6", "p") VXB_FM(4, 6, 0, "%6", "p")

#define VXB_R1(x) x
#define VXB_R2(x) x x
#define VXB_R3(x) x x x
#define VXB_R4(x) x x x x
#define VXB_R5(x) x x x x x
#define VXB_R6(x) x x x x x x
#define VXB_R7(x) x x x x x x x
#define VXB_R8(x) x x x x x x x x
template <int BX>
__device__ __forceinline__ void umma_fold_step(uint32_t d, uint32_t a_lo, uint32_t a_hi,
                                               uint32_t b_lo, uint32_t b_hi, uint32_t id1,
                                               uint32_t id2, uint32_t id3, uint32_t nt,
                                               uint32_t slice_inc, uint32_t blk_inc) {
  static_assert(BX == 2 || BX == 3 || BX == 4 || BX == 6 || BX == 8, "folded step width");
  if (BX == 2) asm volatile(VXB_FOLD_ASM(VXB_FOLD_STEADY_2) VXB_FOLD_OPS);
  if (BX == 3) asm volatile(VXB_FOLD_ASM(VXB_FOLD_STEADY_3) VXB_FOLD_OPS);
  if (BX == 4) asm volatile(VXB_FOLD_ASM(VXB_FOLD_STEADY_4) VXB_FOLD_OPS);
  if (BX == 6) asm volatile(VXB_FOLD_ASM(VXB_FOLD_STEADY_6) VXB_FOLD_OPS);
  if (BX == 8) asm volatile(VXB_FOLD_ASM(VXB_FOLD_STEADY_8) VXB_FOLD_OPS);
}
// first K step of a tile: the d = 0 terms overwrite (accumulate off) before
// any accumulating MMA touches their slice
template <int BX>
__device__ __forceinline__ void umma_fold_first(uint32_t d, uint32_t a_lo, uint32_t a_hi,
                                                uint32_t b_lo, uint32_t b_hi, uint32_t id1,
                                                uint32_t id2, uint32_t id3, uint32_t nt,
                                                uint32_t slice_inc, uint32_t blk_inc) {
  static_assert(BX == 2 || BX == 3 || BX == 4 || BX == 6 || BX == 8, "folded step width");
  if (BX == 2) asm volatile(VXB_FOLD_ASM(VXB_FOLD_FIRST_2) VXB_FOLD_OPS);
  if (BX == 3) asm volatile(VXB_FOLD_ASM(VXB_FOLD_FIRST_3) VXB_FOLD_OPS);
  if (BX == 4) asm volatile(VXB_FOLD_ASM(VXB_FOLD_FIRST_4) VXB_FOLD_OPS);
  if (BX == 6) asm volatile(VXB_FOLD_ASM(VXB_FOLD_FIRST_6) VXB_FOLD_OPS);
  if (BX == 8) asm volatile(VXB_FOLD_ASM(VXB_FOLD_FIRST_8) VXB_FOLD_OPS);
}
#undef VXB_FM
#undef VXB_FOLD_ASM
#undef VXB_FOLD_OPS

// One K step of a streamed-fold slab (conv3d_tc.cu mma_group_stream) as ONE
// asm block: CNT MMAs, every one with its own accumulator column (%5+3k), B
// block offset (%6+3k) and instruction descriptor (%7+3k), handed over in
// issue order; the A start of input slice I is a_lo + I * slice_inc.  The
// issue orders keep neighbours >= 3 input slices apart where the count
// allows (slices i, i' share accumulator slots when |i - i'| <= 2).
// (generated: tools/gen_stream_asm.py)
template <int CNT>
__device__ __forceinline__ void umma_stream_step(uint32_t a_lo, uint32_t a_hi, uint32_t b_lo,
                                                 uint32_t b_hi, uint32_t slice_inc,
                                                 const uint32_t (&d)[8], const uint32_t (&b)[8],
                                                 const uint32_t (&id)[8]) {
  static_assert(CNT >= 1 && CNT <= 8, "slab width");
  if (CNT == 1)
    asm volatile(
      "{\n\t.reg .pred e, p;\n\t.reg .b64 ad, bd;\n\t.reg .b32 al, bl;\n\t"
      "elect.sync _|e, 0xffffffff;\n\tsetp.eq.u32 p, %0, %0;\n\t"
      "mad.lo.u32 al, %4, 0, %0;\n\tadd.u32 bl, %2, %6;\n\tmov.b64 ad, {al, %1};\n\t"
      "mov.b64 bd, {bl, %3};\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%5], ad, bd, %7, p;\n\t"
      "}"
      ::"r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(slice_inc), "r"(d[0]), "r"(b[0]), "r"(id[0])
      : "memory");
  if (CNT == 2)
    asm volatile(
      "{\n\t.reg .pred e, p;\n\t.reg .b64 ad, bd;\n\t.reg .b32 al, bl;\n\t"
      "elect.sync _|e, 0xffffffff;\n\tsetp.eq.u32 p, %0, %0;\n\t"
      "mad.lo.u32 al, %4, 0, %0;\n\tadd.u32 bl, %2, %6;\n\tmov.b64 ad, {al, %1};\n\t"
      "mov.b64 bd, {bl, %3};\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%5], ad, bd, %7, p;\n\t"
      "mad.lo.u32 al, %4, 1, %0;\n\tadd.u32 bl, %2, %9;\n\tmov.b64 ad, {al, %1};\n\t"
      "mov.b64 bd, {bl, %3};\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%8], ad, bd, %10, p;\n\t"
      "}"
      ::"r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(slice_inc), "r"(d[0]), "r"(b[0]), "r"(id[0]), "r"(d[1]), "r"(b[1]), "r"(id[1])
      : "memory");
  if (CNT == 3)
    asm volatile(
      "{\n\t.reg .pred e, p;\n\t.reg .b64 ad, bd;\n\t.reg .b32 al, bl;\n\t"
      "elect.sync _|e, 0xffffffff;\n\tsetp.eq.u32 p, %0, %0;\n\t"
      "mad.lo.u32 al, %4, 0, %0;\n\tadd.u32 bl, %2, %6;\n\tmov.b64 ad, {al, %1};\n\t"
      "mov.b64 bd, {bl, %3};\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%5], ad, bd, %7, p;\n\t"
      "mad.lo.u32 al, %4, 1, %0;\n\tadd.u32 bl, %2, %9;\n\tmov.b64 ad, {al, %1};\n\t"
      "mov.b64 bd, {bl, %3};\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%8], ad, bd, %10, p;\n\t"
      "mad.lo.u32 al, %4, 2, %0;\n\tadd.u32 bl, %2, %12;\n\tmov.b64 ad, {al, %1};\n\t"
      "mov.b64 bd, {bl, %3};\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%11], ad, bd, %13, p;\n\t"
      "}"
      ::"r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(slice_inc), "r"(d[0]), "r"(b[0]), "r"(id[0]), "r"(d[1]), "r"(b[1]), "r"(id[1]), "r"(d[2]), "r"(b[2]), "r"(id[2])
      : "memory");
  if (CNT == 4)
    asm volatile(
      "{\n\t.reg .pred e, p;\n\t.reg .b64 ad, bd;\n\t.reg .b32 al, bl;\n\t"
      "elect.sync _|e, 0xffffffff;\n\tsetp.eq.u32 p, %0, %0;\n\t"
      "mad.lo.u32 al, %4, 0, %0;\n\tadd.u32 bl, %2, %6;\n\tmov.b64 ad, {al, %1};\n\t"
      "mov.b64 bd, {bl, %3};\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%5], ad, bd, %7, p;\n\t"
      "mad.lo.u32 al, %4, 3, %0;\n\tadd.u32 bl, %2, %9;\n\tmov.b64 ad, {al, %1};\n\t"
      "mov.b64 bd, {bl, %3};\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%8], ad, bd, %10, p;\n\t"
      "mad.lo.u32 al, %4, 1, %0;\n\tadd.u32 bl, %2, %12;\n\tmov.b64 ad, {al, %1};\n\t"
      "mov.b64 bd, {bl, %3};\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%11], ad, bd, %13, p;\n\t"
      "mad.lo.u32 al, %4, 2, %0;\n\tadd.u32 bl, %2, %15;\n\tmov.b64 ad, {al, %1};\n\t"
      "mov.b64 bd, {bl, %3};\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%14], ad, bd, %16, p;\n\t"
      "}"
      ::"r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(slice_inc), "r"(d[0]), "r"(b[0]), "r"(id[0]), "r"(d[3]), "r"(b[3]), "r"(id[3]), "r"(d[1]), "r"(b[1]), "r"(id[1]), "r"(d[2]), "r"(b[2]), "r"(id[2])
      : "memory");
  if (CNT == 5)
    asm volatile(
      "{\n\t.reg .pred e, p;\n\t.reg .b64 ad, bd;\n\t.reg .b32 al, bl;\n\t"
      "elect.sync _|e, 0xffffffff;\n\tsetp.eq.u32 p, %0, %0;\n\t"
      "mad.lo.u32 al, %4, 1, %0;\n\tadd.u32 bl, %2, %6;\n\tmov.b64 ad, {al, %1};\n\t"
      "mov.b64 bd, {bl, %3};\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%5], ad, bd, %7, p;\n\t"
      "mad.lo.u32 al, %4, 4, %0;\n\tadd.u32 bl, %2, %9;\n\tmov.b64 ad, {al, %1};\n\t"
      "mov.b64 bd, {bl, %3};\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%8], ad, bd, %10, p;\n\t"
      "mad.lo.u32 al, %4, 0, %0;\n\tadd.u32 bl, %2, %12;\n\tmov.b64 ad, {al, %1};\n\t"
      "mov.b64 bd, {bl, %3};\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%11], ad, bd, %13, p;\n\t"
      "mad.lo.u32 al, %4, 3, %0;\n\tadd.u32 bl, %2, %15;\n\tmov.b64 ad, {al, %1};\n\t"
      "mov.b64 bd, {bl, %3};\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%14], ad, bd, %16, p;\n\t"
      "mad.lo.u32 al, %4, 2, %0;\n\tadd.u32 bl, %2, %18;\n\tmov.b64 ad, {al, %1};\n\t"
      "mov.b64 bd, {bl, %3};\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%17], ad, bd, %19, p;\n\t"
      "}"
      ::"r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(slice_inc), "r"(d[1]), "r"(b[1]), "r"(id[1]), "r"(d[4]), "r"(b[4]), "r"(id[4]), "r"(d[0]), "r"(b[0]), "r"(id[0]), "r"(d[3]), "r"(b[3]), "r"(id[3]), "r"(d[2]), "r"(b[2]), "r"(id[2])
      : "memory");
  if (CNT == 6)
    asm volatile(
      "{\n\t.reg .pred e, p;\n\t.reg .b64 ad, bd;\n\t.reg .b32 al, bl;\n\t"
      "elect.sync _|e, 0xffffffff;\n\tsetp.eq.u32 p, %0, %0;\n\t"
      "mad.lo.u32 al, %4, 2, %0;\n\tadd.u32 bl, %2, %6;\n\tmov.b64 ad, {al, %1};\n\t"
      "mov.b64 bd, {bl, %3};\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%5], ad, bd, %7, p;\n\t"
      "mad.lo.u32 al, %4, 5, %0;\n\tadd.u32 bl, %2, %9;\n\tmov.b64 ad, {al, %1};\n\t"
      "mov.b64 bd, {bl, %3};\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%8], ad, bd, %10, p;\n\t"
      "mad.lo.u32 al, %4, 1, %0;\n\tadd.u32 bl, %2, %12;\n\tmov.b64 ad, {al, %1};\n\t"
      "mov.b64 bd, {bl, %3};\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%11], ad, bd, %13, p;\n\t"
      "mad.lo.u32 al, %4, 4, %0;\n\tadd.u32 bl, %2, %15;\n\tmov.b64 ad, {al, %1};\n\t"
      "mov.b64 bd, {bl, %3};\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%14], ad, bd, %16, p;\n\t"
      "mad.lo.u32 al, %4, 0, %0;\n\tadd.u32 bl, %2, %18;\n\tmov.b64 ad, {al, %1};\n\t"
      "mov.b64 bd, {bl, %3};\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%17], ad, bd, %19, p;\n\t"
      "mad.lo.u32 al, %4, 3, %0;\n\tadd.u32 bl, %2, %21;\n\tmov.b64 ad, {al, %1};\n\t"
      "mov.b64 bd, {bl, %3};\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%20], ad, bd, %22, p;\n\t"
      "}"
      ::"r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(slice_inc), "r"(d[2]), "r"(b[2]), "r"(id[2]), "r"(d[5]), "r"(b[5]), "r"(id[5]), "r"(d[1]), "r"(b[1]), "r"(id[1]), "r"(d[4]), "r"(b[4]), "r"(id[4]), "r"(d[0]), "r"(b[0]), "r"(id[0]), "r"(d[3]), "r"(b[3]), "r"(id[3])
      : "memory");
  if (CNT == 7)
    asm volatile(
      "{\n\t.reg .pred e, p;\n\t.reg .b64 ad, bd;\n\t.reg .b32 al, bl;\n\t"
      "elect.sync _|e, 0xffffffff;\n\tsetp.eq.u32 p, %0, %0;\n\t"
      "mad.lo.u32 al, %4, 3, %0;\n\tadd.u32 bl, %2, %6;\n\tmov.b64 ad, {al, %1};\n\t"
      "mov.b64 bd, {bl, %3};\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%5], ad, bd, %7, p;\n\t"
      "mad.lo.u32 al, %4, 6, %0;\n\tadd.u32 bl, %2, %9;\n\tmov.b64 ad, {al, %1};\n\t"
      "mov.b64 bd, {bl, %3};\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%8], ad, bd, %10, p;\n\t"
      "mad.lo.u32 al, %4, 2, %0;\n\tadd.u32 bl, %2, %12;\n\tmov.b64 ad, {al, %1};\n\t"
      "mov.b64 bd, {bl, %3};\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%11], ad, bd, %13, p;\n\t"
      "mad.lo.u32 al, %4, 5, %0;\n\tadd.u32 bl, %2, %15;\n\tmov.b64 ad, {al, %1};\n\t"
      "mov.b64 bd, {bl, %3};\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%14], ad, bd, %16, p;\n\t"
      "mad.lo.u32 al, %4, 1, %0;\n\tadd.u32 bl, %2, %18;\n\tmov.b64 ad, {al, %1};\n\t"
      "mov.b64 bd, {bl, %3};\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%17], ad, bd, %19, p;\n\t"
      "mad.lo.u32 al, %4, 4, %0;\n\tadd.u32 bl, %2, %21;\n\tmov.b64 ad, {al, %1};\n\t"
      "mov.b64 bd, {bl, %3};\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%20], ad, bd, %22, p;\n\t"
      "mad.lo.u32 al, %4, 0, %0;\n\tadd.u32 bl, %2, %24;\n\tmov.b64 ad, {al, %1};\n\t"
      "mov.b64 bd, {bl, %3};\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%23], ad, bd, %25, p;\n\t"
      "}"
      ::"r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(slice_inc), "r"(d[3]), "r"(b[3]), "r"(id[3]), "r"(d[6]), "r"(b[6]), "r"(id[6]), "r"(d[2]), "r"(b[2]), "r"(id[2]), "r"(d[5]), "r"(b[5]), "r"(id[5]), "r"(d[1]), "r"(b[1]), "r"(id[1]), "r"(d[4]), "r"(b[4]), "r"(id[4]), "r"(d[0]), "r"(b[0]), "r"(id[0])
      : "memory");
  if (CNT == 8)
    asm volatile(
      "{\n\t.reg .pred e, p;\n\t.reg .b64 ad, bd;\n\t.reg .b32 al, bl;\n\t"
      "elect.sync _|e, 0xffffffff;\n\tsetp.eq.u32 p, %0, %0;\n\t"
      "mad.lo.u32 al, %4, 3, %0;\n\tadd.u32 bl, %2, %6;\n\tmov.b64 ad, {al, %1};\n\t"
      "mov.b64 bd, {bl, %3};\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%5], ad, bd, %7, p;\n\t"
      "mad.lo.u32 al, %4, 6, %0;\n\tadd.u32 bl, %2, %9;\n\tmov.b64 ad, {al, %1};\n\t"
      "mov.b64 bd, {bl, %3};\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%8], ad, bd, %10, p;\n\t"
      "mad.lo.u32 al, %4, 2, %0;\n\tadd.u32 bl, %2, %12;\n\tmov.b64 ad, {al, %1};\n\t"
      "mov.b64 bd, {bl, %3};\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%11], ad, bd, %13, p;\n\t"
      "mad.lo.u32 al, %4, 5, %0;\n\tadd.u32 bl, %2, %15;\n\tmov.b64 ad, {al, %1};\n\t"
      "mov.b64 bd, {bl, %3};\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%14], ad, bd, %16, p;\n\t"
      "mad.lo.u32 al, %4, 1, %0;\n\tadd.u32 bl, %2, %18;\n\tmov.b64 ad, {al, %1};\n\t"
      "mov.b64 bd, {bl, %3};\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%17], ad, bd, %19, p;\n\t"
      "mad.lo.u32 al, %4, 4, %0;\n\tadd.u32 bl, %2, %21;\n\tmov.b64 ad, {al, %1};\n\t"
      "mov.b64 bd, {bl, %3};\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%20], ad, bd, %22, p;\n\t"
      "mad.lo.u32 al, %4, 0, %0;\n\tadd.u32 bl, %2, %24;\n\tmov.b64 ad, {al, %1};\n\t"
      "mov.b64 bd, {bl, %3};\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%23], ad, bd, %25, p;\n\t"
      "mad.lo.u32 al, %4, 7, %0;\n\tadd.u32 bl, %2, %27;\n\tmov.b64 ad, {al, %1};\n\t"
      "mov.b64 bd, {bl, %3};\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%26], ad, bd, %28, p;\n\t"
      "}"
      ::"r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(slice_inc), "r"(d[3]), "r"(b[3]), "r"(id[3]), "r"(d[6]), "r"(b[6]), "r"(id[6]), "r"(d[2]), "r"(b[2]), "r"(id[2]), "r"(d[5]), "r"(b[5]), "r"(id[5]), "r"(d[1]), "r"(b[1]), "r"(id[1]), "r"(d[4]), "r"(b[4]), "r"(id[4]), "r"(d[0]), "r"(b[0]), "r"(id[0]), "r"(d[7]), "r"(b[7]), "r"(id[7])
      : "memory");
}

// CNT cta_group::2 MMAs in one asm block: D and the A lo word advance by
// d_inc / a_inc, B and the instruction descriptor are shared (the folded
// CTA-pair walk, mma_group_fold_pair).
#define VXB_PRUN_HEAD                                                        \
  "{\n\t.reg .pred e, p;\n\t.reg .b64 ad, bd;\n\t.reg .b32 al, dd;\n\t"     \
  "elect.sync _|e, 0xffffffff;\n\t"                                          \
  "setp.ne.b32 p, %6, 0;\n\t"                                                \
  "mov.b32 al, %1;\n\tmov.b32 dd, %0;\n\t"                                   \
  "mov.b64 bd, {%3, %4};\n\t"
#define VXB_PRUN_MMA                                                                        \
  "mov.b64 ad, {al, %2};\n\t@e tcgen05.mma.cta_group::2.kind::f16 [dd], ad, bd, %5, p;\n\t" \
  "add.u32 al, al, %8;\n\tadd.u32 dd, dd, %7;\n\t"
#define VXB_PRUN_OPS                                                                      \
  ::"r"(d), "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(accumulate), "r"(d_inc), \
      "r"(a_inc)                                                                          \
      : "memory"
template <int CNT>
__device__ __forceinline__ void umma_pair_run(uint32_t d, uint32_t a_lo, uint32_t a_hi,
                                              uint32_t b_lo, uint32_t b_hi, uint32_t idesc,
                                              uint32_t accumulate, uint32_t d_inc,
                                              uint32_t a_inc) {
  static_assert(CNT >= 1 && CNT <= 10, "run length");
  if (CNT == 1) asm volatile(VXB_PRUN_HEAD VXB_R1(VXB_PRUN_MMA) "}" VXB_PRUN_OPS);
  if (CNT == 2) asm volatile(VXB_PRUN_HEAD VXB_R2(VXB_PRUN_MMA) "}" VXB_PRUN_OPS);
  if (CNT == 3) asm volatile(VXB_PRUN_HEAD VXB_R3(VXB_PRUN_MMA) "}" VXB_PRUN_OPS);
  if (CNT == 4) asm volatile(VXB_PRUN_HEAD VXB_R4(VXB_PRUN_MMA) "}" VXB_PRUN_OPS);
  if (CNT == 5) asm volatile(VXB_PRUN_HEAD VXB_R5(VXB_PRUN_MMA) "}" VXB_PRUN_OPS);
  if (CNT == 6) asm volatile(VXB_PRUN_HEAD VXB_R6(VXB_PRUN_MMA) "}" VXB_PRUN_OPS);
  if (CNT == 7) asm volatile(VXB_PRUN_HEAD VXB_R7(VXB_PRUN_MMA) "}" VXB_PRUN_OPS);
  if (CNT == 8) asm volatile(VXB_PRUN_HEAD VXB_R8(VXB_PRUN_MMA) "}" VXB_PRUN_OPS);
  if (CNT == 9) asm volatile(VXB_PRUN_HEAD VXB_R8(VXB_PRUN_MMA) VXB_PRUN_MMA "}" VXB_PRUN_OPS);
  if (CNT == 10)
    asm volatile(VXB_PRUN_HEAD VXB_R8(VXB_PRUN_MMA) VXB_R2(VXB_PRUN_MMA) "}" VXB_PRUN_OPS);
}
#undef VXB_PRUN_HEAD
#undef VXB_PRUN_MMA
#undef VXB_PRUN_OPS

template <int BX, bool PAIR>
__device__ __forceinline__ void umma_step_elect(uint32_t d, uint32_t a_lo, uint32_t a_hi,
                                                uint32_t b_lo, uint32_t b_hi, uint32_t idesc,
                                                uint32_t accumulate, uint32_t d_inc,
                                                uint32_t a_inc) {
  static_assert(BX == 1 || BX == 2 || BX == 3 || BX == 4 || BX == 6 || BX == 8, "step width");
  if (PAIR) {
    if (BX == 1) asm volatile(VXB_UMMA_HEAD VXB_UMMA_2 "}" VXB_UMMA_OPS);
    if (BX == 2) asm volatile(VXB_UMMA_HEAD VXB_UMMA_2 VXB_UMMA_NEXT VXB_UMMA_2 "}" VXB_UMMA_OPS);
    if (BX == 3)
      asm volatile(VXB_UMMA_HEAD VXB_UMMA_2 VXB_UMMA_NEXT VXB_UMMA_2 VXB_UMMA_NEXT VXB_UMMA_2
                   "}" VXB_UMMA_OPS);
    if (BX == 6)
      asm volatile(VXB_UMMA_HEAD VXB_UMMA_2 VXB_UMMA_NEXT VXB_UMMA_2 VXB_UMMA_NEXT VXB_UMMA_2
                       VXB_UMMA_NEXT VXB_UMMA_2 VXB_UMMA_NEXT VXB_UMMA_2 VXB_UMMA_NEXT VXB_UMMA_2
                   "}" VXB_UMMA_OPS);
    if (BX == 4)
      asm volatile(VXB_UMMA_HEAD VXB_UMMA_2 VXB_UMMA_NEXT VXB_UMMA_2 VXB_UMMA_NEXT VXB_UMMA_2
                       VXB_UMMA_NEXT VXB_UMMA_2 "}" VXB_UMMA_OPS);
    if (BX == 8)
      asm volatile(VXB_UMMA_HEAD VXB_UMMA_2 VXB_UMMA_NEXT VXB_UMMA_2 VXB_UMMA_NEXT VXB_UMMA_2
                       VXB_UMMA_NEXT VXB_UMMA_2 VXB_UMMA_NEXT VXB_UMMA_2 VXB_UMMA_NEXT VXB_UMMA_2
                           VXB_UMMA_NEXT VXB_UMMA_2 VXB_UMMA_NEXT VXB_UMMA_2 "}" VXB_UMMA_OPS);
  } else {
    if (BX == 1) asm volatile(VXB_UMMA_HEAD VXB_UMMA_1 "}" VXB_UMMA_OPS);
    if (BX == 2) asm volatile(VXB_UMMA_HEAD VXB_UMMA_1 VXB_UMMA_NEXT VXB_UMMA_1 "}" VXB_UMMA_OPS);
    if (BX == 3)
      asm volatile(VXB_UMMA_HEAD VXB_UMMA_1 VXB_UMMA_NEXT VXB_UMMA_1 VXB_UMMA_NEXT VXB_UMMA_1
                   "}" VXB_UMMA_OPS);
    if (BX == 6)
      asm volatile(VXB_UMMA_HEAD VXB_UMMA_1 VXB_UMMA_NEXT VXB_UMMA_1 VXB_UMMA_NEXT VXB_UMMA_1
                       VXB_UMMA_NEXT VXB_UMMA_1 VXB_UMMA_NEXT VXB_UMMA_1 VXB_UMMA_NEXT VXB_UMMA_1
                   "}" VXB_UMMA_OPS);
    if (BX == 4)
      asm volatile(VXB_UMMA_HEAD VXB_UMMA_1 VXB_UMMA_NEXT VXB_UMMA_1 VXB_UMMA_NEXT VXB_UMMA_1
                       VXB_UMMA_NEXT VXB_UMMA_1 "}" VXB_UMMA_OPS);
    if (BX == 8)
      asm volatile(VXB_UMMA_HEAD VXB_UMMA_1 VXB_UMMA_NEXT VXB_UMMA_1 VXB_UMMA_NEXT VXB_UMMA_1
                       VXB_UMMA_NEXT VXB_UMMA_1 VXB_UMMA_NEXT VXB_UMMA_1 VXB_UMMA_NEXT VXB_UMMA_1
                           VXB_UMMA_NEXT VXB_UMMA_1 VXB_UMMA_NEXT VXB_UMMA_1 "}" VXB_UMMA_OPS);
  }
}
#undef VXB_UMMA_HEAD
#undef VXB_UMMA_NEXT
#undef VXB_UMMA_1
#undef VXB_UMMA_2
#undef VXB_UMMA_OPS

__device__ __forceinline__ void umma_commit_pair(uint64_t *bar, uint16_t cta_mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"(cta_mask)
      : "memory");
}
__device__ __forceinline__ void umma_commit_mc(uint64_t *bar, uint16_t cta_mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"(cta_mask)
      : "memory");
}

// UMMA shared-memory matrix descriptor, SWIZZLE_NONE (K-major "interleaved"
// canonical layout: 8-row x 16-byte core matrices, rows 16 B apart).
//   lbo: byte distance between the two K-adjacent core matrices
//   sbo: byte distance between M/N-adjacent groups of 8 rows
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // descriptor version (sm_100)
  // base offset 0, lbo mode 0, layout type 0 = SWIZZLE_NONE
  return d;
}

// instruction descriptor: kind::f16, A=B=bf16, D=f32, both K-major
__host__ __device__ constexpr uint32_t idesc_bf16(int m, int n) {
  return (1u << 4)                                  // D format f32
         | (1u << 7)                                // A bf16
         | (1u << 10)                               // B bf16
         | (static_cast<uint32_t>(n >> 3) << 17)    // N / 8
         | (static_cast<uint32_t>(m >> 4) << 24);   // M / 16
}

}  // namespace vxb

// 32-byte global accesses (sm_100: LDG/STG .256); the address must be
// 32-byte aligned
namespace vxb {
__device__ __forceinline__ void ld_nc_v8(const void *p, uint4 &a, uint4 &b) {
  asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z),
                 "=r"(b.w)
               : "l"(p));
}
__device__ __forceinline__ void st_v8(void *p, const uint32_t (&w)[8]) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(w[0]), "r"(w[1]),
               "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
               : "memory");
}
}  // namespace vxb

// packed fp32 pairs (sm_100: FADD2 / FMUL2 / FFMA2, two lanes per
// instruction; the register pairs are free, ptxas keeps them adjacent)
namespace vxb {
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  float2 r;
  asm("{.reg .b64 ra, rb, rr;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "add.rn.f32x2 rr, ra, rb;\n\tmov.b64 {%0, %1}, rr;}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
  float2 r;
  asm("{.reg .b64 ra, rb, rr;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "mul.rn.f32x2 rr, ra, rb;\n\tmov.b64 {%0, %1}, rr;}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 r;
  asm("{.reg .b64 ra, rb, rc, rr;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "mov.b64 rc, {%6, %7};\n\tfma.rn.f32x2 rr, ra, rb, rc;\n\tmov.b64 {%0, %1}, rr;}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return r;
}
}  // namespace vxb

namespace vxb {
// named barrier among `count` threads (warps of one role), id >= 1
__device__ __forceinline__ void named_bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
}  // namespace vxb
