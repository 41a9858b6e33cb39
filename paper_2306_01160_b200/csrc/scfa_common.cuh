// scfa_common.cuh — sm_100a primitives used by every SCFA kernel.
//
// Thin inline-PTX wrappers for the Blackwell async machinery: mbarriers,
// TMA (cp.async.bulk[.tensor]), tcgen05 (TMEM alloc/ld/st, UMMA issue and
// commit) and the shared-memory / instruction descriptors that tie them
// together.  Nothing here is attention-specific.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cfloat>

#ifndef SCFA_DEVICE
#define SCFA_DEVICE __device__ __forceinline__
#endif

namespace scfa {

// ---------------------------------------------------------------- basics

SCFA_DEVICE uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

SCFA_DEVICE uint32_t lane_id() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(r));
  return r;
}

SCFA_DEVICE bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .b32 %%rx;\n\t.reg .pred %%px;\n\t"
      "elect.sync %%rx|%%px, 0xffffffff;\n\t"
      "selp.b32 %0, 1, 0, %%px;\n\t}"
      : "+r"(pred));
  return pred != 0;
}

// ---------------------------------------------------------------- mbarrier

// An mbarrier by its 32-bit shared-memory address (one register, immediate offsets).
struct MBar {
  uint32_t a;
  SCFA_DEVICE MBar() : a(0) {}
  SCFA_DEVICE explicit MBar(uint32_t addr) : a(addr) {}
  SCFA_DEVICE MBar(uint64_t* p) : a(static_cast<uint32_t>(__cvta_generic_to_shared(p))) {}
  SCFA_DEVICE MBar operator+(int i) const { return MBar(a + 8u * static_cast<uint32_t>(i)); }
};

SCFA_DEVICE void mbar_init(MBar bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar.a), "r"(count));
}

SCFA_DEVICE void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

SCFA_DEVICE void mbar_arrive(MBar bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar.a) : "memory");
}

// Arrive without release semantics: for consumers whose data is already in registers
// (tcgen05.ld + wait::ld, ld.shared), so the arrive need not wait for this thread's
// outstanding global stores / reductions to be performed.
SCFA_DEVICE void mbar_arrive_relaxed(MBar bar) {
  asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(bar.a) : "memory");
}

SCFA_DEVICE void mbar_arrive_expect_tx(MBar bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar.a),
               "r"(bytes)
               : "memory");
}

SCFA_DEVICE void mbar_wait(MBar bar, uint32_t parity) {
  uint32_t addr = bar.a;
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(addr),
      "r"(parity), "r"(0x989680)
      : "memory");
}

// Non-blocking probe: has the phase with this parity completed?
SCFA_DEVICE bool mbar_test(MBar bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(bar.a), "r"(parity)
      : "memory");
  return ok != 0;
}

// Wait with back-off, for the warps that mostly wait (producer, MMA issuer, epilogue):
// a failed probe sleeps instead of re-polling, so their spinning does not take issue
// slots from the softmax warps on the same SM sub-partition.
SCFA_DEVICE void mbar_wait_lazy(MBar bar, uint32_t parity, uint32_t sleep_ns = 64) {
  uint32_t ok = 0;
  while (true) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, P1;\n\t}"
        : "=r"(ok)
        : "r"(bar.a), "r"(parity)
        : "memory");
    if (ok) break;
    __nanosleep(sleep_ns);
  }
}

// ---------------------------------------------------------------- proxies

SCFA_DEVICE void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---------------------------------------------------------------- TMA

SCFA_DEVICE void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// 3-D tiled TMA load (coordinates innermost first) completing on `bar`.
SCFA_DEVICE void tma_load_3d(void* smem_dst, const CUtensorMap* map, MBar bar, int c0, int c1,
                             int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar.a), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// TMA row gather: four rows (r0..r3, outer coordinate) of one box_inner-wide column
// window starting at c0 land as four consecutive 128-byte rows at smem_dst (512 B).
// The 128-byte swizzle is a function of the shared-memory address, so 4-row groups
// at 512-byte offsets of a 1024-aligned tile reproduce the tiled SWIZZLE_128B image
// (measured: scripts/gather4_test.cu).
SCFA_DEVICE void tma_gather4(void* smem_dst, const CUtensorMap* map, MBar bar, int c0, int r0, int r1, int r2,
                             int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(bar.a)
      : "memory");
}

// TMA row scatter (the store twin of tma_gather4), tracked by the issuing thread's bulk group.
SCFA_DEVICE void tma_scatter4(const CUtensorMap* map, const void* smem_src, int c0, int r0, int r1, int r2, int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.tile::scatter4.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(smem_src))
      : "memory");
}

// 2-D tiled TMA store of one box (rows r0.., columns c0..).
SCFA_DEVICE void tma_store_2d(const CUtensorMap* map, const void* smem_src, int c0, int r0) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(r0), "r"(smem_u32(smem_src))
               : "memory");
}

SCFA_DEVICE void tma_store_3d(const CUtensorMap* map, const void* smem_src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(smem_src))
               : "memory");
}

SCFA_DEVICE void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// Wait until every committed bulk store of this thread has finished READING shared memory.
SCFA_DEVICE void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
SCFA_DEVICE void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// Plain bulk copy global -> shared (16-byte aligned, size multiple of 16).
SCFA_DEVICE void bulk_load(void* smem_dst, const void* gsrc, uint32_t bytes, MBar bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(gsrc)), "r"(bytes), "r"(bar.a)
      : "memory");
}

// ---------------------------------------------------------------- tcgen05 / TMEM

template <uint32_t kCols>
SCFA_DEVICE void tmem_alloc(uint32_t* smem_slot) {
  static_assert(kCols >= 32 && kCols <= 512 && (kCols & (kCols - 1)) == 0, "TMEM cols pow2");
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(smem_slot)),
               "n"(kCols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::);
}

template <uint32_t kCols>
SCFA_DEVICE void tmem_dealloc(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols));
}

SCFA_DEVICE void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
SCFA_DEVICE void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// Make `bar` track completion of every tcgen05.mma issued so far by this thread.
SCFA_DEVICE void umma_commit(MBar bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          bar.a)
      : "memory");
}

// D[tmem] (+)= A[smem] * B[smem]^T   (kind::f16, bf16 in, fp32 accumulate)
SCFA_DEVICE void umma_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

// D[tmem] (+)= A[tmem] * B[smem]^T
SCFA_DEVICE void umma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

// Instruction descriptor: bf16 x bf16 -> fp32, M x N, A/B major given.
__host__ __device__ constexpr uint32_t make_idesc_bf16(uint32_t M, uint32_t N, bool a_mn_major,
                                                       bool b_mn_major) {
  return (1u << 4)                            // D format: f32
         | (1u << 7)                          // A format: bf16
         | (1u << 10)                         // B format: bf16
         | ((a_mn_major ? 1u : 0u) << 15)     // A major
         | ((b_mn_major ? 1u : 0u) << 16)     // B major
         | ((N >> 3) << 17)                   // N / 8
         | ((M >> 4) << 24);                  // M / 16
}

// Shared-memory matrix descriptor (sm_100 "version 1"), SWIZZLE_128B.
//   K-major : rows of 128 B, 8-row core groups SBO bytes apart (LBO unused = 16 B).
//   MN-major: 64-element (128 B) MN atoms LBO bytes apart, 8-row K groups SBO bytes apart.
SCFA_DEVICE uint64_t make_sdesc_sw128(uint32_t smem_addr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1u) << 46;  // version (sm_100)
  d |= static_cast<uint64_t>(2u) << 61;  // SWIZZLE_128B
  return d;
}

// ---- TMEM <-> registers (32 lanes x 32-bit, one row per thread) ----

#define SCFA_R8(a, i) "=r"(a[i]), "=r"(a[i + 1]), "=r"(a[i + 2]), "=r"(a[i + 3]), \
                      "=r"(a[i + 4]), "=r"(a[i + 5]), "=r"(a[i + 6]), "=r"(a[i + 7])
#define SCFA_W8(a, i) "r"(a[i]), "r"(a[i + 1]), "r"(a[i + 2]), "r"(a[i + 3]), \
                      "r"(a[i + 4]), "r"(a[i + 5]), "r"(a[i + 6]), "r"(a[i + 7])

SCFA_DEVICE void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : SCFA_R8(r, 0), SCFA_R8(r, 8), SCFA_R8(r, 16), SCFA_R8(r, 24)
      : "r"(taddr));
}

SCFA_DEVICE void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : SCFA_R8(r, 0), SCFA_R8(r, 8)
      : "r"(taddr));
}

SCFA_DEVICE void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      SCFA_W8(r, 0), SCFA_W8(r, 8), SCFA_W8(r, 16), SCFA_W8(r, 24)
      : "memory");
}

SCFA_DEVICE void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      SCFA_W8(r, 0), SCFA_W8(r, 8)
      : "memory");
}

// smem -> TMEM copy of a 128-row x 256-bit block (tcgen05.cp; source described by a
// matrix descriptor, as an MMA operand), asynchronous, ordered with the issuing
// thread's tcgen05.mma
SCFA_DEVICE void tmem_cp_128x256b(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}

SCFA_DEVICE void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
SCFA_DEVICE void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// ---------------------------------------------------------------- math

SCFA_DEVICE float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Approximate reciprocal (MUFU.RCP, no IEEE slow-path subroutine: kernels that use
// setmaxnreg must not contain calls).
SCFA_DEVICE float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

SCFA_DEVICE uint32_t pack_bf16(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

// Packed fp32x2 arithmetic (sm_100: FFMA2 / FADD2 / FMUL2) and the 3-input max/min
// (FMNMX3): half the issue slots of the scalar forms in the softmax loops.
SCFA_DEVICE void fma2(float& d0, float& d1, float a0, float a1, float b0, float b1, float c0, float c1) {
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1), "f"(c0), "f"(c1));
}

SCFA_DEVICE void add2(float& d0, float& d1, float a0, float a1, float b0, float b1) {
  asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}

SCFA_DEVICE void mul2(float& d0, float& d1, float a0, float a1, float b0, float b1) {
  asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "mul.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}

SCFA_DEVICE float max3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

SCFA_DEVICE float min3(float a, float b, float c) {
  float d;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// 2^x for a pair on the FMA / ALU pipes instead of MUFU (the softmax loops are MUFU
// bound at D = 64): x clamped to [-126, 127]; floor by the 1.5*2^23 round-down trick,
// degree-3 minimax polynomial for 2^f on [0, 1) (max rel. error 8.8e-5, far below the
// bf16 rounding of P), exponent added in the integer domain.
SCFA_DEVICE void ex2_poly2(float& y0, float& y1, float x0, float x1) {
  x0 = fminf(fmaxf(x0, -126.f), 127.f);
  x1 = fminf(fmaxf(x1, -126.f), 127.f);
  float t0, t1, j0, j1, f0, f1, p0, p1;
  asm("{\n\t.reg .b64 rx, rm, rt;\n\t"
      "mov.b64 rx, {%2, %3};\n\tmov.b64 rm, {%4, %4};\n\t"
      "add.rm.f32x2 rt, rx, rm;\n\tmov.b64 {%0, %1}, rt;\n\t}"
      : "=f"(t0), "=f"(t1)
      : "f"(x0), "f"(x1), "f"(12582912.0f));
  add2(j0, j1, t0, t1, -12582912.0f, -12582912.0f);  // floor(x), exact
  add2(f0, f1, x0, x1, -j0, -j1);                      // fraction in [0, 1)
  fma2(p0, p1, f0, f1, 0.0771190897f, 0.0771190897f, 0.2275643945f, 0.2275643945f);
  fma2(p0, p1, p0, p1, f0, f1, 0.6951461434f, 0.6951461434f);
  fma2(p0, p1, p0, p1, f0, f1, 1.0f, 1.0f);
  y0 = __uint_as_float(__float_as_uint(p0) + (__float_as_uint(t0) << 23));
  y1 = __uint_as_float(__float_as_uint(p1) + (__float_as_uint(t1) << 23));
}

// Named barrier for warps that reach it at different instructions (e.g. the two row
// warpgroups of the D = 128 forward): the non-.aligned form (bar.sync is barrier.sync.aligned,
// which requires every participating thread to execute the same instruction).
SCFA_DEVICE void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("barrier.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

}  // namespace scfa
