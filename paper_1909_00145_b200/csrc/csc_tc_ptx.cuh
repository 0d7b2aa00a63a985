// csc_tc_ptx.cuh -- sm_100a PTX wrappers shared by the tensor-core kernels (csc_tc.cu,
// csc_wgrad_tc.cu): mbarriers, tcgen05 (alloc / mma / commit / ld / st / fences), UMMA shared
// memory descriptors, TMA bulk-tensor loads.  Internal; not part of the ABI.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace csc {
namespace tcx {

constexpr unsigned kFullMask = 0xffffffffu;

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// ---------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra WAIT_%=;\n}\n" ::"r"(
          su32(bar)),
      "r"(parity)
      : "memory");
}
// Wait with a suspend-time hint: the warp sleeps in the barrier unit instead of re-issuing
// try_wait, leaving issue slots to the warps that do the work.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n@!P1 bra WAIT_%=;\n}\n" ::"r"(
          su32(bar)),
      "r"(parity), "r"(20000)
      : "memory");
}
// Wait with an explicit back-off: a failed try_wait sleeps ns nanoseconds before polling again, so
// warps that are not on the critical path stop taking issue slots from the ones that are.
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n"
      : "=r"(ok)
      : "r"(su32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, uint32_t parity, uint32_t ns = 128) {
  while (!mbar_try(bar, parity)) __nanosleep(ns);
}
__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}
// Non-blocking arrival on a named barrier (a producer releasing warps that bar.sync on it).
__device__ __forceinline__ void named_arrive(int id, int nthreads) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}

// ---------------------------------------------------------------- tcgen05
__device__ __forceinline__ void tc_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(dst_smem)), "r"(ncols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t base, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(base), "r"(ncols));
}

// UMMA shared-memory descriptor (sm_100): start, LBO, SBO in 16-byte units, version 1, layout type.
enum : uint32_t { kLayoutNone = 0, kLayout128B32 = 1, kLayout128B = 2, kLayout64B = 4, kLayout32B = 6 };
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(layout) << 61;
  return d;
}
// Instruction descriptor, kind::tf32, fp32 accumulate; a_mn/b_mn: 1 = MN-major operand.
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(a_mn) << 15) |
         (static_cast<uint32_t>(b_mn) << 16) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}

// Warp-collective: every lane calls, one elected lane issues.
__device__ __forceinline__ void mma_commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(su32(bar))
      : "memory");
}

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(taddr), "r"(v[0]),
               "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}
__device__ __forceinline__ void tmem_ld4_nowait(uint32_t taddr, float (&f)[4]) {
  uint32_t v[4];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
               : "r"(taddr)
               : "memory");
#pragma unroll
  for (int i = 0; i < 4; ++i) f[i] = __uint_as_float(v[i]);
}
__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, float (&f)[16]) {
  uint32_t v[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) f[i] = __uint_as_float(v[i]);
}
__device__ __forceinline__ void tmem_ld8_nowait(uint32_t taddr, float (&f)[8]) {
  uint32_t v[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr)
               : "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) f[i] = __uint_as_float(v[i]);
}
// the S accumulator columns of one tap row (exact widths: no TMEM read bandwidth spent on padding)
__device__ __forceinline__ void tmem_ld_x1(uint32_t taddr, float& f) {
  uint32_t v;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(v) : "r"(taddr) : "memory");
  f = __uint_as_float(v);
}
__device__ __forceinline__ void tmem_ld_x2(uint32_t taddr, float& f0, float& f1) {
  uint32_t v0, v1;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];\n" : "=r"(v0), "=r"(v1) : "r"(taddr) : "memory");
  f0 = __uint_as_float(v0);
  f1 = __uint_as_float(v1);
}
template <int S>
__device__ __forceinline__ void tmem_ld_row(uint32_t taddr, float (&y)[S]) {
  int c = 0;
  if constexpr (S >= 8) {
    float t[8];
    tmem_ld8_nowait(taddr, t);
#pragma unroll
    for (int i = 0; i < 8; ++i) y[i] = t[i];
    c = 8;
  }
  if constexpr ((S & 4) != 0) {
    float t[4];
    tmem_ld4_nowait(taddr + c, t);
#pragma unroll
    for (int i = 0; i < 4; ++i) y[(S >= 8 ? 8 : 0) + i] = t[i];
  }
  constexpr int c2 = (S >= 8 ? 8 : 0) + ((S & 4) != 0 ? 4 : 0);
  if constexpr ((S & 2) != 0) tmem_ld_x2(taddr + c2, y[c2], y[c2 + 1]);
  constexpr int c1 = c2 + ((S & 2) != 0 ? 2 : 0);
  if constexpr ((S & 1) != 0) tmem_ld_x1(taddr + c1, y[c1]);
  (void)c;
}

__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

// ---------------------------------------------------------------- TMA
__device__ __forceinline__ void tma_prefetch_desc(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t smem_dst, const void* tmap, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::
          "r"(smem_dst),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(su32(bar))
      : "memory");
}

// The same with an L2 eviction-priority policy (createpolicy): streamed operands read once per kernel are
// loaded evict_first so that the small reused data (residual, partials, masks) stays in L2.
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tma_load_2d_hint(uint32_t smem_dst, const void* tmap, int c0, int c1, uint64_t* bar,
                                                 uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
      "%3}], [%4], %5;\n" ::"r"(smem_dst),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(su32(bar)), "l"(policy)
      : "memory");
}

// ---------------------------------------------------------------- misc
__device__ __forceinline__ void cp_async4(uint32_t smem_dst, const float* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(smem_dst), "l"(src), "r"(valid ? 4 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_async_shared() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// 3xTF32 low part under tensor-core truncation: the MMA reads an fp32 operand as tf32 by
// dropping the low 13 mantissa bits, so x itself serves as the high part and
// lo = x - trunc_tf32(x) is exact in fp32 (it is truncated once more when read as tf32:
// <= 2^-21 relative).
__device__ __forceinline__ float tf32_lo_trunc(float x) {
  return x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}

// 3xTF32 split with round-to-nearest on both parts (ties away from zero), two integer ops each:
// hi = rn_tf32(x), lo = rn_tf32(x - hi) (x - hi is exact in fp32).  Unbiased, unlike the
// truncating split above: representation error <= 2^-22 |x| with random sign.
__device__ __forceinline__ float rn_tf32(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}
__device__ __forceinline__ void tf32_split_rn(float x, float& hi, float& lo) {
  hi = rn_tf32(x);
  lo = rn_tf32(x - hi);
}
// hi = rn_tf32(x), lo = x - hi left for the tensor core to truncate: |lo| <= 2^-11 |x|, and the
// truncation of lo to tf32 costs < 2^-21 |x| with the sign of lo (random w.r.t. x), two integer
// ops and one add instead of five
__device__ __forceinline__ void tf32_split_rn_hi(float x, float& hi, float& lo) {
  hi = rn_tf32(x);
  lo = x - hi;
}

}  // namespace tcx
}  // namespace csc
