// Development microbenchmark (not product code): issue rate of tcgen05.mma kind::tf32
// (M=128, K=8) back to back from one thread, A from TMEM (TS) or smem (SS), for several N.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t sdesc_b32(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)1 << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

template <int MODE, int N>
__global__ void rate(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t mbar;
  __shared__ uint32_t tb;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.f;
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" :: "r"(su32(&tb)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 32) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" :: "r"(su32(&mbar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t t = tb;
  if (threadIdx.x == 0) {
    const uint64_t bd = sdesc_b32(su32(sm), 8 * 128 * 8, 512);
    const uint64_t ad = sdesc_b32(su32(sm + 32768), 8 * 128 * 8, 512);
    const uint32_t id = idesc_tf32(128, N, MODE == 0 ? 0 : 1, 1);
    unsigned long long c0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (MODE == 0) {
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n"
                     :: "r"(t), "r"(t + 256), "l"(bd), "r"(id), "r"(1) : "memory");
      } else {
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                     :: "r"(t), "l"(ad), "l"(bd), "r"(id), "r"(1) : "memory");
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" :: "r"(su32(&mbar)) : "memory");
    asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" :: "r"(su32(&mbar)), "r"(0) : "memory");
    unsigned long long c1 = clock64();
    out[blockIdx.x] = c1 - c0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" :: "r"(t), "r"(512));
}

template <int MODE, int N>
void run(const char* name) {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(rate<MODE, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  const int iters = 4096;
  rate<MODE, N><<<148, 128, 65536>>>(iters, d);
  cudaDeviceSynchronize();
  rate<MODE, N><<<148, 128, 65536>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  const double macs = 128.0 * N * 8;
  printf("%-12s N=%3d: %.1f cycles/MMA  -> %.0f MAC/clk/SM  (%s)\n", name, N, avg / iters, macs / (avg / iters),
         cudaGetErrorString(e));
  cudaFree(d);
}

int main2();
int main() {
  run<0, 64>("TS tf32");
  run<0, 128>("TS tf32");
  run<0, 256>("TS tf32");
  run<1, 64>("SS tf32");
  run<1, 128>("SS tf32");
  run<1, 256>("SS tf32");
  return main2();
}

// ---- pipelined variant: like conv_tc's MMA loop (12 MMAs per slot, commit per slot,
// varying A columns / B addresses), optionally with 16 warps streaming tcgen05.st.
template <int STORES, int LBO = 16 * 128>
__global__ void slots(int nslots, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bars[4];
  __shared__ uint32_t tb;
  const int warp = __shfl_sync(0xffffffff, threadIdx.x >> 5, 0), lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 120000 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.f;
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" :: "r"(su32(&tb)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 32) {
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" :: "r"(su32(&bars[i])), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t t = __shfl_sync(0xffffffff, tb, 0);
  volatile __shared__ int stop;
  if (threadIdx.x == 0) stop = 0;
  __syncthreads();
  if (warp == 0) {
    const uint64_t bd0 = sdesc_b32(su32(sm), LBO, 512);
    const uint32_t id = idesc_tf32(128, 128, 0, 1);
    unsigned long long c0 = clock64();
    for (int s = 0; s < nslots; ++s) {
      const int slot = s & 3;
      if (s >= 4) {
        const uint32_t ph = ((s - 4) >> 2) & 1;
        asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" :: "r"(su32(&bars[slot])), "r"(ph) : "memory");
      }
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      uint64_t bd = bd0;
      for (int e = 0; e < 4; ++e) {
        const uint32_t a = t + 256 + slot * 64 + e * 8;
        asm volatile("{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" :: "r"(t), "r"(a), "l"(bd), "r"(id), "r"(1) : "memory");
        asm volatile("{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" :: "r"(t), "r"(a), "l"(bd + 2048), "r"(id), "r"(1) : "memory");
        asm volatile("{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" :: "r"(t), "r"(a + 32), "l"(bd), "r"(id), "r"(1) : "memory");
        bd += 64;
      }
      asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" :: "r"(su32(&bars[slot])) : "memory");
    }
    // drain
    for (int k = 0; k < 4; ++k) {
      const int s = nslots - 4 + k;
      const uint32_t ph = (s >> 2) & 1;
      asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" :: "r"(su32(&bars[s & 3])), "r"(ph) : "memory");
    }
    unsigned long long c1 = clock64();
    if (lane == 0) { out[blockIdx.x] = c1 - c0; stop = 1; }
  } else if (STORES == 2 && warp >= 8 && warp < 16) {
    const uint32_t tq = t + ((uint32_t)(32 * (warp & 3)) << 16);
    float acc = 0.f;
    int i = 0;
    while (!stop) {
      uint32_t v[16];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                     "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                   : "r"(tq + 128 + ((i * 16) & 127)) : "memory");
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      for (int k = 0; k < 16; ++k) acc += __uint_as_float(v[k]);
      ++i;
    }
    if (acc == 12345.f) out[0] = 0;
  } else if (STORES == 1 && warp >= 8) {
    // 16 warps hammer tcgen05.st into the A slot region (columns 256..511) of their lane quarter
    const uint32_t tq = t + ((uint32_t)(32 * (warp & 3)) << 16);
    uint32_t v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int i = 0;
    while (!stop) {
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" :: "r"(tq + 256 + ((i * 8) & 255)), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]) : "memory");
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
      for (int k = 0; k < 40; ++k) __nanosleep(0);
      ++i;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" :: "r"(t), "r"(512));
}

template <int STORES, int LBO = 16 * 128>
void run_slots() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(slots<STORES, LBO>, cudaFuncAttributeMaxDynamicSharedMemorySize, 120000);
  const int ns = 2048;
  slots<STORES, LBO><<<148, 768, 120000>>>(ns, d);
  cudaError_t e = cudaDeviceSynchronize();
  slots<STORES, LBO><<<148, 768, 120000>>>(ns, d);
  e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  printf("slots stores=%d LBO=%d: %.1f cycles/slot (12 MMA) -> %.1f cycles/MMA (%s)\n", STORES, LBO, avg / ns, avg / ns / 12,
         cudaGetErrorString(e));
  cudaFree(d);
}

int main2() {
  run_slots<0>();
  run_slots<1>();
  run_slots<2>();
  run_slots<0, 104 * 128>();
  run_slots<0, 56 * 128>();
  return 0;
}
