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

int main() {
  run<0, 64>("TS tf32");
  run<0, 128>("TS tf32");
  run<0, 256>("TS tf32");
  run<1, 64>("SS tf32");
  run<1, 128>("SS tf32");
  run<1, 256>("SS tf32");
  return 0;
}
