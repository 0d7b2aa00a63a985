// Development probe (not product code): validates the tcgen05 TF32 building blocks the
// tensor-core kernels use -- SW128 MN-major smem descriptors, the instruction descriptor,
// TMEM alloc / st / ld, SS and TS (A in TMEM) MMAs, commit to an mbarrier, 3xTF32 split.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma_probe umma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// tf32 MN-major operands use SWIZZLE_128B_BASE32B (layout type 1): 128-B rows of 32 fp32,
// 32-byte granules XORed with (row & 3); MN atoms (32 elements) at LBO, K atoms (4 rows) at SBO.
__device__ __forceinline__ uint64_t sdesc_sw128b32(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)1 << 61;  // SWIZZLE_128B_BASE32B
  return d;
}
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// element (k, m) of an MN-major SW128/base32 operand block with BK K-rows: [m atom][k][32]
__device__ __forceinline__ uint32_t sw_off(int k, int m, int BK) {
  const int atom = m >> 5, mm = m & 31;
  return atom * BK * 128 + k * 128 + ((((mm >> 3) ^ (k & 3))) << 5) + (mm & 7) * 4;
}

__device__ __forceinline__ void mma_ss(uint32_t dt, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
               :: "r"(dt), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_ts(uint32_t dt, uint32_t at, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n"
               :: "r"(dt), "r"(at), "l"(b), "r"(idesc), "r"(acc));
}

// MODE 0: SS 1xTF32; 1: TS 1xTF32 (A via tcgen05.st); 2: TS 3xTF32
template <int MODE>
__global__ void probe(const float* A, const float* B, float* C, int KT) {
  extern __shared__ uint8_t smraw[];
  __shared__ uint64_t mbar;
  __shared__ uint32_t tbase_sh;
  const uint32_t raw = smem_u32(smraw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* sm = smraw + (base - raw);
  const int K = KT * 8;
  float* Ah = reinterpret_cast<float*>(sm);                  // K x 128
  float* Bh = reinterpret_cast<float*>(sm + KT * 4096);
  float* Bl = reinterpret_cast<float*>(sm + 2 * KT * 4096);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < K * 128; e += blockDim.x) {
    const int k = e / 128, m = e % 128;
    const uint32_t off = sw_off(k, m, K);
    float a = A[e], b = B[e];
    *reinterpret_cast<float*>(sm + off) = a;
    const float bh = __uint_as_float(__float_as_uint(b) & 0xFFFFE000u);
    *reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(Bh) + off) = b;
    *reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(Bl) + off) = b - bh;
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" :: "r"(smem_u32(&tbase_sh)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 32) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" :: "r"(smem_u32(&mbar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tbase = tbase_sh;
  const uint32_t tD = tbase;              // cols [0,128)
  const uint32_t tA = tbase + 128;        // hi: cols [128, 128+K)
  const uint32_t tAl = tbase + 128 + K;   // lo: cols [128+K, 128+2K)
  if (MODE >= 1 && warp >= 4) {
    // lane quarter (warp % 4): lanes 32*(warp%4) .. +31 = positions m
    const int m = 32 * (warp & 3) + lane;
    for (int kt = 0; kt < KT; ++kt) {
      uint32_t h[8], l[8];
      for (int j = 0; j < 8; ++j) {
        const float a = A[(kt * 8 + j) * 128 + m];
        const float ah = __uint_as_float(__float_as_uint(a) & 0xFFFFE000u);
        h[j] = __float_as_uint(a);
        l[j] = __float_as_uint(a - ah);
      }
      const uint32_t lane_off = (uint32_t)(32 * (warp & 3)) << 16;
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n"
                   :: "r"(tA + lane_off + kt * 8), "r"(h[0]), "r"(h[1]), "r"(h[2]), "r"(h[3]), "r"(h[4]), "r"(h[5]), "r"(h[6]), "r"(h[7]));
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n"
                   :: "r"(tAl + lane_off + kt * 8), "r"(l[0]), "r"(l[1]), "r"(l[2]), "r"(l[3]), "r"(l[4]), "r"(l[5]), "r"(l[6]), "r"(l[7]));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (tid == 0) {
    const uint32_t id_ss = idesc_tf32(128, 128, 1, 1);
    const uint32_t id_ts = idesc_tf32(128, 128, 0, 1);
    for (int kt = 0; kt < KT; ++kt) {
      const uint64_t bd = sdesc_sw128b32(smem_u32(Bh) + kt * 1024, K * 128, 512);
      const uint64_t bld = sdesc_sw128b32(smem_u32(Bl) + kt * 1024, K * 128, 512);
      if (MODE == 0) {
        const uint64_t ad = sdesc_sw128b32(smem_u32(Ah) + kt * 1024, K * 128, 512);
        mma_ss(tD, ad, bd, id_ss, kt > 0);
      } else if (MODE == 1) {
        mma_ts(tD, tA + kt * 8, bd, id_ts, kt > 0);
      } else {
        mma_ts(tD, tA + kt * 8, bd, id_ts, kt > 0);
        mma_ts(tD, tA + kt * 8, bld, id_ts, 1);
        mma_ts(tD, tAl + kt * 8, bd, id_ts, 1);
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" :: "r"(smem_u32(&mbar)) : "memory");
  }
  // wait for the MMAs
  {
    const uint32_t mb = smem_u32(&mbar);
    asm volatile("{\n.reg .pred P1;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra WAIT_%=;\n}\n" :: "r"(mb), "r"(0) : "memory");
  }
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (warp < 4) {
    const int m = 32 * warp + lane;
    for (int n0 = 0; n0 < 128; n0 += 16) {
      uint32_t v[16];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                     "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                   : "r"(tD + ((uint32_t)(32 * warp) << 16) + n0));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      for (int j = 0; j < 16; ++j) C[m * 128 + n0 + j] = __uint_as_float(v[j]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" :: "r"(tbase), "r"(512));
}

int main() {
  const int KT = 4, K = KT * 8;
  std::vector<float> A(K * 128), B(K * 128);
  int bad_total = 0;
  for (int mode = 0; mode < 3; ++mode) {
    srand(1 + mode);
    for (auto& v : A) v = (mode < 2) ? (float)((rand() % 17) - 8) : (float)rand() / RAND_MAX - 0.5f;
    for (auto& v : B) v = (mode < 2) ? (float)((rand() % 13) - 6) * 0.25f : (float)rand() / RAND_MAX - 0.5f;
    float *dA, *dB, *dC;
    CK(cudaMalloc(&dA, A.size() * 4)); CK(cudaMalloc(&dB, B.size() * 4)); CK(cudaMalloc(&dC, 128 * 128 * 4));
    CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemset(dC, 0, 128 * 128 * 4));
    const int smem = 3 * KT * 4096 + 1024;
    if (mode == 0) { CK(cudaFuncSetAttribute(probe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)); probe<0><<<1, 256, smem>>>(dA, dB, dC, KT); }
    if (mode == 1) { CK(cudaFuncSetAttribute(probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)); probe<1><<<1, 256, smem>>>(dA, dB, dC, KT); }
    if (mode == 2) { CK(cudaFuncSetAttribute(probe<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)); probe<2><<<1, 256, smem>>>(dA, dB, dC, KT); }
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<float> C(128 * 128);
    CK(cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost));
    double maxerr = 0, maxref = 0; int bad = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < 128; ++n) {
        double ref = 0;
        for (int k = 0; k < K; ++k) ref += (double)A[k * 128 + m] * (double)B[k * 128 + n];
        const double err = fabs(ref - C[m * 128 + n]);
        maxerr = fmax(maxerr, err); maxref = fmax(maxref, fabs(ref));
        if (mode < 2 && err != 0.0 && bad++ < 5) printf("mode %d mismatch m=%d n=%d got %f ref %f\n", mode, m, n, C[m * 128 + n], ref);
      }
    printf("mode %d: max abs err %.3e (max |ref| %.3e, rel %.3e) %s\n", mode, maxerr, maxref, maxerr / maxref,
           (mode < 2 ? (bad == 0 ? "EXACT" : "MISMATCH") : (maxerr / maxref < 1e-6 ? "OK(3xTF32)" : "BAD")));
    if (mode < 2 && bad) bad_total++;
    if (mode == 2 && maxerr / maxref >= 1e-6) bad_total++;
    cudaFree(dA); cudaFree(dB); cudaFree(dC);
  }
  printf(bad_total ? "PROBE FAILED\n" : "PROBE PASSED\n");
  return bad_total ? 1 : 0;
}
