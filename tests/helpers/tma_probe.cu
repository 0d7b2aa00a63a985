// Development probe (not product code): TMA 2D tile load (SWIZZLE_128B) of a flattened-plane
// fp32 view, as csc_wgrad_tc.cu uses it.  Build: nvcc -gencode arch=compute_100a,code=sm_100a
// -I../../paper_1909_00145_b200/csrc -o tma_probe tma_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "csc_tc_ptx.cuh"
using namespace csc::tcx;

template <int MODE>
__global__ void probe(const __grid_constant__ CUtensorMap tm, const CUtensorMap* tm_glob, float* out, int c0, int c1, int rows) {
  extern __shared__ uint8_t smraw[];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t raw = su32(smraw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* sm = smraw + (base - raw);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (MODE == 0) {
      mbar_arrive_expect_tx(&bar, 128u * rows);
      tma_load_2d(base, &tm, c0, c1, &bar);
    } else if (MODE == 2) {
      mbar_arrive_expect_tx(&bar, 128u * rows);
      tma_load_2d(base, tm_glob, c0, c1, &bar);
    } else {
      mbar_arrive_expect_tx(&bar, 128u * rows);
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::
              "r"(base), "l"(reinterpret_cast<uint64_t>(&tm)), "r"(c0), "r"(c1), "r"(su32(&bar))
          : "memory");
    }
  }
  mbar_wait(&bar, 0);
  for (int e = threadIdx.x; e < rows * 32; e += blockDim.x) out[e] = reinterpret_cast<float*>(sm)[e];
}

typedef CUresult (*PFN_enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                            const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                            CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 0;
  const int swz = argc > 2 ? atoi(argv[2]) : 1;
  const int direct = argc > 3 ? atoi(argv[3]) : 0;
  const int plane = argc > 4 ? atoi(argv[4]) : 74 * 134, nplanes = 15, rows = 5;
  std::vector<float> h(static_cast<size_t>(plane) * nplanes);
  for (size_t i = 0; i < h.size(); ++i) h[i] = static_cast<float>(i);
  float *d, *o;
  cudaMalloc(&d, h.size() * 4);
  cudaMalloc(&o, rows * 32 * 4);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  printf("entry point %p q=%d\n", fp, (int)q);
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)plane, (cuuint64_t)nplanes};
  cuuint64_t str[1] = {(cuuint64_t)plane * 4};
  cuuint32_t box[2] = {32, (cuuint32_t)rows}, es[2] = {1, 1};
  PFN_enc enc = direct ? (PFN_enc)&cuTensorMapEncodeTiled : (PFN_enc)fp;
  CUresult cr = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const unsigned long long* w = reinterpret_cast<const unsigned long long*>(&tm);
  printf("tmap words %llx %llx %llx %llx\n", w[0], w[1], w[2], w[3]);
  CUtensorMap* tg = nullptr;
  cudaMalloc(&tg, sizeof(CUtensorMap));
  cudaMemcpy(tg, &tm, sizeof(CUtensorMap), cudaMemcpyHostToDevice);
  printf("encode %d\n", (int)cr);
  cudaFuncSetAttribute(probe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
  cudaFuncSetAttribute(probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
  cudaFuncSetAttribute(probe<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
  const int c0 = argc > 5 ? atoi(argv[5]) : 134 * 3 + 32, c1 = argc > 6 ? atoi(argv[6]) : 2;
  if (mode == 0) probe<0><<<1, 128, 8192>>>(tm, tg, o, c0, c1, rows);
  else if (mode == 2) probe<2><<<1, 128, 8192>>>(tm, tg, o, c0, c1, rows);
  else probe<1><<<1, 128, 8192>>>(tm, tg, o, c0, c1, rows);
  cudaError_t e = cudaDeviceSynchronize();
  printf("mode %d: %s\n", mode, cudaGetErrorString(e));
  std::vector<float> ho(rows * 32);
  cudaMemcpy(ho.data(), o, rows * 32 * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int r = 0; r < rows; ++r)
    for (int c = 0; c < 32; ++c) {
      // SWIZZLE_128B: 16-B chunk index XOR (row & 7)
      const int chunk = swz ? ((c >> 2) ^ (r & 7)) : (c >> 2);
      const float got = ho[r * 32 + chunk * 4 + (c & 3)];
      const float want = h[(size_t)(c1 + r) * plane + c0 + c];
      if (got != want) ++bad;
    }
  printf("mismatches %d (first row got %g %g want %g)\n", bad, ho[0], ho[1], h[(size_t)c1 * plane + c0]);
  return 0;
}
