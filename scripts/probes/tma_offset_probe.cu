// Probe: does a 2D TMA tiled load accept box start coordinates that are not 16-B aligned in global
// memory (x0 not a multiple of 4 fp32 elements), and negative coordinates (zero fill)?
// nvcc -gencode arch=compute_100a,code=sm_100a -o tma_offset_probe tma_offset_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void probe(const __grid_constant__ CUtensorMap tm, int x0, int y0, float* out, int swz) {
  __shared__ __align__(1024) float buf[32 * 8];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar)));
    asm volatile("fence.proxy.async.shared::cta;\n");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(&bar)), "r"(32 * 8 * 4));
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
            su32(buf)),
        "l"(&tm), "r"(x0), "r"(y0), "r"(su32(&bar))
        : "memory");
    asm volatile(
        "{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W;\n}\n" ::"r"(su32(&bar)));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 32 * 8; i += blockDim.x) out[i] = buf[i];
}

int main() {
  const int W = 1024, H = 64;
  std::vector<float> h(W * H);
  for (int i = 0; i < W * H; ++i) h[i] = static_cast<float>(i);
  float *d, *o;
  cudaMalloc(&d, sizeof(float) * W * H);
  cudaMalloc(&o, sizeof(float) * 256);
  cudaMemcpy(d, h.data(), sizeof(float) * W * H, cudaMemcpyHostToDevice);
  CUtensorMap tm;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(W), static_cast<cuuint64_t>(H)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(W) * 4};
  cuuint32_t box[2] = {32, 8}, es[2] = {1, 1};
  CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, box, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                      CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  int xs[] = {0, 1, 2, 3, 5, 7, 13, -3, -1, 1000};
  for (int x0 : xs) {
    for (int y0 : {0, 3, -2}) {
      probe<<<1, 128>>>(tm, x0, y0, o, 0);
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<float> g(256);
      cudaMemcpy(g.data(), o, sizeof(float) * 256, cudaMemcpyDeviceToHost);
      int bad = 0;
      for (int yy = 0; yy < 8; ++yy)
        for (int xx = 0; xx < 32; ++xx) {
          const int X = x0 + xx, Y = y0 + yy;
          const float want = (X >= 0 && X < W && Y >= 0 && Y < H) ? h[Y * W + X] : 0.f;
          if (g[yy * 32 + xx] != want) ++bad;
        }
      printf("x0 %5d y0 %3d: %s, mismatches %d (first %g)\n", x0, y0, cudaGetErrorString(e), bad, g[0]);
      if (e != cudaSuccess) return 1;
    }
  }
  return 0;
}
