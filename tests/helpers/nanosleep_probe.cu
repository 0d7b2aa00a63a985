// How long does __nanosleep(t) suspend a warp on sm_100a?  (tuning probe for the spin-wait policy)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(unsigned long long* out, unsigned ns) {
  unsigned long long t0 = clock64();
  for (int i = 0; i < 1000; ++i) __nanosleep(ns);
  out[threadIdx.x / 32] = clock64() - t0;
}
int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64 * 8);
  unsigned vals[] = {0, 32, 64, 128, 256, 512, 1000, 2000, 5000};
  for (unsigned ns : vals) {
    k<<<1, 32>>>(d, ns);
    unsigned long long h[2];
    cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    printf("nanosleep(%u): %.1f cycles per call\n", ns, h[0] / 1000.0);
    k<<<1, 256>>>(d, ns);
    cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    printf("  (8 warps) %.1f cycles per call\n", h[0] / 1000.0);
  }
  return 0;
}
