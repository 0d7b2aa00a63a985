// Test-only pin: runs NVIDIA's curand_Philox4x32_10 (curand_philox4x32_x.h) on
// the HOST for (ctr, key) pairs read from stdin and writes the 4 output words to
// stdout.  Used by tests/test_oracle_philox.py to pin the oracle's Philox
// bit-exactly against a library routine.  Not part of the product or oracle.
#define QUALIFIERS static inline __host__ __device__
#include <cstdio>
#include <cstdint>
#include <vector>
#include <vector_types.h>
#include <curand_philox4x32_x.h>

int main() {
  uint64_t count = 0;
  if (fread(&count, sizeof(count), 1, stdin) != 1) return 1;
  std::vector<uint32_t> in(count * 6), out(count * 4);
  if (fread(in.data(), sizeof(uint32_t), in.size(), stdin) != in.size()) return 2;
  for (uint64_t q = 0; q < count; ++q) {
    const uint32_t* p = &in[q * 6];
    uint4 c = make_uint4(p[0], p[1], p[2], p[3]);
    uint2 k = make_uint2(p[4], p[5]);
    uint4 o = curand_Philox4x32_10(c, k);
    out[q * 4 + 0] = o.x; out[q * 4 + 1] = o.y; out[q * 4 + 2] = o.z; out[q * 4 + 3] = o.w;
  }
  fwrite(out.data(), sizeof(uint32_t), out.size(), stdout);
  return 0;
}
