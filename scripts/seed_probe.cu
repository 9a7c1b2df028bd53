// clock64 timing of one CPython seeding (init_by_array) by one thread
#include "../paper_2412_13211_b200/csrc/tl_common.cuh"
#include <cstdio>
__global__ void k(uint32_t* gout, long long* t, int64_t seed, int mode) {
  __shared__ uint32_t row[625];
  long long t0 = clock64();
  if (mode == 0) tl::mt_seed_lane(row, seed, nullptr);
  else tl::mt_seed_lane(row, seed, gout);
  long long t1 = clock64();
  // chain-only reference: 1247 steps of the loop-1 recurrence in registers
  uint32_t prev = (uint32_t)seed;
  #pragma unroll 8
  for (int i = 0; i < 1248; i++) prev = (kTlInitGenrand[i % 624] ^ ((prev ^ (prev >> 30)) * 1664525u)) + 7u;
  long long t2 = clock64();
  t[0] = t1 - t0; t[1] = t2 - t1; gout[700] = prev + row[5];
}
int main() {
  uint32_t* g; long long* t; cudaMalloc(&g, 4096); cudaMalloc(&t, 64);
  long long h[2];
  for (int mode = 0; mode < 2; mode++) {
    for (int r = 0; r < 3; r++) k<<<1, 32>>>(g, t, 12345, mode);
    cudaMemcpy(h, t, 16, cudaMemcpyDeviceToHost);
    printf("mode %d: seed %lld cycles (%.1f/iter)  pure chain %lld (%.1f/iter)\n", mode, h[0], h[0] / 1247.0, h[1], h[1] / 1248.0);
  }
  return 0;
}
