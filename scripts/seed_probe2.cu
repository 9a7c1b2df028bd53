// clock64 timing of CPython seeding (init_by_array) variants, one thread.
// v0: library mt_seed_lane; v1: table values prefetched one group of 8
// ahead into registers (loop 1) and old words one group ahead (loop 2).
#include "../paper_2412_13211_b200/csrc/tl_common.cuh"
#include <cstdio>
using namespace tl;

__device__ __forceinline__ uint32_t s1(uint32_t prev, uint32_t tab, uint32_t key) {
  return (tab ^ ((prev ^ (prev >> 30)) * 1664525u)) + key;
}
__device__ __noinline__ void seed_v1(uint32_t* mt, uint32_t k0, uint32_t* out) {
  const uint32_t* T = kTlInitGenrand;
  uint32_t prev = T[0];
  const uint32_t v1 = s1(prev, T[1], k0);
  mt[1] = v1;
  prev = v1;
  uint32_t a[8], b[8];
#pragma unroll
  for (int k = 0; k < 8; k++) a[k] = T[2 + k];
  // 77 groups of 8: i0 = 2 + 8g
  for (int g = 0; g < 76; g += 2) {
    const int i0 = 2 + 8 * g;
#pragma unroll
    for (int k = 0; k < 8; k++) b[k] = T[i0 + 8 + k];
#pragma unroll
    for (int k = 0; k < 8; k++) { prev = s1(prev, a[k], k0); mt[i0 + k] = prev; }
#pragma unroll
    for (int k = 0; k < 8; k++) a[k] = T[i0 + 16 + k < 624 ? i0 + 16 + k : 623];
#pragma unroll
    for (int k = 0; k < 8; k++) { prev = s1(prev, b[k], k0); mt[i0 + 8 + k] = prev; }
  }
  // group 76: i0 = 610
#pragma unroll
  for (int k = 0; k < 8; k++) { prev = s1(prev, a[k], k0); mt[610 + k] = prev; }
#pragma unroll
  for (int k = 0; k < 6; k++) { prev = s1(prev, T[618 + k], k0); mt[618 + k] = prev; }
  mt[0] = prev;
  prev = s1(prev, v1, k0);
  mt[1] = prev;
  // loop 2
#pragma unroll
  for (int k = 0; k < 8; k++) a[k] = mt[2 + k];
  for (int g = 0; g < 76; g += 2) {
    const int i0 = 2 + 8 * g;
#pragma unroll
    for (int k = 0; k < 8; k++) b[k] = mt[i0 + 8 + k];
#pragma unroll
    for (int k = 0; k < 8; k++) { prev = (a[k] ^ ((prev ^ (prev >> 30)) * 1566083941u)) - (uint32_t)(i0 + k); out[i0 + k] = prev; }
#pragma unroll
    for (int k = 0; k < 8; k++) a[k] = mt[i0 + 16 + k < 624 ? i0 + 16 + k : 623];
#pragma unroll
    for (int k = 0; k < 8; k++) { prev = (b[k] ^ ((prev ^ (prev >> 30)) * 1566083941u)) - (uint32_t)(i0 + 8 + k); out[i0 + 8 + k] = prev; }
  }
#pragma unroll
  for (int k = 0; k < 8; k++) { prev = (a[k] ^ ((prev ^ (prev >> 30)) * 1566083941u)) - (uint32_t)(610 + k); out[610 + k] = prev; }
#pragma unroll
  for (int k = 0; k < 6; k++) { prev = (mt[618 + k] ^ ((prev ^ (prev >> 30)) * 1566083941u)) - (uint32_t)(618 + k); out[618 + k] = prev; }
  out[1] = (mt[1] ^ ((prev ^ (prev >> 30)) * 1566083941u)) - 1u;
  out[0] = 0x80000000u;
}

__global__ void k(uint32_t* gout, long long* t, int64_t seed, int mode) {
  __shared__ uint32_t row[2][625];
  long long t0 = clock64();
  if (mode == 0) mt_seed_lane(row[0], seed, nullptr);
  else seed_v1(row[1], (uint32_t)seed, row[1]);
  long long t1 = clock64();
  t[mode] = t1 - t0;
  for (int i = 0; i < 624; i++) gout[mode * 624 + i] = row[mode][i];
}
int main() {
  uint32_t* g; long long* t; cudaMalloc(&g, 8192); cudaMalloc(&t, 64);
  long long h[2];
  uint32_t hg[1248];
  for (int r = 0; r < 3; r++) { k<<<1, 32>>>(g, t, 12345, 0); k<<<1, 32>>>(g, t, 12345, 1); }
  cudaMemcpy(h, t, 16, cudaMemcpyDeviceToHost);
  cudaMemcpy(hg, g, sizeof(hg), cudaMemcpyDeviceToHost);
  int same = 1;
  for (int i = 0; i < 624; i++) same &= hg[i] == hg[624 + i];
  printf("v0 %lld cycles (%.1f/step)  v1 %lld cycles (%.1f/step)  same=%d\n", h[0], h[0] / 1247.0, h[1], h[1] / 1247.0, same);
  return 0;
}
