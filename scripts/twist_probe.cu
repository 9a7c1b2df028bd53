// cycles per MT19937 block regeneration for several warp/CTA mappings
#include "../paper_2412_13211_b200/csrc/tl_synth_cta.cuh"
#include <cstdio>
using namespace tl;

__global__ void k_cta(uint32_t* out, long long* t, int reps) {
  __shared__ uint32_t mt[624];
  __shared__ uint32_t ring[4096];
  for (int i = threadIdx.x; i < 624; i += blockDim.x) mt[i] = i * 2654435761u;
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < reps; r++) mt_twist_block<7>(mt, ring, r * 624);
  long long t1 = clock64();
  if (threadIdx.x == 0) { t[0] = (t1 - t0) / reps; out[0] = ring[5]; }
}

__global__ void k_warp(uint32_t* out, long long* t, int reps) {
  __shared__ uint32_t mt[624];
  __shared__ uint32_t ring[2048];
  for (int i = threadIdx.x; i < 624; i += 32) mt[i] = i * 2654435761u;
  __syncwarp();
  long long t0 = clock64();
  for (int r = 0; r < reps; r++) mt_twist_warp(mt, ring, r * 624, 2047);
  long long t1 = clock64();
  if (threadIdx.x == 0) { t[1] = (t1 - t0) / reps; out[1] = ring[5]; }
}

int main() {
  uint32_t* o; long long* t; cudaMalloc(&o, 64); cudaMalloc(&t, 64);
  long long h[2];
  for (int it = 0; it < 2; it++) {
    k_cta<<<1, 64>>>(o, t, 100);
    k_warp<<<1, 32>>>(o, t, 100);
  }
  cudaMemcpy(h, t, 16, cudaMemcpyDeviceToHost);
  printf("cycles/block: cta64 3-phase %lld   warp32 grouped %lld\n", h[0], h[1]);
  // contention: 7 CTAs per SM (1036 CTAs)
  for (int it = 0; it < 2; it++) k_cta<<<148 * 7, 64>>>(o, t, 100);
  cudaMemcpy(h, t, 8, cudaMemcpyDeviceToHost);
  printf("cta64 with 7 CTAs/SM: %lld\n", h[0]);
  return 0;
}
