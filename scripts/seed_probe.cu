// init_by_array chain latency by instruction form (one warp, clock64):
//   v0: (old ^ (y * C)) + k as the compiler schedules it (IMAD.IADD / VIADD
//       for the add: an fma-pipe op, two cross-pipe hops per step)
//   v1: the add as a 3-source IADD3 with a runtime-zero third operand (stays
//       on the alu pipe: the multiply is the only fma-pipe op of the step)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/seed_probe scripts/seed_probe.cu
#include <cstdint>
#include <cstdio>

template <int V>
__device__ __forceinline__ uint32_t add3(uint32_t a, uint32_t b, uint32_t z) {
  if constexpr (V == 0) return a + b;
  else return a + b + z;
}

template <int V>
__global__ void k(uint32_t* out, const uint32_t* tab, uint32_t key, uint32_t z, long long* t) {
  __shared__ uint32_t mt[640];
  for (int i = threadIdx.x; i < 640; i += 32) mt[i] = tab[i];
  __syncwarp();
  long long t0 = clock64();
  uint32_t prev = mt[0];
#pragma unroll 8
  for (int i = 1; i < 625; i++) {
    const uint32_t old = mt[i];
    prev = add3<V>(old ^ ((prev ^ (prev >> 30)) * 1664525u), key, z);
    mt[i] = prev;
  }
#pragma unroll 8
  for (int i = 1; i < 624; i++) {
    const uint32_t old = mt[i];
    prev = add3<V>(old ^ ((prev ^ (prev >> 30)) * 1566083941u), (uint32_t)-i, z);
    mt[i] = prev;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) {
    out[V] = prev;
    t[V] = t1 - t0;
  }
}

int main() {
  uint32_t *o, *tab;
  long long* t;
  cudaMalloc(&o, 64);
  cudaMalloc(&tab, 640 * 4);
  cudaMalloc(&t, 64);
  uint32_t h[640];
  for (int i = 0; i < 640; i++) h[i] = 19650218u + i * 2654435761u;
  cudaMemcpy(tab, h, sizeof(h), cudaMemcpyHostToDevice);
  long long ht[2];
  uint32_t ho[2];
  for (int r = 0; r < 3; r++) {
    k<0><<<1, 32>>>(o, tab, 0x12345678u, 0u, t);
    k<1><<<1, 32>>>(o, tab, 0x12345678u, 0u, t);
  }
  cudaMemcpy(ht, t, 16, cudaMemcpyDeviceToHost);
  cudaMemcpy(ho, o, 8, cudaMemcpyDeviceToHost);
  printf("{\"v0_cycles_per_step\": %.2f, \"v1_cycles_per_step\": %.2f, \"same\": %d}\n",
         ht[0] / 1247.0, ht[1] / 1247.0, ho[0] == ho[1]);
  return 0;
}
