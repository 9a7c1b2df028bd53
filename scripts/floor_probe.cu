// Critical-path latency constants of the generator (bench.py's latency
// roofline): one thread, clock64 around dependent chains that mirror
//   (a) CPython init_by_array (Modules/_randommodule.c): 624 + 623 dependent
//       steps, each step's multiply-xor-add on the previous word;
//   (b) _advance_cum (synth.py:192-196): cum += (0.9*limit - cum)*0.05*u,
//       three dependent f64 ops per record (sub, mul, mul then add) with
//       round-to-nearest intrinsics as k_synth_cta issues them.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o scripts/floor_probe scripts/floor_probe.cu
#include <cstdint>
#include <cstdio>

__global__ void k(uint32_t* mt_out, double* cum_out, const double* u, long long* t) {
  __shared__ uint32_t mt[624];
  for (int i = 0; i < 624; i++) mt[i] = 19650218u + i * 2654435761u;
  const uint32_t key = 0x12345678u;
  __syncwarp();
  long long t0 = clock64();
  // init_by_array, key length 1: first loop (max(624, 1) steps), second loop
  // 623.  The old word mt[i] does not depend on the chain: it is generated
  // off the critical path (k_fuzz_reset prefetches it a group ahead), so only
  // the shift / xor / multiply / xor / add on the previous word is timed.
  uint32_t prev = mt[0];
#pragma unroll 4
  for (int i = 1; i < 625; i++) {
    const uint32_t old = 19650218u + (uint32_t)i * 2654435761u;
    const uint32_t v = (old ^ ((prev ^ (prev >> 30)) * 1664525u)) + key;
    mt[i % 624] = v;
    prev = v;
  }
#pragma unroll 4
  for (int i = 1; i < 624; i++) {
    const uint32_t old = 40503u + (uint32_t)i * 2246822519u;
    const uint32_t v = (old ^ ((prev ^ (prev >> 30)) * 1566083941u)) - (uint32_t)i;
    mt[i] = v;
    prev = v;
  }
  long long t1 = clock64();
  double cum = 0.0;
  const double L09 = 4500.0;
#pragma unroll 8
  for (int r = 0; r < 1024; r++)
    cum = __dadd_rn(cum, __dmul_rn(__dmul_rn(__dsub_rn(L09, cum), 0.05), u[r & 255]));
  long long t2 = clock64();
  mt_out[0] = mt[17];
  cum_out[0] = cum;
  t[0] = t1 - t0;
  t[1] = t2 - t1;
}

int main() {
  uint32_t* mo;
  double *co, *u;
  long long* t;
  cudaMalloc(&mo, 4);
  cudaMalloc(&co, 8);
  cudaMalloc(&u, 256 * 8);
  cudaMalloc(&t, 16);
  double hu[256];
  for (int i = 0; i < 256; i++) hu[i] = (i * 0.618033988749895) - (int)(i * 0.618033988749895);
  cudaMemcpy(u, hu, sizeof(hu), cudaMemcpyHostToDevice);
  long long h[2] = {0, 0};
  for (int r = 0; r < 3; r++) k<<<1, 32>>>(mo, co, u, t);
  cudaMemcpy(h, t, 16, cudaMemcpyDeviceToHost);
  printf("{\"init_by_array_cycles\": %lld, \"init_by_array_steps\": 1247, "
         "\"cycles_per_seed_step\": %.2f, \"cum_cycles_per_record\": %.2f, "
         "\"how\": \"scripts/floor_probe.cu: one warp, clock64 around the dependent chains\"}\n",
         h[0], h[0] / 1247.0, h[1] / 1024.0);
  return 0;
}
