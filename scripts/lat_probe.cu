// latency microbenchmark: dependent chains of one instruction kind (clock64)
#include <cstdio>
#include <cstdint>
__global__ void k(double* od, uint32_t* ou, long long* t, double a, uint32_t b) {
  double x = a; uint32_t y = b;
  long long t0 = clock64();
  #pragma unroll 1
  for (int i = 0; i < 1000; i++) { x = __dadd_rn(x, a); }
  long long t1 = clock64();
  #pragma unroll 1
  for (int i = 0; i < 1000; i++) { x = __dmul_rn(x, a); }
  long long t2 = clock64();
  #pragma unroll 1
  for (int i = 0; i < 1000; i++) { y = y * 1664525u; }
  long long t3 = clock64();
  #pragma unroll 1
  for (int i = 0; i < 1000; i++) { y = (y ^ (y >> 30)) * 1664525u + b; }
  long long t4 = clock64();
  float f = (float)a;
  #pragma unroll 1
  for (int i = 0; i < 1000; i++) { f = __fadd_rn(f, 1.5f); }
  long long t5 = clock64();
  #pragma unroll 1
  for (int i = 0; i < 1000; i++) { x = __dadd_rn(x, __dmul_rn(__dmul_rn(__dsub_rn(a, x), 0.05), 0.3)); }
  long long t6 = clock64();
  od[0] = x + f; ou[0] = y;
  t[0] = t1 - t0; t[1] = t2 - t1; t[2] = t3 - t2; t[3] = t4 - t3; t[4] = t5 - t4; t[5] = t6 - t5;
}
int main() {
  double* od; uint32_t* ou; long long* t;
  cudaMalloc(&od, 8); cudaMalloc(&ou, 4); cudaMalloc(&t, 64);
  for (int r = 0; r < 2; r++) k<<<1, 1>>>(od, ou, t, 1.0000001, 12345u);
  long long h[6]; cudaMemcpy(h, t, 48, cudaMemcpyDeviceToHost);
  printf("cycles per op: dadd %.1f  dmul %.1f  imad %.1f  seed-step %.1f  fadd %.1f  cum-step %.1f\n",
         h[0] / 1000.0, h[1] / 1000.0, h[2] / 1000.0, h[3] / 1000.0, h[4] / 1000.0, h[5] / 1000.0);
  return 0;
}
