// fp64 latency (dependent chain, unrolled) and the cum recurrence step
#include <cstdio>
#include <cstdint>
__global__ void k(double* o, long long* t, double a, double b) {
  double x = a, c = 0.0;
  long long t0 = clock64();
  #pragma unroll
  for (int i = 0; i < 256; i++) x = __dadd_rn(x, b);
  long long t1 = clock64();
  #pragma unroll
  for (int i = 0; i < 64; i++) c = __dadd_rn(c, __dmul_rn(__dmul_rn(__dsub_rn(a, c), 0.05), b));
  long long t2 = clock64();
  float f = 0.f;
  #pragma unroll
  for (int i = 0; i < 256; i++) f = __fadd_rn(f, (float)b);
  long long t3 = clock64();
  o[0] = x + c + f; t[0] = t1 - t0; t[1] = t2 - t1; t[2] = t3 - t2;
}
int main() {
  double* o; long long* t; cudaMalloc(&o, 8); cudaMalloc(&t, 32);
  for (int r = 0; r < 3; r++) k<<<1, 32>>>(o, t, 9000.0, 0.37);
  long long h[3]; cudaMemcpy(h, t, 24, cudaMemcpyDeviceToHost);
  printf("dadd latency %.1f  cum step %.1f  fadd latency %.1f cycles\n", h[0] / 256.0, h[1] / 64.0, h[2] / 256.0);
}
