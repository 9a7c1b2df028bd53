// throughput (many warps, independent ops) of conversions vs fp64 vs int ops
#include <cstdio>
#include <cstdint>
template <int OP>
__global__ void k(double* o, long long* t, uint64_t seed) {
  uint64_t a = seed + threadIdx.x * 7919ull + blockIdx.x;
  double acc = 0.0; float facc = 0.f; uint32_t iacc = 0;
  long long t0 = clock64();
  #pragma unroll 8
  for (int i = 0; i < 1024; i++) {
    a = a * 6364136223846793005ull + 1442695040888963407ull;  // keep inputs varying
    if (OP == 0) acc += __ull2double_rn(a >> 11);
    if (OP == 1) facc += __double2float_rn(__longlong_as_double((long long)(a >> 12) | 0x3ff0000000000000ll));
    if (OP == 2) acc = __dmul_rn(acc, 1.0000001) ;
    if (OP == 3) iacc += (uint32_t)(a >> 7) ^ (uint32_t)(a >> 29);
  }
  long long t1 = clock64();
  o[blockIdx.x * blockDim.x + threadIdx.x] = acc + facc + iacc;
  if (threadIdx.x == 0 && blockIdx.x == 0) t[OP] = t1 - t0;
}
int main() {
  double* o; long long* t; cudaMalloc(&o, 148 * 1024 * 8 * 4); cudaMalloc(&t, 64);
  const char* names[4] = {"I2F.F64.U64", "F2F.F32.F64", "DMUL(dep)", "int(xor/shift)"};
  for (int r = 0; r < 2; r++) { k<0><<<148*4, 256>>>(o, t, 1); k<1><<<148*4, 256>>>(o, t, 1); k<2><<<148*4, 256>>>(o, t, 1); k<3><<<148*4, 256>>>(o, t, 1); }
  long long h[4]; cudaMemcpy(h, t, 32, cudaMemcpyDeviceToHost);
  for (int i = 0; i < 4; i++) printf("%s: %.1f cycles per iteration per warp (32 warps/SM)\n", names[i], h[i] / 1024.0);
}
