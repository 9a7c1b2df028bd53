// tl_common.cuh -- shared device primitives for the sm_100a trajlab kernels.
//
// CPython MT19937 (Modules/_randommodule.c) restated for warps:
//   * seeding (init_by_array) is a 1247-step serial chain -> one lane;
//   * block regeneration ("twist") of 624 words is warp-cooperative: word i
//     reads mt[i], mt[i+1] and mt[i+397] (old) or mt[i-227] (already new),
//     so 32 lanes sweep i in order with one __syncwarp between load and store;
//   * random() = ((w0>>5)*2^26 + (w1>>6)) * 2^-53 is exact in f64.
// All f64 arithmetic that must match CPython bytecode uses explicit _rn
// intrinsics (and the library is built with -fmad=false): no contraction.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/trajlab_b200.h"
#include "mt_init_table.h"

namespace tl {

constexpr int kWarp = 32;
constexpr unsigned kFull = 0xffffffffu;
constexpr int kMtN = 624;
constexpr int kMtM = 397;

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

__device__ __forceinline__ uint32_t mt_temper(uint32_t y) {
  y ^= (y >> 11);
  y ^= (y << 7) & 0x9d2c5680u;
  y ^= (y << 15) & 0xefc60000u;
  y ^= (y >> 18);
  return y;
}

__device__ __forceinline__ uint32_t mt_mix(uint32_t a, uint32_t b, uint32_t src) {
  uint32_t y = (a & 0x80000000u) | (b & 0x7fffffffu);
  return src ^ (y >> 1) ^ ((0u - (y & 1u)) & 0x9908b0dfu);
}

// random.Random(int) seeding of one state (one lane).  key = abs(seed) in
// little-endian 32-bit words (1 or 2 words for |seed| < 2^64).
__device__ __noinline__ void mt_seed_lane(uint32_t* mt, int64_t seed) {
  uint64_t n = seed < 0 ? (uint64_t)0 - (uint64_t)seed : (uint64_t)seed;
  const uint32_t k0 = (uint32_t)n, k1 = (uint32_t)(n >> 32);
  const int klen = k1 ? 2 : 1;
  uint32_t prev = kTlInitGenrand[0];
  uint32_t v1 = 0;
  int j = 0;
  // init_by_array first loop: k = max(624, klen) = 624 iterations
#pragma unroll 4
  for (int i = 1; i < kMtN; i++) {
    uint32_t v = (kTlInitGenrand[i] ^ ((prev ^ (prev >> 30)) * 1664525u)) +
                 (j ? k1 : k0) + (uint32_t)j;
    mt[i] = v;
    prev = v;
    if (i == 1) v1 = v;
    j = (j + 1 >= klen) ? 0 : j + 1;
  }
  mt[0] = prev;  // i >= N: mt[0] = mt[N-1], i = 1
  {
    uint32_t v = (v1 ^ ((prev ^ (prev >> 30)) * 1664525u)) + (j ? k1 : k0) + (uint32_t)j;
    mt[1] = v;
    prev = v;
  }
  // second loop: N-1 iterations, i = 2..623 then wrap to i = 1
#pragma unroll 4
  for (int i = 2; i < kMtN; i++) {
    uint32_t v = (mt[i] ^ ((prev ^ (prev >> 30)) * 1566083941u)) - (uint32_t)i;
    mt[i] = v;
    prev = v;
  }
  mt[0] = prev;
  mt[1] = (mt[1] ^ ((prev ^ (prev >> 30)) * 1566083941u)) - 1u;
  mt[0] = 0x80000000u;
}

// Warp-cooperative regeneration of all 624 words in place (CPython's
// genrand "generate N words at one time").  If ring != nullptr the tempered
// outputs are also written to ring[(ring_base + i) & ring_mask].
__device__ __forceinline__ void mt_twist_warp(uint32_t* mt, uint32_t* ring,
                                              uint32_t ring_base,
                                              uint32_t ring_mask) {
  const int lane = lane_id();
#pragma unroll 1
  for (int i0 = 0; i0 < kMtN; i0 += kWarp) {
    const int i = i0 + lane;
    uint32_t nv = 0;
    if (i < kMtN) {
      const int i1 = (i + 1 == kMtN) ? 0 : i + 1;
      const int src = i < kMtN - kMtM ? i + kMtM : i - (kMtN - kMtM);
      nv = mt_mix(mt[i], mt[i1], mt[src]);
    }
    __syncwarp();
    if (i < kMtN) {
      mt[i] = nv;
      if (ring) ring[(ring_base + (uint32_t)i) & ring_mask] = mt_temper(nv);
    }
  }
  __syncwarp();
}

// Serial reader over an MT state for a single lane (script sampling).
struct MtLane {
  uint32_t* mt;
  int idx;
  __device__ __forceinline__ uint32_t genrand() {
    if (idx >= kMtN) {
      // serial regeneration (rare: only when a script needs > 624 words)
      for (int i = 0; i < kMtN; i++) {
        const int i1 = (i + 1 == kMtN) ? 0 : i + 1;
        const int src = i < kMtN - kMtM ? i + kMtM : i - (kMtN - kMtM);
        mt[i] = mt_mix(mt[i], mt[i1], mt[src]);
      }
      idx = 0;
    }
    return mt_temper(mt[idx++]);
  }
  __device__ __forceinline__ double random() {
    uint32_t a = genrand() >> 5, b = genrand() >> 6;
    return __ull2double_rn(((uint64_t)a << 26) | b) * 0x1.0p-53;
  }
  // Lib/random.py _randbelow_with_getrandbits
  __device__ __forceinline__ uint32_t randbelow(uint32_t n) {
    const int k = 32 - __clz(n);
    uint32_t r = genrand() >> (32 - k);
    while (r >= n) r = genrand() >> (32 - k);
    return r;
  }
  __device__ __forceinline__ int32_t randint(int32_t a, int32_t b) {
    return a + (int32_t)randbelow((uint32_t)(b - a + 1));
  }
  __device__ __forceinline__ double uniform(double a, double b) {
    return __dadd_rn(a, __dmul_rn(__dsub_rn(b, a), random()));
  }
};

__device__ __forceinline__ double rand53(uint32_t w0, uint32_t w1) {
  return __ull2double_rn(((uint64_t)(w0 >> 5) << 26) | (w1 >> 6)) * 0x1.0p-53;
}

// Lib/random.py uniform: a + (b - a) * random(), no FMA
__device__ __forceinline__ double uniform_rn(double a, double b, double r) {
  return __dadd_rn(a, __dmul_rn(__dsub_rn(b, a), r));
}

// warp inclusive scan (int)
__device__ __forceinline__ int warp_incl_scan(int v) {
  const int lane = lane_id();
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    int u = __shfl_up_sync(kFull, v, d);
    if (lane >= d) v += u;
  }
  return v;
}

// EVENT_ORDER alphabets (events.py:38-52), local index -> global EventKind
__constant__ uint8_t kAlpha[4][8] = {
    {TL_EV_CONTACT, TL_EV_GRASPED, TL_EV_DROPPED, TL_EV_SUCCESS,
     TL_EV_EXCESSIVE_COLLISIONS, 255, 255, 255},
    {TL_EV_GRASPED, TL_EV_OBJ_AT_GOAL, TL_EV_RELEASED_AT_GOAL,
     TL_EV_RELEASED_OUTSIDE_GOAL, TL_EV_OBJ_LEFT_GOAL, TL_EV_SUCCESS,
     TL_EV_EXCESSIVE_COLLISIONS, 255},
    {TL_EV_CONTACT, TL_EV_OPENED, TL_EV_SLIGHTLY_OPENED, TL_EV_CLOSED,
     TL_EV_SUCCESS, TL_EV_EXCESSIVE_COLLISIONS, 255, 255},
    {TL_EV_CONTACT, TL_EV_CLOSED, TL_EV_SLIGHTLY_CLOSED, TL_EV_OPEN,
     TL_EV_SUCCESS, TL_EV_EXCESSIVE_COLLISIONS, 255, 255}};

}  // namespace tl
