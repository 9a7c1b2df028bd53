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
#include <cstdio>
#include <stdint.h>

#include "../../include/trajlab_b200.h"
#include "mt_init_table.h"

namespace tl {

#ifdef TL_PROFILE
// phase timestamps of one CTA/warp (profiling build only, scripts/phase_probe.py)
__device__ unsigned long long g_tl_prof[128];
#define TL_STAMP(i) do { if (blockIdx.x == 0) g_tl_prof[(i)] = clock64(); } while (0)
#else
#define TL_STAMP(i) do { } while (0)
#endif

#ifdef TL_PHASES
// step timeline of the last launches (profiling build only,
// scripts/step_timeline.py): [kernel][block] = {first start, last end}
// (globaltimer ns); kernel 0 = fuzz reset, 1 = k_scan_emit
__device__ unsigned long long g_tl_step[2][2048][2];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
struct BlockSpan {  // start at construction, end (max over warps) at scope exit
  int k;
  __device__ explicit BlockSpan(int kk) : k(kk) {
    if (blockIdx.x < 2048 && (threadIdx.x & 31) == 0)
      atomicMin(&g_tl_step[k][blockIdx.x][0], gtimer());
  }
  __device__ ~BlockSpan() {
    if (blockIdx.x < 2048 && (threadIdx.x & 31) == 0)
      atomicMax(&g_tl_step[k][blockIdx.x][1], gtimer());
  }
};
#define TL_BLOCK_SPAN(k) BlockSpan tl_span_(k)
#else
#define TL_BLOCK_SPAN(k) do { } while (0)
#endif

// Bounds / invariant checks of the checked build (-DTL_CHECK,
// scripts/gpu_check_build.sh): a failing check prints its site and traps
// (the CUDA context dies, the calling test fails loudly).  compute-sanitizer
// is not available on the GPU pool, so this build + the GPU test suite is
// the memory-safety evidence; the product build compiles them out.
#ifdef TL_CHECK
#define TL_ASSERT(c)                                                              \
  do {                                                                            \
    if (!(c)) {                                                                   \
      printf("TL_ASSERT failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #c, \
             (int)blockIdx.x, (int)threadIdx.x);                                  \
      __trap();                                                                   \
    }                                                                             \
  } while (0)
#else
#define TL_ASSERT(c) do { } while (0)
#endif

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
  // y = (a & UPPER) | (b & LOWER) in one LOP3 with a single mask constant;
  // y & 1 == b & 1, so the MATRIX_A term is a predicate + SEL on b; then one
  // three-way XOR: 5 ALU ops per word (the compiler's own form used 7)
  uint32_t y, mag, r;
  asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(y) : "r"(a), "r"(b), "r"(0x80000000u));
  asm("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\tand.b32 t, %1, 1;\n\tsetp.ne.b32 p, t, 0;\n\t"
      "selp.b32 %0, 0x9908b0df, 0, p;\n\t}" : "=r"(mag) : "r"(b));
  asm("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(r) : "r"(src), "r"(y >> 1), "r"(mag));
  return r;
}

// random.Random(int) seeding of one state (one thread; init_by_array of
// Modules/_randommodule.c).  key = abs(seed) as little-endian 32-bit words
// (1 or 2 words for |seed| < 2^64).  `mt` may be a padded shared-memory row.
// `out` (optional) receives the final state (e.g. a global-memory copy);
// `mt` is the working row (the second loop reads the first loop's values).
// Groups of 8 with exact bounds (622 = 77*8 + 6): no predication, the
// table constants of a group are loaded before its serial chain.
template <int KLEN>
__device__ __forceinline__ uint32_t seed_step1(uint32_t prev, uint32_t tab, int i, uint32_t k0,
                                               uint32_t k1) {
  const int j = KLEN == 1 ? 0 : ((i - 1) & 1);
  const uint32_t key = KLEN == 1 ? k0 : (j ? k1 + 1u : k0);
  return (tab ^ ((prev ^ (prev >> 30)) * 1664525u)) + key;
}

template <int KLEN>
__device__ __forceinline__ void mt_seed_impl(uint32_t* mt, uint32_t k0, uint32_t k1,
                                             uint32_t* out) {
  // The chain is 5 dependent integer ops per step; the table / old-word
  // operands of group g+1 are loaded while group g runs (register double
  // buffer), so no load latency lands on the chain.
  const uint32_t* T = kTlInitGenrand;
  uint32_t prev = T[0];
  // first loop, k = max(624, klen) = 624 iterations: i = 1..623, then i = 1
  const uint32_t v1 = seed_step1<KLEN>(prev, T[1], 1, k0, k1);
  mt[1] = v1;
  prev = v1;
  uint32_t a[8], b[8];
#pragma unroll
  for (int k = 0; k < 8; k++) a[k] = T[2 + k];
  for (int g = 0; g < 76; g += 2) {  // groups i0 = 2 + 8g, g < 76 (2..609)
    const int i0 = 2 + 8 * g;
#pragma unroll
    for (int k = 0; k < 8; k++) b[k] = T[i0 + 8 + k];
#pragma unroll
    for (int k = 0; k < 8; k++) {
      prev = seed_step1<KLEN>(prev, a[k], i0 + k, k0, k1);
      mt[i0 + k] = prev;
    }
#pragma unroll
    for (int k = 0; k < 8; k++) a[k] = T[i0 + 16 + k];  // <= 617 + 8 < 624
#pragma unroll
    for (int k = 0; k < 8; k++) {
      prev = seed_step1<KLEN>(prev, b[k], i0 + 8 + k, k0, k1);
      mt[i0 + 8 + k] = prev;
    }
  }
#pragma unroll
  for (int k = 0; k < 8; k++) {  // group 76: 610..617
    prev = seed_step1<KLEN>(prev, a[k], 610 + k, k0, k1);
    mt[610 + k] = prev;
  }
#pragma unroll
  for (int k = 0; k < 6; k++) {  // 618..623
    prev = seed_step1<KLEN>(prev, T[618 + k], 618 + k, k0, k1);
    mt[618 + k] = prev;
  }
  mt[0] = prev;
  prev = seed_step1<KLEN>(prev, v1, kMtN, k0, k1);  // 624th iteration: i = 1, j = 623 % klen
  mt[1] = prev;
  // second loop: N-1 iterations, i = 2..623 then wrap to i = 1
  auto step2 = [](uint32_t pv, uint32_t old, int i) {
    return (old ^ ((pv ^ (pv >> 30)) * 1566083941u)) - (uint32_t)i;
  };
#pragma unroll
  for (int k = 0; k < 8; k++) a[k] = mt[2 + k];
  for (int g = 0; g < 76; g += 2) {
    const int i0 = 2 + 8 * g;
#pragma unroll
    for (int k = 0; k < 8; k++) b[k] = mt[i0 + 8 + k];
#pragma unroll
    for (int k = 0; k < 8; k++) {
      prev = step2(prev, a[k], i0 + k);
      out[i0 + k] = prev;
    }
#pragma unroll
    for (int k = 0; k < 8; k++) a[k] = mt[i0 + 16 + k];
#pragma unroll
    for (int k = 0; k < 8; k++) {
      prev = step2(prev, b[k], i0 + 8 + k);
      out[i0 + 8 + k] = prev;
    }
  }
#pragma unroll
  for (int k = 0; k < 8; k++) {
    prev = step2(prev, a[k], 610 + k);
    out[610 + k] = prev;
  }
#pragma unroll
  for (int k = 0; k < 6; k++) {
    prev = step2(prev, mt[618 + k], 618 + k);
    out[618 + k] = prev;
  }
  out[1] = step2(prev, mt[1], 1);
  out[0] = 0x80000000u;
}

// init_by_array without per-thread storage of the first loop's output: the
// second loop reads first-loop word i exactly once, at position i, in
// order -- except word 1, which the first loop's 624th iteration rewrites
// and the second loop reads first.  So pass 1 runs the first loop for its
// last word and the final word 1 only; pass 2 regenerates the first loop
// (chain a, the same table reads) in lockstep with the second loop
// (chain b), two independent dependency chains, and streams the final
// state to `out` (shared or global).  Same latency as mt_seed_impl, no
// 2.5 KB working row.
template <int KLEN>
__device__ __forceinline__ void mt_seed_stream_impl(uint32_t k0, uint32_t k1, uint32_t* out) {
  const uint32_t* T = kTlInitGenrand;
  const uint32_t v1 = seed_step1<KLEN>(T[0], T[1], 1, k0, k1);
  uint32_t prev = v1;
  uint32_t a[8], b[8];
#pragma unroll
  for (int k = 0; k < 8; k++) a[k] = T[2 + k];
  for (int g = 0; g < 76; g += 2) {  // i = 2..609
    const int i0 = 2 + 8 * g;
#pragma unroll
    for (int k = 0; k < 8; k++) b[k] = T[i0 + 8 + k];
#pragma unroll
    for (int k = 0; k < 8; k++) prev = seed_step1<KLEN>(prev, a[k], i0 + k, k0, k1);
#pragma unroll
    for (int k = 0; k < 8; k++) a[k] = T[i0 + 16 + k];
#pragma unroll
    for (int k = 0; k < 8; k++) prev = seed_step1<KLEN>(prev, b[k], i0 + 8 + k, k0, k1);
  }
#pragma unroll
  for (int k = 0; k < 8; k++) prev = seed_step1<KLEN>(prev, a[k], 610 + k, k0, k1);
#pragma unroll
  for (int k = 0; k < 6; k++) prev = seed_step1<KLEN>(prev, T[618 + k], 618 + k, k0, k1);
  // mt[0] = mt[623]; 624th iteration: i = 1 (old word = v1), j = 623 % klen
  const uint32_t m1 = seed_step1<KLEN>(prev, v1, kMtN, k0, k1);
  auto step2 = [](uint32_t pv, uint32_t old, int i) {
    return (old ^ ((pv ^ (pv >> 30)) * 1566083941u)) - (uint32_t)i;
  };
  uint32_t pa = v1, pb = m1;
#pragma unroll
  for (int k = 0; k < 8; k++) a[k] = T[2 + k];
  for (int g = 0; g < 76; g += 2) {
    const int i0 = 2 + 8 * g;
#pragma unroll
    for (int k = 0; k < 8; k++) b[k] = T[i0 + 8 + k];
#pragma unroll
    for (int k = 0; k < 8; k++) {
      pa = seed_step1<KLEN>(pa, a[k], i0 + k, k0, k1);
      pb = step2(pb, pa, i0 + k);
      out[i0 + k] = pb;
    }
#pragma unroll
    for (int k = 0; k < 8; k++) a[k] = T[i0 + 16 + k];
#pragma unroll
    for (int k = 0; k < 8; k++) {
      pa = seed_step1<KLEN>(pa, b[k], i0 + 8 + k, k0, k1);
      pb = step2(pb, pa, i0 + 8 + k);
      out[i0 + 8 + k] = pb;
    }
  }
#pragma unroll
  for (int k = 0; k < 8; k++) {
    pa = seed_step1<KLEN>(pa, a[k], 610 + k, k0, k1);
    pb = step2(pb, pa, 610 + k);
    out[610 + k] = pb;
  }
#pragma unroll
  for (int k = 0; k < 6; k++) {
    pa = seed_step1<KLEN>(pa, T[618 + k], 618 + k, k0, k1);
    pb = step2(pb, pa, 618 + k);
    out[618 + k] = pb;
  }
  out[1] = step2(pb, m1, 1);  // wrap: mt[0] = mt[623], i = 1 reads the final word 1
  out[0] = 0x80000000u;
}

__device__ __noinline__ void mt_seed_lane_stream(int64_t seed, uint32_t* out) {
  const uint64_t n = seed < 0 ? (uint64_t)0 - (uint64_t)seed : (uint64_t)seed;
  const uint32_t k0 = (uint32_t)n, k1 = (uint32_t)(n >> 32);
  if (k1) mt_seed_stream_impl<2>(k0, k1, out);
  else mt_seed_stream_impl<1>(k0, 0u, out);
}

// seed one state; the result lands in `out` (== mt for an in-place seed)
__device__ __noinline__ void mt_seed_lane(uint32_t* mt, int64_t seed, uint32_t* out = nullptr) {
  const uint64_t n = seed < 0 ? (uint64_t)0 - (uint64_t)seed : (uint64_t)seed;
  const uint32_t k0 = (uint32_t)n, k1 = (uint32_t)(n >> 32);
  if (!out) out = mt;
  if (k1) mt_seed_impl<2>(mt, k0, k1, out);
  else mt_seed_impl<1>(mt, k0, 0u, out);
}

// Serial reader over a freshly seeded MT state for one thread (script
// sampling).  Words are regenerated lazily in order, in place: word i of a
// block reads mt[i+1] (old) and mt[i+397] (old) or mt[i-227] (already new),
// exactly the values CPython's block regeneration reads.
struct MtLane {
  uint32_t* mt;
  int idx;  // next word of the current block (0 right after seeding)
  int pre;  // words [0, pre) of the first block are already regenerated in place
  // their tempered values at mt[tw + i] (prepare_block_warp), tw = 0: none.
  // An offset, not a pointer: a null test on a shared-memory pointer costs an
  // S2R (shared window) per word in the serial sampler
  int tw = 0;
  // regenerate words [0, n) (n <= 227: they read old words only) with
  // independent loads, so the serial sampler only tempers them
  __device__ __forceinline__ void prepare(int n) {
    for (int i0 = 0; i0 < n; i0 += 8) {
      uint32_t v[8];
#pragma unroll
      for (int k = 0; k < 8; k++) v[k] = mt_mix(mt[i0 + k], mt[i0 + k + 1], mt[i0 + k + kMtM]);
#pragma unroll
      for (int k = 0; k < 8; k++) mt[i0 + k] = v[k];
    }
    pre = n;
  }
  __device__ __forceinline__ uint32_t genrand() {
    if (idx < pre) {
      const uint32_t x = tw ? mt[tw + idx] : mt_temper(mt[idx]);
      idx++;
      return x;
    }
    if (pre) {  // first block prefix consumed; continue lazily
      pre = 0;
      if (idx == kMtN) idx = 0;  // the whole first block was prepared
    }
    const int i = idx;
    const int i1 = i + 1 == kMtN ? 0 : i + 1;
    const int src = i < kMtN - kMtM ? i + kMtM : i - (kMtN - kMtM);
    const uint32_t v = mt_mix(mt[i], mt[i1], mt[src]);
    mt[i] = v;
    idx = i1;
    return mt_temper(v);
  }
  // the same for the whole first block (words [0, 624)), by the 32 lanes of
  // a warp in CPython's three dependency phases (0..226 read old words only,
  // 227..453 read new words 0..226, 454..623 read new 227..396 and word 0);
  // every lane of the warp calls it, then one lane samples with pre = 624;
  // mt[tw_off + i] receives the tempered words (the serial sampler only
  // loads them), tw_off > 0
  __device__ __forceinline__ void prepare_block_warp(int tw_off) {
    uint32_t* tout = mt + tw_off;
    const int lane = lane_id();
    uint32_t v[8];
#pragma unroll
    for (int k = 0; k < 8; k++) {
      const int i = lane + 32 * k;
      if (i < kMtN - kMtM) v[k] = mt_mix(mt[i], mt[i + 1], mt[i + kMtM]);
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 8; k++) {
      const int i = lane + 32 * k;
      if (i < kMtN - kMtM) { mt[i] = v[k]; tout[i] = mt_temper(v[k]); }
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 8; k++) {
      const int i = kMtN - kMtM + lane + 32 * k;
      if (i < 2 * (kMtN - kMtM)) v[k] = mt_mix(mt[i], mt[i + 1], mt[i - (kMtN - kMtM)]);
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 8; k++) {
      const int i = kMtN - kMtM + lane + 32 * k;
      if (i < 2 * (kMtN - kMtM)) { mt[i] = v[k]; tout[i] = mt_temper(v[k]); }
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 6; k++) {
      const int i = 2 * (kMtN - kMtM) + lane + 32 * k;
      if (i < kMtN) v[k] = mt_mix(mt[i], mt[i + 1 == kMtN ? 0 : i + 1], mt[i - (kMtN - kMtM)]);
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 6; k++) {
      const int i = 2 * (kMtN - kMtM) + lane + 32 * k;
      if (i < kMtN) { mt[i] = v[k]; tout[i] = mt_temper(v[k]); }
    }
    __syncwarp();
    idx = 0;
    pre = kMtN;
    tw = tw_off;
  }
  // the first n <= 227 words only (they read old words), by the 32 lanes of a
  // warp, tempered copies at mt[tw_off + i]; the lone sampler continues
  // lazily from word n (the words it usually needs are all in the prefix)
  template <int N>
  __device__ __forceinline__ void prepare_prefix_warp(int tw_off) {
    static_assert(N % 32 == 0 && N <= kMtN - kMtM, "prefix of old-only words");
    const int lane = lane_id();
    uint32_t v[N / 32];
#pragma unroll
    for (int k = 0; k < N / 32; k++) {
      const int i = lane + 32 * k;
      v[k] = mt_mix(mt[i], mt[i + 1], mt[i + kMtM]);
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < N / 32; k++) {
      const int i = lane + 32 * k;
      mt[i] = v[k];
      mt[tw_off + i] = mt_temper(v[k]);
    }
    __syncwarp();
    idx = 0;
    pre = N;
    tw = tw_off;
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

// random() = k * 2^-53 for the 53-bit integer k; the exact conversion is
// followed by an exponent decrement instead of a multiply (k >= 1 keeps the
// result normal; k == 0 gives 0.0)
__device__ __forceinline__ double rand53(uint32_t w0, uint32_t w1) {
  const uint64_t k = ((uint64_t)(w0 >> 5) << 26) | (w1 >> 6);
  const double d = __ull2double_rn(k);
  const double r = __longlong_as_double(__double_as_longlong(d) - (53ll << 52));
  return k ? r : 0.0;
}

// a + span * random() for the 53-bit k of words (w0, w1), given span_s =
// span * 2^-53: span * (k * 2^-53) and span_s * k are the same real number,
// so the rounded product (and sum) equal CPython's uniform(a, a + span)
__device__ __forceinline__ double uniform_k53(double a, double span_s, uint32_t w0, uint32_t w1) {
  const uint32_t hi = w0 >> 11;
  const uint32_t lo = __funnelshift_r(w1, w0 >> 5, 6);  // ((w0 >> 5) << 26) | (w1 >> 6)
  const double k = __ull2double_rn(((uint64_t)hi << 32) | lo);
  return __dadd_rn(a, __dmul_rn(span_s, k));
}

// cp.async (global -> shared, no registers in flight)
__device__ __forceinline__ void cp_async4(uint32_t* sdst, const uint32_t* gsrc) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// Lib/random.py uniform: a + (b - a) * random(), no FMA
// the same with b - a supplied (constant spans are folded at compile time
// with the identical IEEE round-to-nearest subtraction CPython performs)
__device__ __forceinline__ double uniform_span(double a, double span, double r) {
  return __dadd_rn(a, __dmul_rn(span, r));
}
#define TL_UNIFORM(a, b, r) ::tl::uniform_span((a), (double)(b) - (double)(a), (r))

__device__ __forceinline__ double uniform_rn(double a, double b, double r) {
  return __dadd_rn(a, __dmul_rn(__dsub_rn(b, a), r));
}

// warp inclusive scan (int)
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

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
