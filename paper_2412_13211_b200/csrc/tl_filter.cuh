// tl_filter.cuh -- K5: rule-based dataset filter (filter_labels selection).
//
// Reference: /root/reference/pkg/src/trajlab/pipeline.py:276-338.
// filter_labels fills each (quota key, subtask) pool by repeatedly taking
// the head of the allow-rule bucket with the smallest (taken/weight, rule
// position).  Every bucket's key sequence j/w (j = 0, 1, ...) is increasing,
// so that greedy merge emits items in global (j/w, pos) order and the
// selection is exactly the items whose merged rank is < quota.  Hence:
//   1. j = stable rank of each label inside its bucket (episode order),
//   2. per pool, c_b = #items of bucket b with merged rank < quota
//      (binary searches on the bucket counts only; no per-label sort),
//   3. selected = j < c_b.
// Keys use IEEE f64 division exactly like `taken[i] / rule.weight`.
#pragma once
#include "tl_common.cuh"

namespace tl {

constexpr int kFilterTile = 2048;

// per-tile bucket counts: tile_cnt[tile * B + b]
__global__ void __launch_bounds__(256)
    k_filter_hist(const int32_t* __restrict__ bucket, int64_t n, int B,
                  int32_t* __restrict__ tile_cnt) {
  extern __shared__ int32_t h[];
  for (int i = threadIdx.x; i < B; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const int64_t a = (int64_t)blockIdx.x * kFilterTile;
  const int64_t b = min(n, a + kFilterTile);
  for (int64_t i = a + threadIdx.x; i < b; i += blockDim.x) {
    const int k = bucket[i];
    if (k >= 0) atomicAdd(&h[k], 1);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < B; i += blockDim.x) tile_cnt[(int64_t)blockIdx.x * B + i] = h[i];
}

// column-wise exclusive scan over tiles; bucket totals -> cnt[b]
__global__ void k_filter_colscan(int32_t* __restrict__ tile_cnt, int n_tiles, int B,
                                 int64_t* __restrict__ cnt) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  int64_t run = 0;
  for (int t = 0; t < n_tiles; t++) {
    const int64_t idx = (int64_t)t * B + b;
    const int32_t v = tile_cnt[idx];
    tile_cnt[idx] = (int32_t)run;
    run += v;
  }
  cnt[b] = run;
}

// number of j' in [0, n) with (j'/w, pos') < (K, P)
__device__ __forceinline__ int64_t count_below(int64_t n, double w, int pos, double K, int P) {
  int64_t lo = 0, hi = n;  // first j' not below
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    const double k = __ddiv_rn((double)mid, w);
    const bool below = k < K || (k == K && pos < P);
    if (below) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// one thread per pool: c_b for the pool's buckets [b0, b1)
__global__ void k_filter_pool(const int32_t* __restrict__ pool_b0, int n_pools,
                              const double* __restrict__ w, const int64_t* __restrict__ cnt,
                              int64_t quota, int64_t* __restrict__ take,
                              int64_t* __restrict__ pool_selected) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_pools) return;
  const int b0 = pool_b0[p], b1 = pool_b0[p + 1];
  int64_t total = 0;
  for (int b = b0; b < b1; b++) {
    const int pos = b - b0;
    // largest prefix of bucket b whose merged ranks are all < quota
    int64_t lo = 0, hi = cnt[b];
    while (lo < hi) {
      const int64_t j = (lo + hi) >> 1;  // is item j selected?
      const double K = __ddiv_rn((double)j, w[b]);
      int64_t rank = j;                  // earlier items of the same bucket
      for (int b2 = b0; b2 < b1; b2++)
        if (b2 != b) rank += count_below(cnt[b2], w[b2], b2 - b0, K, pos);
      if (rank < quota) lo = j + 1; else hi = j;
    }
    take[b] = lo;
    total += lo;
  }
  pool_selected[p] = total;
}

// stable in-bucket rank per label (one warp per tile, labels in order)
__global__ void __launch_bounds__(32)
    k_filter_select(const int32_t* __restrict__ bucket, int64_t n, int B,
                    const int32_t* __restrict__ tile_off, const int64_t* __restrict__ take,
                    uint8_t* __restrict__ selected) {
  extern __shared__ int32_t run[];
  for (int i = threadIdx.x; i < B; i += 32) run[i] = tile_off[(int64_t)blockIdx.x * B + i];
  __syncwarp();
  const int lane = lane_id();
  const int64_t a = (int64_t)blockIdx.x * kFilterTile;
  const int64_t e = min(n, a + kFilterTile);
  for (int64_t i0 = a; i0 < e; i0 += 32) {
    const int64_t i = i0 + lane;
    const int k = i < e ? bucket[i] : -1;
    const unsigned peers = __match_any_sync(kFull, k);
    const int before = __popc(peers & ((1u << lane) - 1u));
    int rank = 0;
    if (k >= 0) rank = run[k] + before;
    __syncwarp();
    if (k >= 0 && before == 0) run[k] += __popc(peers);
    __syncwarp();
    if (i < e) selected[i] = (k >= 0 && rank < take[k]) ? 1 : 0;
  }
}

}  // namespace tl
