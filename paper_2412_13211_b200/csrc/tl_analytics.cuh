// tl_analytics.cuh -- device counting behind the statistics tables and the
// chained-episode completion curves.
//
// Reference (paths under /root/reference/pkg/src/trajlab/):
//   analytics.py:121-160  mode_table: per-group counts of every mode,
//                         success_once and success_at_end (SoR/SaeR/FR)
//   analytics.py:279-298  progressive_completion: per-slot count of chains
//                         whose every non-auto slot so far succeeded
// The host turns the integer counts into the reference's fractions and
// renderings (analytics.py), so only exact integer work runs here.
#pragma once
#include "tl_common.cuh"

namespace tl {

constexpr int kCountCols = 42;  // 39 modes, success_once, success_at_end, valid labels

// counts[g][c] += 1 for every valid label (status 0) of group g.
// Block-private shared histogram when it fits, global atomics otherwise.
__global__ void k_group_counts(const tl_label* __restrict__ labels,
                               const int32_t* __restrict__ group, int64_t n, int n_groups,
                               unsigned long long* __restrict__ counts, int use_smem) {
  extern __shared__ unsigned int gc_hist[];
  unsigned int* h = gc_hist;
  const int cells = n_groups * kCountCols;
  if (use_smem) {
    for (int i = threadIdx.x; i < cells; i += blockDim.x) h[i] = 0;
    __syncthreads();
  }
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const tl_label L = labels[i];
    if (L.status != 0 || L.mode >= 39) continue;
    const int g = group ? group[i] : 0;
    if (g < 0 || g >= n_groups) continue;
    const int b = g * kCountCols;
    if (use_smem) {
      atomicAdd(&h[b + L.mode], 1u);
      if (L.flags & 1) atomicAdd(&h[b + 39], 1u);
      if (L.flags & 2) atomicAdd(&h[b + 40], 1u);
      atomicAdd(&h[b + 41], 1u);
    } else {
      atomicAdd(&counts[b + L.mode], 1ull);
      if (L.flags & 1) atomicAdd(&counts[b + 39], 1ull);
      if (L.flags & 2) atomicAdd(&counts[b + 40], 1ull);
      atomicAdd(&counts[b + 41], 1ull);
    }
  }
  if (use_smem) {
    __syncthreads();
    for (int i = threadIdx.x; i < cells; i += blockDim.x)
      if (h[i]) atomicAdd(&counts[i], (unsigned long long)h[i]);
  }
}

// One thread per chain: alive &= success_once of each bound slot
// (slot_label >= 0; -1 = auto-success slot, e.g. Nav); per-slot alive
// counts reduced by warp ballot.  n_slots <= 64.
__global__ void k_chain_alive(const tl_label* __restrict__ labels,
                              const int64_t* __restrict__ slot_label, int64_t n_chain,
                              int n_slots, unsigned long long* __restrict__ alive) {
  __shared__ unsigned int h[64];
  for (int i = threadIdx.x; i < 64; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const int lane = lane_id();
  for (int64_t c0 = (int64_t)blockIdx.x * blockDim.x; c0 < n_chain;
       c0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = c0 + threadIdx.x;
    const bool valid = c < n_chain;
    bool ok = valid;
    for (int k = 0; k < n_slots; k++) {
      if (ok) {
        const int64_t li = slot_label[c * n_slots + k];
        if (li >= 0) {
          const tl_label L = labels[li];
          ok = L.status == 0 && (L.flags & 1);
        }
      }
      const unsigned b = __ballot_sync(kFull, ok);
      if (lane == 0 && b) atomicAdd(&h[k], (unsigned)__popc(b));
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < n_slots; k += blockDim.x)
    if (h[k]) atomicAdd(&alive[k], (unsigned long long)h[k]);
}

// filter_labels bucket encoding on the device (pipeline.py:276-304): label
// i of subtask s with quota key k goes to bucket pool_b0[pool[k*4+s]] +
// rule_lut[s*39 + mode] (first allow rule of s containing its mode), or
// -1 when no rule matches / the pool does not exist / the label is invalid.
__global__ void k_filter_buckets(const tl_label* __restrict__ labels,
                                 const int32_t* __restrict__ key, int64_t n,
                                 const int8_t* __restrict__ rule_lut,
                                 const int32_t* __restrict__ pool,
                                 const int32_t* __restrict__ pool_b0, int n_keys,
                                 int32_t* __restrict__ bucket) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const tl_label L = labels[i];
    int b = -1;
    const int k = key[i];
    if (L.status == 0 && L.mode < 39 && L.subtask < 4 && k >= 0 && k < n_keys) {
      const int r = rule_lut[L.subtask * 39 + L.mode];
      const int pl = pool[k * 4 + L.subtask];
      if (r >= 0 && pl >= 0) b = pool_b0[pl] + r;
    }
    bucket[i] = b;
  }
}

}  // namespace tl
