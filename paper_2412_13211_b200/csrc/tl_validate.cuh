// tl_validate.cuh -- structural validation of a record batch on the GPU
// (trajlab.model.validate, model.py:232-281, the per-record invariants).
//
// The reference walks one trajectory's records in Python and appends a
// message per violated invariant.  Here the invariants are per-record bit
// codes computed over the structure-of-arrays planes, one warp per episode,
// 32 records per warp iteration; the only cross-record dependency
// ("cumulative force decreased", model.py:263-265: record i against record
// i-1's cum_robot_force, whatever that value was) is a __shfl_up with the
// previous chunk's last value carried in a register.  The host renders the
// reference's messages from the codes (paper_2412_13211_b200/model.py).
//
// Per record r (vflags[r], TL_VF_* in include/trajlab_b200.h):
//   T_MISMATCH    t[r] != index in episode           (model.py:256-257)
//   CUM_INVALID   cum < 0 or NaN                      (model.py:261-262)
//   CUM_DECREASED not CUM_INVALID and i > 0 and cum < previous cum (:263-264)
//   DEE_INVALID   dist_ee_rest < 0 or NaN             (:266-267)
//   DOG_NEGATIVE  dist_obj_goal not NaN and < 0       (:268-269)
//   FET_NEGATIVE  force_ee_target not NaN and < 0     (:270-271)
//   ART_RANGE     articulated, art_q not NaN, not qmin <= art_q <= qmax
//                 (f64 compare, :272-274; a warning, not an error)
// Binary32 planes compare in f32 against 0 and against each other (exact:
// widening to f64 preserves order); art_q is widened to f64 against the
// f64 bounds, as CPython compares the float read back from a TRJL file.
//
// Algorithmic traffic: 5 planes x sizeof(T) read + 1 B written per record
// (20 B + 1 B at f32) -> HBM-bound.
#pragma once
#include "tl_common.cuh"

namespace tl {

constexpr int kValidateWarps = 8;

template <typename T>
__device__ __forceinline__ bool v_isnan(T x) { return x != x; }

template <typename T>
__global__ void __launch_bounds__(kValidateWarps * 32)
    k_validate(tl_records R, int n_env, const tl_vbounds* __restrict__ vb,
               const int64_t* __restrict__ t_plane, uint8_t* __restrict__ vflags,
               tl_vsummary* __restrict__ vsum) {
  const int warp = threadIdx.x >> 5, lane = lane_id();
  const T* __restrict__ P = reinterpret_cast<const T*>(R.planes);
  const int64_t S = R.plane_stride;
  const int base = 2 * R.dof;
  const T* __restrict__ dee = P + (base + 4) * S;
  const T* __restrict__ dog = P + (base + 5) * S;
  const T* __restrict__ fet = P + (base + 6) * S;
  const T* __restrict__ cum = P + (base + 7) * S;
  const T* __restrict__ art = P + (base + 8) * S;
  for (int e = blockIdx.x * kValidateWarps + warp; e < n_env; e += gridDim.x * kValidateWarps) {
    const int64_t rs = R.rec_start[e];
    const int n = R.n_rec[e];
    const tl_vbounds b = vb[e];
    T carry = T(0);  // cum of the previous chunk's last record
    int n_err = 0, n_warn = 0, first = -1;
    for (int i0 = 0; i0 < n; i0 += 32) {
      const int i = i0 + lane;
      const bool live = i < n;
      const int64_t r = rs + i;
      uint32_t f = 0;
      T c = T(0);
      if (live) {
        c = __ldcs(cum + r);
        const T d = __ldcs(dee + r), g = __ldcs(dog + r), q = __ldcs(fet + r);
        if (t_plane && t_plane[r] != (int64_t)i) f |= TL_VF_T_MISMATCH;
        if (c < T(0) || v_isnan(c)) f |= TL_VF_CUM_INVALID;
        if (d < T(0) || v_isnan(d)) f |= TL_VF_DEE_INVALID;
        if (!v_isnan(g) && g < T(0)) f |= TL_VF_DOG_NEGATIVE;
        if (!v_isnan(q) && q < T(0)) f |= TL_VF_FET_NEGATIVE;
        if (b.has_art) {
          const double a = (double)__ldcs(art + r);
          if (!v_isnan(a) && !(b.art_qmin <= a && a <= b.art_qmax)) f |= TL_VF_ART_RANGE;
        }
      }
      T prev = __shfl_up_sync(kFull, c, 1);
      if (lane == 0) prev = carry;
      if (live && i > 0 && !(f & TL_VF_CUM_INVALID) && c < prev) f |= TL_VF_CUM_DECREASED;
      carry = __shfl_sync(kFull, c, 31);
      if (live && vflags) vflags[r] = (uint8_t)f;
      const unsigned any = __ballot_sync(kFull, f != 0);
      n_err += __popc(__ballot_sync(kFull, (f & ~(uint32_t)TL_VF_ART_RANGE) != 0));
      n_warn += __popc(__ballot_sync(kFull, (f & TL_VF_ART_RANGE) != 0));
      if (first < 0 && any) first = i0 + __ffs(any) - 1;
    }
    if (lane == 0) {
      tl_vsummary s;
      s.n_error_records = n_err;
      s.n_warning_records = n_warn;
      s.first_flagged = first;
      s.too_short = n < 2;  // model.py:252-253
      vsum[e] = s;
    }
  }
}

}  // namespace tl
