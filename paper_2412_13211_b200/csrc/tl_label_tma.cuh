// tl_label_tma.cuh -- the label kernel (K1) with its record planes staged
// through shared memory by bulk async copies (TMA, cp.async.bulk) one chunk
// ahead, so HBM reads overlap the predicate / edge / fold arithmetic.
//
// Same semantics as k_label (tl_label.cuh; reference predicates.py:16-99,
// events.py:94-193, modes.py:235-253).  Mapping: one warp per episode,
// chunks of 128 records (4 per lane).  Lane 0 of each warp arms an mbarrier
// with the chunk's byte count and issues one bulk copy per plane the
// subtask's predicates read (Pick 2*dof+6, Place 2*dof+7, Open/Close
// 2*dof+8 planes of 512 B) into one of two per-warp buffers; while the
// warp folds chunk k, chunk k+1 (or the next episode's chunk 0) is in
// flight.  Episodes that are not 16-byte aligned f32 with a zero rest
// posture take the one-record-per-lane path (label_scalar).
#pragma once
#include "tl_label.cuh"

namespace tl {

constexpr int kTmaChunk = 128;

template <int DOFMAX>
struct LabelTmaSmem {
  static constexpr int kWarps = DOFMAX <= 7 ? 8 : 4;  // 180 KB / 164 KB of buffers
  static constexpr int kPlanes = 2 * DOFMAX + 8;
  float buf[kWarps][2][kPlanes][kTmaChunk];
  tl_cset cs[kWarps];
  unsigned long long bar[kWarps][2];
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "TL_MBAR_WAIT%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra TL_MBAR_WAIT%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// global -> shared bulk copy (TMA), completion counted on the mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

struct TmaEp {
  int64_t rs;
  int n, ci, sub, vec;
};

template <int DOFMAX>
__global__ void __launch_bounds__(LabelTmaSmem<DOFMAX>::kWarps * 32)
    k_label_tma(tl_records R, int n_env, const int32_t* __restrict__ env_cset,
                const tl_cset* __restrict__ csets, tl_rules rules,
                uint8_t* __restrict__ step_mask, uint8_t* __restrict__ step_success,
                tl_label* __restrict__ labels) {
  using SM = LabelTmaSmem<DOFMAX>;
  constexpr int kTmaWarps = SM::kWarps;
  extern __shared__ __align__(128) unsigned char lt_smem_raw[];
  SM& sm = *reinterpret_cast<SM*>(lt_smem_raw);
  const int warp = threadIdx.x >> 5, lane = lane_id();
  const float* __restrict__ P = reinterpret_cast<const float*>(R.planes);
  const int64_t stride = R.plane_stride;
  const int dof = R.dof, f0 = 2 * dof;
  const bool base_ok = (stride & 3) == 0 && (reinterpret_cast<uintptr_t>(R.planes) & 15) == 0 &&
                       (reinterpret_cast<uintptr_t>(R.grasped) & 3) == 0;
  unsigned long long* bar = sm.bar[warp];
  if (lane == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncwarp();
  uint32_t phase[2] = {0u, 0u};
  const int wstride = gridDim.x * kTmaWarps;

  auto ep_info = [&](int e) {
    TmaEp x;
    x.rs = R.rec_start[e];
    x.n = R.n_rec[e];
    x.ci = env_cset[e];
    const tl_cset* cp = &csets[x.ci];
    x.sub = cp->subtask;
    x.vec = base_ok && cp->rest_zero && (x.rs & 3) == 0 &&
            x.rs + (((int64_t)x.n + 3) & ~(int64_t)3) <= stride;
    return x;
  };
  // lane 0: arm buffer b and copy chunk [t0, t0+64) of episode x into it
  auto issue = [&](const TmaEp& x, int t0, int b) {
    if (lane == 0) {
      const int cnt = min(kTmaChunk, x.n - t0);
      const uint32_t sz = (uint32_t)((cnt + 3) & ~3) * 4u;
      const int np = tma_nplanes(x.sub, dof);
      mbar_expect_tx(&bar[b], sz * (uint32_t)np);
      for (int p = 0; p < np; p++)
        bulk_g2s(&sm.buf[warp][b][p][0], P + (int64_t)tma_plane(x.sub, dof, p) * stride + x.rs + t0,
                 sz, &bar[b]);
    }
  };
  auto grasped4 = [&](const TmaEp& x, int t0) -> uint32_t {
    const int tb = t0 + 4 * lane;
    if (x.sub > TL_PLACE || tb >= x.n) return 0u;
    return __ldg(reinterpret_cast<const unsigned int*>(R.grasped + x.rs + tb));
  };

  int e = blockIdx.x * kTmaWarps + warp;
  TmaEp x;
  if (e < n_env) x = ep_info(e);
  bool pre = false;  // chunk 0 of episode e already in flight in buffer cur
  uint32_t g_next = 0;
  int cur = 0;
  for (; e < n_env; e += wstride) {
    stage_cset(&sm.cs[warp], &csets[x.ci]);
    const tl_cset& c = sm.cs[warp];
    const int64_t rs = x.rs;
    const int n = x.n;
    LState S;
    lstate_init(S);
    if (n < 2 && lane == 0) {  // events.py:96-97
      tl_label L;
      L.status = TL_ERR_TOO_SHORT; L.n_events = 0; L.err_index = -1;
      L.subtask = (uint8_t)c.subtask; L.mode = 255; L.flags = 0; L.pad = 0;
      L.d0 = __longlong_as_double(0x7ff8000000000000ll);
      labels[e] = L;
    }
    if (!x.vec || n < 1) {
      if (n > 0 && (n >= 2 || step_success)) {
        double d0 = 0.0, sc_d = 0.0;
        float sc_ru = 0.f;
        if (c.subtask == TL_PLACE) d0 = (double)P[(f0 + 5) * stride + rs];
        if (c.subtask == TL_CLOSE) close_cut(c, (double)P[(f0 + 8) * stride + rs], sc_ru, sc_d);
        label_scalar<float, DOFMAX>(R, c, rs, n, sc_ru, sc_d, S, step_mask, step_success);
        if (n >= 2) finish_label(c, S, d0, rules, &labels[e]);
      }
      if (e + wstride < n_env) x = ep_info(e + wstride);
      pre = false;
      continue;
    }
    if (!pre) {
      issue(x, 0, cur);
      g_next = grasped4(x, 0);
    }
    const int sub = c.subtask;
    double d0 = 0.0, sc_d = 0.0;
    float sc_ru = 0.f;
    TmaEp nx;
    nx.vec = 0;
    for (int t0 = 0; t0 < n; t0 += kTmaChunk) {
      const uint32_t g4 = g_next;
      // prefetch the next chunk: this episode's, or the next episode's first
      if (t0 + kTmaChunk < n) {
        issue(x, t0 + kTmaChunk, cur ^ 1);
        g_next = grasped4(x, t0 + kTmaChunk);
      } else {
        pre = false;
        if (e + wstride < n_env) {
          nx = ep_info(e + wstride);
          if (nx.vec && nx.n > 0) {
            issue(nx, 0, cur ^ 1);
            g_next = grasped4(nx, 0);
            pre = true;
          }
        }
      }
      mbar_wait(&bar[cur], phase[cur]);
      phase[cur] ^= 1u;
      const float(*B)[kTmaChunk] = sm.buf[warp][cur];
      if (t0 == 0) {
        if (sub == TL_PLACE) d0 = (double)B[f0 + 6][0];
        if (sub == TL_CLOSE) close_cut(c, (double)B[f0 + 7][0], sc_ru, sc_d);
      }
      const int tb = t0 + 4 * lane;
      auto get = [&](int p) { return *reinterpret_cast<const float4*>(&B[p][4 * lane]); };
      float4 mq, mqd;
#pragma unroll
      for (int i = 0; i < DOFMAX; i++) {
        if (i < dof) {
          const float4 q = get(i), qd = get(dof + i);
          if (i == 0) {
            mq = make_float4(fabsf(q.x), fabsf(q.y), fabsf(q.z), fabsf(q.w));
            mqd = make_float4(fabsf(qd.x), fabsf(qd.y), fabsf(qd.z), fabsf(qd.w));
          } else {
            mq = make_float4(pymax_step(mq.x, fabsf(q.x)), pymax_step(mq.y, fabsf(q.y)),
                             pymax_step(mq.z, fabsf(q.z)), pymax_step(mq.w, fabsf(q.w)));
            mqd = make_float4(pymax_step(mqd.x, fabsf(qd.x)), pymax_step(mqd.y, fabsf(qd.y)),
                              pymax_step(mqd.z, fabsf(qd.z)), pymax_step(mqd.w, fabsf(qd.w)));
          }
        }
      }
      const float4 vx = get(f0), vy = get(f0 + 1), om = get(f0 + 2), der = get(f0 + 3),
                   cum = get(f0 + 4), x5 = get(f0 + 5);
      const float4 x6 = sub == TL_PICK ? make_float4(0.f, 0.f, 0.f, 0.f) : get(f0 + 6);
      const float4 x7 = sub >= TL_OPEN ? get(f0 + 7) : make_float4(0.f, 0.f, 0.f, 0.f);
      __syncwarp();  // every lane has read buffer `cur` before it is refilled
      uint32_t ind[4], err[4], m[4];
#pragma unroll
      for (int j = 0; j < 4; j++) {
        ind[j] = 0;
        err[j] = 0;
        if (tb + j < n) {
          RecV<float> v;
          v.der = f4get(der, j);
          v.cum = f4get(cum, j);
          v.vx = f4get(vx, j);
          v.vy = f4get(vy, j);
          v.om = f4get(om, j);
          v.qdm = f4get(mqd, j);
          v.jm = f4get(mq, j);
          v.jm_d = 0.0;
          v.tor = 0.f; v.dist = 0.f; v.force = 0.f; v.art = 0.f; v.g = false;
          if (sub == TL_PICK) {
            v.force = f4get(x5, j);
            v.g = (g4 >> (8 * j)) & 0xffu;
          } else if (sub == TL_PLACE) {
            v.tor = f4get(x5, j);
            v.dist = f4get(x6, j);
            v.g = (g4 >> (8 * j)) & 0xffu;
          } else {
            v.tor = f4get(x5, j);
            v.force = f4get(x6, j);
            v.art = f4get(x7, j);
          }
          record_bits(c, v, sc_ru, sc_d, ind[j], err[j]);
          if (step_success)
            step_success[rs + tb + j] = (err[j] & ERR_SUCC) ? 2 : ((ind[j] & IND_SUCCESS) ? 1 : 0);
        }
      }
      uint32_t prev = __shfl_up_sync(kFull, ind[3], 1);
      if (lane == 0) prev = S.prev_ind;
      uint32_t cnt = 0, eor = 0;
#pragma unroll
      for (int j = 0; j < 4; j++) {
        const bool ok = tb + j < n && tb + j > 0;
        m[j] = ok ? edge_mask(sub, j == 0 ? prev : ind[j - 1], ind[j]) : 0u;
        cnt += __popc(m[j]);
        eor |= (tb + j < n) ? err[j] : 0u;
      }
      if (step_mask && tb < n) {
        if (tb + 3 < n) {
          *reinterpret_cast<unsigned int*>(step_mask + rs + tb) =
              m[0] | (m[1] << 8) | (m[2] << 16) | (m[3] << 24);
        } else {
          for (int j = 0; j < 4 && tb + j < n; j++) step_mask[rs + tb + j] = (uint8_t)m[j];
        }
      }
      const int incl = warp_incl_scan((int)cnt);
      const int excl = incl - (int)cnt;
#pragma unroll
      for (int k = 0; k < 7; k++) {
        int pos = -1, before = 0;
#pragma unroll
        for (int j = 0; j < 4; j++) {
          if ((m[j] >> k) & 1u) pos = before + __popc(m[j] & ((1u << k) - 1u));
          before += __popc(m[j]);
        }
        const unsigned bal = __ballot_sync(kFull, pos >= 0);
        if (bal) {
          const int L = 31 - __clz(bal);
          S.last[k] = S.size + __shfl_sync(kFull, excl + pos, L);
        }
      }
      S.size += __shfl_sync(kFull, incl, 31);
      S.err_any |= __reduce_or_sync(kFull, eor);
      S.prev_ind = __shfl_sync(kFull, ind[3], 31);  // only a full chunk carries on
      cur ^= 1;
    }
    if (n >= 2) finish_label(c, S, d0, rules, &labels[e]);
    if (e + wstride < n_env) x = pre ? nx : ep_info(e + wstride);
  }
}

}  // namespace tl
