// tl_realize_seg.cuh -- segment-parallel realize + online labelling.
//
// Same semantics as k_synth_cta (reference synth.py:100-348, events.py:94-193,
// modes.py:235-253) with a different decomposition for latency-bound
// batches, where the longest episode sets the kernel time:
//   * work item = (episode, segment of SEG records), one warp each;
//   * a warp fast-forwards from the episode start: the MT19937 state lives
//     in registers (lane l holds words 32s+l) and each block is regenerated
//     with shuffles only (word i reads words i+1, i+397 (old) or i-227
//     (new): three dependency phases, no barriers); only the advance draws
//     (the serial f64 cum_robot_force recurrence) and object-distance draws
//     are evaluated before the segment;
//   * records of the segment are emitted 32 at a time (one per lane) and
//     labelled into a partial state (|E|, last index per kind, error bits);
//   * k_seg_finalize combines the partials of an episode in order and
//     classifies (modes.py:235-253).
#pragma once
#include "tl_synth.cuh"

namespace tl {

constexpr int kSegWarps = 4;
constexpr int kSegRing = 2048;  // >= 32 records * (4 + 2*(2*7+5)) + 623
constexpr uint32_t kSegMask = kSegRing - 1;

struct SegWarp {
  uint32_t ring[kSegRing];
  int32_t gap[kMaxSteps];
  int32_t tau[kMaxSteps];
  int32_t W[kMaxSteps + 1];
  int32_t hw[kMaxSteps + 1];
  StepSt st[kMaxSteps + 1];
  double dist_after[kMaxSteps];
  double radv[32];
  uint8_t kind[kMaxSteps];
  uint8_t sflag[kMaxSteps];
  int32_t misc[16];
  tl_cset cs;
};

struct SegPartial {  // partial label state of one segment
  int32_t size;
  int32_t last[7];
  uint32_t err_any;
  int32_t err_key;   // (step << 8) | InfeasibleScript code, or INT_MAX
};

// ---- register-resident warp twist ---------------------------------------------
// word(S, l) = state[32*S + l]; slot 19 holds words 608..623 (lanes 0..15).
template <int S>
__device__ __forceinline__ uint32_t twist_word(const uint32_t (&w)[20], int lane) {
  // mt[i+1]: same slot from lane+1, or the next slot's lane 0 (i = 623 -> new mt[0])
  const uint32_t up = __shfl_down_sync(kFull, w[S], 1);
  const uint32_t nx = __shfl_sync(kFull, w[S < 19 ? S + 1 : 0], 0);
  const uint32_t b = (lane < 31 && !(S == 19 && lane == 15)) ? up : nx;
  uint32_t src;
  if (S < 7 || S == 7) {
    // i + 397 = 32*(S+12) + (lane+13): old words
    const uint32_t o1 = __shfl_sync(kFull, w[S + 12 < 20 ? S + 12 : 19], (lane + 13) & 31);
    const uint32_t o2 = __shfl_sync(kFull, w[S + 13 < 20 ? S + 13 : 19], (lane + 13) & 31);
    src = lane < 19 ? o1 : o2;
  }
  if (S >= 7) {
    // i - 227 = 32*(S-7) + (lane-3): new words
    const uint32_t n1 = __shfl_sync(kFull, w[S - 7 >= 0 ? S - 7 : 0], (lane + 29) & 31);
    const uint32_t n2 = __shfl_sync(kFull, w[S - 8 >= 0 ? S - 8 : 0], (lane + 29) & 31);
    const uint32_t nsrc = lane >= 3 ? n1 : n2;
    if (S == 7) src = lane < 3 ? src : nsrc;
    else src = nsrc;
  }
  return mt_mix(w[S], b, src);
}

template <int S>
__device__ __forceinline__ void twist_slot(uint32_t (&w)[20], uint32_t* ring, uint32_t base,
                                           int lane) {
  const uint32_t nv = twist_word<S>(w, lane);
  if (S < 19 || lane < 16) {
    w[S] = nv;
    ring[(base + 32u * S + lane) & kSegMask] = mt_temper(nv);
  }
}

__device__ __forceinline__ void twist_regs(uint32_t (&w)[20], uint32_t* ring, uint32_t base) {
  const int lane = lane_id();
  twist_slot<0>(w, ring, base, lane);   twist_slot<1>(w, ring, base, lane);
  twist_slot<2>(w, ring, base, lane);   twist_slot<3>(w, ring, base, lane);
  twist_slot<4>(w, ring, base, lane);   twist_slot<5>(w, ring, base, lane);
  twist_slot<6>(w, ring, base, lane);   twist_slot<7>(w, ring, base, lane);
  twist_slot<8>(w, ring, base, lane);   twist_slot<9>(w, ring, base, lane);
  twist_slot<10>(w, ring, base, lane);  twist_slot<11>(w, ring, base, lane);
  twist_slot<12>(w, ring, base, lane);  twist_slot<13>(w, ring, base, lane);
  twist_slot<14>(w, ring, base, lane);  twist_slot<15>(w, ring, base, lane);
  twist_slot<16>(w, ring, base, lane);  twist_slot<17>(w, ring, base, lane);
  twist_slot<18>(w, ring, base, lane);  twist_slot<19>(w, ring, base, lane);
  __syncwarp();
}

struct SegParams {
  SynthParams sp;
  int32_t seg;          // records per segment
  int32_t max_seg;      // segments per episode slot (items = n_env * max_seg)
  SegPartial* parts;    // [n_env][max_seg]
};

template <int DOFMAX>
__global__ void __launch_bounds__(kSegWarps * 32)
    k_realize_seg(SegParams q) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const SynthParams& p = q.sp;
  const int warp = threadIdx.x >> 5, lane = lane_id();
  SegWarp& S = reinterpret_cast<SegWarp*>(smem_raw)[warp];
  const int64_t item = (int64_t)blockIdx.x * kSegWarps + warp;
  const int e = (int)(item / q.max_seg), k = (int)(item % q.max_seg);
  if (e >= p.n_env) return;
  const tl_script sc = p.scripts[e];
  const int n_rec = p.out.n_rec[e];
  const int r_lo = k * q.seg;
  if (sc.n_steps < 0 || r_lo >= n_rec) return;  // capacity error / no such segment
  const int r_hi = min(n_rec, r_lo + q.seg);
  const int64_t rs = p.out.rec_start[e];
  const int dof = p.out.dof;
  float* __restrict__ P = reinterpret_cast<float*>(p.out.planes);
  const int64_t stride = p.out.plane_stride;
  const float fnan = __int_as_float(0x7fc00000);
  const uint2* ring2 = reinterpret_cast<const uint2*>(S.ring);

  // MT state of the realize RNG into registers
  uint32_t w[20];
  {
    const uint32_t* src = p.states + (int64_t)e * kMtN;
#pragma unroll
    for (int s = 0; s < 20; s++) w[s] = (s < 19 || lane < 16) ? src[32 * s + lane] : 0u;
  }
  const int art_idx = (sc.subtask == TL_OPEN || sc.subtask == TL_CLOSE) ? sc.art_kind : 0;
  stage_cset(&S.cs, &p.label_csets[sc.subtask * 3 + (art_idx < 0 || art_idx > 2 ? 0 : art_idx)]);
  const tl_cset& c = S.cs;
  RzConst z;
  const int st0 = realizer_init(z, sc, p.th, dof);
  SegPartial part;
  part.size = 0;
#pragma unroll
  for (int i = 0; i < 7; i++) part.last[i] = -1;
  part.err_any = 0;
  part.err_key = 0x7fffffff;
  if (st0 != TL_OK) {  // reported by segment 0 only
    if (lane == 0) {
      part.err_key = (0x7fffff << 8) | st0;
      q.parts[item] = part;
    }
    return;
  }
  const int ns = sc.n_steps;  // <= kMaxSteps (fuzz scripts)
  for (int i = lane; i < ns; i += 32) {
    S.kind[i] = p.step_kind[sc.step_off + i];
    S.gap[i] = p.step_gap[sc.step_off + i];
  }
  __syncwarp();
  if (lane == 0) {  // plan (as k_synth_cta): record/word layout + deterministic state
    PlanSt ps;
    ps.force = (z.has_force && sc.initial_contact) ? 1.2 : 0.0;
    ps.grasped = sc.initial_grasped ? 1 : 0;
    ps.at_rest = 0;
    ps.exc = 0;
    if (z.kind == TL_OPEN) {
      ps.level = sc.initial_level;
      ps.art = sc.initial_level == TL_LVL_LOW ? z.lv_low : sc.initial_level == TL_LVL_SLIGHT ? z.lv_slight : z.lv_open;
    } else if (z.kind == TL_CLOSE) {
      ps.level = sc.initial_level == TL_LVL_CLOSED ? TL_LVL_CLOSED : TL_LVL_OPEN;
      ps.art = z.a_q0;
    } else {
      ps.level = TL_LVL_LOW;
      ps.art = 0.0;
    }
    int32_t wo = 2 * z.ne, r = 0;
    int last_draw = -1, perr = 0, pstep = ns, exc_at = 0x7fffffff;
    S.st[0] = make_st(z, ps, -1);
    for (int s = 0; s < ns; s++) {
      const int g = S.gap[s];
      if (g < 1) { perr = TL_INF_GAP; pstep = s; S.W[s] = wo; S.hw[s] = 0; S.tau[s] = r; break; }
      S.W[s] = wo;
      const int hwv = (ps.exc ? 0 : 2) + (ps.at_rest ? 0 : 2 * z.ne);
      S.hw[s] = hwv;
      wo += (g - 1) * hwv;
      r += g;
      S.tau[s] = r;
      int wev = ps.exc ? 0 : 2;
      int draw = 0;
      const int ec = plan_apply(z, ps, S.kind[s], draw);
      S.sflag[s] = (uint8_t)draw;
      if (ec) { perr = ec; pstep = s; break; }
      if (draw) last_draw = s;
      if (S.kind[s] == TL_EV_EXCESSIVE_COLLISIONS) exc_at = r;
      wev += (draw ? 2 : 0) + (ps.at_rest ? 0 : 2 * z.ne);
      wo += wev;
      S.st[s + 1] = make_st(z, ps, last_draw);
    }
    if (!perr) {
      S.W[ns] = wo;
      S.hw[ns] = (ps.exc ? 0 : 2) + (ps.at_rest ? 0 : 2 * z.ne);
    }
    S.misc[0] = perr;
    S.misc[1] = pstep;
    S.misc[2] = exc_at;
  }
  __syncwarp();
  const int perr = S.misc[0], pstep = S.misc[1], exc_rec = S.misc[2];
  const double dist0 = z.has_goal ? sc.initial_dist_obj_goal : __longlong_as_double(0x7ff8000000000000ll);
  float sc_ru = 0.f;
  double sc_d = 0.0;
  if (c.subtask == TL_CLOSE) {
    const double a0 = z.kind == TL_CLOSE ? z.a_q0 : 0.0;
    close_cut(c, (double)__double2float_rn(a0), sc_ru, sc_d);
  }
  const int r_end = perr ? min(r_hi, S.tau[pstep] + 1) : r_hi;
  double cum = 0.0;
  uint32_t produced = 0;
  uint32_t ind_carry = 0;
  int seg_hint = 0;
  for (int c0 = 0; c0 < r_end; c0 += 32) {
    const int r = c0 + lane;
    const bool valid = r < r_end;
    int o = 0, adv = 0, app = 0, emit = 0, sidx = 0, ev = -1, s = 0;
    if (valid) {
      if (r == 0) {
        emit = 1;
      } else {
        s = seg_hint;
        while (s < ns && S.tau[s] < r) s++;
        if (s < ns && S.tau[s] == r) {
          o = S.W[s] + (S.gap[s] - 1) * S.hw[s];
          adv = !S.st[s].exc;
          ev = S.kind[s];
          const bool failing = perr && s == pstep;
          app = failing ? 0 : (S.sflag[s] & 1);
          emit = failing ? 0 : !S.st[s + 1].at_rest;
          sidx = failing ? s : s + 1;
        } else {
          const int first = (s == 0 ? 0 : S.tau[s - 1]) + 1;
          o = S.W[s] + (r - first) * S.hw[s];
          adv = !S.st[s].exc;
          emit = !S.st[s].at_rest;
          sidx = s;
        }
      }
    }
    seg_hint = __shfl_sync(kFull, s, 0);
    // the chunk needs full records only from r_lo - 1 on (edge at r_lo)
    const bool full = valid && r >= r_lo - 1;
    const int need = valid ? (full ? o + 2 * adv + 2 * app + (emit ? 2 * z.ne : 0)
                                    : o + 2 * adv + 2 * app) : 0;
    const int need_max = __reduce_max_sync(kFull, need);
    while ((int)produced < need_max) {
      twist_regs(w, S.ring, produced);
      produced += kMtN;
    }
    auto rnd = [&](int woff) {
      const uint2 wv = ring2[((uint32_t)woff & kSegMask) >> 1];
      return rand53(wv.x, wv.y);
    };
    int my_err = 0;
    S.radv[lane] = valid && adv ? rnd(o) : 0.0;
    if (valid && app) {
      const double rr = rnd(o + 2 * adv);
      S.dist_after[s] = ev == TL_EV_OBJ_AT_GOAL ? uniform_rn(0.02, 0.12, rr) : uniform_rn(0.3, 0.8, rr);
    }
    __syncwarp();
    double dist_rec = dist0;
    if (valid && z.has_goal) {
      const int ld = S.st[sidx].last_draw;
      dist_rec = ld >= 0 ? S.dist_after[ld] : dist0;
      if (ev >= 0) {
        const int ldb = S.st[s].last_draw;
        const double db = ldb >= 0 ? S.dist_after[ldb] : dist0;
        switch (ev) {  // value-dependent checks of _apply (synth.py:218-260)
          case TL_EV_OBJ_AT_GOAL: if (db <= z.goal) my_err = TL_INF_AT_GOAL_ALREADY; break;
          case TL_EV_OBJ_LEFT_GOAL: if (db > z.goal) my_err = TL_INF_LEFT_NOT_AT_GOAL; break;
          case TL_EV_RELEASED_AT_GOAL: if (db > z.goal) my_err = TL_INF_RAG; break;
          case TL_EV_RELEASED_OUTSIDE_GOAL: if (db <= z.goal) my_err = TL_INF_ROG; break;
          case TL_EV_SUCCESS: if (db > z.goal) my_err = TL_INF_SUCCESS_UNREACHABLE; break;
        }
      }
    }
    if (valid && perr && ev >= 0 && s == pstep && !my_err) my_err = perr;
    const unsigned eb = __ballot_sync(kFull, my_err != 0);
    if (eb) {
      const int L = __ffs(eb) - 1;
      const int code = __shfl_sync(kFull, my_err, L);
      const int step = __shfl_sync(kFull, s, L);
      part.err_key = (step << 8) | code;
      break;
    }
    // cum_robot_force (synth.py:192-196): warp-uniform serial recurrence
    const int cnt = min(32, r_end - c0);
    const int jx = exc_rec >= c0 ? min(cnt, exc_rec - c0) : 0;
    double my_cum = 0.0;
    int j = c0 == 0 ? 1 : 0;
    for (; j + 8 <= jx; j += 8) {
      double rg[8];
#pragma unroll
      for (int kk = 0; kk < 8; kk++) rg[kk] = S.radv[j + kk];
#pragma unroll
      for (int kk = 0; kk < 8; kk++) {
        cum = __dadd_rn(cum, __dmul_rn(__dmul_rn(__dsub_rn(z.L09, cum), 0.05), rg[kk]));
        my_cum = lane == j + kk ? cum : my_cum;
      }
    }
    for (; j < jx; j++) {
      cum = __dadd_rn(cum, __dmul_rn(__dmul_rn(__dsub_rn(z.L09, cum), 0.05), S.radv[j]));
      my_cum = lane == j ? cum : my_cum;
    }
    if (c0 + cnt > exc_rec) {
      cum = z.L105;
      if (lane >= jx) my_cum = cum;
    }
    __syncwarp();
    if (c0 + 32 <= r_lo - 1) continue;  // fast-forward chunk: no records of ours
    // ---- emit (from r_lo - 1: its indicator bits feed the edge at r_lo) ---------
    uint32_t ind = 0, errb = 0;
    if (full) {
      const StepSt stv = S.st[sidx];
      const uint32_t eo = (uint32_t)(o + 2 * adv + 2 * app);
      const bool mine = r >= r_lo;
      float* __restrict__ dst = P + rs + r;
      auto draw = [&](uint32_t kk, double a, double b) -> float {
        if (!emit) return 0.f;
        const uint2 wv = ring2[((eo + 2u * kk) & kSegMask) >> 1];
        return __double2float_rn(uniform_rn(a, b, rand53(wv.x, wv.y)));
      };
      RecV<float> v;
      float mq = 0.f, mqd = 0.f;
#pragma unroll
      for (int i = 0; i < DOFMAX; i++) {
        if (i < dof) {
          const float qv = draw(i, -0.3, 0.3);
          if (mine) *dst = qv;
          dst += stride;
          mq = i == 0 ? fabsf(qv) : pymax_step(mq, fabsf(qv));
        }
      }
#pragma unroll
      for (int i = 0; i < DOFMAX; i++) {
        if (i < dof) {
          const float qd = draw(dof + i, -0.4, 0.4);
          if (mine) *dst = qd;
          dst += stride;
          mqd = i == 0 ? fabsf(qd) : pymax_step(mqd, fabsf(qd));
        }
      }
      const uint32_t k2 = 2 * dof;
      v.tor = draw(k2, -0.05, 0.05);
      v.vx = draw(k2 + 1, -0.2, 0.2);
      v.vy = draw(k2 + 2, -0.2, 0.2);
      v.om = draw(k2 + 3, -0.3, 0.3);
      v.der = draw(k2 + 4, 0.2, 1.0);
      v.dist = z.has_goal ? __double2float_rn(dist_rec) : fnan;
      v.force = stv.force;
      v.cum = __double2float_rn(my_cum);
      v.art = stv.art;
      v.g = stv.grasped != 0;
      v.qdm = mqd;
      v.jm = mq;
      v.jm_d = 0.0;
      if (mine) {
        dst[0] = v.tor;
        dst[stride] = v.vx;
        dst[2 * stride] = v.vy;
        dst[3 * stride] = v.om;
        dst[4 * stride] = v.der;
        dst[5 * stride] = v.dist;
        dst[6 * stride] = v.force;
        dst[7 * stride] = v.cum;
        dst[8 * stride] = v.art;
        p.out.grasped[rs + r] = (uint8_t)v.g;
      }
      record_bits(c, v, sc_ru, sc_d, ind, errb);
    }
    uint32_t prev = __shfl_up_sync(kFull, ind, 1);
    if (lane == 0) prev = ind_carry;
    const bool mine = valid && r >= r_lo;
    const uint32_t mask = (mine && r > 0) ? edge_mask(c.subtask, prev, ind) : 0u;
    if (mine && p.step_mask) p.step_mask[rs + r] = (uint8_t)mask;
    LState L;
    L.size = part.size;
#pragma unroll
    for (int i = 0; i < 7; i++) L.last[i] = part.last[i];
    L.prev_ind = 0;
    L.err_any = part.err_any;
    lstate_fold(L, mask, mine ? errb : 0u);
    part.size = L.size;
#pragma unroll
    for (int i = 0; i < 7; i++) part.last[i] = L.last[i];
    part.err_any = L.err_any;
    ind_carry = __shfl_sync(kFull, ind, 31);
  }
  // a plan error with no event record of its own (gap < 1)
  if (part.err_key == 0x7fffffff && perr) part.err_key = (pstep << 8) | perr;
  if (lane == 0) q.parts[item] = part;
}

// combine the segments of each episode in order, classify, write the label
__global__ void k_seg_finalize(SegParams q) {
  const SynthParams& p = q.sp;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= p.n_env) return;
  const tl_script sc = p.scripts[e];
  tl_label L;
  L.n_events = 0;
  L.err_index = -1;
  L.subtask = (uint8_t)sc.subtask;
  L.mode = 255;
  L.flags = 0;
  L.pad = 0;
  L.d0 = __longlong_as_double(0x7ff8000000000000ll);
  if (sc.n_steps < 0) {
    L.status = TL_ERR_SCRIPT_CAPACITY;
    p.labels[e] = L;
    return;
  }
  const int n_rec = p.out.n_rec[e];
  const int nseg = max(1, (n_rec + q.seg - 1) / q.seg);
  LState S;
  lstate_init(S);
  int err_key = 0x7fffffff;
  for (int k = 0; k < nseg; k++) {
    const SegPartial& pt = q.parts[(int64_t)e * q.max_seg + k];
    err_key = min(err_key, pt.err_key);
#pragma unroll
    for (int i = 0; i < 7; i++)
      if (pt.last[i] >= 0) S.last[i] = S.size + pt.last[i];
    S.size += pt.size;
    S.err_any |= pt.err_any;
  }
  if (err_key != 0x7fffffff) {
    const int step = err_key >> 8;
    L.status = err_key & 0xff;
    L.err_index = step == 0x7fffff ? -1 : step;
    p.labels[e] = L;
    p.out.n_rec[e] = 0;
    return;
  }
  const tl_cset& c = p.label_csets[sc.subtask * 3 + ((sc.subtask == TL_OPEN || sc.subtask == TL_CLOSE) ? sc.art_kind : 0)];
  L.status = label_status(c, S.err_any);
  const double d0 = sc.subtask == TL_PLACE ? (double)__double2float_rn(sc.initial_dist_obj_goal) : L.d0;
  L.d0 = d0;
  if (L.status == TL_OK) {
    Sig zz;
    sig_from_state(zz, c.subtask, S);
    zz.d0 = d0;
    uint8_t fl = 0;
    const int m = classify_sig(c.subtask, zz, p.rules, fl);
    L.n_events = S.size;
    if (m < 0) {
      L.status = -m;
      L.flags = zz.s >= 0 ? 1 : 0;
    } else {
      L.mode = (uint8_t)m;
      L.flags = fl;
    }
  }
  p.labels[e] = L;
}

}  // namespace tl
