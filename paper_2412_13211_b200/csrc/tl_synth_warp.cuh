// tl_synth_warp.cuh -- realize + online labelling with one WARP per episode.
//
// Semantics: reference synth.py:100-348 (_Realizer) fused with
// events.py:94-193 (extract_events) and modes.py:235-253 (classify), the
// same as k_synth_cta; the mapping differs:
//   * every warp is an independent persistent worker (no CTA barriers): it
//     claims an episode by ticket (longest first), plans each script window
//     on lane 0 (exact MT word offset of every record), then walks the
//     records in 32-record waves, one record per lane;
//   * MT19937 blocks are regenerated in place by the warp in CPython's three
//     dependency phases (4-word groups, loads of a phase before its stores,
//     __syncwarp between), tempered words into a per-warp ring;
//   * the serial f64 cum_robot_force recurrence is computed redundantly by
//     all lanes (lane j keeps the value of record r0 + j), so the
//     cum-dependent label bits, the edge masks and the label fold need no
//     shared memory round trip;
//   * per-warp shared memory is ~12.6 KB at arm dof <= 7: 16 episodes in
//     flight per SM (vs 8 three-warp CTAs), and a wave costs the warp's own
//     instruction stream only -- no waiting on the slowest warp of a CTA.
#pragma once
#include "tl_synth.cuh"

namespace tl {

template <int DOFMAX>
struct WarpCfg {
  // >= 32 * (4 + 2 * (2 * DOFMAX + 5)) + 623 words: a wave's draws plus the
  // lookahead of the block that completes them
  static constexpr int kRing = DOFMAX <= 7 ? 2048 : 4096;
  static_assert(kRing >= 32 * (4 + 2 * (2 * DOFMAX + 5)) + 623, "ring too small");
  static constexpr uint32_t kMask = kRing - 1;
  // the ring's first kApron words are mirrored past its end, so one record's
  // 2*(2*dof+5) emit words are contiguous from any start (no wrap per draw)
  static constexpr int kApron = (2 * (2 * DOFMAX + 5) + 3) & ~3;
  static constexpr int kSteps = 32;  // script steps planned per window
};

template <int DOFMAX>
struct WarpSmem {
  static constexpr int kSteps = WarpCfg<DOFMAX>::kSteps;
  alignas(16) uint32_t mt[kMtN];                       // MT state, regenerated in place
  alignas(16) uint32_t wb[WarpCfg<DOFMAX>::kRing + WarpCfg<DOFMAX>::kApron];  // tempered words
  int32_t gap[kSteps];
  int32_t tau[kSteps];
  int32_t W[kSteps + 1];
  int32_t hw[kSteps + 1];
  StepSt st[kSteps + 1];
  double dist_after[kSteps];
  double radv[32];
  double cumw[32];   // the wave's cum_robot_force values (chain step j -> lane j)
  uint8_t kind[kSteps];
  uint8_t sflag[kSteps];
  int32_t misc[16];
  tl_cset cs;
};

// one dependency phase of CPython's block regeneration, in place: group g =
// words 4g..4g+3 reads its own words and word 4g+4 (old; word 0 -- new --
// for the last group) and words i+397 (old, i < 227) or i-227 (new, written
// by an earlier phase).  Every load of the phase precedes every store.
template <int DOFMAX, int G0, int G1>
__device__ __forceinline__ void twist_phase_warp(uint32_t* mt, uint32_t* ring, uint32_t base) {
  constexpr int kPer = (G1 - G0 + 31) / 32;
  constexpr uint32_t kMask = WarpCfg<DOFMAX>::kMask;
  const int lane = lane_id();
  const uint4* mt4 = reinterpret_cast<const uint4*>(mt);
  uint4 nv[kPer];
#pragma unroll
  for (int q = 0; q < kPer; q++) {
    const int g = G0 + lane + 32 * q;
    const int gg = g < G1 ? g : G1 - 1;  // lanes past the phase load a valid group
    const int i = 4 * gg;
    const uint4 cur = mt4[gg];
    // the group's four sources i+k+397 (i+k < 227) or i+k-227 sit one word
    // past a 16-byte boundary: one 128-bit load + the next group's first
    // word (two requests instead of four 4-way conflicted scalar loads);
    // phase 2's first group takes 621..623 and word 0
    int sb;
    if constexpr (G1 * 4 <= kMtN - kMtM) sb = i + kMtM - 1;
    else if constexpr (G0 * 4 >= kMtN - kMtM + 1) sb = i - (kMtN - kMtM) - 1;
    else sb = i < kMtN - kMtM ? i + kMtM - 1 : i - (kMtN - kMtM) - 1;
    const uint4 sa = mt4[sb >> 2];
    const uint32_t s3 = mt[sb + 4 == kMtN ? 0 : sb + 4];
    // word i+4 (old; new word 0 for the block's last group) = the next
    // lane's first word, except at the end of the 32-group chunk
    uint32_t nxt = __shfl_down_sync(kFull, cur.x, 1);
    if (lane == 31 || g + 1 >= G1) {
      if constexpr (G1 * 4 == kMtN) nxt = mt[i + 4 == kMtN ? 0 : i + 4];
      else nxt = mt[i + 4];
    }
    nv[q].x = mt_mix(cur.x, cur.y, sa.y);
    nv[q].y = mt_mix(cur.y, cur.z, sa.z);
    nv[q].z = mt_mix(cur.z, cur.w, sa.w);
    nv[q].w = mt_mix(cur.w, nxt, s3);
  }
  __syncwarp();
#pragma unroll
  for (int q = 0; q < kPer; q++) {
    const int g = G0 + lane + 32 * q;
    if (g < G1) {
      reinterpret_cast<uint4*>(mt)[g] = nv[q];
      const uint4 tv = make_uint4(mt_temper(nv[q].x), mt_temper(nv[q].y), mt_temper(nv[q].z),
                                  mt_temper(nv[q].w));
      reinterpret_cast<uint4*>(ring)[((base + 4u * g) & kMask) >> 2] = tv;
    }
  }
  __syncwarp();
}

template <int DOFMAX>
__device__ __forceinline__ void twist_block_warp(uint32_t* mt, uint32_t* ring, uint32_t base) {
  twist_phase_warp<DOFMAX, 0, 56>(mt, ring, base);     // words 0..223: old words only
  twist_phase_warp<DOFMAX, 56, 112>(mt, ring, base);   // 224..447: new 0..220
  twist_phase_warp<DOFMAX, 112, 156>(mt, ring, base);  // 448..623: new 221..396, word 0
  // the block rewrote ring words [0, kApron): refresh their mirror
  constexpr int kRing = WarpCfg<DOFMAX>::kRing, kApron = WarpCfg<DOFMAX>::kApron;
  const uint32_t b0 = base & WarpCfg<DOFMAX>::kMask;
  if (b0 < (uint32_t)kApron || b0 + kMtN > (uint32_t)kRing) {  // warp-uniform
    if (lane_id() < kApron / 4)
      reinterpret_cast<uint4*>(ring)[kRing / 4 + lane_id()] = reinterpret_cast<const uint4*>(ring)[lane_id()];
    __syncwarp();
  }
}

// longest-first claims (see claim_episode): lane b < 16 holds the exclusive
// end of length buckets 15..15-b
__device__ __forceinline__ int bucket_end_lane(const SynthParams& p) {
  const int lane = lane_id();
  int c = lane < kLenBuckets ? (int)__ldcg(&p.tickets[kTkBucket + kLenBuckets - 1 - lane]) : 0;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int u = __shfl_up_sync(kFull, c, d);
    if (lane >= d) c += u;
  }
  return c;
}

__device__ __forceinline__ int claim_episode_warp(const SynthParams& p, int endv) {
  const int lane = lane_id();
  int t = 0;
  if (lane == 0) t = (int)atomicAdd(&p.tickets[0], 1u);
  t = __shfl_sync(kFull, t, 0);
  if (p.order == nullptr || t >= p.n_env) return t;
  // bucket k = number of bucket ends <= t (the ends increase with b)
  const int k = __popc(__ballot_sync(kFull, lane < kLenBuckets - 1 && t >= endv));
  const int start = __shfl_sync(kFull, endv, k > 0 ? k - 1 : 0);
  return __ldcg(&p.order[(int64_t)(kLenBuckets - 1 - k) * p.n_env + (t - (k > 0 ? start : 0))]);
}

#ifdef TL_PHASES
// per-warp timeline of the last launch (profiling build only,
// scripts/warp_timeline.py): [w][0] start, [w][1] end (globaltimer ns),
// [w][2] records realized, [w][3] episodes
__device__ unsigned long long g_tl_warp[4096][4];
__device__ unsigned long long g_tl_wphase[16];  // clock64 deltas summed over warps, [15] waves
#define TL_WPH(k)                                                                   \
  do {                                                                              \
    const long long _t = clock64();                                                 \
    if (lane == 0) atomicAdd(&g_tl_wphase[(k)], (unsigned long long)(_t - ph_t));   \
    ph_t = _t;                                                                      \
  } while (0)
#else
#define TL_WPH(k) do { } while (0)
#endif

// DOFX: the arm dof when fixed at compile time (7: every fuzz batch and the
// usual realize batch -- the emission then has no dof branches), 0 = runtime
template <bool FUZZ, int DOFMAX, int NW, int DOFX>
__global__ void __launch_bounds__(NW * 32, 16 / NW) k_synth_warp(SynthParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr uint32_t kMask = WarpCfg<DOFMAX>::kMask;
  constexpr int kSteps = WarpCfg<DOFMAX>::kSteps;
  const int warp = threadIdx.x >> 5, lane = lane_id();
  WarpSmem<DOFMAX>& S = reinterpret_cast<WarpSmem<DOFMAX>*>(smem_raw)[warp];
  const int dof = DOFX ? DOFX : p.out.dof;
  float* __restrict__ P = reinterpret_cast<float*>(p.out.planes);
  const int64_t stride = p.out.plane_stride;
  const float fnan = __int_as_float(0x7fc00000);
  const uint2* ring2 = reinterpret_cast<const uint2*>(S.wb);
  const int endv = p.order ? bucket_end_lane(p) : 0;
#ifdef TL_PHASES
  const int gw = blockIdx.x * NW + warp;
  unsigned long long w_recs = 0, w_eps = 0;
  if (lane == 0 && gw < 4096) g_tl_warp[gw][0] = gtimer();
  long long ph_t = clock64();
#endif

  for (int e = claim_episode_warp(p, endv); e < p.n_env; e = claim_episode_warp(p, endv)) {
    // ---------------- script + seeded RNG state -------------------------------
    const tl_script sc = p.scripts[e];
    auto fail = [&](int code, int step) {
      if (lane == 0) {
        tl_label L;
        L.status = code; L.n_events = 0; L.err_index = step;
        L.subtask = (uint8_t)sc.subtask; L.mode = 255; L.flags = 0; L.pad = 0;
        L.d0 = __longlong_as_double(0x7ff8000000000000ll);
        p.labels[e] = L;
        if (FUZZ) p.out.n_rec[e] = 0;
      }
    };
    if (FUZZ && sc.n_steps < 0) {
      if (lane == 0) {
        tl_label L;
        L.status = sc.n_steps == -2 ? TL_E_INVALID : TL_ERR_SCRIPT_CAPACITY;
        L.n_events = 0; L.err_index = -1;
        L.subtask = (uint8_t)sc.subtask; L.mode = 255; L.flags = 0; L.pad = 0;
        L.d0 = __longlong_as_double(0x7ff8000000000000ll);
        p.labels[e] = L;
      }
      continue;
    }
    const int64_t rs = p.out.rec_start[e];
    const int n_rec = p.out.n_rec[e];
    TL_ASSERT(rs >= 0 && n_rec >= 0 && rs + n_rec <= p.out.plane_stride);
    TL_ASSERT(!FUZZ || n_rec <= p.cap_per_env);
    // every load that only needs the script goes out together (one L2 round
    // trip instead of three): the MT state and the cset by cp.async, the
    // first window's step kinds and gaps into lane registers
    const int art_idx = (sc.subtask == TL_OPEN || sc.subtask == TL_CLOSE) ? sc.art_kind : 0;
    const int ns0 = min(sc.n_steps, kSteps);
    const int kind0 = lane < ns0 ? (int)p.step_kind[sc.step_off + lane] : 0;
    const int gap0 = lane < ns0 ? p.step_gap[sc.step_off + lane] : 0;
    {
      __syncwarp();  // the previous episode is done with S.mt and S.cs
      const uint32_t* src = p.states + (int64_t)e * kMtN;
#pragma unroll
      for (int i = lane; i < kMtN / 4; i += 32) cp_async16(S.mt + 4 * i, src + 4 * i);
      const uint32_t* cs = reinterpret_cast<const uint32_t*>(
          &p.label_csets[sc.subtask * 3 + (art_idx < 0 || art_idx > 2 ? 0 : art_idx)]);
      for (int i = lane; i < (int)(sizeof(tl_cset) / 4); i += 32)
        cp_async4(reinterpret_cast<uint32_t*>(&S.cs) + i, cs + i);
      cp_async_commit();
    }
    TL_WPH(9);  // 9: claim + script loads
    RzConst z;
    const int st0 = realizer_init(z, sc, p.th, dof);
    cp_async_wait<0>();
    __syncwarp();
    if (st0 != TL_OK) {
      fail(st0, -1);
      continue;
    }
    TL_WPH(6);  // 6: state + cset arrival, realizer init
    PlanSt ps;  // initial realizer state (synth.py:111-158)
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
    const double dist0 = z.has_goal ? sc.initial_dist_obj_goal : __longlong_as_double(0x7ff8000000000000ll);
    const tl_cset& c = S.cs;
    float sc_ru = 0.f;
    double sc_d = 0.0;
    if (c.subtask == TL_CLOSE) close_cut(c, (double)__double2float_rn(ps.art), sc_ru, sc_d);
    const double d0 = (double)__double2float_rn(dist0);

    LState LS;                 // warp-uniform running label state
    lstate_init(LS);
    uint32_t ind_carry = 0;    // indicator bits of the previous wave's last record
    double cum = 0.0;          // serial f64 recurrence (every lane)
    double dist_carry = dist0;
    int32_t w_carry = 2 * z.ne;
    int32_t tau_prev = 0;
    uint32_t produced = 0;
    int err_code = 0, err_step = -1;
    int s_base = 0;
    const int n_steps = sc.n_steps;
    PlanSt pcarry = ps;
    bool first_window = true;
    for (;;) {
      const int ns = min(n_steps - s_base, kSteps);
      const bool last_window = s_base + ns >= n_steps;
      if (first_window) {  // prefetched with the state
        if (lane < ns) {
          S.kind[lane] = (uint8_t)kind0;
          S.gap[lane] = gap0;
        }
      } else {
        for (int i = lane; i < ns; i += 32) {
          S.kind[i] = p.step_kind[sc.step_off + s_base + i];
          S.gap[i] = p.step_gap[sc.step_off + s_base + i];
        }
      }
      __syncwarp();
      if (lane == 0) {  // plan: record/word layout + deterministic state
        PlanSt q = pcarry;
        int32_t w = w_carry, r = tau_prev;
        int last_draw = -1, perr = 0, pstep = ns;
        int exc_at = 0x7fffffff;  // record of the ExcessiveCollisions jump
        S.st[0] = make_st(z, q, -1);
        for (int s = 0; s < ns; s++) {
          const int g = S.gap[s];
          if (g < 1) { perr = TL_INF_GAP; pstep = s; S.W[s] = w; S.hw[s] = 0; S.tau[s] = r; break; }
          S.W[s] = w;
          const int hwv = (q.exc ? 0 : 2) + (q.at_rest ? 0 : 2 * z.ne);
          S.hw[s] = hwv;
          w += (g - 1) * hwv;
          r += g;
          S.tau[s] = r;
          int wev = q.exc ? 0 : 2;
          int draw = 0;
          const int ec = plan_apply(z, q, S.kind[s], draw);
          S.sflag[s] = (uint8_t)draw;
          if (ec) { perr = ec; pstep = s; break; }
          if (draw) last_draw = s;
          if (S.kind[s] == TL_EV_EXCESSIVE_COLLISIONS) exc_at = r;
          wev += (draw ? 2 : 0) + (q.at_rest ? 0 : 2 * z.ne);
          w += wev;
          S.st[s + 1] = make_st(z, q, last_draw);
        }
        S.misc[14] = pcarry.exc ? -1 : exc_at;
        if (!perr) {
          S.W[ns] = w;
          S.hw[ns] = (q.exc ? 0 : 2) + (q.at_rest ? 0 : 2 * z.ne);
        }
        S.misc[0] = perr; S.misc[1] = pstep; S.misc[2] = w; S.misc[3] = r;
        S.misc[4] = q.grasped; S.misc[5] = q.at_rest; S.misc[6] = q.exc; S.misc[7] = q.level;
        reinterpret_cast<double*>(&S.misc[8])[0] = q.force;
        reinterpret_cast<double*>(&S.misc[10])[0] = q.art;
      }
      __syncwarp();
      TL_WPH(7);  // 7: window load + plan
      const int perr = S.misc[0], pstep = S.misc[1];
      const int exc_rec = S.misc[14];
      const int r_begin = first_window ? 0 : tau_prev + 1;
      int r_end;
      if (perr) r_end = S.tau[pstep] + 1;
      else if (last_window) r_end = n_rec;
      else r_end = S.misc[3] + 1;
      int seg_hint = 0;
      for (int r0 = r_begin; r0 < r_end; r0 += 32) {
        const int r = r0 + lane;
        const bool valid = r < r_end;
        int o = 0, adv = 0, app = 0, emit = 0, sidx = 0, ev = -1, s = seg_hint;
        if (valid) {
          if (r == 0) {
            emit = 1;
          } else {
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
              const int first = (s == 0 ? tau_prev : S.tau[s - 1]) + 1;
              o = S.W[s] + (r - first) * S.hw[s];
              adv = !S.st[s].exc;
              emit = !S.st[s].at_rest;
              sidx = s;
            }
          }
        }
        seg_hint = __shfl_sync(kFull, s, 0);  // lane 0 holds the wave's first record
        TL_WPH(1);  // 1: descriptors
        TL_ASSERT(!valid || (r < n_rec && s <= ns && sidx <= ns));
        const int need = valid ? o + 2 * adv + 2 * app + (emit ? 2 * z.ne : 0) : 0;
        const int need_max = __reduce_max_sync(kFull, need);
        while ((int)produced < need_max) {
          twist_block_warp<DOFMAX>(S.mt, S.wb, produced);
          produced += kMtN;
        }
        TL_WPH(2);  // 2: twist
        auto rnd = [&](int woff) {
          const uint2 wv = ring2[((uint32_t)woff & kMask) >> 1];
          return rand53(wv.x, wv.y);
        };
        S.radv[lane] = valid && adv ? rnd(o) : 0.0;
        TL_ASSERT(!(valid && adv) || ((uint32_t)o + 2u <= produced &&
                                      produced - (uint32_t)o <= (uint32_t)WarpCfg<DOFMAX>::kRing));
        if (valid && app) {
          TL_ASSERT(s < ns);
          const double rr = rnd(o + 2 * adv);
          S.dist_after[s] = ev == TL_EV_OBJ_AT_GOAL ? TL_UNIFORM(0.02, 0.12, rr) : TL_UNIFORM(0.3, 0.8, rr);
        }
        __syncwarp();
        int my_err = 0;
        double dist_rec = dist_carry;
        if (valid && z.has_goal) {
          const int ld = S.st[sidx].last_draw;
          dist_rec = ld >= 0 ? S.dist_after[ld] : dist_carry;
          if (ev >= 0) {
            const int ldb = S.st[s].last_draw;
            const double db = ldb >= 0 ? S.dist_after[ldb] : dist_carry;
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
        {  // the first failing record of the wave ends the episode (nothing of it is kept)
          const int ek = __reduce_min_sync(kFull, my_err ? (((s_base + s) << 8) | my_err) : 0x7fffffff);
          if (ek != 0x7fffffff) {
            err_code = ek & 0xff;
            err_step = ek >> 8;
            break;
          }
        }
        TL_WPH(3);  // 3: draws before emission + error check (+ the twist: phase 2)
        // ---- emit + write, and the cum chain, in one straight-line block -------
        // Every lane runs the emission (invalid lanes' stores are predicated
        // off) and the 32 chain steps are unconditional, so the compiler can
        // interleave the serial f64 chain with the independent draws.
        const int cnt = min(32, r_end - r0);
        const int jx = exc_rec >= r0 ? min(cnt, exc_rec - r0) : 0;  // chain records [j0, jx)
        const int64_t rr = rs + r;
        const StepSt stv = S.st[sidx];
        const uint32_t eo = (uint32_t)(o + 2 * adv + 2 * app);
        float* __restrict__ dst = P + rr;
        // at-rest records select 0.  The record's emit words are contiguous in
        // the ring (apron), and rng.uniform(a, b) = a + (b - a) * (k * 2^-53)
        // is evaluated as a + ((b - a) * 2^-53) * k: the same real product,
        // so the same rounding, with the scaled span folded at compile time
        const uint2* rw = ring2 + ((eo & kMask) >> 1);
        TL_ASSERT(!(valid && emit) || (eo + 2u * (2 * dof + 5) <= produced &&
                                       produced - eo <= (uint32_t)WarpCfg<DOFMAX>::kRing &&
                                       (eo & kMask) + 2u * (2 * dof + 5) <=
                                           (uint32_t)(WarpCfg<DOFMAX>::kRing + WarpCfg<DOFMAX>::kApron)));
        auto draw = [&](const uint2* w, double a, double span) -> float {
          const uint2 wv = *w;
          const float v = __double2float_rn(uniform_k53(a, span * 0x1.0p-53, wv.x, wv.y));
          return emit ? v : 0.f;
        };
        RecV<float> v;
        float mq = 0.f, mqd = 0.f;
#pragma unroll
        for (int i = 0; i < DOFMAX; i++) {
          if (i < dof) {
            const float q = draw(rw + i, -0.3, 0.3 - -0.3);
            if (valid) *dst = q;
            dst += stride;
            mq = i == 0 ? fabsf(q) : pymax_step(mq, fabsf(q));
          }
        }
#pragma unroll
        for (int i = 0; i < DOFMAX; i++) {
          if (i < dof) {
            const float qd = draw(rw + dof + i, -0.4, 0.4 - -0.4);
            if (valid) *dst = qd;
            dst += stride;
            mqd = i == 0 ? fabsf(qd) : pymax_step(mqd, fabsf(qd));
          }
        }
        const uint2* r2 = rw + 2 * dof;
        v.tor = draw(r2, -0.05, 0.05 - -0.05);
        v.vx = draw(r2 + 1, -0.2, 0.2 - -0.2);
        v.vy = draw(r2 + 2, -0.2, 0.2 - -0.2);
        v.om = draw(r2 + 3, -0.3, 0.3 - -0.3);
        v.der = draw(r2 + 4, 0.2, 1.0 - 0.2);
        v.dist = z.has_goal ? __double2float_rn(dist_rec) : fnan;
        v.force = stv.force;
        v.cum = 0.f;  // over = false here; cum_patch_bits applies the real value
        v.art = stv.art;
        v.g = stv.grasped != 0;
        v.qdm = mqd;
        v.jm = mq;
        v.jm_d = 0.0;
        if (valid) {
          dst[0] = v.tor;
          dst[stride] = v.vx;
          dst[2 * stride] = v.vy;
          dst[3 * stride] = v.om;
          dst[4 * stride] = v.der;
          dst[5 * stride] = v.dist;
          dst[6 * stride] = v.force;
          dst[8 * stride] = v.art;
          p.out.grasped[rr] = (uint8_t)v.g;
        }
        // cum_robot_force (synth.py:192-196, :210-213), every lane, lane j
        // keeps record r0 + j.  S.radv is 0.0 for records that do not advance
        // (record 0, after ExcessiveCollisions, past the wave), and cum + 0.0
        // == cum, so all 32 steps run unconditionally; the ExcessiveCollisions
        // record and everything after it take 1.05*limit below.
        // each step's value goes to S.cumw[j] (one broadcast store per step),
        // read back by lane j after the chain
#pragma unroll
        for (int j = 0; j < 32; j++) {
          cum = __dadd_rn(cum, __dmul_rn(__dmul_rn(__dsub_rn(z.L09, cum), 0.05), S.radv[j]));
          S.cumw[j] = cum;
        }
        __syncwarp();
        double my_cum_d = S.cumw[lane];  // record 0: radv 0, cum 0
        if (jx < cnt) {  // the wave reaches the ExcessiveCollisions record (warp-uniform)
          cum = z.L105;
          if (lane >= max(jx, r0 == 0 ? 1 : 0)) my_cum_d = cum;
        }
        const float my_cum = __double2float_rn(my_cum_d);
        uint32_t ind = 0, errb = 0;
        record_bits(c, v, sc_ru, sc_d, ind, errb);
        TL_WPH(4);  // 4: emission || chain
        // ---- patch the cum bits, edges, label fold ------------------------------
        uint32_t indp = 0;
        if (valid) {
          P[rs + r + (int64_t)(2 * dof + 7) * stride] = my_cum;  // cum_robot_force plane
          indp = cum_patch_bits(c, my_cum, ind, errb);
        }
        uint32_t prev = __shfl_up_sync(kFull, indp, 1);
        if (lane == 0) prev = ind_carry;
        const uint32_t mask = (valid && r > 0) ? edge_mask(c.subtask, prev, indp) : 0u;
        if (valid && p.step_mask) p.step_mask[rs + r] = (uint8_t)mask;
        ind_carry = __shfl_sync(kFull, indp, cnt - 1);
        lstate_fold(LS, mask, valid ? errb : 0u);
        __syncwarp();  // S.radv / S.dist_after are rewritten by the next wave
        TL_WPH(5);  // 5: patch + fold
#ifdef TL_PHASES
        if (lane == 0) atomicAdd(&g_tl_wphase[15], 1ull);
#endif
      }
      if (!err_code && perr) { err_code = perr; err_step = s_base + pstep; }
      if (err_code || last_window) break;
      {
        const int ld = S.st[ns].last_draw;
        if (ld >= 0) dist_carry = S.dist_after[ld];
      }
      pcarry.grasped = S.misc[4]; pcarry.at_rest = S.misc[5]; pcarry.exc = S.misc[6]; pcarry.level = S.misc[7];
      pcarry.force = reinterpret_cast<const double*>(&S.misc[8])[0];
      pcarry.art = reinterpret_cast<const double*>(&S.misc[10])[0];
      w_carry = S.misc[2];
      tau_prev = S.misc[3];
      s_base += ns;
      first_window = false;
      __syncwarp();  // the plan arrays are rewritten by the next window
    }
    TL_WPH(10);  // 10: window tails
    if (err_code) {
      fail(err_code, err_step);
    } else {
      const tl_label L = make_label(c, LS, d0, p.rules);
      if (lane == 0) p.labels[e] = L;
    }
#ifdef TL_PHASES
    w_recs += n_rec;
    w_eps++;
#endif
    TL_WPH(8);  // 8: label
  }
#ifdef TL_PHASES
  if (lane == 0 && gw < 4096) {
    g_tl_warp[gw][1] = gtimer();
    g_tl_warp[gw][2] = w_recs;
    g_tl_warp[gw][3] = w_eps;
  }
#endif
  if (p.order) {  // the last CTA out leaves the length buckets at zero for the next launch
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(&p.tickets[2], 1u) == gridDim.x - 1) {
        for (int b = 0; b < kLenBuckets; b++) p.tickets[kTkBucket + b] = 0u;
        p.tickets[2] = 0u;
      }
    }
  }
}

}  // namespace tl
