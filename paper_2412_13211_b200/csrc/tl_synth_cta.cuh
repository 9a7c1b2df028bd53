// tl_synth_cta.cuh -- realize + online labelling with one CTA per episode.
//
// Semantics: reference synth.py:100-348 (_Realizer) fused with
// events.py:94-193 (extract_events) and modes.py:235-253 (classify).
// Mapping (W = records per wave: 64 = 3 warps, 32 = 2 warps for batches
// whose episodes fit 64 records):
//   * thread 0 plans the script window (exact MT word offset of every
//     record and the deterministic per-step state); meanwhile the emission
//     warps regenerate the episode's first MT block;
//   * MT19937 block regeneration in three phases of 4-word groups,
//     double-buffered (old / new block arrays): 3 barriers per block,
//     128-bit shared accesses, tempered words into a ring;
//   * a wave of W records is emitted at once, one record per emission
//     thread, from the ring (4096 / 2048 words: all CTAs of a 1024-episode
//     batch are resident at once);
//   * the serial f64 cum_robot_force recurrence runs on warp 0, eight
//     records per group of vector shared-memory loads, split at the
//     ExcessiveCollisions record (before it every step draws, after it cum
//     is constant), CONCURRENTLY with the emission of the same wave; the
//     cum-dependent label bits are patched in afterwards (cum_patch_bits);
//   * each emission warp folds its 32 event masks into a partial label
//     state, combined in order by warp 0; persistent CTAs prefetch their
//     next episode's seeded state and script by cp.async;
//   * tl_fuzz_ev: the ordered event lists are written by k_scan_emit right
//     after this kernel (tl_label.cuh): an in-kernel form had to wait for the
//     last realized episode of every 32-episode block, and with longest-first
//     claims that is the end of the batch for nearly every block.
#pragma once
#include "tl_synth.cuh"

namespace tl {

#ifdef TL_PHASES
// aggregate phase profiler (profiling build only, scripts/phase_totals.py):
// thread 0 of every CTA adds the clock64 delta since its previous mark to
// g_tl_phase[k]; g_tl_phase[15] counts waves
__device__ unsigned long long g_tl_phase[16];
#define TL_PH(k)                                                              \
  do {                                                                        \
    if (threadIdx.x == 0) {                                                   \
      const long long _t = clock64();                                         \
      atomicAdd(&g_tl_phase[(k)], (unsigned long long)(_t - ph_t));           \
      ph_t = _t;                                                              \
    }                                                                         \
  } while (0)
#else
#define TL_PH(k) do { } while (0)
#endif

// W = records per wave = emission threads (warps 1..W/32); warp 0 runs the
// cum chain.  W = 64 for long episodes; W = 32 (a 2-warp CTA, a quarter of
// the ring, ~1.5x the CTAs per SM) when every episode fits one or two waves.
constexpr int kWave = 64;
template <int W>
__host__ __device__ constexpr int cta_threads() { return W + 32; }

template <int DOFMAX, int W = kWave>
struct CtaCfg {
  // >= W*(4+2*(2*DOFMAX+5)) + 623 words: a wave's draws plus a block's lookahead
  static constexpr int kRing = W == 64 ? (DOFMAX <= 7 ? 4096 : 8192) : (DOFMAX <= 7 ? 2048 : 4096);
  static_assert(kRing >= W * (4 + 2 * (2 * DOFMAX + 5)) + 623, "ring too small");
  static constexpr uint32_t kMask = kRing - 1;
};

template <int DOFMAX, int WAVE = kWave>
struct CtaSmem {
  // script steps planned per window (scripts are re-planned window by
  // window); 48 keeps the 64-record form at 8 CTAs/SM (27.8 KB), the
  // short-episode form plans 32 at a time to fit 12 CTAs/SM
  static constexpr int kSteps = WAVE == 32 ? 32 : 48;
  uint32_t mt[2][kMtN];  // double-buffered MT state (current block, next block)
  uint32_t wb[CtaCfg<DOFMAX, WAVE>::kRing];
  int32_t gap[kSteps];
  int32_t tau[kSteps];
  int32_t W[kSteps + 1];
  int32_t hw[kSteps + 1];
  StepSt st[kSteps + 1];
  double dist_after[kSteps];
  double radv[WAVE];
  float cum32[WAVE];
  uint32_t ind[WAVE];       // indicator bits without the cum patch
  uint32_t eerr[WAVE];
  LState part[WAVE / 32];
  uint8_t kind[kSteps];
  uint8_t sflag[kSteps];
  int32_t misc[16];
  int32_t red[8];
  int32_t tk[2];            // claimed episode tickets (double-buffered by iteration)
  int32_t bend[kLenBuckets];  // longest-first bucket ends (load_bucket_ends)
  tl_cset cs;
  // the CTA's next episode, copied in by cp.async while this one runs
  alignas(16) uint32_t mt_pf[kMtN];
  tl_script sc_pf;
  int64_t rs_pf;
  int32_t nrec_pf;
};

// CPython's block regeneration in 4-word groups (group g = words 4g..4g+3).
// Word i reads words i+1 and i+397 (old, i < 227) or i-227 (new), i.e. a
// group depends on groups 56-57 earlier, so three phases of <= 56 groups
// (0..55 | 56..111 | 112..155) are each internally independent: one group
// per thread, 128-bit shared-memory accesses.
// Double-buffered form: the new block is written to `nw` while every old
// word stays readable in `od`, so a phase needs no barrier between its loads
// and its stores (no write-after-read hazard): 3 barriers per 624-word block.
// Word i reads od[i], od[i+1] (nw[0] for i = 623) and od[i+397] (i < 227) or
// nw[i-227] (i >= 227, written by an earlier phase).
template <int DOFMAX, int W, int G0, int G1>
__device__ __forceinline__ void twist_phase_db(const uint32_t* od, uint32_t* nw, uint32_t* ring,
                                               uint32_t base) {
  static_assert(G1 - G0 <= cta_threads<W>(), "one group per thread");
  const int g = G0 + threadIdx.x;
  if (g < G1) {
    const uint4 cur = reinterpret_cast<const uint4*>(od)[g];
    const int i = 4 * g;
    const uint32_t nxt = i + 4 == kMtN ? nw[0] : od[i + 4];
    auto src = [&](int k) {
      const int ii = i + k;
      return ii < kMtN - kMtM ? od[ii + kMtM] : nw[ii - (kMtN - kMtM)];
    };
    uint4 nv;
    nv.x = mt_mix(cur.x, cur.y, src(0));
    nv.y = mt_mix(cur.y, cur.z, src(1));
    nv.z = mt_mix(cur.z, cur.w, src(2));
    nv.w = mt_mix(cur.w, nxt, src(3));
    reinterpret_cast<uint4*>(nw)[g] = nv;
    const uint4 tv = make_uint4(mt_temper(nv.x), mt_temper(nv.y), mt_temper(nv.z), mt_temper(nv.w));
    reinterpret_cast<uint4*>(ring)[((base + 4u * g) & CtaCfg<DOFMAX, W>::kMask) >> 2] = tv;
  }
  __syncthreads();
}

// The same on the emission warps only (named barrier 1, W threads; W = 32
// takes two groups per thread), so warp 0 can plan the episode meanwhile.
template <int DOFMAX, int W, int G0, int G1>
__device__ __forceinline__ void twist_phase_dbe(const uint32_t* od, uint32_t* nw, uint32_t* ring,
                                                uint32_t base) {
#pragma unroll
  for (int g = G0 + (int)threadIdx.x - 32; g < G1; g += W) {
    const uint4 cur = reinterpret_cast<const uint4*>(od)[g];
    const int i = 4 * g;
    const uint32_t nxt = i + 4 == kMtN ? nw[0] : od[i + 4];
    auto src = [&](int k) {
      const int ii = i + k;
      return ii < kMtN - kMtM ? od[ii + kMtM] : nw[ii - (kMtN - kMtM)];
    };
    uint4 nv;
    nv.x = mt_mix(cur.x, cur.y, src(0));
    nv.y = mt_mix(cur.y, cur.z, src(1));
    nv.z = mt_mix(cur.z, cur.w, src(2));
    nv.w = mt_mix(cur.w, nxt, src(3));
    reinterpret_cast<uint4*>(nw)[g] = nv;
    const uint4 tv = make_uint4(mt_temper(nv.x), mt_temper(nv.y), mt_temper(nv.z), mt_temper(nv.w));
    reinterpret_cast<uint4*>(ring)[((base + 4u * g) & CtaCfg<DOFMAX, W>::kMask) >> 2] = tv;
  }
  asm volatile("bar.sync 1, %0;\n" ::"n"(W) : "memory");
}

template <int DOFMAX, int W>
__device__ __forceinline__ void mt_twist_block_db(const uint32_t* od, uint32_t* nw, uint32_t* ring,
                                                  uint32_t base) {
  twist_phase_db<DOFMAX, W, 0, 56>(od, nw, ring, base);
  twist_phase_db<DOFMAX, W, 56, 112>(od, nw, ring, base);
  twist_phase_db<DOFMAX, W, 112, 156>(od, nw, ring, base);
}

template <int W>
__device__ __forceinline__ int block_max(int v, int32_t* red) {
  const int warp = threadIdx.x >> 5;
  v = __reduce_max_sync(kFull, v);
  if (lane_id() == 0) red[warp] = v;
  __syncthreads();
  int m = red[0];
#pragma unroll
  for (int w = 1; w < cta_threads<W>() / 32; w++) m = max(m, red[w]);
  return m;  // red is rewritten only after later barriers of the wave
}

template <bool FUZZ, int DOFMAX, int W>
__global__ void __launch_bounds__(W + 32, W == 64 ? 8 : 12)
    k_synth_cta(SynthParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CtaSmem<DOFMAX, W>& S = *reinterpret_cast<CtaSmem<DOFMAX, W>*>(smem_raw);
  constexpr uint32_t kMask = CtaCfg<DOFMAX, W>::kMask;
  constexpr int kCtaThreads = cta_threads<W>();
  const int tid = threadIdx.x, warp = tid >> 5, lane = lane_id();
  const int dof = p.out.dof;
  float* __restrict__ P = reinterpret_cast<float*>(p.out.planes);
  const int64_t stride = p.out.plane_stride;
  const float fnan = __int_as_float(0x7fc00000);
  const uint2* ring2 = reinterpret_cast<const uint2*>(S.wb);

  int wave_no = 0;
  bool pf = false;
#ifdef TL_PHASES
  long long ph_t = clock64();
#endif  // the next episode's inputs are in flight to S.*_pf
  // episodes by ticket, in claim order (dynamic load balance across CTAs);
  // the next episode is claimed at the top of the current one so its inputs
  // can be prefetched, parity-buffered in S.tk (>= 1 barrier per iteration)
  if (warp == 0 && p.order) load_bucket_ends(p, S.bend);
  __syncwarp();
  if (tid == 0) S.tk[0] = claim_episode(p, S.bend);
  __syncthreads();
  int e = S.tk[0];
  for (int it = 1; e < p.n_env; it++) {
    if (tid == 0) S.tk[it & 1] = claim_episode(p, S.bend);
    if (tid == 0 && e == 0) TL_STAMP(10);
    TL_PH(9);  // 9: end of the previous episode -> this one (claims, tail)
    // ---------------- script + seeded RNG state -------------------------------
    tl_script sc;
    int64_t rs;
    int n_rec;
    if (pf) {
      cp_async_wait<0>();
      __syncthreads();
      sc = S.sc_pf;
      rs = S.rs_pf;
      n_rec = S.nrec_pf;
      for (int i = tid; i < kMtN / 4; i += kCtaThreads)
        reinterpret_cast<uint4*>(S.mt[0])[i] = reinterpret_cast<const uint4*>(S.mt_pf)[i];
    } else {
      sc = p.scripts[e];
      rs = p.out.rec_start[e];
      n_rec = p.out.n_rec[e];
      const uint32_t* src = p.states + (int64_t)e * kMtN;
      for (int i = tid; i < kMtN; i += kCtaThreads) S.mt[0][i] = src[i];
    }
    pf = false;
    if (FUZZ && sc.n_steps < 0) {
      if (tid == 0) {
        tl_label L;
        L.status = TL_ERR_SCRIPT_CAPACITY; L.n_events = 0; L.err_index = -1;
        L.subtask = (uint8_t)sc.subtask; L.mode = 255; L.flags = 0; L.pad = 0;
        L.d0 = __longlong_as_double(0x7ff8000000000000ll);
        p.labels[e] = L;
      }
      __syncthreads();
      e = S.tk[it & 1];
      continue;
    }
    const int art_idx = (sc.subtask == TL_OPEN || sc.subtask == TL_CLOSE) ? sc.art_kind : 0;
    if (warp == 0) stage_cset(&S.cs, &p.label_csets[sc.subtask * 3 + (art_idx < 0 || art_idx > 2 ? 0 : art_idx)]);
    RzConst z;
    const int st0 = realizer_init(z, sc, p.th, dof);
    __syncthreads();
    const int en = S.tk[it & 1];
    {  // S.*_pf are free again (copied out above): fetch the next episode's inputs
      if (en < p.n_env) {
        const uint32_t* src = p.states + (int64_t)en * kMtN;
        for (int i = tid; i < kMtN / 4; i += kCtaThreads) cp_async16(S.mt_pf + 4 * i, src + 4 * i);
        if (tid < (int)(sizeof(tl_script) / 4))
          cp_async4(reinterpret_cast<uint32_t*>(&S.sc_pf) + tid,
                    reinterpret_cast<const uint32_t*>(&p.scripts[en]) + tid);
        else if (tid < (int)(sizeof(tl_script) / 4) + 2)
          cp_async4(reinterpret_cast<uint32_t*>(&S.rs_pf) + (tid - sizeof(tl_script) / 4),
                    reinterpret_cast<const uint32_t*>(&p.out.rec_start[en]) + (tid - sizeof(tl_script) / 4));
        else if (tid == (int)(sizeof(tl_script) / 4) + 2)
          cp_async4(reinterpret_cast<uint32_t*>(&S.nrec_pf),
                    reinterpret_cast<const uint32_t*>(&p.out.n_rec[en]));
        cp_async_commit();
        pf = true;
      }
    }
    auto fail = [&](int code, int step) {
      if (tid == 0) {
        tl_label L;
        L.status = code; L.n_events = 0; L.err_index = step;
        L.subtask = (uint8_t)sc.subtask; L.mode = 255; L.flags = 0; L.pad = 0;
        L.d0 = __longlong_as_double(0x7ff8000000000000ll);
        p.labels[e] = L;
        if (FUZZ) p.out.n_rec[e] = 0;
      }
    };
    if (st0 != TL_OK) {
      fail(st0, -1);
      __syncthreads();
      e = en;
      continue;
    }
    if (tid == 0 && e == 0) TL_STAMP(11);
    TL_PH(6);  // 6: episode prologue (state copy, init, prefetch issue)
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

    LState LS;                 // live in warp 0
    lstate_init(LS);
    uint32_t ind_carry = 0;    // indicator bits of the previous wave's last record
    double cum = 0.0;          // warp 0: serial f64 recurrence
    double dist_carry = dist0;
    int32_t w_carry = 2 * z.ne;
    int32_t tau_prev = 0;
    uint32_t produced = 0;
    int mt_cur = 0;  // which S.mt buffer holds the current block
    int err_code = 0, err_step = -1;
    int s_base = 0;
    const int n_steps = sc.n_steps;
    PlanSt pcarry = ps;
    bool first_window = true;
    for (;;) {
      const int ns = min(n_steps - s_base, CtaSmem<DOFMAX, W>::kSteps);
      const bool last_window = s_base + ns >= n_steps;
      for (int i = tid; i < ns; i += kCtaThreads) {
        S.kind[i] = p.step_kind[sc.step_off + s_base + i];
        S.gap[i] = p.step_gap[sc.step_off + s_base + i];
      }
      __syncthreads();
      if (first_window && warp > 0) {
        // block 0 of the realize stream is always consumed (record 0 draws):
        // warps 1-2 regenerate it while thread 0 plans
        twist_phase_dbe<DOFMAX, W, 0, 56>(S.mt[0], S.mt[1], S.wb, 0);
        twist_phase_dbe<DOFMAX, W, 56, 112>(S.mt[0], S.mt[1], S.wb, 0);
        twist_phase_dbe<DOFMAX, W, 112, 156>(S.mt[0], S.mt[1], S.wb, 0);
      }
      if (first_window) {
        mt_cur = 1;
        produced = kMtN;
      }
      if (tid == 0) {  // plan: record/word layout + deterministic state
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
      __syncthreads();
      if (tid == 0 && e == 0) TL_STAMP(12);
      TL_PH(7);  // 7: window plan (+ first block twist)
      const int perr = S.misc[0], pstep = S.misc[1];
      const int exc_rec = S.misc[14];
      const int r_begin = first_window ? 0 : tau_prev + 1;
      int r_end;
      if (perr) r_end = S.tau[pstep] + 1;
      else if (last_window) r_end = n_rec;
      else r_end = S.misc[3] + 1;
      int seg_hint = 0;
      const bool emitter = warp > 0;
      const int et = tid - 32;  // record slot of an emission thread
      for (int r0 = r_begin; r0 < r_end && !err_code; r0 += W) {
        const int r = r0 + et;
        const bool valid = emitter && r < r_end;
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
              const int first = (s == 0 ? tau_prev : S.tau[s - 1]) + 1;
              o = S.W[s] + (r - first) * S.hw[s];
              adv = !S.st[s].exc;
              emit = !S.st[s].at_rest;
              sidx = s;
            }
          }
        }
        if (et == 0) S.misc[12] = s;
        const int need = valid ? o + 2 * adv + 2 * app + (emit ? 2 * z.ne : 0) : 0;
        const int need_max = block_max<W>(need, S.red);  // also publishes misc[12]
        seg_hint = S.misc[12];
        const int wbase = 20 + 8 * min(wave_no, 12);  // profiling build only
        if (tid == 0 && e == 0) TL_STAMP(wbase);
        TL_PH(1);  // 1: record descriptors + block max
        while ((int)produced < need_max) {
          mt_twist_block_db<DOFMAX, W>(S.mt[mt_cur], S.mt[mt_cur ^ 1], S.wb, produced);
          mt_cur ^= 1;
          produced += kMtN;
        }
        if (tid == 0 && e == 0) TL_STAMP(wbase + 1);
        TL_PH(2);  // 2: MT twists
        auto rnd = [&](int woff) {
          const uint2 wv = ring2[((uint32_t)woff & kMask) >> 1];
          return rand53(wv.x, wv.y);
        };
        int my_err = 0;
        if (emitter) S.radv[et] = valid && adv ? rnd(o) : 0.0;
        if (valid && app) {
          const double rr = rnd(o + 2 * adv);
          S.dist_after[s] = ev == TL_EV_OBJ_AT_GOAL ? TL_UNIFORM(0.02, 0.12, rr) : TL_UNIFORM(0.3, 0.8, rr);
        }
        if (tid == 0) S.misc[13] = 0x7fffffff;
        __syncthreads();
        if (tid == 0 && e == 0) TL_STAMP(wbase + 2);
        TL_PH(3);  // 3: advance / apply draws
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
        // the wave's InfeasibleScript verdict is read after the next barrier:
        // an erroneous wave's emission only writes inside the failed episode's
        // own record slot, and nothing of it is folded
        if (my_err) atomicMin(&S.misc[13], ((s_base + s) << 8) | my_err);
        const int cnt = min(W, r_end - r0);
        if (!emitter) {
          // cum_robot_force: serial f64 recurrence (synth.py:192-196, :210-213),
          // overlapped with the emission below.  Record 0 never draws; every
          // later record draws until the ExcessiveCollisions record, which
          // jumps to 1.05*limit for good.
          const int jx = exc_rec >= r0 ? min(cnt, exc_rec - r0) : 0;  // draws in [j0, jx)
          int j = 0;
          if (r0 == 0) {
            if (lane == 0) S.cum32[0] = 0.f;
            j = 1;
          }
          for (; j + 8 <= jx; j += 8) {
            double rg[8];
#pragma unroll
            for (int k = 0; k < 8; k++) rg[k] = S.radv[j + k];
            float out[8];
#pragma unroll
            for (int k = 0; k < 8; k++) {
              cum = __dadd_rn(cum, __dmul_rn(__dmul_rn(__dsub_rn(z.L09, cum), 0.05), rg[k]));
              out[k] = __double2float_rn(cum);
            }
            if (lane == 0) {
              S.cum32[j + 0] = out[0]; S.cum32[j + 1] = out[1];
              S.cum32[j + 2] = out[2]; S.cum32[j + 3] = out[3];
              S.cum32[j + 4] = out[4]; S.cum32[j + 5] = out[5];
              S.cum32[j + 6] = out[6]; S.cum32[j + 7] = out[7];
            }
          }
          for (; j < jx; j++) {
            cum = __dadd_rn(cum, __dmul_rn(__dmul_rn(__dsub_rn(z.L09, cum), 0.05), S.radv[j]));
            if (lane == 0) S.cum32[j] = __double2float_rn(cum);
          }
          if (jx < cnt && r0 + cnt > exc_rec) {
            cum = z.L105;
            const float c105 = __double2float_rn(cum);
            for (int k = max(j, 0) + lane; k < cnt; k += 32) S.cum32[k] = c105;
          }
        } else if (valid) {
          // ---- emit + write + indicator bits (cum patched after the barrier) ----
          uint32_t ind = 0, errb = 0;
          const int64_t rr = rs + r;
          const StepSt stv = S.st[sidx];
          const uint32_t eo = (uint32_t)(o + 2 * adv + 2 * app);
          float* __restrict__ dst = P + rr;
          // branch-free: every draw is computed, at-rest records select 0
          // rng.uniform(a, b) with b - a folded at compile time (same RN result)
          auto draw = [&](uint32_t k, double a, double span) -> float {
            const uint2 wv = ring2[((eo + 2u * k) & kMask) >> 1];
            const float v = __double2float_rn(uniform_span(a, span, rand53(wv.x, wv.y)));
            return emit ? v : 0.f;
          };
          RecV<float> v;
          float mq = 0.f, mqd = 0.f;
#pragma unroll
          for (int i = 0; i < DOFMAX; i++) {
            if (i < dof) {
              const float q = draw(i, -0.3, 0.3 - -0.3);
              *dst = q;
              dst += stride;
              mq = i == 0 ? fabsf(q) : pymax_step(mq, fabsf(q));
            }
          }
#pragma unroll
          for (int i = 0; i < DOFMAX; i++) {
            if (i < dof) {
              const float qd = draw(dof + i, -0.4, 0.4 - -0.4);
              *dst = qd;
              dst += stride;
              mqd = i == 0 ? fabsf(qd) : pymax_step(mqd, fabsf(qd));
            }
          }
          const uint32_t k2 = 2 * dof;
          v.tor = draw(k2, -0.05, 0.05 - -0.05);
          v.vx = draw(k2 + 1, -0.2, 0.2 - -0.2);
          v.vy = draw(k2 + 2, -0.2, 0.2 - -0.2);
          v.om = draw(k2 + 3, -0.3, 0.3 - -0.3);
          v.der = draw(k2 + 4, 0.2, 1.0 - 0.2);
          v.dist = z.has_goal ? __double2float_rn(dist_rec) : fnan;
          v.force = stv.force;
          v.cum = 0.f;  // over = false here; cum_patch_bits applies the real value
          v.art = stv.art;
          v.g = stv.grasped != 0;
          v.qdm = mqd;
          v.jm = mq;
          v.jm_d = 0.0;
          dst[0] = v.tor;
          dst[stride] = v.vx;
          dst[2 * stride] = v.vy;
          dst[3 * stride] = v.om;
          dst[4 * stride] = v.der;
          dst[5 * stride] = v.dist;
          dst[6 * stride] = v.force;
          dst[8 * stride] = v.art;
          p.out.grasped[rr] = (uint8_t)v.g;
          record_bits(c, v, sc_ru, sc_d, ind, errb);
          S.ind[et] = ind;
          S.eerr[et] = errb;
        }
        __syncthreads();
        {
          const int ek = S.misc[13];
          if (ek != 0x7fffffff) {
            err_code = ek & 0xff;
            err_step = ek >> 8;
            break;
          }
        }
        if (tid == 0 && e == 0) TL_STAMP(wbase + 3);
        TL_PH(4);  // 4: cum chain || emission
        if (emitter) {
          uint32_t ind = 0, errb = 0, prev = ind_carry;
          if (valid) {
            const float cm = S.cum32[et];
            P[rs + r + (int64_t)(2 * dof + 7) * stride] = cm;  // cum_robot_force plane
            errb = S.eerr[et];
            ind = cum_patch_bits(c, cm, S.ind[et], errb);
            if (et > 0) {
              uint32_t e2 = 0;
              prev = cum_patch_bits(c, S.cum32[et - 1], S.ind[et - 1], e2);
            }
          }
          const uint32_t mask = (valid && r > 0) ? edge_mask(c.subtask, prev, ind) : 0u;
          if (valid && p.step_mask) p.step_mask[rs + r] = (uint8_t)mask;
          // per-warp partial fold, combined in record order by warp 0
          LState part;
          lstate_init(part);
          lstate_fold(part, mask, valid ? errb : 0u);
          if (lane == 0) S.part[warp - 1] = part;
        }
        // indicator bits of the wave's last record (carry into the next wave)
        {
          uint32_t e2 = 0;
          ind_carry = cum_patch_bits(c, S.cum32[cnt - 1], S.ind[cnt - 1], e2);
        }
        __syncthreads();
        if (warp == 0) {
#pragma unroll
          for (int w = 0; w < W / 32; w++) {
            const LState& q = S.part[w];
#pragma unroll
            for (int k = 0; k < 7; k++)
              if (q.last[k] >= 0) LS.last[k] = LS.size + q.last[k];
            LS.size += q.size;
            LS.err_any |= q.err_any;
          }
        }
        // no barrier: S.part is rewritten only after the next wave's barriers
        if (tid == 0 && e == 0) TL_STAMP(wbase + 5);
        TL_PH(5);  // 5: patch + fold
#ifdef TL_PHASES
        if (tid == 0) atomicAdd(&g_tl_phase[15], 1ull);
#endif
        if (e == 0) wave_no++;
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
      __syncthreads();
    }
    if (err_code) {
      fail(err_code, err_step);
    } else if (warp == 0) {
      const tl_label L = make_label(c, LS, d0, p.rules);
      if (lane == 0) p.labels[e] = L;
    }
    __syncthreads();
    if (tid == 0 && e == 0) TL_STAMP(13);
    TL_PH(8);  // 8: label + window tail
    if (tid == 0 && e == gridDim.x) TL_STAMP(14);
    e = en;
  }
  TL_PH(9);
  if (p.order) {  // the last CTA out leaves the length buckets at zero for the next launch
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      if (atomicAdd(&p.tickets[2], 1u) == gridDim.x - 1) {
        for (int b = 0; b < kLenBuckets; b++) p.tickets[kTkBucket + b] = 0u;
        p.tickets[2] = 0u;
      }
    }
  }
}

}  // namespace tl
