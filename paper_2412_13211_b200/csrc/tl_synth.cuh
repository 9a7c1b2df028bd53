// tl_synth.cuh -- random_script + realize building blocks: the reset
// kernels (CPython seeding, script sampling), the realizer constants and
// the deterministic part of _apply; the realize + label kernel itself is
// k_synth_cta (tl_synth_cta.cuh), the batched env in tl_env.cuh.
//
// Reference (paths under /root/reference/pkg/src/trajlab/):
//   synth.py:100-162  _Realizer.__init__  (= reset)
//   synth.py:166-196  _emit / _advance_cum
//   synth.py:205-296  _apply              (= step(action))
//   synth.py:298-348  run / _build / realize
//   synth.py:363-515  random_script / fuzz
//
// Every record t >= 1 is one env step: advance_cum (1 draw before the
// ExcessiveCollisions jump), apply (1 draw for ObjAtGoal/ObjLeftGoal) and
// emit (2*dof+5 draws unless at rest).  Which draws happen depends only on
// the script, not on drawn values, so a per-step plan (one thread,
// O(steps)) fixes the MT word offset of every record and the records of a
// wave are generated in parallel from a ring of tempered MT words.  Only
// cum_robot_force is a true serial f64 recurrence (4 ops per record).
// Object distance draws and their feasibility checks happen at the owning
// event record.
#pragma once
#include "tl_label.cuh"

namespace tl {

constexpr int kMaxSteps = 64;     // script steps planned per window

struct StepSt {          // realizer state after a step (index s+1); [0] = before
  float force, art;      // record values (f32)
  uint8_t grasped, at_rest, exc, level;
  int16_t last_draw;     // window-local step of the latest dist draw, -1 = carry
  int16_t pad;
};

struct RzConst {
  int kind, has_art, has_goal, has_force, dof, ne;
  double limit, L09, L105, goal, qmin, qmax, closed_thresh, sc_thresh,
      lv_low, lv_slight, lv_open, a_q0, sc_art;
  int band_valid;
};

struct SynthParams {
  // fuzz inputs (k_fuzz_reset)
  const int64_t* seeds;
  int32_t fuzz_subtask;
  const uint8_t* subtasks;  // per-episode subtask (tl_fuzz*_mixed), else fuzz_subtask
  tl_fuzz_cfg cfg;
  // scripts (written by k_fuzz_reset, or given for realize)
  tl_script* scripts;
  uint8_t* step_kind;
  int32_t* step_gap;
  // seeded realize-RNG states, [n_env][624] (k_fuzz_reset / k_seed_states)
  uint32_t* states;
  // common
  int32_t n_env;
  int32_t cap_per_env;
  tl_thresholds th;
  const tl_cset* label_csets;   // [subtask*3 + art_kind]
  tl_rules rules;
  tl_records out;
  uint8_t* step_mask;
  tl_label* labels;
  // tl_fuzz_ev: k_scan_emit's tile states + tile counter ([ev_zero] entries),
  // zeroed by the reset kernel (no memset node in the step graph)
  unsigned long long* ev_state;
  int32_t ev_zero;
  // claim counters: [0] episodes (zeroed by the reset kernel), [2] exited
  // CTAs, [4 + b] episodes in length bucket b (left at zero by every
  // k_synth_cta launch; zero-filled scratch before the first).  k_synth_cta
  // takes episodes by ticket and never waits on another CTA.
  unsigned int* tickets;
  // longest-first episode order (fuzz, long-episode configs): bucket b holds
  // the episodes of b+1 64-record waves (b = 15: 16 or more) at
  // order[b * n_env + slot], filled by k_fuzz_reset; null = index order
  int32_t* order;
};

#ifdef TL_BUCKET32
constexpr int kLenBuckets = 32;   // longest-first buckets of 32 records
constexpr int kBucketRecs = 32;
#else
constexpr int kLenBuckets = 16;   // longest-first buckets of 64 records
constexpr int kBucketRecs = 64;
#endif
constexpr int kTkBucket = 4;  // tickets[kTkBucket + b]

// ticket -> episode: tickets walk the length buckets from the longest down
// (LPT order: a long episode claimed last would otherwise set the batch
// time, synth.py run lengths vary ~4x around the mean).  The bucket sizes are
// final once the reset kernel is done: one warp reads them once per launch
// into shared memory (end[k] = exclusive end of buckets 15..15-k).
__device__ __forceinline__ void load_bucket_ends(const SynthParams& p, int* end) {
  const int lane = threadIdx.x & 31;
  int c = lane < kLenBuckets ? (int)__ldcg(&p.tickets[kTkBucket + kLenBuckets - 1 - lane]) : 0;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, c, d);
    if (lane >= d) c += u;
  }
  if (lane < kLenBuckets) end[lane] = c;
}

__device__ __forceinline__ int claim_episode(const SynthParams& p, const int* end) {
  const int t = (int)atomicAdd(&p.tickets[0], 1u);
  if (p.order == nullptr || t >= p.n_env) return t;
  int k = 0;
  while (k < kLenBuckets - 1 && t >= end[k]) k++;
  const int start = k ? end[k - 1] : 0;
  return __ldcg(&p.order[(int64_t)(kLenBuckets - 1 - k) * p.n_env + (t - start)]);
}

__device__ __forceinline__ bool in_alpha(int k, int ev) {
#pragma unroll
  for (int i = 0; i < 7; i++)
    if (kAlpha[k][i] == ev) return true;
  return false;
}

// choices(pop, weights)[0] (Lib/random.py): accumulate + bisect_right
// (N is a compile-time population size: the cumulative weights stay in
// registers)
template <int N>
__device__ __forceinline__ int choices_idx(MtLane& R, const double (&w)[N]) {
  double cum[N];
  double acc = w[0];
  cum[0] = acc;
#pragma unroll
  for (int i = 1; i < N; i++) {
    acc = __dadd_rn(acc, w[i]);
    cum[i] = acc;
  }
  const double total = __dadd_rn(cum[N - 1], 0.0);
  const double x = __dmul_rn(R.random(), total);
  int idx = N - 1;  // bisect_right over cum[0..N-2]: the first i with x < cum[i]
#pragma unroll
  for (int i = N - 2; i >= 0; i--)
    if (x < cum[i]) idx = i;
  return idx;
}

// random_script (synth.py:363-507), one thread.  Returns n_steps, or -1
// when the script does not fit `cap` steps (never for cap = max_events + 4).
__device__ int sample_script(MtLane& R, int kind, const tl_fuzz_cfg& cfg,
                             uint8_t* sk, int32_t* sg, tl_script& sc, int cap, int64_t& gaps) {
  int n = 0;
  bool overflow = false;
  gaps = 0;  // sum of the stored steps' gaps
  auto push = [&](int ev) {
    const int32_t g = R.randint(1, cfg.max_gap);
    if (n < cap) { sk[n] = (uint8_t)ev; sg[n] = g; gaps += g; n++; } else overflow = true;
  };
  if (threadIdx.x == 0) TL_STAMP(4);
  sc.tail = R.randint(1, cfg.max_tail);                                  // :372
  sc.initial_grasped = 0;
  sc.initial_contact = 0;
  sc.initial_dist_obj_goal = 0.5;
  sc.initial_level = TL_LVL_LOW;
  sc.art_kind = TL_ART_FRIDGE;
  sc.arm_dof = 7;
  sc.subtask = kind;
  if (kind == TL_OPEN || kind == TL_CLOSE)                               // :374-376
    sc.art_kind = R.randbelow(2) ? TL_ART_DRAWER : TL_ART_FRIDGE;
  if (kind == TL_PICK) {                                                 // :379-381
    sc.initial_contact = R.random() < 0.25;
    sc.initial_grasped = sc.initial_contact && R.random() < 0.4;
  } else if (kind == TL_PLACE) {                                         // :382-386
    sc.initial_grasped = R.random() < 0.8;
    sc.initial_dist_obj_goal = R.random() < 0.7 ? R.uniform(0.3, 0.9) : R.uniform(0.02, 0.12);
  } else {                                                               // :387-392
    const double w[3] = {0.85, 0.1, 0.05};
    const int c = choices_idx(R, w);
    if (kind == TL_OPEN) sc.initial_level = c == 0 ? TL_LVL_LOW : c == 1 ? TL_LVL_SLIGHT : TL_LVL_OPEN;
    else sc.initial_level = c == 0 ? TL_LVL_HIGH : c == 1 ? TL_LVL_SLIGHT : TL_LVL_CLOSED;
  }
  bool grasped = sc.initial_grasped, contact = sc.initial_contact;       // :394-403
  bool in_goal = sc.initial_dist_obj_goal <= 0.15;
  int level = sc.initial_level;
  bool band = true;
  if (kind == TL_CLOSE) {
    level = sc.initial_level == TL_LVL_CLOSED ? TL_LVL_CLOSED : TL_LVL_OPEN;
    band = sc.initial_level != TL_LVL_CLOSED;
  }
  bool contact_used = contact;                                           // :461
  const long n_target = (long)rint(__dmul_rn((double)R.randint(0, cfg.max_events), cfg.edge_density));
  if (threadIdx.x == 0) TL_STAMP(5);
  for (long it = 0; it < n_target; it++) {                               // :464-474
    // the legal moves (at most 3), packed one byte each into a register
    // (no local-memory array): move i = (mv >> 8i) & 0xff
    uint32_t mv = 0;
    int nm = 0;
    auto add = [&](int ev) { mv |= (uint32_t)ev << (8 * nm); nm++; };
    if (kind == TL_PICK) {
      if (!contact) add(TL_EV_CONTACT);
      if (!grasped && contact) add(TL_EV_GRASPED);
      if (grasped) add(TL_EV_DROPPED);
    } else if (kind == TL_PLACE) {
      add(!grasped ? TL_EV_GRASPED : in_goal ? TL_EV_RELEASED_AT_GOAL : TL_EV_RELEASED_OUTSIDE_GOAL);
      add(in_goal ? TL_EV_OBJ_LEFT_GOAL : TL_EV_OBJ_AT_GOAL);
    } else if (kind == TL_OPEN) {
      if (!contact_used) add(TL_EV_CONTACT);  // Contact is dropped once used (:416-419)
      add(level == TL_LVL_LOW ? TL_EV_SLIGHTLY_OPENED : level == TL_LVL_SLIGHT ? TL_EV_OPENED : TL_EV_CLOSED);
    } else {
      if (!contact_used) add(TL_EV_CONTACT);
      if (level == TL_LVL_OPEN) { if (band) add(TL_EV_SLIGHTLY_CLOSED); }
      else if (level == TL_LVL_SLIGHT) add(TL_EV_CLOSED);
      else add(TL_EV_OPEN);
    }
    if (!nm) break;
    const int m = (int)((mv >> (8 * R.randbelow((uint32_t)nm))) & 0xffu);
    if (m == TL_EV_CONTACT) contact_used = true;
    push(m);
    switch (m) {                                                         // :434-457
      case TL_EV_CONTACT: contact = true; break;
      case TL_EV_GRASPED: grasped = true; break;
      case TL_EV_DROPPED: grasped = false; contact = false; break;
      case TL_EV_RELEASED_AT_GOAL: case TL_EV_RELEASED_OUTSIDE_GOAL: grasped = false; break;
      case TL_EV_OBJ_AT_GOAL: in_goal = true; break;
      case TL_EV_OBJ_LEFT_GOAL: in_goal = false; break;
      case TL_EV_SLIGHTLY_OPENED: level = TL_LVL_SLIGHT; break;
      case TL_EV_OPENED: level = TL_LVL_OPEN; break;
      case TL_EV_CLOSED: level = kind == TL_OPEN ? TL_LVL_LOW : TL_LVL_CLOSED; break;
      case TL_EV_SLIGHTLY_CLOSED: level = TL_LVL_SLIGHT; break;
      case TL_EV_OPEN: level = TL_LVL_OPEN; break;
    }
  }
  if (threadIdx.x == 0) TL_STAMP(6);
  bool feasible;                                                         // :476-483
  if (kind == TL_PICK) feasible = grasped;
  else if (kind == TL_PLACE) feasible = !grasped && in_goal;
  else if (kind == TL_OPEN) feasible = level == TL_LVL_OPEN;
  else feasible = level == TL_LVL_CLOSED;
  const bool want = cfg.edge_density > 0 && R.random() < cfg.success_prob;  // :485
  if (want && feasible) {
    push(TL_EV_SUCCESS);
    const double w[4] = {0.55, 0.2, 0.15, kind == TL_PLACE ? 0.1 : 0.0};
    const int suffix = choices_idx(R, w);
    if (suffix == 1) {
      // the dict literal at :493-496 evaluates gap() for all four subtasks
      int32_t g[4];
      for (int i = 0; i < 4; i++) g[i] = R.randint(1, cfg.max_gap);
      const int brk = kind == TL_PICK ? TL_EV_DROPPED : kind == TL_PLACE ? TL_EV_OBJ_LEFT_GOAL
                    : kind == TL_OPEN ? TL_EV_CLOSED : TL_EV_OPEN;
      if (n < cap) { sk[n] = (uint8_t)brk; sg[n] = g[kind]; gaps += g[kind]; n++; } else overflow = true;
    } else if (suffix == 2) {
      push(TL_EV_EXCESSIVE_COLLISIONS);
    } else if (suffix == 3) {
      push(TL_EV_OBJ_LEFT_GOAL);
      push(TL_EV_OBJ_AT_GOAL);
      push(TL_EV_SUCCESS);
    }
  } else if (cfg.edge_density > 0 && R.random() < 0.15) {               // :504-505
    push(TL_EV_EXCESSIVE_COLLISIONS);
  }
  if (threadIdx.x == 0) TL_STAMP(7);
  sc.n_steps = n;
  return overflow ? -1 : n;
}

// _Realizer.__init__ constants (synth.py:104-148), all lanes
__device__ __forceinline__ int realizer_init(RzConst& z, const tl_script& sc,
                                             const tl_thresholds& th, int dof) {
  const int k = sc.subtask;
  z.kind = k;
  z.dof = dof;
  z.ne = 2 * dof + 5;
  z.has_art = k == TL_OPEN || k == TL_CLOSE;
  z.has_goal = k == TL_PLACE;
  z.has_force = k != TL_PLACE;
  z.limit = k == TL_PICK ? th.coll_pick : k == TL_PLACE ? th.coll_place : th.coll_artic;
  z.L09 = __dmul_rn(z.limit, 0.9);
  z.L105 = __dmul_rn(z.limit, 1.05);
  z.goal = th.goal_radius;
  z.qmin = z.qmax = z.closed_thresh = z.sc_thresh = 0.0;
  z.lv_low = z.lv_slight = z.lv_open = z.a_q0 = z.sc_art = 0.0;
  z.band_valid = 0;
  if (z.has_art) {
    if (sc.art_kind == TL_ART_FRIDGE) { z.qmin = 0.0; z.qmax = 1.6; }
    else if (sc.art_kind == TL_ART_DRAWER) { z.qmin = 0.0; z.qmax = 0.5; }
    else return TL_INF_INIT_LEVEL;
    const double span = __dsub_rn(z.qmax, z.qmin);
    const double ofrac = sc.art_kind == TL_ART_FRIDGE ? th.open_frac_fridge : th.open_frac_drawer;
    const double open_t = __dadd_rn(__dmul_rn(ofrac, span), z.qmin);
    z.closed_thresh = __dadd_rn(__dmul_rn(th.close_frac, span), z.qmin);
    const double so_t = __dadd_rn(__dmul_rn(th.slightly_open_frac, span), z.qmin);
    if (k == TL_OPEN) {
      z.lv_low = z.qmin;
      z.lv_slight = __ddiv_rn(__dadd_rn(so_t, open_t), 2.0);
      z.lv_open = __ddiv_rn(__dadd_rn(open_t, z.qmax), 2.0);
      if (sc.initial_level != TL_LVL_LOW && sc.initial_level != TL_LVL_SLIGHT &&
          sc.initial_level != TL_LVL_OPEN) return TL_INF_INIT_LEVEL;
    } else {
      if (sc.initial_level == TL_LVL_HIGH) z.a_q0 = z.qmax;
      else if (sc.initial_level == TL_LVL_SLIGHT) z.a_q0 = __dadd_rn(z.qmin, __dmul_rn(0.3, span));
      else if (sc.initial_level == TL_LVL_CLOSED) z.a_q0 = z.qmin;
      else return TL_INF_INIT_LEVEL;
      z.sc_thresh = __dsub_rn(z.a_q0, __dmul_rn(th.slightly_close_frac, span));
      z.band_valid = z.sc_thresh > z.closed_thresh;
      z.sc_art = __ddiv_rn(__dadd_rn(z.sc_thresh, z.closed_thresh), 2.0);
    }
  }
  if (k == TL_PICK && sc.initial_grasped && !sc.initial_contact)        // :154-155
    return TL_INF_PICK_GRASPED_NO_CONTACT;
  return TL_OK;
}

// deterministic part of _apply (synth.py:205-296) on the plan state.
// Value-dependent checks (object distance vs goal) are deferred to the
// event record (chunk pass).  Returns 0 or an InfeasibleScript code.
struct PlanSt {
  double force, art;
  int grasped, at_rest, exc, level;
};

__device__ int plan_apply(const RzConst& z, PlanSt& p, int ev, int& draw) {
  const int k = z.kind;
  draw = 0;
  if (!in_alpha(k, ev)) return TL_INF_NOT_IN_ALPHABET;
  if (ev == TL_EV_EXCESSIVE_COLLISIONS) {
    if (p.exc) return TL_INF_LIMIT_EXCEEDED;  // cum = 1.05*limit > limit
    p.exc = 1;
    return 0;
  }
  if (ev == TL_EV_SUCCESS) {
    bool ok;
    if (k == TL_PICK) ok = p.grasped;
    else if (k == TL_PLACE) ok = !p.grasped;  // and dist <= goal (deferred)
    else if (k == TL_OPEN) ok = p.level == TL_LVL_OPEN;
    else ok = p.level == TL_LVL_CLOSED;
    if (!ok || p.at_rest) return TL_INF_SUCCESS_UNREACHABLE;
    p.at_rest = 1;
    return 0;
  }
  p.at_rest = 0;
  switch (ev) {
    case TL_EV_CONTACT:
      if (!z.has_force) return TL_INF_CONTACT_UNDEFINED;
      if (p.force > 0) return TL_INF_CONTACT_AGAIN;
      p.force = 1.2;
      return 0;
    case TL_EV_GRASPED:
      if (p.grasped) return TL_INF_GRASPED_AGAIN;
      if (k == TL_PICK && p.force == 0) return TL_INF_PICK_GRASP_NO_FORCE;
      p.grasped = 1;
      return 0;
    case TL_EV_DROPPED:
      if (!p.grasped) return TL_INF_DROPPED_NOT_GRASPED;
      p.grasped = 0;
      p.force = 0.0;
      return 0;
    case TL_EV_OBJ_AT_GOAL:
    case TL_EV_OBJ_LEFT_GOAL:
      draw = 1;
      return 0;
    case TL_EV_RELEASED_AT_GOAL:
      if (!p.grasped) return TL_INF_RAG;
      p.grasped = 0;
      return 0;
    case TL_EV_RELEASED_OUTSIDE_GOAL:
      if (!p.grasped) return TL_INF_ROG;
      p.grasped = 0;
      return 0;
    case TL_EV_SLIGHTLY_OPENED:
      if (k != TL_OPEN || p.level != TL_LVL_LOW) return TL_INF_SLIGHTLY_OPENED;
      p.level = TL_LVL_SLIGHT;
      p.art = z.lv_slight;
      return 0;
    case TL_EV_OPENED:
      if (k != TL_OPEN || p.level != TL_LVL_SLIGHT) return TL_INF_OPENED;
      p.level = TL_LVL_OPEN;
      p.art = z.lv_open;
      return 0;
    case TL_EV_CLOSED:
      if (k == TL_OPEN) {
        if (p.level != TL_LVL_OPEN) return TL_INF_CLOSED_OPEN;
        p.level = TL_LVL_LOW;
        p.art = z.lv_low;
        return 0;
      }
      if (p.level != TL_LVL_SLIGHT) return TL_INF_CLOSED_CLOSE;
      p.level = TL_LVL_CLOSED;
      p.art = z.qmin;
      return 0;
    case TL_EV_SLIGHTLY_CLOSED:
      if (p.level != TL_LVL_OPEN) return TL_INF_SC_LEVEL;
      if (!z.band_valid) return TL_INF_SC_BAND;
      p.level = TL_LVL_SLIGHT;
      p.art = z.sc_art;
      return 0;
    case TL_EV_OPEN:
      if (p.level != TL_LVL_CLOSED) return TL_INF_OPEN_CLOSE;
      p.level = TL_LVL_OPEN;
      p.art = z.a_q0 > z.closed_thresh ? z.a_q0 : z.qmax;
      return 0;
  }
  return TL_INF_NOT_IN_ALPHABET;
}

__device__ __forceinline__ StepSt make_st(const RzConst& z, const PlanSt& p, int last_draw) {
  StepSt s;
  s.force = z.has_force ? __double2float_rn(p.force) : __int_as_float(0x7fc00000);
  s.art = z.has_art ? __double2float_rn(p.art) : __int_as_float(0x7fc00000);
  s.grasped = (uint8_t)p.grasped;
  s.at_rest = (uint8_t)p.at_rest;
  s.exc = (uint8_t)p.exc;
  s.level = (uint8_t)p.level;
  s.last_draw = (int16_t)last_draw;
  s.pad = 0;
  return s;
}

// random_script + the episode's script record, length bucket and record
// layout (one thread; R = the freshly seeded script RNG).  Returns the
// episode's length bucket; with place_order the thread also takes its slot
// in the longest-first order by a global atomic (else the caller does,
// aggregated per CTA).
__device__ __forceinline__ int reset_script(const SynthParams& p, int64_t e, int64_t seed,
                                            MtLane& R, bool place_order = true) {
  const int ms = p.cfg.max_events + 4;
  tl_script t;
  uint8_t* sk = p.step_kind + e * ms;
  int32_t* sg = p.step_gap + e * ms;
  // at most max_events + 4 = ms steps are ever produced (synth.py:463-505)
  int64_t gaps = 0;
  const int sub = p.subtasks ? (int)p.subtasks[e] : p.fuzz_subtask;
  int ns = -1;
  int64_t nr = 2;
  if (sub >= 0 && sub <= 3) {
    ns = sample_script(R, sub, p.cfg, sk, sg, t, ms, gaps);
    nr = 1 + (ns < 0 ? 0 : gaps);
    const int64_t tmin = ns > 0 ? 0 : 1;
    nr += t.tail > tmin ? t.tail : tmin;
    if (nr < 2) nr = 2;
  } else {
    memset(&t, 0, sizeof(t));
  }
  t.step_off = e * ms;
  t.seed = seed ^ 0x5EED;
  // -1: capacity error, -2: no such subtask (a per-episode TL_E_INVALID)
  t.n_steps = (sub < 0 || sub > 3) ? -2 : (ns < 0 || nr > p.cap_per_env) ? -1 : ns;
  p.scripts[e] = t;
  // length bucket for the realize kernel's longest-first claims
  const int b = t.n_steps < 0 ? 0 : (int)min((int64_t)kLenBuckets - 1, (nr - 1) / kBucketRecs);
  if (p.order && place_order) {
    const unsigned slot = atomicAdd(&p.tickets[kTkBucket + b], 1u);
    p.order[(int64_t)b * p.n_env + slot] = (int32_t)e;
  }
  if (e < p.ev_zero) p.ev_state[e] = 0ull;  // k_scan_emit tile state of this launch
  if (p.out.rec_start) {  // record layout (tl_fuzz); the env reset has none
    p.out.rec_start[e] = e * p.cap_per_env;
    p.out.n_rec[e] = t.n_steps < 0 ? 0 : (int)nr;
  }
  return b;
}

__device__ __forceinline__ void reset_counters(const SynthParams& p) {
  p.tickets[0] = 0u;  // episode claims
  for (int i = p.n_env; i < p.ev_zero; i++) p.ev_state[i] = 0ull;  // tiny batches
}

// ---- reset: seeding + random_script, one thread per RNG ---------------------
// CPython seeding is a 1247-step serial chain per state, so it runs one
// state per thread (32 chains per warp) into padded shared-memory rows
// (stride 625 words: conflict-free), instead of occupying one lane of an
// episode's warp.  Fuzz: even lanes seed the script RNG (seed) and sample
// random_script; odd lanes seed the realize RNG (seed ^ 0x5EED, synth.py:515).
constexpr int kRowWords = kMtN + 1;

// EPW episodes per warp: lanes 2j / 2j+1 own episode j (script RNG +
// random_script / realize RNG).  EPW = 1 for small (latency-bound) batches:
// sampling is serial branchy code, and 16 samplers in one warp diverge.
// STREAM: both lanes seed with mt_seed_lane_stream (no working row), so only
// the script lane's final state needs shared memory: EPW rows instead of
// 2*EPW, twice the warps per SM where shared memory sets the occupancy.
template <int EPW, bool STREAM>
__global__ void __launch_bounds__(32) k_fuzz_reset(SynthParams p) {
  extern __shared__ uint32_t rows[];  // [2*EPW or EPW (STREAM)][kRowWords]
  const int lane = lane_id();
  const int64_t e0 = (int64_t)blockIdx.x * EPW;
  const int64_t e = e0 + (lane >> 1);
  const bool valid = (lane >> 1) < EPW && e < p.n_env;
  uint32_t* row = STREAM ? rows + (lane < 2 * EPW ? lane >> 1 : 0) * kRowWords
                         : rows + (lane < 2 * EPW ? lane : 0) * kRowWords;
  if (lane == 0) TL_STAMP(0);
  if (blockIdx.x == 0 && lane == 0 && p.tickets) reset_counters(p);
  if (valid) {
    const int64_t seed = p.seeds[e];
    // odd lanes: realize RNG, final state written straight to global memory
    if (STREAM)
      mt_seed_lane_stream((lane & 1) ? (seed ^ 0x5EED) : seed,
                          (lane & 1) ? p.states + e * kMtN : row);
    else
      mt_seed_lane(row, (lane & 1) ? (seed ^ 0x5EED) : seed,
                   (lane & 1) ? p.states + e * kMtN : nullptr);
    if (lane == 0) TL_STAMP(1);
    if (!(lane & 1)) {
      MtLane R{row, 0, 0};
      R.prepare(128);
      reset_script(p, e, seed, R);
    }
  }
  if (lane == 0) TL_STAMP(2);
}

#ifdef TL_AB
// Latency form (batches up to a few episodes per SM): a CTA of E warps owns E
// episodes.  Warp 0 seeds all 2E states (lane 2j: script RNG of episode j into
// shared row j, lane 2j+1: realize RNG straight to global memory), so the
// 1247-step chains cost one warp of issue per CTA; then warp j regenerates
// episode j's first MT block with all 32 lanes and its lane 0 samples
// random_script from it -- one sampler per warp, no divergence between
// episodes' branchy sampling code.
template <int E>
__global__ void __launch_bounds__(E * 32) k_fuzz_reset_w(SynthParams p) {
  static_assert(E >= 1 && E <= 16, "2E seeding lanes in one warp");
  extern __shared__ uint32_t rows[];  // [E][kRowWords] states, then [E][kMtN] tempered words
  const int warp = threadIdx.x >> 5, lane = lane_id();
  const int64_t e0 = (int64_t)blockIdx.x * E;
  if (blockIdx.x == 0 && threadIdx.x == 0 && p.tickets) reset_counters(p);
  if (threadIdx.x == 0) TL_STAMP(0);
  if (warp == 0) {
    const int j = lane >> 1;
    const int64_t e = e0 + j;
    if (j < E && e < p.n_env) {
      const int64_t seed = p.seeds[e];
      mt_seed_lane_stream((lane & 1) ? (seed ^ 0x5EED) : seed,
                          (lane & 1) ? p.states + e * kMtN : rows + j * kRowWords);
    }
  }
  if (threadIdx.x == 0) TL_STAMP(1);
  __syncthreads();
  const int64_t e = e0 + warp;
  if (e >= p.n_env) return;
  MtLane R{rows + warp * kRowWords, 0, 0};
  R.prepare_block_warp((E - warp) * kRowWords + warp * kMtN);
  if (threadIdx.x == 0) TL_STAMP(2);
  if (lane == 0) reset_script(p, e, p.seeds[e], R);
  if (threadIdx.x == 0) TL_STAMP(3);
}
#endif

// The same with both states streamed into shared rows 2j / 2j+1 (every
// seeding store is a shared-space store: no generic stores splitting
// between shared and global memory inside the 624-step loops), then the warp
// copies the realize rows to global memory, coalesced, while nothing else
// waits on them; the even lanes then sample random_script.
template <int EPW>
__global__ void __launch_bounds__(32) k_fuzz_reset_sh(SynthParams p) {
  extern __shared__ uint32_t rows[];  // [2*EPW][kRowWords]
  const int lane = lane_id();
  const int64_t e0 = (int64_t)blockIdx.x * EPW;
  const int64_t e = e0 + (lane >> 1);
  const bool valid = (lane >> 1) < EPW && e < p.n_env;
  uint32_t* row = rows + (lane < 2 * EPW ? lane : 0) * kRowWords;
  if (lane == 0) TL_STAMP(0);
  if (blockIdx.x == 0 && lane == 0 && p.tickets) reset_counters(p);
  int64_t seed = 0;
  if (valid) {
    seed = p.seeds[e];
    const int64_t s = (lane & 1) ? (seed ^ 0x5EED) : seed;
    const uint64_t n = s < 0 ? (uint64_t)0 - (uint64_t)s : (uint64_t)s;
    const uint32_t k0 = (uint32_t)n, k1 = (uint32_t)(n >> 32);
    if (k1) mt_seed_stream_impl<2>(k0, k1, row);
    else mt_seed_stream_impl<1>(k0, 0u, row);
  }
  __syncwarp();
  if (lane == 0) TL_STAMP(1);
  const int ne = (int)min((int64_t)EPW, (int64_t)p.n_env - e0);
  for (int q = 0; q < ne; q++) {
    const uint32_t* src = rows + (2 * q + 1) * kRowWords;
    uint32_t* dst = p.states + (e0 + q) * kMtN;
#pragma unroll 4
    for (int i = lane; i < kMtN; i += 32) dst[i] = src[i];
  }
  if (valid && !(lane & 1)) {
    MtLane R{row, 0, 0};
    R.prepare(128);
    reset_script(p, e, seed, R);
  }
  if (lane == 0) TL_STAMP(2);
}

// Mid-size batches: a CTA of E warps owns E episodes.  Warp 0 seeds all 2E
// states into shared rows (lane 2j: script RNG of episode j, 2j+1: realize
// RNG; shared-space stores only), the E warps copy the realize rows out
// (coalesced) and regenerate their episode's first MT block (32 lanes,
// tempered copy), then lane 0 of warp j samples random_script -- one sampler
// per warp, no divergence between episodes -- and takes its longest-first slot.
template <int E>
__global__ void __launch_bounds__(E * 32) k_fuzz_reset_cta(SynthParams p) {
  static_assert(E >= 1 && E <= 16, "2E seeding lanes in one warp");
  // [2E][kRowWords]: the realize rows (odd) take the tempered words once copied out
  extern __shared__ uint32_t rows[];
  const int warp = threadIdx.x >> 5, lane = lane_id();
  const int64_t e0 = (int64_t)blockIdx.x * E;
  TL_BLOCK_SPAN(0);
  if (blockIdx.x == 0 && threadIdx.x == 0 && p.tickets) reset_counters(p);
  if (threadIdx.x == 0) TL_STAMP(0);
  if (warp == 0) {
    const int j = lane >> 1;
    const int64_t e = e0 + j;
    if (j < E && e < p.n_env) {
      const int64_t seed = p.seeds[e];
      const int64_t sd = (lane & 1) ? (seed ^ 0x5EED) : seed;
      const uint64_t n = sd < 0 ? (uint64_t)0 - (uint64_t)sd : (uint64_t)sd;
      const uint32_t k0 = (uint32_t)n, k1 = (uint32_t)(n >> 32);
      uint32_t* row = rows + lane * kRowWords;
      // one chain in place (loop 2 reads loop 1 back from the row): 5 ops per
      // step on the critical path, fewer issued per step than the streamed
      // two-chain form (reset block 37.4k -> 33.6k cycles at 4096 episodes)
      if (k1) mt_seed_impl<2>(row, k0, k1, row);
      else mt_seed_impl<1>(row, k0, 0u, row);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) TL_STAMP(1);
  const int64_t e = e0 + warp;
  if (e < p.n_env) {
    {  // the realize state of this warp's episode, out to global memory
      const uint32_t* src = rows + (2 * warp + 1) * kRowWords;
      uint32_t* dst = p.states + e * kMtN;
#pragma unroll 4
      for (int i = lane; i < kMtN; i += 32) dst[i] = src[i];
    }
    __syncwarp();  // the row is read out before it takes the tempered words
    MtLane R{rows + 2 * warp * kRowWords, 0, 0};
    // the sampler reads ~40 words: regenerate the first 128 with 32 lanes,
    // the rest lazily (a full-block prepare and a CTA-wide order aggregation
    // measured 9k cycles slower per CTA, scripts/reset_probe_env.sh)
    R.prepare_prefix_warp<128>(kRowWords);  // tempered copies into the realize row
    if (threadIdx.x == 0) TL_STAMP(2);
    if (lane == 0) reset_script(p, e, p.seeds[e], R, true);  // its own longest-first slot
  }
  if (threadIdx.x == 0) TL_STAMP(3);
}

// realize path: seed the realize RNG of given scripts (one thread per state,
// streamed straight to global memory: no shared memory)
__global__ void __launch_bounds__(128) k_seed_states(SynthParams p) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e == 0 && p.tickets) {
    p.tickets[0] = 0u;
  }
  if (e < p.n_env) mt_seed_lane_stream(p.scripts[e].seed, p.states + e * kMtN);
}

}  // namespace tl
