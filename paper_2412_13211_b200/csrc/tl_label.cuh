// tl_label.cuh -- predicates, edge-triggered events and mode classification.
//
// Reference (paths under /root/reference/pkg/src/trajlab/):
//   predicates.py:16-99   j_max / is_static / _at_rest / success_step
//   events.py:94-193      extract_events (edge tests in EVENT_ORDER)
//   modes.py:24-253       last_index / _Ctx / rule tables / classify
//
// Mapping: one warp per episode; f32 episodes at arm_dof 7 with aligned
// slots take the vector bodies (4 consecutive records per lane, 128-record
// chunks, k_label<float,7,1>), everything else one record per lane (32-record
// chunks).  Each lane evaluates its records' indicator bits; the previous record's
// bits arrive by __shfl_up (carry across chunks); events are the per-step
// bitmask in EVENT_ORDER bit order.  The event list itself is never stored
// here: classification needs only |E|, the last index of each kind and d0
// (modes.py:42-61), kept as warp-uniform registers (ballot + clz + scan).
//
// Numerics: the reference compares binary32 record values widened to f64
// against f64 thresholds.  For f32 records every such compare is done
// exactly in f32 against a directed-rounding cut (tl_cset, host-built):
//   x <= T <=> x <= rd(T),  x > T <=> x > rd(T),  x >= T <=> x >= ru(T),
//   x < T <=> x < ru(T).
// Differences against a nonzero rest posture (j_max, torso) are f64.
// f64 records (arbitrary doubles, e.g. text logs) use f64 compares.
#pragma once
#include "tl_common.cuh"

namespace tl {

// ---- comparison overloads: f32 value vs cut, f64 value vs threshold -------
__device__ __forceinline__ bool LE(float x, float c, double) { return x <= c; }
__device__ __forceinline__ bool LE(double x, float, double t) { return x <= t; }
__device__ __forceinline__ bool GT(float x, float c, double) { return x > c; }
__device__ __forceinline__ bool GT(double x, float, double t) { return x > t; }
__device__ __forceinline__ bool GE(float x, float c, double) { return x >= c; }
__device__ __forceinline__ bool GE(double x, float, double t) { return x >= t; }
__device__ __forceinline__ bool LT(float x, float c, double) { return x < c; }
__device__ __forceinline__ bool LT(double x, float, double t) { return x < t; }
__device__ __forceinline__ float tabs(float x) { return fabsf(x); }
__device__ __forceinline__ double tabs(double x) { return fabs(x); }

// indicator bits of one record
enum : uint32_t {
  IND_CONTACT = 1u, IND_GRASPED = 2u, IND_SUCCESS = 4u, IND_CUM_LE = 8u,
  IND_CUM_GT = 16u, IND_A = 32u, IND_B = 64u
};
// per-record error bits
enum : uint32_t { ERR_SUCC = 1u, ERR_FORCE = 2u, ERR_DIST = 4u, ERR_ART = 8u };

// Python max() over a generator of |v_i| (a leading NaN sticks, later NaNs
// never win): m = v0; m = v if v > m.
template <class T>
__device__ __forceinline__ T pymax_step(T m, T v) { return v > m ? v : m; }

// Record values the predicates need (lane-private).
template <class T>
struct RecV {
  T der, dist, force, cum, art, tor, vx, vy, om, qdm;
  T jm;          // Python-max |q_i - rest_i| when rest is zero (T path)
  double jm_d;   // same, f64, for a nonzero rest posture
  bool g;
};

// _at_rest (predicates.py:64-72)
template <class T>
__device__ __forceinline__ bool at_rest(const tl_cset& c, const RecV<T>& v, bool torso) {
  if (GT(v.der, c.rd_rest_radius, c.rest_radius)) return false;
  const bool jm_over = c.rest_zero ? GT(v.jm, c.rd_j_arm, c.j_arm) : (v.jm_d > c.j_arm);
  if (jm_over) return false;
  if (torso) {
    const bool tor_over = c.rest_zero
                              ? GT(tabs(v.tor), c.rd_j_tor, c.j_tor)
                              : (fabs(__dsub_rn((double)v.tor, c.rest_tor)) > c.j_tor);
    if (tor_over) return false;
  }
  // is_static (predicates.py:23-27)
  return LE(v.qdm, c.rd_static_qd, c.static_qd) &&
         LE(tabs(v.vx), c.rd_static_v, c.static_v) &&
         LE(tabs(v.vy), c.rd_static_v, c.static_v) &&
         LE(tabs(v.om), c.rd_static_om, c.static_om);
}

// success_step (predicates.py:75-94) + the per-record indicator bits used by
// extract_events (events.py:103-190).  sc_* is the Close slightly-closed cut
// anchored at records[0].art_q (events.py:174-176).
template <class T>
__device__ __forceinline__ void record_bits(const tl_cset& c, const RecV<T>& v,
                                            float sc_ru, double sc_d,
                                            uint32_t& ind, uint32_t& err) {
  const bool over = GT(v.cum, c.rd_limit, c.limit);
  ind = (LE(v.cum, c.rd_limit, c.limit) ? IND_CUM_LE : 0u) | (over ? IND_CUM_GT : 0u);
  err = 0u;
  bool succ = false;
  switch (c.subtask) {
    case TL_PICK:
      succ = !over && v.g && at_rest(c, v, false);
      ind |= (GT(v.force, c.rd_contact, c.contact_eps) ? IND_CONTACT : 0u) |
             (v.g ? IND_GRASPED : 0u);
      err |= isnan(v.force) ? ERR_FORCE : 0u;
      break;
    case TL_PLACE: {
      const bool in = LE(v.dist, c.rd_goal, c.goal_radius);
      if (!over && !v.g && isnan(v.dist)) err |= ERR_SUCC;
      succ = !over && !v.g && in && at_rest(c, v, true);
      ind |= (v.g ? IND_GRASPED : 0u) | (in ? IND_A : 0u) |
             (GT(v.dist, c.rd_goal, c.goal_radius) ? IND_B : 0u);
      err |= isnan(v.dist) ? ERR_DIST : 0u;
      break;
    }
    case TL_OPEN: {
      const bool has_art = c.art_kind != TL_ART_NONE;
      if (!over && (!has_art || isnan(v.art))) err |= ERR_SUCC;
      const bool open = GE(v.art, c.ru_open, c.open_cut);
      succ = !over && has_art && open && at_rest(c, v, true);
      ind |= (GT(v.force, c.rd_contact, c.contact_eps) ? IND_CONTACT : 0u) |
             (open ? IND_A : 0u) |
             (GE(v.art, c.ru_slight_open, c.slight_open_cut) ? IND_B : 0u);
      err |= (isnan(v.force) ? ERR_FORCE : 0u) | (isnan(v.art) ? ERR_ART : 0u);
      break;
    }
    default: {  // TL_CLOSE
      const bool has_art = c.art_kind != TL_ART_NONE;
      if (!over && (!has_art || isnan(v.art))) err |= ERR_SUCC;
      const bool closed = LE(v.art, c.rd_closed, c.closed_cut);
      succ = !over && has_art && closed && at_rest(c, v, true);
      ind |= (GT(v.force, c.rd_contact, c.contact_eps) ? IND_CONTACT : 0u) |
             (closed ? IND_A : 0u) | (LT(v.art, sc_ru, sc_d) ? IND_B : 0u);
      err |= (isnan(v.force) ? ERR_FORCE : 0u) | (isnan(v.art) ? ERR_ART : 0u);
      break;
    }
  }
  if (succ) ind |= IND_SUCCESS;
}

// record_bits split at cum_robot_force: the bits computed with `over` =
// false (cum_patch_bits then applies the real cum).  Exact because every
// success / ERR_SUCC condition of record_bits is conjoined with !over and
// the cum bits depend on nothing else.
__device__ __forceinline__ uint32_t cum_patch_bits(const tl_cset& c, float cum, uint32_t ind,
                                                   uint32_t& err) {
  const bool over = GT(cum, c.rd_limit, c.limit);
  if (over) {
    ind &= ~IND_SUCCESS;
    err &= ~ERR_SUCC;
  }
  return (ind & ~(IND_CUM_LE | IND_CUM_GT)) | (LE(cum, c.rd_limit, c.limit) ? IND_CUM_LE : 0u) |
         (over ? IND_CUM_GT : 0u);
}

// edge tests of extract_events in EVENT_ORDER bit order
__device__ __forceinline__ uint32_t edge_mask(int subtask, uint32_t p, uint32_t c) {
  const uint32_t rise = ~p & c, fall = p & ~c;
  const uint32_t C = (rise & IND_CONTACT) ? 1u : 0u;
  const uint32_t G = (rise & IND_GRASPED) ? 1u : 0u;
  const uint32_t D = (fall & IND_GRASPED) ? 1u : 0u;
  const uint32_t S = (rise & IND_SUCCESS) ? 1u : 0u;
  const uint32_t X = ((p & IND_CUM_LE) && (c & IND_CUM_GT)) ? 1u : 0u;
  const uint32_t Ar = (rise & IND_A) ? 1u : 0u, Af = (fall & IND_A) ? 1u : 0u;
  const uint32_t Br = (rise & IND_B) ? 1u : 0u;
  switch (subtask) {
    case TL_PICK:  // Contact, Grasped, Dropped, Success, ExcessiveCollisions
      return C | (G << 1) | (D << 2) | (S << 3) | (X << 4);
    case TL_PLACE: {  // Grasped, ObjAtGoal, RAG, ROG, ObjLeftGoal, Success, X
      const uint32_t oag = ((p & IND_B) && (c & IND_A)) ? 1u : 0u;
      const uint32_t olg = ((p & IND_A) && (c & IND_B)) ? 1u : 0u;
      const uint32_t rag = (D && (c & IND_A)) ? 1u : 0u;
      const uint32_t rog = (D && !(c & IND_A)) ? 1u : 0u;
      return G | (oag << 1) | (rag << 2) | (rog << 3) | (olg << 4) | (S << 5) | (X << 6);
    }
    default:  // Open: Contact, Opened, SlightlyOpened, Closed, Success, X
              // Close: Contact, Closed, SlightlyClosed, Open, Success, X
      return C | (Ar << 1) | (Br << 2) | (Af << 3) | (S << 4) | (X << 5);
  }
}

__device__ __forceinline__ int alphabet_size(int subtask) {
  return subtask == TL_PICK ? 5 : subtask == TL_PLACE ? 7 : 6;
}

// warp-uniform running label state of one episode
struct LState {
  int size;
  int last[7];
  uint32_t prev_ind;
  uint32_t err_any;
};

__device__ __forceinline__ void lstate_init(LState& S) {
  S.size = 0;
#pragma unroll
  for (int k = 0; k < 7; k++) S.last[k] = -1;
  S.prev_ind = 0;
  S.err_any = 0;
}

// fold one chunk's per-lane event masks into the running state
__device__ __forceinline__ void lstate_fold(LState& S, uint32_t mask, uint32_t err) {
  const int cnt = __popc(mask);
  const int incl = warp_incl_scan(cnt);
  const int excl = incl - cnt;
#pragma unroll
  for (int k = 0; k < 7; k++) {
    const unsigned bal = __ballot_sync(kFull, (mask >> k) & 1u);
    if (bal) {
      const int L = 31 - __clz(bal);
      const int exL = __shfl_sync(kFull, excl, L);
      const uint32_t mL = __shfl_sync(kFull, mask, L);
      S.last[k] = S.size + exL + __popc(mL & ((1u << k) - 1u));
    }
  }
  S.size += __shfl_sync(kFull, incl, 31);
  S.err_any |= __reduce_or_sync(kFull, err);
}

// ---- classification (modes.py) ---------------------------------------------
struct Sig {
  int size, c, g, d, oag, rag, rog, olg, opened, so, closed, sc, open, s, x;
  double d0;
  bool d0_none, s1;
};

__device__ __forceinline__ void sig_clear(Sig& z) {
  z.size = 0;
  z.c = z.g = z.d = z.oag = z.rag = z.rog = z.olg = z.opened = z.so = z.closed =
      z.sc = z.open = z.s = z.x = -1;
  z.d0 = 0.0;
  z.d0_none = false;
  z.s1 = false;
}

__device__ __forceinline__ void sig_set(Sig& z, int kind, int idx) {
  switch (kind) {
    case TL_EV_CONTACT: z.c = idx; break;
    case TL_EV_GRASPED: z.g = idx; break;
    case TL_EV_DROPPED: z.d = idx; break;
    case TL_EV_OBJ_AT_GOAL: z.oag = idx; break;
    case TL_EV_RELEASED_AT_GOAL: z.rag = idx; break;
    case TL_EV_RELEASED_OUTSIDE_GOAL: z.rog = idx; break;
    case TL_EV_OBJ_LEFT_GOAL: z.olg = idx; break;
    case TL_EV_OPENED: z.opened = idx; break;
    case TL_EV_SLIGHTLY_OPENED: z.so = idx; break;
    case TL_EV_CLOSED: z.closed = idx; break;
    case TL_EV_SLIGHTLY_CLOSED: z.sc = idx; break;
    case TL_EV_OPEN: z.open = idx; break;
    case TL_EV_SUCCESS: z.s = idx; break;
    case TL_EV_EXCESSIVE_COLLISIONS: z.x = idx; break;
  }
}

// local kind k of the subtask's alphabet (kAlpha order) -> signature field
__device__ __forceinline__ void sig_from_state(Sig& z, int subtask, const LState& S) {
  sig_clear(z);
  z.size = S.size;
  const int* l = S.last;
  switch (subtask) {
    case TL_PICK:  // Contact, Grasped, Dropped, Success, ExcessiveCollisions
      z.c = l[0]; z.g = l[1]; z.d = l[2]; z.s = l[3]; z.x = l[4];
      break;
    case TL_PLACE:  // Grasped, ObjAtGoal, RAG, ROG, ObjLeftGoal, Success, X
      z.g = l[0]; z.oag = l[1]; z.rag = l[2]; z.rog = l[3]; z.olg = l[4]; z.s = l[5]; z.x = l[6];
      break;
    case TL_OPEN:  // Contact, Opened, SlightlyOpened, Closed, Success, X
      z.c = l[0]; z.opened = l[1]; z.so = l[2]; z.closed = l[3]; z.s = l[4]; z.x = l[5];
      break;
    default:  // Close: Contact, Closed, SlightlyClosed, Open, Success, X
      z.c = l[0]; z.closed = l[1]; z.sc = l[2]; z.open = l[3]; z.s = l[4]; z.x = l[5];
      break;
  }
  z.s1 = z.size == 3 && z.c == 0 && z.g == 1 && z.s == 2;
}

#define TL_GOAL_RADIUS 0.15 /* modes.py:65 literal, independent of thresholds */

// one builtin rule predicate (modes.py:68-205); 1/0 or -status
__device__ int rule_pred(int m, const Sig& z) {
  const bool exc = z.x >= 0;
#define D0_LE(out)                                   \
  do {                                               \
    if (z.d0_none) return -TL_ERR_D0_NONE_LE;        \
    out = z.d0 <= TL_GOAL_RADIUS;                    \
  } while (0)
#define D0_GT(out)                                   \
  do {                                               \
    if (z.d0_none) return -TL_ERR_D0_NONE_GT;        \
    out = z.d0 > TL_GOAL_RADIUS;                     \
  } while (0)
  bool t;
  switch (m) {
    case 0: return z.s1;
    case 1: return !exc && z.d <= z.g;
    case 2: return !exc && z.d > z.g;
    case 3: case 4: return exc;
    case 5: return z.size == 0;
    case 6: return z.c >= 0 && z.g < 0 && z.d < 0;
    case 7: return z.d >= 0 && z.d > z.g;
    case 8: return 1;
    case 9:
      if (!(z.size <= 4)) return 0;
      if (!(z.rag >= 0)) { D0_LE(t); if (!t) return 0; }
      return z.olg <= z.oag && !exc;
    case 10:
      if (!(z.size <= 4)) return 0;
      if (!(z.rog >= 0)) { D0_GT(t); if (!t) return 0; }
      return z.olg <= z.oag && !exc;
    case 11: return z.oag < z.olg && !exc;
    case 12: return z.size > 4 && z.oag >= z.olg && !exc;
    case 13: case 14: return exc;
    case 15: return z.size == 0;
    case 16: return z.size > 0 && z.oag < 0;
    case 17: {
      if (z.oag < 0) return 0;
      bool lat = false;
      if (z.size <= 2) D0_LE(lat);
      if (!lat) lat = z.rag > z.rog && z.rag > z.g;
      return lat && z.olg > z.oag;
    }
    case 18: {
      if (z.oag < 0) return 0;
      bool lat = false;
      if (z.size <= 2) D0_GT(lat);
      if (!lat) lat = z.rog > z.rag && z.rog > z.g;
      return lat && z.olg > z.oag;
    }
    case 19: return z.oag >= 0 && z.g > z.rag && z.g > z.rog;
    case 20: return 1;
    case 21: return !exc && z.opened >= z.closed;
    case 22: return !exc && z.opened < z.closed;
    case 23: case 24: return exc;
    case 25: return z.c < 0;
    case 26: return z.closed >= 0 && z.closed > z.opened && z.closed > z.so;
    case 27: return z.so > z.opened && z.so > z.closed;
    case 28: return z.opened >= 0;
    case 29: return 1;
    case 30: return !exc && z.closed >= z.open;
    case 31: return !exc && z.closed < z.open;
    case 32: case 33: return exc;
    case 34: return z.c < 0;
    case 35: return z.closed >= 0 && z.open > z.closed && z.open > z.sc;
    case 36: return z.sc > z.closed && z.sc > z.open;
    case 37: return z.closed >= 0;
    case 38: return 1;
  }
#undef D0_LE
#undef D0_GT
  return 0;
}

__device__ __forceinline__ bool success_at_end_mode(int m) {  // modes.py:226-232
  return m == 0 || m == 1 || m == 9 || m == 10 || m == 12 || m == 21 || m == 30;
}

// classify (modes.py:235-253): mode id (>=0) or -status; flags out
__device__ int classify_sig(int subtask, const Sig& z, const tl_rules& rules,
                            uint8_t& flags) {
  const bool so = z.s >= 0;
  const int b = so ? 0 : 1;
  const int cnt = rules.count[subtask][b];
  flags = so ? 1u : 0u;
  for (int i = 0; i < cnt; i++) {
    const int m = rules.ids[subtask][b][i];
    const int r = rule_pred(m, z);
    if (r < 0) return r;
    if (r) {
      if (success_at_end_mode(m)) flags |= 2u;
      return m;
    }
  }
  return -TL_ERR_MODE_COVERAGE;
}

// final per-episode status precedence = evaluation order of extract_events
// (events.py:105 success loop, then :112/:127/:153/:172 per-subtask lists)
__device__ __forceinline__ int label_status(const tl_cset& c, uint32_t err_any) {
  const bool art_sub = c.subtask == TL_OPEN || c.subtask == TL_CLOSE;
  const bool has_art = c.art_kind != TL_ART_NONE;
  if (err_any & ERR_SUCC) {
    if (c.subtask == TL_PLACE) return TL_ERR_NAN_SUCCESS_DIST;
    return has_art ? TL_ERR_NAN_ART : TL_ERR_MISSING_ART;
  }
  if (c.subtask != TL_PLACE && (err_any & ERR_FORCE)) return TL_ERR_NAN_FORCE;
  if (c.subtask == TL_PLACE && (err_any & ERR_DIST)) return TL_ERR_NAN_PLACE_DIST;
  if (art_sub && !has_art) return TL_ERR_MISSING_ART;
  if (art_sub && (err_any & ERR_ART)) return TL_ERR_NAN_ART;
  return TL_OK;
}

// Finalise an episode: status + classify.
__device__ __forceinline__ tl_label make_label(const tl_cset& c, const LState& S, double d0,
                                               const tl_rules& rules) {
  tl_label L;
  L.status = label_status(c, S.err_any);
  L.n_events = 0;
  L.err_index = -1;
  L.subtask = (uint8_t)c.subtask;
  L.mode = 255;
  L.flags = 0;
  L.pad = 0;
  L.d0 = c.subtask == TL_PLACE ? d0 : __longlong_as_double(0x7ff8000000000000ll);
  if (L.status == TL_OK) {
    Sig z;
    sig_from_state(z, c.subtask, S);
    z.d0 = d0;
    uint8_t fl = 0;
    const int m = classify_sig(c.subtask, z, rules, fl);
    L.n_events = S.size;  // events exist even when no mode rule matches
    if (m < 0) {
      L.status = -m;
      L.flags = z.s >= 0 ? 1 : 0;
    } else {
      L.mode = (uint8_t)m;
      L.flags = fl;
    }
  }
  return L;
}

// warp-uniform state: lane 0 writes the label
__device__ __forceinline__ void finish_label(const tl_cset& c, const LState& S,
                                             double d0, const tl_rules& rules,
                                             tl_label* out) {
  const tl_label L = make_label(c, S, d0, rules);
  if (lane_id() == 0) *out = L;
}

// stage one cset into a per-warp shared slot
__device__ __forceinline__ void stage_cset(tl_cset* dst, const tl_cset* src) {
  static_assert(sizeof(tl_cset) % 4 == 0, "cset size");
  const uint32_t* s = reinterpret_cast<const uint32_t*>(src);
  uint32_t* d = reinterpret_cast<uint32_t*>(dst);
  __syncwarp();  // every lane is done reading the slot's previous cset
  for (int i = lane_id(); i < (int)(sizeof(tl_cset) / 4); i += 32) d[i] = __ldg(s + i);
  __syncwarp();
}

// Close: slightly-closed cut from records[0].art_q (events.py:174-176)
__device__ __forceinline__ void close_cut(const tl_cset& c, double a0, float& ru, double& d) {
  d = __dsub_rn(a0, c.scf_span);
  ru = __double2float_ru(d);
}

// planes the subtask's predicates read, in buffer order:
// q[dof], qd[dof], v_x, v_y, omega, dist_ee_rest, cum, then
// Pick: force | Place: q_tor, dist_obj_goal | Open/Close: q_tor, force, art
__device__ __forceinline__ int tma_nplanes(int sub, int dof) {
  return 2 * dof + (sub == TL_PICK ? 6 : sub == TL_PLACE ? 7 : 8);
}
__device__ __forceinline__ int tma_plane(int sub, int dof, int p) {
  const int f0 = 2 * dof;
  if (p < f0) return p;
  switch (p - f0) {
    case 0: return f0 + 1;  // v_base_x
    case 1: return f0 + 2;  // v_base_y
    case 2: return f0 + 3;  // omega_base
    case 3: return f0 + 4;  // dist_ee_rest
    case 4: return f0 + 7;  // cum_robot_force
    case 5: return sub == TL_PICK ? f0 + 6 : f0;  // force | q_tor
    case 6: return sub == TL_PLACE ? f0 + 5 : f0 + 6;  // dist_obj_goal | force
    default: return f0 + 8;  // art_q
  }
}

// ---- K1 vector path: 4 consecutive records per lane ----------------------------
__device__ __forceinline__ float4 ldf4(const float* p) {
  return __ldcs(reinterpret_cast<const float4*>(p));  // streamed once: evict-first
}
__device__ __forceinline__ float f4get(const float4& v, int j) {
  return j == 0 ? v.x : j == 1 ? v.y : j == 2 ? v.z : v.w;
}

__device__ __noinline__ void label_vec4(const tl_records& R, const tl_cset& c, int64_t rs, int n,
                                        float sc_ru, double sc_d, LState& S,
                                        uint8_t* step_mask, uint8_t* step_success) {
  const int lane = lane_id();
  const float* __restrict__ P = reinterpret_cast<const float*>(R.planes);
  const int64_t stride = R.plane_stride;
  const int dof = R.dof, f0 = 2 * dof;
  const int sub = c.subtask;
  for (int t0 = 0; t0 < n; t0 += 128) {
    const int tb = t0 + 4 * lane;          // first record of this lane
    const bool any = tb < n;
    const int64_t r = rs + tb;
    float4 der, cum, vx, vy, om, tor, dist, force, art, mq, mqd;
    uint32_t g4 = 0;
    if (any) {
      der = ldf4(P + (f0 + 4) * stride + r);
      cum = ldf4(P + (f0 + 7) * stride + r);
      vx = ldf4(P + (f0 + 1) * stride + r);
      vy = ldf4(P + (f0 + 2) * stride + r);
      om = ldf4(P + (f0 + 3) * stride + r);
      if (sub == TL_PICK) {
        force = ldf4(P + (f0 + 6) * stride + r);
        g4 = __ldcs(reinterpret_cast<const unsigned int*>(R.grasped + r));
      } else if (sub == TL_PLACE) {
        tor = ldf4(P + f0 * stride + r);
        dist = ldf4(P + (f0 + 5) * stride + r);
        g4 = __ldcs(reinterpret_cast<const unsigned int*>(R.grasped + r));
      } else {
        tor = ldf4(P + f0 * stride + r);
        force = ldf4(P + (f0 + 6) * stride + r);
        art = ldf4(P + (f0 + 8) * stride + r);
      }
      // Python max() of |q_i| and |qd_i| per record (predicates.py:20, :24)
      for (int i = 0; i < dof; i++) {
        const float4 q = ldf4(P + i * stride + r);
        const float4 qd = ldf4(P + (dof + i) * stride + r);
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
    uint32_t ind[4], err[4], m[4];
#pragma unroll
    for (int j = 0; j < 4; j++) {
      // branch-free: every lane evaluates its 4 slots, invalid ones are masked
      const bool valid = tb + j < n;
      {
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
          v.force = f4get(force, j);
          v.g = (g4 >> (8 * j)) & 0xffu;
        } else if (sub == TL_PLACE) {
          v.tor = f4get(tor, j);
          v.dist = f4get(dist, j);
          v.g = (g4 >> (8 * j)) & 0xffu;
        } else {
          v.tor = f4get(tor, j);
          v.force = f4get(force, j);
          v.art = f4get(art, j);
        }
        record_bits(c, v, sc_ru, sc_d, ind[j], err[j]);
        ind[j] = valid ? ind[j] : 0u;
        err[j] = valid ? err[j] : 0u;
        if (step_success && valid)
          step_success[r + j] = (err[j] & ERR_SUCC) ? 2 : ((ind[j] & IND_SUCCESS) ? 1 : 0);
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
      eor |= err[j];
    }
    if (step_mask && any) {
      if (tb + 3 < n) {  // one 4-byte store for the lane's 4 masks
        *reinterpret_cast<unsigned int*>(step_mask + r) = m[0] | (m[1] << 8) | (m[2] << 16) | (m[3] << 24);
      } else {
        for (int j = 0; j < 4 && tb + j < n; j++) step_mask[r + j] = (uint8_t)m[j];
      }
    }
    const int incl = warp_incl_scan((int)cnt);
    const int excl = incl - (int)cnt;
#pragma unroll
    for (int k = 0; k < 7; k++) {
      // position (within the lane's events) of the lane's last event of kind k
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
    S.prev_ind = __shfl_sync(kFull, ind[3], 31);
  }
}

// ---- K1 vector path, compile-time arm_dof ---------------------------------------
// Same contract as label_vec4 for aligned f32 episodes with a zero rest
// posture; the arm_dof loop is unrolled so every 128-bit load of a chunk is
// issued before the first use (one HBM latency per chunk instead of one per
// loop trip), the episode's cuts live in registers (no generic reloads after
// the step-mask stores), the predicates are evaluated without short-circuit
// branches (they are pure compares: same values), and the per-kind fold runs
// only over the kinds that occur in the chunk (events are sparse).
struct VCuts {
  float rest_, jarm_, jtor_, sqd_, sv_, som_, lim_, contact_, goal_, a_cut_, b_cut_;
  int sub;
  bool has_art_;
  __device__ float rest() const { return rest_; }
  __device__ float jarm() const { return jarm_; }
  __device__ float jtor() const { return jtor_; }
  __device__ float sqd() const { return sqd_; }
  __device__ float sv() const { return sv_; }
  __device__ float som() const { return som_; }
  __device__ float lim() const { return lim_; }
  __device__ float contact() const { return contact_; }
  __device__ float goal() const { return goal_; }
  __device__ float a_cut() const { return a_cut_; }
  __device__ float b_cut() const { return b_cut_; }
  __device__ bool has_art() const { return has_art_; }
};

__device__ __forceinline__ VCuts vcuts(const tl_cset& c, float sc_ru) {
  VCuts k;
  k.rest_ = c.rd_rest_radius; k.jarm_ = c.rd_j_arm; k.jtor_ = c.rd_j_tor;
  k.sqd_ = c.rd_static_qd; k.sv_ = c.rd_static_v; k.som_ = c.rd_static_om;
  k.lim_ = c.rd_limit; k.contact_ = c.rd_contact; k.goal_ = c.rd_goal;
  k.sub = c.subtask;
  k.has_art_ = c.art_kind != TL_ART_NONE;
  // Open: is_open (>= ru) / slightly_opened (>= ru); Close: is_closed (<= rd) / a_q < ru(a_q0 - 0.05 range)
  k.a_cut_ = k.sub == TL_OPEN ? c.ru_open : c.rd_closed;
  k.b_cut_ = k.sub == TL_OPEN ? c.ru_slight_open : sc_ru;
  return k;
}

__device__ __forceinline__ float4 f4abs(float4 v) {
  return make_float4(fabsf(v.x), fabsf(v.y), fabsf(v.z), fabsf(v.w));
}
__device__ __forceinline__ float4 f4pymax(float4 m, float4 v) {
  return make_float4(pymax_step(m.x, fabsf(v.x)), pymax_step(m.y, fabsf(v.y)),
                     pymax_step(m.z, fabsf(v.z)), pymax_step(m.w, fabsf(v.w)));
}

template <int DOF>
__device__ __forceinline__ void pymax4(const float4 (&v)[DOF], float (&m)[4]) {
#pragma unroll
  for (int j = 0; j < 4; j++) {
    float x = fabsf(f4get(v[0], j));
#pragma unroll
    for (int i = 1; i < DOF; i++) x = fmaxf(x, fabsf(f4get(v[i], j)));
    m[j] = isnan(f4get(v[0], j)) ? f4get(v[0], j) : x;
  }
}

// record_bits (f32 path, zero rest posture), subtask fixed at compile time,
// no short-circuit branches (the predicates are pure compares: same values)
template <int SUB, class K>
__device__ __forceinline__ void record_bits_s(const K& k, float der, float cum, float vx,
                                              float vy, float om, float qdm, float jm, float xa,
                                              float xb, float xc, bool g, uint32_t& ind,
                                              uint32_t& err) {
  const bool over = cum > k.lim();
  const bool rest = !(der > k.rest()) & !(jm > k.jarm()) & (qdm <= k.sqd()) & (fabsf(vx) <= k.sv()) &
                    (fabsf(vy) <= k.sv()) & (fabsf(om) <= k.som());
  ind = ((cum <= k.lim()) ? IND_CUM_LE : 0u) | (over ? IND_CUM_GT : 0u);
  bool succ;
  if (SUB == TL_PICK) {  // xa = force
    succ = !over & g & rest;
    ind |= (xa > k.contact() ? IND_CONTACT : 0u) | (g ? IND_GRASPED : 0u);
    err = isnan(xa) ? ERR_FORCE : 0u;
  } else if (SUB == TL_PLACE) {  // xa = q_tor, xb = dist_obj_goal
    const bool trs = !(fabsf(xa) > k.jtor());
    const bool in = xb <= k.goal();
    const bool dn = isnan(xb);
    succ = !over & !g & in & rest & trs;
    ind |= (g ? IND_GRASPED : 0u) | (in ? IND_A : 0u) | (xb > k.goal() ? IND_B : 0u);
    err = (dn ? ERR_DIST : 0u) | ((!over & !g & dn) ? ERR_SUCC : 0u);
  } else {  // xa = q_tor, xb = art_q, xc = force
    const bool trs = !(fabsf(xa) > k.jtor());
    const bool an = isnan(xb);
    const bool a = SUB == TL_OPEN ? xb >= k.a_cut() : xb <= k.a_cut();
    const bool b = SUB == TL_OPEN ? xb >= k.b_cut() : xb < k.b_cut();
    succ = !over & k.has_art() & a & rest & trs;
    ind |= (xc > k.contact() ? IND_CONTACT : 0u) | (a ? IND_A : 0u) | (b ? IND_B : 0u);
    err = (isnan(xc) ? ERR_FORCE : 0u) | (an ? ERR_ART : 0u) |
          ((!over & (!k.has_art() | an)) ? ERR_SUCC : 0u);
  }
  if (succ) ind |= IND_SUCCESS;
}

constexpr int kLabelWarpsMax = 8;
#ifndef TL_LABEL_L2PF
#define TL_LABEL_L2PF 1
#endif
#ifndef TL_LABEL_QD_SMEM
#define TL_LABEL_QD_SMEM 1  // Pick / Place: qd planes staged in shared memory
#endif
// one staging buffer per block for every subtask's body: [warp][plane][lane]
__device__ __forceinline__ float4 (*qd_stage())[32] {
  __shared__ __align__(16) float4 buf[kLabelWarpsMax * 7][32];
  return buf;
}
#ifndef TL_VEC_INL
#define TL_VEC_INL __forceinline__  // inlined: the running state stays in registers
#endif
// 4 consecutive records per lane, chunks of 128 records.
template <int DOF, int SUB>
__device__ TL_VEC_INL void label_vec_d(const tl_records& R, const tl_cset& c, int64_t rs, int n,
                                         float sc_ru, LState& S, uint8_t* step_mask,
                                         uint8_t* step_success) {
  constexpr int RPL = 4, CH = 32 * RPL;  // 4 consecutive records per lane
  typedef unsigned int G;                 // the lane's 4 grasped bytes / step masks
  const int lane = lane_id();
  constexpr int f0 = 2 * DOF;
  const float* __restrict__ P = reinterpret_cast<const float*>(R.planes) + rs + RPL * lane;
  const uint8_t* __restrict__ GP = R.grasped + rs + RPL * lane;
  const int64_t stride = R.plane_stride;
  const VCuts k = vcuts(c, sc_ru);
  constexpr int XA = SUB == TL_PICK ? f0 + 6 : f0;       // force | q_tor
  constexpr int XB = SUB == TL_PLACE ? f0 + 5 : f0 + 8;  // dist_obj_goal | art_q
  constexpr int NK = SUB == TL_PICK ? 5 : SUB == TL_PLACE ? 7 : 6;  // alphabet size
  // running state in registers, written back at the end
  int size = S.size;
  uint32_t prev_ind = S.prev_ind, err_any = S.err_any;
  // last-index state in shared memory (touched only by chunks with events):
  // keeps registers for the chunk's loads
  __shared__ int s_last[kLabelWarpsMax][8];
  int* last = s_last[threadIdx.x >> 5];
#pragma unroll
  for (int kk = 0; kk < NK; kk++) last[kk] = S.last[kk];
  for (int t0 = 0; t0 < n; t0 += CH) {
    const int tb = t0 + RPL * lane;          // first record of this lane
    const float* __restrict__ p = P + t0;
    uint32_t ind[RPL], err[RPL];
#pragma unroll
    for (int j = 0; j < RPL; j++) ind[j] = err[j] = 0u;
    if (tb < n) {
      // every load of the chunk issued up front; Pick / Place stage the qd
      // planes in shared memory (cp.async: no registers held in flight),
      // which at 64 registers lets ptxas issue the rest in one batch
      constexpr bool kStageQd = TL_LABEL_QD_SMEM && (SUB == TL_PICK || SUB == TL_PLACE);
      static_assert(!kStageQd || DOF <= 7, "qd staging holds 7 planes");
      float4 q[DOF], qd[DOF];
      float4 (*sq)[32] = kStageQd ? qd_stage() + (threadIdx.x >> 5) * 7 : nullptr;
      // Open / Close (qd planes in registers): the next chunk's q / qd planes
      // are prefetched toward L2 while this one is labelled
      constexpr bool kL2Pf = TL_LABEL_L2PF && (SUB == TL_OPEN || SUB == TL_CLOSE);
      if (kL2Pf && tb + CH < n) {
#pragma unroll
        for (int i = 0; i < 2 * DOF; i++)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(p + CH + i * stride));
      }
      if (kStageQd) {
#pragma unroll
        for (int i = 0; i < DOF; i++) cp_async16(&sq[i][lane], p + (DOF + i) * stride);
        cp_async_commit();
#pragma unroll
        for (int i = 0; i < DOF; i++) q[i] = ldf4(p + i * stride);
      } else {
#pragma unroll
        for (int i = 0; i < DOF; i++) {
          q[i] = ldf4(p + i * stride);
          qd[i] = ldf4(p + (DOF + i) * stride);
        }
      }
      const float4 der4 = ldf4(p + (f0 + 4) * stride), cum4 = ldf4(p + (f0 + 7) * stride);
      const float4 vx4 = ldf4(p + (f0 + 1) * stride), vy4 = ldf4(p + (f0 + 2) * stride);
      const float4 om4 = ldf4(p + (f0 + 3) * stride), xa4 = ldf4(p + XA * stride);
      float4 xb4 = make_float4(0.f, 0.f, 0.f, 0.f), xc4 = xb4;
      uint32_t g4 = 0;
      if (SUB != TL_PICK) xb4 = ldf4(p + XB * stride);
      if (SUB == TL_OPEN || SUB == TL_CLOSE) xc4 = ldf4(p + (f0 + 6) * stride);
      if (SUB == TL_PICK || SUB == TL_PLACE) g4 = __ldcs(reinterpret_cast<const G*>(GP + t0));
      float der[RPL], cum[RPL], vx[RPL], vy[RPL], om[RPL], xa[RPL], xb[RPL], xc[RPL];
#pragma unroll
      for (int j = 0; j < RPL; j++) {
        der[j] = f4get(der4, j); cum[j] = f4get(cum4, j); vx[j] = f4get(vx4, j);
        vy[j] = f4get(vy4, j); om[j] = f4get(om4, j); xa[j] = f4get(xa4, j);
        xb[j] = f4get(xb4, j); xc[j] = f4get(xc4, j);
      }
      // Python max() of |q_i| and |qd_i| per record (predicates.py:20, :24)
      float mq[RPL], mqd[RPL];
      pymax4<DOF>(q, mq);
      if (kStageQd) {
        cp_async_wait<0>();
#pragma unroll
        for (int i = 0; i < DOF; i++) qd[i] = sq[i][lane];
      }
      pymax4<DOF>(qd, mqd);
#pragma unroll
      for (int j = 0; j < RPL; j++) {
        record_bits_s<SUB>(k, der[j], cum[j], vx[j], vy[j], om[j], mqd[j], mq[j], xa[j], xb[j],
                           xc[j], (g4 >> (8 * j)) & 0xffu, ind[j], err[j]);
        const bool valid = tb + j < n;
        ind[j] = valid ? ind[j] : 0u;
        err[j] = valid ? err[j] : 0u;
        if (step_success && valid)
          step_success[rs + tb + j] = (err[j] & ERR_SUCC) ? 2 : ((ind[j] & IND_SUCCESS) ? 1 : 0);
      }
    }
    uint32_t prev = __shfl_up_sync(kFull, ind[RPL - 1], 1);
    if (lane == 0) prev = prev_ind;
    uint32_t m[RPL], orm = 0, eor = 0, packed = 0;
#pragma unroll
    for (int j = 0; j < RPL; j++) {
      const bool ok = tb + j < n && tb + j > 0;
      m[j] = ok ? edge_mask(SUB, j == 0 ? prev : ind[j - 1], ind[j]) : 0u;
      orm |= m[j];
      eor |= err[j];
      packed |= m[j] << (8 * j);
    }
    if (step_mask && tb < n) {
      if (tb + RPL - 1 < n) {  // one store for the lane's RPL masks
        *reinterpret_cast<G*>(step_mask + rs + tb) = (G)packed;
      } else {
        for (int j = 0; j < RPL && tb + j < n; j++) step_mask[rs + tb + j] = (uint8_t)m[j];
      }
    }
    orm = __reduce_or_sync(kFull, orm);
    if (orm) {  // warp-uniform: fold only chunks with events, only the kinds present
      int cnt = 0;
#pragma unroll
      for (int j = 0; j < RPL; j++) cnt += __popc(m[j]);
      const int incl = warp_incl_scan(cnt);
      const int excl = incl - cnt;
#pragma unroll
      for (int kk = 0; kk < NK; kk++) {
        if (!((orm >> kk) & 1u)) continue;  // warp-uniform
        // position (within the lane's events) of the lane's last event of kind kk
        int pos = -1, before = 0;
#pragma unroll
        for (int j = 0; j < RPL; j++) {
          if ((m[j] >> kk) & 1u) pos = before + __popc(m[j] & ((1u << kk) - 1u));
          before += __popc(m[j]);
        }
        const unsigned bal = __ballot_sync(kFull, pos >= 0);
        const int L = 31 - __clz(bal);
        last[kk] = size + __shfl_sync(kFull, excl + pos, L);
      }
      size += __shfl_sync(kFull, incl, 31);
    }
    err_any |= __reduce_or_sync(kFull, eor);
    prev_ind = __shfl_sync(kFull, ind[RPL - 1], 31);
  }
  S.size = size;
  S.prev_ind = prev_ind;
  S.err_any = err_any;
#pragma unroll
  for (int kk = 0; kk < NK; kk++) S.last[kk] = last[kk];
}

// one record per lane (any layout, f32 or f64 records, any rest posture)
template <typename T, int DOFMAX>
__device__ __forceinline__ void label_scalar(const tl_records& R, const tl_cset& c, int64_t rs, int n,
                                             float sc_ru, double sc_d, LState& S,
                                             uint8_t* step_mask, uint8_t* step_success) {
  const int lane = lane_id();
  const T* __restrict__ P = reinterpret_cast<const T*>(R.planes);
  const int64_t stride = R.plane_stride;
  const int dof = R.dof;
  const int f0 = 2 * dof;
  for (int t0 = 0; t0 < n; t0 += 32) {
    const int t = t0 + lane;
    const bool valid = t < n;
    const int64_t r = rs + t;
    RecV<T> v;
    uint32_t ind = 0, err = 0;
    if (valid) {
      v.der = P[(f0 + 4) * stride + r];
      v.cum = P[(f0 + 7) * stride + r];
      v.vx = P[(f0 + 1) * stride + r];
      v.vy = P[(f0 + 2) * stride + r];
      v.om = P[(f0 + 3) * stride + r];
      // Python-max of |q_i - rest_i| and of |qd_i|
      T m = 0, mq = 0;
      double md = 0.0;
#pragma unroll
      for (int i = 0; i < DOFMAX; i++) {
        if (i < dof) {
          const T q = P[i * stride + r];
          const T qd = P[(dof + i) * stride + r];
          const T aq = tabs(q), aqd = tabs(qd);
          m = i == 0 ? aq : pymax_step(m, aq);
          mq = i == 0 ? aqd : pymax_step(mq, aqd);
          if (!c.rest_zero) {
            const double dv = fabs(__dsub_rn((double)q, c.rest_arm[i]));
            md = i == 0 ? dv : pymax_step(md, dv);
          }
        }
      }
      v.jm = m;
      v.qdm = mq;
      v.jm_d = md;
      v.tor = 0; v.dist = 0; v.force = 0; v.art = 0; v.g = false;
      if (c.subtask == TL_PICK) {
        v.force = P[(f0 + 6) * stride + r];
        v.g = R.grasped[r] != 0;
      } else if (c.subtask == TL_PLACE) {
        v.tor = P[f0 * stride + r];
        v.dist = P[(f0 + 5) * stride + r];
        v.g = R.grasped[r] != 0;
      } else {
        v.tor = P[f0 * stride + r];
        v.force = P[(f0 + 6) * stride + r];
        v.art = P[(f0 + 8) * stride + r];
      }
      record_bits(c, v, sc_ru, sc_d, ind, err);
      if (step_success) step_success[r] = (err & ERR_SUCC) ? 2 : ((ind & IND_SUCCESS) ? 1 : 0);
    }
    uint32_t prev = __shfl_up_sync(kFull, ind, 1);
    if (lane == 0) prev = S.prev_ind;
    const uint32_t mask = (valid && t > 0) ? edge_mask(c.subtask, prev, ind) : 0u;
    if (valid && step_mask) step_mask[r] = (uint8_t)mask;
    lstate_fold(S, mask, valid ? err : 0u);
    S.prev_ind = __shfl_sync(kFull, ind, 31);
  }
}

// ---- K1: label_records -------------------------------------------------------
constexpr int kLabelWarps = 8;
static_assert(kLabelWarps <= kLabelWarpsMax, "label_vec_d's per-warp state");
#ifndef TL_LABEL_MINB
#define TL_LABEL_MINB 4  // f32, arm_dof <= 7: 4 x 8 warps per SM at <= 64 registers
#endif

// PART 1: only the episodes the compile-time-dof vector bodies take (f32,
// arm_dof 7, zero rest posture, 4-record aligned, >= 2 records); PART 2: all
// others; PART 0: every episode.  f32 / arm_dof <= 7 batches launch PART 1
// then PART 2, so the hot vector kernel's registers are allocated without
// the generic bodies (which share nothing with it at run time).
template <typename T, int DOFMAX, int PART>
__global__ void __launch_bounds__(kLabelWarps * 32, PART == 1 ? TL_LABEL_MINB : 2)
    k_label(tl_records R, int n_env, const int32_t* __restrict__ env_cset,
            const tl_cset* __restrict__ csets, tl_rules rules,
            uint8_t* __restrict__ step_mask, uint8_t* __restrict__ step_success,
            tl_label* __restrict__ labels, int vec_generic) {
  __shared__ tl_cset s_cs[kLabelWarps];
  const int warp = threadIdx.x >> 5, lane = lane_id();
  const T* __restrict__ P = reinterpret_cast<const T*>(R.planes);
  const int64_t stride = R.plane_stride;
  const int dof = R.dof;
  const bool vec_ok = (stride & 3) == 0 && (reinterpret_cast<uintptr_t>(R.planes) & 15) == 0 &&
                      (reinterpret_cast<uintptr_t>(R.grasped) & 3) == 0 &&
                      (reinterpret_cast<uintptr_t>(step_mask) & 7) == 0;  // word mask stores
  auto fast_ok = [&](int ci, int64_t rs, int n) {
    return sizeof(T) == 4 && DOFMAX == 7 && dof == 7 && !vec_generic && n >= 2 && (rs & 3) == 0 &&
           vec_ok && rs + (((int64_t)n + 3) & ~(int64_t)3) <= stride && csets[ci].rest_zero;
  };
  auto process = [&](int e, int ci, int64_t rs, int n) {
    TL_ASSERT(rs >= 0 && n >= 0 && rs + n <= R.plane_stride && ci >= 0);
    stage_cset(&s_cs[warp], &csets[ci]);
    const tl_cset& c = s_cs[warp];
    LState S;
    lstate_init(S);
    if (PART != 1 && n < 2) {  // events.py:96-97
      if (lane == 0) {
        tl_label L;
        L.status = TL_ERR_TOO_SHORT; L.n_events = 0; L.err_index = -1;
        L.subtask = (uint8_t)c.subtask; L.mode = 255; L.flags = 0; L.pad = 0;
        L.d0 = __longlong_as_double(0x7ff8000000000000ll);
        labels[e] = L;
      }
      if (step_success) {  // predicate values are still defined per record
        // fallthrough below handles n == 1 through the generic loop
      } else {
        return;
      }
    }
    const int f0 = 2 * dof;
    double d0 = 0.0;
    float sc_ru = 0.f;
    double sc_d = 0.0;
    if (c.subtask == TL_PLACE) d0 = (double)P[(f0 + 5) * stride + rs];
    if (c.subtask == TL_CLOSE && n > 0) close_cut(c, (double)P[(f0 + 8) * stride + rs], sc_ru, sc_d);
    if (PART == 1) {  // compile-time-dof vector bodies
      switch (c.subtask) {
        case TL_PICK: label_vec_d<7, TL_PICK>(R, c, rs, n, sc_ru, S, step_mask, step_success); break;
        case TL_PLACE: label_vec_d<7, TL_PLACE>(R, c, rs, n, sc_ru, S, step_mask, step_success); break;
        case TL_OPEN: label_vec_d<7, TL_OPEN>(R, c, rs, n, sc_ru, S, step_mask, step_success); break;
        default: label_vec_d<7, TL_CLOSE>(R, c, rs, n, sc_ru, S, step_mask, step_success); break;
      }
      finish_label(c, S, d0, rules, &labels[e]);
      return;
    }
    // f32 episodes whose records are 16-byte aligned: 4 records per lane,
    // 128-bit loads (label_vec4); otherwise one record per lane below.
    if (sizeof(T) == 4 && c.rest_zero && (rs & 3) == 0 && vec_ok &&
        rs + (((int64_t)n + 3) & ~(int64_t)3) <= stride) {
      label_vec4(R, c, rs, n, sc_ru, (double)sc_d, S, step_mask, step_success);
      if (n >= 2) finish_label(c, S, d0, rules, &labels[e]);
      return;
    }
    label_scalar<T, DOFMAX>(R, c, rs, n, sc_ru, sc_d, S, step_mask, step_success);
    if (n >= 2) finish_label(c, S, d0, rules, &labels[e]);
  };
  if constexpr (PART == 2) {
    // 32 episodes per warp iteration: lane l tests episode base + l, the warp
    // then labels the ones the vector kernel left (usually none)
    for (int64_t base = ((int64_t)blockIdx.x * kLabelWarps + warp) * 32; base < n_env;
         base += (int64_t)gridDim.x * kLabelWarps * 32) {
      const int el = (int)base + lane;
      int ci = 0, n = 0;
      int64_t rs = 0;
      bool todo_l = false;
      if (el < n_env) {
        ci = env_cset[el];
        rs = R.rec_start[el];
        n = R.n_rec[el];
        todo_l = !fast_ok(ci, rs, n);
      }
      unsigned todo = __ballot_sync(kFull, todo_l);
      while (todo) {
        const int j = __ffs(todo) - 1;
        todo &= todo - 1;
        process((int)base + j, __shfl_sync(kFull, ci, j), __shfl_sync(kFull, rs, j),
                __shfl_sync(kFull, n, j));
      }
    }
  } else {
    for (int e = blockIdx.x * kLabelWarps + warp; e < n_env; e += gridDim.x * kLabelWarps) {
      const int ci = env_cset[e];
      const int64_t rs = R.rec_start[e];
      const int n = R.n_rec[e];
      if (PART == 1 && !fast_ok(ci, rs, n)) continue;
      process(e, ci, rs, n);
    }
  }
}

// ---- K2: event list emission --------------------------------------------------
constexpr int kEmitWarps = 8;

__global__ void __launch_bounds__(kEmitWarps * 32)
    k_emit(const uint8_t* __restrict__ step_mask, const int64_t* __restrict__ rec_start,
           const int32_t* __restrict__ n_rec, const tl_label* __restrict__ labels,
           const int64_t* __restrict__ ev_off, int n_env, uint8_t* __restrict__ ev_kind,
           int32_t* __restrict__ ev_t) {
  const int warp = threadIdx.x >> 5, lane = lane_id();
  for (int e = blockIdx.x * kEmitWarps + warp; e < n_env; e += gridDim.x * kEmitWarps) {
    if (labels[e].n_events == 0) continue;
    const int sub = labels[e].subtask;
    const int64_t rs = rec_start[e];
    const int n = n_rec[e];
    int64_t base = ev_off[e];
    for (int t0 = 0; t0 < n; t0 += 32) {
      const int t = t0 + lane;
      const uint32_t mask = t < n ? step_mask[rs + t] : 0u;
      const int cnt = __popc(mask);
      const int incl = warp_incl_scan(cnt);
      int64_t pos = base + incl - cnt;
      uint32_t m = mask;
      while (m) {
        const int k = __ffs(m) - 1;
        m &= m - 1;
        ev_kind[pos] = kAlpha[sub][k];
        ev_t[pos] = t;
        pos++;
      }
      base += __shfl_sync(kFull, incl, 31);
    }
  }
}

// ---- scan of event counts -------------------------------------------------------
constexpr int kScanBlock = 1024;

__device__ __forceinline__ int64_t block_excl_scan64(int64_t v, int64_t* sh, int64_t& total) {
  // sh: 32 slots
  const int lane = lane_id(), warp = threadIdx.x >> 5;
  int64_t x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    int64_t u = __shfl_up_sync(kFull, x, d);
    if (lane >= d) x += u;
  }
  if (lane == 31) sh[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int64_t w = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      int64_t u = __shfl_up_sync(kFull, w, d);
      if (lane >= d) w += u;
    }
    sh[lane] = w;
  }
  __syncthreads();
  const int64_t wbase = warp ? sh[warp - 1] : 0;
  total = sh[(blockDim.x >> 5) - 1];
  __syncthreads();
  return wbase + x - v;
}

__global__ void __launch_bounds__(kScanBlock)
    k_scan_tiles(const tl_label* __restrict__ labels, int n, int64_t* __restrict__ ev_off,
                 int64_t* __restrict__ tile_sum) {
  __shared__ int64_t sh[32];
  const int i = blockIdx.x * kScanBlock + threadIdx.x;
  int64_t v = 0;
  if (i < n) v = labels[i].n_events;  // 0 whenever extraction failed
  int64_t total;
  const int64_t ex = block_excl_scan64(v, sh, total);
  if (i < n) ev_off[i] = ex;
  if (threadIdx.x == 0) tile_sum[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kScanBlock)
    k_scan_sums(int64_t* __restrict__ tile_sum, int n_tiles, int64_t* __restrict__ ev_off, int n) {
  __shared__ int64_t sh[32];
  int64_t carry = 0;
  for (int b = 0; b < n_tiles; b += kScanBlock) {
    const int i = b + threadIdx.x;
    const int64_t v = i < n_tiles ? tile_sum[i] : 0;
    int64_t total;
    const int64_t ex = block_excl_scan64(v, sh, total);
    if (i < n_tiles) tile_sum[i] = carry + ex;
    carry += total;
  }
  if (threadIdx.x == 0) ev_off[n] = carry;
}

__global__ void k_scan_add(int64_t* __restrict__ ev_off, const int64_t* __restrict__ tile_off, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) ev_off[i] += tile_off[i / kScanBlock];
}

// ---- classify given event lists (thread per list) --------------------------------
__global__ void k_classify_events(const uint8_t* __restrict__ ev_kind,
                                  const int64_t* __restrict__ ev_off,
                                  const uint8_t* __restrict__ subtask,
                                  const double* __restrict__ d0,
                                  const uint8_t* __restrict__ d0_none, int n,
                                  tl_rules rules, tl_label* __restrict__ out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  const int sub = subtask[e];
  const int64_t a = ev_off[e], b = ev_off[e + 1];
  Sig z;
  sig_clear(z);
  z.size = (int)(b - a);
  for (int64_t i = a; i < b; i++) sig_set(z, ev_kind[i], (int)(i - a));
  z.s1 = z.size == 3 && ev_kind[a] == TL_EV_CONTACT && ev_kind[a + 1] == TL_EV_GRASPED &&
         ev_kind[a + 2] == TL_EV_SUCCESS;
  z.d0 = d0 ? d0[e] : 0.0;
  z.d0_none = d0_none ? d0_none[e] != 0 : false;
  tl_label L;
  L.err_index = -1;
  L.subtask = (uint8_t)sub;
  L.pad = 0;
  L.d0 = z.d0;
  uint8_t fl = 0;
  const int m = classify_sig(sub, z, rules, fl);
  L.status = m < 0 ? -m : TL_OK;
  L.mode = m < 0 ? 255 : (uint8_t)m;
  L.flags = m < 0 ? (z.s >= 0 ? 1 : 0) : fl;
  L.n_events = z.size;
  out[e] = L;
}

// ---- K6: mode histogram ------------------------------------------------------------
__global__ void k_mode_hist(const tl_label* __restrict__ labels, int n,
                            unsigned long long* __restrict__ hist) {
  __shared__ unsigned int h[TL_N_MODES];
  for (int i = threadIdx.x; i < TL_N_MODES; i += blockDim.x) h[i] = 0;
  __syncthreads();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const tl_label L = labels[i];
    if (L.status == TL_OK && L.mode < TL_N_MODES) atomicAdd(&h[L.mode], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < TL_N_MODES; i += blockDim.x)
    if (h[i]) atomicAdd(&hist[i], (unsigned long long)h[i]);
}

}  // namespace tl

namespace tl {

// ---- per-record predicate evaluation (predicates.py:16-99) -------------------
template <typename T, int DOFMAX>
__global__ void __launch_bounds__(kLabelWarps * 32)
    k_predicates(tl_records R, int n_env, const int32_t* __restrict__ env_cset,
                 const tl_cset* __restrict__ csets, const double* __restrict__ a0v,
                 uint8_t* __restrict__ bits, uint8_t* __restrict__ errs,
                 double* __restrict__ jmax) {
  __shared__ tl_cset s_cs[kLabelWarps];
  const int warp = threadIdx.x >> 5, lane = lane_id();
  const T* __restrict__ P = reinterpret_cast<const T*>(R.planes);
  const int64_t stride = R.plane_stride;
  const int dof = R.dof, f0 = 2 * dof;
  for (int e = blockIdx.x * kLabelWarps + warp; e < n_env; e += gridDim.x * kLabelWarps) {
    stage_cset(&s_cs[warp], &csets[env_cset[e]]);
    const tl_cset& c = s_cs[warp];
    const int64_t rs = R.rec_start[e];
    const int n = R.n_rec[e];
    TL_ASSERT(rs >= 0 && n >= 0 && rs + n <= R.plane_stride);
    float sc_ru = 0.f;
    double sc_d = 0.0;
    if (c.subtask == TL_CLOSE && n > 0)
      close_cut(c, a0v ? a0v[e] : (double)P[(f0 + 8) * stride + rs], sc_ru, sc_d);
    for (int t = lane; t < n; t += 32) {
      const int64_t r = rs + t;
      RecV<T> v;
      v.der = P[(f0 + 4) * stride + r];
      v.cum = P[(f0 + 7) * stride + r];
      v.vx = P[(f0 + 1) * stride + r];
      v.vy = P[(f0 + 2) * stride + r];
      v.om = P[(f0 + 3) * stride + r];
      v.tor = P[f0 * stride + r];
      v.dist = P[(f0 + 5) * stride + r];
      v.force = P[(f0 + 6) * stride + r];
      v.art = P[(f0 + 8) * stride + r];
      v.g = R.grasped[r] != 0;
      T m = 0, mq = 0;
      double md = 0.0;
#pragma unroll
      for (int i = 0; i < DOFMAX; i++) {
        if (i < dof) {
          const T q = P[i * stride + r];
          const T qd = P[(dof + i) * stride + r];
          m = i == 0 ? tabs(q) : pymax_step(m, tabs(q));
          mq = i == 0 ? tabs(qd) : pymax_step(mq, tabs(qd));
          const double dv = fabs(__dsub_rn((double)q, c.rest_arm[i]));
          md = i == 0 ? dv : pymax_step(md, dv);
        }
      }
      v.jm = m;
      v.qdm = mq;
      v.jm_d = md;
      uint32_t ind, err;
      record_bits(c, v, sc_ru, sc_d, ind, err);
      const bool stat = LE(v.qdm, c.rd_static_qd, c.static_qd) &&
                        LE(tabs(v.vx), c.rd_static_v, c.static_v) &&
                        LE(tabs(v.vy), c.rd_static_v, c.static_v) &&
                        LE(tabs(v.om), c.rd_static_om, c.static_om);
      // grasped bit is reported for every subtask
      ind = (ind & ~IND_GRASPED) | (v.g ? IND_GRASPED : 0u) |
            (GT(v.force, c.rd_contact, c.contact_eps) ? IND_CONTACT : 0u);
      if (bits) bits[r] = (uint8_t)(ind | (stat ? 128u : 0u));
      if (errs) errs[r] = (uint8_t)(err | (isnan(v.force) ? ERR_FORCE : 0u) |
                                    (isnan(v.dist) ? ERR_DIST : 0u) | (isnan(v.art) ? ERR_ART : 0u));
      if (jmax) jmax[r] = md;
    }
  }
}

}  // namespace tl

namespace tl {

// ---- generic int32 exclusive scan (record counts -> compact offsets) ---------
__global__ void __launch_bounds__(kScanBlock)
    k_scan_i32_tiles(const int32_t* __restrict__ in, int n, int64_t* __restrict__ out,
                     int64_t* __restrict__ tile_sum) {
  __shared__ int64_t sh[32];
  const int i = blockIdx.x * kScanBlock + threadIdx.x;
  const int64_t v = i < n ? in[i] : 0;
  int64_t total;
  const int64_t ex = block_excl_scan64(v, sh, total);
  if (i < n) out[i] = ex;
  if (threadIdx.x == 0) tile_sum[blockIdx.x] = total;
}

// ---- compaction of a padded record layout (one warp per episode) -------------
template <typename T>
__global__ void __launch_bounds__(256)
    k_compact(tl_records src, int n_env, const int64_t* __restrict__ dst_start, tl_records dst,
              int n_planes) {
  const int warp = threadIdx.x >> 5, lane = lane_id();
  const T* __restrict__ sp = reinterpret_cast<const T*>(src.planes);
  T* __restrict__ dp = reinterpret_cast<T*>(dst.planes);
  for (int e = blockIdx.x * 8 + warp; e < n_env; e += gridDim.x * 8) {
    const int64_t a = src.rec_start[e], b = dst_start[e];
    const int n = src.n_rec[e];
    TL_ASSERT(a >= 0 && n >= 0 && a + n <= src.plane_stride && b >= 0 && b + n <= dst.plane_stride);
    for (int t = lane; t < n; t += 32) {
      for (int f = 0; f < n_planes; f++) dp[f * dst.plane_stride + b + t] = sp[f * src.plane_stride + a + t];
      dst.grasped[b + t] = src.grasped[a + t];
    }
    if (lane == 0) {
      dst.rec_start[e] = b;
      dst.n_rec[e] = n;
    }
  }
}

}  // namespace tl

namespace tl {

// k_scan_emit's per-episode body: warp `warp` of the block writes episode e's
// ordered (kind, t) list at out_kind / out_t + base (global, or the tile's
// shared staging area with base relative to the tile)
__device__ __forceinline__ void emit_tile_lists(const uint8_t* __restrict__ step_mask,
                                                const int64_t* __restrict__ rec_start,
                                                const int32_t* __restrict__ n_rec,
                                                const tl_label* __restrict__ labels, int n_env,
                                                int e, int64_t base, uint8_t* out_kind,
                                                int32_t* out_t) {
  const int lane = lane_id();
  if (e >= n_env || labels[e].n_events == 0) return;
  const int sub = labels[e].subtask;
  const int64_t rs = rec_start[e];
  const int n = n_rec[e];
  TL_ASSERT(rs >= 0 && n >= 0);
  // four records per lane (one 32-bit load when the episode's masks are
  // 4-byte aligned), up to eight 128-record chunks loaded before any is
  // processed: the longest episode's chain of dependent loads sets the time
  const uint8_t* sm = step_mask + rs;
  const bool al = (reinterpret_cast<uintptr_t>(sm) & 3) == 0;
  for (int c0 = 0; c0 < n; c0 += 1024) {
    uint32_t w[8];
#pragma unroll
    for (int k = 0; k < 8; k++) {
      const int t = c0 + 128 * k + 4 * lane;
      uint32_t v = 0u;
      if (al && t + 3 < n) {
        v = *reinterpret_cast<const uint32_t*>(sm + t);
      } else {
#pragma unroll
        for (int b = 0; b < 4; b++)
          if (t + b < n) v |= (uint32_t)sm[t + b] << (8 * b);
      }
      w[k] = v;
    }
#pragma unroll
    for (int k = 0; k < 8; k++) {
      if (c0 + 128 * k >= n) break;  // warp-uniform
      const int t4 = c0 + 128 * k + 4 * lane;
      const uint32_t v = w[k];
      const int cnt = __popc(v);
      const int incl = warp_incl_scan(cnt);
      int64_t pos = base + incl - cnt;
#pragma unroll
      for (int b = 0; b < 4; b++) {
        uint32_t m = (v >> (8 * b)) & 0xffu;
        while (m) {
          const int q = __ffs(m) - 1;
          m &= m - 1;
          out_kind[pos] = kAlpha[sub][q];
          out_t[pos] = t4 + b;
          pos++;
        }
      }
      base += __shfl_sync(kFull, incl, 31);
    }
  }
}

// ---- K2 fused: event-offset scan (decoupled look-back) + event emission -------
// One block = 32 warps = a tile of 32 episodes.  Warp 0 scans the tile's
// n_events, publishes the tile aggregate and walks back over predecessor
// tiles (tiles are taken in launch order through a ticket counter, so a
// predecessor is always resident or finished); then warp w emits episode w
// of the tile.  Replaces scan (3 launches) + emit (1 launch) by one.
// A tile's events are one contiguous range of the output: when they fit the
// shared staging area the warps write them there and the block stores the
// range with contiguous, fully used lines (the event lists may live in pinned
// host memory, where scattered 1- and 4-byte stores each cost a PCIe write).
constexpr uint64_t kTileAgg = 1ull << 62, kTilePrefix = 2ull << 62;
constexpr uint64_t kTileValMask = (1ull << 62) - 1;
constexpr int kEvStage = 4096;  // events staged per tile (20 KB)

__global__ void __launch_bounds__(1024)
    k_scan_emit(const uint8_t* __restrict__ step_mask, const int64_t* __restrict__ rec_start,
                const int32_t* __restrict__ n_rec, const tl_label* __restrict__ labels, int n_env,
                int64_t* __restrict__ ev_off, uint8_t* __restrict__ ev_kind,
                int32_t* __restrict__ ev_t, unsigned long long* tile_state) {
  __shared__ int s_tile;
  __shared__ int64_t s_off[32];
  __shared__ int64_t s_tot;
  __shared__ __align__(16) int32_t s_t[kEvStage + 4];
  __shared__ __align__(16) uint8_t s_k[kEvStage + 4];
  TL_BLOCK_SPAN(1);
  const int warp = threadIdx.x >> 5, lane = lane_id();
  const int n_tiles = (n_env + 31) / 32;
  if (threadIdx.x == 0)
    s_tile = (int)atomicAdd(reinterpret_cast<unsigned long long*>(tile_state + n_tiles), 1ull);
  __syncthreads();
  const int tile = s_tile;
  if (warp == 0) {
    const int e = tile * 32 + lane;
    const int64_t cnt = e < n_env ? labels[e].n_events : 0;
    int64_t incl = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int64_t u = __shfl_up_sync(kFull, incl, d);
      if (lane >= d) incl += u;
    }
    const int64_t total = __shfl_sync(kFull, incl, 31);
    int64_t prefix = 0;
    if (tile == 0) {
      if (lane == 0) atomicExch(tile_state, kTilePrefix | (unsigned long long)total);
    } else {
      if (lane == 0) atomicExch(tile_state + tile, kTileAgg | (unsigned long long)total);
      // warp-wide decoupled look-back: 32 predecessor tiles per probe, summed
      // up to the nearest one that already holds its inclusive prefix
      volatile unsigned long long* st = tile_state;
      for (int j = tile - 1; j >= 0;) {
        const int idx = j - lane;
        const unsigned long long v = idx >= 0 ? st[idx] : kTilePrefix;
        const unsigned long long flag = v & ~kTileValMask;
        const unsigned pm = __ballot_sync(kFull, flag == kTilePrefix);
        const unsigned zm = __ballot_sync(kFull, flag == 0);
        const int lim = pm ? __ffs(pm) - 1 : 31;  // lanes 0..lim are needed
        const unsigned need = lim == 31 ? kFull : ((2u << lim) - 1u);
        if (zm & need) continue;                  // a predecessor not published yet
        int64_t c = lane <= lim ? (int64_t)(v & kTileValMask) : 0;
#pragma unroll
        for (int d = 16; d >= 1; d >>= 1) c += __shfl_xor_sync(kFull, c, d);
        prefix += c;
        if (pm) break;
        j -= 32;
      }
      if (lane == 0) atomicExch(tile_state + tile, kTilePrefix | (unsigned long long)(prefix + total));
    }
    prefix = __shfl_sync(kFull, prefix, 0);
    const int64_t off = prefix + incl - cnt;
    s_off[lane] = off;
    if (lane == 0) s_tot = total;
    if (e < n_env) ev_off[e] = off;
    if (e == n_env - 1) ev_off[n_env] = off + cnt;
  }
  __syncthreads();
  const int64_t tile_base = s_off[0];
  const int64_t tile_tot = s_tot;
  const bool staged = tile_tot <= kEvStage && (reinterpret_cast<uintptr_t>(ev_t) & 3u) == 0;
  // staged at the output's phase within a 16-byte (times) / 4-byte (kinds)
  // word, so the copy-out stores whole aligned words from aligned words
  int32_t* gt = ev_t + tile_base;
  uint8_t* gk = ev_kind + tile_base;
  const int sh_t = (int)((reinterpret_cast<uintptr_t>(gt) >> 2) & 3u);
  const int sh_k = (int)(reinterpret_cast<uintptr_t>(gk) & 3u);
  emit_tile_lists(step_mask, rec_start, n_rec, labels, n_env, tile * 32 + warp,
                  staged ? s_off[warp] - tile_base : s_off[warp],
                  staged ? s_k + sh_k : ev_kind, staged ? s_t + sh_t : ev_t);
  if (!staged) return;
  __syncthreads();
  const int n = (int)tile_tot;
  {
    int4* gw = reinterpret_cast<int4*>(gt - sh_t);
    const int4* sw = reinterpret_cast<const int4*>(s_t);
    const int end = sh_t + n;
    for (int v = threadIdx.x; 4 * v < end; v += blockDim.x) {
      if (4 * v >= sh_t && 4 * v + 4 <= end) {
        gw[v] = sw[v];
      } else {
        for (int j = max(4 * v, sh_t); j < min(4 * v + 4, end); j++) (gt - sh_t)[j] = s_t[j];
      }
    }
  }
  {
    uint32_t* gw = reinterpret_cast<uint32_t*>(gk - sh_k);
    const uint32_t* sw = reinterpret_cast<const uint32_t*>(s_k);
    const int end = sh_k + n;
    for (int v = threadIdx.x; 4 * v < end; v += blockDim.x) {
      if (4 * v >= sh_k && 4 * v + 4 <= end) {
        gw[v] = sw[v];
      } else {
        for (int j = max(4 * v, sh_k); j < min(4 * v + 4, end); j++) (gk - sh_k)[j] = s_k[j];
      }
    }
  }
}

}  // namespace tl
