/*
 * trajlab_b200.h -- C ABI of the B200-native trajlab hot path
 * (libtrajlab_b200.so, built from paper_2412_13211_b200/csrc for sm_100a).
 *
 * Plain C: no C++ or torch types cross this boundary.  Every array argument
 * is a DEVICE pointer owned by the caller unless marked (host).  Calls are
 * stream-ordered on the caller's cudaStream_t (passed as void*), return an
 * int status (TL_OK or TL_E_*), and never synchronise the stream.
 * Per-episode failures are NOT call failures: they land in tl_label.status
 * with codes that mirror the reference exception raise sites 1:1.
 *
 * Reference interfaces each entry point replaces (paths relative to
 * /root/reference/pkg/src/trajlab/):
 *   tl_label_records   extract_events (events.py:94-193) + classify
 *                      (modes.py:235-253) + success_step (predicates.py:75-94),
 *                      i.e. label_trajectory (pipeline.py:75-94) for N episodes
 *   tl_emit_events     EventList materialisation (events.py:109-191) /
 *                      LabelRecord.events (pipeline.py:88)
 *   tl_classify_events classify(EventList, rules) (modes.py:235-253)
 *   tl_fuzz            fuzz(seed, kind, config, th) (synth.py:510-515) =
 *                      random_script (synth.py:363-507) + realize
 *                      (synth.py:345-348), fused with labelling
 *   tl_realize         realize(script, seed, th) (synth.py:345-348), fused
 *                      with labelling
 *   tl_filter_select   filter_labels selection (pipeline.py:276-338)
 *   tl_mode_histogram  mode counting of label_batch/mode_table
 *                      (pipeline.py:148-150, analytics.py:140-158)
 *   tl_validate_records validate / check_valid per-record invariants
 *                      (model.py:232-288)
 */
#ifndef TRAJLAB_B200_H
#define TRAJLAB_B200_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TL_ABI_VERSION 1
#define TL_MAX_DOF 16
#define TL_N_MODES 39
#define TL_N_EVENT_KINDS 14

/* ---- enums (model.py:20-43, events.py:20-34 enum order) ---------------- */
enum { TL_PICK = 0, TL_PLACE = 1, TL_OPEN = 2, TL_CLOSE = 3 };
enum { TL_ART_NONE = 0, TL_ART_FRIDGE = 1, TL_ART_DRAWER = 2 };
enum {
  TL_EV_CONTACT = 0, TL_EV_GRASPED, TL_EV_DROPPED, TL_EV_OBJ_AT_GOAL,
  TL_EV_RELEASED_AT_GOAL, TL_EV_RELEASED_OUTSIDE_GOAL, TL_EV_OBJ_LEFT_GOAL,
  TL_EV_OPENED, TL_EV_SLIGHTLY_OPENED, TL_EV_CLOSED, TL_EV_SLIGHTLY_CLOSED,
  TL_EV_OPEN, TL_EV_SUCCESS, TL_EV_EXCESSIVE_COLLISIONS
};
/* EventScript.initial_art_level strings (synth.py:71) */
/* batched env actions (tl_env_step): 0..13 = EventKind applied at this
 * step, or one of these */
enum { TL_ACT_HOLD = 255,     /* no event: _advance_cum + _emit (synth.py:198-201) */
       TL_ACT_IDLE = 254,     /* env does not advance: no record, mask 0 */
       TL_ACT_BAD_GAP = 253   /* raise InfeasibleScript "event gap must be >= 1" */
};
enum { TL_LVL_LOW = 0, TL_LVL_SLIGHT = 1, TL_LVL_OPEN = 2, TL_LVL_HIGH = 3,
       TL_LVL_CLOSED = 4 };

/* ---- status codes --------------------------------------------------------
 * Per-episode (tl_label.status); each names the reference raise site.      */
enum {
  TL_OK = 0,
  TL_ERR_TOO_SHORT = 1,            /* TooShort          events.py:97      */
  TL_ERR_NAN_SUCCESS_DIST = 2,     /* RequiredFieldNaN  predicates.py:86  */
  TL_ERR_NAN_ART = 3,              /* RequiredFieldNaN  predicates.py:46  */
  TL_ERR_NAN_FORCE = 4,            /* RequiredFieldNaN  events.py:87      */
  TL_ERR_NAN_PLACE_DIST = 5,       /* RequiredFieldNaN  events.py:130     */
  TL_ERR_MISSING_ART = 6,          /* MissingArticulation predicates.py:38 */
  TL_ERR_MODE_COVERAGE = 7,        /* ModeCoverageError modes.py:251      */
  TL_ERR_D0_NONE_LE = 8,           /* TypeError None<=float modes.py:100  */
  TL_ERR_D0_NONE_GT = 9,           /* TypeError None>float  modes.py:105  */
  /* InfeasibleScript raise sites (synth.py) */
  TL_INF_PICK_GRASPED_NO_CONTACT = 20, /* :155 */
  TL_INF_NOT_IN_ALPHABET = 21,     /* :209/:296 */
  TL_INF_LIMIT_EXCEEDED = 22,      /* :212 */
  TL_INF_SUCCESS_UNREACHABLE = 23, /* :224 */
  TL_INF_CONTACT_UNDEFINED = 24,   /* :231 */
  TL_INF_CONTACT_AGAIN = 25,       /* :233 */
  TL_INF_GRASPED_AGAIN = 26,       /* :237 */
  TL_INF_PICK_GRASP_NO_FORCE = 27, /* :239 */
  TL_INF_DROPPED_NOT_GRASPED = 28, /* :243 */
  TL_INF_AT_GOAL_ALREADY = 29,     /* :248 */
  TL_INF_LEFT_NOT_AT_GOAL = 30,    /* :252 */
  TL_INF_RAG = 31,                 /* :256 */
  TL_INF_ROG = 32,                 /* :260 */
  TL_INF_SLIGHTLY_OPENED = 33,     /* :264 */
  TL_INF_OPENED = 34,              /* :269 */
  TL_INF_CLOSED_OPEN = 35,         /* :274 */
  TL_INF_SC_LEVEL = 36,            /* :279 */
  TL_INF_SC_BAND = 37,             /* :281 */
  TL_INF_CLOSED_CLOSE = 38,        /* :287 */
  TL_INF_OPEN_CLOSE = 39,          /* :292 */
  TL_INF_GAP = 40,                 /* :302 */
  TL_INF_INIT_LEVEL = 41,          /* :123/:139 */
  TL_ERR_SCRIPT_CAPACITY = 50,     /* script longer than the fuzz capacity */
  /* call-level errors (return values) */
  TL_E_INVALID = 100,
  TL_E_CUDA = 101,
  TL_E_CAPACITY = 102
};

/* ---- Thresholds (thresholds.py:15-31, field order preserved) ------------ */
typedef struct tl_thresholds {
  double rest_radius, goal_radius, j_arm_pick, j_arm_other, j_tor_max,
      static_qd_arm, static_v_base, static_omega, coll_pick, coll_place,
      coll_artic, open_frac_fridge, open_frac_drawer, close_frac,
      slightly_open_frac, slightly_close_frac, contact_eps;
} tl_thresholds;

/* ---- per-episode constant set -------------------------------------------
 * TrajectoryHeader (model.py:51-92) + resolved Thresholds, pre-digested by
 * tl_cset_build into the comparison cuts the predicates use.  Episodes share
 * csets by index (env_cset[e]); the label kernel stages them in shared
 * memory.  Layout is an implementation detail: build with tl_cset_build.   */
typedef struct tl_cset {
  int32_t subtask, art_kind, dof, rest_zero;
  /* f32 cuts: for an f32 value x and f64 threshold T,
   *   x <= T  <=>  x <= rd(T)      x > T  <=>  x > rd(T)
   *   x >= T  <=>  x >= ru(T)      x < T  <=>  x < ru(T)               */
  float rd_rest_radius, rd_goal, rd_static_qd, rd_static_v, rd_static_om,
      rd_limit, rd_contact, ru_open, rd_closed, ru_slight_open, rd_j_arm,
      rd_j_tor;
  /* f64 thresholds (exact path for f64 records / nonzero rest posture) */
  double rest_radius, goal_radius, static_qd, static_v, static_om, limit,
      contact_eps, open_cut, closed_cut, slight_open_cut, j_arm, j_tor,
      rest_tor, scf_span, pad0;
  double rest_arm[TL_MAX_DOF];
} tl_cset;

/* host-only: header fields + resolved thresholds -> cset */
int tl_cset_build(int32_t subtask, int32_t art_kind, double art_qmin,
                  double art_qmax, int32_t arm_dof, const double* rest_arm,
                  double rest_tor, const tl_thresholds* th, tl_cset* out);

/* ---- record batch (structure of arrays, episode-major) ------------------
 * Field planes in TRJL record order (io_binary.py:5-7):
 *   plane f < dof        q_arm[f]
 *   dof <= f < 2dof      qd_arm[f-dof]
 *   2dof + 0..8          q_tor, v_base_x, v_base_y, omega_base, dist_ee_rest,
 *                        dist_obj_goal, force_ee_target, cum_robot_force, art_q
 * Plane f of record r is planes[f*plane_stride + r]; grasped[r] is 0/1.
 * Episode e owns records [rec_start[e], rec_start[e] + n_rec[e]).           */
typedef struct tl_records {
  void* planes;            /* float (dtype 0) or double (dtype 1) */
  uint8_t* grasped;
  int64_t* rec_start;
  int32_t* n_rec;
  int64_t plane_stride;
  int32_t dtype;           /* 0 = f32 (binary32 contract), 1 = f64 */
  int32_t dof;
} tl_records;

/* ---- per-episode label output ------------------------------------------- */
typedef struct tl_label {
  int32_t status;          /* TL_OK or a per-episode code */
  int32_t n_events;
  int32_t err_index;       /* failing script step (realize) or -1 */
  uint8_t subtask;
  uint8_t mode;            /* global mode id 0..38 (MODE_IDS order) */
  uint8_t flags;           /* bit0 success_once, bit1 success_at_end */
  uint8_t pad;
  double d0;               /* initial_dist_obj_goal (Place) else NaN */
} tl_label;

/* classify rule tables (modes.py:68-205).  For subtask s and branch b
 * (0 success, 1 failure): count[s][b] rules, ids[s][b][i] = global mode id
 * of the builtin predicate to evaluate, first match wins.  NULL = MODE_RULES. */
typedef struct tl_rules {
  int8_t count[4][2];
  int8_t ids[4][2][16];
} tl_rules;

/* FuzzConfig (synth.py:354-360) */
typedef struct tl_fuzz_cfg {
  int32_t max_events, max_gap, max_tail, pad;
  double edge_density, success_prob;
} tl_fuzz_cfg;

/* EventScript (synth.py:63-74), one per episode; steps live in the shared
 * step_kind/step_gap arrays at [step_off, step_off + n_steps). */
typedef struct tl_script {
  int64_t step_off;
  int64_t seed;            /* realize RNG seed */
  int32_t n_steps, tail;
  int32_t subtask, art_kind;
  int32_t initial_level, initial_grasped;
  int32_t initial_contact, arm_dof;
  double initial_dist_obj_goal;
} tl_script;

/* ---- entry points --------------------------------------------------------*/
int tl_abi_version(void);
const char* tl_status_name(int code);
int tl_device_sm_count(void);

/* K1: per-step predicates + edge events + mode, one label per episode.
 * step_mask (optional, per record): bit i = i-th kind of the subtask's
 * EVENT_ORDER alphabet fired at that record.  step_success (optional, per
 * record): success_step value 0/1, or 2 where the predicate raises.       */
int tl_label_records(const tl_records* recs, int32_t n_env,
                     const int32_t* env_cset, const tl_cset* csets,
                     int32_t n_cset, const tl_rules* rules /* host, NULL */,
                     uint8_t* step_mask, uint8_t* step_success,
                     tl_label* labels, void* stream);

/* exclusive scan of labels[].n_events (0 for failed episodes) -> ev_off[n+1].
 * scratch >= tl_scan_scratch_bytes(n) device bytes. */
size_t tl_scan_scratch_bytes(int32_t n);
int tl_scan_events(const tl_label* labels, int32_t n, int64_t* ev_off,
                   void* scratch, void* stream);

/* K2: ordered (kind, t) event lists at ev_off[e] (global EventKind ids). */
int tl_emit_events(const uint8_t* step_mask, const int64_t* rec_start,
                   const int32_t* n_rec, const tl_label* labels,
                   const int64_t* ev_off, int32_t n_env, uint8_t* ev_kind,
                   int32_t* ev_t, void* stream);

/* tl_scan_events + tl_emit_events in one launch (single-pass decoupled
 * look-back scan, then emission); scratch >= tl_scan_scratch_bytes(n).    */
int tl_scan_emit_events(const uint8_t* step_mask, const int64_t* rec_start,
                        const int32_t* n_rec, const tl_label* labels,
                        int32_t n_env, int64_t* ev_off, uint8_t* ev_kind,
                        int32_t* ev_t, void* scratch, void* stream);

/* classify given event lists: kinds at [ev_off[e], ev_off[e+1]). */
int tl_classify_events(const uint8_t* ev_kind, const int64_t* ev_off,
                       const uint8_t* subtask, const double* d0,
                       const uint8_t* d0_none, int32_t n,
                       const tl_rules* rules /* host */, tl_label* out,
                       void* stream);

/* K3+K4: for each seed, random_script(seed) -> realize(seed ^ 0x5EED) ->
 * label.  Two launches: a reset kernel (one thread per MT state: CPython
 * seeding + random_script) and the realize+label kernel (one warp per
 * episode).  Records go to out->planes (f32) at rec_start[e] =
 * e*cap_per_env (rec_start and n_rec written).  label_csets (device) is
 * indexed [subtask*3 + articulation kind] (0 none, 1 fridge, 2 drawer).
 * script_kind/script_gap/scripts (optional) receive the sampled scripts
 * (steps at e*(cfg.max_events+4)); scratch >= tl_fuzz_scratch_bytes(),
 * zero-filled before its first use (every call leaves its claim counters at
 * zero again).  Episodes are realized longest-first (length buckets filled
 * by the reset kernel) when cap_per_env > 64; results do not depend on it. */
size_t tl_fuzz_scratch_bytes(int32_t n_env, const tl_fuzz_cfg* cfg /* host */);
int tl_fuzz(const int64_t* seeds, int32_t n_env, int32_t subtask,
            const tl_fuzz_cfg* cfg /* host */,
            const tl_thresholds* th_realize /* host */,
            const tl_cset* label_csets, const tl_rules* rules /* host */,
            tl_records* out /* host struct, device arrays */,
            int32_t cap_per_env, uint8_t* script_kind, int32_t* script_gap,
            tl_script* scripts, uint8_t* step_mask, tl_label* labels,
            void* scratch, void* stream);

/* tl_fuzz + the ordered event lists: ev_off[n+1], (ev_kind, ev_t) at
 * ev_off[e] exactly as tl_scan_emit_events produces them (the reset, realize
 * and k_scan_emit kernels back to back on `stream`).  seeds, labels, ev_off,
 * ev_kind and ev_t may be pinned (mapped) host memory: the reset kernel reads
 * the seeds, the realize kernel writes each label once, and each
 * 32-episode tile's events are stored as one contiguous range of aligned
 * words (zero-copy end to end, bench.py e2e).  step_mask is required;
 * ev_capacity >= 4 * n_env * cap_per_env. */
int tl_fuzz_ev(const int64_t* seeds, int32_t n_env, int32_t subtask,
               const tl_fuzz_cfg* cfg /* host */,
               const tl_thresholds* th_realize /* host */,
               const tl_cset* label_csets, const tl_rules* rules /* host */,
               tl_records* out, int32_t cap_per_env, uint8_t* script_kind,
               int32_t* script_gap, tl_script* scripts, uint8_t* step_mask,
               tl_label* labels, int64_t* ev_off, uint8_t* ev_kind, int32_t* ev_t,
               int64_t ev_capacity, void* scratch, void* stream);

/* tl_fuzz / tl_fuzz_ev with a subtask per episode (subtasks[n_env] u8,
 * device: 0 Pick, 1 Place, 2 Open, 3 Close), one launch sequence for a
 * mixed batch -- e.g. the SetTable chains of C4 (Open, Pick, Place, Close
 * episodes of every chain).  Episode e is fuzz(seeds[e], subtasks[e]); an
 * out-of-range subtask gives that episode status TL_E_INVALID and no
 * records.  The other arguments as for tl_fuzz / tl_fuzz_ev.              */
int tl_fuzz_mixed(const int64_t* seeds, const uint8_t* subtasks, int32_t n_env,
                  const tl_fuzz_cfg* cfg /* host */,
                  const tl_thresholds* th_realize /* host */,
                  const tl_cset* label_csets, const tl_rules* rules /* host */,
                  tl_records* out, int32_t cap_per_env, uint8_t* script_kind,
                  int32_t* script_gap, tl_script* scripts, uint8_t* step_mask,
                  tl_label* labels, void* scratch, void* stream);
int tl_fuzz_ev_mixed(const int64_t* seeds, const uint8_t* subtasks, int32_t n_env,
                     const tl_fuzz_cfg* cfg /* host */,
                     const tl_thresholds* th_realize /* host */,
                     const tl_cset* label_csets, const tl_rules* rules /* host */,
                     tl_records* out, int32_t cap_per_env, uint8_t* script_kind,
                     int32_t* script_gap, tl_script* scripts, uint8_t* step_mask,
                     tl_label* labels, int64_t* ev_off, uint8_t* ev_kind, int32_t* ev_t,
                     int64_t ev_capacity, void* scratch, void* stream);

/* realize given scripts (device array) then label; out->rec_start/n_rec
 * are INPUTS here (host computed the layout).  label_csets indexed
 * [subtask*3 + articulation kind]; episodes may mix subtasks.
 * scratch >= tl_realize_scratch_bytes(n_env).                            */
size_t tl_realize_scratch_bytes(int32_t n_env);
int tl_realize(const tl_script* scripts, const uint8_t* step_kind,
               const int32_t* step_gap, int32_t n_env,
               const tl_thresholds* th_realize /* host */,
               const tl_cset* label_csets /* [4 subtasks][3 art] */,
               const tl_rules* rules /* host */, tl_records* out,
               uint8_t* step_mask, tl_label* labels, void* scratch,
               void* stream);

/* ---- K3 as an environment: reset / step(actions) -------------------------
 * synth.py:100-302 split at the record boundary: reset = _Realizer.__init__
 * + the t = 0 _emit; each step = _advance_cum, _apply(action) unless
 * TL_ACT_HOLD, _emit; one record per env per step.  The edge events of each
 * new record are folded online (events.py:94-193), so tl_env_labels
 * classifies the episode so far without re-reading records.
 * state: opaque device buffer of tl_env_state_bytes(n_env) bytes (realize
 * thresholds, label csets, 128 B per env + the env's MT19937 state).
 * Observations are time-major f32 planes (the tl_records plane order):
 *   obs[f*obs_stride + k*n_env + e], obs_grasped[k*n_env + e],
 *   step_mask[k*n_env + e] (EVENT_ORDER bits of the events that record fired)
 * for step k of the call (reset: k = 0).  An infeasible action (InfeasibleScript
 * in the reference) stops that env: status/err in its label, nothing written.
 * realize(script, seed) == tl_env_reset(script with .seed) followed by the
 * tl_env_script_actions stream; fuzz(seed) == tl_env_reset_fuzz + the same. */
size_t tl_env_state_bytes(int32_t n_env);
int tl_env_reset(void* state, int32_t n_env, int32_t dof, const tl_script* scripts,
                 const tl_thresholds* th_realize /* host */,
                 const tl_cset* label_csets /* device [4 subtasks][3 art] */,
                 float* obs, int64_t obs_stride, uint8_t* obs_grasped,
                 uint8_t* step_mask, void* stream);
/* random_script(seed, subtask, cfg) initial conditions + realize RNG seeded
 * with seed ^ 0x5EED (synth.py:510-515); the sampled scripts go to
 * scripts / script_kind / script_gap (steps at e*(cfg.max_events+4)) so
 * tl_env_script_actions replays fuzz(seed). */
int tl_env_reset_fuzz(void* state, const int64_t* seeds, int32_t n_env, int32_t subtask,
                      const tl_fuzz_cfg* cfg /* host */,
                      const tl_thresholds* th_realize /* host */,
                      const tl_cset* label_csets, tl_script* scripts,
                      uint8_t* script_kind, int32_t* script_gap, float* obs,
                      int64_t obs_stride, uint8_t* obs_grasped, uint8_t* step_mask,
                      void* stream);
int tl_env_step(void* state, int32_t n_env, int32_t dof,
                const uint8_t* actions /* [k_steps][n_env] */, int32_t k_steps,
                float* obs, int64_t obs_stride, uint8_t* obs_grasped,
                uint8_t* step_mask, void* stream);
/* label of every env's episode so far; infeasible envs report the InfeasibleScript
 * code with err_index = record index of the raising action and pad = that action.
 * n_rec (optional) = records emitted (0 for failed envs). */
int tl_env_labels(const void* state, int32_t n_env, const tl_rules* rules /* host */,
                  tl_label* labels, int32_t* n_rec, void* stream);
/* scripts -> actions[k][e] for records t = t0 + k (TL_ACT_HOLD between events,
 * TL_ACT_IDLE past the script's record count). */
int tl_env_script_actions(const tl_script* scripts, const uint8_t* step_kind,
                          const int32_t* step_gap, int32_t n_env, int32_t t0,
                          int32_t k_steps, uint8_t* actions, void* stream);

/* filter_buckets on the device (pipeline.py:276-304) for labels already in
 * episode_id order: bucket[i] = pool_b0[pool[key[i]*4 + subtask]] +
 * rule_lut[subtask*39 + mode] (position of the first allow rule of the
 * subtask containing the mode, -1 none); -1 for invalid labels, unmatched
 * modes or pool < 0.  Feeds tl_filter_select. */
int tl_filter_buckets(const tl_label* labels, const int32_t* key, int64_t n,
                      const int8_t* rule_lut, const int32_t* pool, const int32_t* pool_b0,
                      int32_t n_keys, int32_t* bucket, void* stream);

/* K5: filter_labels selection (pipeline.py:276-338).  Labels are already
 * in episode_id order.  bucket[i] in [-1, n_buckets): the (quota key,
 * subtask) pool's allow-rule position the label falls into (-1 = none).
 * Pool p owns buckets [pool_b0[p], pool_b0[p+1]) in rule order; bucket_w
 * are the rule weights.  Outputs selected[i] (0/1) and pool_selected[p].
 * scratch >= tl_filter_scratch_bytes(n, n_buckets, n_pools) device bytes. */
size_t tl_filter_scratch_bytes(int64_t n, int32_t n_buckets, int32_t n_pools);
int tl_filter_select(const int32_t* bucket, int64_t n, int32_t n_buckets,
                     int32_t n_pools, const int32_t* pool_b0,
                     const double* bucket_w, int64_t quota, uint8_t* selected,
                     int64_t* pool_selected, void* scratch, void* stream);

/* per-record predicates (predicates.py:16-99) for the records of n_env
 * episodes.  bits[r]: bit0 contact (force > contact_eps), bit1 grasped,
 * bit2 success_step, bit3 cum <= limit, bit4 cum > limit (failure_step),
 * bit5 A (Place: dist <= goal, Open: is_open, Close: is_closed), bit6 B
 * (Place: dist > goal, Open: slightly_opened, Close: slightly_closed vs
 * a0), bit7 is_static.  errs[r]: bit0 success_step raises, bit1 force NaN,
 * bit2 dist NaN, bit3 art NaN.  jmax[r] = j_max(q_arm, rest_arm) in f64.
 * a0 (optional, per episode) anchors slightly_closed (default: the
 * episode's records[0].art_q).  Any output pointer may be NULL.           */
int tl_eval_predicates(const tl_records* recs, int32_t n_env,
                       const int32_t* env_cset, const tl_cset* csets,
                       const double* a0, uint8_t* bits, uint8_t* errs,
                       double* jmax, void* stream);

/* exclusive scan of int32 counts -> off[n+1] (e.g. n_rec -> compact
 * rec_start); scratch >= tl_scan_scratch_bytes(n). */
int tl_scan_counts(const int32_t* counts, int32_t n, int64_t* off,
                   void* scratch, void* stream);

/* copy the records of a padded batch (tl_fuzz output) into a compact
 * batch: dst->planes/grasped at dst_start[e]; writes dst->rec_start/n_rec. */
int tl_compact_records(const tl_records* src, int32_t n_env,
                       const int64_t* dst_start, tl_records* dst, void* stream);

/* ---- structural validation (model.py:232-281 validate / check_valid) ----
 * Per-record invariant codes over a record batch.  dof may be 0 when only
 * the 9 scalar planes are present (validation reads dist_ee_rest,
 * dist_obj_goal, force_ee_target, cum_robot_force, art_q).  t (optional,
 * per record, same indexing as the planes): the stored step index, checked
 * against the record's position; NULL = implicit t.  vb[e]: the episode's
 * articulation (has_art = articulation_kind != None) and f64 bounds.
 * vflags[r] (optional) = TL_VF_* bits; vsum[e] = counts of records with an
 * error bit / the warning bit, the first flagged index (-1 if none) and
 * n_rec < 2.  Header checks (arm_dof, rest_arm length, bounds order,
 * Open/Close without articulation) are host-side: they need no records. */
enum {
  TL_VF_T_MISMATCH = 1,     /* "record i has step index t=.., expected i" */
  TL_VF_ARM_LENGTH = 2,     /* host objects only: arm vectors vs arm_dof   */
  TL_VF_CUM_INVALID = 4,    /* "cumulative force invalid at t=i: v"        */
  TL_VF_CUM_DECREASED = 8,  /* "cumulative force decreased at t=i"         */
  TL_VF_DEE_INVALID = 16,   /* "dist_ee_rest invalid at t=i: v"            */
  TL_VF_DOG_NEGATIVE = 32,  /* "dist_obj_goal negative at t=i: v"          */
  TL_VF_FET_NEGATIVE = 64,  /* "force_ee_target negative at t=i: v"        */
  TL_VF_ART_RANGE = 128     /* warning "art_q out of [qmin, qmax] at t=i"  */
};
typedef struct tl_vbounds {
  double art_qmin, art_qmax;
  int32_t has_art, pad;
} tl_vbounds;
typedef struct tl_vsummary {
  int32_t n_error_records, n_warning_records, first_flagged, too_short;
} tl_vsummary;
int tl_validate_records(const tl_records* recs, int32_t n_env, const tl_vbounds* vb,
                        const int64_t* t, uint8_t* vflags, tl_vsummary* vsum,
                        void* stream);

/* K6: counts per global mode id (status==0 only); hist[39] int64, zeroed
 * by the call. */
int tl_mode_histogram(const tl_label* labels, int32_t n, int64_t* hist,
                      void* stream);

/* ---- analytics counting (analytics.py:121-160, :279-298) ----------------
 * counts[g*42 + c] over the valid labels (status 0) of group g (group NULL =
 * one group): c < 39 mode id, 39 success_once, 40 success_at_end, 41 labels.
 * Zeroed by the call.  The host derives SoR/SaeR/FR and the per-mode
 * fractions exactly as mode_table does. */
int tl_group_mode_counts(const tl_label* labels, const int32_t* group, int64_t n,
                         int32_t n_groups, int64_t* counts, void* stream);
/* progressive_completion: slot_label[c*n_slots + k] = label index of chain
 * c's slot k, or -1 for an auto-success slot.  alive[k] = chains whose
 * bound slots 0..k all have success_once (status 0).  n_slots <= 64. */
int tl_chain_progress(const tl_label* labels, const int64_t* slot_label, int64_t n_chain,
                      int32_t n_slots, int64_t* alive, void* stream);

/* ---- the exchange step of the multi-GPU path --------------
 * nccl_comm is the caller's ncclComm_t (one rank per GPU).  Equal-size
 * shards: gathered[r*n_per_rank + i] = rank r's local[i] (pad the last shard).
 * counts is summed in place over ranks (mode histograms, tl_group_mode_counts
 * tables, progressive-completion alive counts).  NCCL is resolved from the
 * process at call time (the library is not linked against it). */
int tl_allgather_labels(void* nccl_comm, const tl_label* local, int64_t n_per_rank,
                        tl_label* gathered, void* stream);
int tl_allreduce_counts(void* nccl_comm, int64_t* counts, int64_t n, void* stream);

#ifdef __cplusplus
}
#endif
#endif
