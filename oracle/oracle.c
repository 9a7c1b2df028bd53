/*
 * oracle.c -- CPU restatement of the reference trajlab hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Compiled with
 * -ffp-contract=off so every double operation rounds exactly like the
 * CPython bytecode it restates (no fused multiply-add).
 *
 * Citations: /root/reference/pkg/src/trajlab/<file>:<line>.
 * Third-party arithmetic restated here (not in /root/reference):
 *   CPython 3.10/3.12 Modules/_randommodule.c (MT19937, init_by_array,
 *   random_random, getrandbits) and Lib/random.py (_randbelow_with_getrandbits,
 *   randint/randrange, choice, choices, uniform) -- unchanged between the
 *   reference run (3.10.12, pkg/test_output.txt:2) and this image (3.12.3);
 *   numpy float32 cast = IEEE round-to-nearest-even.
 */
#include "oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* CPython MT19937                                                     */
/* ------------------------------------------------------------------ */
#define MT_M 397
#define MT_MATRIX_A 0x9908b0dfU
#define MT_UPPER 0x80000000U
#define MT_LOWER 0x7fffffffU

static void init_genrand(or_mt* r, uint32_t s) {
  uint32_t* mt = r->mt;
  mt[0] = s;
  for (int i = 1; i < OR_MT_N; i++)
    mt[i] = 1812433253U * (mt[i - 1] ^ (mt[i - 1] >> 30)) + (uint32_t)i;
  r->index = OR_MT_N;
}

static void init_by_array(or_mt* r, const uint32_t* key, int klen) {
  uint32_t* mt = r->mt;
  init_genrand(r, 19650218U);
  int i = 1, j = 0;
  for (int k = (OR_MT_N > klen ? OR_MT_N : klen); k; k--) {
    mt[i] = (mt[i] ^ ((mt[i - 1] ^ (mt[i - 1] >> 30)) * 1664525U)) + key[j] +
            (uint32_t)j;
    i++;
    j++;
    if (i >= OR_MT_N) { mt[0] = mt[OR_MT_N - 1]; i = 1; }
    if (j >= klen) j = 0;
  }
  for (int k = OR_MT_N - 1; k; k--) {
    mt[i] = (mt[i] ^ ((mt[i - 1] ^ (mt[i - 1] >> 30)) * 1566083941U)) -
            (uint32_t)i;
    i++;
    if (i >= OR_MT_N) { mt[0] = mt[OR_MT_N - 1]; i = 1; }
  }
  mt[0] = 0x80000000U;
}

/* random.Random(int): key = little-endian 32-bit words of abs(seed) */
void or_mt_seed(or_mt* r, int64_t seed) {
  uint64_t n = seed < 0 ? (uint64_t)(-(seed + 1)) + 1u : (uint64_t)seed;
  uint32_t key[2];
  int klen = 1;
  key[0] = (uint32_t)n;
  key[1] = (uint32_t)(n >> 32);
  if (key[1]) klen = 2;
  init_by_array(r, key, klen);
}

uint32_t or_mt_genrand(or_mt* r) {
  uint32_t* mt = r->mt;
  uint32_t y;
  if (r->index >= OR_MT_N) {
    int kk;
    for (kk = 0; kk < OR_MT_N - MT_M; kk++) {
      y = (mt[kk] & MT_UPPER) | (mt[kk + 1] & MT_LOWER);
      mt[kk] = mt[kk + MT_M] ^ (y >> 1) ^ ((y & 1U) ? MT_MATRIX_A : 0U);
    }
    for (; kk < OR_MT_N - 1; kk++) {
      y = (mt[kk] & MT_UPPER) | (mt[kk + 1] & MT_LOWER);
      mt[kk] = mt[kk + (MT_M - OR_MT_N)] ^ (y >> 1) ^ ((y & 1U) ? MT_MATRIX_A : 0U);
    }
    y = (mt[OR_MT_N - 1] & MT_UPPER) | (mt[0] & MT_LOWER);
    mt[OR_MT_N - 1] = mt[MT_M - 1] ^ (y >> 1) ^ ((y & 1U) ? MT_MATRIX_A : 0U);
    r->index = 0;
  }
  y = mt[r->index++];
  y ^= (y >> 11);
  y ^= (y << 7) & 0x9d2c5680U;
  y ^= (y << 15) & 0xefc60000U;
  y ^= (y >> 18);
  return y;
}

/* random_random: (a*67108864.0+b)*(1.0/9007199254740992.0) */
double or_mt_random(or_mt* r) {
  uint32_t a = or_mt_genrand(r) >> 5, b = or_mt_genrand(r) >> 6;
  return ((double)a * 67108864.0 + (double)b) * (1.0 / 9007199254740992.0);
}

static int bit_length(uint32_t n) { return n ? 32 - __builtin_clz(n) : 0; }

/* Lib/random.py _randbelow_with_getrandbits; getrandbits(k<=32) = w>>(32-k) */
uint32_t or_mt_randbelow(or_mt* r, uint32_t n) {
  int k = bit_length(n);
  uint32_t v = or_mt_genrand(r) >> (32 - k);
  while (v >= n) v = or_mt_genrand(r) >> (32 - k);
  return v;
}

static int32_t randint(or_mt* r, int32_t a, int32_t b) {
  return a + (int32_t)or_mt_randbelow(r, (uint32_t)(b - a + 1));
}

static double uniform(or_mt* r, double a, double b) {
  return a + (b - a) * or_mt_random(r);
}

/* choices(population, weights)[0]: accumulate + bisect_right(cum, x, 0, n-1) */
static int choices_idx(or_mt* r, const double* w, int n) {
  double cum[8];
  double acc = 0.0;
  for (int i = 0; i < n; i++) { acc = (i == 0) ? w[0] : acc + w[i]; cum[i] = acc; }
  double total = cum[n - 1] + 0.0;
  double x = or_mt_random(r) * total;
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    int mid = (lo + hi) / 2;
    if (x < cum[mid]) hi = mid; else lo = mid + 1;
  }
  return lo;
}

/* ------------------------------------------------------------------ */
/* Thresholds lookups (thresholds.py:44-60)                            */
/* ------------------------------------------------------------------ */
static double collision_limit(const or_thresholds* th, int kind) {
  switch (kind) {
    case OR_PICK: return th->coll_pick;
    case OR_PLACE: return th->coll_place;
    default: return th->coll_artic;
  }
}

static double open_frac(const or_thresholds* th, int art_kind) {
  return art_kind == OR_ART_FRIDGE ? th->open_frac_fridge : th->open_frac_drawer;
}

/* EVENT_ORDER alphabets (events.py:38-52) */
static const uint8_t ALPHA[4][7] = {
    {OR_EV_CONTACT, OR_EV_GRASPED, OR_EV_DROPPED, OR_EV_SUCCESS,
     OR_EV_EXCESSIVE_COLLISIONS, 255, 255},
    {OR_EV_GRASPED, OR_EV_OBJ_AT_GOAL, OR_EV_RELEASED_AT_GOAL,
     OR_EV_RELEASED_OUTSIDE_GOAL, OR_EV_OBJ_LEFT_GOAL, OR_EV_SUCCESS,
     OR_EV_EXCESSIVE_COLLISIONS},
    {OR_EV_CONTACT, OR_EV_OPENED, OR_EV_SLIGHTLY_OPENED, OR_EV_CLOSED,
     OR_EV_SUCCESS, OR_EV_EXCESSIVE_COLLISIONS, 255},
    {OR_EV_CONTACT, OR_EV_CLOSED, OR_EV_SLIGHTLY_CLOSED, OR_EV_OPEN,
     OR_EV_SUCCESS, OR_EV_EXCESSIVE_COLLISIONS, 255}};

static int in_alphabet(int kind, int ev) {
  for (int i = 0; i < 7; i++)
    if (ALPHA[kind][i] == ev) return 1;
  return 0;
}

/* ------------------------------------------------------------------ */
/* random_script (synth.py:363-507)                                    */
/* ------------------------------------------------------------------ */
int32_t or_random_script(int64_t seed, int32_t kind, const or_fuzz_cfg* cfg,
                         or_script* s, uint8_t* step_kind, int32_t* step_gap,
                         int32_t cap) {
  or_mt rng;
  or_mt_seed(&rng, seed);
  int n = 0;
#define PUSH(k)                                              \
  do {                                                       \
    if (n >= cap) return -1;                                 \
    step_kind[n] = (uint8_t)(k);                             \
    step_gap[n] = randint(&rng, 1, cfg->max_gap);            \
    n++;                                                     \
  } while (0)

  s->subtask = kind;
  s->tail = randint(&rng, 1, cfg->max_tail);                       /* :372 */
  s->initial_grasped = 0;
  s->initial_contact = 0;
  s->initial_dist_obj_goal = 0.5;
  s->initial_level = OR_LVL_LOW;
  s->art_kind = OR_ART_FRIDGE;
  s->arm_dof = 7;
  if (kind == OR_OPEN || kind == OR_CLOSE)                          /* :374-376 */
    s->art_kind = or_mt_randbelow(&rng, 2) ? OR_ART_DRAWER : OR_ART_FRIDGE;

  if (kind == OR_PICK) {                                            /* :379-381 */
    s->initial_contact = or_mt_random(&rng) < 0.25;
    s->initial_grasped = s->initial_contact && or_mt_random(&rng) < 0.4;
  } else if (kind == OR_PLACE) {                                    /* :382-386 */
    s->initial_grasped = or_mt_random(&rng) < 0.8;
    if (or_mt_random(&rng) < 0.7)
      s->initial_dist_obj_goal = uniform(&rng, 0.3, 0.9);
    else
      s->initial_dist_obj_goal = uniform(&rng, 0.02, 0.12);
  } else {                                                          /* :387-392 */
    static const double w[3] = {0.85, 0.1, 0.05};
    int c = choices_idx(&rng, w, 3);
    if (kind == OR_OPEN)
      s->initial_level = c == 0 ? OR_LVL_LOW : c == 1 ? OR_LVL_SLIGHT : OR_LVL_OPEN;
    else
      s->initial_level = c == 0 ? OR_LVL_HIGH : c == 1 ? OR_LVL_SLIGHT : OR_LVL_CLOSED;
  }

  /* generator state (:394-403) */
  int grasped = s->initial_grasped, contact = s->initial_contact;
  int in_goal = s->initial_dist_obj_goal <= 0.15;
  int level = s->initial_level, band = 1;
  if (kind == OR_CLOSE) {
    level = s->initial_level == OR_LVL_CLOSED ? OR_LVL_CLOSED : OR_LVL_OPEN;
    band = s->initial_level != OR_LVL_CLOSED;
  }
  int contact_used = contact;                                       /* :461 */

  double nt = nearbyint((double)randint(&rng, 0, cfg->max_events) * cfg->edge_density);
  long n_target = (long)nt;                                         /* :463 */
  for (long it = 0; it < n_target; it++) {
    int moves[3], nm = 0;
    if (kind == OR_PICK) {                                          /* :406-414 */
      if (!contact) moves[nm++] = OR_EV_CONTACT;
      if (!grasped && contact) moves[nm++] = OR_EV_GRASPED;
      if (grasped) moves[nm++] = OR_EV_DROPPED;
    } else if (kind == OR_PLACE) {                                  /* :415-423 */
      if (!grasped) moves[nm++] = OR_EV_GRASPED;
      else moves[nm++] = in_goal ? OR_EV_RELEASED_AT_GOAL : OR_EV_RELEASED_OUTSIDE_GOAL;
      moves[nm++] = in_goal ? OR_EV_OBJ_LEFT_GOAL : OR_EV_OBJ_AT_GOAL;
    } else if (kind == OR_OPEN) {                                   /* :424-427 */
      moves[nm++] = OR_EV_CONTACT;
      moves[nm++] = level == OR_LVL_LOW ? OR_EV_SLIGHTLY_OPENED
                  : level == OR_LVL_SLIGHT ? OR_EV_OPENED : OR_EV_CLOSED;
    } else {                                                        /* :428-432 */
      moves[nm++] = OR_EV_CONTACT;
      if (level == OR_LVL_OPEN) { if (band) moves[nm++] = OR_EV_SLIGHTLY_CLOSED; }
      else if (level == OR_LVL_SLIGHT) moves[nm++] = OR_EV_CLOSED;
      else moves[nm++] = OR_EV_OPEN;
    }
    if ((kind == OR_OPEN || kind == OR_CLOSE) && contact_used) {    /* :466-467 */
      int k = 0;
      for (int i = 0; i < nm; i++) if (moves[i] != OR_EV_CONTACT) moves[k++] = moves[i];
      nm = k;
    }
    if (!nm) break;
    int mv = moves[or_mt_randbelow(&rng, (uint32_t)nm)];            /* :470 */
    if (mv == OR_EV_CONTACT) contact_used = 1;
    PUSH(mv);                                                       /* :473 */
    switch (mv) {                                                   /* :434-457 */
      case OR_EV_CONTACT: contact = 1; break;
      case OR_EV_GRASPED: grasped = 1; break;
      case OR_EV_DROPPED: grasped = 0; contact = 0; break;
      case OR_EV_RELEASED_AT_GOAL:
      case OR_EV_RELEASED_OUTSIDE_GOAL: grasped = 0; break;
      case OR_EV_OBJ_AT_GOAL: in_goal = 1; break;
      case OR_EV_OBJ_LEFT_GOAL: in_goal = 0; break;
      case OR_EV_SLIGHTLY_OPENED: level = OR_LVL_SLIGHT; break;
      case OR_EV_OPENED: level = OR_LVL_OPEN; break;
      case OR_EV_CLOSED: level = kind == OR_OPEN ? OR_LVL_LOW : OR_LVL_CLOSED; break;
      case OR_EV_SLIGHTLY_CLOSED: level = OR_LVL_SLIGHT; break;
      case OR_EV_OPEN: level = OR_LVL_OPEN; break;
    }
  }

  int feasible;                                                     /* :476-483 */
  if (kind == OR_PICK) feasible = grasped;
  else if (kind == OR_PLACE) feasible = !grasped && in_goal;
  else if (kind == OR_OPEN) feasible = level == OR_LVL_OPEN;
  else feasible = level == OR_LVL_CLOSED;

  int want = cfg->edge_density > 0 && or_mt_random(&rng) < cfg->success_prob; /* :485 */
  if (want && feasible) {
    PUSH(OR_EV_SUCCESS);
    double w[4] = {0.55, 0.2, 0.15, kind == OR_PLACE ? 0.1 : 0.0};  /* :488-491 */
    int suffix = choices_idx(&rng, w, 4);
    if (suffix == 1) {                                              /* :492-497 */
      /* the dict literal at :493-496 builds all four ScriptSteps, so gap()
       * is drawn four times (Pick, Place, Open, Close order) and the
       * subtask's own entry is kept */
      static const int brk[4] = {OR_EV_DROPPED, OR_EV_OBJ_LEFT_GOAL,
                                  OR_EV_CLOSED, OR_EV_OPEN};
      int32_t g[4];
      for (int i = 0; i < 4; i++) g[i] = randint(&rng, 1, cfg->max_gap);
      if (n >= cap) return -1;
      step_kind[n] = (uint8_t)brk[kind];
      step_gap[n] = g[kind];
      n++;
    } else if (suffix == 2) {
      PUSH(OR_EV_EXCESSIVE_COLLISIONS);
    } else if (suffix == 3) {
      PUSH(OR_EV_OBJ_LEFT_GOAL);
      PUSH(OR_EV_OBJ_AT_GOAL);
      PUSH(OR_EV_SUCCESS);
    }
  } else if (cfg->edge_density > 0 && or_mt_random(&rng) < 0.15) { /* :504-505 */
    PUSH(OR_EV_EXCESSIVE_COLLISIONS);
  }
#undef PUSH
  s->n_steps = n;
  return n;
}

/* ------------------------------------------------------------------ */
/* realize (synth.py:97-348)                                           */
/* ------------------------------------------------------------------ */
typedef struct {
  const or_script* s;
  const or_thresholds* th;
  or_mt rng;
  int kind, has_art, has_goal, has_force, dof;
  double limit, qmin, qmax, open_thresh, closed_thresh, slight_open_thresh;
  double lv_low, lv_slight, lv_open, a_q0, sc_thresh;
  int band_valid, art_level, grasped, at_rest;
  double art, force, dist, cum;
  or_record* out;
  int64_t n, cap;
} realizer;

static void r_emit(realizer* R) {                                   /* :166-190 */
  or_record tmp;
  or_record* o = R->n < R->cap ? &R->out[R->n] : &tmp;
  int d = R->dof;
  if (R->at_rest) {
    for (int i = 0; i < d; i++) { o->q_arm[i] = 0.0; o->qd_arm[i] = 0.0; }
    o->q_tor = o->v_base_x = o->v_base_y = o->omega_base = o->dist_ee_rest = 0.0;
  } else {
    for (int i = 0; i < d; i++) o->q_arm[i] = uniform(&R->rng, -0.3, 0.3);
    for (int i = 0; i < d; i++) o->qd_arm[i] = uniform(&R->rng, -0.4, 0.4);
    o->q_tor = uniform(&R->rng, -0.05, 0.05);
    o->v_base_x = uniform(&R->rng, -0.2, 0.2);
    o->v_base_y = uniform(&R->rng, -0.2, 0.2);
    o->omega_base = uniform(&R->rng, -0.3, 0.3);
    o->dist_ee_rest = uniform(&R->rng, 0.2, 1.0);
  }
  o->dist_obj_goal = R->dist;
  o->force_ee_target = R->has_force ? R->force : NAN;
  o->cum_robot_force = R->cum;
  o->art_q = R->art;
  o->grasped = R->grasped;
  /* _build (:312-330): np.float32 quantisation of every float column */
  for (int i = 0; i < d; i++) {
    o->q_arm[i] = (double)(float)o->q_arm[i];
    o->qd_arm[i] = (double)(float)o->qd_arm[i];
  }
  o->q_tor = (double)(float)o->q_tor;
  o->v_base_x = (double)(float)o->v_base_x;
  o->v_base_y = (double)(float)o->v_base_y;
  o->omega_base = (double)(float)o->omega_base;
  o->dist_ee_rest = (double)(float)o->dist_ee_rest;
  o->dist_obj_goal = (double)(float)o->dist_obj_goal;
  o->force_ee_target = (double)(float)o->force_ee_target;
  o->cum_robot_force = (double)(float)o->cum_robot_force;
  o->art_q = (double)(float)o->art_q;
  R->n++;
}

static void r_advance_cum(realizer* R) {                            /* :192-196 */
  double headroom = R->limit * 0.9 - R->cum;
  if (headroom > 0) R->cum += uniform(&R->rng, 0.0, headroom * 0.05);
}

static void r_hold(realizer* R, int64_t steps) {                    /* :198-201 */
  for (int64_t i = 0; i < steps; i++) { r_advance_cum(R); r_emit(R); }
}

static int r_apply(realizer* R, int ev) {                           /* :205-296 */
  const or_thresholds* th = R->th;
  int k = R->kind;
  if (!in_alphabet(k, ev)) return OR_INF_NOT_IN_ALPHABET;
  if (ev == OR_EV_EXCESSIVE_COLLISIONS) {
    if (R->cum > R->limit) return OR_INF_LIMIT_EXCEEDED;
    R->cum = R->limit * 1.05;
    return 0;
  }
  if (ev == OR_EV_SUCCESS) {
    int ok;
    if (k == OR_PICK) ok = R->grasped;
    else if (k == OR_PLACE) ok = !R->grasped && R->dist <= th->goal_radius;
    else if (k == OR_OPEN) ok = R->art_level == OR_LVL_OPEN;
    else ok = R->art_level == OR_LVL_CLOSED;
    if (!ok || R->at_rest) return OR_INF_SUCCESS_UNREACHABLE;
    R->at_rest = 1;
    return 0;
  }
  R->at_rest = 0;
  switch (ev) {
    case OR_EV_CONTACT:
      if (!R->has_force) return OR_INF_CONTACT_UNDEFINED;
      if (R->force > 0) return OR_INF_CONTACT_AGAIN;
      R->force = 1.2;
      return 0;
    case OR_EV_GRASPED:
      if (R->grasped) return OR_INF_GRASPED_AGAIN;
      if (k == OR_PICK && R->force == 0) return OR_INF_PICK_GRASP_NO_FORCE;
      R->grasped = 1;
      return 0;
    case OR_EV_DROPPED:
      if (!R->grasped) return OR_INF_DROPPED_NOT_GRASPED;
      R->grasped = 0;
      R->force = 0.0;
      return 0;
    case OR_EV_OBJ_AT_GOAL:
      if (R->dist <= th->goal_radius) return OR_INF_AT_GOAL_ALREADY;
      R->dist = uniform(&R->rng, 0.02, 0.12);
      return 0;
    case OR_EV_OBJ_LEFT_GOAL:
      if (R->dist > th->goal_radius) return OR_INF_LEFT_NOT_AT_GOAL;
      R->dist = uniform(&R->rng, 0.3, 0.8);
      return 0;
    case OR_EV_RELEASED_AT_GOAL:
      if (!R->grasped || R->dist > th->goal_radius) return OR_INF_RAG;
      R->grasped = 0;
      return 0;
    case OR_EV_RELEASED_OUTSIDE_GOAL:
      if (!R->grasped || R->dist <= th->goal_radius) return OR_INF_ROG;
      R->grasped = 0;
      return 0;
    case OR_EV_SLIGHTLY_OPENED:
      if (k != OR_OPEN || R->art_level != OR_LVL_LOW) return OR_INF_SLIGHTLY_OPENED;
      R->art_level = OR_LVL_SLIGHT;
      R->art = R->lv_slight;
      return 0;
    case OR_EV_OPENED:
      if (k != OR_OPEN || R->art_level != OR_LVL_SLIGHT) return OR_INF_OPENED;
      R->art_level = OR_LVL_OPEN;
      R->art = R->lv_open;
      return 0;
    case OR_EV_CLOSED:
      if (k == OR_OPEN) {
        if (R->art_level != OR_LVL_OPEN) return OR_INF_CLOSED_OPEN;
        R->art_level = OR_LVL_LOW;
        R->art = R->lv_low;
        return 0;
      }
      if (k == OR_CLOSE) {
        if (R->art_level != OR_LVL_SLIGHT) return OR_INF_CLOSED_CLOSE;
        R->art_level = OR_LVL_CLOSED;
        R->art = R->qmin;
        return 0;
      }
      return OR_INF_NOT_IN_ALPHABET;
    case OR_EV_SLIGHTLY_CLOSED:
      if (R->art_level != OR_LVL_OPEN) return OR_INF_SC_LEVEL;
      if (!R->band_valid) return OR_INF_SC_BAND;
      R->art_level = OR_LVL_SLIGHT;
      R->art = (R->sc_thresh + R->closed_thresh) / 2;
      return 0;
    case OR_EV_OPEN:
      if (k == OR_CLOSE) {
        if (R->art_level != OR_LVL_CLOSED) return OR_INF_OPEN_CLOSE;
        R->art_level = OR_LVL_OPEN;
        R->art = R->a_q0 > R->closed_thresh ? R->a_q0 : R->qmax;
        return 0;
      }
      return OR_INF_NOT_IN_ALPHABET;
  }
  return OR_INF_NOT_IN_ALPHABET;
}

int64_t or_realize_len(const or_script* s) {
  int64_t n = 1;
  for (int i = 0; i < s->n_steps; i++) n += s->step_gap[i];
  int64_t tail = s->tail;
  int64_t m = s->n_steps ? 0 : 1;
  n += tail > m ? tail : m;
  if (n < 2) n = 2;
  return n;
}

int64_t or_realize(const or_script* s, int64_t seed, const or_thresholds* th,
                   or_record* out, int64_t cap, int32_t* err_step) {
  realizer R;
  memset(&R, 0, sizeof(R));
  R.s = s;
  R.th = th;
  R.out = out;
  R.cap = cap;
  R.dof = s->arm_dof;
  or_mt_seed(&R.rng, seed);                                         /* :103 */
  int k = s->subtask;
  R.kind = k;
  R.has_art = k == OR_OPEN || k == OR_CLOSE;
  R.has_goal = k == OR_PLACE;
  R.has_force = k != OR_PLACE;
  R.limit = collision_limit(th, k);
  *err_step = -1;
  if (R.has_art) {                                                  /* :111-148 */
    if (s->art_kind == OR_ART_FRIDGE) { R.qmin = 0.0; R.qmax = 1.6; }
    else if (s->art_kind == OR_ART_DRAWER) { R.qmin = 0.0; R.qmax = 0.5; }
    else return -OR_INF_INIT_LEVEL;
    double span = R.qmax - R.qmin;
    double ofrac = open_frac(th, s->art_kind);
    R.open_thresh = ofrac * span + R.qmin;
    R.closed_thresh = th->close_frac * span + R.qmin;
    R.slight_open_thresh = th->slightly_open_frac * span + R.qmin;
    if (k == OR_OPEN) {
      R.lv_low = R.qmin;
      R.lv_slight = (R.slight_open_thresh + R.open_thresh) / 2;
      R.lv_open = (R.open_thresh + R.qmax) / 2;
      int lv = s->initial_level;
      if (lv == OR_LVL_LOW) R.art = R.lv_low;
      else if (lv == OR_LVL_SLIGHT) R.art = R.lv_slight;
      else if (lv == OR_LVL_OPEN) R.art = R.lv_open;
      else return -OR_INF_INIT_LEVEL;
      R.art_level = lv;
    } else {
      int lv = s->initial_level;
      if (lv == OR_LVL_HIGH) R.a_q0 = R.qmax;
      else if (lv == OR_LVL_SLIGHT) R.a_q0 = R.qmin + 0.3 * span;
      else if (lv == OR_LVL_CLOSED) R.a_q0 = R.qmin;
      else return -OR_INF_INIT_LEVEL;
      R.sc_thresh = R.a_q0 - th->slightly_close_frac * span;
      R.band_valid = R.sc_thresh > R.closed_thresh;
      R.art = R.a_q0;
      R.art_level = lv == OR_LVL_CLOSED ? OR_LVL_CLOSED : OR_LVL_OPEN;
    }
  } else {
    R.art = NAN;
  }
  R.grasped = s->initial_grasped;                                   /* :152-158 */
  R.force = (R.has_force && s->initial_contact) ? 1.2 : 0.0;
  if (k == OR_PICK && R.grasped && !s->initial_contact)
    return -OR_INF_PICK_GRASPED_NO_CONTACT;
  R.dist = R.has_goal ? s->initial_dist_obj_goal : NAN;
  R.at_rest = 0;
  R.cum = 0.0;

  r_emit(&R);                                                       /* :298-310 */
  for (int i = 0; i < s->n_steps; i++) {
    if (s->step_gap[i] < 1) { *err_step = i; return -OR_INF_GAP; }
    r_hold(&R, s->step_gap[i] - 1);
    r_advance_cum(&R);
    int e = r_apply(&R, s->step_kind[i]);
    if (e) { *err_step = i; return -e; }
    r_emit(&R);
  }
  int64_t tail = s->tail, m = s->n_steps ? 0 : 1;
  r_hold(&R, tail > m ? tail : m);
  if (R.n < 2) r_hold(&R, 1);
  return R.n;
}

/* ------------------------------------------------------------------ */
/* predicates (predicates.py:16-99)                                    */
/* ------------------------------------------------------------------ */
/* Python max() over a generator: first element wins unless a later one is
 * strictly greater (NaN never compares greater, a leading NaN sticks). */
static double py_max_absdiff(const double* q, const double* r, int n) {
  double m = fabs(q[0] - (r ? r[0] : 0.0));
  for (int i = 1; i < n; i++) {
    double v = fabs(q[i] - (r ? r[i] : 0.0));
    if (v > m) m = v;
  }
  return m;
}

static int is_static(const or_record* rec, const or_thresholds* th, int dof) {
  return py_max_absdiff(rec->qd_arm, NULL, dof) <= th->static_qd_arm &&
         fabs(rec->v_base_x) <= th->static_v_base &&
         fabs(rec->v_base_y) <= th->static_v_base &&
         fabs(rec->omega_base) <= th->static_omega;
}

static int at_rest(const or_record* rec, const or_header* h,
                   const or_thresholds* th, double jlim, int torso) {
  if (rec->dist_ee_rest > th->rest_radius) return 0;
  double jm = h->arm_dof > 0 ? py_max_absdiff(rec->q_arm, h->rest_arm, h->arm_dof) : 0.0;
  if (jm > jlim) return 0;
  if (torso && fabs(rec->q_tor - h->rest_tor) > th->j_tor_max) return 0;
  return is_static(rec, th, h->arm_dof);
}

int32_t or_success_step(const or_record* rec, const or_header* h,
                        const or_thresholds* th, int32_t* err) {
  int k = h->subtask;
  *err = 0;
  if (rec->cum_robot_force > collision_limit(th, k)) return 0;
  double span = h->art_qmax - h->art_qmin;
  switch (k) {
    case OR_PICK:
      return rec->grasped && at_rest(rec, h, th, th->j_arm_pick, 0);
    case OR_PLACE:
      if (rec->grasped) return 0;
      if (isnan(rec->dist_obj_goal)) { *err = OR_ERR_NAN_SUCCESS_DIST; return 0; }
      return rec->dist_obj_goal <= th->goal_radius &&
             at_rest(rec, h, th, th->j_arm_other, 1);
    case OR_OPEN:
      if (h->art_kind == OR_ART_NONE) { *err = OR_ERR_MISSING_ART; return 0; }
      if (isnan(rec->art_q)) { *err = OR_ERR_NAN_ART; return 0; }
      return rec->art_q >= open_frac(th, h->art_kind) * span + h->art_qmin &&
             at_rest(rec, h, th, th->j_arm_other, 1);
    default:
      if (h->art_kind == OR_ART_NONE) { *err = OR_ERR_MISSING_ART; return 0; }
      if (isnan(rec->art_q)) { *err = OR_ERR_NAN_ART; return 0; }
      return rec->art_q <= th->close_frac * span + h->art_qmin &&
             at_rest(rec, h, th, th->j_arm_other, 1);
  }
}

/* ------------------------------------------------------------------ */
/* extract_events (events.py:94-193)                                   */
/* ------------------------------------------------------------------ */
int32_t or_extract_events(const or_record* recs, int64_t n, const or_header* h,
                          const or_thresholds* th, uint8_t* ev_kind,
                          int32_t* ev_t, int32_t cap, double* d0) {
  if (n < 2) return -OR_ERR_TOO_SHORT;                              /* :96-97 */
  int k = h->subtask;
  double limit = collision_limit(th, k);
  uint8_t* succ = (uint8_t*)malloc((size_t)n);
  uint8_t* a = (uint8_t*)malloc((size_t)n);
  uint8_t* b = (uint8_t*)malloc((size_t)n);
  int32_t ne = 0, err = 0;
#define EMIT(kind, t)                                  \
  do {                                                 \
    if (ne < cap) { ev_kind[ne] = (uint8_t)(kind); ev_t[ne] = (int32_t)(t); } \
    ne++;                                              \
  } while (0)
  for (int64_t t = 0; t < n && !err; t++) succ[t] = (uint8_t)or_success_step(&recs[t], h, th, &err); /* :105 */
  if (err) goto done;
  *d0 = NAN;
  double span = h->art_qmax - h->art_qmin;
  if (k == OR_PICK || k == OR_OPEN || k == OR_CLOSE) {               /* _contact_flags :83-91 */
    for (int64_t t = 0; t < n; t++) {
      double f = recs[t].force_ee_target;
      if (isnan(f)) { err = OR_ERR_NAN_FORCE; goto done; }
      a[t] = f > th->contact_eps;
    }
  }
  if (k == OR_PICK) {                                               /* :113-124 */
    for (int64_t t = 1; t < n; t++) {
      if (!a[t - 1] && a[t]) EMIT(OR_EV_CONTACT, t);
      if (!recs[t - 1].grasped && recs[t].grasped) EMIT(OR_EV_GRASPED, t);
      if (recs[t - 1].grasped && !recs[t].grasped) EMIT(OR_EV_DROPPED, t);
      if (!succ[t - 1] && succ[t]) EMIT(OR_EV_SUCCESS, t);
      if (recs[t - 1].cum_robot_force <= limit && limit < recs[t].cum_robot_force)
        EMIT(OR_EV_EXCESSIVE_COLLISIONS, t);
    }
  } else if (k == OR_PLACE) {                                       /* :126-150 */
    for (int64_t t = 0; t < n; t++)
      if (isnan(recs[t].dist_obj_goal)) { err = OR_ERR_NAN_PLACE_DIST; goto done; }
    *d0 = recs[0].dist_obj_goal;
    double r = th->goal_radius;
    for (int64_t t = 1; t < n; t++) {
      double dp = recs[t - 1].dist_obj_goal, dc = recs[t].dist_obj_goal;
      int gp = recs[t - 1].grasped, gc = recs[t].grasped;
      if (!gp && gc) EMIT(OR_EV_GRASPED, t);
      if (dp > r && r >= dc) EMIT(OR_EV_OBJ_AT_GOAL, t);
      if (gp && !gc) EMIT(dc <= r ? OR_EV_RELEASED_AT_GOAL : OR_EV_RELEASED_OUTSIDE_GOAL, t);
      if (dp <= r && r < dc) EMIT(OR_EV_OBJ_LEFT_GOAL, t);
      if (!succ[t - 1] && succ[t]) EMIT(OR_EV_SUCCESS, t);
      if (recs[t - 1].cum_robot_force <= limit && limit < recs[t].cum_robot_force)
        EMIT(OR_EV_EXCESSIVE_COLLISIONS, t);
    }
  } else if (k == OR_OPEN) {                                        /* :152-169 */
    if (h->art_kind == OR_ART_NONE) { err = OR_ERR_MISSING_ART; goto done; }
    double ocut = open_frac(th, h->art_kind) * span + h->art_qmin;
    double scut = th->slightly_open_frac * span + h->art_qmin;
    for (int64_t t = 0; t < n; t++)
      if (isnan(recs[t].art_q)) { err = OR_ERR_NAN_ART; goto done; }
    for (int64_t t = 0; t < n; t++) { b[t] = recs[t].art_q >= ocut; succ[t] |= (uint8_t)((recs[t].art_q >= scut) << 1); }
    for (int64_t t = 1; t < n; t++) {
      int sp = succ[t - 1] & 1, sc = succ[t] & 1;
      int lp = (succ[t - 1] >> 1) & 1, lc = (succ[t] >> 1) & 1;
      if (!a[t - 1] && a[t]) EMIT(OR_EV_CONTACT, t);
      if (!b[t - 1] && b[t]) EMIT(OR_EV_OPENED, t);
      if (!lp && lc) EMIT(OR_EV_SLIGHTLY_OPENED, t);
      if (b[t - 1] && !b[t]) EMIT(OR_EV_CLOSED, t);
      if (!sp && sc) EMIT(OR_EV_SUCCESS, t);
      if (recs[t - 1].cum_robot_force <= limit && limit < recs[t].cum_robot_force)
        EMIT(OR_EV_EXCESSIVE_COLLISIONS, t);
    }
  } else {                                                          /* :171-190 */
    if (h->art_kind == OR_ART_NONE) { err = OR_ERR_MISSING_ART; goto done; }
    double ccut = th->close_frac * span + h->art_qmin;
    for (int64_t t = 0; t < n; t++)
      if (isnan(recs[t].art_q)) { err = OR_ERR_NAN_ART; goto done; }
    double sc_thresh = recs[0].art_q - th->slightly_close_frac * span;
    for (int64_t t = 0; t < n; t++) { b[t] = recs[t].art_q <= ccut; succ[t] |= (uint8_t)((recs[t].art_q < sc_thresh) << 1); }
    for (int64_t t = 1; t < n; t++) {
      int sp = succ[t - 1] & 1, sc = succ[t] & 1;
      int lp = (succ[t - 1] >> 1) & 1, lc = (succ[t] >> 1) & 1;
      if (!a[t - 1] && a[t]) EMIT(OR_EV_CONTACT, t);
      if (!b[t - 1] && b[t]) EMIT(OR_EV_CLOSED, t);
      if (!lp && lc) EMIT(OR_EV_SLIGHTLY_CLOSED, t);
      if (b[t - 1] && !b[t]) EMIT(OR_EV_OPEN, t);
      if (!sp && sc) EMIT(OR_EV_SUCCESS, t);
      if (recs[t - 1].cum_robot_force <= limit && limit < recs[t].cum_robot_force)
        EMIT(OR_EV_EXCESSIVE_COLLISIONS, t);
    }
  }
#undef EMIT
done:
  free(succ);
  free(a);
  free(b);
  return err ? -err : ne;
}

/* ------------------------------------------------------------------ */
/* classify (modes.py:24-253)                                          */
/* ------------------------------------------------------------------ */
#define GOAL_RADIUS 0.15 /* modes.py:65 literal */
static const int MODE_BASE[4] = {0, 9, 21, 30};
static const int N_SUCC[4] = {4, 5, 3, 3};
static const int N_MODES[4] = {9, 12, 9, 9};

typedef struct { int size; int last[OR_EV_COUNT]; double d0; int d0_none; int s1; } sig_t;

/* evaluates one builtin rule (global mode id); returns 1/0 or -status */
static int rule_pred(int m, const sig_t* c) {
  const int* L = c->last;
  int exc = L[OR_EV_EXCESSIVE_COLLISIONS] >= 0;
#define D0_LE(res) do { if (c->d0_none) return -OR_ERR_D0_NONE_LE; res = c->d0 <= GOAL_RADIUS; } while (0)
#define D0_GT(res) do { if (c->d0_none) return -OR_ERR_D0_NONE_GT; res = c->d0 > GOAL_RADIUS; } while (0)
  int x;
  switch (m) {
    /* pick (:68-92) */
    case 0: return c->s1;
    case 1: return !exc && L[OR_EV_DROPPED] <= L[OR_EV_GRASPED];
    case 2: return !exc && L[OR_EV_DROPPED] > L[OR_EV_GRASPED];
    case 3: return exc;
    case 4: return exc;
    case 5: return c->size == 0;
    case 6: return L[OR_EV_CONTACT] >= 0 && L[OR_EV_GRASPED] < 0 && L[OR_EV_DROPPED] < 0;
    case 7: return L[OR_EV_DROPPED] >= 0 && L[OR_EV_DROPPED] > L[OR_EV_GRASPED];
    case 8: return 1;
    /* place (:95-147) */
    case 9:
      if (!(c->size <= 4)) return 0;
      if (!(L[OR_EV_RELEASED_AT_GOAL] >= 0)) { D0_LE(x); if (!x) return 0; }
      return L[OR_EV_OBJ_LEFT_GOAL] <= L[OR_EV_OBJ_AT_GOAL] && !exc;
    case 10:
      if (!(c->size <= 4)) return 0;
      if (!(L[OR_EV_RELEASED_OUTSIDE_GOAL] >= 0)) { D0_GT(x); if (!x) return 0; }
      return L[OR_EV_OBJ_LEFT_GOAL] <= L[OR_EV_OBJ_AT_GOAL] && !exc;
    case 11: return L[OR_EV_OBJ_AT_GOAL] < L[OR_EV_OBJ_LEFT_GOAL] && !exc;
    case 12: return c->size > 4 && L[OR_EV_OBJ_AT_GOAL] >= L[OR_EV_OBJ_LEFT_GOAL] && !exc;
    case 13: return exc;
    case 14: return exc;
    case 15: return c->size == 0;
    case 16: return c->size > 0 && L[OR_EV_OBJ_AT_GOAL] < 0;
    case 17:
    case 18: {
      if (L[OR_EV_OBJ_AT_GOAL] < 0) return 0;
      int latest = 0;
      if (c->size <= 2) {
        if (m == 17) D0_LE(latest); else D0_GT(latest);
      }
      if (!latest) {
        int a = m == 17 ? L[OR_EV_RELEASED_AT_GOAL] : L[OR_EV_RELEASED_OUTSIDE_GOAL];
        int b = m == 17 ? L[OR_EV_RELEASED_OUTSIDE_GOAL] : L[OR_EV_RELEASED_AT_GOAL];
        latest = a > b && a > L[OR_EV_GRASPED];
      }
      return latest && L[OR_EV_OBJ_LEFT_GOAL] > L[OR_EV_OBJ_AT_GOAL];
    }
    case 19:
      return L[OR_EV_OBJ_AT_GOAL] >= 0 && L[OR_EV_GRASPED] > L[OR_EV_RELEASED_AT_GOAL] &&
             L[OR_EV_GRASPED] > L[OR_EV_RELEASED_OUTSIDE_GOAL];
    case 20: return 1;
    /* open (:150-176) */
    case 21: return !exc && L[OR_EV_OPENED] >= L[OR_EV_CLOSED];
    case 22: return !exc && L[OR_EV_OPENED] < L[OR_EV_CLOSED];
    case 23: return exc;
    case 24: return exc;
    case 25: return L[OR_EV_CONTACT] < 0;
    case 26: return L[OR_EV_CLOSED] >= 0 && L[OR_EV_CLOSED] > L[OR_EV_OPENED] &&
                    L[OR_EV_CLOSED] > L[OR_EV_SLIGHTLY_OPENED];
    case 27: return L[OR_EV_SLIGHTLY_OPENED] > L[OR_EV_OPENED] &&
                    L[OR_EV_SLIGHTLY_OPENED] > L[OR_EV_CLOSED];
    case 28: return L[OR_EV_OPENED] >= 0;
    case 29: return 1;
    /* close (:179-205) */
    case 30: return !exc && L[OR_EV_CLOSED] >= L[OR_EV_OPEN];
    case 31: return !exc && L[OR_EV_CLOSED] < L[OR_EV_OPEN];
    case 32: return exc;
    case 33: return exc;
    case 34: return L[OR_EV_CONTACT] < 0;
    case 35: return L[OR_EV_CLOSED] >= 0 && L[OR_EV_OPEN] > L[OR_EV_CLOSED] &&
                    L[OR_EV_OPEN] > L[OR_EV_SLIGHTLY_CLOSED];
    case 36: return L[OR_EV_SLIGHTLY_CLOSED] > L[OR_EV_CLOSED] &&
                    L[OR_EV_SLIGHTLY_CLOSED] > L[OR_EV_OPEN];
    case 37: return L[OR_EV_CLOSED] >= 0;
    case 38: return 1;
  }
#undef D0_LE
#undef D0_GT
  return 0;
}

static int success_at_end_mode(int m) {                             /* :226-232 */
  return m == 0 || m == 1 || m == 9 || m == 10 || m == 12 || m == 21 || m == 30;
}

int32_t or_classify(int32_t subtask, const uint8_t* kinds, int32_t n, double d0,
                    int32_t d0_none, const int32_t* rule_order, int32_t n_rules,
                    int32_t* success_once, int32_t* success_at_end) {
  sig_t c;
  c.size = n;
  for (int i = 0; i < OR_EV_COUNT; i++) c.last[i] = -1;
  for (int i = 0; i < n; i++) c.last[kinds[i]] = i;
  c.d0 = d0;
  c.d0_none = d0_none;
  c.s1 = n == 3 && kinds[0] == OR_EV_CONTACT && kinds[1] == OR_EV_GRASPED &&
         kinds[2] == OR_EV_SUCCESS;
  int succ = c.last[OR_EV_SUCCESS] >= 0;
  *success_once = succ;
  *success_at_end = 0;
  int order[16], no = 0;
  if (!rule_order) {
    int base = MODE_BASE[subtask];
    if (succ) for (int i = 0; i < N_SUCC[subtask]; i++) order[no++] = base + i;
    else for (int i = N_SUCC[subtask]; i < N_MODES[subtask]; i++) order[no++] = base + i;
  } else {
    /* rule_order = [n_succ, ids..., n_fail, ids...] */
    int ns = rule_order[0];
    const int32_t* p = succ ? rule_order + 1 : rule_order + 2 + ns;
    int cnt = succ ? ns : rule_order[1 + ns];
    for (int i = 0; i < cnt && i < 16; i++) order[no++] = p[i];
    (void)n_rules;
  }
  for (int i = 0; i < no; i++) {
    int r = rule_pred(order[i], &c);
    if (r < 0) return r;
    if (r) {
      *success_at_end = success_at_end_mode(order[i]);
      return order[i];
    }
  }
  return -OR_ERR_MODE_COVERAGE;
}

/* ------------------------------------------------------------------ */
/* filter_labels selection loop (pipeline.py:276-338)                  */
/* ------------------------------------------------------------------ */
int64_t or_filter_select(int64_t n, const int32_t* pool, const int32_t* subtask,
                         const int32_t* rule, int32_t n_pools,
                         const double* rule_w, const int32_t* n_rules,
                         int64_t quota, uint8_t* selected,
                         int64_t* pool_selected) {
  /* bucket = (pool, rule position); lists in episode order (:289-298) */
  int64_t nb = (int64_t)n_pools * 16;
  int64_t* cnt = (int64_t*)calloc((size_t)nb + 1, sizeof(int64_t));
  int32_t* pool_sub = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n_pools > 0 ? n_pools : 1));
  for (int p = 0; p < n_pools; p++) pool_sub[p] = -1;
  for (int64_t i = 0; i < n; i++) {
    selected[i] = 0;
    if (rule[i] < 0) continue;
    cnt[(int64_t)pool[i] * 16 + rule[i] + 1]++;
    pool_sub[pool[i]] = subtask[i];
  }
  for (int64_t b = 0; b < nb; b++) cnt[b + 1] += cnt[b];
  int64_t* items = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  int64_t* fill = (int64_t*)calloc((size_t)nb, sizeof(int64_t));
  for (int64_t i = 0; i < n; i++) {
    if (rule[i] < 0) continue;
    int64_t b = (int64_t)pool[i] * 16 + rule[i];
    items[cnt[b] + fill[b]++] = i;
  }
  int64_t total = 0;
  for (int p = 0; p < n_pools; p++) {                                /* :302-326 */
    int s = pool_sub[p];
    int64_t sel = 0;
    if (s >= 0) {
      int nr = n_rules[s];
      int64_t taken[16] = {0}, cur[16] = {0};
      while (sel < quota) {
        int best = -1;
        double best_key = 0.0;
        for (int pos = 0; pos < nr; pos++) {
          int64_t b = (int64_t)p * 16 + pos;
          if (cur[pos] >= cnt[b + 1] - cnt[b]) continue;
          double key = (double)taken[pos] / rule_w[s * 16 + pos];
          if (best < 0 || key < best_key) { best = pos; best_key = key; }
        }
        if (best < 0) break;
        int64_t b = (int64_t)p * 16 + best;
        selected[items[cnt[b] + cur[best]]] = 1;
        cur[best]++;
        taken[best]++;
        sel++;
      }
    }
    if (pool_selected) pool_selected[p] = sel;
    total += sel;
  }
  free(cnt);
  free(pool_sub);
  free(items);
  free(fill);
  return total;
}

/* ------------------------------------------------------------------ */
/* Batched fuzz -> extract_events -> classify (CPU baseline)           */
/* tests/test_acceptance.py:30-36 loop, optionally multi-threaded       */
/* ------------------------------------------------------------------ */
typedef struct {
  int64_t s0, s1;
  int32_t kind;
  const or_fuzz_cfg* cfg;
  const or_thresholds* th;
  uint8_t* mode_out;
  int32_t* nev_out;
  int64_t* nrec_out;
  uint8_t* flags_out;   /* optional: bit 0 success_once, bit 1 success_at_end */
  double* d0_out;       /* optional: initial_dist_obj_goal (NaN if absent) */
  int64_t ev_stride;    /* optional event lists: ev_*_out[i * ev_stride + k] */
  uint8_t* ev_kind_out;
  int32_t* ev_t_out;
  int64_t base;
  int64_t records;
} job_t;

static void* fuzz_job(void* arg) {
  job_t* J = (job_t*)arg;
  int cap_steps = J->cfg->max_events + 8;
  uint8_t* sk = (uint8_t*)malloc((size_t)cap_steps);
  int32_t* sg = (int32_t*)malloc(sizeof(int32_t) * (size_t)cap_steps);
  int64_t rcap = 1 + (int64_t)cap_steps * J->cfg->max_gap + J->cfg->max_tail + 2;
  or_record* recs = (or_record*)malloc(sizeof(or_record) * (size_t)rcap);
  uint8_t* ek = (uint8_t*)malloc((size_t)(4 * rcap));
  int32_t* et = (int32_t*)malloc(sizeof(int32_t) * (size_t)(4 * rcap));
  or_header h;
  memset(&h, 0, sizeof(h));
  h.subtask = J->kind;
  h.arm_dof = 7;
  for (int64_t seed = J->s0; seed < J->s1; seed++) {
    or_script s;
    int32_t ns = or_random_script(seed, J->kind, J->cfg, &s, sk, sg, cap_steps);
    s.step_kind = sk;
    s.step_gap = sg;
    (void)ns;
    int32_t es;
    int64_t n = or_realize(&s, seed ^ 0x5EED, J->th, recs, rcap, &es);
    int32_t mode = -1, nev = 0, so = 0, se = 0;
    double d0 = NAN;
    if (n > 0) {
      h.art_kind = (J->kind == OR_OPEN || J->kind == OR_CLOSE) ? s.art_kind : OR_ART_NONE;
      h.art_qmin = h.art_kind == OR_ART_FRIDGE ? 0.0 : h.art_kind == OR_ART_DRAWER ? 0.0 : NAN;
      h.art_qmax = h.art_kind == OR_ART_FRIDGE ? 1.6 : h.art_kind == OR_ART_DRAWER ? 0.5 : NAN;
      nev = or_extract_events(recs, n, &h, J->th, ek, et, (int32_t)(4 * rcap), &d0);
      if (nev >= 0) mode = or_classify(J->kind, ek, nev, d0, 0, NULL, 0, &so, &se);
      J->records += n;
    }
    int64_t i = seed - J->base;
    if (J->mode_out) J->mode_out[i] = (uint8_t)(mode < 0 ? 255 : mode);
    if (J->nev_out) J->nev_out[i] = nev;
    if (J->nrec_out) J->nrec_out[i] = n;
    if (J->flags_out) J->flags_out[i] = (uint8_t)((mode >= 0 && so ? 1 : 0) | (mode >= 0 && se ? 2 : 0));
    if (J->d0_out) J->d0_out[i] = d0;
    if (J->ev_kind_out && nev > 0) {
      const int64_t m = nev < J->ev_stride ? nev : J->ev_stride;
      memcpy(J->ev_kind_out + i * J->ev_stride, ek, (size_t)m);
      memcpy(J->ev_t_out + i * J->ev_stride, et, sizeof(int32_t) * (size_t)m);
    }
  }
  free(sk);
  free(sg);
  free(recs);
  free(ek);
  free(et);
  return NULL;
}

int64_t or_fuzz_label_batch_ex(int64_t seed0, int64_t n, int32_t subtask,
                               const or_fuzz_cfg* cfg, const or_thresholds* th,
                               int32_t n_threads, uint8_t* mode_out,
                               int32_t* n_events_out, int64_t* n_records_out,
                               uint8_t* flags_out, double* d0_out, int64_t ev_stride,
                               uint8_t* ev_kind_out, int32_t* ev_t_out) {
  if (n_threads < 1) n_threads = 1;
  if (n_threads > 256) n_threads = 256;
  job_t jobs[256];
  pthread_t tid[256];
  for (int i = 0; i < n_threads; i++) {
    jobs[i].s0 = seed0 + n * i / n_threads;
    jobs[i].s1 = seed0 + n * (i + 1) / n_threads;
    jobs[i].kind = subtask;
    jobs[i].cfg = cfg;
    jobs[i].th = th;
    jobs[i].mode_out = mode_out;
    jobs[i].nev_out = n_events_out;
    jobs[i].nrec_out = n_records_out;
    jobs[i].flags_out = flags_out;
    jobs[i].d0_out = d0_out;
    jobs[i].ev_stride = ev_stride;
    jobs[i].ev_kind_out = ev_stride > 0 ? ev_kind_out : NULL;
    jobs[i].ev_t_out = ev_t_out;
    jobs[i].base = seed0;
    jobs[i].records = 0;
  }
  if (n_threads == 1) {
    fuzz_job(&jobs[0]);
  } else {
    for (int i = 0; i < n_threads; i++) pthread_create(&tid[i], NULL, fuzz_job, &jobs[i]);
    for (int i = 0; i < n_threads; i++) pthread_join(tid[i], NULL);
  }
  int64_t total = 0;
  for (int i = 0; i < n_threads; i++) total += jobs[i].records;
  return total;
}

int64_t or_fuzz_label_batch(int64_t seed0, int64_t n, int32_t subtask,
                            const or_fuzz_cfg* cfg, const or_thresholds* th,
                            int32_t n_threads, uint8_t* mode_out,
                            int32_t* n_events_out, int64_t* n_records_out) {
  return or_fuzz_label_batch_ex(seed0, n, subtask, cfg, th, n_threads, mode_out, n_events_out,
                                n_records_out, NULL, NULL, 0, NULL, NULL);
}
