// tl_env.cuh -- batched subtask environment: reset / step(actions) with
// online labelling, one thread per environment.
//
// Reference (paths under /root/reference/pkg/src/trajlab/):
//   synth.py:100-162  _Realizer.__init__           -> reset (+ the t = 0 _emit, :299)
//   synth.py:192-196  _advance_cum
//   synth.py:205-296  _apply                        -> step(action)
//   synth.py:166-190  _emit                         -> the step's observation
//   synth.py:298-310  run: every record t >= 1 is _advance_cum; [_apply]; _emit
//   events.py:94-193  edge events, folded online    -> step_mask
//   modes.py:235-253  classify                      -> tl_env_labels
//
// realize(script) is exactly reset + one step per record, the action being
// the script step's event on its event record and TL_ACT_HOLD elsewhere.
//
// State (one opaque device buffer, tl_env_state_bytes):
//   EnvHdr                  realize thresholds + the 12 label csets
//   EnvSt[n]                128 B per env: realizer scalars + label fold
//   uint32 mt[n][624]       CPython MT19937 state per env, regenerated
//                           lazily in place (word i of a block reads mt[i],
//                           mt[i+1] and mt[i+397] / mt[i-227], all written
//                           >= 227 words earlier), so a step's <= 2*(2dof+7)
//                           words have no intra-step dependencies: every
//                           load of a step is issued (global -> shared) before
//                           any store.  4096 envs = 10 MB of MT state: L2
//                           resident across steps.
// Observations are time-major: plane f of step k of env e at
// obs[f*obs_stride + k*n_env + e] (coalesced across the warp).
#pragma once
#include "tl_synth.cuh"

namespace tl {

constexpr int kEnvThreads = 64;

struct EnvHdr {
  tl_thresholds th;   // realize thresholds (synth.py:100)
  tl_cset cs[12];     // label csets [subtask*3 + art_kind]
  int32_t n_env, dof, pad[2];
};

struct __align__(16) EnvSt {
  double cum, force, dist, art;  // _Realizer scalars (f64)
  double d0, sc_d;               // label: Place d0 = records[0].dist, Close sc cut (f64)
  int32_t t;                     // index of the latest record (0 after reset)
  int32_t status;                // 0 or the InfeasibleScript code (env stops)
  int32_t err_t;                 // record index whose action raised
  int32_t mt_idx;                // next MT word of the current block
  int32_t size;                  // label fold: |E|
  int32_t last[7];               // label fold: last index per alphabet kind
  uint32_t prev_ind, err_any;
  float sc_ru;
  uint8_t subtask, art_kind, init_level, grasped, at_rest, level, err_act, active;
  int32_t pad[1];
};
static_assert(sizeof(EnvSt) == 128, "EnvSt is one 128-byte line");

__host__ __device__ inline size_t env_align(size_t x) { return (x + 255) & ~(size_t)255; }
__host__ __device__ inline size_t env_st_off() { return env_align(sizeof(EnvHdr)); }
__host__ __device__ inline size_t env_mt_off(int n) {
  return env_st_off() + env_align((size_t)n * sizeof(EnvSt));
}
__host__ __device__ inline size_t env_bytes(int n) {
  return env_mt_off(n) + env_align((size_t)n * kMtN * 4);
}

struct EnvParams {
  EnvHdr* hdr;
  // reset: header contents by value / source pointer (written into hdr by
  // the reset kernel itself, so a captured CUDA graph replays them)
  tl_thresholds th;
  const tl_cset* src_cs;
  EnvSt* st;
  uint32_t* mt;
  int32_t n_env;
  int32_t dof;
  // reset
  const tl_script* scripts;
  // step
  const uint8_t* actions;     // [k_steps][n_env]
  int32_t k_steps;
  // outputs (time-major)
  float* obs;
  int64_t obs_stride;
  uint8_t* obs_grasped;
  uint8_t* step_mask;         // [k_steps][n_env], may be null
  // labels
  tl_rules rules;
  tl_label* labels;
  int32_t* n_rec;
};

// Realize thresholds from the per-env script fields (synth.py:104-148).
__device__ __forceinline__ int env_rz(RzConst& z, const EnvSt& s, const tl_thresholds& th,
                                      int dof) {
  tl_script sc;
  sc.subtask = s.subtask;
  sc.art_kind = s.art_kind;
  sc.initial_level = s.init_level;
  sc.initial_grasped = 0;
  sc.initial_contact = 0;
  return realizer_init(z, sc, th, dof);
}

// Stage the raw MT words a step consumes: old[j] = mt[idx+j] (j <= nw) and
// src[j] = mt[idx+j+397 | idx+j-227] (j < nw), global -> registers ->
// shared.  Fully unrolled over the compile-time maximum (predicated), so
// all of a step's loads are in flight together (one L2 round trip).
template <int MAXW>
__device__ __forceinline__ void env_stage(const uint32_t* __restrict__ mt, int idx, int nw,
                                          uint32_t* __restrict__ so, uint32_t* __restrict__ ss) {
  uint32_t o[MAXW + 1], r[MAXW];
#pragma unroll
  for (int j = 0; j <= MAXW; j++) {
    int i = idx + j;
    i = i >= kMtN ? i - kMtN : i;
    if (j <= nw) o[j] = __ldcg(mt + i);
  }
#pragma unroll
  for (int j = 0; j < MAXW; j++) {
    int i = idx + j;
    i = i >= kMtN ? i - kMtN : i;
    if (j < nw) r[j] = __ldcg(mt + (i < kMtN - kMtM ? i + kMtM : i - (kMtN - kMtM)));
  }
#pragma unroll
  for (int j = 0; j <= MAXW; j++)
    if (j <= nw) so[j] = o[j];
#pragma unroll
  for (int j = 0; j < MAXW; j++)
    if (j < nw) ss[j] = r[j];
}

// Pipelined form: cp.async (global -> shared, no registers) of the full
// window a step can consume, [idx, idx + MAXW] and its MAXW sources
// ((i + 397) mod 624).  Issued for step k+1 as soon as step k's plan fixes
// idx' = idx + nw: the window never overlaps the words step k regenerates
// (they precede idx'; their sources lie >= 227 words behind), so the
// copies overlap step k's arithmetic.
// (cp_async4 / cp_async_commit / cp_async_wait: tl_common.cuh)

template <int MAXW>
__device__ __forceinline__ void env_stage_async(const uint32_t* __restrict__ mt, int idx,
                                                uint32_t* so, uint32_t* ss) {
  int i = idx;
#pragma unroll
  for (int j = 0; j <= MAXW; j++) {
    cp_async4(so + j, mt + i);
    i = i + 1 == kMtN ? 0 : i + 1;
  }
  i = idx + kMtM;
  i = i >= kMtN ? i - kMtN : i;
#pragma unroll
  for (int j = 0; j < MAXW; j++) {
    cp_async4(ss + j, mt + i);
    i = i + 1 == kMtN ? 0 : i + 1;
  }
  cp_async_commit();
}

// Regenerate staged words j, j+1 (in place in global memory) and return
// random() of their tempered outputs (Modules/_randommodule.c genrand,
// random_random).
__device__ __forceinline__ double env_rand(uint32_t* __restrict__ mt, int idx, int j,
                                           const uint32_t* so, const uint32_t* ss) {
  const uint32_t v0 = mt_mix(so[j], so[j + 1], ss[j]);
  const uint32_t v1 = mt_mix(so[j + 1], so[j + 2], ss[j + 1]);
  int i0 = idx + j, i1 = i0 + 1;
  i0 = i0 >= kMtN ? i0 - kMtN : i0;
  i1 = i1 >= kMtN ? i1 - kMtN : i1;
  __stcg(mt + i0, v0);
  __stcg(mt + i1, v1);
  return rand53(mt_temper(v0), mt_temper(v1));
}

// _emit (synth.py:166-190) + the record's indicator bits and edge events.
// Draw k of the emission goes to plane k (q_arm, qd_arm, q_tor, v_x, v_y,
// omega, dist_ee_rest: the draw order is the plane order).
template <int DOFMAX>
__device__ __forceinline__ void env_emit(const EnvParams& p, EnvSt& s, const RzConst& z,
                                         const tl_cset& c, uint32_t* __restrict__ mt, int idx,
                                         int j0, const uint32_t* so, const uint32_t* ss,
                                         int64_t col, uint32_t& ind, uint32_t& err) {
  const int dof = z.dof;
  const int64_t st = p.obs_stride;
  float* __restrict__ dst = p.obs + col;
  const bool emit = !s.at_rest;
  RecV<float> v;
  float mq = 0.f, mqd = 0.f;
  double md = 0.0;
#pragma unroll
  for (int i = 0; i < DOFMAX; i++) {
    if (i < dof) {
      const float q = emit ? __double2float_rn(TL_UNIFORM(-0.3, 0.3, env_rand(mt, idx, j0 + 2 * i, so, ss))) : 0.f;
      dst[(int64_t)i * st] = q;
      mq = i == 0 ? fabsf(q) : pymax_step(mq, fabsf(q));
      if (!c.rest_zero) {
        const double dv = fabs(__dsub_rn((double)q, c.rest_arm[i]));
        md = i == 0 ? dv : pymax_step(md, dv);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < DOFMAX; i++) {
    if (i < dof) {
      const float qd = emit ? __double2float_rn(TL_UNIFORM(-0.4, 0.4, env_rand(mt, idx, j0 + 2 * (dof + i), so, ss))) : 0.f;
      dst[(int64_t)(dof + i) * st] = qd;
      mqd = i == 0 ? fabsf(qd) : pymax_step(mqd, fabsf(qd));
    }
  }
  const int k2 = 2 * dof;
  auto draw = [&](int k, double a, double span) -> float {
    return emit ? __double2float_rn(uniform_span(a, span, env_rand(mt, idx, j0 + 2 * (k2 + k), so, ss))) : 0.f;
  };
  v.tor = draw(0, -0.05, 0.05 - -0.05);
  v.vx = draw(1, -0.2, 0.2 - -0.2);
  v.vy = draw(2, -0.2, 0.2 - -0.2);
  v.om = draw(3, -0.3, 0.3 - -0.3);
  v.der = draw(4, 0.2, 1.0 - 0.2);
  const float fnan = __int_as_float(0x7fc00000);
  v.dist = z.has_goal ? __double2float_rn(s.dist) : fnan;
  v.force = z.has_force ? __double2float_rn(s.force) : fnan;
  v.cum = __double2float_rn(s.cum);
  v.art = z.has_art ? __double2float_rn(s.art) : fnan;
  v.g = s.grasped != 0;
  v.jm = mq;
  v.qdm = mqd;
  v.jm_d = md;
  float* d2 = dst + (int64_t)k2 * st;
  d2[0] = v.tor;
  d2[st] = v.vx;
  d2[2 * st] = v.vy;
  d2[3 * st] = v.om;
  d2[4 * st] = v.der;
  d2[5 * st] = v.dist;
  d2[6 * st] = v.force;
  d2[7 * st] = v.cum;
  d2[8 * st] = v.art;
  if (p.obs_grasped) p.obs_grasped[col] = s.grasped;
  if (s.t == 0) {  // events.py:174-176: slightly-closed cut anchored at records[0]
    if (c.subtask == TL_CLOSE) close_cut(c, (double)v.art, s.sc_ru, s.sc_d);
    s.d0 = (double)v.dist;
  }
  record_bits(c, v, s.sc_ru, s.sc_d, ind, err);
}

// fold one record's event mask into the running label state
__device__ __forceinline__ void env_fold(EnvSt& s, uint32_t m, uint32_t err) {
#pragma unroll
  for (int k = 0; k < 7; k++)
    if ((m >> k) & 1u) s.last[k] = s.size + __popc(m & ((1u << k) - 1u));
  s.size += __popc(m);
  s.err_any |= err;
}

__device__ __forceinline__ void env_load(EnvSt& s, const EnvSt* src) {
  const uint4* a = reinterpret_cast<const uint4*>(src);
  uint4* b = reinterpret_cast<uint4*>(&s);
#pragma unroll
  for (int i = 0; i < 8; i++) b[i] = __ldcg(a + i);
}
__device__ __forceinline__ void env_store(EnvSt* dst, const EnvSt& s) {
  const uint4* a = reinterpret_cast<const uint4*>(&s);
  uint4* b = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int i = 0; i < 8; i++) __stcg(b + i, a[i]);
}

template <int DOFMAX>
struct EnvSmem {
  static constexpr int kWords = 2 * (2 + 2 * DOFMAX + 5);  // max words per step
  static constexpr int kBuf = 2 * kWords + 1;              // old[kWords+1] + src[kWords]
  static constexpr int kStride = 2 * kBuf + 1;             // two buffers; odd: conflict-free
  tl_cset cs[12];  // label csets, staged once per block (no reloads after stores)
  uint32_t buf[kEnvThreads * kStride];
};

template <int DOFMAX>
__device__ __forceinline__ void env_stage_csets(EnvSmem<DOFMAX>& sm, const tl_cset* cs) {
  const uint32_t* s = reinterpret_cast<const uint32_t*>(cs);
  uint32_t* d = reinterpret_cast<uint32_t*>(sm.cs);
  for (int i = threadIdx.x; i < (int)(sizeof(sm.cs) / 4); i += blockDim.x) d[i] = __ldg(s + i);
  __syncthreads();
}

// reset: _Realizer.__init__ + _emit at t = 0.  MT rows already seeded
// (k_seed_states / k_fuzz_reset).  Infeasible starts (synth.py:123/139/155)
// set status and emit nothing.
template <int DOFMAX>
__global__ void __launch_bounds__(kEnvThreads) k_env_reset(EnvParams p) {
  extern __shared__ __align__(16) unsigned char env_smem_raw[];
  EnvSmem<DOFMAX>& sm = *reinterpret_cast<EnvSmem<DOFMAX>*>(env_smem_raw);
  env_stage_csets(sm, p.src_cs);
  if (blockIdx.x == 0) {  // header for the step kernels
    if (threadIdx.x == 0) {
      p.hdr->th = p.th;
      p.hdr->n_env = p.n_env;
      p.hdr->dof = p.dof;
    }
    const uint32_t* src = reinterpret_cast<const uint32_t*>(sm.cs);
    uint32_t* dst = reinterpret_cast<uint32_t*>(p.hdr->cs);
    for (int i = threadIdx.x; i < (int)(sizeof(sm.cs) / 4); i += blockDim.x) dst[i] = src[i];
  }
  const int e = blockIdx.x * kEnvThreads + threadIdx.x;
  if (e >= p.n_env) return;
  const tl_script sc = p.scripts[e];
  EnvSt s;
  memset(&s, 0, sizeof(s));
  s.subtask = (uint8_t)sc.subtask;
  s.art_kind = (uint8_t)(sc.subtask >= TL_OPEN ? sc.art_kind : TL_ART_NONE);
  s.init_level = (uint8_t)sc.initial_level;
  for (int k = 0; k < 7; k++) s.last[k] = -1;
  s.err_t = -1;
  RzConst z;
  int code = sc.n_steps < 0 ? TL_ERR_SCRIPT_CAPACITY : env_rz(z, s, p.th, p.dof);
  if (!code && sc.subtask == TL_PICK && sc.initial_grasped && !sc.initial_contact)
    code = TL_INF_PICK_GRASPED_NO_CONTACT;                               // synth.py:154-155
  const bool art_ok = sc.art_kind >= 0 && sc.art_kind <= 2;
  const int ci = sc.subtask * 3 + (s.art_kind <= 2 ? s.art_kind : 0);
  if (code) {
    s.status = code;
    s.err_t = 0;
    env_store(&p.st[e], s);
    if (p.step_mask) p.step_mask[e] = 0;
    return;
  }
  (void)art_ok;
  s.grasped = (uint8_t)(sc.initial_grasped != 0);
  s.force = (z.has_force && sc.initial_contact) ? 1.2 : 0.0;
  s.dist = z.has_goal ? sc.initial_dist_obj_goal : __longlong_as_double(0x7ff8000000000000ll);
  s.cum = 0.0;
  s.at_rest = 0;
  s.active = 1;
  if (z.has_art) {
    if (z.kind == TL_OPEN) {
      s.level = (uint8_t)sc.initial_level;
      s.art = sc.initial_level == TL_LVL_LOW ? z.lv_low
              : sc.initial_level == TL_LVL_SLIGHT ? z.lv_slight : z.lv_open;
    } else {
      s.level = sc.initial_level == TL_LVL_CLOSED ? TL_LVL_CLOSED : TL_LVL_OPEN;
      s.art = z.a_q0;
    }
  } else {
    s.art = __longlong_as_double(0x7ff8000000000000ll);
  }
  const tl_cset& c = sm.cs[ci];
  uint32_t* mt = p.mt + (size_t)e * kMtN;
  uint32_t* so = sm.buf + threadIdx.x * EnvSmem<DOFMAX>::kStride;
  uint32_t* ss = so + EnvSmem<DOFMAX>::kWords + 1;
  const int nw = 2 * z.ne;
  env_stage<EnvSmem<DOFMAX>::kWords>(mt, 0, nw, so, ss);
  uint32_t ind, err;
  env_emit<DOFMAX>(p, s, z, c, mt, 0, 0, so, ss, e, ind, err);
  s.mt_idx = nw;
  s.prev_ind = ind;
  s.err_any = err;
  if (p.step_mask) p.step_mask[e] = 0;
  env_store(&p.st[e], s);
}

// step: k_steps records per env (actions[k][e]): _advance_cum, _apply, _emit.
// LPE lanes (4 or 8) share one env: the plan is computed redundantly by the
// group, the MT window copies, the draws and the plane stores are split LPE
// ways (draw d -> lane d % LPE: the pre-draws of cum / dist are draws
// 0..pre-1, plane k is draw pre + k), and lane 0 gathers the record for the
// label fold.
constexpr int kEnvQThreads = 128;             // 128 / LPE envs per block

template <int DOFMAX, int LPE>
struct EnvQSmem {
  static constexpr int kEnvs = kEnvQThreads / LPE;
  static constexpr int kWords = 2 * (2 + 2 * DOFMAX + 5);  // max words per step
  static constexpr int kBuf = 2 * kWords + 1;              // old[kWords+1] + src[kWords]
  static constexpr int kStride = 2 * kBuf + 1;             // two buffers per env; odd
  tl_cset cs[12];
  uint32_t buf[kEnvs * kStride];
};

// lane q of the env's lane group copies words j = q, q+LPE, ... of the window
template <int MAXW, int LPE>
__device__ __forceinline__ void env_stage_async_q(const uint32_t* __restrict__ mt, int idx,
                                                  uint32_t* so, uint32_t* ss, int q) {
#pragma unroll
  for (int j0 = 0; j0 <= MAXW; j0 += LPE) {
    const int j = j0 + q;
    if (j <= MAXW) {
      int i = idx + j;
      i = i >= kMtN ? i - kMtN : i;
      cp_async4(so + j, mt + i);
    }
  }
#pragma unroll
  for (int j0 = 0; j0 < MAXW; j0 += LPE) {
    const int j = j0 + q;
    if (j < MAXW) {
      int i = idx + j + kMtM;
      i = i >= kMtN ? i - kMtN : i;
      i = i >= kMtN ? i - kMtN : i;
      cp_async4(ss + j, mt + i);
    }
  }
  cp_async_commit();
}

// STAGED: the 12 label csets are staged into shared memory once per block
// (multi-step launches); single-step launches read the env's cset through L1
// at use instead -- the staging round trip and block barrier were ~0.8 us of
// a ~5.6 us single-step launch (scripts/ab_env_api.sh)
template <int DOFMAX, int LPE, bool STAGED>
__global__ void __launch_bounds__(kEnvQThreads) k_env_step(EnvParams p) {
  using SM = EnvQSmem<DOFMAX, LPE>;
  constexpr int kQuad = LPE;  // lanes per env (4 or 8)
  extern __shared__ __align__(16) unsigned char env_smem_raw[];
  SM& sm = *reinterpret_cast<SM*>(env_smem_raw);
  if (STAGED) {
    const uint32_t* src = reinterpret_cast<const uint32_t*>(p.hdr->cs);
    uint32_t* d = reinterpret_cast<uint32_t*>(sm.cs);
    for (int i = threadIdx.x; i < (int)(sizeof(sm.cs) / 4); i += blockDim.x) d[i] = __ldg(src + i);
    __syncthreads();
  }
  const int q = threadIdx.x & (kQuad - 1);
  const int le = threadIdx.x / kQuad;
  const int e = blockIdx.x * SM::kEnvs + le;
  const int qbase = lane_id() & ~(kQuad - 1);
  const unsigned qmask = ((1u << kQuad) - 1u) << qbase;
  if (e >= p.n_env) return;  // whole quads leave together
  EnvSt s;
  env_load(s, &p.st[e]);
  const int n = p.n_env;
  if (s.status || !s.active) {
    if (p.step_mask)
      for (int k = q; k < p.k_steps; k += kQuad) p.step_mask[(int64_t)k * n + e] = 0;
    return;
  }
  RzConst z;
  env_rz(z, s, p.hdr->th, p.dof);
  const tl_cset& c = STAGED ? sm.cs[s.subtask * 3 + s.art_kind]
                            : p.hdr->cs[s.subtask * 3 + s.art_kind];  // L1-cached reads at use
  uint32_t* mt = p.mt + (size_t)e * kMtN;
  uint32_t* row = sm.buf + le * SM::kStride;
  const int dof = z.dof, ne = z.ne;
  const int64_t st = p.obs_stride;
  const float fnan = __int_as_float(0x7fc00000);
  int cur = 0;  // buffer holding the window at s.mt_idx
  env_stage_async_q<SM::kWords, LPE>(mt, s.mt_idx, row, row + SM::kWords + 1, q);
  int a_next = p.actions[e];
  for (int k = 0; k < p.k_steps; k++) {
    const int64_t col = (int64_t)k * n + e;
    const bool stamp = e == 0 && q == 0 && k == 5;  // profiling build only
    if (stamp) TL_STAMP(100);
    const int a = a_next;
    if (k + 1 < p.k_steps) a_next = p.actions[col + n];  // prefetch
    if (a == TL_ACT_IDLE || s.status) {
      if (q == 0 && p.step_mask) p.step_mask[col] = 0;
      continue;
    }
    if (a == TL_ACT_BAD_GAP) {  // run(): "event gap must be >= 1" (synth.py:301-302)
      s.status = TL_INF_GAP;
      s.err_t = s.t + 1;
      s.err_act = (uint8_t)a;
      if (q == 0 && p.step_mask) p.step_mask[col] = 0;
      continue;
    }
    // draw plan: known before any draw (synth.py:192-196, :205-296)
    const double head = __dsub_rn(z.L09, s.cum);
    const int adv = head > 0.0;
    int code = 0, app = 0;
    // _apply's checks (state after _advance_cum: only cum > limit reads cum,
    // and advance never crosses 0.9*limit, so the pre-advance cum decides)
    if (a != TL_ACT_HOLD) {
      PlanSt ps;
      ps.force = s.force;
      ps.art = s.art;
      ps.grasped = s.grasped;
      ps.at_rest = s.at_rest;
      ps.exc = s.cum > z.limit;
      ps.level = s.level;
      code = a > TL_EV_EXCESSIVE_COLLISIONS ? TL_INF_NOT_IN_ALPHABET : plan_apply(z, ps, a, app);
      if (!code && z.has_goal) {  // value-dependent checks (synth.py:218-260)
        const bool in = s.dist <= z.goal;
        if (a == TL_EV_OBJ_AT_GOAL && in) code = TL_INF_AT_GOAL_ALREADY;
        else if (a == TL_EV_OBJ_LEFT_GOAL && !in) code = TL_INF_LEFT_NOT_AT_GOAL;
        else if (a == TL_EV_RELEASED_AT_GOAL && !in) code = TL_INF_RAG;
        else if (a == TL_EV_RELEASED_OUTSIDE_GOAL && in) code = TL_INF_ROG;
        else if (a == TL_EV_SUCCESS && !in) code = TL_INF_SUCCESS_UNREACHABLE;
      }
      if (code) {
        s.status = code;
        s.err_t = s.t + 1;
        s.err_act = (uint8_t)a;
        if (q == 0 && p.step_mask) p.step_mask[col] = 0;
        continue;
      }
      s.force = ps.force;
      s.art = ps.art;
      s.grasped = (uint8_t)ps.grasped;
      s.at_rest = (uint8_t)ps.at_rest;
      s.level = (uint8_t)ps.level;
    }
    if (stamp) TL_STAMP(101);
    const bool emit = !s.at_rest;
    const int pre = adv + app;
    const int nw = 2 * (pre + (emit ? ne : 0));
    const int idx = s.mt_idx;
    const int ni = idx + nw;
    s.mt_idx = ni >= kMtN ? ni - kMtN : ni;
    const uint32_t* so = row + cur * SM::kBuf;
    const uint32_t* ss = so + SM::kWords + 1;
    {  // next step's window into the other buffer; this one complete quad-wide
      uint32_t* no = row + (cur ^ 1) * SM::kBuf;
      env_stage_async_q<SM::kWords, LPE>(mt, s.mt_idx, no, no + SM::kWords + 1, q);
      cp_async_wait<1>();
      __syncwarp(qmask);
      cur ^= 1;
    }
    if (stamp) TL_STAMP(102);
    // this lane's draws: d = q, q + 4, ... over pre-draws then planes
    double r_pre = 0.0;
    float mq = 0.f, mqd = 0.f, sc5[5] = {0.f, 0.f, 0.f, 0.f, 0.f};
    double md = 0.0;
    const int nd = pre + ne;
    // unrolled to the compile-time maximum so the independent draws of a
    // lane interleave (the loop-carried form serialised ~470 cycles each)
    constexpr int kMaxIt = (2 + 2 * DOFMAX + 5 + kQuad - 1) / kQuad;
#pragma unroll
    for (int it = 0; it < kMaxIt; it++) {
      const int d = q + it * kQuad;
      if (d >= nd) continue;
      const bool draw = d < pre || emit;
      const double r = draw ? env_rand(mt, idx, 2 * d, so, ss) : 0.0;
      if (d < pre) {
        r_pre = r;  // lane 0: cum (or dist), lane 1: dist
        continue;
      }
      const int kf = d - pre;  // plane
      double lo, span;  // rng.uniform bounds of plane kf, b - a folded at compile time
      if (kf < dof) { lo = -0.3; span = 0.3 - -0.3; }
      else if (kf < 2 * dof) { lo = -0.4; span = 0.4 - -0.4; }
      else {
        const int j = kf - 2 * dof;
        lo = j == 0 ? -0.05 : j == 3 ? -0.3 : j == 4 ? 0.2 : -0.2;
        span = j == 0 ? 0.05 - -0.05 : j == 3 ? 0.3 - -0.3 : j == 4 ? 1.0 - 0.2 : 0.2 - -0.2;
      }
      const float v = emit ? __double2float_rn(uniform_span(lo, span, r)) : 0.f;
      p.obs[(int64_t)kf * st + col] = v;
      if (kf < dof) {
        mq = fmaxf(mq, fabsf(v));  // generated values are never NaN: max is order-free
        if (!c.rest_zero) md = fmax(md, fabs(__dsub_rn((double)v, c.rest_arm[kf])));
      } else if (kf < 2 * dof) {
        mqd = fmaxf(mqd, fabsf(v));
      } else {
        const int j = kf - 2 * dof;
        sc5[0] = j == 0 ? v : sc5[0];
        sc5[1] = j == 1 ? v : sc5[1];
        sc5[2] = j == 2 ? v : sc5[2];
        sc5[3] = j == 3 ? v : sc5[3];
        sc5[4] = j == 4 ? v : sc5[4];
      }
    }
    if (stamp) TL_STAMP(103);
    // cum / dist from the pre-draws (lanes 0 and adv), identical on all lanes
    if (adv) {
      const double rc = __shfl_sync(qmask, r_pre, qbase);
      s.cum = __dadd_rn(s.cum, __dmul_rn(__dmul_rn(head, 0.05), rc));
    }
    if (a == TL_EV_EXCESSIVE_COLLISIONS) s.cum = z.L105;                 // synth.py:210-213
    if (app) {
      const double rd = __shfl_sync(qmask, r_pre, qbase + adv);
      s.dist = a == TL_EV_OBJ_AT_GOAL ? TL_UNIFORM(0.02, 0.12, rd) : TL_UNIFORM(0.3, 0.8, rd);
    }
    s.t += 1;
    const float vdist = z.has_goal ? __double2float_rn(s.dist) : fnan;
    const float vforce = z.has_force ? __double2float_rn(s.force) : fnan;
    const float vcum = __double2float_rn(s.cum);
    const float vart = z.has_art ? __double2float_rn(s.art) : fnan;
    if (q < 4) {
      const int f = 2 * dof + 5 + q;  // dist, force, cum, art: one plane per lane
      p.obs[(int64_t)f * st + col] = q == 0 ? vdist : q == 1 ? vforce : q == 2 ? vcum : vart;
    }
    if (stamp) TL_STAMP(104);
    // gather the record's predicate inputs on lane 0
#pragma unroll
    for (int x = 1; x < kQuad; x <<= 1) {
      mq = fmaxf(mq, __shfl_xor_sync(qmask, mq, x));
      mqd = fmaxf(mqd, __shfl_xor_sync(qmask, mqd, x));
    }
    if (!c.rest_zero) {
#pragma unroll
      for (int x = 1; x < kQuad; x <<= 1) md = fmax(md, __shfl_xor_sync(qmask, md, x));
    }
    float sv[5];
#pragma unroll
    for (int j = 0; j < 5; j++)
      sv[j] = __shfl_sync(qmask, sc5[j], qbase + ((pre + 2 * dof + j) & (kQuad - 1)));
    if (stamp) TL_STAMP(105);
    if (q == 0) {
      if (p.obs_grasped) p.obs_grasped[col] = s.grasped;
      RecV<float> v;
      v.tor = sv[0]; v.vx = sv[1]; v.vy = sv[2]; v.om = sv[3]; v.der = sv[4];
      v.dist = vdist; v.force = vforce; v.cum = vcum; v.art = vart;
      v.g = s.grasped != 0;
      v.jm = mq; v.qdm = mqd; v.jm_d = md;
      uint32_t ind, err;
      record_bits(c, v, s.sc_ru, s.sc_d, ind, err);
      const uint32_t m = edge_mask(c.subtask, s.prev_ind, ind);
      env_fold(s, m, err);
      s.prev_ind = ind;
      if (p.step_mask) p.step_mask[col] = (uint8_t)m;
    }
    if (stamp) TL_STAMP(106);
  }
  cp_async_wait<0>();
  if (q == 0) env_store(&p.st[e], s);
}

// labels of the episodes so far (classify(extract_events(records[0..t])))
__global__ void k_env_labels(EnvParams p) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= p.n_env) return;
  EnvSt s;
  env_load(s, &p.st[e]);
  tl_label L;
  const int ci = s.subtask * 3 + (s.art_kind <= 2 ? s.art_kind : 0);
  if (s.status) {
    L.status = s.status;
    L.n_events = 0;
    L.err_index = s.err_t;
    L.subtask = s.subtask;
    L.mode = 255;
    L.flags = 0;
    L.pad = s.err_act;
    L.d0 = __longlong_as_double(0x7ff8000000000000ll);
  } else if (s.t < 1) {  // events.py:96-97
    L.status = TL_ERR_TOO_SHORT;
    L.n_events = 0;
    L.err_index = -1;
    L.subtask = s.subtask;
    L.mode = 255;
    L.flags = 0;
    L.pad = 0;
    L.d0 = __longlong_as_double(0x7ff8000000000000ll);
  } else {
    LState S;
    S.size = s.size;
#pragma unroll
    for (int k = 0; k < 7; k++) S.last[k] = s.last[k];
    S.prev_ind = s.prev_ind;
    S.err_any = s.err_any;
    L = make_label(p.hdr->cs[ci], S, s.d0, p.rules);
  }
  p.labels[e] = L;
  if (p.n_rec) p.n_rec[e] = s.status ? 0 : s.t + 1;
}

// script -> per-step actions (synth.py:298-310): record t >= 1 of env e
// gets the event of the script step whose event record it is, TL_ACT_HOLD
// on hold records up to the script's record count, TL_ACT_IDLE after it.
// A step with gap < 1 turns the record where run() raises into
// TL_ACT_BAD_GAP.  actions[k][e] is record t = t0 + k.
__global__ void k_env_script_actions(const tl_script* __restrict__ scripts,
                                     const uint8_t* __restrict__ step_kind,
                                     const int32_t* __restrict__ step_gap, int n_env, int t0,
                                     int k_steps, uint8_t* __restrict__ actions) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n_env) return;
  const tl_script sc = scripts[e];
  const int ns = sc.n_steps < 0 ? 0 : sc.n_steps;
  const int32_t* gap = step_gap + sc.step_off;
  int64_t nrec = 1;
  bool bad = false;
  for (int i = 0; i < ns; i++) {
    bad |= gap[i] < 1;
    nrec += gap[i];
  }
  const int tmin = ns ? 0 : 1;
  nrec += sc.tail > tmin ? sc.tail : tmin;
  if (nrec < 2) nrec = 2;
  int si = 0;
  int64_t tau_prev = 0;  // event record of step si - 1 (0 = the reset record)
  for (int k = 0; k < k_steps; k++) {
    const int64_t t = (int64_t)t0 + k;
    while (si < ns && gap[si] >= 1 && tau_prev + gap[si] < t) tau_prev += gap[si++];
    uint8_t a;
    if (sc.n_steps < 0 || t < 1) a = TL_ACT_IDLE;
    else if (si < ns && gap[si] < 1) a = t == tau_prev + 1 ? TL_ACT_BAD_GAP : TL_ACT_IDLE;
    else if (si < ns && tau_prev + gap[si] == t) a = step_kind[sc.step_off + si];
    else a = (bad || t < nrec) ? TL_ACT_HOLD : TL_ACT_IDLE;  // bad: holds before the raise
    actions[(int64_t)k * n_env + e] = a;
  }
}

}  // namespace tl
