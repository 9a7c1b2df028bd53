// trajlab_b200.cu -- C ABI of libtrajlab_b200.so (see include/trajlab_b200.h).
// Single translation unit: kernels live in the tl_*.cuh headers.
#include <algorithm>
#include <dlfcn.h>
#include <nccl.h>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "tl_common.cuh"
#include "tl_label.cuh"
#ifdef TL_AB
#include "tl_label_tma.cuh"  // A/B probe build only (slower TMA-staged labeller)
#endif
#include "tl_synth.cuh"
#include "tl_synth_warp.cuh"
#ifdef TL_AB
#include "tl_synth_cta.cuh"  // A/B probe build only (one CTA per episode)
#endif
#include "tl_filter.cuh"
#include "tl_env.cuh"
#include "tl_analytics.cuh"
#include "tl_validate.cuh"

namespace {

using namespace tl;

cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int check_launch() {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "trajlab_b200: CUDA error: %s\n", cudaGetErrorString(e));
    return TL_E_CUDA;
  }
  return TL_OK;
}

int sm_count() {
  int dev = 0, n = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

// default rule tables = MODE_RULES (modes.py:208-213): success rules then
// failure rules of each subtask, in declaration order
tl_rules default_rules() {
  static const int base[4] = {0, 9, 21, 30}, ns[4] = {4, 5, 3, 3}, nm[4] = {9, 12, 9, 9};
  tl_rules r;
  memset(&r, 0, sizeof(r));
  for (int s = 0; s < 4; s++) {
    r.count[s][0] = (int8_t)ns[s];
    for (int i = 0; i < ns[s]; i++) r.ids[s][0][i] = (int8_t)(base[s] + i);
    r.count[s][1] = (int8_t)(nm[s] - ns[s]);
    for (int i = ns[s]; i < nm[s]; i++) r.ids[s][1][i - ns[s]] = (int8_t)(base[s] + i);
  }
  return r;
}

tl_rules rules_or_default(const tl_rules* r) { return r ? *r : default_rules(); }

// largest float <= x / smallest float >= x (x finite or inf; NaN stays NaN)
float rd_f32(double x) {
  float f = (float)x;
  if (std::isnan(x)) return f;
  if ((double)f > x) f = std::nextafter(f, -INFINITY);
  return f;
}
float ru_f32(double x) {
  float f = (float)x;
  if (std::isnan(x)) return f;
  if ((double)f < x) f = std::nextafter(f, INFINITY);
  return f;
}

template <class F>
void set_max_smem(F* k, int bytes) {
  static std::mutex mu;
  std::lock_guard<std::mutex> g(mu);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

// Launch-shape overrides exist only in the A/B probe build (-DTL_AB,
// scripts/*_ab.sh); the product library has one code path per config.
#ifdef TL_AB
const char* ab_env(const char* name) { return getenv(name); }
#else
constexpr const char* ab_env(const char*) { return nullptr; }
#endif

int blocks_for(int n_items, int per_block, int max_blocks) {
  int b = (n_items + per_block - 1) / per_block;
  if (b > max_blocks) b = max_blocks;
  return b < 1 ? 1 : b;
}

}  // namespace

// ---- the one exchange step over NCCL helpers ------------------
// NCCL is resolved at call time from the process (the library that created
// the caller's communicator, e.g. torch's bundled copy), never linked, so
// libtrajlab_b200.so loads without NCCL and cannot pull in a second copy.
namespace {
using AllGatherFn = ncclResult_t (*)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                                     cudaStream_t);
using AllReduceFn = ncclResult_t (*)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
                                     ncclComm_t, cudaStream_t);
template <class F>
F nccl_sym(const char* name) {
  void* f = dlsym(RTLD_DEFAULT, name);
  if (!f) {
    static void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // an already-loaded NCCL
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h) f = dlsym(h, name);
  }
  return reinterpret_cast<F>(f);
}
}  // namespace


extern "C" {

int tl_abi_version(void) { return TL_ABI_VERSION; }

int tl_device_sm_count(void) { return sm_count(); }

const char* tl_status_name(int code) {
  switch (code) {
    case TL_OK: return "OK";
    case TL_ERR_TOO_SHORT: return "TooShort";
    case TL_ERR_NAN_SUCCESS_DIST: case TL_ERR_NAN_ART: case TL_ERR_NAN_FORCE:
    case TL_ERR_NAN_PLACE_DIST: return "RequiredFieldNaN";
    case TL_ERR_MISSING_ART: return "MissingArticulation";
    case TL_ERR_MODE_COVERAGE: return "ModeCoverageError";
    case TL_ERR_D0_NONE_LE: case TL_ERR_D0_NONE_GT: return "TypeError";
    case TL_ERR_SCRIPT_CAPACITY: return "ScriptCapacity";
    case TL_E_INVALID: return "InvalidArgument";
    case TL_E_CUDA: return "CudaError";
    case TL_E_CAPACITY: return "Capacity";
    default:
      if (code >= TL_INF_PICK_GRASPED_NO_CONTACT && code <= TL_INF_INIT_LEVEL) return "InfeasibleScript";
      return "Unknown";
  }
}

// TrajectoryHeader + Thresholds -> cset (predicates.py:43-94 thresholds,
// thresholds.py:44-60 lookups).  All f64 arithmetic in the reference order.
int tl_cset_build(int32_t subtask, int32_t art_kind, double art_qmin, double art_qmax,
                  int32_t arm_dof, const double* rest_arm, double rest_tor,
                  const tl_thresholds* th, tl_cset* out) {
  if (!th || !out || subtask < 0 || subtask > 3 || arm_dof < 1 || arm_dof > TL_MAX_DOF ||
      art_kind < 0 || art_kind > 2)
    return TL_E_INVALID;
  tl_cset c;
  memset(&c, 0, sizeof(c));
  c.subtask = subtask;
  c.art_kind = art_kind;
  c.dof = arm_dof;
  int zero = rest_tor == 0.0;
  for (int i = 0; i < arm_dof; i++) {
    c.rest_arm[i] = rest_arm ? rest_arm[i] : 0.0;
    if (c.rest_arm[i] != 0.0) zero = 0;
  }
  c.rest_zero = zero;
  c.rest_tor = rest_tor;
  const double limit = subtask == TL_PICK ? th->coll_pick : subtask == TL_PLACE ? th->coll_place : th->coll_artic;
  const double span = art_qmax - art_qmin;  // (qmax - qmin)
  const double ofrac = art_kind == TL_ART_FRIDGE ? th->open_frac_fridge : th->open_frac_drawer;
  volatile double t;  // keep each product rounded before the add (no FMA)
  t = ofrac * span;
  c.open_cut = t + art_qmin;
  t = th->close_frac * span;
  c.closed_cut = t + art_qmin;
  t = th->slightly_open_frac * span;
  c.slight_open_cut = t + art_qmin;
  t = th->slightly_close_frac * span;
  c.scf_span = t;
  c.rest_radius = th->rest_radius;
  c.goal_radius = th->goal_radius;
  c.static_qd = th->static_qd_arm;
  c.static_v = th->static_v_base;
  c.static_om = th->static_omega;
  c.limit = limit;
  c.contact_eps = th->contact_eps;
  c.j_arm = subtask == TL_PICK ? th->j_arm_pick : th->j_arm_other;
  c.j_tor = th->j_tor_max;
  c.rd_rest_radius = rd_f32(c.rest_radius);
  c.rd_goal = rd_f32(c.goal_radius);
  c.rd_static_qd = rd_f32(c.static_qd);
  c.rd_static_v = rd_f32(c.static_v);
  c.rd_static_om = rd_f32(c.static_om);
  c.rd_limit = rd_f32(limit);
  c.rd_contact = rd_f32(c.contact_eps);
  c.ru_open = ru_f32(c.open_cut);
  c.rd_closed = rd_f32(c.closed_cut);
  c.ru_slight_open = ru_f32(c.slight_open_cut);
  c.rd_j_arm = rd_f32(c.j_arm);
  c.rd_j_tor = rd_f32(c.j_tor);
  *out = c;
  return TL_OK;
}

int tl_label_records(const tl_records* recs, int32_t n_env, const int32_t* env_cset,
                     const tl_cset* csets, int32_t n_cset, const tl_rules* rules,
                     uint8_t* step_mask, uint8_t* step_success, tl_label* labels,
                     void* stream) {
  if (!recs || !labels || !env_cset || !csets || n_env < 0 || n_cset < 1 || recs->dof < 1 ||
      recs->dof > TL_MAX_DOF || (recs->dtype != 0 && recs->dtype != 1))
    return TL_E_INVALID;
  if (n_env == 0) return TL_OK;
  const tl_rules r = rules_or_default(rules);
  // 128 blocks (of 8 warps) per SM, grid-stride beyond: each warp labels ~7
  // episodes of a 2^20-episode batch, and the episodes in flight stay close
  // in memory (measured: 16/SM 84 %, 128/SM 89 %, one block per 8 episodes 78 %
  // of HBM on the Pick sizing run)
  const char* gm = ab_env("TL_LABEL_GRID_PER_SM");
  const int grid = blocks_for(n_env, kLabelWarps, sm_count() * (gm ? std::max(1, atoi(gm)) : 128));
  const dim3 blk(kLabelWarps * 32);
  const bool small = recs->dof <= 7;
  const int vgen = ab_env("TL_LABEL_V4GEN") != nullptr;  // A/B: runtime-dof vec4 body
#ifdef TL_AB
  // TL_LABEL_TMA=1: the shared-memory (TMA bulk copy) staged variant, slower
  // than the register path + L2 bulk prefetch (profiles/r1_ncu_summary.md)
  if (recs->dtype == 0 && ab_env("TL_LABEL_TMA")) {
    if (small) {
      using SM7 = LabelTmaSmem<7>;
      set_max_smem(k_label_tma<7>, (int)sizeof(SM7));
      k_label_tma<7><<<blocks_for(n_env, SM7::kWarps, sm_count()), SM7::kWarps * 32, sizeof(SM7),
                       S(stream)>>>(*recs, n_env, env_cset, csets, r, step_mask, step_success,
                                    labels);
    } else {
      using SM16 = LabelTmaSmem<16>;
      set_max_smem(k_label_tma<16>, (int)sizeof(SM16));
      k_label_tma<16><<<blocks_for(n_env, SM16::kWarps, sm_count()), SM16::kWarps * 32,
                        sizeof(SM16), S(stream)>>>(*recs, n_env, env_cset, csets, r, step_mask,
                                                   step_success, labels);
    }
    return check_launch();
  }
#endif
  if (recs->dtype == 0) {
    if (small) {  // vector-body episodes, then everything else (k_label PART 1 / 2)
      k_label<float, 7, 1><<<grid, blk, 0, S(stream)>>>(*recs, n_env, env_cset, csets, r, step_mask, step_success, labels, vgen);
      k_label<float, 7, 2><<<grid, blk, 0, S(stream)>>>(*recs, n_env, env_cset, csets, r, step_mask, step_success, labels, vgen);
    } else {
      k_label<float, 16, 0><<<grid, blk, 0, S(stream)>>>(*recs, n_env, env_cset, csets, r, step_mask, step_success, labels, vgen);
    }
  } else {
    if (small) k_label<double, 7, 0><<<grid, blk, 0, S(stream)>>>(*recs, n_env, env_cset, csets, r, step_mask, step_success, labels, vgen);
    else k_label<double, 16, 0><<<grid, blk, 0, S(stream)>>>(*recs, n_env, env_cset, csets, r, step_mask, step_success, labels, vgen);
  }
  return check_launch();
}

size_t tl_scan_scratch_bytes(int32_t n) {
  const size_t tiles = ((size_t)(n > 0 ? n : 1) + kScanBlock - 1) / kScanBlock;
  const size_t tiles32 = ((size_t)(n > 0 ? n : 1) + 31) / 32 + 1;
  return (tiles > tiles32 ? tiles : tiles32) * sizeof(int64_t);
}

int tl_scan_emit_events(const uint8_t* step_mask, const int64_t* rec_start, const int32_t* n_rec,
                        const tl_label* labels, int32_t n_env, int64_t* ev_off, uint8_t* ev_kind,
                        int32_t* ev_t, void* scratch, void* stream) {
  if (!ev_off || n_env < 0 || (n_env > 0 && (!step_mask || !rec_start || !n_rec || !labels ||
                                             !ev_kind || !ev_t || !scratch)))
    return TL_E_INVALID;
  if (n_env == 0) {
    cudaMemsetAsync(ev_off, 0, sizeof(int64_t), S(stream));
    return check_launch();
  }
  const int tiles = (n_env + 31) / 32;
  cudaMemsetAsync(scratch, 0, (size_t)(tiles + 1) * sizeof(unsigned long long), S(stream));
  k_scan_emit<<<tiles, 1024, 0, S(stream)>>>(step_mask, rec_start, n_rec, labels, n_env, ev_off,
                                              ev_kind, ev_t,
                                              reinterpret_cast<unsigned long long*>(scratch));
  return check_launch();
}

int tl_scan_events(const tl_label* labels, int32_t n, int64_t* ev_off, void* scratch, void* stream) {
  if (!ev_off || n < 0 || (n > 0 && (!labels || !scratch))) return TL_E_INVALID;
  if (n == 0) {
    cudaMemsetAsync(ev_off, 0, sizeof(int64_t), S(stream));
    return check_launch();
  }
  const int tiles = (n + kScanBlock - 1) / kScanBlock;
  int64_t* tile = reinterpret_cast<int64_t*>(scratch);
  k_scan_tiles<<<tiles, kScanBlock, 0, S(stream)>>>(labels, n, ev_off, tile);
  k_scan_sums<<<1, kScanBlock, 0, S(stream)>>>(tile, tiles, ev_off, n);
  k_scan_add<<<(n + 255) / 256, 256, 0, S(stream)>>>(ev_off, tile, n);
  return check_launch();
}

int tl_emit_events(const uint8_t* step_mask, const int64_t* rec_start, const int32_t* n_rec,
                   const tl_label* labels, const int64_t* ev_off, int32_t n_env, uint8_t* ev_kind,
                   int32_t* ev_t, void* stream) {
  if (n_env < 0 || (n_env > 0 && (!step_mask || !rec_start || !n_rec || !labels || !ev_off ||
                                  !ev_kind || !ev_t)))
    return TL_E_INVALID;
  if (n_env == 0) return TL_OK;
  const int grid = blocks_for(n_env, kEmitWarps, sm_count() * 128);  // as k_label
  k_emit<<<grid, kEmitWarps * 32, 0, S(stream)>>>(step_mask, rec_start, n_rec, labels, ev_off, n_env, ev_kind, ev_t);
  return check_launch();
}

int tl_classify_events(const uint8_t* ev_kind, const int64_t* ev_off, const uint8_t* subtask,
                       const double* d0, const uint8_t* d0_none, int32_t n, const tl_rules* rules,
                       tl_label* out, void* stream) {
  if (n < 0 || (n > 0 && (!ev_off || !subtask || !out))) return TL_E_INVALID;
  if (n == 0) return TL_OK;
  const tl_rules r = rules_or_default(rules);
  k_classify_events<<<(n + 127) / 128, 128, 0, S(stream)>>>(ev_kind, ev_off, subtask, d0, d0_none, n, r, out);
  return check_launch();
}

// fuzz reset shape by batch size: the seeding chains are latency-bound and
// more warps contend for issue, while the sampler is branchy code that
// diverges across the episodes of a warp (measured: scripts/reset_epw_ab*.sh,
// scripts/ab_env.sh; the A/B build keeps the other shapes behind env knobs)
static void launch_fuzz_reset(SynthParams& sp, void* stream) {
  const int n = sp.n_env, sms = sm_count();
#ifdef TL_AB
  // TL_RESET_W=8|16: the warp-per-sampler form (k_fuzz_reset_w), measured
  // 1-2% slower on the headline step than the lane-per-sampler kernel below
  const char* fw = ab_env("TL_RESET_W");
  const int wform = fw ? atoi(fw) : 0;
  if (wform == 8) {
    k_fuzz_reset_w<8><<<(n + 7) / 8, 8 * 32, 8 * (kRowWords + kMtN) * 4, S(stream)>>>(sp);
    return;
  }
  if (wform == 16) {
    set_max_smem(k_fuzz_reset_w<16>, 16 * (kRowWords + kMtN) * 4);
    k_fuzz_reset_w<16><<<(n + 15) / 16, 16 * 32, 16 * (kRowWords + kMtN) * 4, S(stream)>>>(sp);
    return;
  }
  if (const char* fc = ab_env("TL_RESET_CTA")) {
    const int e = atoi(fc);
    if (e == 16) {
      const int smem = 16 * 2 * kRowWords * 4;
      set_max_smem(k_fuzz_reset_cta<16>, smem);
      k_fuzz_reset_cta<16><<<(n + 15) / 16, 16 * 32, smem, S(stream)>>>(sp);
    } else {
      const int smem = 8 * 2 * kRowWords * 4;
      set_max_smem(k_fuzz_reset_cta<8>, smem);
      k_fuzz_reset_cta<8><<<(n + 7) / 8, 8 * 32, smem, S(stream)>>>(sp);
    }
    return;
  }
  if (ab_env("TL_RESET_SH")) {
    const int e = atoi(ab_env("TL_RESET_SH"));
    const int smem = 2 * e * kRowWords * 4;
    if (e == 4) {
      set_max_smem(k_fuzz_reset_sh<4>, smem);
      k_fuzz_reset_sh<4><<<(n + 3) / 4, 32, smem, S(stream)>>>(sp);
    } else if (e == 2) {
      k_fuzz_reset_sh<2><<<(n + 1) / 2, 32, smem, S(stream)>>>(sp);
    } else {
      set_max_smem(k_fuzz_reset_sh<8>, smem);
      k_fuzz_reset_sh<8><<<(n + 7) / 8, 32, smem, S(stream)>>>(sp);
    }
    return;
  }
  if (const char* force = ab_env("TL_RESET_EPW")) {
    const int epw = atoi(force);
    const bool stream_seed = epw >= 2 && ab_env("TL_RESET_ROWS2") == nullptr;
    const int smem = (stream_seed ? 1 : 2) * epw * kRowWords * 4;
    if (epw == 2 && stream_seed) { set_max_smem(k_fuzz_reset<2, true>, smem); k_fuzz_reset<2, true><<<(n + 1) / 2, 32, smem, S(stream)>>>(sp); }
    else if (epw == 2) { set_max_smem(k_fuzz_reset<2, false>, smem); k_fuzz_reset<2, false><<<(n + 1) / 2, 32, smem, S(stream)>>>(sp); }
    else if (epw == 4 && stream_seed) { set_max_smem(k_fuzz_reset<4, true>, smem); k_fuzz_reset<4, true><<<(n + 3) / 4, 32, smem, S(stream)>>>(sp); }
    else if (epw == 4) { set_max_smem(k_fuzz_reset<4, false>, smem); k_fuzz_reset<4, false><<<(n + 3) / 4, 32, smem, S(stream)>>>(sp); }
    else if (epw == 16) { set_max_smem(k_fuzz_reset<16, true>, smem); k_fuzz_reset<16, true><<<(n + 15) / 16, 32, smem, S(stream)>>>(sp); }
    else { set_max_smem(k_fuzz_reset<8, true>, smem); k_fuzz_reset<8, true><<<(n + 7) / 8, 32, smem, S(stream)>>>(sp); }
    return;
  }
#endif
  if ((int64_t)n <= (int64_t)sms * 64) {
    // a CTA of 8 warps per 8 episodes: warp 0 seeds the 16 states into shared
    // rows, one random_script sampler per warp, longest-first slots per CTA
    // (scripts/ab_env.sh: -2.3% on the 4096-env step, -4.5% at 1024, -2.8% C3
    // against the lane-per-sampler forms)
    const int smem = 8 * 2 * kRowWords * 4;
    set_max_smem(k_fuzz_reset_cta<8>, smem);
    k_fuzz_reset_cta<8><<<(n + 7) / 8, 8 * 32, smem, S(stream)>>>(sp);
  } else {
    // large batches (throughput): streamed seeding, one shared row per episode
    set_max_smem(k_fuzz_reset<8, true>, 8 * kRowWords * 4);
    k_fuzz_reset<8, true><<<(n + 7) / 8, 32, 8 * kRowWords * 4, S(stream)>>>(sp);
  }
}

#ifdef TL_AB
typedef void (*SynthKernel)(SynthParams);
static SynthKernel synth_kernel(int w, bool fuzz, bool small) {
  if (w == 32)
    return fuzz ? (small ? k_synth_cta<true, 7, 32> : k_synth_cta<true, 16, 32>)
                : (small ? k_synth_cta<false, 7, 32> : k_synth_cta<false, 16, 32>);
  return fuzz ? (small ? k_synth_cta<true, 7, 64> : k_synth_cta<true, 16, 64>)
              : (small ? k_synth_cta<false, 7, 64> : k_synth_cta<false, 16, 64>);
}
#endif

typedef void (*SynthWarpKernel)(SynthParams);
#ifndef TL_SYNTH_NW
#define TL_SYNTH_NW 2
#endif
constexpr int kSynthWarps = TL_SYNTH_NW;  // warps (independent episodes) per CTA of k_synth_warp

static int launch_synth(SynthParams& sp, bool fuzz, void* stream) {
  // realize + label: one warp per episode (tl_synth_warp.cuh)
  const bool small = sp.out.dof <= 7;
  if (fuzz) {
    launch_fuzz_reset(sp, stream);
  } else {
    k_seed_states<<<(sp.n_env + 127) / 128, 128, 0, S(stream)>>>(sp);
  }
#ifdef TL_AB
  if (ab_env("TL_SYNTH_CTA")) {  // the one-CTA-per-episode kernel (tl_synth_cta.cuh)
    const char* fw = ab_env("TL_SYNTH_WAVE");
    const int W = fw ? (atoi(fw) == 32 ? 32 : 64)
                     : (sp.cap_per_env > 0 && sp.cap_per_env <= 64 ? 32 : 64);
    const int threads = W + 32;
    const int smem = W == 32 ? (small ? (int)sizeof(CtaSmem<7, 32>) : (int)sizeof(CtaSmem<16, 32>))
                             : (small ? (int)sizeof(CtaSmem<7, 64>) : (int)sizeof(CtaSmem<16, 64>));
    SynthKernel k = synth_kernel(W, fuzz, small);
    set_max_smem(k, smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, threads, smem);
    if (per_sm < 1) per_sm = 1;
    k<<<blocks_for(sp.n_env, 1, sm_count() * per_sm), threads, smem, S(stream)>>>(sp);
    return check_launch();
  }
#endif
  const bool d7 = sp.out.dof == 7;
  const SynthWarpKernel k =
      fuzz ? (d7 ? k_synth_warp<true, 7, kSynthWarps, 7>
                 : small ? k_synth_warp<true, 7, kSynthWarps, 0> : k_synth_warp<true, 16, kSynthWarps, 0>)
           : (d7 ? k_synth_warp<false, 7, kSynthWarps, 7>
                 : small ? k_synth_warp<false, 7, kSynthWarps, 0> : k_synth_warp<false, 16, kSynthWarps, 0>);
  const int smem = kSynthWarps * (small ? (int)sizeof(WarpSmem<7>) : (int)sizeof(WarpSmem<16>));
  set_max_smem(k, smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kSynthWarps * 32, smem);
  if (per_sm < 1) per_sm = 1;
  // long episodes and at most ~2 per warp slot: the batch time is the longest
  // episodes' latency, so 12 warps per SM (less issue contention for them)
  // beat 16 (scripts/ab_env2.sh: -1.5% on the 4096-env Place step; the
  // short-episode C3 batch and a 16384-env batch want all 16)
  if (sp.order && (int64_t)sp.n_env <= (int64_t)sm_count() * 32)
    per_sm = std::min(per_sm, 12 / kSynthWarps);
  if (const char* f = ab_env("TL_SYNTH_CTAS")) per_sm = std::min(per_sm, std::max(1, atoi(f)));
  const int grid = blocks_for(sp.n_env, kSynthWarps, sm_count() * per_sm);
  if (ab_env("TL_DEBUG"))
    fprintf(stderr, "k_synth_warp: %d CTAs/SM x %d warps (smem %d B), grid %d\n", per_sm,
            kSynthWarps, smem, grid);
  k<<<grid, kSynthWarps * 32, smem, S(stream)>>>(sp);
  return check_launch();
}

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }


size_t tl_fuzz_scratch_bytes(int32_t n_env, const tl_fuzz_cfg* cfg) {
  const size_t n = n_env > 0 ? (size_t)n_env : 1, ms = cfg ? (size_t)(cfg->max_events + 4) : 64;
  return align256(n * kMtN * 4) + align256(n * sizeof(tl_script)) + align256(n * ms) +
         align256(n * ms * 4) + align256((n + 1) * 8)  // + k_scan_emit tile states (tl_fuzz_ev)
         + align256(n * kLenBuckets * 4)          // + longest-first episode order
         + 256;                                   // + episode / emission tickets
}

size_t tl_realize_scratch_bytes(int32_t n_env) {
  return align256((size_t)(n_env > 0 ? n_env : 1) * kMtN * 4) + 256;  // states + tickets
}

static int fuzz_impl(const int64_t* seeds, const uint8_t* subtasks, int32_t n_env, int32_t subtask,
                     const tl_fuzz_cfg* cfg,
                     const tl_thresholds* th_realize, const tl_cset* label_csets,
                     const tl_rules* rules, tl_records* out, int32_t cap_per_env,
                     uint8_t* script_kind, int32_t* script_gap, tl_script* scripts,
                     uint8_t* step_mask, tl_label* labels, int64_t* ev_off, uint8_t* ev_kind,
                     int32_t* ev_t, void* scratch, void* stream) {
  if (!cfg || !th_realize || !label_csets || !out || !labels || !scratch || n_env < 0 ||
      (!subtasks && (subtask < 0 || subtask > 3)) || out->dtype != 0 || out->dof < 1 || out->dof > TL_MAX_DOF ||
      cfg->max_gap < 1 || cfg->max_tail < 1 || cfg->max_events < 0 ||
      cap_per_env < 2 || (script_kind && !script_gap) ||
      (!script_kind && script_gap))
    return TL_E_INVALID;
  if (n_env == 0) return TL_OK;
  const size_t n = (size_t)n_env, ms = (size_t)(cfg->max_events + 4);
  char* base = reinterpret_cast<char*>(scratch);
  SynthParams sp;
  memset(&sp, 0, sizeof(sp));
  // the claim counters come first: at a fixed offset for any n_env, so the
  // zero state every call leaves them in holds across calls of other sizes
  sp.tickets = reinterpret_cast<unsigned int*>(base);
  base += 256;
  sp.states = reinterpret_cast<uint32_t*>(base);
  base += align256(n * kMtN * 4);
  sp.scripts = scripts ? scripts : reinterpret_cast<tl_script*>(base);
  base += align256(n * sizeof(tl_script));
  sp.step_kind = script_kind ? script_kind : reinterpret_cast<uint8_t*>(base);
  base += align256(n * ms);
  sp.step_gap = script_gap ? script_gap : reinterpret_cast<int32_t*>(base);
  base += align256(n * ms * 4);
  sp.ev_state = reinterpret_cast<unsigned long long*>(base);
  base += align256((n + 1) * 8);
  sp.order = reinterpret_cast<int32_t*>(base);
  if (cap_per_env <= 64) sp.order = nullptr;  // every episode fits one wave: index order
  sp.seeds = seeds;
  sp.fuzz_subtask = subtask;
  sp.subtasks = subtasks;
  sp.cfg = *cfg;
  sp.n_env = n_env;
  sp.cap_per_env = cap_per_env;
  sp.th = *th_realize;
  sp.label_csets = label_csets;
  sp.rules = rules_or_default(rules);
  sp.out = *out;
  sp.step_mask = step_mask;
  sp.labels = labels;
  if (ev_off) {  // tl_fuzz_ev: ordered event lists by k_scan_emit right after the realize kernel
    const int tiles = (n_env + 31) / 32;
    sp.ev_zero = tiles + 1;  // tile states + the tile counter, zeroed by the reset kernel
    const int rc = launch_synth(sp, true, stream);
    if (rc != TL_OK) return rc;
    k_scan_emit<<<tiles, 1024, 0, S(stream)>>>(step_mask, out->rec_start, out->n_rec, labels, n_env,
                                                ev_off, ev_kind, ev_t, sp.ev_state);
    return check_launch();
  }
  return launch_synth(sp, true, stream);
}

int tl_fuzz(const int64_t* seeds, int32_t n_env, int32_t subtask, const tl_fuzz_cfg* cfg,
            const tl_thresholds* th_realize, const tl_cset* label_csets, const tl_rules* rules,
            tl_records* out, int32_t cap_per_env, uint8_t* script_kind, int32_t* script_gap,
            tl_script* scripts, uint8_t* step_mask, tl_label* labels, void* scratch,
            void* stream) {
  return fuzz_impl(seeds, nullptr, n_env, subtask, cfg, th_realize, label_csets, rules, out, cap_per_env,
                   script_kind, script_gap, scripts, step_mask, labels, nullptr, nullptr, nullptr,
                   scratch, stream);
}

int tl_fuzz_ev(const int64_t* seeds, int32_t n_env, int32_t subtask, const tl_fuzz_cfg* cfg,
               const tl_thresholds* th_realize, const tl_cset* label_csets, const tl_rules* rules,
               tl_records* out, int32_t cap_per_env, uint8_t* script_kind, int32_t* script_gap,
               tl_script* scripts, uint8_t* step_mask, tl_label* labels, int64_t* ev_off,
               uint8_t* ev_kind, int32_t* ev_t, int64_t ev_capacity, void* scratch,
               void* stream) {
  if (!ev_off || !ev_kind || !ev_t || !step_mask ||
      ev_capacity < (int64_t)n_env * cap_per_env * 4)  // <= 4 events per record (Open/Close)
    return TL_E_INVALID;
  if (n_env == 0) return cudaMemsetAsync(ev_off, 0, 8, S(stream)) ? TL_E_CUDA : TL_OK;
  return fuzz_impl(seeds, nullptr, n_env, subtask, cfg, th_realize, label_csets, rules, out, cap_per_env,
                   script_kind, script_gap, scripts, step_mask, labels, ev_off, ev_kind, ev_t,
                   scratch, stream);
}

int tl_fuzz_mixed(const int64_t* seeds, const uint8_t* subtasks, int32_t n_env,
                  const tl_fuzz_cfg* cfg, const tl_thresholds* th_realize,
                  const tl_cset* label_csets, const tl_rules* rules, tl_records* out,
                  int32_t cap_per_env, uint8_t* script_kind, int32_t* script_gap,
                  tl_script* scripts, uint8_t* step_mask, tl_label* labels, void* scratch,
                  void* stream) {
  if (!subtasks && n_env > 0) return TL_E_INVALID;
  return fuzz_impl(seeds, subtasks, n_env, 0, cfg, th_realize, label_csets, rules, out,
                   cap_per_env, script_kind, script_gap, scripts, step_mask, labels, nullptr,
                   nullptr, nullptr, scratch, stream);
}

int tl_fuzz_ev_mixed(const int64_t* seeds, const uint8_t* subtasks, int32_t n_env,
                     const tl_fuzz_cfg* cfg, const tl_thresholds* th_realize,
                     const tl_cset* label_csets, const tl_rules* rules, tl_records* out,
                     int32_t cap_per_env, uint8_t* script_kind, int32_t* script_gap,
                     tl_script* scripts, uint8_t* step_mask, tl_label* labels, int64_t* ev_off,
                     uint8_t* ev_kind, int32_t* ev_t, int64_t ev_capacity, void* scratch,
                     void* stream) {
  if ((!subtasks && n_env > 0) || !ev_off || !ev_kind || !ev_t || !step_mask ||
      ev_capacity < (int64_t)n_env * cap_per_env * 4)
    return TL_E_INVALID;
  if (n_env == 0) return cudaMemsetAsync(ev_off, 0, 8, S(stream)) ? TL_E_CUDA : TL_OK;
  return fuzz_impl(seeds, subtasks, n_env, 0, cfg, th_realize, label_csets, rules, out,
                   cap_per_env, script_kind, script_gap, scripts, step_mask, labels, ev_off,
                   ev_kind, ev_t, scratch, stream);
}

int tl_realize(const tl_script* scripts, const uint8_t* step_kind, const int32_t* step_gap,
               int32_t n_env, const tl_thresholds* th_realize, const tl_cset* label_csets,
               const tl_rules* rules, tl_records* out, uint8_t* step_mask, tl_label* labels,
               void* scratch, void* stream) {
  if (!scripts || !th_realize || !label_csets || !out || !labels || !scratch || n_env < 0 ||
      out->dtype != 0 || out->dof < 1 || out->dof > TL_MAX_DOF)
    return TL_E_INVALID;
  if (n_env == 0) return TL_OK;
  SynthParams sp;
  memset(&sp, 0, sizeof(sp));
  sp.scripts = const_cast<tl_script*>(scripts);
  sp.step_kind = const_cast<uint8_t*>(step_kind);
  sp.step_gap = const_cast<int32_t*>(step_gap);
  sp.states = reinterpret_cast<uint32_t*>(scratch);
  sp.tickets = reinterpret_cast<unsigned int*>(reinterpret_cast<char*>(scratch) +
                                               align256((size_t)n_env * kMtN * 4));
  sp.n_env = n_env;
  sp.th = *th_realize;
  sp.label_csets = label_csets;
  sp.rules = rules_or_default(rules);
  sp.out = *out;
  sp.step_mask = step_mask;
  sp.labels = labels;
  return launch_synth(sp, false, stream);
}

// ---- batched env ------------------------------------------------------------
size_t tl_env_state_bytes(int32_t n_env) { return env_bytes(n_env > 0 ? n_env : 1); }

static EnvParams env_params(void* state, int32_t n_env, int32_t dof) {
  EnvParams ep;
  memset(&ep, 0, sizeof(ep));
  char* b = reinterpret_cast<char*>(state);
  ep.hdr = reinterpret_cast<EnvHdr*>(b);
  ep.st = reinterpret_cast<EnvSt*>(b + env_st_off());
  ep.mt = reinterpret_cast<uint32_t*>(b + env_mt_off(n_env));
  ep.n_env = n_env;
  ep.dof = dof;
  return ep;
}

// The header (realize thresholds, label csets, sizes) is written by the
// reset kernel from its by-value parameters: no host-memory copy is captured
// into CUDA graphs.
static void env_set_hdr(EnvParams& ep, const tl_thresholds* th, const tl_cset* csets) {
  ep.th = *th;
  ep.src_cs = csets;
}

static int env_launch_reset(EnvParams& ep, void* stream) {
  const int grid = (ep.n_env + kEnvThreads - 1) / kEnvThreads;
  if (ep.dof <= 7) {
    set_max_smem(k_env_reset<7>, (int)sizeof(EnvSmem<7>));
    k_env_reset<7><<<grid, kEnvThreads, sizeof(EnvSmem<7>), S(stream)>>>(ep);
  } else {
    set_max_smem(k_env_reset<16>, (int)sizeof(EnvSmem<16>));
    k_env_reset<16><<<grid, kEnvThreads, sizeof(EnvSmem<16>), S(stream)>>>(ep);
  }
  return check_launch();
}

static bool env_obs_ok(const float* obs, int64_t stride, int64_t cols) {
  return obs && stride >= cols;
}

int tl_env_reset(void* state, int32_t n_env, int32_t dof, const tl_script* scripts,
                 const tl_thresholds* th_realize, const tl_cset* label_csets, float* obs,
                 int64_t obs_stride, uint8_t* obs_grasped, uint8_t* step_mask, void* stream) {
  if (!state || !scripts || !th_realize || !label_csets || n_env < 0 || dof < 1 ||
      dof > TL_MAX_DOF || (n_env > 0 && !env_obs_ok(obs, obs_stride, n_env)))
    return TL_E_INVALID;
  if (n_env == 0) return TL_OK;
  EnvParams ep = env_params(state, n_env, dof);
  env_set_hdr(ep, th_realize, label_csets);
  SynthParams sp;
  memset(&sp, 0, sizeof(sp));
  sp.scripts = const_cast<tl_script*>(scripts);
  sp.states = ep.mt;
  sp.n_env = n_env;
  k_seed_states<<<(n_env + 127) / 128, 128, 0, S(stream)>>>(sp);
  ep.scripts = scripts;
  ep.obs = obs;
  ep.obs_stride = obs_stride;
  ep.obs_grasped = obs_grasped;
  ep.step_mask = step_mask;
  return env_launch_reset(ep, stream);
}

int tl_env_reset_fuzz(void* state, const int64_t* seeds, int32_t n_env, int32_t subtask,
                      const tl_fuzz_cfg* cfg, const tl_thresholds* th_realize,
                      const tl_cset* label_csets, tl_script* scripts, uint8_t* script_kind,
                      int32_t* script_gap, float* obs, int64_t obs_stride, uint8_t* obs_grasped,
                      uint8_t* step_mask, void* stream) {
  if (!state || !seeds || !cfg || !th_realize || !label_csets || !scripts || !script_kind ||
      !script_gap || n_env < 0 || subtask < 0 || subtask > 3 || cfg->max_gap < 1 ||
      cfg->max_tail < 1 || cfg->max_events < 0 ||
      (n_env > 0 && !env_obs_ok(obs, obs_stride, n_env)))
    return TL_E_INVALID;
  if (n_env == 0) return TL_OK;
  const int dof = 7;  // random_script builds arm_dof = 7 scripts (synth.py:63-74)
  EnvParams ep = env_params(state, n_env, dof);
  env_set_hdr(ep, th_realize, label_csets);
  SynthParams sp;
  memset(&sp, 0, sizeof(sp));
  sp.seeds = seeds;
  sp.fuzz_subtask = subtask;
  sp.cfg = *cfg;
  sp.scripts = scripts;
  sp.step_kind = script_kind;
  sp.step_gap = script_gap;
  sp.states = ep.mt;
  sp.n_env = n_env;
  sp.cap_per_env = 0x7fffffff;
  launch_fuzz_reset(sp, stream);
  ep.scripts = scripts;
  ep.obs = obs;
  ep.obs_stride = obs_stride;
  ep.obs_grasped = obs_grasped;
  ep.step_mask = step_mask;
  return env_launch_reset(ep, stream);
}

int tl_env_step(void* state, int32_t n_env, int32_t dof, const uint8_t* actions,
                int32_t k_steps, float* obs, int64_t obs_stride, uint8_t* obs_grasped,
                uint8_t* step_mask, void* stream) {
  if (!state || n_env < 0 || dof < 1 || dof > TL_MAX_DOF || k_steps < 0 ||
      (n_env > 0 && k_steps > 0 && (!actions || !env_obs_ok(obs, obs_stride, (int64_t)k_steps * n_env))))
    return TL_E_INVALID;
  if (n_env == 0 || k_steps == 0) return TL_OK;
  EnvParams ep = env_params(state, n_env, dof);
  ep.actions = actions;
  ep.k_steps = k_steps;
  ep.obs = obs;
  ep.obs_stride = obs_stride;
  ep.obs_grasped = obs_grasped;
  ep.step_mask = step_mask;
  // 8 lanes per env while the batch leaves SMs idle (latency-bound), 4 when
  // it fills the GPU (less redundant per-env planning); 16 measured slower
  bool wide = (int64_t)n_env * 8 <= (int64_t)sm_count() * 1024;
  if (const char* f = ab_env("TL_ENV_LPE")) wide = atoi(f) == 8;
  auto go = [&](auto kern, int lpe, size_t smem) {
    set_max_smem(kern, (int)smem);
    const int per_block = kEnvQThreads / lpe;
    kern<<<(n_env + per_block - 1) / per_block, kEnvQThreads, smem, S(stream)>>>(ep);
  };
  const bool staged = k_steps > 1;
  if (dof <= 7) {
    if (wide) {
      if (staged) go(k_env_step<7, 8, true>, 8, sizeof(EnvQSmem<7, 8>));
      else go(k_env_step<7, 8, false>, 8, sizeof(EnvQSmem<7, 8>));
    } else {
      if (staged) go(k_env_step<7, 4, true>, 4, sizeof(EnvQSmem<7, 4>));
      else go(k_env_step<7, 4, false>, 4, sizeof(EnvQSmem<7, 4>));
    }
  } else {
    if (wide) {
      if (staged) go(k_env_step<16, 8, true>, 8, sizeof(EnvQSmem<16, 8>));
      else go(k_env_step<16, 8, false>, 8, sizeof(EnvQSmem<16, 8>));
    } else {
      if (staged) go(k_env_step<16, 4, true>, 4, sizeof(EnvQSmem<16, 4>));
      else go(k_env_step<16, 4, false>, 4, sizeof(EnvQSmem<16, 4>));
    }
  }
  return check_launch();
}

int tl_env_labels(const void* state, int32_t n_env, const tl_rules* rules, tl_label* labels,
                  int32_t* n_rec, void* stream) {
  if (!state || !labels || n_env < 0) return TL_E_INVALID;
  if (n_env == 0) return TL_OK;
  EnvParams ep = env_params(const_cast<void*>(state), n_env, 7);
  ep.rules = rules_or_default(rules);
  ep.labels = labels;
  ep.n_rec = n_rec;
  k_env_labels<<<(n_env + 127) / 128, 128, 0, S(stream)>>>(ep);
  return check_launch();
}

int tl_env_script_actions(const tl_script* scripts, const uint8_t* step_kind,
                          const int32_t* step_gap, int32_t n_env, int32_t t0, int32_t k_steps,
                          uint8_t* actions, void* stream) {
  if (!scripts || !step_kind || !step_gap || !actions || n_env < 0 || k_steps < 0 || t0 < 0)
    return TL_E_INVALID;
  if (n_env == 0 || k_steps == 0) return TL_OK;
  k_env_script_actions<<<(n_env + 127) / 128, 128, 0, S(stream)>>>(scripts, step_kind, step_gap,
                                                                  n_env, t0, k_steps, actions);
  return check_launch();
}

// ---- analytics counting ------------------------------------------------------
int tl_group_mode_counts(const tl_label* labels, const int32_t* group, int64_t n,
                         int32_t n_groups, int64_t* counts, void* stream) {
  if (!labels || !counts || n < 0 || n_groups < 1) return TL_E_INVALID;
  const size_t bytes = (size_t)n_groups * kCountCols * sizeof(int64_t);
  if (cudaMemsetAsync(counts, 0, bytes, S(stream))) return TL_E_CUDA;
  if (n == 0) return TL_OK;
  const int cells = n_groups * kCountCols;
  const int use_smem = cells <= 8192;
  const int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)sm_count() * 4);
  k_group_counts<<<grid, 256, use_smem ? cells * 4 : 0, S(stream)>>>(
      labels, group, n, n_groups, reinterpret_cast<unsigned long long*>(counts), use_smem);
  return check_launch();
}

int tl_chain_progress(const tl_label* labels, const int64_t* slot_label, int64_t n_chain,
                      int32_t n_slots, int64_t* alive, void* stream) {
  if (!labels || !slot_label || !alive || n_chain < 0 || n_slots < 1 || n_slots > 64)
    return TL_E_INVALID;
  if (cudaMemsetAsync(alive, 0, (size_t)n_slots * sizeof(int64_t), S(stream))) return TL_E_CUDA;
  if (n_chain == 0) return TL_OK;
  const int grid = (int)std::min<int64_t>((n_chain + 255) / 256, (int64_t)sm_count() * 4);
  k_chain_alive<<<grid, 256, 0, S(stream)>>>(labels, slot_label, n_chain, n_slots,
                                            reinterpret_cast<unsigned long long*>(alive));
  return check_launch();
}

int tl_filter_buckets(const tl_label* labels, const int32_t* key, int64_t n,
                      const int8_t* rule_lut, const int32_t* pool, const int32_t* pool_b0,
                      int32_t n_keys, int32_t* bucket, void* stream) {
  if (!labels || !key || !rule_lut || !pool || !pool_b0 || !bucket || n < 0 || n_keys < 1)
    return TL_E_INVALID;
  if (n == 0) return TL_OK;
  const int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)sm_count() * 8);
  k_filter_buckets<<<grid, 256, 0, S(stream)>>>(labels, key, n, rule_lut, pool, pool_b0, n_keys,
                                               bucket);
  return check_launch();
}

// ---- the one exchange step over NCCL ----------------------------
int tl_allgather_labels(void* nccl_comm, const tl_label* local, int64_t n_per_rank,
                        tl_label* gathered, void* stream) {
  if (!nccl_comm || !local || !gathered || n_per_rank < 0) return TL_E_INVALID;
  static AllGatherFn f = nccl_sym<AllGatherFn>("ncclAllGather");
  if (!f) return TL_E_CUDA;
  const ncclResult_t r = f(local, gathered, (size_t)n_per_rank * sizeof(tl_label), ncclUint8,
                           reinterpret_cast<ncclComm_t>(nccl_comm), S(stream));
  return r == ncclSuccess ? TL_OK : TL_E_CUDA;
}

int tl_allreduce_counts(void* nccl_comm, int64_t* counts, int64_t n, void* stream) {
  if (!nccl_comm || !counts || n < 0) return TL_E_INVALID;
  static AllReduceFn f = nccl_sym<AllReduceFn>("ncclAllReduce");
  if (!f) return TL_E_CUDA;
  const ncclResult_t r = f(counts, counts, (size_t)n, ncclInt64, ncclSum,
                           reinterpret_cast<ncclComm_t>(nccl_comm), S(stream));
  return r == ncclSuccess ? TL_OK : TL_E_CUDA;
}

size_t tl_filter_scratch_bytes(int64_t n, int32_t n_buckets, int32_t n_pools) {
  const int64_t tiles = (n + kFilterTile - 1) / kFilterTile;
  const size_t a = (size_t)(tiles > 0 ? tiles : 1) * (size_t)(n_buckets > 0 ? n_buckets : 1) * 4;
  const size_t a8 = (a + 15) & ~(size_t)15;
  return a8 + 2 * (size_t)(n_buckets > 0 ? n_buckets : 1) * 8 + (size_t)(n_pools + 1) * 0;
}

int tl_filter_select(const int32_t* bucket, int64_t n, int32_t n_buckets, int32_t n_pools,
                     const int32_t* pool_b0, const double* bucket_w, int64_t quota,
                     uint8_t* selected, int64_t* pool_selected, void* scratch, void* stream) {
  if (n < 0 || n_buckets < 0 || n_pools < 0 || quota < 0 || !scratch ||
      (n > 0 && (!bucket || !selected)) || (n_pools > 0 && (!pool_b0 || !pool_selected)))
    return TL_E_INVALID;
  if (n_buckets * 4 > 200 * 1024) return TL_E_CAPACITY;
  const int64_t tiles = (n + kFilterTile - 1) / kFilterTile;
  int32_t* tile_cnt = reinterpret_cast<int32_t*>(scratch);
  const size_t a = (size_t)(tiles > 0 ? tiles : 1) * (size_t)(n_buckets > 0 ? n_buckets : 1) * 4;
  int64_t* cnt = reinterpret_cast<int64_t*>(reinterpret_cast<char*>(scratch) + ((a + 15) & ~(size_t)15));
  int64_t* take = cnt + (n_buckets > 0 ? n_buckets : 1);
  const int hsmem = n_buckets * 4;
  if (hsmem > 48 * 1024) {
    set_max_smem(k_filter_hist, hsmem);
    set_max_smem(k_filter_select, hsmem);
  }
  if (n_buckets > 0) {
    if (tiles > 0) k_filter_hist<<<(unsigned)tiles, 256, hsmem, S(stream)>>>(bucket, n, n_buckets, tile_cnt);
    else cudaMemsetAsync(tile_cnt, 0, (size_t)n_buckets * 4, S(stream));
    k_filter_colscan<<<(n_buckets + 127) / 128, 128, 0, S(stream)>>>(tile_cnt, (int)tiles, n_buckets, cnt);
  }
  if (n_pools > 0)
    k_filter_pool<<<(n_pools + 127) / 128, 128, 0, S(stream)>>>(pool_b0, n_pools, bucket_w, cnt, quota, take, pool_selected);
  if (tiles > 0) {
    if (n_buckets > 0)
      k_filter_select<<<(unsigned)tiles, 32, hsmem, S(stream)>>>(bucket, n, n_buckets, tile_cnt, take, selected);
    else
      cudaMemsetAsync(selected, 0, (size_t)n, S(stream));
  }
  return check_launch();
}

int tl_eval_predicates(const tl_records* recs, int32_t n_env, const int32_t* env_cset,
                       const tl_cset* csets, const double* a0, uint8_t* bits, uint8_t* errs,
                       double* jmax, void* stream) {
  if (!recs || !env_cset || !csets || n_env < 0 || recs->dof < 1 || recs->dof > TL_MAX_DOF ||
      (recs->dtype != 0 && recs->dtype != 1))
    return TL_E_INVALID;
  if (n_env == 0) return TL_OK;
  // 128 blocks (of 8 warps) per SM, grid-stride beyond: each warp labels ~7
  // episodes of a 2^20-episode batch, and the episodes in flight stay close
  // in memory (measured: 16/SM 84 %, 128/SM 89 %, one block per 8 episodes 78 %
  // of HBM on the Pick sizing run)
  const char* gm = ab_env("TL_LABEL_GRID_PER_SM");
  const int grid = blocks_for(n_env, kLabelWarps, sm_count() * (gm ? std::max(1, atoi(gm)) : 128));
  const dim3 blk(kLabelWarps * 32);
  if (recs->dtype == 0) {
    if (recs->dof <= 7) k_predicates<float, 7><<<grid, blk, 0, S(stream)>>>(*recs, n_env, env_cset, csets, a0, bits, errs, jmax);
    else k_predicates<float, 16><<<grid, blk, 0, S(stream)>>>(*recs, n_env, env_cset, csets, a0, bits, errs, jmax);
  } else {
    if (recs->dof <= 7) k_predicates<double, 7><<<grid, blk, 0, S(stream)>>>(*recs, n_env, env_cset, csets, a0, bits, errs, jmax);
    else k_predicates<double, 16><<<grid, blk, 0, S(stream)>>>(*recs, n_env, env_cset, csets, a0, bits, errs, jmax);
  }
  return check_launch();
}

int tl_scan_counts(const int32_t* counts, int32_t n, int64_t* off, void* scratch, void* stream) {
  if (!off || n < 0 || (n > 0 && (!counts || !scratch))) return TL_E_INVALID;
  if (n == 0) {
    cudaMemsetAsync(off, 0, sizeof(int64_t), S(stream));
    return check_launch();
  }
  const int tiles = (n + kScanBlock - 1) / kScanBlock;
  int64_t* tile = reinterpret_cast<int64_t*>(scratch);
  k_scan_i32_tiles<<<tiles, kScanBlock, 0, S(stream)>>>(counts, n, off, tile);
  k_scan_sums<<<1, kScanBlock, 0, S(stream)>>>(tile, tiles, off, n);
  k_scan_add<<<(n + 255) / 256, 256, 0, S(stream)>>>(off, tile, n);
  return check_launch();
}

int tl_compact_records(const tl_records* src, int32_t n_env, const int64_t* dst_start,
                       tl_records* dst, void* stream) {
  if (!src || !dst || !dst_start || n_env < 0 || src->dtype != dst->dtype || src->dof != dst->dof)
    return TL_E_INVALID;
  if (n_env == 0) return TL_OK;
  const int np_ = 2 * src->dof + 9;
  const int grid = blocks_for(n_env, 8, sm_count() * 8);
  if (src->dtype == 0) k_compact<float><<<grid, 256, 0, S(stream)>>>(*src, n_env, dst_start, *dst, np_);
  else k_compact<double><<<grid, 256, 0, S(stream)>>>(*src, n_env, dst_start, *dst, np_);
  return check_launch();
}

#ifdef TL_PHASES
extern "C" int tl_warp_timeline(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, g_tl_warp, sizeof(g_tl_warp)) == cudaSuccess ? TL_OK : TL_E_CUDA;
}
extern "C" int tl_step_timeline(unsigned long long* out, int reset) {
  if (cudaMemcpyFromSymbol(out, g_tl_step, sizeof(g_tl_step)) != cudaSuccess) return TL_E_CUDA;
  if (reset) {  // starts to +inf, ends to 0
    static unsigned long long z[2][2048][2];
    for (int k = 0; k < 2; k++)
      for (int b = 0; b < 2048; b++) z[k][b][0] = ~0ull, z[k][b][1] = 0ull;
    if (cudaMemcpyToSymbol(g_tl_step, z, sizeof(z)) != cudaSuccess) return TL_E_CUDA;
  }
  return TL_OK;
}
extern "C" int tl_warp_phases(unsigned long long* out, int reset) {
  if (cudaMemcpyFromSymbol(out, g_tl_wphase, sizeof(g_tl_wphase)) != cudaSuccess) return TL_E_CUDA;
  if (reset) {
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(g_tl_wphase, z, sizeof(z));
  }
  return TL_OK;
}
#endif
#if defined(TL_PHASES) && defined(TL_AB)
extern "C" int tl_phase_read(unsigned long long* out, int reset) {
  if (cudaMemcpyFromSymbol(out, g_tl_phase, sizeof(unsigned long long) * 16) != cudaSuccess) return TL_E_CUDA;
  if (reset) {
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(g_tl_phase, z, sizeof(z));
  }
  return TL_OK;
}
#endif

#ifdef TL_PROFILE
int tl_prof_read(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, g_tl_prof, sizeof(unsigned long long) * 128) == cudaSuccess ? 0 : TL_E_CUDA;
}
#endif

int tl_validate_records(const tl_records* recs, int32_t n_env, const tl_vbounds* vb,
                        const int64_t* t, uint8_t* vflags, tl_vsummary* vsum, void* stream) {
  if (!recs || n_env < 0 || recs->dof < 0 || recs->dof > TL_MAX_DOF || recs->dtype < 0 ||
      recs->dtype > 1)
    return TL_E_INVALID;
  if (n_env == 0) return TL_OK;
  if (!vb || !vsum || !recs->planes || !recs->rec_start || !recs->n_rec) return TL_E_INVALID;
  const int grid = blocks_for(n_env, kValidateWarps, sm_count() * 16);
  if (recs->dtype == 0)
    k_validate<float><<<grid, kValidateWarps * 32, 0, S(stream)>>>(*recs, n_env, vb, t, vflags, vsum);
  else
    k_validate<double><<<grid, kValidateWarps * 32, 0, S(stream)>>>(*recs, n_env, vb, t, vflags, vsum);
  return check_launch();
}

int tl_mode_histogram(const tl_label* labels, int32_t n, int64_t* hist, void* stream) {
  if (!hist || n < 0 || (n > 0 && !labels)) return TL_E_INVALID;
  cudaMemsetAsync(hist, 0, TL_N_MODES * sizeof(int64_t), S(stream));
  if (n > 0)
    k_mode_hist<<<blocks_for(n, 256, sm_count() * 4), 256, 0, S(stream)>>>(
        labels, n, reinterpret_cast<unsigned long long*>(hist));
  return check_launch();
}

}  // extern "C"
