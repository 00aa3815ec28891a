// cog_kernels.cu -- B200 (sm_100a) kernels of the Cascade-of-Gaussians hot
// path and the C-ABI declared in include/cog_b200.h.
//
// Kernels (one launch each, all asynchronous on the caller's stream):
//   prior_kernel     training prior: one CTA stages 32 pixels x N frames of
//                    one stream in shared memory, builds per-pixel 256-bin
//                    histograms for each trailing window (bin-major,
//                    conflict-free, no atomics), smooths them with the
//                    grid-normalised Gaussian over the distinct sample
//                    values only, and writes the f32 tables, the peak, the
//                    pooled residue counts and the dynamics class.
//   warmup_kernel    GMM warm-up: one thread per plane-pixel streams the N
//                    training frames with the mixture in registers
//                    (binary64), records the channel-0 adaptation
//                    statistics for grouping and seeds the mode references.
//   step_kernel      the fused per-frame step: persistent CTAs sweep
//                    stride-aligned warp tiles (stride rows x cw columns),
//                    run skip/copy gating, confidence, cascade descent and
//                    bookkeeping per plane-pixel, resolve copies from the
//                    tile's shared-memory labels, write the union mask, and
//                    reduce level counts + per-group partials (exact
//                    integer/fixed-point sums, so the result is independent
//                    of CTA count and order).  The last CTA of each stream
//                    applies the group update, the illumination test and the
//                    frame statistics.  A pending illumination reset or a
//                    scheduled reorder is applied lazily per pixel at the
//                    start of the next frame (they touch disjoint state).
//   finalize_kernel  the same tail for row-band shards after an all-reduce.
//   pending_kernel   materialises a pending reset / reorder on demand.
//   baseline_kernel  plain mixture over all planes (gmm.classify_frame).
//   export/import    reference-layout (f64 / i64) views of the packed state.
#include "cog_device.cuh"
#include "../../include/cog_b200.h"

#include <cmath>
#include <mutex>

using namespace cog;

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int STEP_THREADS = 256;
constexpr int PRIOR_PIX = 32;
constexpr int STATS_WORDS = 16;
#ifndef DEEP_THREADS
#define DEEP_THREADS 256  // deep_kernel CTA size
#endif
#ifndef DEEP_MINB
#define DEEP_MINB 2  // deep_kernel CTAs per SM the registers must allow
#endif
#ifndef DEEP_AHEAD
#define DEEP_AHEAD 1  // deep_kernel item pipeline (build-time A/B switch)
#endif

// accumulator layout (u64 words, per stream)
__host__ __device__ inline int acc_kind(int c, int k) { return c * 7 + k; }
__host__ __device__ inline int acc_fg(int d) { return 7 * d; }
__host__ __device__ inline int acc_grp(int d, int G, int c, int g) {
  return 7 * d + 1 + (c * G + g) * 6;
}
// last word: nonzero when this frame's pass cleared the packed hit bytes
// (cog_state.hitq) of every plane-pixel -- reset, reorder or fold
__host__ __device__ inline int acc_flag(int d, int G) {
  return 7 * d + 1 + 6 * d * G;
}
__host__ __device__ inline int acc_words(int d, int G) {
  return 7 * d + 2 + 6 * d * G;
}
// frames the packed hit bytes may collect before they are folded into the
// wide counters (a byte holds 255)
constexpr uint32_t HITQ_FOLD_AGE = 250;
// per (c, g): 0 hit count, 1 sum v over hits, 2 conf hi, 3 conf lo,
//             4 sum v over all members, 5 member count
constexpr int CONF_SPLIT = 26;  // conf fixed point: q = floor(conf * 2^52)

struct StepArgs {
  cog_geom g;
  cog_params q;
  cog_state s;
  const uint8_t* frame;
  uint8_t* mask;
  void* conf;
  uint8_t* kind;
  int64_t* stats;
  int64_t frame_index;
  int reorder_now;
  int fuse_finalize;
  int cw, iters, tiles_x, n_tiles;
  int two_ended;  // the worklist was filled from both ends (hot_flush)
  cog_peers peers;  // n_ranks > 1: cross-shard sum over peer mailboxes
};

// ---------------------------------------------------------------------------
// Hot prior layout (tabq).  The float32 step reads ONE entry of a pixel's
// 256-bin prior per frame (at the pixel's value v).  Pixel-major (the
// reference's [P][256]) every lookup of a warp is a random DRAM line.  The
// hot copy is tile-major -- per plane [n_tiles][256][SL], the SL slots of a
// bin being the pixels of one warp tile (stride rows x cw columns, slot =
// row * cw + col, SL = iters * 32) -- so lanes of a warp that see the same
// value share a line, and it holds phat = table / peak quantised to u16, so
// a 128-B line covers two bins (a warp tile's ~17 distinct values touch
// ~9 lines instead of 17).  The exact f32 table stays in the reference
// layout for the binary64 paths, the decisions the u16 value cannot settle,
// and model files.
// ---------------------------------------------------------------------------
struct TabGeo {
  uint32_t W, st, cw, tiles_x, SL;
  size_t plane;  // floats per plane
};

__host__ __device__ inline void tile_shape(int st, int H, int W, int& cw,
                                           int& iters, int& tiles_x,
                                           int& n_tiles) {
  const int m = (32 / (st * st)) > 0 ? 32 / (st * st) : 1;
  cw = st * m;
  iters = (st * cw + 31) / 32;
  tiles_x = (W + cw - 1) / cw;
  n_tiles = tiles_x * ((H + st - 1) / st);
}

__host__ __device__ inline TabGeo tab_geo(const cog_geom& g) {
  int cw, iters, tiles_x, n_tiles;
  tile_shape(g.stride, g.height, g.width, cw, iters, tiles_x, n_tiles);
  TabGeo t;
  t.W = (uint32_t)g.width;
  t.st = (uint32_t)g.stride;
  t.cw = (uint32_t)cw;
  t.tiles_x = (uint32_t)tiles_x;
  t.SL = (uint32_t)(iters * 32);
  t.plane = (size_t)n_tiles * 256 * t.SL;
  return t;
}

// offset of pixel p's bin 0 inside its plane's table; bin v is at + v * SL
__device__ __forceinline__ size_t tab_pix(const TabGeo& t, size_t p) {
  const uint32_t y = (uint32_t)(p / t.W), x = (uint32_t)(p - (size_t)y * t.W);
  const uint32_t ty = y / t.st, r = y - ty * t.st;
  const uint32_t tx = x / t.cw, col = x - tx * t.cw;
  return (size_t)(ty * t.tiles_x + tx) * 256 * t.SL + r * t.cw + col;
}

__device__ __forceinline__ double clip_rint(double x) {
  double r = rint(x);
  return r < 0.0 ? 0.0 : (r > 255.0 ? 255.0 : r);
}

// ---------------------------------------------------------------------------
// One plane of one stream, by value (cold-path functions take it in
// registers; no pointer-to-struct round trips through local memory).
// ---------------------------------------------------------------------------
template <typename T>
struct PlaneRef {
  T* mix;              // this plane's mixture records, R elements each
  uint16_t* meta;
  uint32_t* dyn;
  uint32_t* streak;
  uint32_t* hits;
  uint32_t* hitq;      // packed hit bytes of the float32 hot pass, or null
  const float* table;  // this plane's prior, reference layout [P][256]
  const float* peak;
  size_t P;
  int R, KB;           // record length and K bucket (w_k at 2 * KB + k)
};

template <typename T>
__device__ __forceinline__ PlaneRef<T> plane_ref(const StepArgs& a, int s,
                                                 int c) {
  const size_t P = (size_t)a.g.height * a.g.width;
  const size_t sc = (size_t)s * a.g.depth + c;
  PlaneRef<T> r;
  r.KB = kbucket(a.g.k);
  r.R = rec_elems(r.KB);
  r.mix = (T*)a.s.mix + sc * P * (size_t)r.R;
  r.meta = a.s.meta + sc * P;
  r.dyn = a.s.dyn + sc * P;
  r.streak = a.s.streak + sc * P;
  r.hits = a.s.hits + sc * 5 * P;
  r.hitq = a.s.hitq ? a.s.hitq + sc * P : nullptr;
  r.table = a.s.table + sc * P * 256;
  r.peak = a.s.peak + sc * P;
  r.P = P;
  return r;
}

// mode k of plane-pixel p
template <typename T>
__device__ __forceinline__ T* rec_of(const PlaneRef<T>& r, size_t p) {
  return r.mix + p * (size_t)r.R;
}
template <typename T>
__device__ __forceinline__ T* w_of(const PlaneRef<T>& r, size_t p, int k) {
  return r.mix + p * (size_t)r.R + 2 * r.KB + k;
}

// the whole record in one round of 16-byte loads; e keeps dead slots and
// padding so the record can be stored back whole (KMAX is the bucket)
template <typename T, int KMAX>
__device__ __forceinline__ void load_mix_r(const PlaneRef<T>& r, size_t p,
                                           int n, Mix<KMAX>& x,
                                           T (&e)[rec_elems(KMAX)]) {
  rec_load<rec_elems(KMAX)>(rec_of(r, p), e);
  rec_to_mix<KMAX, T>(e, n, x);
}

template <typename T, int KMAX>
__device__ __forceinline__ void store_mix_r(const PlaneRef<T>& r, size_t p,
                                            int n, const Mix<KMAX>& x,
                                            T (&e)[rec_elems(KMAX)]) {
  mix_to_rec<KMAX, T>(x, n, e);
  rec_store<rec_elems(KMAX)>(rec_of(r, p), e);
}

// ---------------------------------------------------------------------------
// Cold paths (rare per frame): kept out of line so the hot loop stays small.
// ---------------------------------------------------------------------------

// Illumination reset of one plane-pixel (cascade.py:361-391, per-pixel part)
template <typename T, int KMAX>
__device__ __noinline__ void cold_reset(PlaneRef<T> r, size_t p,
                                        double init_var) {
  uint32_t meta = r.meta[p];
  uint32_t dyn = r.dyn[p];
  int n = meta_count(meta);
  Mix<KMAX> x;
  T e[rec_elems(KMAX)];
  load_mix_r<T, KMAX>(r, p, n, x, e);
  double v = (double)dyn_chp(dyn);
#pragma unroll
  for (int k = 0; k < KMAX; ++k) {
    if (k < n) {
      x.mu[k] = v;
      x.var[k] = init_var;
    }
  }
  int inv[KMAX];
  sort_modes<KMAX>(x, n, inv);
  store_mix_r<T, KMAX>(r, p, n, x, e);
  r.meta[p] = (uint16_t)meta_with_refs(meta,
                                       select_inv<KMAX>(inv, meta_ref(meta, 0)),
                                       select_inv<KMAX>(inv, meta_ref(meta, 1)));
  // streak, clock, waking, hits -> 0; last_active -> -1; label, chp kept
  r.dyn[p] = pack_dyn(dyn_chp(dyn), dyn_label(dyn), 0, -1, 0);
  r.streak[p] = 0;
#pragma unroll
  for (int l = 0; l < 5; ++l) r.hits[l * r.P + p] = 0;
  if (r.hitq) r.hitq[p] = 0u;
}

// Level reorder of one plane-pixel (cascade.py:393-417)
template <typename T>
__device__ __noinline__ void cold_reorder(PlaneRef<T> r, size_t p,
                                          double group_mu) {
  uint32_t meta = r.meta[p];
  int code[3];
  long long nh[3];
  double nm[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    code[j] = meta_mid(meta, j);
    nh[j] = 1;                                              // -(-1)
    nm[j] = __longlong_as_double(0x7ff0000000000000ll);     // -(-inf)
    if (code[j] >= 0) {
      nh[j] = -(long long)r.hits[(size_t)code[j] * r.P + p];
      if (r.hitq && code[j] < 4) nh[j] -= (r.hitq[p] >> (8 * code[j])) & 0xFFu;
      double lmu = group_mu;
      if (code[j] != L_GROUP) {
        int k = meta_ref(meta, code[j] == L_MEAN ? 0 : 1);
        lmu = ldrw(rec_of(r, p) + 2 * k);
      }
      nm[j] = -(double)r.table[p * 256 + (size_t)clip_rint(lmu)];
    }
  }
  // np.lexsort((-mass, -hv)): primary -hv, secondary -mass, stable
  int out[3] = {-1, -1, -1};
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    int rank = 0;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      bool less = (nh[j] < nh[i]) || (nh[j] == nh[i] && nm[j] < nm[i]);
      bool tie = (nh[j] == nh[i]) && (nm[j] == nm[i]);
      rank += less || (j < i && tie);
    }
#pragma unroll
    for (int t = 0; t < 3; ++t)
      if (rank == t) out[t] = code[i];
  }
  r.meta[p] = (uint16_t)meta_with_mids(meta, out[0], out[1], out[2]);
#pragma unroll
  for (int l = 0; l < 5; ++l) r.hits[l * r.P + p] = 0;
  if (r.hitq) r.hitq[p] = 0u;
}

// the float32 hot pass's packed hit bytes folded into the wide counters
// (before a byte can wrap: finalize_stream's frame count)
template <typename T>
__device__ __forceinline__ void cold_fold_hits(PlaneRef<T> r, size_t p) {
  const uint32_t q = r.hitq[p];
  if (!q) return;
#pragma unroll
  for (int l = 0; l < 4; ++l) {
    const uint32_t b = (q >> (8 * l)) & 0xFFu;
    if (b) r.hits[l * r.P + p] += b;
  }
  r.hitq[p] = 0u;
}

// MEANVAR level hit: mean+variance update of mode rs, re-sort, remap refs
// (kernels_numba.py:312-334)
template <typename T, int KMAX>
__device__ __noinline__ void cold_meanvar(PlaneRef<T> r, size_t p,
                                          uint32_t meta, int rs, double v,
                                          double rho, double var_floor) {
  const int n = meta_count(meta);
  Mix<KMAX> x;
  T e[rec_elems(KMAX)];
  load_mix_r<T, KMAX>(r, p, n, x, e);
#pragma unroll
  for (int k = 0; k < KMAX; ++k) {
    if (k == rs) {
      double mm = (1.0 - rho) * x.mu[k] + rho * v;
      x.mu[k] = mm;
      double dd = v - mm;
      double s2 = (1.0 - rho) * x.var[k] + rho * (dd * dd);
      if (s2 < var_floor) s2 = var_floor;
      x.var[k] = s2;
    }
  }
  int inv[KMAX];
  sort_modes<KMAX>(x, n, inv);
  store_mix_r<T, KMAX>(r, p, n, x, e);
  r.meta[p] = (uint16_t)meta_with_refs(meta,
                                       select_inv<KMAX>(inv, meta_ref(meta, 0)),
                                       select_inv<KMAX>(inv, meta_ref(meta, 1)));
}

// Full mixture update (last level, compat mode and the baseline); remap
// the cascade's mode references unless compat (kernels_numba.py:218-237,
// 335-342).  Returns the label.
template <typename T, int KMAX>
__device__ __noinline__ int cold_gmm(PlaneRef<T> r, size_t p, uint32_t meta,
                                     double v, double rho, GmmPar gp,
                                     int kcap, int remap) {
  int n = meta_count(meta);
  Mix<KMAX> x;
  T e[rec_elems(KMAX)];
  load_mix_r<T, KMAX>(r, p, n, x, e);
  int inv[KMAX];
  int label = gmm_step<KMAX>(x, n, kcap, v, rho, gp, inv);
  store_mix_r<T, KMAX>(r, p, n, x, e);
  uint32_t nm = meta_with_count(meta, n);
  if (remap)
    nm = meta_with_refs(nm, select_inv<KMAX>(inv, meta_ref(meta, 0)),
                        select_inv<KMAX>(inv, meta_ref(meta, 1)));
  r.meta[p] = (uint16_t)nm;
  return label;
}

// ---------------------------------------------------------------------------
// The cascade pass of one plane-pixel, hot path (kernels_numba.py:188-359).
// Decides the kind, confidence and rate and does all bookkeeping, but
// leaves the two deep updates (MEANVAR hit: mean+var update and re-sort;
// GMM fall-through: full mixture update) to the caller's dense deep pass:
// `deep` returns DEEP_NONE / DEEP_MEANVAR / DEEP_GMM / DEEP_COMPAT.
// The dyn word is written here unless the kind is COPY or the label is not
// known yet (GMM): then it is returned in dyn_out (label bit 0).
// ---------------------------------------------------------------------------
struct Flags {
  bool sampling, grouping, rate, chp, literal, compat;
};

struct GroupConst {
  bool ok;       // pixel grouped and groups exist
  double mu;     // g_mu
  double thr;    // lam * sqrt(g_var)
};

enum Deep : int { DEEP_NONE = 0, DEEP_MEANVAR = 1, DEEP_GMM = 2,
                  DEEP_COMPAT = 3 };

struct HotOut {
  int kind, label, deep, rsel;
  double conf, rho;
  uint32_t dyn;
};

// Everything the common path reads, issued as two independent rounds of
// loads before any decision: round 1 needs only the pixel index, round 2
// the round-1 values (table entry at v; the mode the confidence reads).
template <typename T>
struct Pre {
  int vb;
  uint32_t dyn, meta, streak;
  float peak, tv;
  T mu0, var0, mu1, var1;  // the MEAN (ref0) and MEANVAR (ref1) modes
};

// false for pixels the sampling gate will skip or copy (no table / mode
// reads for them)
__device__ __forceinline__ bool will_evaluate(bool sampling, uint32_t dyn,
                                              int vb, bool on_lattice,
                                              double eps) {
  if (!sampling) return true;
  const int chp = dyn_chp(dyn);
  const bool changed = (double)(vb > chp ? vb - chp : chp - vb) > eps;
  if (dyn_clock(dyn) > 0) return changed;
  if (dyn_waking(dyn) == 1) return changed || on_lattice;
  return true;
}

template <typename T>
__device__ __forceinline__ void preload_r1(const PlaneRef<T>& pr, size_t p,
                                           const uint8_t* frame_c, Pre<T>& x) {
  x.vb = frame_c[p];
  x.dyn = pr.dyn[p];
  x.meta = pr.meta[p];
  x.streak = pr.streak[p];
  x.peak = __ldg(pr.peak + p);
}

template <typename T>
__device__ __forceinline__ void preload_r2(const PlaneRef<T>& pr, size_t p,
                                           bool sampling, bool compat,
                                           bool on_lattice, double eps,
                                           Pre<T>& x) {
  x.tv = 0.0f;
  x.mu0 = x.mu1 = (T)0;
  x.var0 = x.var1 = (T)1;
  if (compat || !will_evaluate(sampling, x.dyn, x.vb, on_lattice, eps)) return;
  // one 32-B sector of a 1 KB row: bypass L1 (no 128-B line fill)
  x.tv = __ldcg(pr.table + p * 256 + (size_t)x.vb);
  const int r0 = meta_ref(x.meta, 0), r1 = meta_ref(x.meta, 1);
  const T* rec = rec_of(pr, p);
  x.mu0 = rec[2 * r0];
  x.var0 = rec[2 * r0 + 1];
  if (r1 != r0) {
    x.mu1 = rec[2 * r1];
    x.var1 = rec[2 * r1 + 1];
  } else {
    x.mu1 = x.mu0;
    x.var1 = x.var0;
  }
}

// ---------------------------------------------------------------------------
// float32-state mode: confidence and level tests in fp32 with filtered
// decisions.  Every comparison whose fp32 operands are within a relative
// margin of each other (far above the fp32 error bound, ~1e-6) is redone in
// binary64 exactly as the reference does; all decisions are therefore the
// reference's, while continuous values (conf, rho) carry fp32 rounding.
// ---------------------------------------------------------------------------
constexpr float FILTER_MARGIN = 1e-5f;
constexpr float MATCH_ABS_MARGIN = 3e-5f;  // > fp32 rounding of |v - mu| (v <= 255)

// reference form: |v - mu| <= lam * sqrt(var)
__device__ __noinline__ bool match_exact(double v, double mu, double var,
                                         double lam) {
  return fabs(v - mu) <= lam * sqrt(var);
}

// reference confidence (kernels_numba.py:243-270), binary64
__device__ __noinline__ double conf_exact(double v, double prev, double mu_top,
                                          double den, double tv, double peak,
                                          double wa, double wb, double wc,
                                          double prior_floor, int literal) {
  const double phat = tv / peak;
  double bterm = fabs(v - prev) / 255.0;
  if (!literal) bterm = 1.0 - bterm;
  double gterm = fabs(v - mu_top) / den;
  if (gterm > 1.0) gterm = 1.0;
  if (!literal) gterm = 1.0 - gterm;
  if (phat < prior_floor) {
    const double dd = wb + wc;
    return dd > 0.0 ? (wb * bterm + wc * gterm) / dd : 0.0;
  }
  return wa * phat + wb * bterm + wc * gterm;
}

template <typename T>
__device__ __forceinline__ void hot_px(const StepArgs& a, const Flags& f,
                                       const PlaneRef<T>& pr, size_t p,
                                       const Pre<T>& pre, bool on_lattice,
                                       const double* s_bt, double wa,
                                       double wb, double wc,
                                       const GroupConst& gc, HotOut& o) {
  const cog_params& q = a.q;
  const size_t P = pr.P;
  const int vb = pre.vb;
  const uint32_t dyn = pre.dyn;
  const int chp = dyn_chp(dyn);
  const int last_label = dyn_label(dyn);
  int waking = dyn_waking(dyn);
  const int last_active = dyn_active(dyn);
  int clock = dyn_clock(dyn);
  const double v = (double)vb;
  const int dv = vb > chp ? vb - chp : chp - vb;
  const bool changed = (double)dv > q.chp_epsilon;
  bool zero_streak = false;
  o.deep = DEEP_NONE;
  o.rsel = 0;
  o.rho = 0.0;

  if (f.sampling && clock > 0) {
    if (!changed) {
      clock -= 1;
      if (clock == 0) waking = 1;
      o.kind = K_SKIP;
      o.label = last_label;
      o.conf = 0.0;
      o.dyn = pack_dyn(vb, last_label, waking, last_active, clock);
      pr.dyn[p] = o.dyn;
      return;
    }
    clock = 0;
    waking = 0;
    zero_streak = true;
  } else if (f.sampling && waking == 1) {
    waking = 0;
    if (!changed && !on_lattice) {
      o.kind = K_COPY;
      o.label = last_label;
      o.conf = 0.0;
      o.dyn = pack_dyn(vb, 0, 0, last_active, q.sleep_frames);
      return;
    }
  }

  const uint32_t meta = pre.meta;
  if (f.compat) {
    // kind from the pre-update rank-0 mode; the full update is deep work
    const int n = meta_count(meta);
    int active = L_GMM;
    const T* rec = rec_of(pr, p);
    if (n > 0 && fabs(v - ldrw(rec)) <= q.match_lambda * sqrt(ldrw(rec + 1)))
      active = L_MEAN;
    atomicAdd(pr.hits + (size_t)active * P + p, 1u);  // RED: no round trip
    o.kind = active;
    o.label = 0;
    o.conf = 0.0;
    o.deep = DEEP_COMPAT;
    o.rho = q.learning_rate;
    o.dyn = pack_dyn(vb, 0, waking, active, clock);
    return;
  }

  // ---- evaluation, branch-minimal: every level test is computed, the
  // active level is the first hit in mid_order (kernels_numba.py:239-342)
  const int r0 = meta_ref(meta, 0), r1 = meta_ref(meta, 1);
  const int c0 = (meta >> 4) & 3, c1 = (meta >> 6) & 3, c2 = (meta >> 8) & 3;
  int top = c0;  // raw codes: 0 = none, 1 group, 2 mean, 3 mean+var
  if (top == L_GROUP && !f.grouping) top = c1;
  const bool group_top = (top == L_GROUP && gc.ok);
  const bool top1 = (top == L_MEANVAR);
  double conf;
  bool t0, t1;
  if constexpr (sizeof(T) == 4) {
    // fp32 values; every decision filtered to the binary64 one
    const float vf = (float)vb;
    const float lamf = (float)q.match_lambda;
    // sqrt via MUFU.RSQ (~2 ulp): only feeds filtered decisions / fp32 conf
    const float v0f = (float)pre.var0, v1f = (float)pre.var1;
    const float s0 = v0f * rsqrtf(v0f), s1 = v1f * rsqrtf(v1f);
    const float mt = group_top ? (float)gc.mu : (top1 ? (float)pre.mu1 : (float)pre.mu0);
    const float dn = group_top ? (float)gc.thr : lamf * (top1 ? s1 : s0);
    const float ph = __fdividef(pre.tv, pre.peak);
    const float bt = (float)s_bt[dv];
    float gt = fminf(__fdividef(fabsf(vf - mt), dn), 1.0f);
    if (!f.literal) gt = 1.0f - gt;
    const float pf = (float)q.prior_floor;
    float cf;
    if (ph < pf) {
      const float dd = (float)(wb + wc);
      cf = dd > 0.0f ? __fdividef((float)wb * bt + (float)wc * gt, dd) : 0.0f;
    } else {
      cf = (float)wa * ph + (float)wb * bt + (float)wc * gt;
    }
    const float ct = (float)q.confidence_threshold;
    conf = (double)cf;
    if (fabsf(ph - pf) <= FILTER_MARGIN * pf + 1e-30f ||
        fabsf(cf - ct) <= FILTER_MARGIN) {
      const double den =
          group_top ? gc.thr
                    : q.match_lambda * sqrt((double)(top1 ? pre.var1 : pre.var0));
      conf = conf_exact(v, (double)chp,
                        group_top ? gc.mu : (double)(top1 ? pre.mu1 : pre.mu0),
                        den, (double)pre.tv, (double)pre.peak, wa, wb, wc,
                        q.prior_floor, f.literal);
    }
    const float thr0 = lamf * s0, thr1 = lamf * s1;
    const float g0 = fabsf(vf - (float)pre.mu0) - thr0;
    const float g1 = fabsf(vf - (float)pre.mu1) - thr1;
    t0 = g0 <= 0.0f;
    t1 = g1 <= 0.0f;
    if (fabsf(g0) <= FILTER_MARGIN * thr0 + MATCH_ABS_MARGIN)
      t0 = match_exact(v, (double)pre.mu0, (double)pre.var0, q.match_lambda);
    if (fabsf(g1) <= FILTER_MARGIN * thr1 + MATCH_ABS_MARGIN)
      t1 = match_exact(v, (double)pre.mu1, (double)pre.var1, q.match_lambda);
  } else {
    // binary64 throughout, the reference's operation order
    const double thr0 = q.match_lambda * sqrt((double)pre.var0);
    const double thr1 = (r1 == r0) ? thr0 : q.match_lambda * sqrt((double)pre.var1);
    const double mu_top = group_top ? gc.mu : (double)(top1 ? pre.mu1 : pre.mu0);
    const double den = group_top ? gc.thr : (top1 ? thr1 : thr0);
    const double phat = (double)pre.tv / (double)pre.peak;
    const double bterm = s_bt[dv];
    double gterm = fabs(v - mu_top) / den;
    if (gterm > 1.0) gterm = 1.0;
    if (!f.literal) gterm = 1.0 - gterm;
    if (phat < q.prior_floor) {
      const double dd = wb + wc;
      conf = dd > 0.0 ? (wb * bterm + wc * gterm) / dd : 0.0;
    } else {
      conf = wa * phat + wb * bterm + wc * gterm;
    }
    t0 = fabs(v - (double)pre.mu0) <= thr0;
    t1 = fabs(v - (double)pre.mu1) <= thr1;
  }
  double rho = q.learning_rate;
  if (f.rate) {
    double relax = 1.0 - conf;
    if (relax < q.rate_floor) relax = q.rate_floor;
    rho = q.learning_rate * relax;
  }
  const bool hitG = f.grouping && gc.ok && fabs(v - gc.mu) <= gc.thr;
  int active = -1;
  int label = 0;
  if (f.chp && !changed) {
    active = L_CHP;
    label = last_label;
  } else {
    bool done = false;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int code = j == 0 ? c0 : (j == 1 ? c1 : c2);
      if (!done && code == 0) done = true;
      bool hit = (code == L_GROUP) ? hitG : (code == L_MEAN ? t0 : t1);
      const int rr = (code == L_MEAN) ? r0 : r1;
      if (!done && hit && code != L_GROUP && rr > 0) {
        // a matched mode outside the background weight prefix is not a hit
        double acc = 0.0;
        for (int k = 0; k < rr; ++k) acc = acc + ldrw(w_of(pr, p, k));
        hit = acc <= q.background_threshold;
      }
      if (!done && hit) {
        active = code;
        done = true;
      }
    }
    if (active == L_MEAN) {
      st(rec_of(pr, p) + 2 * r0, (1.0 - rho) * (double)pre.mu0 + rho * v);
    } else if (active == L_MEANVAR) {
      o.deep = DEEP_MEANVAR;
      o.rsel = r1;
    } else if (active < 0) {
      active = L_GMM;
      o.deep = DEEP_GMM;
    }
  }

  // ---- streak / sampling bookkeeping (label-independent)
  uint32_t sk = zero_streak ? 0u : pre.streak;
  if (conf > q.confidence_threshold)
    sk = (sk == 0xffffffffu) ? sk : sk + 1u;
  else
    sk = 0u;
  pr.streak[p] = sk;
  atomicAdd(pr.hits + (size_t)active * P + p, 1u);  // RED: no round trip
  if (f.sampling && (long long)sk >= (long long)q.saturation_frames)
    clock = q.sleep_frames;
  o.kind = active;
  o.label = label;
  o.conf = conf;
  o.rho = rho;
  o.dyn = pack_dyn(vb, label, waking, active, clock);
  if (o.deep != DEEP_GMM) pr.dyn[p] = o.dyn;
}

// ---------------------------------------------------------------------------
// Frame tail for one stream: group update, illumination test, stats.
// Runs on one CTA; `acc` holds the stream's summed partials.
// ---------------------------------------------------------------------------
template <typename T>
__device__ double exact_group_conf(const StepArgs& a, int s, int c, int g) {
  // parity/debug mode: the reference's sequential np.bincount order
  const size_t P = (size_t)a.g.height * a.g.width;
  const uint8_t* kind = a.kind + ((size_t)s * a.g.depth + c) * P;
  const T* conf = (const T*)a.conf + ((size_t)s * a.g.depth + c) * P;
  const uint16_t* gid = a.s.gid + (size_t)s * P;
  double acc = 0.0;
  for (size_t p = 0; p < P; ++p)
    if (kind[p] == L_GROUP && gid[p] == (uint16_t)g) acc = acc + (double)conf[p];
  return acc;
}

// ---------------------------------------------------------------------------
// One-shot all-reduce of a row-band shard's frame partials over peer
// mailboxes (include/cog_b200.h, cog_peers).  Both run in ONE CTA, after
// every CTA's contribution has reached `acc` (the caller's done counter).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void st_release_sys(unsigned long long* p,
                                               unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(
    const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys(
    const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// this rank's partials into its slot of every rank's mailbox, then the flags
__device__ void p2p_push(const cog_peers& pr, const unsigned long long* acc,
                         int words) {
  const size_t slot = (size_t)words + 1;
  const size_t off =
      ((size_t)(pr.seq & 1ull) * (size_t)pr.n_ranks + (size_t)pr.rank) * slot;
  for (int r = 0; r < pr.n_ranks; ++r) {
    unsigned long long* dst = (unsigned long long*)pr.mailbox[r] + off;
    for (int i = threadIdx.x; i < words; i += blockDim.x)
      dst[i] = __ldcg(acc + i);
  }
  __threadfence_system();
  __syncthreads();
  if ((int)threadIdx.x < pr.n_ranks)
    st_release_sys((unsigned long long*)pr.mailbox[threadIdx.x] + off + words,
                   pr.seq);
}

// wait for every rank's slot of this step in the own mailbox; acc = their
// sum.  The wait is bounded (P2P_WAIT_NS): a peer that never arrives must
// not hang the GPU -- returns false then (the frame's sums are incomplete;
// the caller flags the frame's stats row)
constexpr unsigned long long P2P_WAIT_NS = 10ull * 1000 * 1000 * 1000;
__device__ bool p2p_wait_sum(const cog_peers& pr, unsigned long long* acc,
                             int words) {
  __shared__ int s_late;
  const size_t slot = (size_t)words + 1;
  const unsigned long long* box = (const unsigned long long*)pr.mailbox[pr.rank] +
                                  (size_t)(pr.seq & 1ull) * (size_t)pr.n_ranks * slot;
  if (threadIdx.x == 0) s_late = 0;
  __syncthreads();
  if ((int)threadIdx.x < pr.n_ranks) {
    const unsigned long long* flag = box + (size_t)threadIdx.x * slot + words;
    unsigned long long t0 = 0, spins = 0;
    while (ld_acquire_sys(flag) != pr.seq) {
      __nanosleep(64);
      if ((++spins & 1023ull) == 0) {
        unsigned long long now;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
        if (t0 == 0) t0 = now;
        else if (now - t0 > P2P_WAIT_NS) {
          s_late = 1;
          break;
        }
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < words; i += blockDim.x) {
    unsigned long long v = 0ull;
    for (int r = 0; r < pr.n_ranks; ++r)
      v += ld_relaxed_sys(box + (size_t)r * slot + i);
    acc[i] = v;
  }
  __threadfence();
  __syncthreads();
  return s_late == 0;
}

template <typename T>
__device__ void finalize_stream(const StepArgs& a, int s,
                                unsigned long long* acc, int64_t* stats,
                                uint32_t* sync) {
  const int d = a.g.depth, G = a.g.n_groups;
  const cog_params& q = a.q;
  __shared__ int s_fired, s_cleared;
  __shared__ long long s_tot[7 * MAXD + 1];
  __syncthreads();
  if (threadIdx.x == 0) s_cleared = __ldcg(acc + acc_flag(d, G)) != 0ull;
  for (int i = threadIdx.x; i <= 7 * d; i += blockDim.x)
    s_tot[i] = (long long)__ldcg(acc + i);
  __syncthreads();
  if (threadIdx.x == 0) {
    long long tot[7] = {0, 0, 0, 0, 0, 0, 0};
    for (int c = 0; c < d; ++c)
      for (int k = 0; k < 7; ++k) tot[k] += s_tot[acc_kind(c, k)];
    long long fg = s_tot[acc_fg(d)];
    double thresh = q.illumination_fraction * (double)a.g.total_pixels *
                    (double)d;
    int fired = (!q.compat && (double)tot[L_GMM] > thresh) ? 1 : 0;
    int64_t* row = stats + (size_t)s * STATS_WORDS;
    row[0] = a.frame_index;
    row[1] = tot[0];
    row[2] = tot[1];
    row[3] = tot[2];
    row[4] = tot[3];
    row[5] = tot[4];
    row[6] = tot[5] + tot[6];
    row[7] = fg;
    row[8] = tot[4];
    row[9] = fired;
    for (int i = 10; i < STATS_WORDS; ++i) row[i] = 0;
    s_fired = fired;
  }
  __syncthreads();
  const int fired = s_fired;
  double* gmu = a.s.g_mu + (size_t)s * d * G;
  double* gvar = a.s.g_var + (size_t)s * d * G;
  for (int it = threadIdx.x; it < d * G; it += blockDim.x) {
    int c = it / G, g = it % G;
    unsigned long long e[6];
#pragma unroll
    for (int j = 0; j < 6; ++j) e[j] = __ldcg(acc + acc_grp(d, G, c, g) + j);
    unsigned long long cnt = e[0];
    if (q.grouping_on && cnt > 0) {
      double cd = (double)cnt;
      double vbar = (double)e[1] / cd;
      double csum = q.exact_group_sums
                        ? exact_group_conf<T>(a, s, c, g)
                        : (double)e[2] * (1.0 / (double)(1ull << CONF_SPLIT)) +
                              (double)e[3] * (1.0 / 4503599627370496.0);
      double cbar = csum / cd;
      double rho = 1.0 - cbar;
      if (rho < q.rate_floor) rho = q.rate_floor;
      rho = q.learning_rate * rho;
      double m = (1.0 - rho) * gmu[it] + rho * vbar;
      double dlt = vbar - m;
      double s2 = (1.0 - rho) * gvar[it] + rho * dlt * dlt;
      gmu[it] = m;
      gvar[it] = s2 < q.variance_floor ? q.variance_floor : s2;
    }
    unsigned long long members = e[5];
    if (fired && members > 0) {
      gmu[it] = (double)e[4] / (double)members;
      gvar[it] = q.initial_variance;
    }
  }
  __syncthreads();
  const int words = acc_words(d, G);
  for (int i = threadIdx.x; i < words; i += blockDim.x) acc[i] = 0ull;
  if (threadIdx.x == 0) {
    // bit 0: pending reset for the next frame; bits 8..15: frames counted
    // into the packed hit bytes (hitq) since they were last cleared -- by
    // this frame's reset / reorder / fold (hot_pending), after which this
    // frame's own hits have been counted
    const uint32_t age = sync[1] >> 8;
    const uint32_t na = s_cleared ? 1u : (age < 0xFFFFu ? age + 1u : age);
    sync[1] = (fired ? 1u : 0u) | (na << 8);
    sync[0] = 0u;               // done counter
    sync[2] = 0u;               // tile counter
    sync[3] = 0u;               // worklist length
  }
}

// ---------------------------------------------------------------------------
// fused per-frame step.  Work unit = a warp tile of `stride` rows x cw
// columns (cw a multiple of the stride), fetched from a per-stream atomic
// counter (dynamic balance).  Every copy pixel's anchor sits in row 0 of
// the same warp tile, so copy resolution is a warp shuffle and the frame
// loop has no block barrier.  Per warp tile:
//   1. hot pass, plane by plane: kinds, confidences, cheap levels and all
//      bookkeeping; MEANVAR hits and GMM fall-throughs are queued
//   2. deep pass: the queued plane-pixels of all planes run densely, one
//      per lane (instead of one divergent pass per plane)
//   3. finish: GMM labels patched in, copies resolved, union mask written
// Partial sums go to warp-private shared slices (plain adds).
// ---------------------------------------------------------------------------
constexpr int STEP_WARPS = STEP_THREADS / 32;
constexpr int QCAP = 32 * MAXD;
// worklist slots per stream: every plane-pixel at most once per frame
__host__ __device__ inline size_t dq_capacity(int d, size_t P) {
  return (size_t)d * P;
}

// bterm tables |v - prev| / 255 (literal) and 1 - that (reference form,
// kernels_numba.py:255-257), computed once on the host in IEEE binary64
// (correctly rounded, as the device division) and uploaded per device, so
// no CTA spends its prologue on 256 binary64 divisions
__device__ double g_bterm[2][256];

// worklist item code (u64): valid | deep << 1 | rsel << 3 | plane << 6 |
// v << 8 | p << 16 (32 bits) | copy mask << 48 (15 bits) | deferred << 63;
// the copy mask and the deferred flag come from the float32 hot pass only
constexpr int ITEM_COPY_SHIFT = 48;
constexpr unsigned long long ITEM_DEFERRED = 1ull << 63;

constexpr int WQ_CAP = 128;  // warp-private worklist buffer (flushed when full)

struct WarpScratch {  // one per warp, in dynamic shared memory
  uint32_t qcode[QCAP];
  double qrho[QCAP];
  uint32_t dw[MAXD][32];
  uint32_t glab[32];
  unsigned long long wq_code[WQ_CAP];
  double wq_rho[WQ_CAP];
};

// move the warp's buffered worklist items to the stream's global worklist
// (one atomic per flush)
__device__ __forceinline__ void flush_wq(WarpScratch& ws, int& wq_n,
                                         uint32_t* counter,
                                         unsigned long long* dq_code,
                                         double* dq_rho, int lane) {
  __syncwarp();
  unsigned base = 0;
  if (lane == 0) base = atomicAdd(counter, (unsigned)wq_n);
  base = __shfl_sync(0xffffffffu, base, 0);
  for (int e = lane; e < wq_n; e += 32) {
    dq_code[(size_t)base + e] = ws.wq_code[e];
    dq_rho[(size_t)base + e] = ws.wq_rho[e];
  }
  __syncwarp();
  wq_n = 0;
}

// ---------------------------------------------------------------------------
// Per-tile work shared by both step kernels.  `fill(c, pre)` provides plane
// c's preloaded values (global loads or shared-memory stages).
// ---------------------------------------------------------------------------
struct TileCtx {
  int s, d, G, lane, it, ty, tx, col, stride, cw, W;
  size_t P, p;
  bool valid, on_lat, member;
  int gid, cls;
};

struct StepShared {
  const double* bt;
  const double* gmu;
  const double* gthr;
  unsigned long long* wacc;
  WarpScratch* ws;
  uint32_t* lk;            // lane-private kind counts [d*7][32]
  uint32_t* lg;            // lane-private group sums [d*G][4][32] (or null)
  unsigned long long* lq;  // lane-private group conf sums [d*G][32]
};

// lane-private group partials only while they stay small
constexpr int LANE_GROUP_SLOTS = 16;  // d * G

__host__ __device__ inline size_t lane_acc_bytes(int d, int G) {
  size_t b = (size_t)d * 7 * 32 * 4;
  if (d * G <= LANE_GROUP_SLOTS) b += (size_t)d * G * 32 * (4 * 4 + 8);
  return b;
}

template <typename T, int KMAX, typename Fill>
__device__ __forceinline__ void tile_pass(const StepArgs& a, const Flags& f,
                                          const TileCtx& t, const StepShared& sh,
                                          unsigned& row0_lbl, int& wq_n,
                                          unsigned long long& fg_count,
                                          unsigned long long* dq_code,
                                          double* dq_rho, uint32_t* sync,
                                          Fill fill) {
  const int s = t.s, d = t.d, G = t.G, lane = t.lane, it = t.it;
  const size_t P = t.P, p = t.p;
  const bool valid = t.valid, member = t.member;
  const int gid = t.gid;
  WarpScratch& ws = *sh.ws;
  T* confo = (T*)a.conf + (size_t)s * d * P;
  uint8_t* kindo = a.kind + (size_t)s * d * P;
  const GmmPar gp{a.q.match_lambda, a.q.background_threshold,
                  a.q.variance_floor, a.q.initial_variance};
  double wa = 0.0, wb = 0.0, wc = 0.0;
  if (valid) {
    wa = a.q.weights[3 * t.cls];
    wb = a.q.weights[3 * t.cls + 1];
    wc = a.q.weights[3 * t.cls + 2];
  }
  unsigned lbits = 0, copybits = 0, gmmbits = 0, latebits = 0;
  int nq = 0;
  ws.glab[lane] = 0u;

  // ---- 1. hot pass, plane by plane
#pragma unroll 1
  for (int c = 0; c < d; ++c) {
    const PlaneRef<T> pr = plane_ref<T>(a, s, c);
    HotOut o;
    o.kind = 0;
    o.label = 0;
    o.deep = DEEP_NONE;
    o.conf = 0.0;
    o.rho = 0.0;
    o.rsel = 0;
    o.dyn = 0;
    Pre<T> pre;
    fill(c, pre);
    if (valid) {
      GroupConst gc;
      gc.ok = member;
      gc.mu = member ? sh.gmu[c * G + gid] : 0.0;
      gc.thr = member ? sh.gthr[c * G + gid] : 0.0;
      hot_px<T>(a, f, pr, p, pre, t.on_lat, sh.bt, wa, wb, wc, gc, o);
      st(confo + (size_t)c * P + p, o.conf);
      kindo[(size_t)c * P + p] = (uint8_t)o.kind;
    }
    const int vb = pre.vb;
    lbits |= ((unsigned)o.label & 1u) << c;
    if (o.kind == K_COPY && valid) {
      copybits |= 1u << c;
      ws.dw[c][lane] = o.dyn;
    }
    const bool labeled_later = valid && (o.deep == DEEP_GMM ||
                                         o.deep == DEEP_COMPAT);
    if (labeled_later) {
      gmmbits |= 1u << c;
      ws.dw[c][lane] = o.dyn;
    }
    // deep work: in-warp when this plane has copy pixels (their anchors
    // need final labels now), else onto the stream's global worklist
    const bool dq = valid && o.deep != DEEP_NONE;
    const unsigned qm = __ballot_sync(FULL, dq);
    const bool inline_plane =
        __ballot_sync(FULL, valid && o.kind == K_COPY) != 0u;
    if (qm && inline_plane) {
      if (dq) {
        const int pos = nq + __popc(qm & ((1u << lane) - 1u));
        ws.qcode[pos] = (uint32_t)lane | ((uint32_t)c << 5) |
                        ((uint32_t)o.deep << 7) | ((uint32_t)o.rsel << 9) |
                        ((uint32_t)vb << 12);
        ws.qrho[pos] = o.rho;
      }
      nq += __popc(qm);
    } else if (qm) {
      if (wq_n + __popc(qm) > WQ_CAP)
        flush_wq(ws, wq_n, sync + 3, dq_code, dq_rho, lane);
      if (dq) {
        const int pos = wq_n + __popc(qm & ((1u << lane) - 1u));
        ws.wq_code[pos] = 1ull | ((unsigned long long)o.deep << 1) |
                          ((unsigned long long)o.rsel << 3) |
                          ((unsigned long long)c << 6) |
                          ((unsigned long long)vb << 8) |
                          ((unsigned long long)p << 16);
        ws.wq_rho[pos] = o.rho;
        gmmbits &= ~((unsigned)labeled_later << c);  // label patched later
        if (labeled_later) latebits |= 1u << c;
      }
      wq_n += __popc(qm);
    }

    // ---- per-plane partial sums (label-independent), lane-private
    if (valid) sh.lk[(c * 7 + o.kind) * 32 + lane] += 1u;
    if (sh.lg) {
      if (member) {
        const int slot = c * G + gid;
        uint32_t* e = sh.lg + slot * 4 * 32 + lane;
        e[0] += (uint32_t)vb;   // sum v over all members
        e[32] += 1u;            // member count
        if (o.kind == L_GROUP) {
          e[64] += 1u;          // hit count
          e[96] += (uint32_t)vb;
          const double cq = o.conf * 4503599627370496.0;  // 2^52
          sh.lq[slot * 32 + lane] += cq > 0.0 ? (unsigned long long)cq : 0ull;
        }
      }
      continue;
    }
    unsigned todo = __ballot_sync(FULL, member);
    while (todo) {
      const int leader = __ffs(todo) - 1;
      const int g = __shfl_sync(FULL, gid, leader);
      const bool mine = member && gid == g;
      const unsigned mm = __ballot_sync(FULL, mine);
      todo &= ~mm;
      const unsigned sall = warp_sum_u32(mine ? (unsigned)vb : 0u);
      const bool hit = mine && o.kind == L_GROUP;
      const unsigned hm = __ballot_sync(FULL, hit);
      unsigned sv = 0, q2 = 0, q1 = 0, q0 = 0;
      if (hm) {
        unsigned long long qv = 0;
        if (hit) {
          const double cq = o.conf * 4503599627370496.0;  // 2^52
          qv = cq > 0.0 ? (unsigned long long)cq : 0ull;
        }
        sv = warp_sum_u32(hit ? (unsigned)vb : 0u);
        q2 = warp_sum_u32((unsigned)(qv >> 40));
        q1 = warp_sum_u32((unsigned)((qv >> 20) & 0xFFFFFu));
        q0 = warp_sum_u32((unsigned)(qv & 0xFFFFFu));
      }
      if (lane == 0) {
        unsigned long long* e = sh.wacc + acc_grp(d, G, c, g);
        e[4] += sall;
        e[5] += (unsigned long long)__popc(mm);
        if (hm) {
          const unsigned long long Q = ((unsigned long long)q2 << 40) +
                                       ((unsigned long long)q1 << 20) +
                                       (unsigned long long)q0;
          e[0] += (unsigned long long)__popc(hm);
          e[1] += sv;
          e[2] += Q >> CONF_SPLIT;
          e[3] += Q & ((1ull << CONF_SPLIT) - 1ull);
        }
      }
    }
  }

  // ---- 2. in-warp deep pass (planes with copy pixels only)
  __syncwarp();
  for (int e = lane; e < nq; e += 32) {
    const uint32_t code = ws.qcode[e];
    const int owner = code & 31, c = (code >> 5) & 3;
    const int kindq = (code >> 7) & 3, rs = (code >> 9) & 7;
    const double v = (double)((code >> 12) & 0xFF);
    const int oidx = it * 32 + owner;
    const int orow = oidx / t.cw, ocol = oidx - orow * t.cw;
    const size_t op =
        (size_t)(t.ty * t.stride + orow) * t.W + (t.tx * t.cw + ocol);
    const PlaneRef<T> pr = plane_ref<T>(a, s, c);
    const uint32_t meta = pr.meta[op];
    if (kindq == DEEP_MEANVAR) {
      cold_meanvar<T, KMAX>(pr, op, meta, rs, v, ws.qrho[e],
                            a.q.variance_floor);
    } else {
      const int lbl = cold_gmm<T, KMAX>(pr, op, meta, v, ws.qrho[e], gp,
                                        a.g.k, kindq == DEEP_GMM);
      if (lbl) atomicOr(&ws.glab[owner], 1u << c);
    }
  }
  __syncwarp();

  // ---- 3. finish: GMM labels, copy resolution, union mask
  const unsigned glab = ws.glab[lane];
  int fg = 0;
#pragma unroll 1
  for (int c = 0; c < d; ++c) {
    int label = (int)((lbits >> c) & 1u);
    if ((gmmbits >> c) & 1u) {
      label = (int)((glab >> c) & 1u);
      a.s.dyn[((size_t)s * d + c) * P + p] =
          ws.dw[c][lane] | ((uint32_t)label << 8);
    } else if ((latebits >> c) & 1u) {
      // the deep kernel sets the label bit (and the mask) if foreground
      label = 0;
      a.s.dyn[((size_t)s * d + c) * P + p] = ws.dw[c][lane];
    }
    const int src = (it == 0) ? label : (int)((row0_lbl >> c) & 1u);
    const int al = __shfl_sync(FULL, src, t.col - t.col % t.stride);
    if ((copybits >> c) & 1u) {
      label = al;
      a.s.dyn[((size_t)s * d + c) * P + p] =
          ws.dw[c][lane] | ((uint32_t)al << 8);
    }
    if (it == 0) row0_lbl |= ((unsigned)label & 1u) << c;
    fg |= label;
  }
  if (valid) a.mask[(size_t)s * P + p] = fg ? 255 : 0;
  fg_count += __popc(__ballot_sync(FULL, valid && fg));
  __syncwarp();
}

// shared prologue: constant tables, group constants, partial slices
struct StepSmem {
  double* bt;
  double* gmu;
  double* gthr;
  unsigned long long* acc_all;
  WarpScratch* ws;
  uint32_t* lane;        // lane-private partials, lane_bytes per warp
  size_t lane_bytes;
};

__device__ __forceinline__ StepShared step_shared(const StepSmem& m, int warp,
                                                  int d, int G, int words) {
  StepShared sh;
  sh.bt = m.bt;
  sh.gmu = m.gmu;
  sh.gthr = m.gthr;
  sh.wacc = m.acc_all + warp * words;
  sh.ws = m.ws + warp;
  uint32_t* base = (uint32_t*)((unsigned char*)m.lane + warp * m.lane_bytes);
  sh.lk = base;
  sh.lg = nullptr;
  sh.lq = nullptr;
  if (d * G <= LANE_GROUP_SLOTS && G > 0) {
    sh.lg = base + d * 7 * 32;
    sh.lq = (unsigned long long*)(sh.lg + d * G * 4 * 32);
  }
  return sh;
}

// fold the lane-private partials into the warp slice (end of kernel)
__device__ __forceinline__ void fold_lane_partials(const StepShared& sh, int d,
                                                   int G, int lane) {
  __syncwarp();
  for (int i = lane; i < d * 7; i += 32) {
    unsigned long long t = 0;
    for (int l = 0; l < 32; ++l) t += sh.lk[i * 32 + l];
    sh.wacc[acc_kind(i / 7, i % 7)] += t;
  }
  if (sh.lg) {
    for (int slot = lane; slot < d * G; slot += 32) {
      unsigned long long sv = 0, cn = 0, hc = 0, hv = 0, cq = 0;
      for (int l = 0; l < 32; ++l) {
        const uint32_t* e = sh.lg + slot * 4 * 32 + l;
        sv += e[0];
        cn += e[32];
        hc += e[64];
        hv += e[96];
        cq += sh.lq[slot * 32 + l];
      }
      unsigned long long* g = sh.wacc + acc_grp(d, G, slot / G, slot % G);
      g[0] += hc;
      g[1] += hv;
      g[2] += cq >> CONF_SPLIT;
      g[3] += cq & ((1ull << CONF_SPLIT) - 1ull);
      g[4] += sv;
      g[5] += cn;
    }
  }
  __syncwarp();
}

__device__ __forceinline__ StepSmem step_prologue(const StepArgs& a,
                                                  const Flags& f, int warps,
                                                  double* s_mem) {
  const int s = blockIdx.y, d = a.g.depth, G = a.g.n_groups;
  const int words = acc_words(d, G);
  StepSmem m;
  m.bt = s_mem;
  m.gmu = s_mem + 256;
  m.gthr = m.gmu + d * G;
  m.acc_all = (unsigned long long*)(m.gthr + d * G);
  m.ws = (WarpScratch*)(m.acc_all + warps * words);
  m.lane = (uint32_t*)(m.ws + warps);
  m.lane_bytes = lane_acc_bytes(d, G);
  for (size_t i = threadIdx.x; i < (size_t)warps * m.lane_bytes / 4;
       i += blockDim.x)
    m.lane[i] = 0u;
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    const double b = (double)i / 255.0;
    m.bt[i] = f.literal ? b : 1.0 - b;
  }
  const double* gmu = a.s.g_mu + (size_t)s * d * G;
  const double* gvar = a.s.g_var + (size_t)s * d * G;
  for (int i = threadIdx.x; i < d * G; i += blockDim.x) {
    m.gmu[i] = gmu[i];
    m.gthr[i] = a.q.match_lambda * sqrt(gvar[i]);
  }
  for (int i = threadIdx.x; i < warps * words; i += blockDim.x)
    m.acc_all[i] = 0ull;
  __syncthreads();
  return m;
}

__device__ __forceinline__ void step_publish(const StepArgs& a,
                                             const StepSmem& m, int warps) {
  const int s = blockIdx.y;
  const int words = acc_words(a.g.depth, a.g.n_groups);
  __syncthreads();
  unsigned long long* gacc =
      (unsigned long long*)a.s.accum + (size_t)s * words;
  for (int i = threadIdx.x; i < words; i += blockDim.x) {
    unsigned long long v = 0;
    for (int w = 0; w < warps; ++w) v += m.acc_all[w * words + i];
    if (v) atomicAdd(gacc + i, v);
  }
}

#ifndef COG_STEP_MINB
#define COG_STEP_MINB 2
#endif

// ---------------------------------------------------------------------------
// general step kernel: any stride / geometry; plane state loaded from global
// memory (the next plane's first round issued before the current plane).
// ---------------------------------------------------------------------------
template <typename T, int KMAX>
__global__ void __launch_bounds__(STEP_THREADS, COG_STEP_MINB)
    step_kernel(const StepArgs a) {
  extern __shared__ double s_mem[];
  const Flags f{a.q.sampling_on != 0, a.q.grouping_on != 0,
                a.q.rate_scaling_on != 0, a.q.chp_on != 0,
                a.q.literal_conf != 0, a.q.compat != 0};
  const StepSmem m = step_prologue(a, f, STEP_WARPS, s_mem);
  const int s = blockIdx.y;
  const int d = a.g.depth, G = a.g.n_groups;
  const int H = a.g.height, W = a.g.width, stride = a.g.stride;
  const size_t P = (size_t)H * W;
  const int words = acc_words(d, G);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const StepShared sh = step_shared(m, warp, d, G, words);
  uint32_t* sync = a.s.sync + (size_t)s * 4;
  const bool do_reset = (*(volatile uint32_t*)(sync + 1) & 1u) != 0;
  const bool do_reorder = a.reorder_now != 0;
  const uint8_t* frame = a.frame + (size_t)s * d * P;
  const uint8_t* cls = a.s.cls + (size_t)s * P;
  const uint16_t* gidp = a.s.gid + (size_t)s * P;
  const int cw = a.cw, npx = stride * cw;
  unsigned long long fg_count = 0;
  const size_t dq_cap = dq_capacity(d, P);
  unsigned long long* dq_code = (unsigned long long*)a.s.deepq + (size_t)s * dq_cap;
  double* dq_rho = a.s.deeprho + (size_t)s * dq_cap;
  int wq_n = 0;

  // tile indices from a per-stream counter, fetched one tile ahead
  int next_wt = 0;
  if (lane == 0) next_wt = (int)atomicAdd(sync + 2, 1u);
  for (;;) {
    const int wt = __shfl_sync(FULL, next_wt, 0);
    if (wt >= a.n_tiles) break;
    if (lane == 0) next_wt = (int)atomicAdd(sync + 2, 1u);
    unsigned row0_lbl = 0;
    TileCtx t;
    t.s = s; t.d = d; t.G = G; t.lane = lane; t.stride = stride;
    t.cw = cw; t.W = W; t.P = P;
    t.ty = wt / a.tiles_x;
    t.tx = wt - t.ty * a.tiles_x;
    for (int it = 0; it < a.iters; ++it) {
      const int idx = it * 32 + lane;
      const int r = idx / cw;
      t.it = it;
      t.col = idx - r * cw;
      const int y = t.ty * stride + r, x = t.tx * cw + t.col;
      t.valid = (idx < npx) && (y < H) && (x < W);
      t.p = t.valid ? (size_t)y * W + x : 0;
      t.on_lat = ((a.g.row0 + y) % stride == 0) && (x % stride == 0);
      t.gid = (int)UNGROUPED;
      t.cls = 0;
      if (t.valid) {
        t.gid = gidp[t.p];
        t.cls = cls[t.p];
      }
      t.member = t.valid && G > 0 && t.gid != (int)UNGROUPED;
      // pending illumination reset / scheduled reorder (rare)
      if (t.valid && (do_reset || do_reorder)) {
#pragma unroll 1
        for (int c = 0; c < d; ++c) {
          const PlaneRef<T> pr = plane_ref<T>(a, s, c);
          if (do_reset) cold_reset<T, KMAX>(pr, t.p, a.q.initial_variance);
          if (do_reorder)
            cold_reorder<T>(pr, t.p, t.member ? m.gmu[c * G + t.gid]
                                              : (G > 0 ? m.gmu[c * G] : 0.0));
        }
      }
      const size_t p = t.p;
      const bool valid = t.valid, on_lat = t.on_lat;
      // first-round loads of plane c+1 are issued before plane c is
      // evaluated (the callback runs once per plane, in order)
      Pre<T> nxt;
      nxt.vb = 0;
      nxt.dyn = nxt.meta = nxt.streak = 0u;
      nxt.peak = 1.0f;
      if (valid) preload_r1<T>(plane_ref<T>(a, s, 0), p, frame, nxt);
      tile_pass<T, KMAX>(
          a, f, t, sh, row0_lbl, wq_n, fg_count, dq_code, dq_rho, sync,
          [&](int c, Pre<T>& pre) {
            pre = nxt;
            nxt.vb = 0;
            nxt.dyn = nxt.meta = nxt.streak = 0u;
            nxt.peak = 1.0f;
            if (valid && c + 1 < d)
              preload_r1<T>(plane_ref<T>(a, s, c + 1), p,
                            frame + (size_t)(c + 1) * P, nxt);
            pre.tv = 0.0f;
            pre.mu0 = pre.mu1 = (T)0;
            pre.var0 = pre.var1 = (T)1;
            if (!valid) return;
            preload_r2<T>(plane_ref<T>(a, s, c), p, f.sampling, f.compat,
                          on_lat, a.q.chp_epsilon, pre);
          });
    }
  }
  if (wq_n) flush_wq(*sh.ws, wq_n, sync + 3, dq_code, dq_rho, lane);
  fold_lane_partials(sh, d, G, lane);
  if (lane == 0) sh.wacc[acc_fg(d)] += fg_count;
  step_publish(a, m, STEP_WARPS);
}

// ---------------------------------------------------------------------------
// deep kernel: the stream's worklist of MEANVAR hits and GMM fall-throughs,
// one plane-pixel per thread (dense warps).  GMM labels are OR-ed into the
// dyn word and the mask; a pixel turning foreground here is counted exactly
// once (atomicOr on its mask word returns the previous byte).  The last CTA
// of each stream finalizes the frame.
// ---------------------------------------------------------------------------
// One worklist item (a MEANVAR hit or a GMM fall-through of one plane-pixel,
// kernels_numba.py:312-342): full binary64 mixture update, stable re-sort,
// mode references remapped.  A GMM label sets the label bit in dyn and --
// unless the mask is formed by a union pass -- ORs the pixel's mask byte;
// returns 1 iff that byte went 0 -> 255 (counted once per pixel).
// A label that only becomes known in the deep pass (GMM fall-through,
// deferred plane-pixel): the label bit of dyn and the mask byte of pixel p
// and of the copy pixels that read their label from it (cmask: bit b is the
// pixel b + 1 of the anchor's stride x stride block in row-major order,
// kernels_numba.py:363-373).  Returns how many mask bytes went 0 -> 255.
__device__ __forceinline__ unsigned or_mask_byte(uint8_t* m) {
  const uintptr_t addr = (uintptr_t)m;
  unsigned* word = (unsigned*)(addr & ~(uintptr_t)3);
  const unsigned sh = (unsigned)(addr & 3) * 8;
  const unsigned old = atomicOr(word, 0xFFu << sh);
  return ((old >> sh) & 0xFFu) == 0u;
}

__device__ __noinline__ unsigned late_label(const StepArgs& a, int s, int c,
                                            size_t p, unsigned cmask) {
  const size_t P = (size_t)a.g.height * a.g.width;
  uint32_t* dyn = a.s.dyn + ((size_t)s * a.g.depth + c) * P;
  uint8_t* mask = a.mask + (size_t)s * P;
  dyn[p] |= 1u << 8;
  unsigned newly = or_mask_byte(mask + p);
  const int st = a.g.stride;
  for (int b = 0; cmask; ++b, cmask >>= 1) {
    if (!(cmask & 1u)) continue;
    const int idx = b + 1, r = idx / st, dc = idx - r * st;
    const size_t q = p + (size_t)r * a.g.width + dc;
    dyn[q] |= 1u << 8;
    newly += or_mask_byte(mask + q);
  }
  return newly;
}

template <typename T, int KMAX>
__device__ __forceinline__ unsigned deep_item(const StepArgs& a, int s,
                                              unsigned long long code,
                                              double rho) {
  const size_t P = (size_t)a.g.height * a.g.width;
  const GmmPar gp{a.q.match_lambda, a.q.background_threshold,
                  a.q.variance_floor, a.q.initial_variance};
  const int kindq = (int)((code >> 1) & 3), rs = (int)((code >> 3) & 7);
  const int c = (int)((code >> 6) & 3);
  const double v = (double)((code >> 8) & 0xFF);
  const size_t p = (size_t)((code >> 16) & 0xFFFFFFFFull);
  const PlaneRef<T> pr = plane_ref<T>(a, s, c);
  // meta and the whole mixture record in one round of loads
  const uint32_t meta = pr.meta[p];
  Mix<KMAX> x;
  T e[rec_elems(KMAX)];
  load_mix_r<T, KMAX>(pr, p, meta_count(meta), x, e);
  int n = meta_count(meta);
  int inv[KMAX];
  unsigned newly = 0;
  if (kindq == DEEP_MEANVAR) {
#pragma unroll
    for (int k = 0; k < KMAX; ++k) {
      if (k == rs) {
        const double mm = (1.0 - rho) * x.mu[k] + rho * v;
        x.mu[k] = mm;
        const double dd = v - mm;
        double s2 = (1.0 - rho) * x.var[k] + rho * (dd * dd);
        if (s2 < a.q.variance_floor) s2 = a.q.variance_floor;
        x.var[k] = s2;
      }
    }
    sort_modes<KMAX>(x, n, inv);
    store_mix_r<T, KMAX>(pr, p, n, x, e);
    pr.meta[p] = (uint16_t)meta_with_refs(
        meta, select_inv<KMAX>(inv, meta_ref(meta, 0)),
        select_inv<KMAX>(inv, meta_ref(meta, 1)));
  } else {
    const int lbl = gmm_step<KMAX>(x, n, a.g.k, v, rho, gp, inv);
    store_mix_r<T, KMAX>(pr, p, n, x, e);
    uint32_t nm = meta_with_count(meta, n);
    if (kindq == DEEP_GMM)
      nm = meta_with_refs(nm, select_inv<KMAX>(inv, meta_ref(meta, 0)),
                          select_inv<KMAX>(inv, meta_ref(meta, 1)));
    pr.meta[p] = (uint16_t)nm;
    if (lbl) newly = late_label(a, s, c, p, (unsigned)(code >> 48) & 0x7FFFu);
  }
  return newly;
}

// ---------------------------------------------------------------------------
// float32-state worklist item in fp32 arithmetic.  The mixture is stored in
// fp32, so the binary64 update of deep_item only differs from this one in
// the last bits of the stored values (within the fp32 tolerance); every
// DECISION -- the match test, the background prefix of the label, the
// order of the re-sort -- is filtered: one whose fp32 operands lie within a
// 1e-5 relative margin makes the item fall back to the binary64 deep_item
// (nothing is written before that), so decisions are the reference's
// (kernels_numba.py:76-134, 312-334).  It replaces ~25 binary64 divisions
// and square roots per item by single-instruction approximations, which
// matters when the worklist is long (busy scenes, C5).
// ---------------------------------------------------------------------------
__device__ __forceinline__ float d32_rsqrt(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float d32_rcp(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// stable descending order by w / sqrt(var); false on a near tie.  The
// mixture was sorted before the update and an update moves one mode's key,
// so nearly always the order stands: `same` = every adjacent pair is still
// in order by more than the margin (inv is the identity, nothing moves)
template <int KMAX>
__device__ __forceinline__ bool d32_sort(float (&mu)[KMAX], float (&var)[KMAX],
                                         float (&w)[KMAX], int n,
                                         int (&inv)[KMAX], bool& same) {
  float key[KMAX];
#pragma unroll
  for (int k = 0; k < KMAX; ++k)
    key[k] = k < n ? w[k] * d32_rsqrt(var[k]) : 0.0f;
  same = true;
#pragma unroll
  for (int k = 0; k + 1 < KMAX; ++k)
    if (k + 1 < n)
      same &= key[k] - key[k + 1] >
              1e-5f * fmaxf(fabsf(key[k]), fabsf(key[k + 1])) + 1e-30f;
#pragma unroll
  for (int k = 0; k < KMAX; ++k) inv[k] = k;
  if (same) return true;
  bool ok = true;
#pragma unroll
  for (int i = 0; i < KMAX; ++i) {
    int r = i;
    if (i < n) {
      r = 0;
#pragma unroll
      for (int j = 0; j < KMAX; ++j) {
        if (j < n && j != i) {
          ok &= fabsf(key[j] - key[i]) >
                1e-5f * fmaxf(fabsf(key[j]), fabsf(key[i])) + 1e-30f;
          r += (key[j] > key[i]);
        }
      }
    }
    inv[i] = r;
  }
  if (!ok) return false;
  float m2[KMAX], v2[KMAX], w2[KMAX];
#pragma unroll
  for (int t = 0; t < KMAX; ++t) {
    m2[t] = mu[t];
    v2[t] = var[t];
    w2[t] = w[t];
  }
#pragma unroll
  for (int i = 0; i < KMAX; ++i)
#pragma unroll
    for (int t = 0; t < KMAX; ++t)
      if (i < n && inv[i] == t) {
        m2[t] = mu[i];
        v2[t] = var[i];
        w2[t] = w[i];
      }
#pragma unroll
  for (int t = 0; t < KMAX; ++t) {
    mu[t] = m2[t];
    var[t] = v2[t];
    w[t] = w2[t];
  }
  return true;
}

// returns 1 if the pixel's mask byte went 0 -> 255; ok = false: undecided
// in fp32, nothing written (the caller runs deep_item)
template <int KMAX>
__device__ __forceinline__ unsigned deep_item_f32(const StepArgs& a, int s,
                                                  unsigned long long code,
                                                  double rho_d, bool& ok) {
  const size_t P = (size_t)a.g.height * a.g.width;
  const int kindq = (int)((code >> 1) & 3), rs = (int)((code >> 3) & 7);
  const int c = (int)((code >> 6) & 3);
  const float v = (float)((code >> 8) & 0xFF);
  const size_t p = (size_t)((code >> 16) & 0xFFFFFFFFull);
  const PlaneRef<float> pr = plane_ref<float>(a, s, c);
  const uint32_t meta = pr.meta[p];
  constexpr int R = rec_elems(KMAX), WO = rec_w(KMAX);
  float e[R];
  rec_load<R>(rec_of(pr, p), e);
  float mu[KMAX], var[KMAX], w[KMAX];
#pragma unroll
  for (int k = 0; k < KMAX; ++k) {
    mu[k] = e[2 * k];
    var[k] = e[2 * k + 1];
    w[k] = e[WO + k];
    if (k >= a.g.k) {
      mu[k] = 0.0f;
      var[k] = 1.0f;
      w[k] = 0.0f;
    }
  }
  int n = meta_count(meta);
  const float rho = (float)rho_d, om = 1.0f - rho;
  const float lam = (float)a.q.match_lambda;
  const float vfloor = (float)a.q.variance_floor;
  int label = 0;
  ok = true;
  if (kindq == DEEP_MEANVAR) {
#pragma unroll
    for (int k = 0; k < KMAX; ++k) {
      if (k == rs) {
        const float mm = om * mu[k] + rho * v;
        const float dd = v - mm;
        mu[k] = mm;
        var[k] = fmaxf(om * var[k] + rho * (dd * dd), vfloor);
      }
    }
  } else {
    // match: first live mode within lam * sigma (filtered)
    int hit = -1;
#pragma unroll
    for (int k = 0; k < KMAX; ++k) {
      if (hit < 0 && ok && k < n) {
        const float thr = lam * (var[k] * d32_rsqrt(var[k]));
        const float gap = fabsf(v - mu[k]) - thr;
        const float m = 1e-5f * thr + 3e-5f;
        if (gap < -m)
          hit = k;
        else if (gap <= m)
          ok = false;
      }
    }
    if (!ok) return 0;
    if (hit >= 0) {
      float sw = 0.0f;
#pragma unroll
      for (int k = 0; k < KMAX; ++k) {
        if (k < n) {
          w[k] = om * w[k] + (k == hit ? rho : 0.0f);
          sw += w[k];
        }
      }
      const float rsw = d32_rcp(sw);
      float acc = 0.0f;
      int b = n;
      bool found = false;
      const float tbg = (float)a.q.background_threshold;
#pragma unroll
      for (int k = 0; k < KMAX; ++k) {
        if (k < n) {
          w[k] *= rsw;
          if (k == hit) {
            const float mm = om * mu[k] + rho * v;
            const float dd = v - mm;
            mu[k] = mm;
            var[k] = fmaxf(om * var[k] + rho * (dd * dd), vfloor);
          }
          if (!found) {
            acc += w[k];
            ok &= fabsf(acc - tbg) > 1e-5f * tbg;  // prefix decision
            if (acc > tbg) {
              b = k + 1;
              found = true;
            }
          }
        }
      }
      if (!ok) return 0;
      label = (hit + 1 <= b) ? 0 : 1;
    } else {
      const int slot = n < a.g.k ? n : n - 1;
      if (n < a.g.k) n = n + 1;
      float sw = 0.0f;
#pragma unroll
      for (int k = 0; k < KMAX; ++k) {
        if (k == slot) {
          mu[k] = v;
          var[k] = (float)a.q.initial_variance;
          w[k] = rho;
        }
        if (k < n) sw += w[k];
      }
      if (sw == 0.0f) {
#pragma unroll
        for (int k = 0; k < KMAX; ++k)
          if (k < n) w[k] = (k == slot) ? 1.0f : 0.0f;
      } else {
        const float r_ = d32_rcp(sw);
#pragma unroll
        for (int k = 0; k < KMAX; ++k)
          if (k < n) w[k] *= r_;
      }
      label = 1;
    }
  }
  int inv[KMAX];
  bool same;
  if (!d32_sort<KMAX>(mu, var, w, n, inv, same)) {
    ok = false;
    return 0;
  }
  if (same && kindq == DEEP_MEANVAR) {
    // the order stands: only mode rs changed, the refs stay
    float2 mv = make_float2(0.0f, 1.0f);
#pragma unroll
    for (int k = 0; k < KMAX; ++k)
      if (k == rs) mv = make_float2(mu[k], var[k]);
    *reinterpret_cast<float2*>(rec_of(pr, p) + 2 * rs) = mv;
    return 0;
  }
  // ---- write back (deep_item's bookkeeping): the whole record
#pragma unroll
  for (int k = 0; k < KMAX; ++k) {
    if (k < n) {
      e[2 * k] = mu[k];
      e[2 * k + 1] = var[k];
      e[WO + k] = w[k];
    }
  }
  rec_store<R>(rec_of(pr, p), e);
  if (kindq == DEEP_MEANVAR) {
    pr.meta[p] = (uint16_t)meta_with_refs(
        meta, select_inv<KMAX>(inv, meta_ref(meta, 0)),
        select_inv<KMAX>(inv, meta_ref(meta, 1)));
    return 0;
  }
  uint32_t nm = meta_with_count(meta, n);
  if (kindq == DEEP_GMM)
    nm = meta_with_refs(nm, select_inv<KMAX>(inv, meta_ref(meta, 0)),
                        select_inv<KMAX>(inv, meta_ref(meta, 1)));
  pr.meta[p] = (uint16_t)nm;
  unsigned newly = 0;
  if (label) newly = late_label(a, s, c, p, (unsigned)(code >> 48) & 0x7FFFu);
  return newly;
}

// A plane-pixel the float32 hot pass deferred (an fp32 decision inside its
// filter margin): the general binary64 step of kernels_numba.py:188-359
// (hot_px) from its untouched state, with the exact f32 table entry, then
// everything the hot pass would have done for it -- confidence / kind
// outputs, its kind count and group partials (into the stream's summed
// partials, before the frame tail reads them), the deep update, and its
// label (with its copies').  Returns the mask bytes that went 0 -> 255.
template <int KMAX>
__device__ __noinline__ unsigned deferred_item(const StepArgs& a, int s,
                                               unsigned long long code,
                                               unsigned long long* gacc) {
  using T = float;
  const int D = a.g.depth, G = a.g.n_groups;
  const size_t P = (size_t)a.g.height * a.g.width;
  const int c = (int)((code >> 6) & 3);
  const int vb = (int)((code >> 8) & 0xFF);
  const size_t p = (size_t)((code >> 16) & 0xFFFFFFFFull);
  const unsigned cmask = (unsigned)(code >> 48) & 0x7FFFu;
  const PlaneRef<T> pr = plane_ref<T>(a, s, c);
  const Flags f{a.q.sampling_on != 0, a.q.grouping_on != 0,
                a.q.rate_scaling_on != 0, a.q.chp_on != 0,
                a.q.literal_conf != 0, a.q.compat != 0};
  Pre<T> x;
  x.vb = vb;
  x.dyn = pr.dyn[p];
  x.meta = pr.meta[p];
  x.streak = pr.streak[p];
  x.tv = __ldcg(pr.table + p * 256 + vb);
  x.peak = pr.peak[p];
  {
    const T* rec = rec_of(pr, p);
    const int r0 = meta_ref(x.meta, 0), r1 = meta_ref(x.meta, 1);
    x.mu0 = rec[2 * r0];
    x.var0 = rec[2 * r0 + 1];
    x.mu1 = rec[2 * r1];
    x.var1 = rec[2 * r1 + 1];
  }
  const int W = a.g.width, st = a.g.stride;
  const int y = (int)(p / (size_t)W), xx = (int)(p - (size_t)y * W);
  const bool on_lat = ((a.g.row0 + y) % st == 0) && (xx % st == 0);
  const int cls = a.s.cls[(size_t)s * P + p];
  const int gid = a.s.gid[(size_t)s * P + p];
  const bool member = G > 0 && gid != (int)UNGROUPED;
  GroupConst gc;
  gc.ok = member;
  gc.mu = 0.0;
  gc.thr = 0.0;
  if (member) {
    const size_t gi = ((size_t)s * D + c) * G + gid;
    gc.mu = a.s.g_mu[gi];
    gc.thr = a.q.match_lambda * sqrt(a.s.g_var[gi]);
  }
  HotOut h;
  h.kind = 0;
  h.label = 0;
  h.deep = DEEP_NONE;
  h.conf = 0.0;
  h.rho = 0.0;
  h.rsel = 0;
  h.dyn = 0;
  hot_px<T>(a, f, pr, p, x, on_lat, g_bterm[f.literal ? 1 : 0],
            a.q.weights[3 * cls], a.q.weights[3 * cls + 1],
            a.q.weights[3 * cls + 2], gc, h);
  const size_t o = ((size_t)s * D + c) * P + p;
  ((T*)a.conf)[o] = (T)h.conf;
  a.kind[o] = (uint8_t)h.kind;
  atomicAdd(gacc + acc_kind(0, h.kind), 1ull);
  if (member && h.kind == L_GROUP) {
    unsigned long long* e = gacc + acc_grp(D, G, c, gid);
    const double cq = h.conf * 4503599627370496.0;  // 2^52
    const unsigned long long qv = cq > 0.0 ? (unsigned long long)cq : 0ull;
    atomicAdd(e + 0, 1ull);
    atomicAdd(e + 1, (unsigned long long)vb);
    atomicAdd(e + 2, qv >> CONF_SPLIT);
    atomicAdd(e + 3, qv & ((1ull << CONF_SPLIT) - 1ull));
  }
  int label = h.label;
  if (h.deep == DEEP_MEANVAR) {
    cold_meanvar<T, KMAX>(pr, p, x.meta, h.rsel, (double)vb, h.rho,
                          a.q.variance_floor);
  } else if (h.deep == DEEP_GMM) {
    const GmmPar gp{a.q.match_lambda, a.q.background_threshold,
                    a.q.variance_floor, a.q.initial_variance};
    label = cold_gmm<T, KMAX>(pr, p, x.meta, (double)vb, h.rho, gp, a.g.k, 1);
    pr.dyn[p] = h.dyn;
  }
  return label ? late_label(a, s, c, p, cmask) : 0u;
}

// the binary64 update of a float32 worklist item whose fp32 decision was
// too close to call: out of line, so the fp32 path keeps few registers
template <int KMAX>
__device__ __noinline__ unsigned deep_item_f64_of_f32(const StepArgs* __restrict__ ap,
                                                      int s,
                                                      unsigned long long code,
                                                      double rho) {
  return deep_item<float, KMAX>(*ap, s, code, rho);
}

template <typename T, int KMAX>
__global__ void __launch_bounds__(DEEP_THREADS, DEEP_MINB) deep_kernel(const StepArgs a) {
  __shared__ int s_last;
  __shared__ unsigned long long s_fg;
  // launched with programmatic stream serialization after fast_kernel: wait
  // for its results (a no-op under a normal launch)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int s = blockIdx.y;
  const int d = a.g.depth;
  const size_t P = (size_t)a.g.height * a.g.width;
  uint32_t* sync = a.s.sync + (size_t)s * 4;
  const size_t dq_cap = dq_capacity(d, P);
  unsigned long long* dq_code = (unsigned long long*)a.s.deepq + (size_t)s * dq_cap;
  const double* dq_rho = a.s.deeprho + (size_t)s * dq_cap;
  // hot_kernel's worklist is two-ended (cog_hot.cuh, hot_flush): n_a items
  // at the front, n_b at the back; virtual index i runs over the front
  // items, a gap up to the next warp boundary, then the back items -- so a
  // warp holds one item type.  Every other step kernel fills the front only
  const size_t n_b = *(volatile uint32_t*)(sync + 3);
  const size_t n_a = a.two_ended ? *(volatile uint32_t*)(sync + 2) : n_b;
  const size_t a32 = (n_a + 31) & ~(size_t)31;
  const size_t n = a.two_ended ? a32 + n_b : n_a;
  if (threadIdx.x == 0) s_fg = 0;
  __syncthreads();
  unsigned fg = 0;
  const int words = acc_words(d, a.g.n_groups);
  unsigned long long* gacc =
      (unsigned long long*)a.s.accum + (size_t)s * words;
  // warp-granular round robin over the CTAs (warp 0 of every CTA first):
  // a short worklist spreads over all SMs instead of filling the first
  // few CTAs
  const size_t wpc = blockDim.x >> 5;
  const size_t gw = (size_t)(threadIdx.x >> 5) * gridDim.x + blockIdx.x;
  // Software pipeline over this thread's items (DEEP_AHEAD): the code and
  // rho of the item two rounds ahead are loaded, the mixture record and meta
  // word of the item one round ahead are prefetched into L2, while the
  // current item is processed -- an item's dependent round trips (item ->
  // record -> update) then overlap the previous items' work.
  const size_t vstep = (size_t)gridDim.x * wpc * 32;
  auto item_index = [&](size_t v) -> size_t {
    return v < n_a ? v : dq_cap - 1 - (v - a32);
  };
  auto fetch = [&](size_t v, unsigned long long& code, double& rho) {
    code = 0ull;
    rho = 0.0;
    if (v < n && !(v >= n_a && v < a32)) {
      const size_t i = item_index(v);
      code = dq_code[i];
      rho = dq_rho[i];
    }
  };
  auto prefetch = [&](unsigned long long code) {
    const int c = (int)((code >> 6) & 3);
    const size_t p = (size_t)((code >> 16) & 0xFFFFFFFFull);
    const PlaneRef<T> pr = plane_ref<T>(a, s, c);
    asm volatile("prefetch.global.L2 [%0];" ::"l"(rec_of(pr, p)));
    asm volatile("prefetch.global.L2 [%0];" ::"l"(pr.meta + p));
  };
  size_t vi = gw * 32 + (threadIdx.x & 31);
  unsigned long long code = 0ull, code1 = 0ull;
  double rho = 0.0, rho1 = 0.0;
  fetch(vi, code, rho);
#if DEEP_AHEAD
  fetch(vi + vstep, code1, rho1);
#endif
  for (; vi < n; vi += vstep) {
#if DEEP_AHEAD
    unsigned long long code2;
    double rho2;
    fetch(vi + 2 * vstep, code2, rho2);
    if (code1 & 1ull) prefetch(code1);
#endif
    const unsigned long long cur = code;
    const double cur_rho = rho;
#if DEEP_AHEAD
    code = code1;
    rho = rho1;
    code1 = code2;
    rho1 = rho2;
#else
    fetch(vi + vstep, code, rho);
#endif
    if (!(cur & 1ull)) continue;
    dq_code[item_index(vi)] = 0ull;
    if constexpr (sizeof(T) == 4) {
      if (cur & ITEM_DEFERRED) {
        fg += deferred_item<KMAX>(a, s, cur, gacc);
        continue;
      }
      if (!a.q.compat) {  // fp32 arithmetic, binary64 fallback near ties
        bool ok;
        const unsigned nw = deep_item_f32<KMAX>(a, s, cur, cur_rho, ok);
        if (ok) {
          fg += nw;
          continue;
        }
        fg += deep_item_f64_of_f32<KMAX>(&a, s, cur, cur_rho);
        continue;
      }
    }
    fg += deep_item<T, KMAX>(a, s, cur, cur_rho);
  }
  for (int o = 16; o > 0; o >>= 1) fg += __shfl_xor_sync(FULL, fg, o);
  if ((threadIdx.x & 31) == 0 && fg) atomicAdd(&s_fg, (unsigned long long)fg);
  __syncthreads();
  if (threadIdx.x == 0 && s_fg) atomicAdd(gacc + acc_fg(d), s_fg);
  const bool p2p = a.peers.n_ranks > 1;
  if (!a.fuse_finalize && !p2p) return;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned t = atomicAdd(sync, 1u);
    s_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (p2p) {
    // row-band shard: the partials go to every rank's mailbox from here;
    // fused, this CTA also waits for the other shards' and sums them
    p2p_push(a.peers, gacc, words);
    if (!a.fuse_finalize) return;
    const bool in_time = p2p_wait_sum(a.peers, gacc, words);
    finalize_stream<T>(a, s, gacc, a.stats, sync);
    if (!in_time && threadIdx.x == 0)
      a.stats[(size_t)s * STATS_WORDS + STATS_WORDS - 1] = -1;  // peer missing
    return;
  }
  finalize_stream<T>(a, s, gacc, a.stats, sync);
}

// hot prior of one stream: reference-layout table f32[d][P][256] + peak ->
// tile-major u16 phat (cascade.py:213-216, phat = table / peak in binary64,
// stored as round(phat * 65535)); one thread per entry, coalesced reads
__global__ void tabq_build_kernel(TabGeo tg, int d, size_t P,
                                  const float* __restrict__ table,
                                  const float* __restrict__ peak,
                                  uint16_t* tabq) {
  const size_t n = (size_t)d * P * 256;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const size_t c = i / (P * 256), rem = i - c * P * 256;
    const size_t p = rem >> 8, v = rem & 255;
    const double ph = (double)table[i] / (double)peak[c * P + p];
    double q = rint(ph * 65535.0);
    q = q < 0.0 ? 0.0 : (q > 65535.0 ? 65535.0 : q);
    tabq[c * tg.plane + tab_pix(tg, p) + v * tg.SL] = (uint16_t)q;
  }
}

template <typename T>
__global__ void finalize_kernel(const StepArgs a) {
  const int s = blockIdx.x;
  const int words = acc_words(a.g.depth, a.g.n_groups);
  unsigned long long* acc = (unsigned long long*)a.s.accum + (size_t)s * words;
  bool in_time = true;
  if (a.peers.n_ranks > 1) in_time = p2p_wait_sum(a.peers, acc, words);
  finalize_stream<T>(a, s, acc, a.stats, a.s.sync + (size_t)s * 4);
  if (!in_time && threadIdx.x == 0)
    a.stats[(size_t)s * STATS_WORDS + STATS_WORDS - 1] = -1;  // peer missing
}

template <typename T, int KMAX>
__global__ void __launch_bounds__(256) pending_kernel(const StepArgs a) {
  const int s = blockIdx.y;
  const int d = a.g.depth, G = a.g.n_groups;
  const size_t P = (size_t)a.g.height * a.g.width;
  uint32_t* sync = a.s.sync + (size_t)s * 4;
  const bool do_reset = (*(volatile uint32_t*)(sync + 1) & 1u) != 0;
  const bool do_reorder = a.reorder_now != 0;
  if (!do_reset && !do_reorder) return;
  const double* gmu = a.s.g_mu + (size_t)s * d * G;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < d * P;
       i += (size_t)gridDim.x * blockDim.x) {
    const int c = (int)(i / P);
    const size_t p = i % P;
    const PlaneRef<T> pr = plane_ref<T>(a, s, c);
    if (do_reset) cold_reset<T, KMAX>(pr, p, a.q.initial_variance);
    if (do_reorder) {
      const int gid = a.s.gid[(size_t)s * P + p];
      const double gm = G > 0 ? gmu[(size_t)c * G + (gid == (int)UNGROUPED ? 0 : gid)] : 0.0;
      cold_reorder<T>(pr, p, gm);
    }
  }
}

// clears the pending flag after pending_kernel (separate launch: every CTA
// of pending_kernel must have read the flag first)
__global__ void clear_pending_kernel(uint32_t* sync, int streams,
                                     int reorder_now) {
  int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= streams) return;
  // a reset or a reorder cleared the packed hit bytes too: their age restarts
  const uint32_t v = sync[(size_t)s * 4 + 1];
  if (reorder_now || (v & 1u)) sync[(size_t)s * 4 + 1] = 0u;
}

// ---------------------------------------------------------------------------
// training: prior
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
    prior_kernel(const uint8_t* __restrict__ frames, int N, int d, int64_t P,
                 const double* __restrict__ kern,
                 const int32_t* __restrict__ windows, int nw, float* tables,
                 float* peak, uint16_t* hist_out, double t1, double t2,
                 double peaky, uint32_t* residue, uint8_t* cls) {
  extern __shared__ __align__(16) unsigned char psm[];
  uint8_t* samp = psm;                                          // [N][32]
  uint16_t* hist = (uint16_t*)(psm + (((size_t)N * 32 + 15) & ~(size_t)15));
  const int64_t p0 = (int64_t)blockIdx.x * PRIOR_PIX;
  const int npx = (int)min((int64_t)PRIOR_PIX, P - p0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nwarps = blockDim.x >> 5;
  unsigned rc0 = 0, rc1 = 0, rc2 = 0;

  for (int c = 0; c < d; ++c) {
    for (int e = tid; e < N * 32; e += blockDim.x) {
      int i = e >> 5, t = e & 31;
      samp[e] = (t < npx) ? frames[((size_t)i * d + c) * P + p0 + t] : 0;
    }
    for (int e = tid; e < 256 * 32; e += blockDim.x) hist[e] = 0;
    __syncthreads();
    if (tid < npx) {
      int prev = samp[tid];
      for (int i = 1; i < N; ++i) {
        int cur = samp[i * 32 + tid];
        double rr = (double)abs(cur - prev);
        int b = (rr >= t1) + (rr >= t2);
        rc0 += (b == 0);
        rc1 += (b == 1);
        rc2 += (b == 2);
        prev = cur;
      }
    }
    int prev_w = 0;
    for (int j = 0; j < nw; ++j) {
      const int wj = windows[j];
      if (tid < npx) {
        for (int i = N - wj; i < N - prev_w; ++i)
          hist[samp[i * 32 + tid] * 32 + tid] += 1;
      }
      prev_w = wj;
      __syncthreads();
      const bool last = (j == nw - 1);
      if (last && hist_out) {
        for (int e = tid; e < npx * 256; e += blockDim.x) {
          int t = e >> 8, bin = e & 255;
          hist_out[((size_t)c * P + p0 + t) * 256 + bin] = hist[bin * 32 + t];
        }
      }
      const double inv_n = (double)wj;
      for (int t = warp; t < npx; t += nwarps) {
        double acc[8];
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) acc[jj] = 0.0;
        for (int chunk = 0; chunk < 8; ++chunk) {
          unsigned cnt = hist[(chunk * 32 + lane) * 32 + t];
          unsigned m = __ballot_sync(FULL, cnt != 0);
          while (m) {
            const int b = __ffs(m) - 1;
            m &= m - 1;
            const double cd = (double)__shfl_sync(FULL, cnt, b);
            const double* row = kern + (size_t)(chunk * 32 + b) * 256;
#pragma unroll
            for (int jj = 0; jj < 8; ++jj)
              acc[jj] = acc[jj] + cd * __ldg(row + jj * 32 + lane);
          }
        }
        float mx = 0.0f;
        float* trow = tables + (((size_t)j * d + c) * P + p0 + t) * 256;
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          float fv = (float)(acc[jj] / inv_n);
          trow[jj * 32 + lane] = fv;
          mx = fmaxf(mx, fv);
        }
        if (last) {
#pragma unroll
          for (int o = 16; o > 0; o >>= 1)
            mx = fmaxf(mx, __shfl_xor_sync(FULL, mx, o));
          if (lane == 0) peak[(size_t)c * P + p0 + t] = mx > 0.0f ? mx : 1.0f;
        }
      }
      __syncthreads();
    }
  }
  if (tid < npx) {
    const double den = (double)(N - 1) * (double)d;
    const double o0 = (double)rc0 / den, o1 = (double)rc1 / den;
    uint8_t k = 2;
    if (o1 >= peaky) k = 1;
    if (o0 >= peaky) k = 0;
    cls[p0 + tid] = k;
    if (residue) {
      residue[(p0 + tid) * 3 + 0] = rc0;
      residue[(p0 + tid) * 3 + 1] = rc1;
      residue[(p0 + tid) * 3 + 2] = rc2;
    }
  }
}

// ---------------------------------------------------------------------------
// training: GMM warm-up, adaptation statistics, mode references
// ---------------------------------------------------------------------------
struct WarmArgs {
  cog_geom g;
  cog_params q;
  cog_state s;
  const uint8_t* frames;
  int N;
  double* features;
  double* w_final;
};

template <int KMAX>
__device__ __forceinline__ void warm_init(Mix<KMAX>& m, double v0,
                                          double init_var) {
#pragma unroll
  for (int k = 0; k < KMAX; ++k) {
    m.mu[k] = 0.0;
    m.var[k] = init_var;
    m.w[k] = 0.0;
  }
  m.mu[0] = v0;
  m.w[0] = 1.0;
}

template <typename T, int KMAX>
__global__ void __launch_bounds__(128) warmup_kernel(const WarmArgs a) {
  const int c = blockIdx.y;
  const int d = a.g.depth, K = a.g.k;
  const size_t P = (size_t)a.g.height * a.g.width;
  const size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const GmmPar gp{a.q.match_lambda, a.q.background_threshold,
                  a.q.variance_floor, a.q.initial_variance};
  const double lr = a.q.learning_rate;
  const uint8_t* fr = a.frames;
  const int N = a.N;
  const bool series = (c == 0) && a.features != nullptr;
  Mix<KMAX> m;
  int inv[KMAX];
  int n = 1;
  warm_init<KMAX>(m, (double)fr[(size_t)c * P + p], a.q.initial_variance);
  double sv = m.var[0], sw = m.w[0];
  for (int i = 1; i < N; ++i) {
    double v = (double)fr[((size_t)i * d + c) * P + p];
    gmm_step<KMAX>(m, n, K, v, lr, gp, inv);
    if (series) {
      sv = sv + m.var[0];
      sw = sw + m.w[0];
    }
  }
  if (series) {
    // numpy var(axis=0, ddof=0): sequential mean, then sequential sum of
    // squared deviations -- recompute the series rather than storing it
    const double mv = sv / (double)N, mw = sw / (double)N;
    Mix<KMAX> r;
    int rn = 1;
    warm_init<KMAX>(r, (double)fr[(size_t)c * P + p], a.q.initial_variance);
    double dv = r.var[0] - mv, dw = r.w[0] - mw;
    double qv = dv * dv, qw = dw * dw;
    for (int i = 1; i < N; ++i) {
      double v = (double)fr[((size_t)i * d + c) * P + p];
      gmm_step<KMAX>(r, rn, K, v, lr, gp, inv);
      dv = r.var[0] - mv;
      dw = r.w[0] - mw;
      qv = qv + dv * dv;
      qw = qw + dw * dw;
    }
    a.features[p * 2 + 0] = qv / (double)N;
    a.features[p * 2 + 1] = qw / (double)N;
    if (a.w_final) a.w_final[p] = m.w[0];
  }
  // store the mixture record (dead slots hold the canonical (0, init_var,
  // 0), padding zero)
  {
    T e[rec_elems(KMAX)];
#pragma unroll
    for (int i = 0; i < rec_elems(KMAX); ++i) e[i] = (T)0;
#pragma unroll
    for (int k = 0; k < KMAX; ++k) {
      if (k < K) {
        e[2 * k] = (T)m.mu[k];
        e[2 * k + 1] = (T)m.var[k];
        e[rec_w(KMAX) + k] = (T)m.w[k];
      }
    }
    rec_store<rec_elems(KMAX)>(
        (T*)a.s.mix + ((size_t)c * P + p) * rec_elems(KMAX), e);
  }
  // mode references: lexsort((-tie, -mass)) over all K slots
  // (cascade.py:218-235); dead slots carry (-inf, -inf)
  const float* trow = a.s.table + ((size_t)c * P + p) * 256;
  double nm[KMAX], nt[KMAX];
  const double PINF = __longlong_as_double(0x7ff0000000000000ll);
#pragma unroll
  for (int k = 0; k < KMAX; ++k) {
    nm[k] = PINF;
    nt[k] = PINF;
    if (k < n) {
      nm[k] = -(double)trow[(size_t)clip_rint(m.mu[k])];
      nt[k] = -(m.w[k] / sqrt(m.var[k]));
    }
  }
  int ref0 = 0, ref1 = 0;
#pragma unroll
  for (int i = 0; i < KMAX; ++i) {
    if (i >= K) continue;
    int r = 0;
#pragma unroll
    for (int j = 0; j < KMAX; ++j) {
      if (j >= K) continue;
      bool less = (nm[j] < nm[i]) || (nm[j] == nm[i] && nt[j] < nt[i]);
      bool tie = (nm[j] == nm[i]) && (nt[j] == nt[i]);
      r += less || (j < i && tie);
    }
    if (r == 0) ref0 = i;
    if (r == 1) ref1 = i;
  }
  if (n < 2) ref1 = ref0;
  const size_t pi = (size_t)c * P + p;
  a.s.meta[pi] = (uint16_t)pack_meta(n, L_MEAN, L_MEANVAR, -1, ref0, ref1);
  a.s.dyn[pi] = pack_dyn(fr[((size_t)(N - 1) * d + c) * P + p], 0, 0, -1, 0);
  a.s.streak[pi] = 0u;
#pragma unroll
  for (int l = 0; l < 5; ++l) a.s.hits[((size_t)c * 5 + l) * P + p] = 0u;
  if (a.s.hitq) a.s.hitq[pi] = 0u;
}

__global__ void set_levels_kernel(cog_geom g, uint16_t* meta,
                                  const uint16_t* gid) {
  const size_t P = (size_t)g.height * g.width;
  const size_t total = (size_t)g.streams * g.depth * P;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const size_t s = i / ((size_t)g.depth * P);
    const size_t p = i % P;
    const bool grouped = gid[s * P + p] != UNGROUPED;
    uint32_t m = meta[i];
    meta[i] = (uint16_t)(grouped ? meta_with_mids(m, L_GROUP, L_MEAN, L_MEANVAR)
                                 : meta_with_mids(m, L_MEAN, L_MEANVAR, -1));
  }
}

// ---------------------------------------------------------------------------
// baseline mixture (gmm.classify_frame)
// ---------------------------------------------------------------------------
template <typename T, int KMAX>
__global__ void __launch_bounds__(256) baseline_kernel(const StepArgs a) {
  const int d = a.g.depth, K = a.g.k;
  const size_t P = (size_t)a.g.height * a.g.width;
  const size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const GmmPar gp{a.q.match_lambda, a.q.background_threshold,
                  a.q.variance_floor, a.q.initial_variance};
  int fg = 0;
  for (int c = 0; c < d; ++c) {
    const PlaneRef<T> pr = plane_ref<T>(a, 0, c);
    uint16_t* metap = a.s.meta + (size_t)c * P + p;
    uint32_t meta = *metap;
    int n = meta_count(meta);
    Mix<KMAX> x;
    T e[rec_elems(KMAX)];
    load_mix_r<T, KMAX>(pr, p, n, x, e);
    int inv[KMAX];
    int n0 = n;
    fg |= gmm_step<KMAX>(x, n, K, (double)a.frame[(size_t)c * P + p],
                         a.q.learning_rate, gp, inv);
    store_mix_r<T, KMAX>(pr, p, n, x, e);
    if (n != n0) *metap = (uint16_t)meta_with_count(meta, n);
  }
  a.mask[p] = fg ? 255 : 0;
}

// ---------------------------------------------------------------------------
// state export / import (reference layouts)
// ---------------------------------------------------------------------------
template <typename T>
__global__ void export_kernel(cog_geom g, cog_state s, cog_ref_state o) {
  const size_t P = (size_t)g.height * g.width;
  const int d = g.depth, K = g.k;
  const int R = rec_elems(kbucket(K)), WO = rec_w(kbucket(K));
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < d * P;
       i += (size_t)gridDim.x * blockDim.x) {
    const size_t c = i / P, p = i % P;
    const T* rec = (const T*)s.mix + i * R;
    for (int k = 0; k < K; ++k) {
      const size_t dst = i * K + k;
      o.mu[dst] = (double)rec[2 * k];
      o.var[dst] = (double)rec[2 * k + 1];
      o.w[dst] = (double)rec[WO + k];
    }
    uint32_t m = s.meta[i], dy = s.dyn[i];
    o.count[i] = meta_count(m);
    for (int j = 0; j < 3; ++j) o.mid[i * 3 + j] = (int8_t)meta_mid(m, j);
    o.ref[i * 2 + 0] = (int8_t)meta_ref(m, 0);
    o.ref[i * 2 + 1] = (int8_t)meta_ref(m, 1);
    o.chp[i] = (uint8_t)dyn_chp(dy);
    o.label[i] = (uint8_t)dyn_label(dy);
    o.active[i] = (int8_t)dyn_active(dy);
    o.waking[i] = (uint8_t)dyn_waking(dy);
    o.clock[i] = dyn_clock(dy);
    o.streak[i] = s.streak[i];
    const uint32_t hq = s.hitq ? s.hitq[i] : 0u;
    for (int l = 0; l < 5; ++l)
      o.hits[i * 5 + l] = (long long)s.hits[(c * 5 + l) * P + p] +
                          (l < 4 ? (long long)((hq >> (8 * l)) & 0xFFu) : 0ll);
  }
}

template <typename T>
__global__ void import_kernel(cog_geom g, cog_state s, cog_ref_state in) {
  const size_t P = (size_t)g.height * g.width;
  const int d = g.depth, K = g.k;
  const int R = rec_elems(kbucket(K)), WO = rec_w(kbucket(K));
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < d * P;
       i += (size_t)gridDim.x * blockDim.x) {
    const size_t c = i / P, p = i % P;
    T* rec = (T*)s.mix + i * R;
    for (int k = 0; k < K; ++k) {
      const size_t src = i * K + k;
      st(rec + 2 * k, in.mu[src]);
      st(rec + 2 * k + 1, in.var[src]);
      st(rec + WO + k, in.w[src]);
    }
    s.meta[i] = (uint16_t)pack_meta((int)in.count[i], in.mid[i * 3],
                                    in.mid[i * 3 + 1], in.mid[i * 3 + 2],
                                    in.ref[i * 2], in.ref[i * 2 + 1]);
    long long ck = in.clock[i];
    s.dyn[i] = pack_dyn(in.chp[i], in.label[i] & 1, in.waking[i] & 1,
                        in.active[i], (int)(ck < 0 ? 0 : (ck > 65535 ? 65535 : ck)));
    long long sk = in.streak[i];
    s.streak[i] = (uint32_t)(sk < 0 ? 0 : (sk > 0xffffffffll ? 0xffffffffll : sk));
    for (int l = 0; l < 5; ++l) {
      long long h = in.hits[i * 5 + l];
      s.hits[(c * 5 + l) * P + p] =
          (uint32_t)(h < 0 ? 0 : (h > 0xffffffffll ? 0xffffffffll : h));
    }
    if (s.hitq) s.hitq[i] = 0u;
  }
}

#include "cog_lean.cuh"
#include "cog_fast.cuh"
#include "cog_hot.cuh"

// ---------------------------------------------------------------------------
// training: k-means assignment step (grouping.py:116-118): squared distance
// to every centre over the two features, (x0 - c0)^2 + (x1 - c1)^2 in
// binary64 (no contraction, so each value is numpy's), argmin with the
// lowest index on ties and the first NaN winning (numpy argmin).  One
// thread per point; `changed` is set if any label differs from the previous.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
    kmeans_assign_kernel(const double* __restrict__ pts, int64_t n,
                         const double* __restrict__ ctr, int k,
                         int64_t* __restrict__ label, uint32_t* changed) {
  unsigned any = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double x0 = pts[2 * i], x1 = pts[2 * i + 1];
    int best = 0;
    double bv = 0.0;
    for (int j = 0; j < k; ++j) {
      const double d0 = x0 - ctr[2 * j], d1 = x1 - ctr[2 * j + 1];
      const double d = d0 * d0 + d1 * d1;
      if (j == 0) {
        bv = d;
        if (isnan(d)) break;
      } else if (isnan(d)) {
        best = j;
        break;
      } else if (d < bv) {
        bv = d;
        best = j;
      }
    }
    if (label[i] != best) {
      label[i] = best;
      any = 1;
    }
  }
  if (__any_sync(FULL, any) && (threadIdx.x & 31) == 0) atomicOr(changed, 1u);
}

// ---------------------------------------------------------------------------
// training: the grouping's axis-0 reductions (grouping.py:100-161).  numpy
// sums the rows of a C-contiguous (n, dims) array one after another, so the
// reference's cluster means / deviations are SEQUENTIAL binary64 sums in
// index order -- not re-associable.  One warp per (label, column) chain:
// the warp loads 32 rows at a time (coalesced, next chunk in flight), then
// adds the matching rows' terms in index order (every lane keeps the same
// accumulator; the loop runs over the matching lanes only).  The chains of
// all labels and columns run side by side, each at one dependent DADD per
// member.  term = x (square = 0) or (x - shift[chain])^2 (square = 1).
// Also the chain's min and max (np.ptp) and the label's member count.
// ---------------------------------------------------------------------------
// The same sums for dims dividing 32, one warp per label: the lanes stage a
// tile of SEQ_TILE rows (masked rows as +0.0, which leaves a sum unchanged)
// in shared memory with coalesced loads, then lane f < dims adds its column
// of the tile in row order -- one shared load and one dependent DADD per
// row -- while the next tile's loads are in flight.
constexpr int SEQ_TILE = 128;
template <int DIMS>
__global__ void __launch_bounds__(32)
    seq_sums_tiled_kernel(const double* __restrict__ x, int64_t n,
                          const int64_t* __restrict__ label,
                          const double* __restrict__ shift, int square,
                          double* out, double* minmax, long long* count) {
  constexpr int PER = SEQ_TILE * DIMS / 32;  // elements per lane per tile
  __shared__ double buf[SEQ_TILE * DIMS];
  const int j = blockIdx.x, lane = threadIdx.x;
  const int f = lane % DIMS;                 // every element of this lane
  const double sh = shift ? shift[j * DIMS + f] : 0.0;
  double mn = __longlong_as_double(0x7ff0000000000000ll), mx = -mn;
  long long cnt = 0;
  double acc = 0.0;
  double t[PER], raw[PER];
  long long lb[PER];
  // raw loads of a tile (clamped rows), consumed by finish() after the
  // previous tile's adds, so they are in flight while lane f adds
  auto fetch = [&](int64_t i0) {
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      int64_t i = i0 + (q * 32 + lane) / DIMS;   // row of tile element e
      if (i >= n) i = n - 1;
      raw[q] = x[i * DIMS + f];
      lb[q] = label ? label[i] : (long long)j;
    }
  };
  auto finish = [&](int64_t i0) {
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int64_t i = i0 + (q * 32 + lane) / DIMS;
      const bool m = i < n && lb[q] == (long long)j;
      t[q] = 0.0;
      if (m) {
        const double v = raw[q];
        mn = fmin(mn, v);
        mx = fmax(mx, v);
        const double dv = v - sh;
        t[q] = square ? dv * dv : v;
        cnt += (f == 0);
      }
    }
  };
  if (n > 0) {
    fetch(0);
    finish(0);
  }
  for (int64_t i0 = 0; i0 < n; i0 += SEQ_TILE) {
    __syncwarp();
#pragma unroll
    for (int q = 0; q < PER; ++q) buf[q * 32 + lane] = t[q];
    __syncwarp();
    const bool more = i0 + SEQ_TILE < n;
    if (more) fetch(i0 + SEQ_TILE);
    if (lane < DIMS) {
#pragma unroll 16
      for (int r = 0; r < SEQ_TILE; ++r) acc = acc + buf[r * DIMS + lane];
    }
    if (more) finish(i0 + SEQ_TILE);
  }
  // lanes with the same f hold partial min / max / counts
  for (int o = 16; o >= DIMS; o >>= 1) {
    mn = fmin(mn, __shfl_xor_sync(FULL, mn, o));
    mx = fmax(mx, __shfl_xor_sync(FULL, mx, o));
    cnt += __shfl_xor_sync(FULL, cnt, o);
  }
  if (lane < DIMS) {
    out[j * DIMS + lane] = acc;
    if (minmax) {
      minmax[2 * (j * DIMS + lane)] = mn;
      minmax[2 * (j * DIMS + lane) + 1] = mx;
    }
    if (count && lane == 0) count[j] = cnt;
  }
}

__global__ void __launch_bounds__(32)
    seq_sums_kernel(const double* __restrict__ x, int64_t n, int dims,
                    const int64_t* __restrict__ label, int k,
                    const double* __restrict__ shift, int square, double* out,
                    double* minmax, long long* count) {
  const int chain = blockIdx.x, j = chain / dims, f = chain - j * dims;
  const int lane = threadIdx.x;
  const double sh = shift ? shift[chain] : 0.0;
  double acc = 0.0;
  double mn = __longlong_as_double(0x7ff0000000000000ll), mx = -mn;
  long long cnt = 0;
  double t_cur = 0.0, t_nxt = 0.0;
  bool m_cur = false, m_nxt = false;
  auto load = [&](int64_t i0, double& t, bool& m) {
    const int64_t i = i0 + lane;
    m = i < n && (!label || label[i] == (int64_t)j);
    t = 0.0;
    if (m) {
      const double v = x[i * dims + f];
      mn = fmin(mn, v);
      mx = fmax(mx, v);
      const double dv = v - sh;
      t = square ? dv * dv : v;
    }
  };
  load(0, t_cur, m_cur);
  for (int64_t i0 = 0; i0 < n; i0 += 32) {
    if (i0 + 32 < n) load(i0 + 32, t_nxt, m_nxt);
    unsigned bal = __ballot_sync(FULL, m_cur);
    cnt += __popc(bal);
    while (bal) {
      const int l = __ffs(bal) - 1;
      bal &= bal - 1;
      acc = acc + __shfl_sync(FULL, t_cur, l);
    }
    t_cur = t_nxt;
    m_cur = m_nxt;
    m_nxt = false;
  }
  for (int o = 16; o > 0; o >>= 1) {
    mn = fmin(mn, __shfl_xor_sync(FULL, mn, o));
    mx = fmax(mx, __shfl_xor_sync(FULL, mx, o));
  }
  if (lane == 0) {
    out[chain] = acc;
    if (minmax) {
      minmax[2 * chain] = mn;
      minmax[2 * chain + 1] = mx;
    }
    if (count && f == 0) count[j] = cnt;
  }
}

// farthest-point seeding step (grouping.py:100-112): far[i] = min(far[i],
// |pts[i] - c|^2) (first: far[i] = |pts[i] - c|^2), then np.argmax(far) =
// the lowest index of the largest value, in two passes over `best`
// (best[0] = max bits of far, best[1] = lowest index holding it; far >= 0,
// so its bit pattern orders like the value)
__global__ void __launch_bounds__(256)
    far_update_kernel(const double* __restrict__ pts, int64_t n, double c0,
                      double c1, int first, double* __restrict__ far,
                      unsigned long long* best) {
  unsigned long long m = 0ull;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double d0 = pts[2 * i] - c0, d1 = pts[2 * i + 1] - c1;
    double d = d0 * d0 + d1 * d1;
    if (!first) d = fmin(far[i], d);  // np.minimum(far, d)
    far[i] = d;
    const unsigned long long b = (unsigned long long)__double_as_longlong(d);
    m = b > m ? b : m;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long t = __shfl_xor_sync(FULL, m, o);
    m = t > m ? t : m;
  }
  if ((threadIdx.x & 31) == 0 && m) atomicMax(best, m);
}

__global__ void __launch_bounds__(256)
    far_argmax_kernel(const double* __restrict__ far, int64_t n,
                      unsigned long long* best) {
  const unsigned long long want = best[0];
  unsigned long long m = ~0ull;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if ((unsigned long long)__double_as_longlong(far[i]) == want)
      m = (unsigned long long)i < m ? (unsigned long long)i : m;
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long t = __shfl_xor_sync(FULL, m, o);
    m = t < m ? t : m;
  }
  if ((threadIdx.x & 31) == 0 && m != ~0ull) atomicMin(best + 1, m);
}

// ---------------------------------------------------------------------------
// training: pooled group statistics (grouping.py:189-192) for pools too big
// for numpy's in-memory expression: per (group, plane) the exact integer sums
// of x and x^2 over every training frame of every member pixel.  One thread
// per pixel (coalesced over the frames), shared-memory accumulation per CTA,
// one 64-bit atomic per entry per CTA.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
    pool_sums_kernel(const uint8_t* __restrict__ values, int N, int d,
                     int64_t P, const int32_t* __restrict__ member, int G,
                     unsigned long long* sums) {
  extern __shared__ unsigned long long ps[];  // [G][d][2]
  for (int i = threadIdx.x; i < G * d * 2; i += blockDim.x) ps[i] = 0ull;
  __syncthreads();
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < P;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int g = member[p];
    if (g < 0 || g >= G) continue;
    for (int c = 0; c < d; ++c) {
      unsigned long long s1 = 0, s2 = 0;
      for (int i = 0; i < N; ++i) {
        const unsigned x = values[((int64_t)i * d + c) * P + p];
        s1 += x;
        s2 += x * x;
      }
      atomicAdd(&ps[(g * d + c) * 2], s1);
      atomicAdd(&ps[(g * d + c) * 2 + 1], s2);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < G * d * 2; i += blockDim.x)
    if (ps[i]) atomicAdd(sums + i, ps[i]);
}

// ---------------------------------------------------------------------------
// evaluation: confusion counts (16 pixels a thread, warp reductions, one
// 64-bit atomic per count per warp)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
    confusion_kernel(const uint8_t* __restrict__ pred,
                     const uint8_t* __restrict__ truth, int64_t n,
                     unsigned long long* counts) {
  unsigned tp = 0, fp = 0, tn = 0, fn = 0, ex = 0;
  const int64_t nv = n / 16;
  const bool aligned = (((uintptr_t)pred | (uintptr_t)truth) & 15) == 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  auto one = [&](unsigned pv, unsigned tv) {
    const bool known = tv == 0u || tv == 255u;
    const bool pf = pv == 255u, tf = tv == 255u;
    tp += known && pf && tf;
    fp += known && pf && !tf;
    tn += known && !pf && !tf;
    fn += known && !pf && tf;
    ex += !known;
  };
  int64_t start = 0;
  if (aligned) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv;
         i += stride) {
      const uint4 a = __ldcs((const uint4*)pred + i);
      const uint4 b = __ldcs((const uint4*)truth + i);
      const unsigned pa[4] = {a.x, a.y, a.z, a.w};
      const unsigned tb[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int w = 0; w < 4; ++w)
#pragma unroll
        for (int j = 0; j < 4; ++j)
          one((pa[w] >> (8 * j)) & 0xFFu, (tb[w] >> (8 * j)) & 0xFFu);
    }
    start = nv * 16;
  }
  for (int64_t i = start + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
       i < n; i += stride)
    one(pred[i], truth[i]);
  const unsigned v[5] = {tp, fp, tn, fn, ex};
#pragma unroll
  for (int q = 0; q < 5; ++q) {
    const unsigned r = warp_sum_u32(v[q]);
    if ((threadIdx.x & 31) == 0 && r)
      atomicAdd(counts + q, (unsigned long long)r);
  }
}

// ---------------------------------------------------------------------------
// host helpers
// ---------------------------------------------------------------------------
int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

void ensure_bterm() {
  static bool done[64] = {false};
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  if (dev < 0 || dev >= 64 || done[dev]) return;
  double t[2][256];
  for (int i = 0; i < 256; ++i) {
    const double b = (double)i / 255.0;
    t[1][i] = b;
    t[0][i] = 1.0 - b;
  }
  cudaMemcpyToSymbol(g_bterm, t, sizeof(t));
  // the level-walk table of hot_kernel (cog_hot.cuh): for the level codes
  // (c0, c1, c2) and the 2-bit test states of GROUP / MEAN / MEANVAR, the
  // first code whose test is not a miss decides (kernels_numba.py:286-334)
  uint8_t wt[64 * 64];
  for (int codes = 0; codes < 64; ++codes) {
    for (int st = 0; st < 64; ++st) {
      int out = L_GMM;
      for (int j = 0; j < 3; ++j) {
        const int code = (codes >> (2 * j)) & 3;
        if (code == 0) break;  // mid_order entry -1: the walk ends
        const int state = (st >> (2 * (code - 1))) & 3;
        if (state == 0) continue;  // miss: next level
        out = state == 1 ? code : 0xFF;  // hit, or undecided
        break;
      }
      wt[codes * 64 + st] = (uint8_t)out;
    }
  }
  cudaMemcpyToSymbol(g_walk, wt, sizeof(wt));
  done[dev] = true;
}

// occupancy queries cost microseconds; the per-frame launch path asks the
// same (kernel, block, smem) question every frame -> memoise
int cached_occupancy(const void* fn, int threads, size_t smem) {
  struct Entry { const void* fn; int threads; size_t smem; int occ; };
  static Entry cache[64];
  static int n = 0;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  for (int i = 0; i < n; ++i)
    if (cache[i].fn == fn && cache[i].threads == threads &&
        cache[i].smem == smem)
      return cache[i].occ;
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem);
  if (occ < 1) occ = 1;
  if (n < 64) cache[n++] = Entry{fn, threads, smem, occ};
  return occ;
}

int check_geom(const cog_geom* g) {
  if (!g) return COG_EINVAL;
  if (g->height < 1 || g->width < 1 || g->depth < 1 || g->depth > MAXD)
    return COG_EINVAL;
  if (g->k < 1 || g->k > 8) return COG_EUNSUPPORTED;
  if (g->stride < 1 || g->stride > 16 || g->streams < 1 || g->n_groups < 0)
    return COG_EUNSUPPORTED;
  if (g->row0 % g->stride) return COG_EINVAL;
  return COG_OK;
}

int launch_status() {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? COG_OK : (int)e;
}

StepArgs make_args(const cog_geom* g, const cog_params* q, const cog_state* s) {
  StepArgs a{};
  a.g = *g;
  if (q) a.q = *q;
  a.s = *s;
  tile_shape(g->stride, g->height, g->width, a.cw, a.iters, a.tiles_x,
             a.n_tiles);
  return a;
}

template <typename T>
using StepFn = void (*)(const StepArgs);

template <typename T>
StepFn<T> pick_step(int K) {
  if (K <= 3) return step_kernel<T, 3>;
  if (K <= 5) return step_kernel<T, 5>;
  return step_kernel<T, 8>;
}
template <typename T>
StepFn<T> pick_pending(int K) {
  if (K <= 3) return pending_kernel<T, 3>;
  if (K <= 5) return pending_kernel<T, 5>;
  return pending_kernel<T, 8>;
}
template <typename T>
StepFn<T> pick_baseline(int K) {
  if (K <= 3) return baseline_kernel<T, 3>;
  if (K <= 5) return baseline_kernel<T, 5>;
  return baseline_kernel<T, 8>;
}

template <typename T>
StepFn<T> pick_deep(int K) {
  if (K <= 3) return deep_kernel<T, 3>;
  if (K <= 5) return deep_kernel<T, 5>;
  return deep_kernel<T, 8>;
}

// step-kernel choice (cog_params.variant): 0 automatic, 1 general, 2 lean;
// a kernel is used only where its shared memory fits (per-warp group
// partials grow with the group count), so any valid configuration runs
constexpr size_t SMEM_CAP = 200 * 1024;

template <typename T>
StepFn<T> pick_lean(int K, int d) {
  if (d == 1) {
    if (K <= 3) return lean_kernel<T, 3, 1>;
    if (K <= 5) return lean_kernel<T, 5, 1>;
    return lean_kernel<T, 8, 1>;
  }
  if (K <= 3) return lean_kernel<T, 3, 3>;
  if (K <= 5) return lean_kernel<T, 5, 3>;
  return lean_kernel<T, 8, 3>;
}

bool lean_ok(const StepArgs& a) {
  return (a.q.variant == 0 || a.q.variant == 2) && a.iters == 1 &&
         (a.g.depth == 1 || a.g.depth == 3) && a.g.stride <= 5 &&
         lean_smem_bytes(a.g.depth, a.g.n_groups) <= SMEM_CAP;
}

size_t step_smem_bytes(const StepArgs& a) {
  const int warps = STEP_WARPS;
  return 256 * 8 + (size_t)2 * a.g.depth * a.g.n_groups * 8 +
         (size_t)warps * acc_words(a.g.depth, a.g.n_groups) * 8 +
         (size_t)warps * sizeof(WarpScratch) +
         (size_t)warps * lane_acc_bytes(a.g.depth, a.g.n_groups);
}

template <typename T>
int launch_lean(const StepArgs& a, cudaStream_t st) {
  auto fn = pick_lean<T>(a.g.k, a.g.depth);
  const size_t smem = lean_smem_bytes(a.g.depth, a.g.n_groups);
  if (smem > SMEM_CAP) return COG_EUNSUPPORTED;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
  const int occ = cached_occupancy((const void*)fn, LEAN_THREADS, smem);
  const int need = (a.n_tiles + LEAN_WARPS - 1) / LEAN_WARPS;
  int per_stream = (num_sms() * occ) / a.g.streams;  // one wave
  if (per_stream < 1) per_stream = 1;
  int gx = need < per_stream ? need : per_stream;
  if (gx < 1) gx = 1;
  fn<<<dim3(gx, a.g.streams), LEAN_THREADS, smem, st>>>(a);
  return launch_status();
}

template <int KMAX, int D>
int launch_fast_k(const StepArgs& a, cudaStream_t st) {
  auto fn = fast_kernel<KMAX, D>;
  const size_t smem = fast_smem_bytes(a.g.depth, a.g.n_groups);
  if (smem > SMEM_CAP) return COG_EUNSUPPORTED;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
  const int occ = cached_occupancy((const void*)fn, LEAN_THREADS, smem);
  // static schedule over every resident slot (at most one tile per warp
  // more than another, spread over the CTAs by the kernel's warp ranking)
  const long long units = (long long)a.n_tiles;
  // rounded down: every CTA of every stream resident in one wave (a CTA in
  // a second wave would start only when a first-wave one ends)
  int per_stream = (num_sms() * occ) / a.g.streams;
  if (per_stream < 1) per_stream = 1;
  long long gxl = (units + LEAN_WARPS - 1) / LEAN_WARPS;
  if (gxl > per_stream) gxl = per_stream;
  int gx = (int)gxl;
  if (gx < 1) gx = 1;
  const FastConst k = make_fast_const(a.q);
  fn<<<dim3(gx, a.g.streams), LEAN_THREADS, smem, st>>>(a, k);
  return launch_status();
}

int launch_fast(const StepArgs& a, cudaStream_t st) {
  if (a.g.depth == 1) {
    if (a.g.k <= 3) return launch_fast_k<3, 1>(a, st);
    if (a.g.k <= 5) return launch_fast_k<5, 1>(a, st);
    return launch_fast_k<8, 1>(a, st);
  }
  if (a.g.k <= 3) return launch_fast_k<3, 3>(a, st);
  if (a.g.k <= 5) return launch_fast_k<5, 3>(a, st);
  return launch_fast_k<8, 3>(a, st);
}

template <int KMAX, int D, int ST, int FL, bool PIPE, bool BIG>
int launch_hot_k(const StepArgs& a, cudaStream_t st) {
  auto fn = hot_kernel<KMAX, D, ST, FL, PIPE, BIG>;
  constexpr bool big = BIG;
  const size_t smem = hot_smem_bytes(a.g.depth, a.g.n_groups, big, PIPE);
  if (smem > SMEM_CAP) return COG_EUNSUPPORTED;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
  // the whole unified L1/shared array as shared memory: the occupancy is
  // then bounded by the registers, not by a small default carveout
  cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                       (int)cudaSharedmemCarveoutMaxShared);
  const int threads = 32 * D * HOT_TPB;
  const int occ = cached_occupancy((const void*)fn, threads, smem);
  // HOT_TPB tiles per CTA at a time, CTAs striding over the tiles; every
  // CTA of every stream resident in one wave
  int per_stream = (num_sms() * occ) / a.g.streams;
  if (per_stream < 1) per_stream = 1;
  const int need = (a.n_tiles + HOT_TPB - 1) / HOT_TPB;
  const int gx = need < per_stream ? need : per_stream;
  FastConst k = make_fast_const(a.q);
  k.P = a.g.height * a.g.width;
  k.wpad = (acc_words(a.g.depth, big ? 0 : a.g.n_groups) + 1) & ~1;
  if (PIPE && HOT_MASK_ATOMIC != 0 && D > 1) {
    // the plane warps OR their foreground bytes into a zeroed mask
    const cudaError_t e = cudaMemsetAsync(
        a.mask, 0, (size_t)a.g.streams * a.g.height * a.g.width, st);
    if (e != cudaSuccess) return (int)e;
  }
  fn<<<dim3(gx < 1 ? 1 : gx, a.g.streams), threads, smem, st>>>(a, k);
  return launch_status();
}

// the group sums and constants move to global memory when they would not
// fit comfortably in shared memory (hundreds of groups): any group count runs
template <int KMAX, int D, int ST, int FL, bool PIPE>
int launch_hot_b(const StepArgs& a, cudaStream_t st) {
  if (hot_smem_bytes(a.g.depth, a.g.n_groups, false, false) > 24 * 1024)
    return launch_hot_k<KMAX, D, ST, FL, PIPE, true>(a, st);
  return launch_hot_k<KMAX, D, ST, FL, PIPE, false>(a, st);
}

// the production configuration (stride 2, the reference's default feature
// switches) is compiled in; anything else reads them at run time
template <int KMAX, int D>
int launch_hot_cfg(const StepArgs& a, cudaStream_t st) {
  const int fl = (a.q.sampling_on ? HF_SAMPLING : 0) |
                 (a.q.grouping_on ? HF_GROUPING : 0) |
                 (a.q.chp_on ? HF_CHP : 0) |
                 (a.q.rate_scaling_on ? HF_RATE : 0) |
                 (a.q.literal_conf ? HF_LITERAL : 0);
  if (a.g.stride == 2 && fl == HF_DEFAULT) {
    // the pipelined variant copies 16-byte chunks of 16-pixel rows: every
    // row of every round-1 array must start on a 16-byte boundary
    const uintptr_t bases = (uintptr_t)a.frame | (uintptr_t)a.s.dyn |
                            (uintptr_t)a.s.streak | (uintptr_t)a.s.meta |
                            (uintptr_t)a.s.gid | (uintptr_t)a.s.cls |
                            (uintptr_t)a.mask;
    if (HOT_PIPE && a.g.width % 16 == 0 && (bases & 15) == 0)
      return launch_hot_b<KMAX, D, 2, HF_DEFAULT, true>(a, st);
    return launch_hot_b<KMAX, D, 2, HF_DEFAULT, false>(a, st);
  }
  return launch_hot_b<KMAX, D, 0, -1, false>(a, st);
}

int launch_hotpass(const StepArgs& a, cudaStream_t st) {
  if (a.g.depth == 1) {
    if (a.g.k <= 3) return launch_hot_cfg<3, 1>(a, st);
    if (a.g.k <= 5) return launch_hot_cfg<5, 1>(a, st);
    return launch_hot_cfg<8, 1>(a, st);
  }
  if (a.g.k <= 3) return launch_hot_cfg<3, 3>(a, st);
  if (a.g.k <= 5) return launch_hot_cfg<5, 3>(a, st);
  return launch_hot_cfg<8, 3>(a, st);
}

template <typename T>
int launch_hot(const StepArgs& a, cudaStream_t st) {
  if (lean_ok(a)) return launch_lean<T>(a, st);
  auto fn = pick_step<T>(a.g.k);
  const int threads = STEP_THREADS;
  const int warps = threads / 32;
  const size_t smem = step_smem_bytes(a);
  if (smem > SMEM_CAP) return COG_EUNSUPPORTED;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
  const int occ = cached_occupancy((const void*)fn, threads, smem);
  const int need = (a.n_tiles + warps - 1) / warps;
  int per_stream = (num_sms() * occ) / a.g.streams;  // one wave
  if (per_stream < 1) per_stream = 1;
  int gx = need < per_stream ? need : per_stream;
  if (gx < 1) gx = 1;
  fn<<<dim3(gx, a.g.streams), threads, smem, st>>>(a);
  return launch_status();
}

bool fast_ok(const StepArgs& a, bool f32) {
  const unsigned long long span = (unsigned long long)a.g.streams *
                                  a.g.depth * (a.g.k > 5 ? a.g.k : 5) *
                                  (unsigned long long)a.g.height * a.g.width;
  const unsigned long long recs = (unsigned long long)a.g.streams *
                                  a.g.depth * (unsigned long long)a.g.height *
                                  a.g.width * rec_elems(kbucket(a.g.k));
  return f32 && (a.q.variant == 0 || a.q.variant == 3) &&
         a.s.tabq != nullptr && a.iters == 1 &&
         a.g.stride <= 4 && (a.g.depth == 1 || a.g.depth == 3) &&
         span < (1ull << 32) && recs < (1ull << 32) &&
         !a.q.exact_group_sums && !a.q.compat &&
         (a.q.variant == 3
              ? fast_smem_bytes(a.g.depth, a.g.n_groups) <= SMEM_CAP
              : true);
}

template <typename T>
int launch_deep(const StepArgs& a, cudaStream_t st, bool pdl) {
  auto fn = pick_deep<T>(a.g.k);
  const size_t P = (size_t)a.g.height * a.g.width;
  size_t dg = (P * a.g.depth / 8 + DEEP_THREADS - 1) / DEEP_THREADS;  // ~12% items
  // grid-stride over the worklist, one wave
  const size_t per_sm =
      (size_t)cached_occupancy((const void*)fn, DEEP_THREADS, 0);
  size_t cap = (size_t)num_sms() * per_sm / a.g.streams;
  if (cap < 1) cap = 1;
  if (dg > cap) dg = cap;
  if (dg < 1) dg = 1;
  if (!pdl) {
    fn<<<dim3((unsigned)dg, a.g.streams), DEEP_THREADS, 0, st>>>(a);
    return launch_status();
  }
  // programmatic dependent launch: the deep grid is scheduled while the
  // hot kernel drains and waits (griddepcontrol.wait) for its results
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)dg, a.g.streams);
  cfg.blockDim = dim3(DEEP_THREADS);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, fn, a);
  return e == cudaSuccess ? COG_OK : (int)e;
}

template <typename T>
int launch_step(const StepArgs& a, cudaStream_t st) {
  ensure_bterm();
  // float32 state: the fast kernel; otherwise lean / general
  const bool fast = fast_ok(a, sizeof(T) == 4);
  StepArgs b = a;
  b.two_ended = fast && a.q.variant != 3;
  int rc = fast ? (a.q.variant == 3 ? launch_fast(b, st) : launch_hotpass(b, st))
                : launch_hot<T>(b, st);
  if (rc) return rc;
  // programmatic dependent launch of the deep pass behind the fast kernel:
  // its CTAs are scheduled while the hot kernel drains (they wait in
  // griddepcontrol.wait), which hides the launch gap
  return launch_deep<T>(b, st, fast);
}

}  // namespace

// ===========================================================================
// C-ABI
// ===========================================================================
extern "C" {

const char* cog_version(void) {
  return "cog_b200 2.0 (sm_100a, binary64 decisions, fused step, record "
         "mixtures, u16 hot prior)";
}

int64_t cog_accum_words(int32_t depth, int32_t n_groups) {
  return acc_words(depth, n_groups);
}

int64_t cog_deepq_slots(int32_t depth, int64_t n_pix) {
  return (int64_t)dq_capacity(depth, (size_t)n_pix);
}

int64_t cog_mix_elems(int32_t k) {
  if (k < 1 || k > 8) return -1;
  return rec_elems(kbucket(k));
}

int64_t cog_tabq_elems(const cog_geom* geom) {
  if (!geom || check_geom(geom)) return -1;
  return (int64_t)(tab_geo(*geom).plane * (size_t)geom->depth);
}

int cog_tabq_build(const cog_geom* geom, const float* table, const float* peak,
                   uint16_t* tabq, void* stream) {
  int rc = check_geom(geom);
  if (rc) return rc;
  if (!table || !peak || !tabq) return COG_EINVAL;
  const size_t P = (size_t)geom->height * geom->width;
  const size_t n = (size_t)geom->depth * P * 256;
  size_t blocks = (n + 255) / 256;
  const size_t cap = (size_t)num_sms() * 16;
  if (blocks > cap) blocks = cap;
  tabq_build_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
      tab_geo(*geom), geom->depth, P, table, peak, tabq);
  return launch_status();
}

int cog_prior_build(const uint8_t* frames, int32_t n_frames, int32_t depth,
                    int64_t n_pix, const double* kern, const int32_t* windows,
                    int32_t n_windows, float* tables, float* peak,
                    uint16_t* hist, double residue_t1, double residue_t2,
                    double peaky_threshold, uint32_t* residue, uint8_t* cls,
                    void* stream) {
  if (!frames || !kern || !windows || !tables || !peak || !cls)
    return COG_EINVAL;
  if (n_frames < 2 || depth < 1 || n_pix < 1 || n_windows < 1)
    return COG_EINVAL;
  const size_t smem = (((size_t)n_frames * 32 + 15) & ~(size_t)15) +
                      256 * 32 * sizeof(uint16_t);
  if (smem > 200 * 1024) return COG_EUNSUPPORTED;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(prior_kernel,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const unsigned blocks = (unsigned)((n_pix + PRIOR_PIX - 1) / PRIOR_PIX);
  prior_kernel<<<blocks, 256, smem, (cudaStream_t)stream>>>(
      frames, n_frames, depth, n_pix, kern, windows, n_windows, tables, peak,
      hist, residue_t1, residue_t2, peaky_threshold, residue, cls);
  return launch_status();
}

int cog_gmm_warmup(const cog_geom* geom, const cog_params* prm,
                   const cog_state* st, const uint8_t* frames,
                   int32_t n_frames, double* features, double* w_final,
                   void* stream) {
  int rc = check_geom(geom);
  if (rc) return rc;
  if (!prm || !st || !frames || n_frames < 1) return COG_EINVAL;
  WarmArgs a{};
  a.g = *geom;
  a.q = *prm;
  a.s = *st;
  a.frames = frames;
  a.N = n_frames;
  a.features = features;
  a.w_final = w_final;
  const size_t P = (size_t)geom->height * geom->width;
  dim3 grid((unsigned)((P + 127) / 128), geom->depth);
  cudaStream_t s = (cudaStream_t)stream;
  const int K = geom->k;
  if (geom->state_f64) {
    if (K <= 3) warmup_kernel<double, 3><<<grid, 128, 0, s>>>(a);
    else if (K <= 5) warmup_kernel<double, 5><<<grid, 128, 0, s>>>(a);
    else warmup_kernel<double, 8><<<grid, 128, 0, s>>>(a);
  } else {
    if (K <= 3) warmup_kernel<float, 3><<<grid, 128, 0, s>>>(a);
    else if (K <= 5) warmup_kernel<float, 5><<<grid, 128, 0, s>>>(a);
    else warmup_kernel<float, 8><<<grid, 128, 0, s>>>(a);
  }
  return launch_status();
}

int cog_set_levels(const cog_geom* geom, const cog_state* st, void* stream) {
  int rc = check_geom(geom);
  if (rc) return rc;
  if (!st || !st->meta || !st->gid) return COG_EINVAL;
  set_levels_kernel<<<num_sms() * 4, 256, 0, (cudaStream_t)stream>>>(
      *geom, st->meta, st->gid);
  return launch_status();
}

int cog_step(const cog_geom* geom, const cog_params* prm, const cog_state* st,
             const uint8_t* frame, uint8_t* mask, void* conf, uint8_t* kind,
             int64_t* stats, int64_t frame_index, int32_t reorder_now,
             int32_t fuse_finalize, void* stream) {
  int rc = check_geom(geom);
  if (rc) return rc;
  if (!prm || !st || !frame || !mask || !conf || !kind || !stats)
    return COG_EINVAL;
  if (((uintptr_t)st->sync & 15) != 0) return COG_EINVAL;  // 64-bit atomics
  StepArgs a = make_args(geom, prm, st);
  a.frame = frame;
  a.mask = mask;
  a.conf = conf;
  a.kind = kind;
  a.stats = stats;
  a.frame_index = frame_index;
  a.reorder_now = reorder_now;
  a.fuse_finalize = fuse_finalize;
  cudaStream_t s = (cudaStream_t)stream;
  return geom->state_f64 ? launch_step<double>(a, s) : launch_step<float>(a, s);
}

int cog_step_host(const cog_geom* geom, const cog_params* prm,
                  const cog_state* st, const uint8_t* host_frame,
                  uint8_t* dev_frame, uint8_t* dev_mask, void* conf,
                  uint8_t* kind, int64_t* dev_stats, uint8_t* host_mask,
                  int64_t* host_stats, int64_t frame_index,
                  int32_t reorder_now, void* stream, void* copy_stream,
                  void* down_stream, void* up_event, void* done_event) {
  int rc = check_geom(geom);
  if (rc) return rc;
  if (!host_frame || !dev_frame || !host_mask || !host_stats || !up_event ||
      !done_event || geom->streams != 1)
    return COG_EINVAL;
  const size_t P = (size_t)geom->height * geom->width;
  cudaStream_t s = (cudaStream_t)stream, cs = (cudaStream_t)copy_stream;
  cudaError_t e = cudaMemcpyAsync(dev_frame, host_frame, P * geom->depth,
                                  cudaMemcpyHostToDevice, cs);
  if (e == cudaSuccess) e = cudaEventRecord((cudaEvent_t)up_event, cs);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(s, (cudaEvent_t)up_event, 0);
  if (e != cudaSuccess) return (int)e;
  rc = cog_step(geom, prm, st, dev_frame, dev_mask, conf, kind, dev_stats,
                frame_index, reorder_now, 1, stream);
  if (rc) return rc;
  // downloads on their own stream (when given): the next frame's step does
  // not queue behind this frame's device->host copies
  cudaStream_t ds = down_stream ? (cudaStream_t)down_stream : s;
  e = cudaSuccess;
  if (ds != s) {
    e = cudaEventRecord((cudaEvent_t)done_event, s);  // the step is done
    if (e == cudaSuccess) e = cudaStreamWaitEvent(ds, (cudaEvent_t)done_event, 0);
  }
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(host_mask, dev_mask, P, cudaMemcpyDeviceToHost, ds);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(host_stats, dev_stats, 16 * sizeof(int64_t),
                        cudaMemcpyDeviceToHost, ds);
  if (e == cudaSuccess) e = cudaEventRecord((cudaEvent_t)done_event, ds);
  return e == cudaSuccess ? COG_OK : (int)e;
}

int cog_pool_sums(const uint8_t* values, int32_t n_frames, int32_t depth,
                  int64_t n_pix, const int32_t* member, int32_t n_groups,
                  uint64_t* sums, void* stream) {
  if (!values || !member || !sums || n_frames < 1 || depth < 1 ||
      depth > MAXD || n_pix < 0 || n_groups < 1)
    return COG_EINVAL;
  const size_t smem = (size_t)n_groups * depth * 2 * 8;
  if (smem > 48 * 1024) return COG_EUNSUPPORTED;
  if (n_pix == 0) return COG_OK;
  int64_t blocks = (n_pix + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  pool_sums_kernel<<<(unsigned)blocks, 256, smem, (cudaStream_t)stream>>>(
      values, n_frames, depth, n_pix, member, n_groups,
      (unsigned long long*)sums);
  return launch_status();
}

int cog_kmeans_assign(const double* points, int64_t n, const double* centers,
                      int32_t k, int64_t* label, uint32_t* changed,
                      void* stream) {
  if (!points || !centers || !label || !changed || n < 0 || k < 1)
    return COG_EINVAL;
  if (n == 0) return COG_OK;
  int64_t blocks = (n + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 16;
  if (blocks > cap) blocks = cap;
  kmeans_assign_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
      points, n, centers, k, label, changed);
  return launch_status();
}

int cog_seq_sums(const double* x, int64_t n, int32_t dims,
                 const int64_t* label, int32_t k, const double* shift,
                 int32_t square, double* out, double* minmax, int64_t* count,
                 void* stream) {
  if (!x || !out || n < 0 || dims < 1 || k < 1) return COG_EINVAL;
  if (square && !shift) return COG_EINVAL;
  if (dims == 1 || dims == 2) {
    auto fn = dims == 1 ? seq_sums_tiled_kernel<1> : seq_sums_tiled_kernel<2>;
    fn<<<(unsigned)k, 32, 0, (cudaStream_t)stream>>>(
        x, n, label, shift, square, out, minmax, (long long*)count);
    return launch_status();
  }
  seq_sums_kernel<<<(unsigned)(k * dims), 32, 0, (cudaStream_t)stream>>>(
      x, n, dims, label, k, shift, square, out, minmax, (long long*)count);
  return launch_status();
}

int cog_far_step(const double* points, int64_t n, const double* centre,
                 int32_t first, double* far, uint64_t* best, void* stream) {
  if (!points || !centre || !far || !best || n < 1) return COG_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  int64_t blocks = (n + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 16;
  if (blocks > cap) blocks = cap;
  const unsigned long long init[2] = {0ull, ~0ull};
  cudaError_t e = cudaMemcpyAsync(best, init, sizeof(init),
                                  cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return (int)e;
  far_update_kernel<<<(unsigned)blocks, 256, 0, s>>>(
      points, n, centre[0], centre[1], first, far, (unsigned long long*)best);
  far_argmax_kernel<<<(unsigned)blocks, 256, 0, s>>>(
      far, n, (unsigned long long*)best);
  return launch_status();
}

int cog_confusion(const uint8_t* predicted, const uint8_t* truth, int64_t n,
                  uint64_t* counts, void* stream) {
  if (!predicted || !truth || !counts || n < 0) return COG_EINVAL;
  if (n == 0) return COG_OK;
  int64_t blocks = (n / 16 + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  confusion_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
      predicted, truth, n, (unsigned long long*)counts);
  return launch_status();
}

void* cog_event_create(void) {
  cudaEvent_t ev = nullptr;
  if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess)
    return nullptr;
  return (void*)ev;
}

int cog_event_destroy(void* event) {
  return event ? (int)cudaEventDestroy((cudaEvent_t)event) : COG_EINVAL;
}

int cog_event_sync(void* event) {
  return event ? (int)cudaEventSynchronize((cudaEvent_t)event) : COG_EINVAL;
}

int cog_event_query(void* event) {
  if (!event) return COG_EINVAL;
  const cudaError_t e = cudaEventQuery((cudaEvent_t)event);
  if (e == cudaSuccess) return 1;
  if (e == cudaErrorNotReady) {
    cudaGetLastError();
    return 0;
  }
  return -(int)e;
}

int cog_finalize(const cog_geom* geom, const cog_params* prm,
                 const cog_state* st, int64_t* stats, int64_t frame_index,
                 void* stream) {
  int rc = check_geom(geom);
  if (rc) return rc;
  if (!prm || !st || !stats) return COG_EINVAL;
  StepArgs a = make_args(geom, prm, st);
  a.stats = stats;
  a.frame_index = frame_index;
  if (geom->state_f64)
    finalize_kernel<double><<<geom->streams, 128, 0, (cudaStream_t)stream>>>(a);
  else
    finalize_kernel<float><<<geom->streams, 128, 0, (cudaStream_t)stream>>>(a);
  return launch_status();
}

int64_t cog_mailbox_words(int32_t depth, int32_t n_groups, int32_t n_ranks) {
  if (depth < 1 || depth > MAXD || n_groups < 0 || n_ranks < 1 ||
      n_ranks > COG_MAX_RANKS)
    return -1;
  return 2ll * n_ranks * ((int64_t)acc_words(depth, n_groups) + 1);
}

static int check_peers(const cog_geom* geom, const cog_peers* pr) {
  if (!pr || pr->n_ranks < 2 || pr->n_ranks > COG_MAX_RANKS || pr->rank < 0 ||
      pr->rank >= pr->n_ranks || pr->seq == 0 || geom->streams != 1)
    return COG_EINVAL;
  for (int r = 0; r < pr->n_ranks; ++r)
    if (!pr->mailbox[r]) return COG_EINVAL;
  return COG_OK;
}

int cog_step_p2p(const cog_geom* geom, const cog_params* prm,
                 const cog_state* st, const uint8_t* frame, uint8_t* mask,
                 void* conf, uint8_t* kind, int64_t* stats,
                 int64_t frame_index, int32_t reorder_now, int32_t fuse,
                 const cog_peers* peers, void* stream) {
  int rc = check_geom(geom);
  if (rc) return rc;
  if (!prm || !st || !frame || !mask || !conf || !kind || !stats)
    return COG_EINVAL;
  rc = check_peers(geom, peers);
  if (rc) return rc;
  if (((uintptr_t)st->sync & 15) != 0) return COG_EINVAL;  // 64-bit atomics
  StepArgs a = make_args(geom, prm, st);
  a.frame = frame;
  a.mask = mask;
  a.conf = conf;
  a.kind = kind;
  a.stats = stats;
  a.frame_index = frame_index;
  a.reorder_now = reorder_now;
  a.fuse_finalize = fuse ? 1 : 0;
  a.peers = *peers;
  cudaStream_t s = (cudaStream_t)stream;
  return geom->state_f64 ? launch_step<double>(a, s) : launch_step<float>(a, s);
}

int cog_finalize_p2p(const cog_geom* geom, const cog_params* prm,
                     const cog_state* st, int64_t* stats, int64_t frame_index,
                     const cog_peers* peers, void* stream) {
  int rc = check_geom(geom);
  if (rc) return rc;
  if (!prm || !st || !stats) return COG_EINVAL;
  rc = check_peers(geom, peers);
  if (rc) return rc;
  StepArgs a = make_args(geom, prm, st);
  a.stats = stats;
  a.frame_index = frame_index;
  a.peers = *peers;
  if (geom->state_f64)
    finalize_kernel<double><<<1, 128, 0, (cudaStream_t)stream>>>(a);
  else
    finalize_kernel<float><<<1, 128, 0, (cudaStream_t)stream>>>(a);
  return launch_status();
}

int cog_apply_pending(const cog_geom* geom, const cog_params* prm,
                      const cog_state* st, int32_t reorder_now, void* stream) {
  int rc = check_geom(geom);
  if (rc) return rc;
  if (!prm || !st) return COG_EINVAL;
  StepArgs a = make_args(geom, prm, st);
  a.reorder_now = reorder_now;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t work = (size_t)geom->depth * geom->height * geom->width;
  unsigned gx = (unsigned)((work + 255) / 256);
  const unsigned cap = (unsigned)num_sms() * 8;
  if (gx > cap) gx = cap;
  dim3 grid(gx, geom->streams);
  if (geom->state_f64) pick_pending<double>(geom->k)<<<grid, 256, 0, s>>>(a);
  else pick_pending<float>(geom->k)<<<grid, 256, 0, s>>>(a);
  rc = launch_status();
  if (rc) return rc;
  clear_pending_kernel<<<(geom->streams + 127) / 128, 128, 0, s>>>(
      st->sync, geom->streams, reorder_now);
  return launch_status();
}

int cog_baseline_frame(const cog_geom* geom, const cog_params* prm,
                       const cog_state* st, const uint8_t* frame,
                       uint8_t* mask, void* stream) {
  int rc = check_geom(geom);
  if (rc) return rc;
  if (!prm || !st || !frame || !mask) return COG_EINVAL;
  StepArgs a = make_args(geom, prm, st);
  a.frame = frame;
  a.mask = mask;
  const size_t P = (size_t)geom->height * geom->width;
  const unsigned blocks = (unsigned)((P + 255) / 256);
  cudaStream_t s = (cudaStream_t)stream;
  if (geom->state_f64) pick_baseline<double>(geom->k)<<<blocks, 256, 0, s>>>(a);
  else pick_baseline<float>(geom->k)<<<blocks, 256, 0, s>>>(a);
  return launch_status();
}

int cog_export_state(const cog_geom* geom, const cog_state* st,
                     const cog_ref_state* out, void* stream) {
  int rc = check_geom(geom);
  if (rc) return rc;
  if (!st || !out) return COG_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  unsigned blocks = (unsigned)num_sms() * 4;
  if (geom->state_f64) export_kernel<double><<<blocks, 256, 0, s>>>(*geom, *st, *out);
  else export_kernel<float><<<blocks, 256, 0, s>>>(*geom, *st, *out);
  return launch_status();
}

int cog_import_state(const cog_geom* geom, const cog_state* st,
                     const cog_ref_state* in, void* stream) {
  int rc = check_geom(geom);
  if (rc) return rc;
  if (!st || !in) return COG_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  unsigned blocks = (unsigned)num_sms() * 4;
  if (geom->state_f64) import_kernel<double><<<blocks, 256, 0, s>>>(*geom, *st, *in);
  else import_kernel<float><<<blocks, 256, 0, s>>>(*geom, *st, *in);
  return launch_status();
}

}  // extern "C"
