// cog_fast.cuh -- the float32-state step kernel (the throughput path).
// Included inside the anonymous namespace of cog_kernels.cu.
//
// Work unit = one stride-aligned warp tile (stride rows x cw columns, so
// every copy pixel's anchor is in row 0 of the same warp); thread = one
// pixel, planes processed one after another in a non-unrolled loop (the
// reference's planes are independent, cascade.py:281) so a thread holds one
// plane's state at a time.  The union mask is written per tile; labels that
// arrive with the deep kernel (GMM fall-throughs) are OR-ed in there.
//
// Loads per plane-pixel, in two dependent rounds:
//   round 1 (pixel index): frame byte, dyn, meta, streak -- for all planes
//            of the tile up front;
//   round 2 (needs v and meta): the hot prior phat(v) from the u16
//            tile-major table, and -- only when the cascade can reach a
//            mode level or the confidence reads a mode (the group test is
//            settled from shared memory first; ~75 % of plane-pixels stop
//            at the group level) -- the (mu, var) pairs of the two
//            referenced modes from the pixel's 64-B mixture record, one
//            8-byte load each, same DRAM burst.
// The per-plane-pixel work is split by frequency:
//   * fast path (the common case: evaluated pixel, sampling clock idle, not
//     compat, no decision within the filter margins): the cascade in fp32
//     with float constants precomputed on the host (FastConst), integer
//     change test, one level walk.  It makes exactly the reference's
//     decisions: an fp32 comparison whose operands lie within its margin
//     (the u16 prior's quantisation, 7.7e-6, plus 1e-5 relative) bails out;
//   * slow path: the general hot_px (binary64 fallbacks from the exact f32
//     table, SKIP/COPY gating, compat) for the rare plane-pixels that need
//     it; its exact loads (table entry, peak, modes) are issued only then.
//   * group partials: a warp-tile is nearly always group-homogeneous, so the
//     partials are one set of warp reductions added by lane 0 into the
//     warp's private shared slice (no atomics); mixed tiles loop.

constexpr int FQ_CAP = 64;  // per-warp worklist buffer (one global atomic per flush)

// u16 hot prior: phat = q / 65535 with q = round(phat * 65535), so
// |phat - q / 65535| <= 0.5 / 65535 (+ the fp32 product's rounding)
constexpr float PH_Q = 1.0f / 65535.0f;
constexpr float PH_QERR = 7.7e-6f;

struct FastConst {
  float lam, pf, ct, pf_margin;
  float w[9];
  float wbc_inv[3];  // 1 / (wb + wc) per class, 0 if wb + wc <= 0
  float ct_margin[3];  // |conf - ct| below this -> exact path, per class
  int eps_i;         // changed  <=>  |v - chp| > eps_i
  int sat;           // saturation_frames (clamped to int)
  int P;             // hot_kernel: pixels per plane (height * width)
  int wpad;          // hot_kernel: words of a warp's partial slice in shared
};

FastConst make_fast_const(const cog_params& q) {
  FastConst k{};
  k.lam = (float)q.match_lambda;
  k.pf = (float)q.prior_floor;
  k.ct = (float)q.confidence_threshold;
  k.pf_margin = PH_QERR + FILTER_MARGIN * fabsf(k.pf);
  for (int i = 0; i < 9; ++i) k.w[i] = (float)q.weights[i];
  for (int c = 0; c < 3; ++c) {
    const double dd = q.weights[3 * c + 1] + q.weights[3 * c + 2];
    k.wbc_inv[c] = dd > 0.0 ? (float)(1.0 / dd) : 0.0f;
    k.ct_margin[c] = FILTER_MARGIN + fabsf(k.w[3 * c]) * PH_QERR;
  }
  // |v - chp| is an integer: d > eps  <=>  d > floor(eps)  (eps >= 0)
  const double e = q.chp_epsilon;
  k.eps_i = e < 0.0 ? -1 : (e >= 1e9 ? 1000000000 : (int)floor(e));
  k.sat = q.saturation_frames;
  return k;
}

// general path for the rare plane-pixels (returns by value: taking the
// address of the caller's HotOut would pin it to local memory)
template <typename T>
__device__ __forceinline__ HotOut hot_px_slow(const StepArgs* __restrict__ a,
                                              int s, int c, uint32_t p,
                                              Pre<T> pre, bool on_lat,
                                              const double* s_bt, int cls,
                                              bool member, double gmu,
                                              double gthr) {
  const Flags f{a->q.sampling_on != 0, a->q.grouping_on != 0,
                a->q.rate_scaling_on != 0, a->q.chp_on != 0,
                a->q.literal_conf != 0, a->q.compat != 0};
  const PlaneRef<T> pr = plane_ref<T>(*a, s, c);
  GroupConst gc;
  gc.ok = member;
  gc.mu = gmu;
  gc.thr = gthr;
  HotOut h;
  h.kind = 0;
  h.label = 0;
  h.deep = DEEP_NONE;
  h.conf = 0.0;
  h.rho = 0.0;
  h.rsel = 0;
  h.dyn = 0;
  hot_px<T>(*a, f, pr, p, pre, on_lat, s_bt, a->q.weights[3 * cls],
            a->q.weights[3 * cls + 1], a->q.weights[3 * cls + 2], gc, h);
  return h;
}

// single-instruction MUFU approximations (rel. error ~1 ulp): every value
// they feed is either continuous (within the fp32 tolerance) or a decision
// protected by the filter margins; operands are normal, positive floats
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float rsqrt_approx(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// filtered fp32 match: 1 hit, 0 miss, -1 undecided (within the margin)
// (margin: relative to the threshold plus a few ulp of 255 absolute, so the
// fp32 rounding of |v - mu| and of the threshold can never flip it)
__device__ __forceinline__ int fmatch(float vf, float mu, float thr) {
  const float gap = fabsf(vf - mu) - thr;
  const float m = FILTER_MARGIN * thr + MATCH_ABS_MARGIN;
  if (gap < -m) return 1;
  if (gap > m) return 0;
  return -1;
}

// exact operands of the binary64 path: f32 table entry at v, peak, and the
// two referenced modes (from the record)
__device__ __forceinline__ void load_exact(const float* table,
                                           const float* peak, const float* rec,
                                           uint32_t o, Pre<float>& x) {
  x.tv = __ldcg(table + (size_t)o * 256 + x.vb);
  x.peak = __ldg(peak + o);
  const uint32_t r0 = (x.meta >> 10) & 7u, r1 = x.meta >> 13;
  const float2 m0 = *reinterpret_cast<const float2*>(rec + 2 * r0);
  const float2 m1 = *reinterpret_cast<const float2*>(rec + 2 * r1);
  x.mu0 = m0.x;
  x.var0 = m0.y;
  x.mu1 = m1.x;
  x.var1 = m1.y;
}

#ifndef COG_FAST_MINB
#define COG_FAST_MINB 3
#endif

template <int KMAX, int D>
__global__ void __launch_bounds__(LEAN_THREADS, COG_FAST_MINB)
    fast_kernel(const __grid_constant__ StepArgs a,
                const __grid_constant__ FastConst k) {
  using T = float;
  constexpr int R = rec_elems(KMAX), WO = rec_w(KMAX);
  extern __shared__ double s_mem[];
  const int s = blockIdx.y;
  const int G = a.g.n_groups, K = a.g.k;
  const int H = a.g.height, W = a.g.width, stride = a.g.stride;
  const uint32_t P = (uint32_t)H * (uint32_t)W;
  const int words = acc_words(D, G);
  const int wpad = (words + 1) & ~1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool sampling = a.q.sampling_on != 0, grouping = a.q.grouping_on != 0;
  const bool compat = a.q.compat != 0, literal = a.q.literal_conf != 0;
  const bool chp_on = a.q.chp_on != 0, rate_on = a.q.rate_scaling_on != 0;

  // ---- shared: bterm tables (double for the slow path, float), group
  // constants, warp-private partial slices, warp worklist buffers
  double* s_bt = s_mem;
  double* s_gmu = s_bt + 256;
  double* s_gthr = s_gmu + D * G;
  unsigned long long* s_wacc =
      (unsigned long long*)(s_gthr + D * G);            // [warps][wpad]
  unsigned long long* s_qc = s_wacc + LEAN_WARPS * wpad; // [warps][FQ_CAP]
  double* s_qr = (double*)(s_qc + LEAN_WARPS * FQ_CAP);  // [warps][FQ_CAP]
  float* s_btf = (float*)(s_qr + LEAN_WARPS * FQ_CAP);   // [256]
  float* s_gmuf = s_btf + 256;                           // [D*G]
  float* s_gthrf = s_gmuf + D * G;                       // [D*G]
  for (int i = threadIdx.x; i < 256; i += LEAN_THREADS) {
    const double b = g_bterm[literal ? 1 : 0][i];
    s_bt[i] = b;
    s_btf[i] = (float)b;
  }
  {
    const double* gmu = a.s.g_mu + (size_t)s * D * G;
    const double* gvar = a.s.g_var + (size_t)s * D * G;
    for (int i = threadIdx.x; i < D * G; i += LEAN_THREADS) {
      s_gmu[i] = gmu[i];
      s_gthr[i] = a.q.match_lambda * sqrt(gvar[i]);
      s_gmuf[i] = (float)s_gmu[i];
      s_gthrf[i] = (float)s_gthr[i];
    }
  }
  for (int i = threadIdx.x; i < LEAN_WARPS * wpad; i += LEAN_THREADS)
    s_wacc[i] = 0ull;
  __syncthreads();
  // let the frame's deep kernel be scheduled now (it waits on this grid's
  // completion before touching anything); hides the launch gap
  asm volatile("griddepcontrol.launch_dependents;");
  unsigned long long* wacc = s_wacc + warp * wpad;
  unsigned long long* qc = s_qc + warp * FQ_CAP;
  double* qr = s_qr + warp * FQ_CAP;

  // 32-bit element indices from the state arrays' own bases (the launcher
  // guarantees streams * d * max(K, 5) * P and the record elements < 2^32);
  // the bases stay uniform
  const uint32_t sP = (uint32_t)s * D * P;      // [s][d][P] arrays
  const uint32_t sK = (uint32_t)s * D;          // plane index base
  const uint32_t s1 = (uint32_t)s * P;          // [s][P] arrays
  T* const mix_s = (T*)a.s.mix;
  T* const conf_s = (T*)a.conf;
  const float* const table_s = a.s.table;
  const float* const peak_s = a.s.peak;
  const uint16_t* const tabq_s = a.s.tabq;
  uint32_t* sync = a.s.sync + (size_t)s * 4;
  const size_t dq_cap = dq_capacity(D, P);
  unsigned long long* dq_code =
      (unsigned long long*)a.s.deepq + (size_t)s * dq_cap;
  double* dq_rho = a.s.deeprho + (size_t)s * dq_cap;
  const bool do_reset = (*(volatile uint32_t*)(sync + 1) & 1u) != 0;
  const bool do_reorder = a.reorder_now != 0;
  const GmmPar gp{a.q.match_lambda, a.q.background_threshold,
                  a.q.variance_floor, a.q.initial_variance};

  const int cw = a.cw;
  const int lrow = lane / cw, lcol = lane - lrow * cw;
  const bool lane_ok = lane < stride * cw;
  const bool on_lat = (lrow == 0) && (lcol % stride == 0);
  const int anchor = lcol - lcol % stride;

  unsigned long long kc = 0ull;  // pooled kind counts, 7 x 9 bits
  int kc_units = 0;
  int wq_n = 0;

  // static tile assignment over every resident slot: tile j of warp rank r
  // is r + j * nw.  Ranks are CTA-major (a CTA's warps on adjacent tiles:
  // shared rows stay in the same DRAM pages and L2 lines) when every warp
  // has many tiles; with few tiles per warp (C2: 2-3) the one-tile
  // difference between warps decides the SM balance, and ranks interleaved
  // over the CTAs spread the longer warps evenly.
  const int nw = gridDim.x * LEAN_WARPS;
  const bool spread = a.n_tiles / nw < 8;
  int wt = spread ? warp * gridDim.x + blockIdx.x
                  : blockIdx.x * LEAN_WARPS + warp;
  int ty = wt / a.tiles_x, tx = wt - ty * a.tiles_x;
  const int dty = nw / a.tiles_x, dtx = nw - dty * a.tiles_x;
  const int kc_flush = 511 / D;  // D counts per tile per 9-bit field
  unsigned fg_count = 0;
  for (; wt < a.n_tiles; wt += nw) {
    const int tile = wt;
    const int y = ty * stride + lrow, x_ = tx * cw + lcol;
    tx += dtx;
    ty += dty;
    if (tx >= a.tiles_x) {
      tx -= a.tiles_x;
      ty += 1;
    }
    const bool valid = lane_ok && y < H && x_ < W;
    const uint32_t p = valid ? (uint32_t)y * (uint32_t)W + (uint32_t)x_ : 0u;

    if (do_reset || do_reorder) {
      if (valid) {
        const int g0 = a.s.gid[s1 + p];
        const bool mem = G > 0 && g0 != (int)UNGROUPED;
#pragma unroll 1
        for (int c = 0; c < D; ++c) {
          const PlaneRef<T> pr = plane_ref<T>(a, s, c);
          if (do_reset) cold_reset<T, KMAX>(pr, p, a.q.initial_variance);
          if (do_reorder)
            cold_reorder<T>(pr, p, mem ? s_gmu[c * G + g0]
                                       : (G > 0 ? s_gmu[c * G] : 0.0));
        }
      }
      __syncwarp();
    }
    const int gid = valid ? (int)a.s.gid[s1 + p] : (int)UNGROUPED;
    const int cls = valid ? (int)a.s.cls[s1 + p] : 0;
    const bool member = valid && G > 0 && gid != (int)UNGROUPED;
    const float wa = k.w[3 * cls], wb = k.w[3 * cls + 1], wc = k.w[3 * cls + 2];
    const float ct_m = k.ct_margin[cls];
    const unsigned any_member = __ballot_sync(FULL, member);
    int fg = 0;

    // round 1 of every plane up front (pixel-indexed loads), then the
    // planes one at a time in a non-unrolled loop (the reference's planes
    // are independent, cascade.py:281): one dependent load round per plane,
    // a small register footprint
    Pre<T> n0, n1, n2;
    auto load1 = [&](int c, Pre<T>& x) {
      x.vb = 0;
      x.dyn = x.meta = x.streak = 0u;
      if (valid) {
        const uint32_t o = sP + (uint32_t)c * P + p;
        x.vb = a.frame[o];
        x.dyn = a.s.dyn[o];
        x.meta = a.s.meta[o];
        x.streak = a.s.streak[o];
      }
    };
    load1(0, n0);
    if (D > 1) load1(1, n1);
    if (D > 2) load1(2, n2);
#pragma unroll 1
    for (int c = 0; c < D; ++c) {
    const uint32_t o = sP + (uint32_t)c * P + p;
    T* const rec = mix_s + o * R;  // this plane-pixel's mixture record
    Pre<T> x = n0;
    if (D > 1) n0 = n1;
    if (D > 2) n1 = n2;
    x.tv = 0.0f;
    x.peak = 1.0f;
    x.mu0 = x.mu1 = 0.0f;
    x.var0 = x.var1 = 1.0f;
    const int gidx = member ? c * G + gid : 0;
    const float vf = (float)x.vb;
    const int chp = x.dyn & 0xFF;
    const int dv = abs(x.vb - chp);
    const bool changed = dv > k.eps_i;
    // rare gating states (sleeping / waking clock) and compat go to the
    // general path with exact operands
    bool slow = compat || (sampling && ((x.dyn >> 9 & 1u) || (x.dyn >> 16)));
    const bool ev = valid && !compat &&
                    will_evaluate(sampling, x.dyn, x.vb, on_lat,
                                  a.q.chp_epsilon);
    const uint32_t meta = x.meta;
    const uint32_t c0 = (meta >> 4) & 3u, c1 = (meta >> 6) & 3u,
                   c2 = (meta >> 8) & 3u;
    uint32_t top = c0;
    if (top == L_GROUP && !grouping) top = c1;
    const bool gtop = top == L_GROUP && member;
    const float gm = member ? s_gmuf[gidx] : 0.0f;
    const float gt_thr = member ? s_gthrf[gidx] : 1.0f;
    // the group test from shared memory: does the level walk stop at GROUP
    // before any mode level?  (only GROUP codes ahead of the first mode
    // code matter; an undecided test loads the modes and bails later)
    int ghit = (grouping && member) ? fmatch(vf, gm, gt_thr) : 0;
    bool need_modes = !gtop;
    if (!(chp_on && !changed)) {
      const bool walk_stops = (c0 == L_GROUP && ghit == 1);
      need_modes |= !walk_stops;
    }
    uint16_t q16 = 0;

    // ---- round 2: hot prior at v; the referenced modes if needed
    if (ev && !slow) {
      q16 = __ldcg(tabq_s + (((size_t)(sK + c) * a.n_tiles + tile) * 256 +
                             x.vb) * 32 + lane);
      if (need_modes) {
        const uint32_t r0 = (meta >> 10) & 7u, r1 = meta >> 13;
        const float2 m0 = *reinterpret_cast<const float2*>(rec + 2 * r0);
        const float2 m1 = *reinterpret_cast<const float2*>(rec + 2 * r1);
        x.mu0 = m0.x;
        x.var0 = m0.y;
        x.mu1 = m1.x;
        x.var1 = m1.y;
      }
    } else if (ev) {
      load_exact(table_s, peak_s, rec, o, x);
    }
    HotOut ho;
    ho.kind = 0;
    ho.label = 0;
    ho.deep = DEEP_NONE;
    ho.conf = 0.0;
    ho.rho = 0.0;
    ho.rsel = 0;
    ho.dyn = 0;
    if (valid) {
      const uint32_t dyn = x.dyn;
      int active = -1, label = 0;
      float cf = 0.0f;
      double rho = 0.0;
      uint32_t r0 = 0, r1 = 0;
      if (!slow) {
        r0 = (meta >> 10) & 7u;
        r1 = meta >> 13;
        const bool top1 = top == L_MEANVAR;
        float thr0 = 1.0f, thr1 = 1.0f;
        if (need_modes) {
          thr0 = k.lam * (x.var0 * rsqrt_approx(x.var0));
          thr1 = k.lam * (x.var1 * rsqrt_approx(x.var1));
        }
        const float mt = gtop ? gm : (top1 ? x.mu1 : x.mu0);
        const float dn = gtop ? gt_thr : (top1 ? thr1 : thr0);
        const float ph = (float)q16 * PH_Q;
        const float bt = s_btf[dv];
        float gt = fminf(fabsf(vf - mt) * rcp_approx(dn), 1.0f);
        if (!literal) gt = 1.0f - gt;
        if (ph < k.pf)
          cf = (wb * bt + wc * gt) * k.wbc_inv[cls];
        else
          cf = wa * ph + wb * bt + wc * gt;
        slow = fabsf(ph - k.pf) <= k.pf_margin ||
               fabsf(cf - k.ct) <= ct_m;
        if (chp_on && !changed) {
          active = L_CHP;
          label = (dyn >> 8) & 1u;
        } else {
          // first hit in mid_order; an undecided test on the path bails
#pragma unroll
          for (int j = 0; j < 3; ++j) {
            const uint32_t code = j == 0 ? c0 : (j == 1 ? c1 : c2);
            if (active >= 0 || code == 0) break;
            int hit;
            uint32_t rr = 0;
            if (code == L_GROUP) {
              hit = ghit;
            } else if (code == L_MEAN) {
              rr = r0;
              hit = fmatch(vf, x.mu0, thr0);
            } else {
              rr = r1;
              hit = fmatch(vf, x.mu1, thr1);
            }
            if (hit < 0) {
              slow = true;
              break;
            }
            if (hit && rr > 0) {
              // matched mode must sit inside the background weight prefix
              double acc = 0.0;
              for (uint32_t q = 0; q < rr; ++q)
                acc = acc + (double)rec[WO + q];
              hit = acc <= a.q.background_threshold;
            }
            if (hit) active = (int)code;
          }
          if (active < 0) active = L_GMM;
        }
        if (!slow) {
          rho = a.q.learning_rate;
          if (rate_on) {
            double relax = 1.0 - (double)cf;
            if (relax < a.q.rate_floor) relax = a.q.rate_floor;
            rho = a.q.learning_rate * relax;
          }
        } else {
          load_exact(table_s, peak_s, rec, o, x);  // rare: exact operands
        }
      }
      if (slow) {
        ho = hot_px_slow<T>(&a, s, c, p, x, on_lat, s_bt, cls, member,
                            member ? s_gmu[gidx] : 0.0,
                            member ? s_gthr[gidx] : 0.0);
      } else {
        // ---- bookkeeping of the fast path (kernels_numba.py:335-359)
        if (active == L_MEAN) {
          rec[2 * r0] = (float)((1.0 - rho) * (double)x.mu0 + rho * (double)x.vb);
        } else if (active == L_MEANVAR) {
          ho.deep = DEEP_MEANVAR;
          ho.rsel = (int)r1;
        } else if (active == L_GMM) {
          ho.deep = DEEP_GMM;
        }
        uint32_t sk = x.streak;
        if (cf > k.ct)
          sk = (sk == 0xffffffffu) ? sk : sk + 1u;
        else
          sk = 0u;
        a.s.streak[o] = sk;
        atomicAdd(a.s.hits + (((sK + c) * 5 + (uint32_t)active) * P + p), 1u);
        const int clock = (sampling && (long long)sk >= (long long)k.sat)
                              ? a.q.sleep_frames : (int)(dyn >> 16);
        ho.kind = active;
        ho.label = label;
        ho.conf = (double)cf;
        ho.rho = rho;
        ho.dyn = pack_dyn(x.vb, label, (dyn >> 9) & 1u, active, clock);
        if (active != L_GMM) a.s.dyn[o] = ho.dyn;
      }
      st(conf_s + o, ho.conf);
      a.kind[o] = (uint8_t)ho.kind;
      kc += 1ull << (9 * ho.kind);
    }
    int label = ho.label & 1;
    const bool is_copy = valid && ho.kind == K_COPY;
    const bool dq = valid && ho.deep != DEEP_NONE;
    const unsigned qm = __ballot_sync(FULL, dq);
    bool late = false;   // label arrives with the deep kernel
    bool gmm_now = false;
    if (qm) {
      if (__ballot_sync(FULL, is_copy)) {
        // copies in this plane-tile need their anchors' final labels now
        if (dq) {
          PlaneRef<T> pr = plane_ref<T>(a, s, c);
          if (ho.deep == DEEP_MEANVAR) {
            cold_meanvar<T, KMAX>(pr, p, x.meta, ho.rsel, (double)x.vb,
                                  ho.rho, a.q.variance_floor);
          } else {
            label = cold_gmm<T, KMAX>(pr, p, x.meta, (double)x.vb, ho.rho,
                                      gp, K, ho.deep == DEEP_GMM);
            gmm_now = true;
          }
        }
      } else {
        const int nq = __popc(qm);
        if (wq_n + nq > FQ_CAP) {
          unsigned base = 0;
          if (lane == 0) base = atomicAdd(sync + 3, (unsigned)wq_n);
          base = __shfl_sync(FULL, base, 0);
          __syncwarp();
          for (int e = lane; e < wq_n; e += 32) {
            dq_code[(size_t)base + e] = qc[e];
            dq_rho[(size_t)base + e] = qr[e];
          }
          __syncwarp();
          wq_n = 0;
        }
        if (dq) {
          const int pos = wq_n + __popc(qm & ((1u << lane) - 1u));
          qc[pos] = 1ull | ((unsigned long long)ho.deep << 1) |
                    ((unsigned long long)ho.rsel << 3) |
                    ((unsigned long long)c << 6) |
                    ((unsigned long long)x.vb << 8) |
                    ((unsigned long long)p << 16);
          qr[pos] = ho.rho;
          late = ho.deep == DEEP_GMM || ho.deep == DEEP_COMPAT;
        }
        wq_n += nq;
      }
    }

    // ---- labels of this plane: GMM now / later, copies from anchors
    if (gmm_now) a.s.dyn[o] = ho.dyn | ((uint32_t)label << 8);
    if (late) {
      label = 0;  // the deep kernel sets the label bit
      a.s.dyn[o] = ho.dyn;
    }
    const int al = __shfl_sync(FULL, label, anchor);
    if (is_copy) {
      label = al;
      a.s.dyn[o] = ho.dyn | ((uint32_t)al << 8);
    }
    fg |= label;

    // ---- group partials (exact sums) into the warp's private slice
    if (any_member) {
      unsigned todo = any_member;
      while (todo) {
        const int leader = __ffs(todo) - 1;
        const int g = __shfl_sync(FULL, gid, leader);
        const bool mine = member && gid == g;
        const unsigned mm = __ballot_sync(FULL, mine);
        todo &= ~mm;
        const unsigned sall = warp_sum_u32(mine ? (unsigned)x.vb : 0u);
        const bool hit = mine && ho.kind == L_GROUP;
        const unsigned hm = __ballot_sync(FULL, hit);
        unsigned sv = 0, qh = 0, ql = 0;
        if (hm) {
          unsigned long long qv = 0;
          if (hit) {
            const double cq = ho.conf * 4503599627370496.0;  // 2^52
            qv = cq > 0.0 ? (unsigned long long)cq : 0ull;
          }
          sv = warp_sum_u32(hit ? (unsigned)x.vb : 0u);
          qh = warp_sum_u32((unsigned)(qv >> CONF_SPLIT));
          ql = warp_sum_u32((unsigned)(qv & ((1ull << CONF_SPLIT) - 1ull)));
        }
        if (lane == 0) {
          unsigned long long* e = wacc + acc_grp(D, G, c, g);
          e[4] += sall;
          e[5] += (unsigned long long)__popc(mm);
          if (hm) {
            e[0] += (unsigned long long)__popc(hm);
            e[1] += sv;
            e[2] += qh;
            e[3] += ql;
          }
        }
      }
    }
    }  // planes

    if (valid) a.mask[s1 + p] = fg ? 255 : 0;
    fg_count += __popc(__ballot_sync(FULL, valid && fg));
    if (++kc_units >= kc_flush) {
#pragma unroll
      for (int q = 0; q < 7; ++q) {
        const unsigned v = warp_sum_u32((unsigned)((kc >> (9 * q)) & 511u));
        if (lane == 0) wacc[acc_kind(0, q)] += v;
      }
      kc = 0ull;
      kc_units = 0;
    }
  }
  if (wq_n) {
    unsigned base = 0;
    if (lane == 0) base = atomicAdd(sync + 3, (unsigned)wq_n);
    base = __shfl_sync(FULL, base, 0);
    __syncwarp();
    for (int e = lane; e < wq_n; e += 32) {
      dq_code[(size_t)base + e] = qc[e];
      dq_rho[(size_t)base + e] = qr[e];
    }
  }
#pragma unroll
  for (int q = 0; q < 7; ++q) {
    const unsigned v = warp_sum_u32((unsigned)((kc >> (9 * q)) & 511u));
    if (lane == 0) wacc[acc_kind(0, q)] += v;
  }
  if (lane == 0) wacc[acc_fg(D)] += fg_count;
  __syncthreads();
  unsigned long long* gacc = (unsigned long long*)a.s.accum + (size_t)s * words;
  for (int i = threadIdx.x; i < words; i += LEAN_THREADS) {
    unsigned long long v = 0;
#pragma unroll
    for (int w = 0; w < LEAN_WARPS; ++w) v += s_wacc[w * wpad + i];
    if (v) atomicAdd(gacc + i, v);
  }
}

__host__ inline size_t fast_smem_bytes(int d, int G) {
  const size_t words = (size_t)acc_words(d, G);
  return 256 * 8 + (size_t)2 * d * G * 8 +
         (size_t)LEAN_WARPS * ((words + 1) & ~(size_t)1) * 8 +
         (size_t)LEAN_WARPS * FQ_CAP * 16 + 256 * 4 + (size_t)2 * d * G * 4;
}
