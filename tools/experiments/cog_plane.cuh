// cog_plane.cuh -- plane_kernel: the float32-state hot pass of the frame
// step with one thread per PLANE-pixel (kernels_numba.py:188-359; the
// reference runs its planes independently, cascade.py:281).  Included
// inside the anonymous namespace of cog_kernels.cu, after cog_frame.cuh.
//
// Layout of a CTA iteration: NT warp tiles (stride rows x cw columns, as
// everywhere) x D planes; warp (t, c) owns plane c of tile t, one lane per
// pixel.  A thread therefore carries one plane's state: a short serial
// path and a small register footprint (many resident warps hide the two
// load rounds), instead of fast_kernel's three planes per thread (80
// registers, spills, ~550 instructions per plane-pixel).  The planes of a
// pixel meet in shared memory: each warp writes its lane labels, one
// barrier per iteration (double-buffered), and the plane-0 warp of the
// tile ORs them into the mask.  Copies resolve in-warp (anchor = row 0 of
// the same tile and plane).  Rare cases run in place: fp32 decisions inside
// the filter margin are redone in binary64 out of line, a pending
// illumination reset / scheduled reorder is applied per plane-pixel first
// (cold_reset / cold_reorder), and a warp with copies does its deep updates
// in place so the anchors' labels are final.  MEANVAR hits and GMM
// fall-throughs otherwise go to the stream's deep worklist (deep_kernel).

#ifndef COG_PLANE_MINB
#define COG_PLANE_MINB 1
#endif

template <int D>
struct PlaneShape {
  static constexpr int NT = (D == 1) ? 8 : 4;  // tiles per CTA iteration
  static constexpr int WARPS = NT * D;
  static constexpr int THREADS = WARPS * 32;
};

__host__ inline size_t plane_smem_bytes(int d, int G, int warps, int nt) {
  const size_t words = (size_t)acc_words(d, G);
  return (size_t)warps * ((words + 1) & ~(size_t)1) * 8 +  // partials
         (size_t)warps * FQ_CAP * 16 +                      // worklist bufs
         (size_t)2 * nt * d * 32 +                          // labels x2
         256 * 4 + (size_t)2 * d * G * 4;                   // bterm, groups
}

template <int KMAX, int D>
__global__ void __launch_bounds__(PlaneShape<D>::THREADS, COG_PLANE_MINB)
    plane_kernel(const __grid_constant__ StepArgs a,
                 const __grid_constant__ FastConst k) {
  using T = float;
  constexpr int NT = PlaneShape<D>::NT;
  constexpr int WARPS = PlaneShape<D>::WARPS;
  extern __shared__ unsigned long long pk_mem[];
  const int s = blockIdx.y;
  const int G = a.g.n_groups, K = a.g.k;
  const int H = a.g.height, W = a.g.width, stride = a.g.stride;
  const uint32_t P = (uint32_t)H * (uint32_t)W;
  const int words = acc_words(D, G);
  const int wpad = (words + 1) & ~1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tl = warp / D, c = warp - tl * D;  // tile slot, plane
  const bool sampling = a.q.sampling_on != 0, grouping = a.q.grouping_on != 0;
  const bool literal = a.q.literal_conf != 0;
  const bool chp_on = a.q.chp_on != 0, rate_on = a.q.rate_scaling_on != 0;

  unsigned long long* s_wacc = pk_mem;                     // [WARPS][wpad]
  unsigned long long* s_qc = s_wacc + WARPS * wpad;        // [WARPS][FQ_CAP]
  double* s_qr = (double*)(s_qc + WARPS * FQ_CAP);         // [WARPS][FQ_CAP]
  uint8_t* s_lab = (uint8_t*)(s_qr + WARPS * FQ_CAP);      // [2][NT][D][32]
  float* s_btf = (float*)(s_lab + 2 * NT * D * 32);        // [256]
  float* s_gmuf = s_btf + 256;                             // [D*G]
  float* s_gthrf = s_gmuf + D * G;                         // [D*G]
  for (int i = threadIdx.x; i < 256; i += WARPS * 32)
    s_btf[i] = (float)g_bterm[literal ? 1 : 0][i];
  {
    const double* gmu = a.s.g_mu + (size_t)s * D * G;
    const double* gvar = a.s.g_var + (size_t)s * D * G;
    for (int i = threadIdx.x; i < D * G; i += WARPS * 32) {
      s_gmuf[i] = (float)gmu[i];
      s_gthrf[i] = (float)(a.q.match_lambda * sqrt(gvar[i]));
    }
  }
  for (int i = threadIdx.x; i < WARPS * wpad; i += WARPS * 32)
    s_wacc[i] = 0ull;
  __syncthreads();
  unsigned long long* wacc = s_wacc + warp * wpad;
  unsigned long long* qc = s_qc + warp * FQ_CAP;
  double* qr = s_qr + warp * FQ_CAP;

  // this warp's plane: every per-plane-pixel array from its own base
  const uint32_t sc = (uint32_t)s * D + (uint32_t)c;
  const uint8_t* frame_c = a.frame + (size_t)sc * P;
  uint32_t* dyn_c = a.s.dyn + (size_t)sc * P;
  uint16_t* meta_c = a.s.meta + (size_t)sc * P;
  uint32_t* stk_c = a.s.streak + (size_t)sc * P;
  const float* peak_c = a.s.peak + (size_t)sc * P;
  const float* tab_c = a.s.table + (size_t)sc * P * 256;
  T* mu_c = (T*)a.s.mu + (size_t)sc * K * P;
  T* var_c = (T*)a.s.var + (size_t)sc * K * P;
  T* w_c = (T*)a.s.w + (size_t)sc * K * P;
  uint32_t* hits_c = a.s.hits + (size_t)sc * 5 * P;
  T* conf_c = (T*)a.conf + (size_t)sc * P;
  uint8_t* kind_c = a.kind + (size_t)sc * P;
  const uint16_t* gid_s = a.s.gid + (size_t)s * P;
  const uint8_t* cls_s = a.s.cls + (size_t)s * P;
  uint8_t* mask_s = a.mask + (size_t)s * P;

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

  unsigned long long kc = 0ull;  // kind counts of this plane, 7 x 9 bits
  int kc_units = 0;
  int wq_n = 0;
  unsigned fg_count = 0;
  int buf = 0;

  const int n_iter = (a.n_tiles + NT - 1) / NT;
  for (int it = blockIdx.x; it < n_iter; it += gridDim.x) {
    const int tile = it * NT + tl;
    const int ty = tile / a.tiles_x, tx = tile - ty * a.tiles_x;
    const int y = ty * stride + lrow, x_ = tx * cw + lcol;
    const bool valid = tile < a.n_tiles && lane_ok && y < H && x_ < W;
    const uint32_t p = valid ? (uint32_t)y * (uint32_t)W + (uint32_t)x_ : 0u;

    if (do_reset || do_reorder) {
      if (valid) {
        const PlaneRef<T> pr = plane_ref<T>(a, s, c);
        const int g0 = gid_s[p];
        const bool mem = G > 0 && g0 != (int)UNGROUPED;
        if (do_reset) cold_reset<T, KMAX>(pr, p, a.q.initial_variance);
        if (do_reorder)
          cold_reorder<T>(pr, p, mem ? (double)a.s.g_mu[(size_t)s * D * G + c * G + g0]
                                     : (G > 0 ? a.s.g_mu[(size_t)s * D * G + c * G] : 0.0));
      }
      __syncwarp();
    }

    // ---- round 1: pixel-indexed loads
    int vb = 0, gid = (int)UNGROUPED, cls = 0;
    uint32_t dy = 0u, meta = 0u, stk = 0u;
    float peak = 1.0f;
    if (valid) {
      vb = frame_c[p];
      dy = dyn_c[p];
      meta = meta_c[p];
      stk = stk_c[p];
      peak = __ldg(peak_c + p);
      gid = gid_s[p];
      cls = cls_s[p];
    }
    const bool member = valid && G > 0 && gid != (int)UNGROUPED;
    const int dv = abs(vb - (int)(dy & 0xFFu));
    const bool changed = dv > k.eps_i;
    // ---- sampling gate (kernels_numba.py:193-216)
    int kind = -1;      // SKIP / COPY decided here, else the active level
    bool zs = false;    // woke on change: streak restarts
    if (valid && sampling) {
      if (dy >> 16) {
        if (!changed) kind = K_SKIP;
        else zs = true;
      } else if ((dy >> 9 & 1u) && !changed && !on_lat) {
        kind = K_COPY;
      }
    }
    const bool eval = valid && kind < 0;
    const uint32_t r0 = (meta >> 10) & 7u, r1 = meta >> 13;

    // ---- round 2: table entry at v, the referenced modes, weight prefix
    float tv = 0.0f, mu0 = 0.0f, var0 = 1.0f, mu1 = 0.0f, var1 = 1.0f;
    float wq[KMAX > 1 ? KMAX - 1 : 1];
#pragma unroll
    for (int q = 0; q < (KMAX > 1 ? KMAX - 1 : 1); ++q) wq[q] = 0.0f;
    if (eval) {
      tv = __ldcg(tab_c + (((size_t)p << 8) | (uint32_t)vb));
      mu0 = mu_c[r0 * P + p];
      var0 = var_c[r0 * P + p];
      if (r1 != r0) {
        mu1 = mu_c[r1 * P + p];
        var1 = var_c[r1 * P + p];
      } else {
        mu1 = mu0;
        var1 = var0;
      }
      const uint32_t rm = r0 > r1 ? r0 : r1;
#pragma unroll
      for (int q = 0; q < KMAX - 1; ++q)
        if ((uint32_t)q < rm) wq[q] = w_c[(uint32_t)q * P + p];
    }

    // ---- decisions (fp32, filtered; binary64 out of line in the margin)
    int label = 0;
    float cf = 0.0f;
    bool sat = false;
    const int gidx = member ? c * G + gid : 0;
    if (eval) {
      const float wa = k.w[3 * cls], wb = k.w[3 * cls + 1], wc = k.w[3 * cls + 2];
      const float vf = (float)vb;
      const uint32_t c0 = (meta >> 4) & 3u, c1 = (meta >> 6) & 3u,
                     c2 = (meta >> 8) & 3u;
      uint32_t top = c0;
      if (top == L_GROUP && !grouping) top = c1;
      const bool gtop = top == L_GROUP && member;
      const bool top1 = top == L_MEANVAR;
      const float thr0 = k.lam * (var0 * rsqrt_approx(var0)),
                  thr1 = k.lam * (var1 * rsqrt_approx(var1));
      const float gm = member ? s_gmuf[gidx] : 0.0f;
      const float gt_thr = member ? s_gthrf[gidx] : 1.0f;
      const float mt = gtop ? gm : (top1 ? mu1 : mu0);
      const float dn = gtop ? gt_thr : (top1 ? thr1 : thr0);
      const float ph = tv * rcp_approx(peak);
      const float bt = s_btf[dv];
      float gt = fminf(fabsf(vf - mt) * rcp_approx(dn), 1.0f);
      if (!literal) gt = 1.0f - gt;
      if (ph < k.pf)
        cf = (wb * bt + wc * gt) * k.wbc_inv[cls];
      else
        cf = wa * ph + wb * bt + wc * gt;
      sat = cf > k.ct;
      if (fabsf(ph - k.pf) <= FILTER_MARGIN * k.pf + 1e-30f ||
          fabsf(cf - k.ct) <= FILTER_MARGIN) {
        const double ce = frame_conf_exact(
            &a, gtop ? (int)((size_t)s * D * G + gidx) : -1, vb,
            (int)(dy & 0xFFu), top1 ? mu1 : mu0, top1 ? var1 : var0, tv,
            peak, cls);
        sat = ce > a.q.confidence_threshold;
        cf = (float)ce;
      }
      if (chp_on && !changed) {
        kind = L_CHP;
        label = (dy >> 8) & 1u;
      } else {
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          const uint32_t code = j == 0 ? c0 : (j == 1 ? c1 : c2);
          if (kind >= 0 || code == 0) break;
          int hit;
          uint32_t rr = 0;
          if (code == L_GROUP) {
            hit = (grouping && member) ? fmatch(vf, gm, gt_thr) : 0;
          } else if (code == L_MEAN) {
            rr = r0;
            hit = fmatch(vf, mu0, thr0);
          } else {
            rr = r1;
            hit = fmatch(vf, mu1, thr1);
          }
          if (hit < 0) {
            if (code == L_GROUP) {
              const size_t gi = (size_t)s * D * G + gidx;
              hit = match_exact((double)vb, a.s.g_mu[gi], a.s.g_var[gi],
                                a.q.match_lambda);
            } else {
              hit = match_exact((double)vb, (double)(code == L_MEAN ? mu0 : mu1),
                                (double)(code == L_MEAN ? var0 : var1),
                                a.q.match_lambda);
            }
          }
          if (hit && rr > 0) {
            // matched mode must sit inside the background weight prefix
            double acc = 0.0;
#pragma unroll
            for (int q = 0; q < KMAX - 1; ++q)
              if ((uint32_t)q < rr) acc = acc + (double)wq[q];
            hit = acc <= a.q.background_threshold;
          }
          if (hit) kind = (int)code;
        }
        if (kind < 0) kind = L_GMM;
      }
    }

    // ---- bookkeeping (kernels_numba.py:335-359)
    int deep = DEEP_NONE;
    double rho = 0.0;
    uint32_t dnew = 0u;
    if (valid) {
      if (kind == K_SKIP) {
        // clock -1, waking on its last tick; label, last_active kept
        const int clock = (int)(dy >> 16) - 1;
        label = (dy >> 8) & 1u;
        dnew = pack_dyn(vb, label, clock == 0 ? 1 : (int)((dy >> 9) & 1u),
                        (int)((dy >> 10) & 7u) - 1, clock);
      } else if (kind == K_COPY) {
        // label from the anchor below
        dnew = pack_dyn(vb, 0, 0, (int)((dy >> 10) & 7u) - 1, a.q.sleep_frames);
      } else {
        rho = a.q.learning_rate;
        if (rate_on) {
          double relax = 1.0 - (double)cf;
          if (relax < a.q.rate_floor) relax = a.q.rate_floor;
          rho = a.q.learning_rate * relax;
        }
        if (kind == L_MEAN)
          st(mu_c + (r0 * P + p), (1.0 - rho) * (double)mu0 + rho * (double)vb);
        else if (kind == L_MEANVAR)
          deep = DEEP_MEANVAR;
        else if (kind == L_GMM)
          deep = DEEP_GMM;
        uint32_t sk = zs ? 0u : stk;
        if (sat)
          sk = (sk == 0xffffffffu) ? sk : sk + 1u;
        else
          sk = 0u;
        stk_c[p] = sk;
        atomicAdd(hits_c + ((uint32_t)kind * P + p), 1u);
        // after the gate an evaluated pixel has clock 0 and waking 0
        // (sampling on); with sampling off both are carried unchanged
        const int clock = sampling ? ((long long)sk >= (long long)k.sat
                                          ? a.q.sleep_frames : 0)
                                   : (int)(dy >> 16);
        const int waking = sampling ? 0 : (int)((dy >> 9) & 1u);
        dnew = pack_dyn(vb, label, waking, kind, clock);
      }
      st(conf_c + p, (double)cf);
      kind_c[p] = (uint8_t)kind;
      kc += 1ull << (9 * kind);
    }

    // ---- deep work: queued, or in place when copies need final labels
    const bool is_copy = kind == K_COPY;
    const bool dq = deep != DEEP_NONE;
    const unsigned qm = __ballot_sync(FULL, dq);
    if (qm) {
      if (__ballot_sync(FULL, is_copy)) {
        if (dq) {
          const PlaneRef<T> pr = plane_ref<T>(a, s, c);
          if (deep == DEEP_MEANVAR)
            cold_meanvar<T, KMAX>(pr, p, meta, (int)r1, (double)vb, rho,
                                  a.q.variance_floor);
          else
            label = cold_gmm<T, KMAX>(pr, p, meta, (double)vb, rho, gp, K, 1);
          dnew |= (uint32_t)label << 8;
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
          qc[pos] = 1ull | ((unsigned long long)deep << 1) |
                    ((unsigned long long)(deep == DEEP_MEANVAR ? r1 : 0u) << 3) |
                    ((unsigned long long)c << 6) |
                    ((unsigned long long)vb << 8) |
                    ((unsigned long long)p << 16);
          qr[pos] = rho;
        }
        wq_n += nq;
      }
    }
    const int al = __shfl_sync(FULL, label, anchor);
    if (is_copy) {
      label = al;
      dnew |= (uint32_t)al << 8;
    }
    if (valid) dyn_c[p] = dnew;  // a GMM label arrives with the deep pass

    // ---- group partials (exact sums) into the warp's private slice
    const unsigned any_member = __ballot_sync(FULL, member);
    if (any_member) {
      unsigned todo = any_member;
      while (todo) {
        const int leader = __ffs(todo) - 1;
        const int g = __shfl_sync(FULL, gid, leader);
        const bool mine = member && gid == g;
        const unsigned mm = __ballot_sync(FULL, mine);
        todo &= ~mm;
        const unsigned sall = warp_sum_u32(mine ? (unsigned)vb : 0u);
        const bool hit = mine && kind == L_GROUP;
        const unsigned hm = __ballot_sync(FULL, hit);
        unsigned sv = 0, qh = 0, ql = 0;
        if (hm) {
          unsigned long long qv = 0;
          if (hit) {
            const double cq = (double)cf * 4503599627370496.0;  // 2^52
            qv = cq > 0.0 ? (unsigned long long)cq : 0ull;
          }
          sv = warp_sum_u32(hit ? (unsigned)vb : 0u);
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

    // ---- union mask: planes meet in shared memory (one barrier)
    uint8_t* lab = s_lab + (size_t)buf * NT * D * 32;
    lab[(tl * D + c) * 32 + lane] = (uint8_t)(label & 1);
    __syncthreads();
    if (c == 0) {
      int fg = 0;
#pragma unroll
      for (int cc = 0; cc < D; ++cc) fg |= lab[(tl * D + cc) * 32 + lane];
      if (valid) mask_s[p] = fg ? 255 : 0;
      fg_count += __popc(__ballot_sync(FULL, valid && fg));
    }
    buf ^= 1;
    if (++kc_units >= 511) {
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
  for (int i = threadIdx.x; i < words; i += WARPS * 32) {
    unsigned long long v = 0;
    for (int w = 0; w < WARPS; ++w) v += s_wacc[w * wpad + i];
    if (v) atomicAdd(gacc + i, v);
  }
}
