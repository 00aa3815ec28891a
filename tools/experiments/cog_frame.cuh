// cog_frame.cuh -- frame_kernel: the float32-state hot pass of the frame
// step (kernels_numba.py:188-359 for the common case).  Included inside the
// anonymous namespace of cog_kernels.cu, after cog_fast.cuh.
//
// Why a second hot kernel: fast_kernel (LIST = false) is latency-bound --
// one dependent load round per plane (table entry at v, the referenced
// modes), a third for the background-weight prefix, and the general
// binary64 path inlined beside the fast one (80 registers, spills, 3 CTAs
// per SM).  frame_kernel restructures the warp tile around one load round:
//   * the frame bytes and meta words of the NEXT tile are prefetched while
//     the current tile computes, so every address of a tile is known when
//     it starts: table entry at v, both referenced modes and the weight
//     prefix of every plane go out as one batch;
//   * pass 1 makes every plane's decisions without writing anything: the
//     sampling gate (SKIP, wake on change), the confidence and the level
//     walk in fp32, filtered as in fast_kernel -- an fp32 decision inside
//     the filter margin is redone in binary64 in place (out of line);
//   * a tile with a COPY pixel (its anchor's final label is needed) is
//     deferred whole -- appended to the stream's deferred-tile list and
//     left untouched -- and fast_kernel<LIST = true> runs it after this
//     kernel through the general path, which resolves copies.  Frames
//     with a pending illumination reset or reorder, and compat mode, defer
//     every tile;
//   * pass 2 does the bookkeeping, queues MEANVAR hits and GMM
//     fall-throughs for the deep worklist, and accumulates the exact
//     partials exactly as fast_kernel does.
// The deferred list shares the worklist buffer: tiles from the back (count
// in sync[2]), worklist items from the front (count in sync[3]).  A
// deferred tile queues nothing, so items + tiles <= d * P always fits.

#ifdef COG_PROF  // debug counters of the deferral reasons (cog_debug_prof)
#define FRAME_DBG(i) atomicAdd(&g_prof[i], 1ull)
#else
#define FRAME_DBG(i)
#endif

#ifndef COG_FRAME_MINB
#define COG_FRAME_MINB 3
#endif

__host__ inline size_t frame_smem_bytes(int d, int G) {
  const size_t words = (size_t)acc_words(d, G);
  return (size_t)LEAN_WARPS * ((words + 1) & ~(size_t)1) * 8 +
         (size_t)LEAN_WARPS * FQ_CAP * 16 + 256 * 4 + (size_t)2 * d * G * 4;
}

// the reference's binary64 confidence for a plane-pixel whose fp32 one
// fell inside the filter margin (kernels_numba.py:243-270); gi >= 0 selects
// the group (g_mu, g_var) as the top level.  Out of line: small register footprint
// at the (rare) call site.
__device__ __noinline__ double frame_conf_exact(const StepArgs* __restrict__ a,
                                                int gi, int vb, int chp,
                                                float mu_top, float var_top,
                                                float tv, float peak, int cls) {
  double mtd, dnd;
  if (gi >= 0) {
    mtd = a->s.g_mu[gi];
    dnd = a->q.match_lambda * sqrt(a->s.g_var[gi]);
  } else {
    mtd = (double)mu_top;
    dnd = a->q.match_lambda * sqrt((double)var_top);
  }
  const double ce = conf_exact((double)vb, (double)chp, mtd, dnd, (double)tv,
                               (double)peak, a->q.weights[3 * cls],
                               a->q.weights[3 * cls + 1],
                               a->q.weights[3 * cls + 2], a->q.prior_floor,
                               a->q.literal_conf);
  return ce;
}

template <int KMAX, int D>
__global__ void __launch_bounds__(LEAN_THREADS, COG_FRAME_MINB)
    frame_kernel(const __grid_constant__ StepArgs a,
                 const __grid_constant__ FastConst k) {
  using T = float;
  extern __shared__ unsigned long long f_mem[];
  const int s = blockIdx.y;
  const int G = a.g.n_groups, K = a.g.k;
  const int H = a.g.height, W = a.g.width, stride = a.g.stride;
  const uint32_t P = (uint32_t)H * (uint32_t)W;
  const int words = acc_words(D, G);
  const int wpad = (words + 1) & ~1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool sampling = a.q.sampling_on != 0, grouping = a.q.grouping_on != 0;
  const bool literal = a.q.literal_conf != 0;
  const bool chp_on = a.q.chp_on != 0, rate_on = a.q.rate_scaling_on != 0;

  // ---- shared: warp-private partial slices, warp worklist buffers, the
  // float bterm table and group constants
  unsigned long long* s_wacc = f_mem;                      // [warps][wpad]
  unsigned long long* s_qc = s_wacc + LEAN_WARPS * wpad;   // [warps][FQ_CAP]
  double* s_qr = (double*)(s_qc + LEAN_WARPS * FQ_CAP);    // [warps][FQ_CAP]
  float* s_btf = (float*)(s_qr + LEAN_WARPS * FQ_CAP);     // [256]
  float* s_gmuf = s_btf + 256;                             // [D*G]
  float* s_gthrf = s_gmuf + D * G;                         // [D*G]
  for (int i = threadIdx.x; i < 256; i += LEAN_THREADS)
    s_btf[i] = (float)g_bterm[literal ? 1 : 0][i];
  {
    const double* gmu = a.s.g_mu + (size_t)s * D * G;
    const double* gvar = a.s.g_var + (size_t)s * D * G;
    for (int i = threadIdx.x; i < D * G; i += LEAN_THREADS) {
      s_gmuf[i] = (float)gmu[i];
      s_gthrf[i] = (float)(a.q.match_lambda * sqrt(gvar[i]));
    }
  }
  for (int i = threadIdx.x; i < LEAN_WARPS * wpad; i += LEAN_THREADS)
    s_wacc[i] = 0ull;
  __syncthreads();
  asm volatile("griddepcontrol.launch_dependents;");
  unsigned long long* wacc = s_wacc + warp * wpad;
  unsigned long long* qc = s_qc + warp * FQ_CAP;
  double* qr = s_qr + warp * FQ_CAP;

  const uint32_t sP = (uint32_t)s * D * P;  // [s][d][P] arrays
  const uint32_t sK = (uint32_t)s * D;      // plane index base
  const uint32_t s1 = (uint32_t)s * P;      // [s][P] arrays
  T* const mu_s = (T*)a.s.mu;
  T* const var_s = (T*)a.s.var;
  T* const w_s = (T*)a.s.w;
  T* const conf_s = (T*)a.conf;
  uint32_t* sync = a.s.sync + (size_t)s * 4;
  const size_t dq_cap = dq_capacity(D, P);
  unsigned long long* dq_code =
      (unsigned long long*)a.s.deepq + (size_t)s * dq_cap;
  double* dq_rho = a.s.deeprho + (size_t)s * dq_cap;
  const bool defer_all = a.q.compat != 0 || a.reorder_now != 0 ||
                         (*(volatile uint32_t*)(sync + 1) & 1u) != 0;

  const int cw = a.cw;
  const int lrow = lane / cw, lcol = lane - lrow * cw;
  const bool lane_ok = lane < stride * cw;
  const bool on_lat = (lrow == 0) && (lcol % stride == 0);

  unsigned long long kc = 0ull;  // pooled kind counts, 7 x 9 bits
  int kc_units = 0;
  const int kc_flush = 511 / D;
  int wq_n = 0;
  unsigned fg_count = 0;

  auto defer_tile = [&](int tile) {
    if (lane == 0) {
      const unsigned j = atomicAdd(sync + 2, 1u);
      dq_code[dq_cap - 1 - j] = ((unsigned long long)tile << 1) | 1ull;
    }
  };

  // static, balanced tile assignment: tile j of warp gw is gw + j * nw
  const int nw = gridDim.x * LEAN_WARPS;
  int wt = blockIdx.x * LEAN_WARPS + warp;
  if (defer_all) {
    for (; wt < a.n_tiles; wt += nw) defer_tile(wt);
    wt = a.n_tiles;  // nothing else to do (partials stay zero)
  }
  int ty = wt / a.tiles_x, tx = wt - ty * a.tiles_x;
  const int dty = nw / a.tiles_x, dtx = nw - dty * a.tiles_x;

  // pixel of this lane in tile (ty, tx)
  auto pix = [&](int t, int yy, int xx, uint32_t& p) {
    const int y = yy * stride + lrow, x_ = xx * cw + lcol;
    const bool v = t < a.n_tiles && lane_ok && y < H && x_ < W;
    p = v ? (uint32_t)y * (uint32_t)W + (uint32_t)x_ : 0u;
    return v;
  };

  // ---- prefetch of the first tile: frame bytes and meta words
  uint32_t pf_p;
  bool pf_valid = pix(wt, ty, tx, pf_p);
  int pf_vb[D];
  uint32_t pf_meta[D];
#pragma unroll
  for (int c = 0; c < D; ++c) {
    pf_vb[c] = 0;
    pf_meta[c] = 0u;
    if (pf_valid) {
      pf_vb[c] = a.frame[sP + (uint32_t)c * P + pf_p];
      pf_meta[c] = a.s.meta[sP + (uint32_t)c * P + pf_p];
    }
  }

  for (; wt < a.n_tiles; wt += nw) {
    const int tile = wt;
    const uint32_t p = pf_p;
    const bool valid = pf_valid;
    int vbs[D];
    uint32_t metas[D];
#pragma unroll
    for (int c = 0; c < D; ++c) {
      vbs[c] = pf_vb[c];
      metas[c] = pf_meta[c];
    }
    // ---- prefetch the next tile's frame bytes and meta words
    tx += dtx;
    ty += dty;
    if (tx >= a.tiles_x) {
      tx -= a.tiles_x;
      ty += 1;
    }
    pf_valid = pix(wt + nw, ty, tx, pf_p);
#pragma unroll
    for (int c = 0; c < D; ++c) {
      if (pf_valid) {
        pf_vb[c] = a.frame[sP + (uint32_t)c * P + pf_p];
        pf_meta[c] = a.s.meta[sP + (uint32_t)c * P + pf_p];
      }
    }

    // ---- one round of loads for every plane of this tile
    const int gid = valid ? (int)a.s.gid[s1 + p] : (int)UNGROUPED;
    const int cls = valid ? (int)a.s.cls[s1 + p] : 0;
    uint32_t dyn[D], stk[D];
    float peak[D], tv[D], mu0[D], var0[D], mu1[D], var1[D];
    float wq[D][KMAX > 1 ? KMAX - 1 : 1];
#pragma unroll
    for (int c = 0; c < D; ++c) {
      const uint32_t o = sP + (uint32_t)c * P + p;
      const uint32_t mb = (sK + c) * K * P + p;
      const uint32_t r0 = (metas[c] >> 10) & 7u, r1 = metas[c] >> 13;
      const uint32_t rm = r0 > r1 ? r0 : r1;
      dyn[c] = stk[c] = 0u;
      peak[c] = 1.0f;
      tv[c] = 0.0f;
      mu0[c] = mu1[c] = 0.0f;
      var0[c] = var1[c] = 1.0f;
#pragma unroll
      for (int q = 0; q < (KMAX > 1 ? KMAX - 1 : 1); ++q) wq[c][q] = 0.0f;
      if (valid) {
        dyn[c] = a.s.dyn[o];
        stk[c] = a.s.streak[o];
        peak[c] = __ldg(a.s.peak + o);
        tv[c] = __ldcg(a.s.table + (((size_t)o << 8) | (uint32_t)vbs[c]));
        mu0[c] = mu_s[mb + r0 * P];
        var0[c] = var_s[mb + r0 * P];
        if (r1 != r0) {
          mu1[c] = mu_s[mb + r1 * P];
          var1[c] = var_s[mb + r1 * P];
        }
#pragma unroll
        for (int q = 0; q < KMAX - 1; ++q)
          if ((uint32_t)q < rm) wq[c][q] = w_s[mb + (uint32_t)q * P];
      }
    }
    const bool member = valid && G > 0 && gid != (int)UNGROUPED;
    const float wa = k.w[3 * cls], wb = k.w[3 * cls + 1], wc = k.w[3 * cls + 2];

    // ---- pass 1: every plane's decisions, no writes
    int res[D];   // kind | label << 3 | zero_streak << 4 | conf > ct << 5
    float cfs[D];
    bool slow = false;
#pragma unroll
    for (int c = 0; c < D; ++c) {
      res[c] = 0;
      cfs[c] = 0.0f;
      if (!valid) continue;
      const uint32_t meta = metas[c];
      const uint32_t r0 = (meta >> 10) & 7u, r1 = meta >> 13;
      if (r1 == r0) {
        mu1[c] = mu0[c];
        var1[c] = var0[c];
      }
      const int vb = vbs[c];
      const uint32_t dy = dyn[c];
      const int dv = abs(vb - (int)(dy & 0xFFu));
      const bool changed = dv > k.eps_i;
      // sampling gate (kernels_numba.py:193-216): SKIP and wake-on-change
      // here; a COPY (anchor label needed) defers the tile
      int zs = 0;
      if (sampling && (dy >> 16)) {
        if (!changed) {
          res[c] = K_SKIP | (int)(((dy >> 8) & 1u) << 3);
          continue;
        }
        zs = 1;  // woke on change: clock, waking, streak -> 0
      } else if (sampling && (dy >> 9 & 1u)) {
        if (!changed && !on_lat) {
          slow = true;
          FRAME_DBG(0);
          continue;
        }
      }
      const float vf = (float)vb;
      const uint32_t c0 = (meta >> 4) & 3u, c1 = (meta >> 6) & 3u,
                     c2 = (meta >> 8) & 3u;
      uint32_t top = c0;
      if (top == L_GROUP && !grouping) top = c1;
      const bool gtop = top == L_GROUP && member;
      const bool top1 = top == L_MEANVAR;
      const float sd0 = var0[c] * rsqrt_approx(var0[c]),
                  sd1 = var1[c] * rsqrt_approx(var1[c]);
      const float thr0 = k.lam * sd0, thr1 = k.lam * sd1;
      const int gidx = member ? c * G + gid : 0;
      const float gm = member ? s_gmuf[gidx] : 0.0f;
      const float gt_thr = member ? s_gthrf[gidx] : 1.0f;
      const float mt = gtop ? gm : (top1 ? mu1[c] : mu0[c]);
      const float dn = gtop ? gt_thr : (top1 ? thr1 : thr0);
      const float ph = tv[c] * rcp_approx(peak[c]);
      const float bt = s_btf[dv];
      float gt = fminf(fabsf(vf - mt) * rcp_approx(dn), 1.0f);
      if (!literal) gt = 1.0f - gt;
      float cf;
      if (ph < k.pf)
        cf = (wb * bt + wc * gt) * k.wbc_inv[cls];
      else
        cf = wa * ph + wb * bt + wc * gt;
      bool sat = cf > k.ct;
      if (fabsf(ph - k.pf) <= FILTER_MARGIN * k.pf + 1e-30f ||
          fabsf(cf - k.ct) <= FILTER_MARGIN) {
        // inside the filter margin: the reference's binary64 confidence
        // (kernels_numba.py:254-270), in place (rare, out of line)
        FRAME_DBG(2);
        const double ce = frame_conf_exact(
            &a, gtop ? (int)((size_t)s * D * G + gidx) : -1, vb,
            (int)(dy & 0xFFu), top1 ? mu1[c] : mu0[c],
            top1 ? var1[c] : var0[c], tv[c], peak[c], cls);
        sat = ce > a.q.confidence_threshold;
        cf = (float)ce;
      }
      int active = -1, label = 0;
      if (chp_on && !changed) {
        active = L_CHP;
        label = (dy >> 8) & 1u;
      } else {
        // first hit in mid_order; an undecided test on the path defers
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          const uint32_t code = j == 0 ? c0 : (j == 1 ? c1 : c2);
          if (active >= 0 || code == 0) break;
          int hit;
          uint32_t rr = 0;
          if (code == L_GROUP) {
            hit = (grouping && member) ? fmatch(vf, gm, gt_thr) : 0;
          } else if (code == L_MEAN) {
            rr = r0;
            hit = fmatch(vf, mu0[c], thr0);
          } else {
            rr = r1;
            hit = fmatch(vf, mu1[c], thr1);
          }
          if (hit < 0) {
            // undecided in fp32: the reference's binary64 test (rare)
            FRAME_DBG(3);
            if (code == L_GROUP) {
              const size_t gi = (size_t)s * D * G + gidx;
              hit = match_exact((double)vb, a.s.g_mu[gi], a.s.g_var[gi],
                                a.q.match_lambda);
            } else {
              hit = code == L_MEAN
                        ? match_exact((double)vb, (double)mu0[c],
                                      (double)var0[c], a.q.match_lambda)
                        : match_exact((double)vb, (double)mu1[c],
                                      (double)var1[c], a.q.match_lambda);
            }
          }
          if (hit && rr > 0) {
            // matched mode must sit inside the background weight prefix
            double acc = 0.0;
#pragma unroll
            for (int q = 0; q < KMAX - 1; ++q)
              if ((uint32_t)q < rr) acc = acc + (double)wq[c][q];
            hit = acc <= a.q.background_threshold;
          }
          if (hit) active = (int)code;
        }
        if (active < 0) active = L_GMM;
      }
      res[c] = active | (label << 3) | (zs << 4) | ((int)sat << 5);
      cfs[c] = cf;
    }
    if (lane == 0) FRAME_DBG(5);
    if (__any_sync(FULL, slow)) {
      if (lane == 0) FRAME_DBG(4);
      defer_tile(tile);
      continue;
    }

    // ---- pass 2: bookkeeping (kernels_numba.py:335-359), deep queue,
    // exact partials
    int fg = 0;
    const unsigned any_member = __ballot_sync(FULL, member);
#pragma unroll
    for (int c = 0; c < D; ++c) {
      const uint32_t o = sP + (uint32_t)c * P + p;
      const int active = res[c] & 7, label = (res[c] >> 3) & 1;
      const float cf = cfs[c];
      const int vb = vbs[c];
      int deep = DEEP_NONE;
      double rho = 0.0;
      if (valid && active == K_SKIP) {
        // clock -1, waking on its last tick; label, last_active kept
        const uint32_t dy = dyn[c];
        const int clock = (int)(dy >> 16) - 1;
        a.s.dyn[o] = pack_dyn(vb, label, clock == 0 ? 1 : (int)((dy >> 9) & 1u),
                              (int)((dy >> 10) & 7u) - 1, clock);
        st(conf_s + o, 0.0);
        a.kind[o] = (uint8_t)K_SKIP;
        kc += 1ull << (9 * K_SKIP);
        fg |= label;
      } else if (valid) {
        const uint32_t meta = metas[c];
        const uint32_t r0 = (meta >> 10) & 7u;
        const uint32_t mb = (sK + c) * K * P + p;
        rho = a.q.learning_rate;
        if (rate_on) {
          double relax = 1.0 - (double)cf;
          if (relax < a.q.rate_floor) relax = a.q.rate_floor;
          rho = a.q.learning_rate * relax;
        }
        if (active == L_MEAN)
          st(mu_s + (mb + r0 * P), (1.0 - rho) * (double)mu0[c] + rho * (double)vb);
        else if (active == L_MEANVAR)
          deep = DEEP_MEANVAR;
        else if (active == L_GMM)
          deep = DEEP_GMM;
        uint32_t sk = ((res[c] >> 4) & 1) ? 0u : stk[c];
        if ((res[c] >> 5) & 1)
          sk = (sk == 0xffffffffu) ? sk : sk + 1u;
        else
          sk = 0u;
        a.s.streak[o] = sk;
        atomicAdd(a.s.hits + (((sK + c) * 5 + (uint32_t)active) * P + p), 1u);
        // after the gate an evaluated pixel has clock 0 and waking 0
        // (sampling on); with sampling off both are carried unchanged
        const uint32_t dy = dyn[c];
        const int clock = sampling ? ((long long)sk >= (long long)k.sat
                                          ? a.q.sleep_frames : 0)
                                   : (int)(dy >> 16);
        const int waking = sampling ? 0 : (int)((dy >> 9) & 1u);
        // a GMM label arrives with the deep pass (it ORs the label bit)
        a.s.dyn[o] = pack_dyn(vb, label, waking, active, clock);
        st(conf_s + o, (double)cf);
        a.kind[o] = (uint8_t)active;
        kc += 1ull << (9 * active);
        fg |= label;
      }
      const bool dq = deep != DEEP_NONE;
      const unsigned qm = __ballot_sync(FULL, dq);
      if (qm) {
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
          const uint32_t r1 = metas[c] >> 13;
          qc[pos] = 1ull | ((unsigned long long)deep << 1) |
                    ((unsigned long long)(deep == DEEP_MEANVAR ? r1 : 0u) << 3) |
                    ((unsigned long long)c << 6) |
                    ((unsigned long long)vb << 8) |
                    ((unsigned long long)p << 16);
          qr[pos] = rho;
        }
        wq_n += nq;
      }

      // ---- group partials (exact sums) into the warp's private slice
      if (any_member) {
        unsigned todo = any_member;
        while (todo) {
          const int leader = __ffs(todo) - 1;
          const int g = __shfl_sync(FULL, gid, leader);
          const bool mine = member && gid == g;
          const unsigned mm = __ballot_sync(FULL, mine);
          todo &= ~mm;
          const unsigned sall = warp_sum_u32(mine ? (unsigned)vb : 0u);
          const bool hit = mine && active == L_GROUP;
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
