// cog_vec.cuh -- the float32-state step kernel with 128-bit vector access
// (included inside the anonymous namespace of cog_kernels.cu, after
// cog_fast.cuh, whose FastConst / fmatch / hot_px_slow it reuses).
//
// Work unit = one plane of one stride-aligned warp tile of 128 pixels; each
// lane owns 4 consecutive pixels of a row (stride 1: 1 x 128, stride 2:
// 2 x 64, stride 4: 4 x 32 pixels), so
//   * the per-pixel state words move as 16-byte vectors (dyn, streak, peak,
//     conf: uint4/float4; meta, group ids: 8 bytes; frame bytes, classes,
//     kinds: 4 bytes) -- one load/store instruction per array per 4 pixels;
//   * the referenced modes of the 4 pixels are one float4 per array when the
//     4 pixels share their mode references (the common case);
//   * per-unit overhead (index math, ballots, worklist compaction, group
//     reductions) is paid once per 128 plane-pixels instead of per 32;
//   * every copy pixel's anchor (y - y % s, x - x % s) is in row 0 of the
//     same warp and in the same 4-pixel group, so copy resolution is a
//     shuffle of the anchor lane's 4 label bits.
// Decisions are the fast kernel's (filtered fp32, exact binary64 fallback
// per plane-pixel through hot_px_slow).  The union mask is formed by the
// deep kernel's union pass.

#ifndef COG_VEC_MINB
#define COG_VEC_MINB 2
#endif

struct FastEval {
  int active, label;
  float cf;
  double rho;
  uint32_t r0, r1;
  bool slow;
};

// fast-path decision for one plane-pixel (kernels_numba.py:239-342 with
// filtered fp32 comparisons; slow = a comparison was undecided or the
// pixel's gating state is not the plain "evaluate" one)
__device__ __forceinline__ FastEval fast_eval(
    const StepArgs& a, const FastConst& k, int vb, uint32_t dyn,
    uint32_t meta, float tv, float peak, float mu0, float var0, float mu1,
    float var1, bool member, float gm, float gthr, float wa, float wb,
    float wc, float wbc, const float* s_btf, const float* wbase, uint32_t P) {
  const bool sampling = a.q.sampling_on != 0, grouping = a.q.grouping_on != 0;
  FastEval e;
  e.active = -1;
  e.label = 0;
  e.cf = 0.0f;
  e.rho = 0.0;
  e.r0 = (meta >> 10) & 7u;
  e.r1 = meta >> 13;
  e.slow = a.q.compat != 0 || (sampling && ((dyn >> 9) & 1u || (dyn >> 16)));
  if (e.slow) return e;
  const int chp = dyn & 0xFF;
  const int dv = abs(vb - chp);
  const bool changed = dv > k.eps_i;
  const float vf = (float)vb;
  const uint32_t c0 = (meta >> 4) & 3u, c1 = (meta >> 6) & 3u,
                 c2 = (meta >> 8) & 3u;
  uint32_t top = c0;
  if (top == L_GROUP && !grouping) top = c1;
  const bool gtop = top == L_GROUP && member;
  const bool top1 = top == L_MEANVAR;
  const float thr0 = k.lam * (var0 * rsqrtf(var0));
  const float thr1 = k.lam * (var1 * rsqrtf(var1));
  const float mt = gtop ? gm : (top1 ? mu1 : mu0);
  const float dn = gtop ? gthr : (top1 ? thr1 : thr0);
  const float ph = __fdividef(tv, peak);
  const float bt = s_btf[dv];
  float gt = fminf(__fdividef(fabsf(vf - mt), dn), 1.0f);
  if (!a.q.literal_conf) gt = 1.0f - gt;
  float cf;
  if (ph < k.pf)
    cf = (wb * bt + wc * gt) * wbc;
  else
    cf = wa * ph + wb * bt + wc * gt;
  e.cf = cf;
  e.slow = fabsf(ph - k.pf) <= FILTER_MARGIN * k.pf + 1e-30f ||
           fabsf(cf - k.ct) <= FILTER_MARGIN;
  if (a.q.chp_on && !changed) {
    e.active = L_CHP;
    e.label = (dyn >> 8) & 1u;
  } else {
    int active = -1;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const uint32_t code = j == 0 ? c0 : (j == 1 ? c1 : c2);
      if (active >= 0 || code == 0) break;
      int hit;
      uint32_t rr = 0;
      if (code == L_GROUP) {
        hit = (grouping && member) ? fmatch(vf, gm, gthr) : 0;
      } else if (code == L_MEAN) {
        rr = e.r0;
        hit = fmatch(vf, mu0, thr0);
      } else {
        rr = e.r1;
        hit = fmatch(vf, mu1, thr1);
      }
      if (hit < 0) {
        e.slow = true;
        break;
      }
      if (hit && rr > 0) {
        // a matched mode must sit inside the background weight prefix
        double acc = 0.0;
        for (uint32_t q = 0; q < rr; ++q) acc = acc + (double)wbase[q * P];
        hit = acc <= a.q.background_threshold;
      }
      if (hit) active = (int)code;
    }
    e.active = active < 0 ? (int)L_GMM : active;
  }
  if (!e.slow) {
    double rho = a.q.learning_rate;
    if (a.q.rate_scaling_on) {
      double relax = 1.0 - (double)cf;
      if (relax < a.q.rate_floor) relax = a.q.rate_floor;
      rho = a.q.learning_rate * relax;
    }
    e.rho = rho;
  }
  return e;
}

__device__ __forceinline__ uint32_t u16_at(uint2 v, int j) {
  const uint32_t w = j < 2 ? v.x : v.y;
  return (j & 1) ? (w >> 16) : (w & 0xFFFFu);
}
__device__ __forceinline__ uint32_t u8_at(uint32_t v, int j) {
  return (v >> (8 * j)) & 0xFFu;
}
template <typename V>
__device__ __forceinline__ auto lane4(const V& v, int j) {
  return j == 0 ? v.x : (j == 1 ? v.y : (j == 2 ? v.z : v.w));
}
template <typename V, typename S>
__device__ __forceinline__ void set4(V& v, int j, S x) {
  if (j == 0) v.x = x;
  else if (j == 1) v.y = x;
  else if (j == 2) v.z = x;
  else v.w = x;
}

template <int KMAX>
__global__ void __launch_bounds__(LEAN_THREADS, COG_VEC_MINB)
    vec_kernel(const __grid_constant__ StepArgs a,
               const __grid_constant__ FastConst k) {
  using T = float;
  extern __shared__ double s_mem[];
  const int s = blockIdx.y;
  const int D = a.g.depth, G = a.g.n_groups, K = a.g.k;
  const int H = a.g.height, W = a.g.width, stride = a.g.stride;
  const uint32_t P = (uint32_t)H * (uint32_t)W;
  const int words = acc_words(D, G);
  const int wpad = (words + 1) & ~1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool sampling = a.q.sampling_on != 0, compat = a.q.compat != 0;

  // ---- shared (same layout as fast_kernel)
  double* s_bt = s_mem;
  double* s_gmu = s_bt + 256;
  double* s_gthr = s_gmu + D * G;
  unsigned long long* s_wacc = (unsigned long long*)(s_gthr + D * G);
  unsigned long long* s_qc = s_wacc + LEAN_WARPS * wpad;
  double* s_qr = (double*)(s_qc + LEAN_WARPS * FQ_CAP);
  float* s_btf = (float*)(s_qr + LEAN_WARPS * FQ_CAP);
  float* s_gmuf = s_btf + 256;
  float* s_gthrf = s_gmuf + D * G;
  for (int i = threadIdx.x; i < 256; i += LEAN_THREADS) {
    const double b = (double)i / 255.0;
    s_bt[i] = a.q.literal_conf ? b : 1.0 - b;
    s_btf[i] = (float)s_bt[i];
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
  unsigned long long* wacc = s_wacc + warp * wpad;
  unsigned long long* qc = s_qc + warp * FQ_CAP;
  double* qr = s_qr + warp * FQ_CAP;

  const uint32_t sP = (uint32_t)s * D * P;
  const uint32_t sK = (uint32_t)s * D;
  const uint32_t s1 = (uint32_t)s * P;
  T* const mu_s = (T*)a.s.mu;
  T* const var_s = (T*)a.s.var;
  T* const w_s = (T*)a.s.w;
  uint32_t* sync = a.s.sync + (size_t)s * 4;
  const size_t dq_cap = dq_capacity(D, P);
  unsigned long long* dq_code =
      (unsigned long long*)a.s.deepq + (size_t)s * dq_cap;
  double* dq_rho = a.s.deeprho + (size_t)s * dq_cap;
  const bool do_reset = (*(volatile uint32_t*)(sync + 1) & 1u) != 0;
  const bool do_reorder = a.reorder_now != 0;
  const GmmPar gp{a.q.match_lambda, a.q.background_threshold,
                  a.q.variance_floor, a.q.initial_variance};

  // lane geometry: lanes_row lanes a row, 4 pixels a lane
  const int lanes_row = 32 / stride;
  const int lrow = lane / lanes_row, lg = lane - lrow * lanes_row;
  const int tile_w = lanes_row * 4;
  const int tiles_x = (W + tile_w - 1) / tile_w;
  const int n_tiles = tiles_x * ((H + stride - 1) / stride);
  const int anchor = lg;  // row-0 lane with the same 4-pixel group

  unsigned long long kc = 0ull;  // pooled kind counts, 7 x 9 bits
  int kc_units = 0;
  int wq_n = 0;

  const int n_units = n_tiles * D;
  const int nw = gridDim.x * LEAN_WARPS;
  for (int u = blockIdx.x * LEAN_WARPS + warp; u < n_units; u += nw) {
    const int wt = u / D, c = u - wt * D;
    const int ty = wt / tiles_x, tx = wt - ty * tiles_x;
    const int y = ty * stride + lrow, x0 = tx * tile_w + lg * 4;
    const bool valid = y < H && x0 < W;  // W % 4 == 0: all 4 or none
    const uint32_t p = valid ? (uint32_t)y * (uint32_t)W + (uint32_t)x0 : 0u;
    const uint32_t o = sP + (uint32_t)c * P + p;      // 4-aligned
    const uint32_t mb = (sK + c) * K * P + p;          // mode 0 of pixel 0

    if (do_reset || do_reorder) {
      if (valid) {
        const PlaneRef<T> pr = plane_ref<T>(a, s, c);
        for (int j = 0; j < 4; ++j) {
          const int g0 = a.s.gid[s1 + p + j];
          const bool mem = G > 0 && g0 != (int)UNGROUPED;
          if (do_reset) cold_reset<T, KMAX>(pr, p + j, a.q.initial_variance);
          if (do_reorder)
            cold_reorder<T>(pr, p + j, mem ? s_gmu[c * G + g0]
                                           : (G > 0 ? s_gmu[c * G] : 0.0));
        }
      }
      __syncwarp();
    }

    // ---- round 1: 4 pixels of every pixel-indexed array, vector loads
    uint32_t fr4 = 0, cls4 = 0;
    uint2 meta4 = make_uint2(0, 0), gid4 = make_uint2(0xFFFFFFFFu, 0xFFFFFFFFu);
    uint4 dyn4 = make_uint4(0, 0, 0, 0), stk4 = make_uint4(0, 0, 0, 0);
    float4 pk4 = make_float4(1.f, 1.f, 1.f, 1.f);
    if (valid) {
      fr4 = *(const uint32_t*)(a.frame + o);
      dyn4 = *(const uint4*)(a.s.dyn + o);
      meta4 = *(const uint2*)(a.s.meta + o);
      stk4 = *(const uint4*)(a.s.streak + o);
      pk4 = __ldg((const float4*)(a.s.peak + o));
      gid4 = *(const uint2*)(a.s.gid + s1 + p);
      cls4 = *(const uint32_t*)(a.s.cls + s1 + p);
    }
    // ---- round 2: table entries and referenced modes
    float tv[4] = {0.f, 0.f, 0.f, 0.f};
    float4 m0 = make_float4(0.f, 0.f, 0.f, 0.f), v0 = make_float4(1.f, 1.f, 1.f, 1.f);
    float4 m1 = m0, v1 = v0;
    bool evm[4];
    uint32_t ev_any = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      evm[j] = valid && !compat &&
               will_evaluate(sampling, lane4(dyn4, j), (int)u8_at(fr4, j),
                             lrow == 0 && (j % stride) == 0, a.q.chp_epsilon);
      ev_any |= (uint32_t)evm[j] << j;
      if (evm[j])
        tv[j] = __ldcg(a.s.table + (((size_t)(o + j) << 8) | u8_at(fr4, j)));
    }
    if (ev_any) {
      const uint32_t refs0 = (u16_at(meta4, 0) >> 10);
      const bool same = ((u16_at(meta4, 1) >> 10) == refs0) &&
                        ((u16_at(meta4, 2) >> 10) == refs0) &&
                        ((u16_at(meta4, 3) >> 10) == refs0);
      if (same) {
        const uint32_t r0 = refs0 & 7u, r1 = refs0 >> 3;
        m0 = *(const float4*)(mu_s + mb + r0 * P);
        v0 = *(const float4*)(var_s + mb + r0 * P);
        if (r1 != r0) {
          m1 = *(const float4*)(mu_s + mb + r1 * P);
          v1 = *(const float4*)(var_s + mb + r1 * P);
        } else {
          m1 = m0;
          v1 = v0;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (!evm[j]) continue;
          const uint32_t mt = u16_at(meta4, j);
          const uint32_t r0 = (mt >> 10) & 7u, r1 = mt >> 13;
          set4(m0, j, mu_s[mb + j + r0 * P]);
          set4(v0, j, var_s[mb + j + r0 * P]);
          set4(m1, j, mu_s[mb + j + r1 * P]);
          set4(v1, j, var_s[mb + j + r1 * P]);
        }
      }
    }

    // ---- the 4 plane-pixels
    float4 cf4 = make_float4(0.f, 0.f, 0.f, 0.f);
    uint4 dout = dyn4;
    uint32_t kind4 = 0, labels = 0, slowbits = 0, copybits = 0;
    uint32_t latebits = 0, nowbits = 0, skn[4];
    int deepk[4], rsel[4];
    double rhov[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      deepk[j] = DEEP_NONE;
      rsel[j] = 0;
      rhov[j] = 0.0;
      skn[j] = lane4(stk4, j);
      if (!valid) continue;
      const uint32_t pj = p + j, oj = o + j;
      const int vb = (int)u8_at(fr4, j);
      const uint32_t dyn = lane4(dyn4, j), meta = u16_at(meta4, j);
      const int gid = (int)u16_at(gid4, j), cls = (int)u8_at(cls4, j);
      const bool member = G > 0 && gid != (int)UNGROUPED;
      const int gidx = member ? c * G + gid : 0;
      const FastEval e = fast_eval(
          a, k, vb, dyn, meta, tv[j], lane4(pk4, j), lane4(m0, j),
          lane4(v0, j), lane4(m1, j), lane4(v1, j), member,
          member ? s_gmuf[gidx] : 0.0f, member ? s_gthrf[gidx] : 1.0f,
          k.w[3 * cls], k.w[3 * cls + 1], k.w[3 * cls + 2], k.wbc_inv[cls],
          s_btf, w_s + mb + j, P);
      HotOut ho;
      if (e.slow) {
        Pre<T> x;
        x.vb = vb;
        x.dyn = dyn;
        x.meta = meta;
        x.streak = lane4(stk4, j);
        x.peak = lane4(pk4, j);
        x.tv = tv[j];
        x.mu0 = lane4(m0, j);
        x.var0 = lane4(v0, j);
        x.mu1 = lane4(m1, j);
        x.var1 = lane4(v1, j);
        ho = hot_px_slow<T>(&a, s, c, pj, x, lrow == 0 && (j % stride) == 0,
                            s_bt, cls, member, member ? s_gmu[gidx] : 0.0,
                            member ? s_gthr[gidx] : 0.0);
        slowbits |= 1u << j;
      } else {
        // bookkeeping of the fast path (kernels_numba.py:335-359)
        const int active = e.active;
        ho.kind = active;
        ho.label = e.label;
        ho.conf = (double)e.cf;
        ho.rho = e.rho;
        ho.rsel = 0;
        ho.deep = DEEP_NONE;
        if (active == L_MEAN) {
          st(mu_s + (mb + j + e.r0 * P),
             (1.0 - e.rho) * (double)lane4(m0, j) + e.rho * (double)vb);
        } else if (active == L_MEANVAR) {
          ho.deep = DEEP_MEANVAR;
          ho.rsel = (int)e.r1;
        } else if (active == L_GMM) {
          ho.deep = DEEP_GMM;
        }
        uint32_t sk = lane4(stk4, j);
        if (e.cf > k.ct)
          sk = (sk == 0xffffffffu) ? sk : sk + 1u;
        else
          sk = 0u;
        skn[j] = sk;
        atomicAdd(a.s.hits + (((sK + c) * 5 + (uint32_t)active) * P + pj), 1u);
        const int clock = (sampling && (long long)sk >= (long long)k.sat)
                              ? a.q.sleep_frames : (int)(dyn >> 16);
        ho.dyn = pack_dyn(vb, e.label, (dyn >> 9) & 1u, active, clock);
      }
      set4(cf4, j, (float)ho.conf);
      kind4 |= (uint32_t)ho.kind << (8 * j);
      kc += 1ull << (9 * ho.kind);
      labels |= ((uint32_t)ho.label & 1u) << j;
      if (ho.kind == K_COPY) copybits |= 1u << j;
      set4(dout, j, ho.dyn);
      deepk[j] = ho.deep;
      rsel[j] = ho.rsel;
      rhov[j] = ho.rho;
      (void)oj;
    }
    if (valid) {
      *(float4*)((T*)a.conf + o) = cf4;
      *(uint32_t*)(a.kind + o) = kind4;
      if (!slowbits) {
        *(uint4*)(a.s.streak + o) = make_uint4(skn[0], skn[1], skn[2], skn[3]);
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (!((slowbits >> j) & 1u)) a.s.streak[o + j] = skn[j];
      }
    }

    // ---- deep work: in-lane when this plane-tile has copy pixels (their
    // anchors need final labels now), else onto the dense worklist
    uint32_t dqbits = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) dqbits |= (uint32_t)(deepk[j] != DEEP_NONE) << j;
    if (__any_sync(FULL, dqbits != 0)) {
      if (__any_sync(FULL, copybits != 0)) {
        const PlaneRef<T> pr = plane_ref<T>(a, s, c);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (!((dqbits >> j) & 1u)) continue;
          const uint32_t mt = u16_at(meta4, j);
          const double v = (double)u8_at(fr4, j);
          if (deepk[j] == DEEP_MEANVAR) {
            cold_meanvar<T, KMAX>(pr, p + j, mt, rsel[j], v, rhov[j],
                                  a.q.variance_floor);
          } else {
            const int lbl = cold_gmm<T, KMAX>(pr, p + j, mt, v, rhov[j], gp,
                                              K, deepk[j] == DEEP_GMM);
            labels = (labels & ~(1u << j)) | ((uint32_t)(lbl & 1) << j);
            nowbits |= 1u << j;
          }
        }
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const bool dq = (dqbits >> j) & 1u;
          const unsigned qm = __ballot_sync(FULL, dq);
          if (!qm) continue;
          const int nq = __popc(qm);
          if (wq_n + nq > FQ_CAP) {
            unsigned base = 0;
            if (lane == 0) base = atomicAdd(sync + 3, (unsigned)wq_n);
            base = __shfl_sync(FULL, base, 0);
            __syncwarp();
            for (int e2 = lane; e2 < wq_n; e2 += 32) {
              dq_code[(size_t)base + e2] = qc[e2];
              dq_rho[(size_t)base + e2] = qr[e2];
            }
            __syncwarp();
            wq_n = 0;
          }
          if (dq) {
            const int pos = wq_n + __popc(qm & ((1u << lane) - 1u));
            qc[pos] = 1ull | ((unsigned long long)deepk[j] << 1) |
                      ((unsigned long long)rsel[j] << 3) |
                      ((unsigned long long)c << 6) |
                      ((unsigned long long)u8_at(fr4, j) << 8) |
                      ((unsigned long long)(p + j) << 16);
            qr[pos] = rhov[j];
            if (deepk[j] == DEEP_GMM || deepk[j] == DEEP_COMPAT)
              latebits |= 1u << j;
          }
          wq_n += nq;
        }
      }
    }
    // ---- final labels: late GMM labels arrive with the deep kernel (0
    // now), copies take their anchors' labels
    labels &= ~latebits;
    const uint32_t alab = __shfl_sync(FULL, labels, anchor);
    if (copybits) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if ((copybits >> j) & 1u) {
          const uint32_t aj = j - j % stride;  // anchor pixel in the group
          labels = (labels & ~(1u << j)) | (((alab >> aj) & 1u) << j);
        }
    }
    if (valid) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        set4(dout, j, (lane4(dout, j) & ~(1u << 8)) | (((labels >> j) & 1u) << 8));
      *(uint4*)(a.s.dyn + o) = dout;
    }

    // ---- group partials (exact sums) into the warp's private slice
    const unsigned any_member = __ballot_sync(
        FULL, valid && G > 0 && (gid4.x != 0xFFFFFFFFu || gid4.y != 0xFFFFFFFFu));
    if (any_member) {
      // per-lane pre-aggregation over the 4 pixels, per distinct group
#pragma unroll 1
      for (int j0 = 0; j0 < 4; ++j0) {
        // handle the group of pixel j0 unless an earlier pixel had it
        const int g_l = valid ? (int)u16_at(gid4, j0) : (int)UNGROUPED;
        bool dup = false;
        for (int j = 0; j < j0; ++j)
          dup |= (int)u16_at(gid4, j) == g_l;
        const bool has = valid && G > 0 && g_l != (int)UNGROUPED && !dup;
        unsigned todo = __ballot_sync(FULL, has);
        while (todo) {
          const int leader = __ffs(todo) - 1;
          const int g = __shfl_sync(FULL, g_l, leader);
          const bool mine = has && g_l == g;
          todo &= ~__ballot_sync(FULL, mine);
          unsigned sall = 0, cnt = 0, hits = 0, sv = 0;
          unsigned long long qv = 0;
          if (valid) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              if ((int)u16_at(gid4, j) != g || !mine) continue;
              const unsigned vb = u8_at(fr4, j);
              sall += vb;
              cnt += 1;
              if (u8_at(kind4, j) == L_GROUP) {
                hits += 1;
                sv += vb;
                const double cq = (double)lane4(cf4, j) * 4503599627370496.0;
                qv += cq > 0.0 ? (unsigned long long)cq : 0ull;
              }
            }
          }
          const unsigned r_sall = warp_sum_u32(sall);
          const unsigned r_cnt = warp_sum_u32(cnt);
          const unsigned r_hits = warp_sum_u32(hits);
          unsigned r_sv = 0;
          unsigned long long Q = 0;
          if (r_hits) {
            // a lane holds up to 4 x 2^52: split in 20-bit pieces so the
            // 32-bit warp sums cannot overflow
            r_sv = warp_sum_u32(sv);
            const unsigned q2 = warp_sum_u32((unsigned)(qv >> 40));
            const unsigned q1 = warp_sum_u32((unsigned)((qv >> 20) & 0xFFFFFu));
            const unsigned q0 = warp_sum_u32((unsigned)(qv & 0xFFFFFu));
            Q = ((unsigned long long)q2 << 40) +
                ((unsigned long long)q1 << 20) + (unsigned long long)q0;
          }
          if (lane == 0) {
            unsigned long long* e = wacc + acc_grp(D, G, c, g);
            e[4] += r_sall;
            e[5] += r_cnt;
            if (r_hits) {
              e[0] += r_hits;
              e[1] += r_sv;
              e[2] += Q >> CONF_SPLIT;
              e[3] += Q & ((1ull << CONF_SPLIT) - 1ull);
            }
          }
        }
      }
    }
    if (++kc_units >= 127) {  // 4 counts a unit per field: flush before 511
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
    for (int e2 = lane; e2 < wq_n; e2 += 32) {
      dq_code[(size_t)base + e2] = qc[e2];
      dq_rho[(size_t)base + e2] = qr[e2];
    }
  }
#pragma unroll
  for (int q = 0; q < 7; ++q) {
    const unsigned v = warp_sum_u32((unsigned)((kc >> (9 * q)) & 511u));
    if (lane == 0) wacc[acc_kind(0, q)] += v;
  }
  __syncthreads();
  unsigned long long* gacc = (unsigned long long*)a.s.accum + (size_t)s * words;
  for (int i = threadIdx.x; i < words; i += LEAN_THREADS) {
    unsigned long long v = 0;
#pragma unroll
    for (int w = 0; w < LEAN_WARPS; ++w) v += s_wacc[w * wpad + i];
    if (v) atomicAdd(gacc + i, v);
  }
}
