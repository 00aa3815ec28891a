// cog_lean.cuh -- the lean per-frame step kernel (included inside the
// anonymous namespace of cog_kernels.cu, after the shared helpers).
//
// Same work unit and the same per-plane-pixel decisions as the general
// step kernel (hot_px: kernels_numba.py:188-359), organised for occupancy:
//   * one thread = one pixel, all D planes (D a template parameter); one warp
//     = one stride-aligned tile (stride rows x cw columns, so every copy
//     pixel's anchor sits in row 0 of the same warp);
//   * every load of the tile is issued before any decision: round 1 (frame
//     bytes, dyn, meta, streak, peak, class, group id of all planes) then
//     round 2 (table entry at v, the two referenced modes) -- ~10 independent
//     loads in flight per thread, 24-32 warps per SM hide the latency;
//   * 32-bit element offsets inside a plane, per-stream base pointers set
//     once per CTA (the general kernel spent 30% of its instructions on
//     64-bit address arithmetic);
//   * statistics: pooled kind counts packed in one u64 register per lane
//     (7 x 9-bit fields, flushed before they can overflow), foreground count
//     by ballot, group partials by warp reductions into a CTA slice in
//     shared memory (exact integer / 2^-52 fixed-point sums, so the totals
//     do not depend on CTA count or order);
//   * MEANVAR hits and GMM fall-throughs go to the stream's dense worklist
//     through a per-warp shared buffer (one global atomic per 64 items); a
//     plane-tile that holds copy pixels runs its deep items in-warp so the
//     copies see their anchors' final labels.
// The deep kernel then runs the worklist and its last CTA finalizes the
// frame, exactly as after the general kernel.

constexpr int LEAN_THREADS = 256;
constexpr int LEAN_WARPS = LEAN_THREADS / 32;
constexpr int LQ_CAP = 64;  // per-warp worklist buffer

#ifndef COG_LEAN_MINB
#define COG_LEAN_MINB 3
#endif

__host__ __device__ inline size_t lean_smem_bytes(int d, int G) {
  const size_t words = (size_t)acc_words(d, G);
  return 256 * 8 + (size_t)2 * d * G * 8 + ((words + 1) & ~(size_t)1) * 8 +
         (size_t)LEAN_WARPS * LQ_CAP * 16;
}

template <int D>
__device__ __forceinline__ void lean_flush_kinds(unsigned long long& kc,
                                                 unsigned long long* s_acc,
                                                 int lane) {
#pragma unroll
  for (int k = 0; k < 7; ++k) {
    const unsigned v = warp_sum_u32((unsigned)((kc >> (9 * k)) & 511u));
    if (lane == 0 && v) atomicAdd(s_acc + acc_kind(0, k), (unsigned long long)v);
  }
  kc = 0ull;
}

template <typename T, int KMAX, int D>
__global__ void __launch_bounds__(LEAN_THREADS, COG_LEAN_MINB)
    lean_kernel(const StepArgs a) {
  extern __shared__ double s_mem[];
  const Flags f{a.q.sampling_on != 0, a.q.grouping_on != 0,
                a.q.rate_scaling_on != 0, a.q.chp_on != 0,
                a.q.literal_conf != 0, a.q.compat != 0};
  const int s = blockIdx.y;
  const int G = a.g.n_groups, K = a.g.k;
  const int H = a.g.height, W = a.g.width, stride = a.g.stride;
  const uint32_t P = (uint32_t)H * (uint32_t)W;
  const int words = acc_words(D, G);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

  // ---- shared prologue
  double* s_bt = s_mem;
  double* s_gmu = s_bt + 256;
  double* s_gthr = s_gmu + D * G;
  unsigned long long* s_acc = (unsigned long long*)(s_gthr + D * G);
  unsigned long long* s_qc =
      s_acc + ((words + 1) & ~1) + (size_t)warp * LQ_CAP;
  double* s_qr = (double*)(s_acc + ((words + 1) & ~1) +
                           (size_t)LEAN_WARPS * LQ_CAP) +
                 (size_t)warp * LQ_CAP;
  for (int i = threadIdx.x; i < 256; i += LEAN_THREADS) {
    const double b = (double)i / 255.0;
    s_bt[i] = f.literal ? b : 1.0 - b;
  }
  {
    const double* gmu = a.s.g_mu + (size_t)s * D * G;
    const double* gvar = a.s.g_var + (size_t)s * D * G;
    for (int i = threadIdx.x; i < D * G; i += LEAN_THREADS) {
      s_gmu[i] = gmu[i];
      s_gthr[i] = a.q.match_lambda * sqrt(gvar[i]);
    }
  }
  for (int i = threadIdx.x; i < words; i += LEAN_THREADS) s_acc[i] = 0ull;
  __syncthreads();

  // ---- per-stream bases (planes are P apart, records R elements)
  const size_t sD = (size_t)s * D;
  const uint8_t* frame = a.frame + sD * P;
  uint32_t* dynb = a.s.dyn + sD * P;
  uint16_t* metab = a.s.meta + sD * P;
  uint32_t* stkb = a.s.streak + sD * P;
  const float* peakb = a.s.peak + sD * P;
  uint32_t* hitsb = a.s.hits + sD * 5 * P;
  const float* tabb = a.s.table + sD * P * 256;   // reference layout
  constexpr int R = rec_elems(KMAX);
  T* mixb = (T*)a.s.mix + sD * P * R;
  T* confb = (T*)a.conf + sD * P;
  uint8_t* kindb = a.kind + sD * P;
  uint8_t* maskb = a.mask + (size_t)s * P;
  const uint8_t* clsb = a.s.cls + (size_t)s * P;
  const uint16_t* gidb = a.s.gid + (size_t)s * P;
  uint32_t* sync = a.s.sync + (size_t)s * 4;
  const size_t dq_cap = dq_capacity(D, P);
  unsigned long long* dq_code =
      (unsigned long long*)a.s.deepq + (size_t)s * dq_cap;
  double* dq_rho = a.s.deeprho + (size_t)s * dq_cap;
  const bool do_reset = (*(volatile uint32_t*)(sync + 1) & 1u) != 0;
  const bool do_reorder = a.reorder_now != 0;
  const GmmPar gp{a.q.match_lambda, a.q.background_threshold,
                  a.q.variance_floor, a.q.initial_variance};
  const double eps = a.q.chp_epsilon;

  // lane geometry inside a tile (row 0 holds every copy anchor)
  const int cw = a.cw;
  const int lrow = lane / cw, lcol = lane - lrow * cw;
  const bool lane_ok = lane < stride * cw;
  const bool on_lat = (lrow == 0) && (lcol % stride == 0);
  const int anchor = lcol - lcol % stride;  // lane of this pixel's anchor

  unsigned long long kc = 0ull;  // pooled kind counts, 7 x 9 bits
  int kc_tiles = 0;
  constexpr int KC_FLUSH = 511 / D;
  unsigned fg_count = 0;
  int wq_n = 0;

  const int nw = gridDim.x * LEAN_WARPS;
  for (int wt = blockIdx.x * LEAN_WARPS + warp; wt < a.n_tiles; wt += nw) {
    const int ty = wt / a.tiles_x, tx = wt - ty * a.tiles_x;
    const int y = ty * stride + lrow, x = tx * cw + lcol;
    const bool valid = lane_ok && y < H && x < W;
    const uint32_t p = valid ? (uint32_t)y * (uint32_t)W + (uint32_t)x : 0u;
    int gid = (int)UNGROUPED, cls = 0;

    // pending illumination reset / scheduled reorder (rare)
    if (do_reset || do_reorder) {
      if (valid) {
        const int g0 = gidb[p];
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

    // ---- round 1: everything addressed by the pixel index
    Pre<T> pre[D];
#pragma unroll
    for (int c = 0; c < D; ++c) {
      pre[c].vb = 0;
      pre[c].dyn = pre[c].meta = pre[c].streak = 0u;
      pre[c].peak = 1.0f;
      pre[c].tv = 0.0f;
      pre[c].mu0 = pre[c].mu1 = (T)0;
      pre[c].var0 = pre[c].var1 = (T)1;
    }
    if (valid) {
      gid = gidb[p];
      cls = clsb[p];
#pragma unroll
      for (int c = 0; c < D; ++c) {
        const uint32_t o = (uint32_t)c * P + p;
        pre[c].vb = frame[o];
        pre[c].dyn = dynb[o];
        pre[c].meta = metab[o];
        pre[c].streak = stkb[o];
        pre[c].peak = __ldg(peakb + o);
      }
    }
    // ---- round 2: table entry at v, the MEAN / MEANVAR modes
#pragma unroll
    for (int c = 0; c < D; ++c) {
      const bool ev = valid && !f.compat &&
                      will_evaluate(f.sampling, pre[c].dyn, pre[c].vb, on_lat,
                                    eps);
      if (ev) {
        const size_t o = (size_t)c * P + p;
        pre[c].tv = __ldcg(tabb + o * 256 + pre[c].vb);
        const int r0 = meta_ref(pre[c].meta, 0), r1 = meta_ref(pre[c].meta, 1);
        const T* rec = mixb + o * R;
        pre[c].mu0 = rec[2 * r0];
        pre[c].var0 = rec[2 * r0 + 1];
        if (r1 != r0) {
          pre[c].mu1 = rec[2 * r1];
          pre[c].var1 = rec[2 * r1 + 1];
        } else {
          pre[c].mu1 = pre[c].mu0;
          pre[c].var1 = pre[c].var0;
        }
      }
    }

    const bool member = valid && G > 0 && gid != (int)UNGROUPED;
    double wa = 0.0, wb = 0.0, wc = 0.0;
    if (valid) {
      wa = a.q.weights[3 * cls];
      wb = a.q.weights[3 * cls + 1];
      wc = a.q.weights[3 * cls + 2];
    }
    const unsigned any_member = __ballot_sync(FULL, member);

    unsigned lbits = 0, copybits = 0, gmmbits = 0;
    uint32_t dyn_late[D];

#pragma unroll
    for (int c = 0; c < D; ++c) {
      const uint32_t o = (uint32_t)c * P + p;
      PlaneRef<T> pr;
      pr.mix = mixb + (size_t)c * P * R;
      pr.R = R;
      pr.KB = KMAX;
      pr.meta = metab + (size_t)c * P;
      pr.dyn = dynb + (size_t)c * P;
      pr.streak = stkb + (size_t)c * P;
      pr.hits = hitsb + (size_t)c * 5 * P;
      pr.table = tabb + (size_t)c * P * 256;
      pr.peak = peakb + (size_t)c * P;
      pr.P = P;
      HotOut ho;
      ho.kind = 0;
      ho.label = 0;
      ho.deep = DEEP_NONE;
      ho.conf = 0.0;
      ho.rho = 0.0;
      ho.rsel = 0;
      ho.dyn = 0;
      if (valid) {
        GroupConst gc;
        gc.ok = member;
        gc.mu = member ? s_gmu[c * G + gid] : 0.0;
        gc.thr = member ? s_gthr[c * G + gid] : 0.0;
        hot_px<T>(a, f, pr, p, pre[c], on_lat, s_bt, wa, wb, wc, gc, ho);
        st(confb + o, ho.conf);
        kindb[o] = (uint8_t)ho.kind;
        kc += 1ull << (9 * ho.kind);
      }
      dyn_late[c] = ho.dyn;
      lbits |= ((unsigned)ho.label & 1u) << c;
      const bool is_copy = valid && ho.kind == K_COPY;
      if (is_copy) copybits |= 1u << c;
      const bool dq = valid && ho.deep != DEEP_NONE;
      const bool late = dq && (ho.deep == DEEP_GMM || ho.deep == DEEP_COMPAT);
      const unsigned qm = __ballot_sync(FULL, dq);
      if (qm) {
        if (__ballot_sync(FULL, is_copy)) {
          // copies in this plane-tile need their anchors' final labels now
          if (dq) {
            if (ho.deep == DEEP_MEANVAR) {
              cold_meanvar<T, KMAX>(pr, p, pre[c].meta, ho.rsel,
                                    (double)pre[c].vb, ho.rho,
                                    a.q.variance_floor);
            } else {
              const int lbl = cold_gmm<T, KMAX>(
                  pr, p, pre[c].meta, (double)pre[c].vb, ho.rho, gp, K,
                  ho.deep == DEEP_GMM);
              lbits |= ((unsigned)lbl & 1u) << c;
              gmmbits |= 1u << c;  // dyn written with its label below
            }
          }
        } else {
          const int nq = __popc(qm);
          if (wq_n + nq > LQ_CAP) {
            unsigned base = 0;
            if (lane == 0) base = atomicAdd(sync + 3, (unsigned)wq_n);
            base = __shfl_sync(FULL, base, 0);
            __syncwarp();
            for (int e = lane; e < wq_n; e += 32) {
              dq_code[(size_t)base + e] = s_qc[e];
              dq_rho[(size_t)base + e] = s_qr[e];
            }
            __syncwarp();
            wq_n = 0;
          }
          if (dq) {
            const int pos = wq_n + __popc(qm & ((1u << lane) - 1u));
            s_qc[pos] = 1ull | ((unsigned long long)ho.deep << 1) |
                        ((unsigned long long)ho.rsel << 3) |
                        ((unsigned long long)c << 6) |
                        ((unsigned long long)pre[c].vb << 8) |
                        ((unsigned long long)p << 16);
            s_qr[pos] = ho.rho;
          }
          wq_n += nq;
          if (late) gmmbits |= 1u << (8 + c);  // label arrives via deep kernel
        }
      }
      // ---- group partials of this plane (exact sums)
      if (any_member) {
        unsigned todo = any_member;
        while (todo) {
          const int leader = __ffs(todo) - 1;
          const int g = __shfl_sync(FULL, gid, leader);
          const bool mine = member && gid == g;
          const unsigned mm = __ballot_sync(FULL, mine);
          todo &= ~mm;
          const unsigned sall = warp_sum_u32(mine ? (unsigned)pre[c].vb : 0u);
          const bool hit = mine && ho.kind == L_GROUP;
          const unsigned hm = __ballot_sync(FULL, hit);
          unsigned sv = 0, qh = 0, ql = 0;
          if (hm) {
            unsigned long long qv = 0;
            if (hit) {
              const double cq = ho.conf * 4503599627370496.0;  // 2^52
              qv = cq > 0.0 ? (unsigned long long)cq : 0ull;
            }
            sv = warp_sum_u32(hit ? (unsigned)pre[c].vb : 0u);
            qh = warp_sum_u32((unsigned)(qv >> CONF_SPLIT));
            ql = warp_sum_u32((unsigned)(qv & ((1ull << CONF_SPLIT) - 1ull)));
          }
          if (lane == 0) {
            unsigned long long* e = s_acc + acc_grp(D, G, c, g);
            atomicAdd(e + 4, (unsigned long long)sall);
            atomicAdd(e + 5, (unsigned long long)__popc(mm));
            if (hm) {
              atomicAdd(e + 0, (unsigned long long)__popc(hm));
              atomicAdd(e + 1, (unsigned long long)sv);
              atomicAdd(e + 2, (unsigned long long)qh);
              atomicAdd(e + 3, (unsigned long long)ql);
            }
          }
        }
      }
    }

    // ---- finish: labels, copy resolution, dyn words, union mask
    int fg = 0;
#pragma unroll
    for (int c = 0; c < D; ++c) {
      int label = (int)((lbits >> c) & 1u);
      const uint32_t o = (uint32_t)c * P + p;
      if ((gmmbits >> c) & 1u) {
        if (valid) dynb[o] = dyn_late[c] | ((uint32_t)label << 8);
      } else if ((gmmbits >> (8 + c)) & 1u) {
        label = 0;  // the deep kernel ORs in the label bit and the mask
        if (valid) dynb[o] = dyn_late[c];
      }
      const int al = __shfl_sync(FULL, label, anchor);
      if ((copybits >> c) & 1u) {
        label = al;
        dynb[o] = dyn_late[c] | ((uint32_t)al << 8);
      }
      fg |= label;
    }
    if (valid) maskb[p] = fg ? 255 : 0;
    fg_count += __popc(__ballot_sync(FULL, valid && fg));
    if (++kc_tiles >= KC_FLUSH) {
      lean_flush_kinds<D>(kc, s_acc, lane);
      kc_tiles = 0;
    }
  }
  if (wq_n) {
    unsigned base = 0;
    if (lane == 0) base = atomicAdd(sync + 3, (unsigned)wq_n);
    base = __shfl_sync(FULL, base, 0);
    __syncwarp();
    for (int e = lane; e < wq_n; e += 32) {
      dq_code[(size_t)base + e] = s_qc[e];
      dq_rho[(size_t)base + e] = s_qr[e];
    }
  }
  lean_flush_kinds<D>(kc, s_acc, lane);
  if (lane == 0 && fg_count)
    atomicAdd(s_acc + acc_fg(D), (unsigned long long)fg_count);
  __syncthreads();
  unsigned long long* gacc = (unsigned long long*)a.s.accum + (size_t)s * words;
  for (int i = threadIdx.x; i < words; i += LEAN_THREADS) {
    const unsigned long long v = s_acc[i];
    if (v) atomicAdd(gacc + i, v);
  }
}
