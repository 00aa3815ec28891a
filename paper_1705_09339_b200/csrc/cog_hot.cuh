// cog_hot.cuh -- the float32-state hot pass of the frame step (the
// throughput path).  Included inside the anonymous namespace of
// cog_kernels.cu, after cog_fast.cuh (FastConst, fmatch, the u16 prior).
//
// Work unit: one stride-aligned warp tile (stride rows x cw columns, so
// every copy pixel's anchor is in row 0 of the same tile).  A CTA is D
// warps; warp c runs plane c of the tile, one thread per plane-pixel (the
// reference's planes are independent, cascade.py:281), and the planes meet
// once per tile in shared memory for the union mask.  One thread therefore
// holds one plane-pixel's state: no plane loop, no register rotation, no
// spills, and ~60 warps per SM in flight.
//
// The hot loop has no calls and no binary64 fallback.  A plane-pixel whose
// fp32 decision lies inside a filter margin (the u16 prior's quantisation
// plus 1e-5 relative, see cog_fast.cuh) is DEFERRED: the hot pass writes
// nothing for it and queues it on the stream's worklist, where deep_kernel
// runs the general binary64 step (hot_px) for it.  MEANVAR hits and GMM
// fall-throughs are queued as before.  A label that only becomes known in
// the deep pass (GMM, deferred) is OR-ed into dyn and the mask there --
// together with the labels of the copy pixels that read it
// (kernels_numba.py:363-373): the queued item carries their positions.
//
// Loads per plane-pixel, in two dependent rounds: the frame byte, dyn,
// meta, streak (+ the pixel's class and group id); then the hot prior
// phat(v) from the u16 tile-major table and -- only when the cascade can
// reach a mode level or the confidence reads a mode -- the (mu, var) pairs
// of the two referenced modes, 8 bytes each from the 64-B record.

constexpr int HQ_CAP = 64;  // per-warp worklist buffer (one global atomic per flush)
// tiles evaluated side by side by one CTA (D warps each): fewer CTAs per
// frame, so fewer prologues and partial-sum flushes on small frames
#ifndef HOT_TPB
#define HOT_TPB 2  // 1..4
#endif
constexpr int HOT_QCAP_BYTES = HQ_CAP * 16;

// pending illumination reset / scheduled reorder of the plane-pixels this
// thread evaluates (the CTA's tiles, plane c): out of line, called once per
// frame, so the hot loop's registers never live across a call
template <int KMAX>
__device__ __noinline__ void hot_pending(const StepArgs* __restrict__ ap,
                                         int s, int c, int slot,
                                         bool do_reset, bool do_reorder,
                                         bool do_fold) {
  using T = float;
  const StepArgs& a = *ap;
  const int lane = threadIdx.x & 31;
  const int H = a.g.height, W = a.g.width, stride = a.g.stride;
  const int G = a.g.n_groups, D = a.g.depth;
  const uint32_t P = (uint32_t)H * (uint32_t)W;
  const int cw = a.cw;
  const int lrow = lane / cw, lcol = lane - lrow * cw;
  const bool lane_ok = lane < stride * cw;
  const PlaneRef<T> pr = plane_ref<T>(a, s, c);
  const double* gmu = a.s.g_mu + ((size_t)s * D + c) * G;
  for (int t = blockIdx.x * HOT_TPB + slot; t < a.n_tiles;
       t += gridDim.x * HOT_TPB) {
    const int ty = t / a.tiles_x, tx = t - ty * a.tiles_x;
    const int y = ty * stride + lrow, x = tx * cw + lcol;
    if (!(lane_ok && y < H && x < W)) continue;
    const uint32_t p = (uint32_t)y * (uint32_t)W + (uint32_t)x;
    if (do_reset) cold_reset<T, KMAX>(pr, p, a.q.initial_variance);
    if (do_reorder) {
      const int g0 = a.s.gid[(size_t)s * P + p];
      cold_reorder<T>(pr, p, (G > 0 && g0 != (int)UNGROUPED)
                                 ? gmu[g0] : (G > 0 ? gmu[0] : 0.0));
    }
    // neither of the two left anything in the packed hit bytes
    if (do_fold && !do_reset && !do_reorder) cold_fold_hits<T>(pr, p);
  }
}

// The level walk as a table (kernels_numba.py:286-334): the first level in
// mid_order whose test is not a miss decides.  Index = the three 2-bit level
// codes of meta (bits 4-9) * 64 + the test states of the three levels
// (2 bits each, GROUP / MEAN / MEANVAR: 0 miss, 1 hit, 3 undecided); value =
// the active level, L_GMM when every test misses or the order ends, 0xFF
// when an undecided test decides.
__device__ __align__(16) uint8_t g_walk[64 * 64];

// shared memory of one CTA; `big`: the group sums and constants do not fit
// (hundreds of groups) and live in global memory instead
// the pipelined variant's per-warp ring of round-1 stages (HOT_NS tiles in
// flight per warp): dyn[32] u32, streak[32] u32, meta[32] u16, gid[32] u16,
// frame[32] u8, cls[32] u8
#ifndef HOT_NS
#define HOT_NS 4
#endif
#ifndef HOT_PIPE
#define HOT_PIPE 1  // build-time A/B switch (tools/gpu_ab_build.sh)
#endif
constexpr int HOT_STAGE_BYTES = 592;
constexpr int HS_DYN = 0, HS_STREAK = 128, HS_META = 256, HS_GID = 320,
              HS_FRAME = 384, HS_CLS = 416,
              HS_PIX = 448,  // u32[32]: each lane's pixel index, ~0 = invalid
              HS_TILE = 576; // u32: the tile's index

// shared memory of one CTA, fixed-size parts first (compile-time offsets):
// the level-walk table, class constants, the tiles' label words, the
// per-warp worklist buffers, the pipelined ring; then the per-warp partial
// slices and the group constants, whose size depends on the group count
__host__ __device__ constexpr int hot_off_cw() { return 64 * 64; }
__host__ __device__ constexpr int hot_off_ctm() { return hot_off_cw() + 48; }
__host__ __device__ constexpr int hot_off_lab() { return hot_off_ctm() + 32; }
__host__ __device__ constexpr int hot_off_qc(int d) {
  return hot_off_lab() + ((2 * d * HOT_TPB * 4 + 15) & ~15);
}
__host__ __device__ constexpr int hot_off_qr(int d) {
  return hot_off_qc(d) + d * HOT_TPB * HOT_QCAP_BYTES / 2;
}
__host__ __device__ constexpr int hot_off_ring(int d) {
  return hot_off_qr(d) + d * HOT_TPB * HOT_QCAP_BYTES / 2;
}
__host__ __device__ constexpr int hot_off_var(int d, bool pipe) {
  return hot_off_ring(d) + (pipe ? d * HOT_TPB * HOT_NS * HOT_STAGE_BYTES : 0);
}
// `big`: the group sums and constants do not fit (hundreds of groups) and
// live in global memory instead
__host__ __device__ inline size_t hot_smem_bytes(int d, int G, bool big,
                                                 bool pipe = false) {
  const int g = big ? 0 : G;
  const int warps = d * HOT_TPB;
  const size_t wpad = ((size_t)acc_words(d, g) + 1) & ~(size_t)1;
  return (size_t)hot_off_var(d, pipe) + (size_t)warps * wpad * 8 +
         (size_t)2 * d * g * 4 + 16;
}

// one plane-pixel's loads, handed from the front half of the tile loop
// (gates + loads) to the back half (evaluation + writes); in the pipelined
// variant the front half runs one tile ahead of the back half
struct HotIn {
  uint32_t p;     // pixel index (0 for an invalid lane)
  uint32_t dyn, sk;
  uint32_t mf;    // meta | the front half's gates << 16 (HI_*)
  uint32_t pk;    // v | cls << 8 | gid << 16
  uint32_t q16;   // hot prior at v (its own register: packing it would
                  // wait for the load in the front half)
  float2 m0, m1;  // the two referenced modes (mu, var)
};
enum : uint32_t { HI_VALID = 1u << 16, HI_SKIP = 1u << 17, HI_COPY = 1u << 18,
                  HI_GHIT_SHIFT = 19 };  // ghit & 3 at bits 19-20

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src,
                                           uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst),
               "l"(src), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// A warp's buffered worklist items go out two-ended, so that the deep pass
// runs warps of one item type: fp32 MEANVAR updates grow from the front of
// the stream's worklist (count in sync[2]), GMM fall-throughs and deferred
// plane-pixels from its back (count in sync[3]); one 64-bit atomic reserves
// both ranges.  The capacity is every plane-pixel, so the ends cannot meet.
#ifndef HOT_TWO_ENDED
#define HOT_TWO_ENDED 1  // build-time A/B switch (tools/gpu_ab_build.sh)
#endif
static_assert(HQ_CAP == 64, "hot_flush moves two entries per lane");
__device__ __forceinline__ void hot_flush(const unsigned long long* qc,
                                          const double* qr, int n,
                                          uint32_t* sync,
                                          unsigned long long* dq_code,
                                          double* dq_rho, size_t dq_cap,
                                          int lane) {
  __syncwarp();
  const bool v0 = lane < n, v1 = lane + 32 < n;
  const unsigned long long c0 = v0 ? qc[lane] : 0ull;
  const unsigned long long c1 = v1 ? qc[lane + 32] : 0ull;
  const bool a0 = v0 && (!HOT_TWO_ENDED ||
                        (((c0 >> 1) & 3ull) == (unsigned long long)DEEP_MEANVAR &&
                         !(c0 & ITEM_DEFERRED)));
  const bool a1 = v1 && (!HOT_TWO_ENDED ||
                        (((c1 >> 1) & 3ull) == (unsigned long long)DEEP_MEANVAR &&
                         !(c1 & ITEM_DEFERRED)));
  const unsigned ma0 = __ballot_sync(FULL, a0), ma1 = __ballot_sync(FULL, a1);
  const unsigned mb0 = __ballot_sync(FULL, v0 && !a0);
  const unsigned mb1 = __ballot_sync(FULL, v1 && !a1);
  const unsigned na = __popc(ma0) + __popc(ma1);
  unsigned long long old = 0ull;
  if (lane == 0)
    old = atomicAdd(reinterpret_cast<unsigned long long*>(sync + 2),
                    (unsigned long long)na |
                        ((unsigned long long)((unsigned)n - na) << 32));
  const unsigned base_a = __shfl_sync(FULL, (unsigned)old, 0);
  const unsigned base_b = __shfl_sync(FULL, (unsigned)(old >> 32), 0);
  const unsigned lt = (1u << lane) - 1u;
  if (v0) {
    const size_t i = a0 ? (size_t)base_a + __popc(ma0 & lt)
                        : dq_cap - 1 - ((size_t)base_b + __popc(mb0 & lt));
    dq_code[i] = c0;
    dq_rho[i] = qr[lane];
  }
  if (v1) {
    const size_t i =
        a1 ? (size_t)base_a + __popc(ma0) + __popc(ma1 & lt)
           : dq_cap - 1 - ((size_t)base_b + __popc(mb0) + __popc(mb1 & lt));
    dq_code[i] = c1;
    dq_rho[i] = qr[lane + 32];
  }
  __syncwarp();
}

// compile-time configuration of a hot_kernel instantiation: FL < 0 reads
// the feature switches from the params, else bit 0 sampling, 1 grouping,
// 2 change-hypothesis probe, 3 rate scaling, 4 literal confidence; ST = 0
// reads the stride from the geometry
enum : int { HF_SAMPLING = 1, HF_GROUPING = 2, HF_CHP = 4, HF_RATE = 8,
             HF_LITERAL = 16 };
constexpr int HF_DEFAULT = HF_SAMPLING | HF_GROUPING | HF_CHP | HF_RATE;

#ifndef COG_HOT_MINB
#define COG_HOT_MINB 30
#endif
// The pipelined variant (16-pixel rows, 4-byte aligned mask words) builds the
// union mask without a rendezvous of the tile's plane warps: the launcher
// zeroes the mask, each plane warp ORs the bytes of its foreground labels
// into it with word atomics (nothing to do for an all-background tile, the
// common case), and the bytes a warp turned 0 -> 255 are its share of the
// foreground count -- the same rule the deep pass uses for late labels.
#ifndef HOT_MASK_ATOMIC
#define HOT_MASK_ATOMIC 1  // build-time A/B switch (tools/gpu_ab_build.sh)
#endif

// PIPE (stride 2, rows 16-byte aligned): the round-1 arrays of the warp's
// next HOT_NS - 1 tiles are in flight as 16-byte cp.async copies into the
// warp's shared ring, and the front half (gates, prior and mode loads) of
// tile j + 1 is issued before the back half of tile j runs, so both load
// rounds overlap a whole tile of evaluation without holding registers
template <int KMAX, int D, int ST, int FL, bool PIPE, bool BIG>
__global__ void __launch_bounds__(32 * D * HOT_TPB, COG_HOT_MINB / (D * HOT_TPB))
    hot_kernel(const __grid_constant__ StepArgs a,
               const __grid_constant__ FastConst k) {
  static_assert(!PIPE || ST == 2, "the pipelined ring is laid out for stride 2");
  using T = float;
  constexpr int R = rec_elems(KMAX), WO = rec_w(KMAX);
  extern __shared__ __align__(16) unsigned char h_raw[];
  const int s = blockIdx.y;
  const int G = a.g.n_groups;
  const int H = a.g.height, W = a.g.width;
  const int stride = ST > 0 ? ST : a.g.stride;
  const int cw = ST > 0 ? ST * (32 / (ST * ST) > 0 ? 32 / (ST * ST) : 1) : a.cw;
  const uint32_t P = (uint32_t)k.P;  // H * W (launcher)
  const int words = acc_words(D, G);
  constexpr bool big = BIG;  // group sums / constants in global memory
  const int sG = big ? 0 : G;
  const int wpad = k.wpad;   // (acc_words(D, sG) + 1) & ~1 (launcher)
  constexpr int NW = D * HOT_TPB;   // warps per CTA
  constexpr int NT = 32 * NW;       // threads per CTA
  // read once (volatile: the compiler would otherwise re-read %tid.x, a
  // slow special-register move, all over the loop instead of keeping it)
  unsigned tid_x;
  asm volatile("mov.u32 %0, %%tid.x;" : "=r"(tid_x));
  const int lane = tid_x & 31;
  const int w = tid_x >> 5;
  // this warp's tile of the CTA's HOT_TPB and its plane (no division)
  const int slot = (w >= D) + (HOT_TPB > 2 && w >= 2 * D) +
                   (HOT_TPB > 3 && w >= 3 * D);
  const int c = w - slot * D;
  const bool sampling = FL < 0 ? a.q.sampling_on != 0 : (FL & HF_SAMPLING) != 0;
  const bool grouping = FL < 0 ? a.q.grouping_on != 0 : (FL & HF_GROUPING) != 0;
  const bool chp_on = FL < 0 ? a.q.chp_on != 0 : (FL & HF_CHP) != 0;
  const bool rate_on = FL < 0 ? a.q.rate_scaling_on != 0 : (FL & HF_RATE) != 0;
  const bool literal = FL < 0 ? a.q.literal_conf != 0 : (FL & HF_LITERAL) != 0;

  // ---- shared: warp-private partial slices (lane 0 adds, no atomics),
  // per-warp worklist buffers, the level-walk table, the per-class
  // confidence constants, group constants (float), the tiles' per-plane
  // label words (double buffered)
  uint8_t* const s_walk = h_raw;                                    // [64 * 64]
  float4* const s_cw = (float4*)(h_raw + hot_off_cw());             // [3] wa wb wc 1/(wb+wc)
  float* const s_ctm = (float*)(h_raw + hot_off_ctm());             // [3] conf margins
  unsigned* const s_lab = (unsigned*)(h_raw + hot_off_lab());       // [2][NW]
  unsigned long long* const s_qc =
      (unsigned long long*)(h_raw + hot_off_qc(D));                 // [NW][HQ_CAP]
  double* const s_qr = (double*)(h_raw + hot_off_qr(D));            // [NW][HQ_CAP]
  unsigned long long* const s_wacc =
      (unsigned long long*)(h_raw + hot_off_var(D, PIPE));          // [NW][wpad]
  float* const s_gmu = (float*)(s_wacc + NW * wpad);                // [D*G]
  float* const s_gthr = s_gmu + D * sG;                             // [D*G]
  const double* gmu_d = a.s.g_mu + (size_t)s * D * G;
  const double* gvar_d = a.s.g_var + (size_t)s * D * G;
  for (int i = threadIdx.x; i < D * sG; i += NT) {
    s_gmu[i] = (float)gmu_d[i];
    s_gthr[i] = (float)(a.q.match_lambda * sqrt(gvar_d[i]));
  }
  for (int i = threadIdx.x; i < NW * wpad; i += NT) s_wacc[i] = 0ull;
  for (int i = threadIdx.x; i < 64 * 64 / 16; i += NT)
    reinterpret_cast<uint4*>(s_walk)[i] = reinterpret_cast<const uint4*>(g_walk)[i];
  if (threadIdx.x < 3) {
    const int q = threadIdx.x;
    s_cw[q] = make_float4(k.w[3 * q], k.w[3 * q + 1], k.w[3 * q + 2],
                          k.wbc_inv[q]);
    s_ctm[q] = k.ct_margin[q];
  }
  __syncthreads();
  // let the frame's deep kernel be scheduled now (it waits on this grid's
  // completion before touching anything); hides the launch gap
  asm volatile("griddepcontrol.launch_dependents;");
  unsigned long long* const wacc = s_wacc + w * wpad;
  unsigned long long* const qc = s_qc + w * HQ_CAP;
  double* const qr = s_qr + w * HQ_CAP;

  // 32-bit element indices from the state arrays' own bases (the launcher
  // guarantees streams * d * 5 * P and the record elements < 2^32)
  const uint32_t s1 = (uint32_t)s * P;                  // [s][P] arrays
  const uint32_t plane = ((uint32_t)s * D + c) * P;     // [s][d][P] arrays
  T* const mix_s = (T*)a.s.mix;
  T* const conf_s = (T*)a.conf;
  unsigned long long* const gacc =
      (unsigned long long*)a.s.accum + (size_t)s * words;
  uint32_t* const sync = a.s.sync + (size_t)s * 4;
  const size_t dq_cap = dq_capacity(D, P);
  unsigned long long* const dq_code =
      (unsigned long long*)a.s.deepq + (size_t)s * dq_cap;
  double* const dq_rho = a.s.deeprho + (size_t)s * dq_cap;
  const uint32_t pend = *(volatile uint32_t*)(sync + 1);
  const bool do_reset = (pend & 1u) != 0;
  const bool do_reorder = a.reorder_now != 0;
  // the packed hit bytes are folded into the wide counters before a byte
  // can wrap (finalize_stream counts the frames since they were cleared)
  uint32_t* const hitq = a.s.hitq;
  const bool do_fold = hitq != nullptr && (pend >> 8) >= HITQ_FOLD_AGE;
  // this warp's plane of the hot prior: tile t, bin v, slot at
  // (t * 256 + v) * 32 + slot
  const uint16_t* const tq =
      a.s.tabq + ((size_t)s * D + c) * (size_t)a.n_tiles * 8192 + lane;

  const int lrow = lane / cw, lcol = lane - lrow * cw;
  const bool lane_ok = lane < stride * cw;
  const bool on_lat = (lrow == 0) && (lcol % stride == 0);
  const int anchor = lcol - lcol % stride;

  // ---- a pending illumination reset / scheduled reorder (rare, uniform
  // over the grid): applied per plane-pixel before the frame's own pass,
  // over the same tiles this thread evaluates below
  if (do_reset || do_reorder || do_fold) {
    hot_pending<KMAX>(&a, s, c, slot, do_reset, do_reorder, do_fold);
    // every plane-pixel's packed hit bytes are zero now: their age restarts
    if (hitq != nullptr && blockIdx.x == 0 && threadIdx.x == 0)
      atomicAdd(gacc + acc_flag(D, G), 1ull);
  }

  unsigned long long kc = 0ull;  // kind counts, 7 x 9 bits
  int kc_units = 0;
  int wq_n = 0;
  unsigned fg_count = 0;
  constexpr bool AMASK = PIPE && HOT_MASK_ATOMIC != 0 && D > 1;
  // the CTA's tiles: round r covers tiles (blockIdx.x + r * gridDim.x) *
  // HOT_TPB + slot; t = ty * tiles_x + tx advanced without a division
  const int step = gridDim.x * HOT_TPB;
  const int dty = step / a.tiles_x, dtx = step - dty * a.tiles_x;
  const int t_first = blockIdx.x * HOT_TPB + slot;
  const int n_it = ((int)a.n_tiles - (int)(blockIdx.x * HOT_TPB) + step - 1) / step;

  // ---- front half of a tile: the gates that decide which loads are
  // needed, then the loads.  Round 1 comes from global memory, or from the
  // ring stage `st` the copies have filled
  auto front = [&](int t, int ty_, int tx_, const unsigned char* st) -> HotIn {
    HotIn in;
    bool valid;
    uint32_t p;
    if (PIPE) {
      p = *reinterpret_cast<const uint32_t*>(st + HS_PIX + lane * 4);
      t = *reinterpret_cast<const int*>(st + HS_TILE);
      valid = p != 0xFFFFFFFFu;
      if (!valid) p = 0u;
    } else {
      const int y = ty_ * stride + lrow, x = tx_ * cw + lcol;
      valid = lane_ok && t < a.n_tiles && y < H && x < W;
      p = valid ? (uint32_t)y * (uint32_t)W + (uint32_t)x : 0u;
    }
    const uint32_t o = plane + p;
    int vb, gid, cls;
    uint32_t dyn, meta, sk;
    if (PIPE) {
      dyn = *reinterpret_cast<const uint32_t*>(st + HS_DYN + lane * 4);
      sk = *reinterpret_cast<const uint32_t*>(st + HS_STREAK + lane * 4);
      meta = *reinterpret_cast<const uint16_t*>(st + HS_META + lane * 2);
      gid = *reinterpret_cast<const uint16_t*>(st + HS_GID + lane * 2);
      vb = st[HS_FRAME + lane];
      cls = st[HS_CLS + lane];
    } else {
      // addresses are in range for every lane; invalid lanes read pixel 0
      // and write nothing
      vb = a.frame[o];
      dyn = a.s.dyn[o];
      meta = a.s.meta[o];
      sk = a.s.streak[o];
      gid = a.s.gid[s1 + p];
      cls = a.s.cls[s1 + p];
    }
    const bool member = valid && G > 0 && gid != (int)UNGROUPED;
    const int gidx = member ? c * G + gid : 0;
    const int dv = abs(vb - (int)(dyn & 0xFF));
    const bool changed = dv > k.eps_i;
    const bool asleep = sampling && (dyn >> 16) != 0u;
    const bool waking = sampling && !asleep && ((dyn >> 9) & 1u);
    const bool skip = asleep && !changed;
    const bool copy = waking && !changed && !on_lat;
    const bool ev = valid && !skip && !copy;
    const uint32_t c0 = (meta >> 4) & 3u, c1 = (meta >> 6) & 3u;
    const uint32_t r0 = (meta >> 10) & 7u, r1 = (meta >> 13) & 7u;
    const uint32_t top = (c0 == L_GROUP && !grouping) ? c1 : c0;
    const bool gtop = top == L_GROUP && member;
    float gm = 0.0f, gthr = 1.0f;
    if (member) {
      if (!big) {
        gm = s_gmu[gidx];
        gthr = s_gthr[gidx];
      } else {
        gm = (float)gmu_d[gidx];
        gthr = (float)(a.q.match_lambda * sqrt(gvar_d[gidx]));
      }
    }
    const int ghit = (grouping && member) ? fmatch((float)vb, gm, gthr) : 0;
    const bool chp_hit = chp_on && !changed;
    // the modes are needed unless the confidence reads the group and the
    // walk stops at the group level (or the probe) before any mode level
    const bool need =
        ev && !(gtop && (chp_hit || (c0 == L_GROUP && ghit == 1)));
    const T* const rec = mix_s + o * R;  // this plane-pixel's mixture record
    uint32_t q16 = 0u;
    in.m0 = make_float2(0.0f, 1.0f);
    in.m1 = in.m0;
    if (ev) q16 = __ldcg(tq + ((size_t)t * 256 + vb) * 32);
    if (need) {
      in.m0 = *reinterpret_cast<const float2*>(rec + 2 * r0);
      in.m1 = *reinterpret_cast<const float2*>(rec + 2 * r1);
    }
    in.p = p;
    in.dyn = dyn;
    in.sk = sk;
    in.q16 = q16;
    in.mf = (meta & 0xFFFFu) | (valid ? HI_VALID : 0u) | (skip ? HI_SKIP : 0u) |
            (copy ? HI_COPY : 0u) | (((uint32_t)ghit & 3u) << HI_GHIT_SHIFT);
    in.pk = (uint32_t)vb | ((uint32_t)cls << 8) | ((uint32_t)gid << 16);
    return in;
  };

  // ---- the pipelined variant's copy stream: lane l < 28 moves one 16-byte
  // chunk of one round-1 array per tile (rows of 16 pixels: dyn / streak 4
  // chunks a row, meta / gid 2, frame / cls 1)
  const char* cbase = nullptr;  // array base + plane + the chunk's row / column
  int csh = 0, crow = 0;
  uint32_t cdst = 0;            // shared address of the chunk in stage 0
  unsigned char* ring = nullptr;
  if (PIPE) {
    ring = h_raw + hot_off_ring(D) + w * (HOT_NS * HOT_STAGE_BYTES);
    int l = lane, chunk = 0;
    uint32_t d0 = 0;
    if (l < 8) {
      cbase = (const char*)(a.s.dyn + plane); csh = 2; crow = l >> 2; chunk = l & 3;
      d0 = HS_DYN + crow * 64;
    } else if (l < 16) {
      l -= 8;
      cbase = (const char*)(a.s.streak + plane); csh = 2; crow = l >> 2; chunk = l & 3;
      d0 = HS_STREAK + crow * 64;
    } else if (l < 20) {
      l -= 16;
      cbase = (const char*)(a.s.meta + plane); csh = 1; crow = l >> 1; chunk = l & 1;
      d0 = HS_META + crow * 32;
    } else if (l < 24) {
      l -= 20;
      cbase = (const char*)(a.s.gid + s1); csh = 1; crow = l >> 1; chunk = l & 1;
      d0 = HS_GID + crow * 32;
    } else if (l < 26) {
      l -= 24;
      cbase = (const char*)(a.frame + plane); csh = 0; crow = l;
      d0 = HS_FRAME + crow * 16;
    } else if (l < 28) {
      l -= 26;
      cbase = (const char*)(a.s.cls + s1); csh = 0; crow = l;
      d0 = HS_CLS + crow * 16;
    }
    cbase += chunk * 16;
    cdst = (uint32_t)__cvta_generic_to_shared(ring) + d0 + chunk * 16;
  }
  // copy tile (t, ty_, tx_) of this warp into ring stage `sidx`; rows past
  // the frame and tiles past the end are zero-filled
  auto copy_tile = [&](int t, int ty_, int tx_, int sidx) {
    __syncwarp();  // the stage's previous tile has been read by every lane
    {
      // each lane's pixel of this tile and the tile index ride along, so
      // the front half needs no cursor of its own
      unsigned char* st = ring + sidx * HOT_STAGE_BYTES;
      const int y = ty_ * 2 + lrow;
      const bool v = t < a.n_tiles && y < H;
      *reinterpret_cast<uint32_t*>(st + HS_PIX + lane * 4) =
          v ? (uint32_t)y * (uint32_t)W + (uint32_t)(tx_ * 16 + lcol)
            : 0xFFFFFFFFu;
      if (lane == 0) *reinterpret_cast<int*>(st + HS_TILE) = t;
    }
    if (lane < 28) {
      const int y = ty_ * 2 + crow;
      const bool ok = t < a.n_tiles && y < H;
      const size_t pix = ok ? (size_t)y * W + (size_t)tx_ * 16 : 0;
      cp_async16(cdst + sidx * HOT_STAGE_BYTES, cbase + (pix << csh),
                 ok ? 16u : 0u);
    }
    cp_async_commit();
  };
  auto advance = [&](int& ty_, int& tx_) {
    ty_ += dty;
    tx_ += dtx;
    if (tx_ >= a.tiles_x) {
      tx_ -= a.tiles_x;
      ty_ += 1;
    }
  };

  // the tile cursor: of the copies when pipelined, else of the front half
  int ty = t_first / a.tiles_x, tx = t_first - ty * a.tiles_x;
  int tf = t_first;
  HotIn nxt;
  if (PIPE) {
    // the pending pass wrote through other lanes than the ones that copy
    __syncwarp();
#pragma unroll
    for (int j = 0; j < HOT_NS - 1; ++j) {
      copy_tile(tf, ty, tx, j);
      tf += step;
      advance(ty, tx);
    }
    cp_async_wait<HOT_NS - 2>();
    __syncwarp();
    nxt = front(0, 0, 0, ring);
  }
  for (int it = 0; it < n_it; ++it) {
    HotIn in;
    if (PIPE) {
      copy_tile(tf, ty, tx, (it + HOT_NS - 1) % HOT_NS);
      tf += step;
      advance(ty, tx);
      in = nxt;
      if (it + 1 < n_it) {
        cp_async_wait<HOT_NS - 2>();
        __syncwarp();
        nxt = front(0, 0, 0, ring + ((it + 1) % HOT_NS) * HOT_STAGE_BYTES);
      }
    } else {
      in = front(tf, ty, tx, nullptr);
      tf += step;
      advance(ty, tx);
    }

    // ---- back half: the loaded values and the front half's gates
    const bool valid = (in.mf & HI_VALID) != 0u;
    const uint32_t p = in.p;
    const uint32_t o = plane + p;
    const int vb = in.pk & 0xFF;
    const int cls = (in.pk >> 8) & 3u;
    const int gid = in.pk >> 16;
    const uint32_t dyn = in.dyn, sk = in.sk;
    const uint32_t meta = in.mf & 0xFFFFu;
    const uint32_t q16 = in.q16;
    const float2 m0 = in.m0, m1 = in.m1;
    const bool member = valid && G > 0 && gid != (int)UNGROUPED;
    const int gidx = member ? c * G + gid : 0;
    const int dv = abs(vb - (int)(dyn & 0xFF));
    const bool changed = dv > k.eps_i;
    const int last_label = (dyn >> 8) & 1u;

    // ---- sampling gate (kernels_numba.py:189-216): skip, copy, evaluate
    // (after waking on a change the streak restarts)
    const bool asleep = sampling && (dyn >> 16) != 0u;
    const bool skip = (in.mf & HI_SKIP) != 0u;
    const bool copy = (in.mf & HI_COPY) != 0u;
    const bool ev = valid && !skip && !copy;

    // ---- level codes, the group test from shared memory
    const uint32_t c0 = (meta >> 4) & 3u, c1 = (meta >> 6) & 3u;
    const uint32_t r0 = (meta >> 10) & 7u, r1 = (meta >> 13) & 7u;
    const uint32_t top = (c0 == L_GROUP && !grouping) ? c1 : c0;
    const bool gtop = top == L_GROUP && member;
    const float vf = (float)vb;
    float gm = 0.0f, gthr = 1.0f;
    if (member) {
      if (!big) {
        gm = s_gmu[gidx];
        gthr = s_gthr[gidx];
      } else {
        gm = (float)gmu_d[gidx];
        gthr = (float)(a.q.match_lambda * sqrt(gvar_d[gidx]));
      }
    }
    const bool chp_hit = chp_on && !changed;
    T* const rec = mix_s + o * R;  // this plane-pixel's mixture record

    // ---- evaluation (kernels_numba.py:239-359) in fp32; a decision whose
    // fp32 operands lie inside the filter margin defers the plane-pixel
    const float thr0 = k.lam * (m0.y * rsqrt_approx(m0.y));
    const float thr1 = k.lam * (m1.y * rsqrt_approx(m1.y));
    const float4 cwv = s_cw[cls];  // wa, wb, wc, 1 / (wb + wc)
    const float wa = cwv.x, wb = cwv.y, wc = cwv.z;
    const bool top1 = top == L_MEANVAR;
    const float mt = gtop ? gm : (top1 ? m1.x : m0.x);
    const float dn = gtop ? gthr : (top1 ? thr1 : thr0);
    const float ph = (float)q16 * PH_Q;
    const float btl = (float)dv * (1.0f / 255.0f);
    const float bt = literal ? btl : 1.0f - btl;
    const float gtl = fminf(fabsf(vf - mt) * rcp_approx(dn), 1.0f);
    const float gt = literal ? gtl : 1.0f - gtl;
    const float wbc = __fmaf_rn(wb, bt, __fmul_rn(wc, gt));
    const bool floor_ = ph < k.pf;
    const float cf_ev = floor_ ? __fmul_rn(wbc, cwv.w) : __fmaf_rn(wa, ph, wbc);
    const float ct_m = s_ctm[cls];
    bool deferred = ev && (fabsf(ph - k.pf) <= k.pf_margin ||
                           fabsf(cf_ev - k.ct) <= ct_m);
    // the level tests, then the first decisive one in mid_order (table)
    const uint32_t codes = ((meta >> 4) & 63u) << 6;
    uint32_t sg = (in.mf >> HI_GHIT_SHIFT) & 3u;  // 0 miss, 1 hit, 3 undecided
    uint32_t sm0 = (uint32_t)fmatch(vf, m0.x, thr0) & 3u;
    uint32_t sm1 = (uint32_t)fmatch(vf, m1.x, thr1) & 3u;
    auto walk = [&]() {
      const int v = s_walk[codes | sg | (sm0 << 2) | (sm1 << 4)];
      return v == 0xFF ? -1 : v;
    };
    int active = L_CHP, label = chp_hit ? last_label : 0;
    if (!chp_hit) {
      active = walk();
      // a matched mode must also sit inside the background weight prefix,
      // else the walk continues (kernels_numba.py:298-311); only when the
      // matched mode is not the first one
      for (int guard = 0; guard < 2 && ev; ++guard) {
        const bool m = active == L_MEAN && r0 > 0;
        const bool mv = active == L_MEANVAR && r1 > 0;
        if (!m && !mv) break;
        const uint32_t rr = m ? r0 : r1;
        // w_0 .. w_{K-2} in one round of 8-byte loads, summed in the
        // reference's order in binary64
        float wv[KMAX];
#pragma unroll
        for (int i = 0; i + 1 < KMAX; i += 2) {
          const float2 t2 = *reinterpret_cast<const float2*>(rec + WO + i);
          wv[i] = t2.x;
          wv[i + 1] = t2.y;
        }
        double acc = 0.0;
#pragma unroll
        for (int q = 0; q + 1 < KMAX; ++q)
          if ((uint32_t)q < rr) acc = acc + (double)wv[q];
        if (acc <= a.q.background_threshold) break;
        if (m) sm0 = 0u;
        else sm1 = 0u;
        active = walk();
      }
    }
    if (active < 0) {
      deferred |= ev;
      active = L_GMM;
    }
    const bool fast = ev && !deferred;
    const int deep = !fast ? DEEP_NONE
                           : (active == L_MEANVAR ? DEEP_MEANVAR
                                                  : (active == L_GMM ? DEEP_GMM
                                                                     : DEEP_NONE));
    double rho = a.q.learning_rate;
    if (rate_on) {
      double relax = 1.0 - (double)cf_ev;
      if (relax < a.q.rate_floor) relax = a.q.rate_floor;
      rho = a.q.learning_rate * relax;
    }
    const uint32_t la_bits = dyn & (7u << 10);  // last_active + 1, kept
    int kind;
    uint32_t dyn_out;
    float cf = 0.0f;
    if (skip) {
      // asleep and unchanged (kernels_numba.py:194-203)
      const uint32_t clk = (dyn >> 16) - 1u;
      kind = K_SKIP;
      label = last_label;
      dyn_out = (uint32_t)vb | ((uint32_t)last_label << 8) |
                (((uint32_t)(clk == 0u) | ((dyn >> 9) & 1u)) << 9) | la_bits |
                (clk << 16);
    } else if (copy) {
      // waking, unchanged, off the lattice (kernels_numba.py:207-216)
      kind = K_COPY;
      label = 0;
      dyn_out = (uint32_t)vb | la_bits | ((uint32_t)a.q.sleep_frames << 16);
    } else {
      // ---- bookkeeping (kernels_numba.py:335-359)
      kind = active;
      cf = cf_ev;
      const uint32_t skn0 = (asleep || !fast) ? 0u : sk;  // woke: restart
      const uint32_t skn =
          cf_ev > k.ct ? (skn0 == 0xffffffffu ? skn0 : skn0 + 1u) : 0u;
      uint32_t clock = 0u, wk = 0u;
      if (!sampling) {
        clock = dyn >> 16;
        wk = (dyn >> 9) & 1u;
      } else if ((long long)skn >= (long long)k.sat) {
        clock = (uint32_t)a.q.sleep_frames;
      }
      dyn_out = (uint32_t)vb | ((uint32_t)label << 8) | (wk << 9) |
                ((uint32_t)(active + 1) << 10) | (clock << 16);
      if (fast) {
        a.s.streak[o] = skn;
        // one dense RED per plane-pixel: a byte per level below GMM
        if (hitq != nullptr && active < L_GMM)
          atomicAdd(hitq + o, 1u << (8 * active));
        else
          atomicAdd(a.s.hits + (plane * 5 + (uint32_t)active * P + p), 1u);
        if (active == L_MEAN)
          rec[2 * r0] = (float)((1.0 - rho) * (double)m0.x + rho * (double)vb);
      }
    }

    // ---- copies take the anchor's label when it is known now; a label
    // that arrives with the deep pass (GMM, deferred) is written there,
    // for the anchor and its copies
    const bool late = deferred || deep == DEEP_GMM;
    const int now = late ? 0 : label;
    const int al = __shfl_sync(FULL, now, anchor);
    const bool is_copy = valid && copy;
    const int lab_now = is_copy ? al : now;
    if (valid && !deferred)
      a.s.dyn[o] = dyn_out | ((uint32_t)(is_copy ? al : (deep == DEEP_GMM ? 0 : label)) << 8);
    const unsigned cm = __ballot_sync(FULL, is_copy);

    // ---- worklist: MEANVAR hits, GMM fall-throughs, deferred plane-pixels
    const bool item = valid && (deferred || deep != DEEP_NONE);
    const unsigned qm = __ballot_sync(FULL, item);
    if (qm) {
      const int nq = __popc(qm);
      if (wq_n + nq > HQ_CAP) {
        hot_flush(qc, qr, wq_n, sync, dq_code, dq_rho, dq_cap, lane);
        wq_n = 0;
      }
      if (item) {
        unsigned cmk = 0;
        if (late && on_lat && cm) {
          // the copies of this anchor: lanes (r, anchor + dc) of the tile
          int b = 0;
          for (int r = 0; r < stride; ++r)
            for (int dc = 0; dc < stride; ++dc) {
              if (r == 0 && dc == 0) continue;
              if ((cm >> (r * cw + lcol + dc)) & 1u) cmk |= 1u << b;
              ++b;
            }
        }
        const int pos = wq_n + __popc(qm & ((1u << lane) - 1u));
        qc[pos] = 1ull | ((unsigned long long)deep << 1) |
                  ((unsigned long long)(deep == DEEP_MEANVAR ? r1 : 0u) << 3) |
                  ((unsigned long long)c << 6) |
                  ((unsigned long long)vb << 8) |
                  ((unsigned long long)p << 16) |
                  ((unsigned long long)cmk << ITEM_COPY_SHIFT) |
                  (deferred ? ITEM_DEFERRED : 0ull);
        qr[pos] = rho;
      }
      wq_n += nq;
    }

    // ---- outputs, kind counts
    if (valid && !deferred) {
      conf_s[o] = cf;
      a.kind[o] = (uint8_t)kind;
      kc += 1ull << (9 * kind);
    }

    // ---- group partials (exact sums) into the warp's private slice, or
    // straight into the stream's sums when they live in global memory
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
        const bool hit = mine && !deferred && kind == L_GROUP;
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
          if (!big) {
            unsigned long long* e = wacc + acc_grp(D, G, c, g);
            e[4] += sall;
            e[5] += (unsigned long long)__popc(mm);
            if (hm) {
              e[0] += (unsigned long long)__popc(hm);
              e[1] += sv;
              e[2] += qh;
              e[3] += ql;
            }
          } else {
            unsigned long long* e = gacc + acc_grp(D, G, c, g);
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
    if (++kc_units >= 511) {
#pragma unroll
      for (int q = 0; q < 7; ++q) {
        const unsigned v = warp_sum_u32((unsigned)((kc >> (9 * q)) & 511u));
        if (lane == 0) wacc[acc_kind(0, q)] += v;
      }
      kc = 0ull;
      kc_units = 0;
    }

    // ---- union mask of the tile (labels known now; late ones are OR-ed
    // in by the deep pass)
    const unsigned lb = __ballot_sync(FULL, valid && lab_now != 0);
    if (D == 1) {
      if (valid) a.mask[s1 + p] = (lb >> lane) & 1u ? 255 : 0;
      fg_count += __popc(lb);
    } else if (AMASK) {
      // lanes 0, 4, 8, ... own one aligned mask word (4 pixels of a row)
      const unsigned nib = (lb >> (lane & 28)) & 0xFu;
      if ((lane & 3) == 0 && nib != 0u) {
        const unsigned word = ((nib * 0x00204081u) & 0x01010101u) * 0xFFu;
        const unsigned old =
            atomicOr(reinterpret_cast<unsigned*>(a.mask + s1 + p), word);
        fg_count += __popc(word & ~old) >> 3;   // per lane; summed below
      }
    } else {
      unsigned* lab = s_lab + (it & 1) * NW + slot * D;
      if (lane == 0) lab[c] = lb;
      // the D warps of this tile only (named barrier 1 + slot; the ids are
      // compile-time constants, so the CTA reserves HOT_TPB + 1 barriers)
      if (HOT_TPB == 1 || slot == 0)
        asm volatile("bar.sync 1, %0;" ::"n"(32 * D) : "memory");
      else if (HOT_TPB == 2 || slot == 1)
        asm volatile("bar.sync 2, %0;" ::"n"(32 * D) : "memory");
      else if (HOT_TPB == 3 || slot == 2)
        asm volatile("bar.sync 3, %0;" ::"n"(32 * D) : "memory");
      else
        asm volatile("bar.sync 4, %0;" ::"n"(32 * D) : "memory");
      if (c == 0) {
        unsigned u = 0;
#pragma unroll
        for (int j = 0; j < D; ++j) u |= lab[j];
        if (valid) a.mask[s1 + p] = (u >> lane) & 1u ? 255 : 0;
        fg_count += __popc(u & __ballot_sync(FULL, valid));
      }
    }
  }
  if (wq_n) hot_flush(qc, qr, wq_n, sync, dq_code, dq_rho, dq_cap, lane);
#pragma unroll
  for (int q = 0; q < 7; ++q) {
    const unsigned v = warp_sum_u32((unsigned)((kc >> (9 * q)) & 511u));
    if (lane == 0) wacc[acc_kind(0, q)] += v;
  }
  if (AMASK) fg_count = warp_sum_u32(fg_count);
  if (lane == 0) wacc[acc_fg(D)] += fg_count;
  __syncthreads();
  const int sw = acc_words(D, sG);  // words held in shared
  for (int i = threadIdx.x; i < sw; i += NT) {
    unsigned long long v = 0;
#pragma unroll
    for (int j = 0; j < NW; ++j) v += s_wacc[j * wpad + i];
    if (v) atomicAdd(gacc + i, v);
  }
}
