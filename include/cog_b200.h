/*
 * cog_b200.h -- C-ABI of the B200-native Cascade-of-Gaussians hot path.
 *
 * Plain pointers and sizes; every pointer is a DEVICE pointer unless stated
 * otherwise; every call is asynchronous on `stream` (a cudaStream_t passed
 * as void*).  Return value: 0 on success, a positive cudaError_t from the
 * launch, or a negative COG_E* code for rejected arguments (nothing is
 * launched then).  The caller owns every buffer; nothing is allocated here.
 *
 * Each entry point replaces one reference interface of the `cogbg`
 * package (paths under /root/reference/pkg/src/cogbg/):
 *
 *   cog_prior_build      scene_prior.build_kde              :92-112
 *                        scene_prior.compute_residue_histogram :171-189
 *                        scene_prior.classify_pixel_dynamics :192-202
 *                        cascade.CascadeEngine._finalize_tables :213-216
 *   cog_gmm_warmup       training.train_engine GMM loop      :38-52
 *                        gmm.init_plane                      gmm.py:89-100
 *                        grouping.behavior_features           grouping.py:85-91
 *                        cascade.CascadeEngine._seed_level_order (mode refs) :218-235
 *   cog_set_levels       cascade.CascadeEngine._seed_level_order (level order) :236-241
 *   cog_step             kernels_numba.cascade_frame          :152-360
 *                        kernels_numba.resolve_copies         :363-373
 *                        cascade.CascadeEngine.process_frame  :261-318
 *                        cascade.CascadeEngine._update_groups :320-344
 *                        cascade.CascadeEngine._collect_stats :346-359
 *   cog_finalize         the per-frame tail of process_frame  :303-317
 *                        (group update, stats, illumination test) for
 *                        row-band shards after the partials are summed
 *   cog_apply_pending    cascade.CascadeEngine._reset_on_illumination :361-391
 *                        cascade.CascadeEngine.reorder_levels :393-417
 *   cog_baseline_frame   gmm.classify_frame                   gmm.py:112-133
 *                        (kernels_numba.baseline_frame :137-149)
 *   cog_export_state /   the engine's numpy state views, in the reference
 *   cog_import_state     dtypes and layouts (cascade.py:143-158), used by
 *                        model_io.save_model / load_model (model_io.py:61-227)
 *
 * State layout in HBM (one stream; `streams` copies back to back):
 *   mix      T[depth][P][R]   one record per plane-pixel (T = float or
 *            double): (mu_k, var_k) at [2k, 2k+1], w_k at [2*KB + k],
 *            KB = 3 / 5 / 8 for k <= 3 / <= 5 / <= 8, R = cog_mix_elems(k)
 *            (16 or 32: a pixel's whole mixture is one 64-B / 128-B float32
 *            record, so a full-mixture update touches one line instead of
 *            3k scattered ones)
 *   meta     u16[depth][P]   count | mid_order | mode_ref (packed)
 *   dyn      u32[depth][P]   chp_prev | last_label | waking | last_active | clock
 *   streak   u32[depth][P]
 *   hits     u32[depth][5][P]
 *   table    f32[depth][P][256] the reference-layout prior (exact values:
 *            binary64 paths, model files, host views)
 *   peak     f32[depth][P]
 *   tabq     u16, the hot prior of the float32 step: phat = table / peak
 *            quantised to round(phat * 65535), tile-major -- per plane
 *            [n_tiles][256][SL], bin v of the pixel in slot
 *            (row * cw + col) of warp tile t (stride rows x cw columns,
 *            SL = 32 * ceil(stride * cw / 32)) at (t * 256 + v) * SL + slot,
 *            so lanes of a warp that see the same value (or a neighbouring
 *            one) share a line; cog_tabq_elems() per stream, built by
 *            cog_tabq_build(); NULL for float64 engines
 *   cls      u8[P], gid u16[P] (0xFFFF = ungrouped)
 *   g_mu, g_var  f64[depth][G], g_members u32[G]
 *   accum    u64[cog_accum_words()], sync u32[4] (16-byte aligned: done
 *            counter, pending bits + hit-byte age, and the worklist's two
 *            counts, reserved together by one 64-bit atomic)
 *   deepq    u64 + f64 [cog_deepq_slots()]  per-frame worklist of MEANVAR /
 *            GMM plane-pixels (consumed and re-zeroed by the deep pass); the
 *            float32 hot pass fills it from both ends -- fp32 MEANVAR items
 *            from the front, GMM / deferred items from the back -- so the
 *            deep pass runs warps of one item type
 */
#ifndef COG_B200_H
#define COG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define COG_OK 0
#define COG_EINVAL (-1)
#define COG_EUNSUPPORTED (-2)

typedef struct cog_geom {
  int64_t total_pixels; /* pixels of the FULL frame (illumination threshold) */
  int32_t height;       /* rows held by this engine (a row band or a frame) */
  int32_t width;
  int32_t depth;        /* planes, 1..4 */
  int32_t k;            /* k_max, 1..8 */
  int32_t stride;       /* sampling lattice stride, 1..32 */
  int32_t n_groups;     /* G (groups per stream, max over streams) */
  int32_t streams;      /* independent streams stored back to back */
  int32_t state_f64;    /* 0: float32 mixture storage, 1: float64 */
  int32_t row0;         /* global row of this band's first row (% stride == 0) */
  int32_t pad_;
} cog_geom;

typedef struct cog_params {
  double learning_rate, match_lambda, background_threshold, variance_floor;
  double initial_variance, chp_epsilon, confidence_threshold, prior_floor;
  double rate_floor, illumination_fraction;
  double weights[9]; /* dynamics class c -> (alpha, beta, gamma) at [3c..3c+2] */
  int32_t saturation_frames, sleep_frames;
  int32_t sampling_on, grouping_on, rate_scaling_on, chp_on;
  int32_t literal_conf, compat;
  int32_t exact_group_sums; /* parity/debug: sum group confidences in the
                               reference's sequential pixel order (one
                               thread per group; small frames only) */
  int32_t variant;          /* step kernel: 0 automatic (fast for float32
                               state, lean / general for float64), 1 the
                               general kernel, 2 the lean kernel -- a parity
                               knob for tests, never read from the env */
} cog_params;

typedef struct cog_state {
  void *mix;
  uint16_t *meta;
  uint32_t *dyn;
  uint32_t *streak;
  uint32_t *hits;
  const float *table;
  const float *peak;
  const uint16_t *tabq;
  const uint8_t *cls;
  const uint16_t *gid;
  double *g_mu, *g_var;
  const uint32_t *g_members;
  uint64_t *accum;
  uint32_t *sync;
  uint64_t *deepq;   /* u64[cog_deepq_slots()] worklist (zero-initialised) */
  double *deeprho;   /* f64[cog_deepq_slots()] */
  uint32_t *hitq;    /* u32[depth][P] or NULL: the float32 hot pass counts
                        its CHP / GROUP / MEAN / MEANVAR hits here, one
                        byte per level in one word per plane-pixel (one
                        dense RED instead of one per level plane);
                        hits = hits + the bytes of hitq.  Folded back into
                        `hits` before a byte can wrap and wherever hits is
                        read or zeroed (reorder, reset, export). */
} cog_state;

/* Words of `accum` per stream (kinds, foreground, group partials). */
int64_t cog_accum_words(int32_t depth, int32_t n_groups);

/* Worklist slots per stream (deep-level plane-pixels of one frame). */
int64_t cog_deepq_slots(int32_t depth, int64_t n_pix);

/* Elements (of the state type) of one plane-pixel's mixture record. */
int64_t cog_mix_elems(int32_t k);

/* u16 elements of one stream's hot prior table (all planes), or -1. */
int64_t cog_tabq_elems(const cog_geom *geom);

/* Build one stream's hot prior tabq u16 from its reference-layout table
 * f32[depth][P][256] and peak f32[depth][P] (cascade.py:213-216:
 * phat = table / peak), round(phat * 65535) in binary64, tile-major. */
int cog_tabq_build(const cog_geom *geom, const float *table,
                   const float *peak, uint16_t *tabq, void *stream);

/* Scene prior for one stream: frames u8[N][depth][P].  Writes, for each
 * trailing window windows[j] (ascending, last == N), tables
 * f32[n_windows][depth][P][256]; peak f32[depth][P] of the last window
 * (<= 0 -> 1); optional hist u16[depth][P][256] (last window counts);
 * residue u32[P][3] (optional) and the dynamics class u8[P].
 * kern: f64[256][256] smoothing matrix (scene_prior._kernel_matrix). */
int cog_prior_build(const uint8_t *frames, int32_t n_frames, int32_t depth,
                    int64_t n_pix, const double *kern, const int32_t *windows,
                    int32_t n_windows, float *tables, float *peak,
                    uint16_t *hist, double residue_t1, double residue_t2,
                    double peaky_threshold, uint32_t *residue, uint8_t *cls,
                    void *stream);

/* GMM warm-up over N training frames u8[N][depth][P] for one stream.
 * Needs the stream's table (reference layout) already built.
 * Writes the mixture (state dtype per geom.state_f64), meta (count + mode
 * references ranked by prior mass, ties by w/sigma; mid_order left as
 * "ungrouped"), dyn (chp_prev = last frame), zeroes streak and hits.
 * Optional: features f64[P][2] (temporal variance of channel-0 rank-0
 * variance / weight series) and w_final f64[P]. */
int cog_gmm_warmup(const cog_geom *geom, const cog_params *prm,
                   const cog_state *st, const uint8_t *frames,
                   int32_t n_frames, double *features, double *w_final,
                   void *stream);

/* Level order seeding from the group map (grouped -> GROUP,MEAN,MEANVAR). */
int cog_set_levels(const cog_geom *geom, const cog_state *st, void *stream);

/* One frame for all streams: frame u8[streams][depth][P].  Outputs mask
 * u8[streams][P] (0/255), conf T[streams][depth][P], kind u8[streams]
 * [depth][P] and stats i64[streams][16] = {frame, n_chp, n_group, n_mean,
 * n_meanvar, n_gmm, n_skipped, n_foreground, unexplained, fired, ...}.
 * reorder_now: apply the scheduled level reorder before this frame.
 * fuse_finalize: 1 = the last CTA of each stream finalizes the frame
 * (single engine); 0 = leave the summed partials in accum for an external
 * all-reduce followed by cog_finalize (row-band shards). */
int cog_step(const cog_geom *geom, const cog_params *prm, const cog_state *st,
             const uint8_t *frame, uint8_t *mask, void *conf, uint8_t *kind,
             int64_t *stats, int64_t frame_index, int32_t reorder_now,
             int32_t fuse_finalize, void *stream);

int cog_finalize(const cog_geom *geom, const cog_params *prm,
                 const cog_state *st, int64_t *stats, int64_t frame_index,
                 void *stream);

/* Row-band shards on several GPUs: the cross-shard sum of the frame's exact
 * partials (what cascade.py:301-313, 320-344 computes over the whole frame)
 * as a one-shot all-reduce over peer memory, fused into the step's tail.
 * Every rank owns a mailbox of cog_mailbox_words() u64 words, mapped into
 * every peer (CUDA IPC / symmetric memory): [2 parities][n_ranks slots]
 * [accum words + 1 flag].  The last CTA of the step stores the rank's
 * partials into its slot of EVERY rank's mailbox (stores over NVLink), then
 * the flag (= seq, release at system scope); it -- fuse = 1 -- or
 * cog_finalize_p2p -- fuse = 0 -- waits for the n_ranks flags of its own
 * mailbox (acquire), sums the slots (integers: any order gives the same
 * sum) and runs the frame tail, identically on every rank.  seq > 0 must
 * be the same on every rank for the same frame and grow by one per step;
 * slots alternate by seq parity (a rank can only be one step ahead).
 * fuse = 1 makes the kernels of different ranks wait on one another: one
 * shard per GPU only.  streams must be 1. */
#define COG_MAX_RANKS 16
typedef struct cog_peers {
  int32_t n_ranks, rank;
  uint64_t seq;
  uint64_t *mailbox[COG_MAX_RANKS]; /* rank r's mailbox, as mapped here */
} cog_peers;

int64_t cog_mailbox_words(int32_t depth, int32_t n_groups, int32_t n_ranks);

int cog_step_p2p(const cog_geom *geom, const cog_params *prm,
                 const cog_state *st, const uint8_t *frame, uint8_t *mask,
                 void *conf, uint8_t *kind, int64_t *stats,
                 int64_t frame_index, int32_t reorder_now, int32_t fuse,
                 const cog_peers *peers, void *stream);

int cog_finalize_p2p(const cog_geom *geom, const cog_params *prm,
                     const cog_state *st, int64_t *stats, int64_t frame_index,
                     const cog_peers *peers, void *stream);

/* Materialise a pending illumination reset (device flag) and/or a level
 * reorder (reorder_now) so the state reads as the reference's would. */
int cog_apply_pending(const cog_geom *geom, const cog_params *prm,
                      const cog_state *st, int32_t reorder_now, void *stream);

/* Plain per-pixel mixture over all planes of one frame (baseline model):
 * state uses st->mix/meta (count only); mask u8[P] 0/255. */
int cog_baseline_frame(const cog_geom *geom, const cog_params *prm,
                       const cog_state *st, const uint8_t *frame,
                       uint8_t *mask, void *stream);

/* Reference-layout views of one stream's state (device buffers):
 * mu/var/w f64[d][P][K]; count i64[d][P]; mid i8[d][P][3]; ref i8[d][P][2];
 * chp u8[d][P]; label u8[d][P]; active i8[d][P]; waking u8[d][P];
 * streak i64[d][P]; clock i64[d][P]; hits i64[d][P][5]. */
typedef struct cog_ref_state {
  double *mu, *var, *w;
  int64_t *count;
  int8_t *mid, *ref;
  uint8_t *chp, *label;
  int8_t *active;
  uint8_t *waking;
  int64_t *streak, *clock, *hits;
} cog_ref_state;

int cog_export_state(const cog_geom *geom, const cog_state *st,
                     const cog_ref_state *out, void *stream);
int cog_import_state(const cog_geom *geom, const cog_state *st,
                     const cog_ref_state *in, void *stream);

/* One host frame end to end, for the host-facing API (one call per frame
 * instead of a dozen runtime calls from Python): H2D of `host_frame`
 * (pinned, d*P bytes) into `dev_frame` on `copy_stream`, recorded in
 * `up_event`; `stream` waits for it and runs the step (fused finalize);
 * mask (P bytes) and stats (16 x i64) are copied back into the pinned
 * `host_mask` / `host_stats` on `down_stream` (NULL: on `stream`; a stream
 * of its own keeps the next frame's step from queueing behind these
 * copies) and completion is recorded in `done_event`.
 * Replaces the per-frame body of CascadeEngine.process_frame
 * (cascade.py:261-318) for host frames.  Events come from
 * cog_event_create. */
int cog_step_host(const cog_geom *geom, const cog_params *prm,
                  const cog_state *st, const uint8_t *host_frame,
                  uint8_t *dev_frame, uint8_t *dev_mask, void *conf,
                  uint8_t *kind, int64_t *dev_stats, uint8_t *host_mask,
                  int64_t *host_stats, int64_t frame_index,
                  int32_t reorder_now, void *stream, void *copy_stream,
                  void *down_stream, void *up_event, void *done_event);

/* Pooled training statistics of big groups (grouping.py:189-192): values
 * u8[N][depth][P], member i32[P] (group 0..n_groups-1, -1 = none), all on
 * the device; ACCUMULATES into sums u64[n_groups][depth][2] the exact
 * integer sums of x and x^2 over every frame of every member pixel (zero it
 * first).  n_groups * depth <= 3072. */
int cog_pool_sums(const uint8_t *values, int32_t n_frames, int32_t depth,
                  int64_t n_pix, const int32_t *member, int32_t n_groups,
                  uint64_t *sums, void *stream);

/* k-means assignment step of the grouping (grouping.py:116-118): points
 * f64[n][2], centers f64[k][2] (device); label i64[n] is overwritten with
 * each point's nearest centre (numpy's squared distance, lowest index on
 * ties) and *changed (u32, device, zeroed by the caller) is set to 1 if any
 * label changed. */
int cog_kmeans_assign(const double *points, int64_t n, const double *centers,
                      int32_t k, int64_t *label, uint32_t *changed,
                      void *stream);

/* The grouping's axis-0 reductions (cogbg/grouping.py:100-161: the k-means
 * centre update `pts[label == j].mean(axis=0)`, standardise's mean / std,
 * the sigma-band's per-cluster mean / std / ptp).  numpy adds the rows of a
 * C-contiguous (n, dims) f64 array one after another, so these are
 * sequential binary64 sums in index order; this reproduces them bit for bit.
 * For chain (j, f), j < k, f < dims:  out[j * dims + f] = sum, over the rows
 * i with label[i] == j in index order (label NULL: every row, k = 1), of
 * x[i][f] (square = 0) or (x[i][f] - shift[j * dims + f])^2 (square = 1);
 * minmax[2 * chain], [2 * chain + 1] = min / max of x over those rows (or
 * NULL); count[j] = rows with label j (or NULL).  All device pointers. */
int cog_seq_sums(const double *x, int64_t n, int32_t dims, const int64_t *label,
                 int32_t k, const double *shift, int32_t square, double *out,
                 double *minmax, int64_t *count, void *stream);

/* One farthest-point seeding step (cogbg/grouping.py:100-112): far[i] =
 * |points[i] - centre|^2 (first != 0) or min(far[i], ...), points f64[n][2],
 * centre f64[2] on the HOST; best u64[2] on the device receives the bit
 * pattern of max(far) and np.argmax(far), the lowest index holding it. */
int cog_far_step(const double *points, int64_t n, const double *centre,
                 int32_t first, double *far, uint64_t *best, void *stream);

/* Confusion counts of predicted vs truth masks u8[n] (evaluation.
 * confusion_counts, cogbg/evaluation.py:72-89): truth 0 = background,
 * 255 = foreground, anything else excluded; predicted foreground = 255.
 * ACCUMULATES into counts u64[5] = {tp, fp, tn, fn, excluded} (zero it to
 * start a sequence), so a whole run is scored on the device and read once. */
int cog_confusion(const uint8_t *predicted, const uint8_t *truth, int64_t n,
                  uint64_t *counts, void *stream);

/* cudaEvent_t helpers (timing disabled): create returns NULL on failure;
 * sync blocks until the event completes; query returns 1 done, 0 not yet,
 * negative on error. */
void *cog_event_create(void);
int cog_event_destroy(void *event);
int cog_event_sync(void *event);
int cog_event_query(void *event);

/* Version / build string (host pointer, static). */
const char *cog_version(void);

#ifdef __cplusplus
}
#endif

#endif /* COG_B200_H */
