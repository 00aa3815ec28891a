/*
 * cog_oracle.c -- CPU ORACLE (test infrastructure only, never the product).
 *
 * Plain-C restatement of the reference's per-pixel kernels, used by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * as the checker and the CPU baseline.  Only those three may load it.
 *
 * Follows, operation for operation and in the same IEEE-754 binary64 order
 * (built with -O2 -ffp-contract=off, no -ffast-math, like numba without
 * fastmath):
 *   _sort_modes      /root/reference/pkg/src/cogbg/kernels_numba.py:30-73
 *   _gmm_step        /root/reference/pkg/src/cogbg/kernels_numba.py:76-134
 *   baseline_frame   /root/reference/pkg/src/cogbg/kernels_numba.py:137-149
 *   cascade_frame    /root/reference/pkg/src/cogbg/kernels_numba.py:152-360
 *   resolve_copies   /root/reference/pkg/src/cogbg/kernels_numba.py:363-373
 *
 * Parity pin: tests/test_oracle.py checks this file against golden vectors
 * produced by the real reference (tests/golden/make_golden.py).
 *
 * The only liberty taken is an optional OpenMP split of the pixel loop
 * (pixels are independent within one plane pass; the 7 level counters are
 * integer sums, so the result does not depend on the thread count).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

enum { L_CHP = 0, L_GROUP = 1, L_MEAN = 2, L_MEANVAR = 3, L_GMM = 4,
       K_SKIP = 5, K_COPY = 6 };

#define KCAP 64

/* stable insertion sort of one pixel's live modes by w/sqrt(var), desc;
 * inv[old] = new slot (identity for dead slots). */
static void sort_pixel(double *mu, double *var, double *w, int64_t n, int kmax,
                       int64_t *inv)
{
    double key[KCAP], tmp[KCAP];
    int64_t perm[KCAP];
    for (int64_t k = 0; k < n; k++) {
        key[k] = w[k] / sqrt(var[k]);
        perm[k] = k;
    }
    for (int64_t i = 1; i < n; i++) {
        double ki = key[i];
        int64_t pi = perm[i];
        int64_t j = i - 1;
        while (j >= 0 && key[j] < ki) {
            key[j + 1] = key[j];
            perm[j + 1] = perm[j];
            j--;
        }
        key[j + 1] = ki;
        perm[j + 1] = pi;
    }
    int moved = 0;
    for (int64_t j = 0; j < n; j++)
        if (perm[j] != j) { moved = 1; break; }
    if (moved) {
        for (int64_t j = 0; j < n; j++) inv[perm[j]] = j;
        for (int64_t j = 0; j < n; j++) tmp[j] = mu[perm[j]];
        for (int64_t j = 0; j < n; j++) mu[j] = tmp[j];
        for (int64_t j = 0; j < n; j++) tmp[j] = var[perm[j]];
        for (int64_t j = 0; j < n; j++) var[j] = tmp[j];
        for (int64_t j = 0; j < n; j++) tmp[j] = w[perm[j]];
        for (int64_t j = 0; j < n; j++) w[j] = tmp[j];
    } else {
        for (int64_t j = 0; j < n; j++) inv[j] = j;
    }
    for (int64_t j = n; j < kmax; j++) inv[j] = j;
}

/* full Stauffer-Grimson update of one pixel; returns 0 bg / 1 fg */
static int gmm_pixel(double *mu, double *var, double *w, int64_t *count,
                     int kmax, double v, double alpha, double lam, double t_bg,
                     double var_floor, double init_var, int64_t *inv)
{
    int64_t n = *count;
    int64_t hit = -1;
    for (int64_t k = 0; k < n; k++) {
        if (fabs(v - mu[k]) <= lam * sqrt(var[k])) { hit = k; break; }
    }
    int label;
    if (hit >= 0) {
        for (int64_t k = 0; k < n; k++) w[k] = (1.0 - alpha) * w[k];
        w[hit] = w[hit] + alpha;
        double s = 0.0;
        for (int64_t k = 0; k < n; k++) s = s + w[k];
        for (int64_t k = 0; k < n; k++) w[k] = w[k] / s;
        double m = (1.0 - alpha) * mu[hit] + alpha * v;
        mu[hit] = m;
        double dd = v - m;
        double s2 = (1.0 - alpha) * var[hit] + alpha * (dd * dd);
        if (s2 < var_floor) s2 = var_floor;
        var[hit] = s2;
        double acc = 0.0;
        int64_t b = n;
        for (int64_t k = 0; k < n; k++) {
            acc = acc + w[k];
            if (acc > t_bg) { b = k + 1; break; }
        }
        label = (hit + 1 <= b) ? 0 : 1;
    } else {
        int64_t slot;
        if (n < kmax) { slot = n; n = n + 1; *count = n; }
        else slot = n - 1;
        mu[slot] = v;
        var[slot] = init_var;
        w[slot] = alpha;
        double s = 0.0;
        for (int64_t k = 0; k < n; k++) s = s + w[k];
        if (s == 0.0) {
            for (int64_t k = 0; k < n; k++) w[k] = 0.0;
            w[slot] = 1.0;
        } else {
            for (int64_t k = 0; k < n; k++) w[k] = w[k] / s;
        }
        label = 1;
    }
    sort_pixel(mu, var, w, *count, kmax, inv);
    return label;
}

static int oracle_threads(int threads)
{
#ifdef _OPENMP
    if (threads <= 0) threads = omp_get_max_threads();
    return threads;
#else
    (void)threads;
    return 1;
#endif
}

/* kernels_numba.baseline_frame: one plane of P pixels, state (P,K) f64 */
int cogo_baseline_frame(int64_t P, int K, const uint8_t *vals, double *mu,
                        double *var, double *w, int64_t *count, double alpha,
                        double lam, double t_bg, double var_floor,
                        double init_var, uint8_t *out_label, int threads)
{
    if (K < 1 || K > KCAP) return -1;
    int nt = oracle_threads(threads);
    (void)nt;
#pragma omp parallel for schedule(static) num_threads(nt) if (nt > 1)
    for (int64_t p = 0; p < P; p++) {
        int64_t inv[KCAP];
        out_label[p] = (uint8_t)gmm_pixel(mu + p * K, var + p * K, w + p * K,
                                          count + p, K, (double)vals[p], alpha,
                                          lam, t_bg, var_floor, init_var, inv);
    }
    return 0;
}

/* kernels_numba.cascade_frame: one cascade pass over one plane */
int cogo_cascade_frame(
    int64_t P, int K,
    const uint8_t *vals, double *mu, double *var, double *w, int64_t *count,
    uint8_t *chp_prev, uint8_t *last_label, int8_t *mid_order,
    int8_t *mode_ref, int64_t *hits, int64_t *streak, int8_t *last_active,
    int64_t *clock, uint8_t *waking, const uint8_t *on_lattice,
    const int64_t *group_id, const double *g_mu, const double *g_var,
    const float *table, const double *peak, const double *wa,
    const double *wb, const double *wc,
    double base_rate, double lam, double t_bg, double var_floor,
    double init_var, double eps_chp, double conf_thresh, double prior_floor,
    double rate_floor, int64_t saturation_frames, int64_t sleep_frames,
    int sampling_on, int grouping_on, int rate_scaling_on, int chp_on,
    int literal_conf, int compat,
    uint8_t *out_label, uint8_t *out_kind, double *out_conf,
    int64_t *out_counts, int threads)
{
    if (K < 1 || K > KCAP) return -1;
    int64_t c0 = 0, c1 = 0, c2 = 0, c3 = 0, c4 = 0, c5 = 0, c6 = 0;
    int nt = oracle_threads(threads);
    (void)nt;
#pragma omp parallel for schedule(static) num_threads(nt) if (nt > 1) \
    reduction(+ : c0, c1, c2, c3, c4, c5, c6)
    for (int64_t p = 0; p < P; p++) {
        int64_t inv[KCAP];
        double *pmu = mu + p * K, *pvar = var + p * K, *pw = w + p * K;
        int8_t *mid = mid_order + p * 3, *ref = mode_ref + p * 2;
        int64_t *ph = hits + p * 5;
        double v = (double)vals[p];
        double prev = (double)chp_prev[p];
        int changed = fabs(v - prev) > eps_chp;

        if (sampling_on && clock[p] > 0) {
            if (!changed) {
                clock[p] -= 1;
                if (clock[p] == 0) waking[p] = 1;
                chp_prev[p] = vals[p];
                out_label[p] = last_label[p];
                out_kind[p] = K_SKIP;
                out_conf[p] = 0.0;
                c5++;
                continue;
            }
            clock[p] = 0;
            waking[p] = 0;
            streak[p] = 0;
        } else if (sampling_on && waking[p] == 1) {
            waking[p] = 0;
            if (!changed && on_lattice[p] == 0) {
                chp_prev[p] = vals[p];
                clock[p] = sleep_frames;
                out_label[p] = last_label[p];
                out_kind[p] = K_COPY;
                out_conf[p] = 0.0;
                c6++;
                continue;
            }
        }

        if (compat) {
            int active = L_GMM;
            if (count[p] > 0 && fabs(v - pmu[0]) <= lam * sqrt(pvar[0]))
                active = L_MEAN;
            int label = gmm_pixel(pmu, pvar, pw, count + p, K, v, base_rate,
                                  lam, t_bg, var_floor, init_var, inv);
            out_label[p] = (uint8_t)label;
            out_kind[p] = (uint8_t)active;
            out_conf[p] = 0.0;
            if (active == L_MEAN) c2++; else c4++;
            ph[active] += 1;
            last_active[p] = (int8_t)active;
            last_label[p] = (uint8_t)label;
            chp_prev[p] = vals[p];
            continue;
        }

        /* confidence from pre-update state */
        int top = mid[0];
        if (top == L_GROUP && !grouping_on) top = mid[1];
        double mu_top, sig_top;
        if (top == L_GROUP) {
            mu_top = g_mu[group_id[p]];
            sig_top = sqrt(g_var[group_id[p]]);
        } else if (top == L_MEANVAR) {
            mu_top = pmu[ref[1]];
            sig_top = sqrt(pvar[ref[1]]);
        } else {
            mu_top = pmu[ref[0]];
            sig_top = sqrt(pvar[ref[0]]);
        }
        /* the engine keeps the f32 table and promotes at use
           (cascade.py:192, 213-216: _tables64 = float64(f32 table)) */
        double phat = (double)table[p * 256 + vals[p]] / peak[p];
        double bterm = fabs(v - prev) / 255.0;
        if (!literal_conf) bterm = 1.0 - bterm;
        double gterm = fabs(v - mu_top) / (lam * sig_top);
        if (gterm > 1.0) gterm = 1.0;
        if (!literal_conf) gterm = 1.0 - gterm;
        double conf;
        if (phat < prior_floor) {
            double denom = wb[p] + wc[p];
            conf = denom > 0.0 ? (wb[p] * bterm + wc[p] * gterm) / denom : 0.0;
        } else {
            conf = wa[p] * phat + wb[p] * bterm + wc[p] * gterm;
        }
        double rho;
        if (rate_scaling_on) {
            double relax = 1.0 - conf;
            if (relax < rate_floor) relax = rate_floor;
            rho = base_rate * relax;
        } else {
            rho = base_rate;
        }

        int active = -1;
        int label = 0;
        if (chp_on && !changed) {
            active = L_CHP;
            label = last_label[p];
        } else {
            for (int j = 0; j < 3; j++) {
                int code = mid[j];
                if (code < 0) break;
                if (code == L_GROUP) {
                    if (!grouping_on) continue;
                    int64_t g = group_id[p];
                    if (fabs(v - g_mu[g]) <= lam * sqrt(g_var[g])) {
                        active = L_GROUP;
                        label = 0;
                        break;
                    }
                } else if (code == L_MEAN) {
                    int r = ref[0];
                    if (fabs(v - pmu[r]) <= lam * sqrt(pvar[r])) {
                        double acc = 0.0;
                        for (int k = 0; k < r; k++) acc = acc + pw[k];
                        if (acc <= t_bg) {
                            active = L_MEAN;
                            label = 0;
                            pmu[r] = (1.0 - rho) * pmu[r] + rho * v;
                            break;
                        }
                    }
                } else {
                    int r = ref[1];
                    if (fabs(v - pmu[r]) <= lam * sqrt(pvar[r])) {
                        double acc = 0.0;
                        for (int k = 0; k < r; k++) acc = acc + pw[k];
                        if (acc <= t_bg) {
                            active = L_MEANVAR;
                            label = 0;
                            double m = (1.0 - rho) * pmu[r] + rho * v;
                            pmu[r] = m;
                            double dd = v - m;
                            double s2 = (1.0 - rho) * pvar[r] + rho * (dd * dd);
                            if (s2 < var_floor) s2 = var_floor;
                            pvar[r] = s2;
                            sort_pixel(pmu, pvar, pw, count[p], K, inv);
                            ref[0] = (int8_t)inv[ref[0]];
                            ref[1] = (int8_t)inv[ref[1]];
                            break;
                        }
                    }
                }
            }
            if (active < 0) {
                active = L_GMM;
                label = gmm_pixel(pmu, pvar, pw, count + p, K, v, rho, lam,
                                  t_bg, var_floor, init_var, inv);
                ref[0] = (int8_t)inv[ref[0]];
                ref[1] = (int8_t)inv[ref[1]];
            }
        }

        if (conf > conf_thresh) streak[p] += 1;
        else streak[p] = 0;
        ph[active] += 1;
        last_active[p] = (int8_t)active;
        last_label[p] = (uint8_t)label;
        chp_prev[p] = vals[p];
        out_label[p] = (uint8_t)label;
        out_kind[p] = (uint8_t)active;
        out_conf[p] = conf;
        switch (active) {
        case 0: c0++; break;
        case 1: c1++; break;
        case 2: c2++; break;
        case 3: c3++; break;
        default: c4++; break;
        }
        if (sampling_on && streak[p] >= saturation_frames)
            clock[p] = sleep_frames;
    }
    out_counts[0] = c0; out_counts[1] = c1; out_counts[2] = c2;
    out_counts[3] = c3; out_counts[4] = c4; out_counts[5] = c5;
    out_counts[6] = c6;
    return 0;
}

/* kernels_numba.resolve_copies */
int cogo_resolve_copies(int64_t P, const uint8_t *out_kind, uint8_t *out_label,
                        uint8_t *last_label, int64_t width, int64_t stride)
{
    for (int64_t p = 0; p < P; p++) {
        if (out_kind[p] == K_COPY) {
            int64_t y = p / width, x = p % width;
            int64_t q = (y - y % stride) * width + (x - x % stride);
            uint8_t lbl = out_label[q];
            out_label[p] = lbl;
            last_label[p] = lbl;
        }
    }
    return 0;
}

/* Stable re-sort of the given pixels' live modes by w/sqrt(var)
 * (kernels_numpy.sort_subset, /root/reference/pkg/src/cogbg/kernels_numpy.py:24-38);
 * writes inv (P_sel, K). */
int cogo_sort_pixels(int64_t n_sel, const int64_t *idx, int K, double *mu,
                     double *var, double *w, const int64_t *count,
                     int64_t *inv_out)
{
    if (K < 1 || K > KCAP) return -1;
    for (int64_t i = 0; i < n_sel; i++) {
        int64_t p = idx[i];
        sort_pixel(mu + p * K, var + p * K, w + p * K, count[p], K,
                   inv_out + i * K);
    }
    return 0;
}

/* ---------------------------------------------------------------------
 * Helpers that let the oracle run BASELINE configs at full geometry (C3:
 * 2 Mpx, C4: 8 Mpx) in host memory and time; each restates one numpy
 * expression of the reference.
 * ------------------------------------------------------------------- */

/* f32 KDE tables of one plane (scene_prior.build_kde :104-111, then the
 * engine's astype(float32), cascade.py:192): counts = histogram of the N
 * values of each pixel, table[g] = (sum_s counts[s] * kern[s][g]) / N.
 * values u8[N][P] (one plane, frame-major), out f32[P][256].  The dot
 * products run over the nonzero bins in ascending order (zero bins add
 * +0.0); BLAS may sum the 256 products in another order, which moves the
 * binary64 result by at most an ulp and, after rounding to float32,
 * leaves the table identical (pinned on the reference's goldens,
 * tests/test_oracle.py). */
int cogo_kde_tables32(int64_t P, int N, const uint8_t *values,
                      const double *kern, float *out, int threads)
{
    int nt = oracle_threads(threads);
    (void)nt;
    const int64_t B = 64;
    int64_t nb = (P + B - 1) / B;
#pragma omp parallel for schedule(dynamic, 16) num_threads(nt) if (nt > 1)
    for (int64_t b = 0; b < nb; b++) {
        int64_t p0 = b * B, p1 = p0 + B < P ? p0 + B : P;
        uint16_t hist[64][256];
        memset(hist, 0, sizeof(hist));
        for (int i = 0; i < N; i++) {
            const uint8_t *row = values + (int64_t)i * P;
            for (int64_t p = p0; p < p1; p++) hist[p - p0][row[p]]++;
        }
        for (int64_t p = p0; p < p1; p++) {
            const uint16_t *h = hist[p - p0];
            int s_idx[256], ns = 0;
            for (int s = 0; s < 256; s++)
                if (h[s]) s_idx[ns++] = s;
            float *o = out + p * 256;
            for (int g = 0; g < 256; g++) {
                double acc = 0.0;
                for (int j = 0; j < ns; j++) {
                    int s = s_idx[j];
                    acc = acc + (double)h[s] * kern[s * 256 + g];
                }
                o[g] = (float)(acc / (double)N);
            }
        }
    }
    return 0;
}

/* k-means assignment step (grouping.py:116-118):
 * dist = ((f[:, None, :] - c[None]) ** 2).sum(axis=2); argmin(axis=1)
 * (first minimum on ties).  f f64[n][2], c f64[k][2]; writes label i64[n];
 * returns 1 if any label changed. */
int cogo_kmeans_assign(int64_t n, const double *f, int k, const double *c,
                       int64_t *label, int threads)
{
    int nt = oracle_threads(threads);
    (void)nt;
    int changed = 0;
#pragma omp parallel for schedule(static) num_threads(nt) if (nt > 1) \
    reduction(| : changed)
    for (int64_t i = 0; i < n; i++) {
        double best = 0.0;
        int64_t arg = 0;
        for (int j = 0; j < k; j++) {
            double d0 = f[2 * i] - c[2 * j], d1 = f[2 * i + 1] - c[2 * j + 1];
            double dd = d0 * d0 + d1 * d1;
            if (j == 0 || dd < best || (isnan(dd) && !isnan(best))) {
                best = dd;
                arg = j;
            }
        }
        if (label[i] != arg) changed = 1;
        label[i] = arg;
    }
    return changed;
}

/* Group sums of one plane for _update_groups (cascade.py:320-344): over the
 * pixels with kind == GROUP, in pixel order like np.bincount: cnt[g],
 * vsum[g] (sum of v as f64) and csum[g] (sum of conf, sequential). */
int cogo_group_sums(int64_t P, const uint8_t *kind, const uint8_t *vals,
                    const double *conf, const int64_t *group_id, int64_t G,
                    int64_t *cnt, double *vsum, double *csum)
{
    for (int64_t g = 0; g < G; g++) {
        cnt[g] = 0;
        vsum[g] = 0.0;
        csum[g] = 0.0;
    }
    for (int64_t p = 0; p < P; p++) {
        if (kind[p] != L_GROUP) continue;
        int64_t g = group_id[p];
        cnt[g] += 1;
        vsum[g] = vsum[g] + (double)vals[p];
        csum[g] = csum[g] + conf[p];
    }
    return 0;
}
