// cog_device.cuh -- device-side building blocks of the CoG hot path (sm_100a).
//
// Arithmetic contract: every decision and update is evaluated in IEEE
// binary64 in the reference's operation order, with FMA contraction off
// (the whole extension is built with -fmad=false; CUDA's double '/' and
// sqrt are correctly rounded).  From identical state this reproduces the
// reference's kernels bit for bit:
//   mixture update + sort   kernels_numba.py:30-134
//   cascade descent          kernels_numba.py:188-359
// State may be *stored* as float32 (promoted on load, rounded on store).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace cog {

enum Level : int {
  L_CHP = 0, L_GROUP = 1, L_MEAN = 2, L_MEANVAR = 3, L_GMM = 4,
  K_SKIP = 5, K_COPY = 6
};

constexpr int MAXD = 4;                 // planes per frame handled per thread
constexpr uint16_t UNGROUPED = 0xFFFF;  // group id of ungrouped pixels

// ----------------------------------------------------------------------------
// Packed per-plane-pixel words.
//
// meta (u16): count[0:4] | mid0[4:6] | mid1[6:8] | mid2[8:10] | ref0[10:13] |
//             ref1[13:16]; a mid code is the level (1..3) or 0 for "-1".
// dyn  (u32): chp_prev[0:8] | last_label[8] | waking[9] |
//             last_active+1 [10:13] | clock[16:32]
// ----------------------------------------------------------------------------
__device__ __forceinline__ int meta_count(uint32_t m) { return m & 15u; }
__device__ __forceinline__ int meta_mid(uint32_t m, int j) {
  int c = (m >> (4 + 2 * j)) & 3u;
  return c ? c : -1;
}
__device__ __forceinline__ int meta_ref(uint32_t m, int j) {
  return (m >> (10 + 3 * j)) & 7u;
}
__host__ __device__ __forceinline__ uint32_t enc_mid(int code) {
  return code < 0 ? 0u : (uint32_t)code & 3u;
}
__device__ __forceinline__ uint32_t pack_meta(int count, int m0, int m1, int m2,
                                              int r0, int r1) {
  return (uint32_t)count | (enc_mid(m0) << 4) | (enc_mid(m1) << 6) |
         (enc_mid(m2) << 8) | ((uint32_t)r0 << 10) | ((uint32_t)r1 << 13);
}
__device__ __forceinline__ uint32_t meta_with_count(uint32_t m, int n) {
  return (m & ~15u) | (uint32_t)n;
}
__device__ __forceinline__ uint32_t meta_with_refs(uint32_t m, int r0, int r1) {
  return (m & 0x03FFu) | ((uint32_t)r0 << 10) | ((uint32_t)r1 << 13);
}
__device__ __forceinline__ uint32_t meta_with_mids(uint32_t m, int m0, int m1,
                                                   int m2) {
  return (m & ~0x3F0u) | (enc_mid(m0) << 4) | (enc_mid(m1) << 6) |
         (enc_mid(m2) << 8);
}

__device__ __forceinline__ int dyn_chp(uint32_t d) { return d & 0xFFu; }
__device__ __forceinline__ int dyn_label(uint32_t d) { return (d >> 8) & 1u; }
__device__ __forceinline__ int dyn_waking(uint32_t d) { return (d >> 9) & 1u; }
__device__ __forceinline__ int dyn_active(uint32_t d) {
  return (int)((d >> 10) & 7u) - 1;
}
__device__ __forceinline__ int dyn_clock(uint32_t d) { return d >> 16; }
__device__ __forceinline__ uint32_t pack_dyn(int chp, int label, int waking,
                                             int active, int clock) {
  return (uint32_t)chp | ((uint32_t)label << 8) | ((uint32_t)waking << 9) |
         ((uint32_t)(active + 1) << 10) | ((uint32_t)clock << 16);
}

// ----------------------------------------------------------------------------
// Mixture record of one plane-pixel in HBM (cog_b200.h): KB = the K bucket
// of the kernel instantiation (k_max <= KB), R elements of the state type:
// (mu_k, var_k) at [2k, 2k+1], w_k at [2*KB + k], the rest padding.  One
// record is 64 B (KB <= 5) or 128 B of float32: a pixel's whole mixture is
// one aligned DRAM burst, and (mu, var) of one mode one 8-byte load.
// ----------------------------------------------------------------------------
__host__ __device__ constexpr int kbucket(int K) {
  return K <= 3 ? 3 : (K <= 5 ? 5 : 8);
}
__host__ __device__ constexpr int rec_elems(int KB) { return KB <= 5 ? 16 : 32; }
__host__ __device__ constexpr int rec_w(int KB) { return 2 * KB; }

// ----------------------------------------------------------------------------
// Register-resident mixture of one plane-pixel, binary64.
// ----------------------------------------------------------------------------
template <int KMAX>
struct Mix {
  double mu[KMAX], var[KMAX], w[KMAX];
};

// Stable descending order by w/sqrt(var) over the n live modes
// (kernels_numba.py:30-73).  The stable insertion sort's final slot of mode
// i is #{j: key_j > key_i} + #{j < i: key_j == key_i}; computing it as a
// rank keeps everything in registers.  inv[old] = new slot.
template <int KMAX>
__device__ __forceinline__ void sort_modes(Mix<KMAX>& m, int n,
                                           int (&inv)[KMAX]) {
  double key[KMAX];
#pragma unroll
  for (int k = 0; k < KMAX; ++k) {
    key[k] = 0.0;
    if (k < n) key[k] = m.w[k] / sqrt(m.var[k]);
  }
  bool moved = false;
#pragma unroll
  for (int i = 0; i < KMAX; ++i) {
    int r = i;
    if (i < n) {
      r = 0;
#pragma unroll
      for (int j = 0; j < KMAX; ++j)
        if (j < n) r += (key[j] > key[i]) || (j < i && key[j] == key[i]);
    }
    inv[i] = r;
    moved |= (r != i);
  }
  if (moved) {
    Mix<KMAX> o = m;
#pragma unroll
    for (int i = 0; i < KMAX; ++i) {
#pragma unroll
      for (int t = 0; t < KMAX; ++t) {
        if (i < n && inv[i] == t) {
          m.mu[t] = o.mu[i];
          m.var[t] = o.var[i];
          m.w[t] = o.w[i];
        }
      }
    }
  }
}

struct GmmPar {
  double lam, t_bg, var_floor, init_var;
};

// Full mixture update (kernels_numba.py:76-134).  n is the live count (in/
// out), kcap the configured k_max.  Returns 0 background / 1 foreground.
template <int KMAX>
__device__ __forceinline__ int gmm_step(Mix<KMAX>& m, int& n, int kcap,
                                        double v, double alpha,
                                        const GmmPar& g, int (&inv)[KMAX]) {
  int hit = -1;
#pragma unroll
  for (int k = 0; k < KMAX; ++k) {
    if (hit < 0 && k < n) {
      if (fabs(v - m.mu[k]) <= g.lam * sqrt(m.var[k])) hit = k;
    }
  }
  int label;
  if (hit >= 0) {
#pragma unroll
    for (int k = 0; k < KMAX; ++k)
      if (k < n) m.w[k] = (1.0 - alpha) * m.w[k];
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < KMAX; ++k) {
      if (k == hit) m.w[k] = m.w[k] + alpha;
    }
#pragma unroll
    for (int k = 0; k < KMAX; ++k)
      if (k < n) s = s + m.w[k];
#pragma unroll
    for (int k = 0; k < KMAX; ++k)
      if (k < n) m.w[k] = m.w[k] / s;
#pragma unroll
    for (int k = 0; k < KMAX; ++k) {
      if (k == hit) {
        double mm = (1.0 - alpha) * m.mu[k] + alpha * v;
        m.mu[k] = mm;
        double dd = v - mm;
        double s2 = (1.0 - alpha) * m.var[k] + alpha * (dd * dd);
        if (s2 < g.var_floor) s2 = g.var_floor;
        m.var[k] = s2;
      }
    }
    double acc = 0.0;
    int b = n;
    bool found = false;
#pragma unroll
    for (int k = 0; k < KMAX; ++k) {
      if (!found && k < n) {
        acc = acc + m.w[k];
        if (acc > g.t_bg) {
          b = k + 1;
          found = true;
        }
      }
    }
    label = (hit + 1 <= b) ? 0 : 1;
  } else {
    int slot;
    if (n < kcap) {
      slot = n;
      n = n + 1;
    } else {
      slot = n - 1;
    }
#pragma unroll
    for (int k = 0; k < KMAX; ++k) {
      if (k == slot) {
        m.mu[k] = v;
        m.var[k] = g.init_var;
        m.w[k] = alpha;
      }
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < KMAX; ++k)
      if (k < n) s = s + m.w[k];
    if (s == 0.0) {
#pragma unroll
      for (int k = 0; k < KMAX; ++k)
        if (k < n) m.w[k] = (k == slot) ? 1.0 : 0.0;
    } else {
#pragma unroll
      for (int k = 0; k < KMAX; ++k)
        if (k < n) m.w[k] = m.w[k] / s;
    }
    label = 1;
  }
  sort_modes<KMAX>(m, n, inv);
  return label;
}

template <int KMAX>
__device__ __forceinline__ int select_inv(const int (&inv)[KMAX], int r) {
  int out = r;
#pragma unroll
  for (int k = 0; k < KMAX; ++k)
    if (k == r) out = inv[k];
  return out;
}

// ----------------------------------------------------------------------------
// Typed state access (float32 or float64 storage, binary64 arithmetic).
// ----------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ double ld(const T* p) {
  return (double)__ldg(p);
}
template <typename T>
__device__ __forceinline__ double ldrw(const T* p) {
  return (double)*p;
}
__device__ __forceinline__ void st(float* p, double v) { *p = (float)v; }
__device__ __forceinline__ void st(double* p, double v) { *p = v; }

// whole record <-> registers with 16-byte vector accesses (R is a multiple
// of 4 floats / 2 doubles; records are 64-B aligned)
template <int R>
__device__ __forceinline__ void rec_load(const float* rec, float (&e)[R]) {
#pragma unroll
  for (int i = 0; i < R / 4; ++i) {
    const float4 v = reinterpret_cast<const float4*>(rec)[i];
    e[4 * i] = v.x;
    e[4 * i + 1] = v.y;
    e[4 * i + 2] = v.z;
    e[4 * i + 3] = v.w;
  }
}
template <int R>
__device__ __forceinline__ void rec_load(const double* rec, double (&e)[R]) {
#pragma unroll
  for (int i = 0; i < R / 2; ++i) {
    const double2 v = reinterpret_cast<const double2*>(rec)[i];
    e[2 * i] = v.x;
    e[2 * i + 1] = v.y;
  }
}
template <int R>
__device__ __forceinline__ void rec_store(float* rec, const float (&e)[R]) {
#pragma unroll
  for (int i = 0; i < R / 4; ++i)
    reinterpret_cast<float4*>(rec)[i] =
        make_float4(e[4 * i], e[4 * i + 1], e[4 * i + 2], e[4 * i + 3]);
}
template <int R>
__device__ __forceinline__ void rec_store(double* rec, const double (&e)[R]) {
#pragma unroll
  for (int i = 0; i < R / 2; ++i)
    reinterpret_cast<double2*>(rec)[i] = make_double2(e[2 * i], e[2 * i + 1]);
}

// record elements <-> binary64 mixture (live modes only; dead slots and
// padding keep their stored values)
template <int KMAX, typename T>
__device__ __forceinline__ void rec_to_mix(const T (&e)[rec_elems(KMAX)],
                                           int n, Mix<KMAX>& x) {
#pragma unroll
  for (int k = 0; k < KMAX; ++k) {
    x.mu[k] = 0.0;
    x.var[k] = 1.0;
    x.w[k] = 0.0;
    if (k < n) {
      x.mu[k] = (double)e[2 * k];
      x.var[k] = (double)e[2 * k + 1];
      x.w[k] = (double)e[rec_w(KMAX) + k];
    }
  }
}
template <int KMAX, typename T>
__device__ __forceinline__ void mix_to_rec(const Mix<KMAX>& x, int n,
                                           T (&e)[rec_elems(KMAX)]) {
#pragma unroll
  for (int k = 0; k < KMAX; ++k) {
    if (k < n) {
      e[2 * k] = (T)x.mu[k];
      e[2 * k + 1] = (T)x.var[k];
      e[rec_w(KMAX) + k] = (T)x.w[k];
    }
  }
}

// warp-wide sums of unsigned values (REDUX on sm_80+)
__device__ __forceinline__ unsigned warp_sum_u32(unsigned v) {
  return __reduce_add_sync(0xffffffffu, v);
}

}  // namespace cog
