// prost_phases.cuh — the phase kernels of one tracker frame (see
// prost_kernels.cuh for the overall structure).  Templated on the element type
// T (float: the product path; double: the parity instantiation), the compiled
// subspace bound K (runtime k <= K) and the coordinates-per-thread VEC.
#pragma once

#include "prost_kernels.cuh"

namespace prost {

template <typename T, int VEC>
__device__ __forceinline__ void load_weights(const Args& a, const uint8_t* lab, int pix,
                                             T (&w)[VEC]) {
  uint8_t l[VEC];
  ld_lab<VEC>(lab + pix, l);
#pragma unroll
  for (int e = 0; e < VEC; ++e)
    w[e] = (pix + e < a.P) ? (l[e] ? (T)a.omega : (T)1) : (T)0;
}

__device__ __forceinline__ float norm_div(float x, float s) { return __fdiv_rn(x, s); }
__device__ __forceinline__ double norm_div(double x, double s) { return __ddiv_rn(x, s); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }

// Normalized frame coordinates (pipeline.py:148-156; mean update 120-132).
// `upd`: this frame folds into the running mean (frames_seen = `seen`);
// `wr`: write the updated mean back.
template <typename T, int VEC>
__device__ __forceinline__ void normalized(const Args& a, size_t off, bool upd, bool wr, T seen,
                                           T stdv, T (&xh)[VEC], bool& bad) {
  T xv[VEC];
  if (a.xu8) {  // 8-bit frames (TMEM path; the periodic-QR relabel reads them too)
    const uint8_t* X8 = static_cast<const uint8_t*>(a.x) + off;
#pragma unroll
    for (int e = 0; e < VEC; ++e) xv[e] = (T)((double)X8[e] * (1.0 / 255.0));
  } else {
    VecIO<T, VEC>::ldg(static_cast<const T*>(a.x) + off, xv);
  }
#pragma unroll
  for (int e = 0; e < VEC; ++e) bad |= !isfinite(xv[e]);
  if (!a.pipeline) {
#pragma unroll
    for (int e = 0; e < VEC; ++e) xh[e] = xv[e];
    return;
  }
  T* M = static_cast<T*>(a.mean) + off;
  T mv[VEC];
  VecIO<T, VEC>::ld(M, mv);
  if (upd) {
#pragma unroll
    for (int e = 0; e < VEC; ++e) mv[e] = add_rn(mv[e], norm_div(sub_rn(xv[e], mv[e]), seen));
    if (wr) VecIO<T, VEC>::st(M, mv);
  }
#pragma unroll
  for (int e = 0; e < VEC; ++e) xh[e] = norm_div(sub_rn(xv[e], mv[e]), stdv);
}

__device__ __forceinline__ double running_std(const Ctl* c) {
  // pipeline.py:134-140
  if (c->pcount < 2) return STD_FLOOR;
  const double cnt = (double)c->pcount;
  const double var = (c->psumsq - c->psum * c->psum / cnt) / (cnt - 1.0);
  return fmax(sqrt(fmax(var, 0.0)), STD_FLOOR);
}

// Scalar tails of the phases with a reduction (shared by the phase kernels and
// k_xlogic, which runs them after the cross-rank sum in exchange mode).

// red: [0] sum x, [1] sum x^2, [2] non-finite count (thread 0)
__device__ __forceinline__ void tail_stats(Ctl* c, const Args& a, int s, const double* red) {
  if (red[2] > 0.0) {
    c->status = ST_NONFINITE;
    c->t = step_size(a, c->frame_index);
    write_info(c, a, s);
  } else {
    c->psum += red[0];
    c->psumsq += red[1];
    c->pcount += a.n_real;
    c->pseen += 1;
    c->std_cur = running_std(c);
    c->update_stats = 1;
    c->status = ST_OK;
  }
}

// red: [0..K) U^T x, [K] non-finite count (warp 0)
template <int K>
__device__ __forceinline__ void tail_cold(Ctl* c, const Args& a, int s, int lane, const double* red) {
  if (red[K] > 0.0) {
    if (lane == 0) {
      c->status = ST_NONFINITE;
      c->t = step_size(a, c->frame_index);
      write_info(c, a, s);
    }
  } else if (lane < a.k) {
    c->y[lane] = red[lane];
  }
}

// red: packed upper triangle of U^T U (thread 0): Cholesky R, R^-1, reset the
// QR counter (manifold.py:192-196)
__device__ __forceinline__ void tail_gram(Ctl* c, const Args& a, int s, const double* red) {
  __shared__ double Rm[KMAX * KMAX];
  const int k = a.k;
  auto Gat = [&](int i, int j) {
    if (i > j) { const int t = i; i = j; j = t; }
    return red[i * k - i * (i - 1) / 2 + (j - i)];
  };
  for (int i = 0; i < KMAX * KMAX; ++i) Rm[i] = 0.0;
  for (int j = 0; j < k; ++j) {
    double dsum = Gat(j, j);
    for (int l = 0; l < j; ++l) dsum -= Rm[l * KMAX + j] * Rm[l * KMAX + j];
    const double rjj = sqrt(fmax(dsum, 1e-300));
    Rm[j * KMAX + j] = rjj;
    for (int i = j + 1; i < k; ++i) {
      double o = Gat(j, i);
      for (int l = 0; l < j; ++l) o -= Rm[l * KMAX + j] * Rm[l * KMAX + i];
      Rm[j * KMAX + i] = o / rjj;
    }
  }
  // R^{-1}, upper triangular, column by column
  double* Ri = a.rinv + (size_t)s * KMAX * KMAX;
  for (int i = 0; i < KMAX * KMAX; ++i) Ri[i] = 0.0;
  for (int j = 0; j < k; ++j) {
    Ri[j * KMAX + j] = 1.0 / Rm[j * KMAX + j];
    for (int i = j - 1; i >= 0; --i) {
      double o = 0.0;
      for (int l = i + 1; l <= j; ++l) o += Rm[i * KMAX + l] * Ri[l * KMAX + j];
      Ri[i * KMAX + j] = -o / Rm[i * KMAX + i];
    }
  }
  c->since_qr = 0;
}

// ---------------------------------------------------------------------------
// k_stats: frame start.  Pipeline frames inside the statistics window fold the
// raw frame's sums into the running statistics (pipeline.py:120-132) and
// reject non-finite frames; every other frame only fixes the normalization
// scale (freezing it at frame i_init, jobs.py:201-209).

template <typename T, int VEC>
__global__ void __launch_bounds__(NT) k_stats(const __grid_constant__ Args a) {
  pdl_enter();
  const int s = a.s0 + blockIdx.y;
  Ctl* c = a.ctl + s;
  if (c->p0_next == c->frame_index + 1) {  // this frame started in the previous geodesic sweep
    mark_go(a, s, 0);
    return;
  }
  const bool upd = a.pipeline && !c->frozen && c->frame_index < a.i_init;
  mark_go(a, s, upd);
  if (!upd) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      double sd = 1.0;
      if (a.pipeline) {
        sd = c->frozen ? c->pstd : running_std(c);
        if (!c->frozen) {
          c->frozen = 1;
          c->pstd = sd;
        }
      }
      c->std_cur = sd;
      c->update_stats = 0;
      c->status = ST_OK;
    }
    return;
  }
  __shared__ double sm[NW * 3];
  __shared__ double red[3];
  double s1 = 0.0, s2 = 0.0, nf = 0.0;
  const int ng = a.Pp / VEC;
  const T* X = static_cast<const T*>(a.x) + (size_t)s * a.np;
  const uint8_t* X8 = static_cast<const uint8_t*>(a.x) + (size_t)s * a.np;
  for (int q = blockIdx.x * NT + threadIdx.x; q < ng; q += a.chunks * NT) {
    const int pix = q * VEC;
    for (int ch = 0; ch < a.C; ++ch) {
      T xv[VEC];
      if (a.xu8) {  // 8-bit frames read directly (TMA-fed streamed path), frameio.py:136
#pragma unroll
        for (int e = 0; e < VEC; ++e) xv[e] = (T)((double)X8[(size_t)ch * a.Pp + pix + e] * (1.0 / 255.0));
      } else {
        VecIO<T, VEC>::ldg(X + (size_t)ch * a.Pp + pix, xv);
      }
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        if (pix + e < a.P) {
          const double v = (double)xv[e];
          s1 += v;
          s2 += v * v;
          nf += isfinite(v) ? 0.0 : 1.0;
        }
      }
    }
  }
  cta_stage(s1, sm, 0, 3);
  cta_stage(s2, sm, 1, 3);
  cta_stage(nf, sm, 2, 3);
  if (!cta_finish(a, s, sm, 3, red)) return;
  if (threadIdx.x == 0) tail_stats(c, a, s, red);
}

// ---------------------------------------------------------------------------
// k_cold: y = U^T x on a stream's first frame (fit.py:86-87, tracker.py:136).

template <typename T, int K, int VEC>
__global__ void __launch_bounds__(NT) k_cold(const __grid_constant__ Args a) {
  pdl_enter();
  const int s = a.s0 + blockIdx.y;
  Ctl* c = a.ctl + s;
  __shared__ int go, upd;
  __shared__ double sstd, sseen;
  if (threadIdx.x == 0) {
    go = c->status == ST_OK && c->frame_index == 0;
    upd = c->update_stats;
    sstd = c->std_cur;
    sseen = (double)c->pseen;
  }
  __syncthreads();
  mark_go(a, s, go);
  if (!go) return;
  __shared__ double sm[NW * (K + 1)];
  __shared__ double red[K + 1];
  T acc[K];
#pragma unroll
  for (int j = 0; j < K; ++j) acc[j] = (T)0;
  bool bad = false;
  const int ng = a.Pp / VEC;
  const T* U = static_cast<const T*>(a.U) + (size_t)s * a.k * a.np;
  for (int q = blockIdx.x * NT + threadIdx.x; q < ng; q += a.chunks * NT) {
    const int pix = q * VEC;
    for (int ch = 0; ch < a.C; ++ch) {
      const size_t off = (size_t)ch * a.Pp + pix;
      T xh[VEC];
      normalized<T, VEC>(a, (size_t)s * a.np + off, upd, false, (T)sseen, (T)sstd, xh, bad);
#pragma unroll
      for (int e = 0; e < VEC; ++e)
        if (pix + e >= a.P) xh[e] = (T)0;
#pragma unroll
      for (int j = 0; j < K; ++j) {
        if (j < a.k) {
          T u[VEC];
          VecIO<T, VEC>::ldg(U + (size_t)j * a.np + off, u);
#pragma unroll
          for (int e = 0; e < VEC; ++e) acc[j] += u[e] * xh[e];
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < K; ++j) cta_stage((double)acc[j], sm, j, K + 1);
  cta_stage(bad ? 1.0 : 0.0, sm, K, K + 1);
  if (!cta_finish(a, s, sm, K + 1, red)) return;
  if (threadIdx.x < 32) tail_cold<K>(c, a, s, threadIdx.x, red);
}

// ---------------------------------------------------------------------------
// k_pass0: r = x - U y, its cost and coordinate gradient (fit.py:96-104).

template <typename T, int K, int VEC>
__global__ void __launch_bounds__(NT, PROST_MINB) k_pass0(const __grid_constant__ Args a) {
  pdl_enter();
  const int s = a.s0 + blockIdx.y;
  Ctl* c = a.ctl + s;
  __shared__ int go, upd;
  __shared__ double sstd, sseen, sy[K];
  if (threadIdx.x == 0) {
    go = c->status == ST_OK && c->p0_next != c->frame_index + 1;
    upd = c->update_stats;
    sstd = c->std_cur;
    sseen = (double)c->pseen;
  }
  if (threadIdx.x < K) sy[threadIdx.x] = threadIdx.x < a.k ? c->y[threadIdx.x] : 0.0;
  __syncthreads();
  mark_go(a, s, go);
  if (!go) return;
  constexpr int NV = K + 3;
  __shared__ double sm[NW * NV];
  __shared__ double red[NV];
  T y[K], acc[K];
#pragma unroll
  for (int j = 0; j < K; ++j) {
    y[j] = (T)sy[j];
    acc[j] = (T)0;
  }
  double cost = 0.0;
  T gsq = (T)0;
  bool bad = false;
  const int ng = a.Pp / VEC;
  const T* U = static_cast<const T*>(a.U) + (size_t)s * a.k * a.np;
  T* R = static_cast<T*>(a.r) + (size_t)s * a.np;
  const uint8_t* L = a.lab + (size_t)s * a.Pp;
  for (int q = blockIdx.x * NT + threadIdx.x; q < ng; q += a.chunks * NT) {
    const int pix = q * VEC;
    T w[VEC];
    load_weights<T, VEC>(a, L, pix, w);
    for (int ch = 0; ch < a.C; ++ch) {
      const size_t off = (size_t)ch * a.Pp + pix;
      T xh[VEC];
      normalized<T, VEC>(a, (size_t)s * a.np + off, upd, true, (T)sseen, (T)sstd, xh, bad);
      T u[K][VEC];
      T uy[VEC];
#pragma unroll
      for (int e = 0; e < VEC; ++e) uy[e] = (T)0;
#pragma unroll
      for (int j = 0; j < K; ++j) {
        if (j < a.k) {
          VecIO<T, VEC>::ldg(U + (size_t)j * a.np + off, u[j]);
        } else {
#pragma unroll
          for (int e = 0; e < VEC; ++e) u[j][e] = (T)0;
        }
#pragma unroll
        for (int e = 0; e < VEC; ++e) uy[e] += u[j][e] * y[j];
      }
      T r[VEC];
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        r[e] = sub_rn(xh[e], uy[e]);
        T tw, g;
        penalty(r[e], w[e], a, tw, g);
        cost += (double)tw;
        gsq += g * g;
#pragma unroll
        for (int j = 0; j < K; ++j) acc[j] += u[j][e] * g;
      }
      VecIO<T, VEC>::st(R + off, r);
    }
  }
  cta_stage(cost, sm, 0, NV);
#pragma unroll
  for (int j = 0; j < K; ++j) cta_stage((double)acc[j], sm, 1 + j, NV);
  cta_stage((double)gsq, sm, K + 1, NV);
  cta_stage(bad ? 1.0 : 0.0, sm, K + 2, NV);
  if (!cta_finish(a, s, sm, NV, red)) return;
  if (threadIdx.x < 32) after_pass0<K>(c, a, s, threadIdx.x, red);
}

// ---------------------------------------------------------------------------
// k_iter: one CG iteration's U pass (fit.py:108-141).

template <typename T, int K, int VEC>
__global__ void __launch_bounds__(NT, PROST_MINB) k_iter(const __grid_constant__ Args a) {
  pdl_enter();
  const int s = a.s0 + blockIdx.y;
  Ctl* c = a.ctl + s;
  __shared__ int go, lo;
  __shared__ double sd[K], spend;
  if (threadIdx.x == 0) {
    go = c->status == ST_OK && c->active;
    lo = c->gwin_lo;
    spend = c->pend_alpha;
  }
  if (threadIdx.x < K) sd[threadIdx.x] = threadIdx.x < a.k ? c->d[threadIdx.x] : 0.0;
  __syncthreads();
  mark_go(a, s, go);
  if (!go) return;
  constexpr int NV = WC + WG * (K + 1);
  __shared__ double sm[NW * NV];
  __shared__ double red[NV];
  // large k: the direction stays in shared memory (broadcast reads) so that
  // u, the two speculative gradients and d do not exceed the register budget
  constexpr bool DSM = K > 16;
  __shared__ T sdt[K];
  T d[DSM ? 1 : K];
  if (DSM) {
    if (threadIdx.x < K) sdt[threadIdx.x] = (T)sd[threadIdx.x];
    __syncthreads();
  } else {
#pragma unroll
    for (int j = 0; j < (DSM ? 1 : K); ++j) d[j] = (T)sd[j];
  }
  T al[WC];
  {
    double v = a.step0;
#pragma unroll
    for (int m = 0; m < WC; ++m) {
      al[m] = (T)v;
      v *= a.shrink;
    }
  }
  const T pend = (T)spend;
  const int wlo = lo;
  double cost[WC];
#pragma unroll
  for (int m = 0; m < WC; ++m) cost[m] = 0.0;
  T gacc[WG][K], gsq[WG];
#pragma unroll
  for (int mm = 0; mm < WG; ++mm) {
    gsq[mm] = (T)0;
#pragma unroll
    for (int j = 0; j < K; ++j) gacc[mm][j] = (T)0;
  }
  const int ng = a.Pp / VEC;
  const T* U = static_cast<const T*>(a.U) + (size_t)s * a.k * a.np;
  T* R = static_cast<T*>(a.r) + (size_t)s * a.np;
  T* UD = static_cast<T*>(a.ud) + (size_t)s * a.np;
  const uint8_t* L = a.lab + (size_t)s * a.Pp;
  for (int q = blockIdx.x * NT + threadIdx.x; q < ng; q += a.chunks * NT) {
    const int pix = q * VEC;
    T w[VEC];
    load_weights<T, VEC>(a, L, pix, w);
    for (int ch = 0; ch < a.C; ++ch) {
      const size_t off = (size_t)ch * a.Pp + pix;
      T r[VEC], ud[VEC];
      VecIO<T, VEC>::ld(R + off, r);
      if (spend != 0.0) {
        VecIO<T, VEC>::ld(UD + off, ud);
#pragma unroll
        for (int e = 0; e < VEC; ++e) r[e] = trial(r[e], pend, ud[e]);
        VecIO<T, VEC>::st(R + off, r);
      }
      T u[K][VEC];
#pragma unroll
      for (int e = 0; e < VEC; ++e) ud[e] = (T)0;
#pragma unroll
      for (int j = 0; j < K; ++j) {
        if (j < a.k) {
          VecIO<T, VEC>::ldg(U + (size_t)j * a.np + off, u[j]);
        } else {
#pragma unroll
          for (int e = 0; e < VEC; ++e) u[j][e] = (T)0;
        }
        const T dj = DSM ? sdt[j] : d[DSM ? 0 : j];
#pragma unroll
        for (int e = 0; e < VEC; ++e) ud[e] += u[j][e] * dj;
      }
      VecIO<T, VEC>::st(UD + off, ud);
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        T gs[WG];
#pragma unroll
        for (int mm = 0; mm < WG; ++mm) gs[mm] = (T)0;
#pragma unroll
        for (int m = 0; m < WC; ++m) {
          T tw, g;
          penalty(trial(r[e], al[m], ud[e]), w[e], a, tw, g);
          cost[m] += (double)tw;
#pragma unroll
          for (int mm = 0; mm < WG; ++mm)
            if (m == wlo + mm) gs[mm] = g;
        }
#pragma unroll
        for (int mm = 0; mm < WG; ++mm) {
          gsq[mm] += gs[mm] * gs[mm];
#pragma unroll
          for (int j = 0; j < K; ++j) gacc[mm][j] += u[j][e] * gs[mm];
        }
      }
    }
  }
#pragma unroll
  for (int m = 0; m < WC; ++m) cta_stage(cost[m], sm, m, NV);
#pragma unroll
  for (int mm = 0; mm < WG; ++mm) {
#pragma unroll
    for (int j = 0; j < K; ++j) cta_stage((double)gacc[mm][j], sm, WC + mm * (K + 1) + j, NV);
    cta_stage((double)gsq[mm], sm, WC + mm * (K + 1) + K, NV);
  }
  if (!cta_finish(a, s, sm, NV, red)) return;
  if (threadIdx.x < 32) after_iter<K>(c, a, s, threadIdx.x, red, wlo);
}

// ---------------------------------------------------------------------------
// k_lsfb: further Armijo trials over the stored residual and u_dir only.

template <typename T, int VEC>
__global__ void __launch_bounds__(NT) k_lsfb(const __grid_constant__ Args a) {
  pdl_enter();
  const int s = a.s0 + blockIdx.y;
  Ctl* c = a.ctl + s;
  __shared__ int go, m0;
  if (threadIdx.x == 0) {
    go = c->status == ST_OK && c->active && c->need_lsfb;
    m0 = c->ls_next;
  }
  __syncthreads();
  mark_go(a, s, go);
  if (!go) return;
  __shared__ double sm[NW * LSW];
  __shared__ double red[LSW];
  const int base = m0;
  const int cnt = (a.max_bt - base) < LSW ? (a.max_bt - base) : LSW;
  T al[LSW];
  {
    double v = alpha_at(a, base);
#pragma unroll
    for (int m = 0; m < LSW; ++m) {
      al[m] = (T)v;
      v *= a.shrink;
    }
  }
  double cost[LSW];
#pragma unroll
  for (int m = 0; m < LSW; ++m) cost[m] = 0.0;
  const int ng = a.Pp / VEC;
  const T* R = static_cast<const T*>(a.r) + (size_t)s * a.np;
  const T* UD = static_cast<const T*>(a.ud) + (size_t)s * a.np;
  const uint8_t* L = a.lab + (size_t)s * a.Pp;
  for (int q = blockIdx.x * NT + threadIdx.x; q < ng; q += a.chunks * NT) {
    const int pix = q * VEC;
    T w[VEC];
    load_weights<T, VEC>(a, L, pix, w);
    for (int ch = 0; ch < a.C; ++ch) {
      const size_t off = (size_t)ch * a.Pp + pix;
      T r[VEC], ud[VEC];
      VecIO<T, VEC>::ld(R + off, r);
      VecIO<T, VEC>::ld(UD + off, ud);
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
#pragma unroll
        for (int m = 0; m < LSW; ++m) {
          if (m < cnt) {
            T tw, g;
            penalty(trial(r[e], al[m], ud[e]), w[e], a, tw, g);
            cost[m] += (double)tw;
          }
        }
      }
    }
  }
#pragma unroll
  for (int m = 0; m < LSW; ++m) cta_stage(cost[m], sm, m, LSW);
  if (!cta_finish(a, s, sm, LSW, red)) return;
  if (threadIdx.x < 32) after_lsfb(c, a, s, threadIdx.x, red, base);
}

// ---------------------------------------------------------------------------
// k_gradfb: coordinate gradient at an accepted step outside the window.

template <typename T, int K, int VEC>
__global__ void __launch_bounds__(NT, PROST_MINB) k_gradfb(const __grid_constant__ Args a) {
  pdl_enter();
  const int s = a.s0 + blockIdx.y;
  Ctl* c = a.ctl + s;
  __shared__ int go;
  __shared__ double salpha;
  if (threadIdx.x == 0) {
    go = c->status == ST_OK && c->active && c->need_gradfb;
    salpha = c->acc_alpha;
  }
  __syncthreads();
  mark_go(a, s, go);
  if (!go) return;
  constexpr int NV = K + 1;
  __shared__ double sm[NW * NV];
  __shared__ double red[NV];
  const T alpha = (T)salpha;
  T acc[K];
#pragma unroll
  for (int j = 0; j < K; ++j) acc[j] = (T)0;
  T gsq = (T)0;
  const int ng = a.Pp / VEC;
  const T* U = static_cast<const T*>(a.U) + (size_t)s * a.k * a.np;
  const T* R = static_cast<const T*>(a.r) + (size_t)s * a.np;
  const T* UD = static_cast<const T*>(a.ud) + (size_t)s * a.np;
  const uint8_t* L = a.lab + (size_t)s * a.Pp;
  for (int q = blockIdx.x * NT + threadIdx.x; q < ng; q += a.chunks * NT) {
    const int pix = q * VEC;
    T w[VEC];
    load_weights<T, VEC>(a, L, pix, w);
    for (int ch = 0; ch < a.C; ++ch) {
      const size_t off = (size_t)ch * a.Pp + pix;
      T r[VEC], ud[VEC], g[VEC];
      VecIO<T, VEC>::ld(R + off, r);
      VecIO<T, VEC>::ld(UD + off, ud);
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        T tw;
        penalty(trial(r[e], alpha, ud[e]), w[e], a, tw, g[e]);
        gsq += g[e] * g[e];
      }
#pragma unroll
      for (int j = 0; j < K; ++j) {
        if (j < a.k) {
          T u[VEC];
          VecIO<T, VEC>::ldg(U + (size_t)j * a.np + off, u);
#pragma unroll
          for (int e = 0; e < VEC; ++e) acc[j] += u[e] * g[e];
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < K; ++j) cta_stage((double)acc[j], sm, j, NV);
  cta_stage((double)gsq, sm, K, NV);
  if (!cta_finish(a, s, sm, NV, red)) return;
  if (threadIdx.x < 32) after_gradfb<K>(c, a, s, threadIdx.x, red);
}

// ---------------------------------------------------------------------------
// k_geo: rank-one geodesic step of U along the projected gradient, then the
// relabel / background / residual epilogue against the updated basis.
// QR = true: apply the inverse Cholesky factor of U'^T U' instead (periodic
// re-orthonormalization, manifold.py:192-196) and run the same epilogue.

template <typename T, int K, int VEC, bool QR>
__global__ void __launch_bounds__(NT, PROST_MINB) k_geo(const __grid_constant__ Args a) {
  pdl_enter();
  const int s = a.s0 + blockIdx.y;
  Ctl* c = a.ctl + s;
  __shared__ int go, dogeo, relabel;
  __shared__ double sv[K], sg[K], sy[K], sc[6];
  __shared__ double srinv[QR ? K * K : 1];
  if (threadIdx.x == 0) {
    go = c->status == ST_OK && (!QR || c->qr_now);
    dogeo = QR ? 1 : c->do_geo;
    relabel = QR ? 1 : !c->qr_now;
    sc[0] = c->geo_a;
    sc[1] = c->geo_s;
    sc[2] = c->geo_ln;
    sc[3] = c->pend_alpha;
    sc[4] = c->std_cur;
  }
  if (threadIdx.x < K) {
    const int j = threadIdx.x;
    sv[j] = j < a.k ? c->v[j] : 0.0;
    sg[j] = j < a.k ? c->grad[j] : 0.0;
    sy[j] = j < a.k ? c->y[j] : 0.0;
  }
  if (QR) {
    for (int i = threadIdx.x; i < K * K; i += NT) {
      const int l = i / K, j = i % K;
      srinv[i] = (l < a.k && j < a.k) ? a.rinv[(size_t)s * KMAX * KMAX + l * KMAX + j] : 0.0;
    }
  }
  __syncthreads();
  if (!go) return;
  const T ga = (T)sc[0], gsn = (T)sc[1], ln = (T)sc[2], pend = (T)sc[3], stdv = (T)sc[4];
  const bool do_geo = dogeo, do_lab = relabel;
  T v[K], gr[K], y[K];
#pragma unroll
  for (int j = 0; j < K; ++j) {
    v[j] = (T)sv[j];
    gr[j] = (T)sg[j];
    y[j] = (T)sy[j];
  }
  const int ng = a.Pp / VEC;
  T* U = static_cast<T*>(a.U) + (size_t)s * a.k * a.np;
  const T* R = static_cast<const T*>(a.r) + (size_t)s * a.np;
  const T* UD = static_cast<const T*>(a.ud) + (size_t)s * a.np;
  uint8_t* L = a.lab + (size_t)s * a.Pp;
  T* BG = a.bg_out ? static_cast<T*>(a.bg_out) + (size_t)s * a.np : nullptr;
  T* RES = a.res_out ? static_cast<T*>(a.res_out) + (size_t)s * a.np : nullptr;
  T* FRES = (!QR && a.fitres_out) ? static_cast<T*>(a.fitres_out) + (size_t)s * a.np : nullptr;
  for (int q = blockIdx.x * NT + threadIdx.x; q < ng; q += a.chunks * NT) {
    const int pix = q * VEC;
    T w[VEC];
    load_weights<T, VEC>(a, L, pix, w);
    T mx[VEC];
#pragma unroll
    for (int e = 0; e < VEC; ++e) mx[e] = (T)0;
    for (int ch = 0; ch < a.C; ++ch) {
      const size_t off = (size_t)ch * a.Pp + pix;
      if (FRES) {  // FitResult.residual: x - U y after the fit (fit.py:50-63)
        T r[VEC], ud[VEC];
        VecIO<T, VEC>::ld(R + off, r);
        if (sc[3] != 0.0) {
          VecIO<T, VEC>::ld(UD + off, ud);
#pragma unroll
          for (int e = 0; e < VEC; ++e) r[e] = trial(r[e], pend, ud[e]);
        }
        VecIO<T, VEC>::st(FRES + off, r);
      }
      T u[K][VEC];
#pragma unroll
      for (int j = 0; j < K; ++j) {
        if (j < a.k) {
          VecIO<T, VEC>::ld(U + (size_t)j * a.np + off, u[j]);
        } else {
#pragma unroll
          for (int e = 0; e < VEC; ++e) u[j][e] = (T)0;
        }
      }
      if (do_geo) {
        if constexpr (QR) {
          // U'' = U' R^{-1} (R upper triangular)
          T nu[K][VEC];
#pragma unroll
          for (int j = 0; j < K; ++j) {
#pragma unroll
            for (int e = 0; e < VEC; ++e) nu[j][e] = (T)0;
#pragma unroll
            for (int l = 0; l <= j; ++l) {
              const T rl = (T)srinv[l * K + j];
#pragma unroll
              for (int e = 0; e < VEC; ++e) nu[j][e] += u[l][e] * rl;
            }
          }
#pragma unroll
          for (int j = 0; j < K; ++j)
#pragma unroll
            for (int e = 0; e < VEC; ++e) u[j][e] = nu[j][e];
        } else {
          T r[VEC], ud[VEC];
          VecIO<T, VEC>::ld(R + off, r);
          if (sc[3] != 0.0) {
            VecIO<T, VEC>::ld(UD + off, ud);
#pragma unroll
            for (int e = 0; e < VEC; ++e) r[e] = trial(r[e], pend, ud[e]);
          }
#pragma unroll
          for (int e = 0; e < VEC; ++e) {
            T tw, g;
            penalty(r[e], w[e], a, tw, g);
            const T eta = -g;  // cost.py:103-112
            T uv = (T)0, ug = (T)0;
#pragma unroll
            for (int j = 0; j < K; ++j) {
              uv += u[j][e] * v[j];
              ug += u[j][e] * gr[j];
            }
            const T proj = eta - ug;  // manifold.py:127
            const T coef = ga * uv - gsn * (proj / ln);
#pragma unroll
            for (int j = 0; j < K; ++j) u[j][e] += coef * v[j];
          }
        }
#pragma unroll
        for (int j = 0; j < K; ++j)
          if (j < a.k) VecIO<T, VEC>::st(U + (size_t)j * a.np + off, u[j]);
      }
      if (do_lab) {
        T xh[VEC];
        bool bad = false;
        normalized<T, VEC>(a, (size_t)s * a.np + off, false, false, (T)1, stdv, xh, bad);
        T bgn[VEC], rr[VEC];
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
          T acc = (T)0;
#pragma unroll
          for (int j = 0; j < K; ++j) acc += u[j][e] * y[j];
          bgn[e] = acc;
          rr[e] = sub_rn(xh[e], acc);
          mx[e] = fmax(mx[e], fabs(rr[e]));
        }
        if (RES) VecIO<T, VEC>::st(RES + off, rr);
        if (BG) {
          T b[VEC];
          if (a.pipeline) {
            T mv[VEC];
            VecIO<T, VEC>::ld(static_cast<const T*>(a.mean) + (size_t)s * a.np + off, mv);
#pragma unroll
            for (int e = 0; e < VEC; ++e)
              b[e] = fmin(fmax(add_rn(bgn[e] * stdv, mv[e]), (T)0), (T)1);
          } else {
#pragma unroll
            for (int e = 0; e < VEC; ++e) b[e] = bgn[e];
          }
          VecIO<T, VEC>::st(BG + off, b);
        }
      }
    }
    if (do_lab) {
      uint8_t lb[VEC];
#pragma unroll
      for (int e = 0; e < VEC; ++e)
        lb[e] = (pix + e < a.P && (double)mx[e] >= a.delta) ? 1 : 0;
      st_lab<VEC>(L + pix, lb);
      if (a.raw_out) st_lab<VEC>(a.raw_out + (size_t)s * a.Pp + pix, lb);
    }
  }
}

// ---------------------------------------------------------------------------
// k_gram: G = U'^T U' for streams due for re-orthonormalization; the last CTA
// factors G = R^T R (Cholesky, R upper with positive diagonal — the same Q as
// the reference's sign-fixed Householder QR) and stores R^{-1}.

template <typename T, int K, int VEC>
__global__ void __launch_bounds__(NT) k_gram(const __grid_constant__ Args a) {
  pdl_enter();
  const int s = a.s0 + blockIdx.y;
  Ctl* c = a.ctl + s;
  __shared__ int go;
  if (threadIdx.x == 0) go = c->status == ST_OK && c->qr_now;
  __syncthreads();
  mark_go(a, s, go);
  if (!go) return;
  constexpr int NP = K * (K + 1) / 2;
  __shared__ double sm[NW * NP];
  __shared__ double red[NP];
  const int k = a.k;
  const int np_ = k * (k + 1) / 2;
  const int ng = a.Pp / VEC;
  const T* U = static_cast<const T*>(a.U) + (size_t)s * a.k * a.np;
  int pr = 0;
  for (int ia = 0; ia < k; ++ia) {
    for (int ib = ia; ib < k; ++ib, ++pr) {
      double acc = 0.0;
      for (int q = blockIdx.x * NT + threadIdx.x; q < ng; q += a.chunks * NT) {
        const int pix = q * VEC;
        for (int ch = 0; ch < a.C; ++ch) {
          const size_t off = (size_t)ch * a.Pp + pix;
          T ua[VEC], ub[VEC];
          VecIO<T, VEC>::ld(U + (size_t)ia * a.np + off, ua);
          VecIO<T, VEC>::ld(U + (size_t)ib * a.np + off, ub);
#pragma unroll
          for (int e = 0; e < VEC; ++e) acc += (double)ua[e] * (double)ub[e];
        }
      }
      cta_stage(acc, sm, pr, np_);
    }
  }
  if (!cta_finish(a, s, sm, np_, red)) return;
  if (threadIdx.x == 0) tail_gram(c, a, s, red);
}

// ---------------------------------------------------------------------------
// Label-row halos over peer memory (pixel sharding, prost_xpeer_open): this
// rank's first label row goes to the rank above (its row below), its last row
// to the rank below (its row above); the flag carries the frame number.
static __global__ void __launch_bounds__(NT) k_halo_push(const __grid_constant__ Args a) {
  pdl_enter();
  const int s = a.s0 + blockIdx.y;
  const int W = a.width, H = a.height, par = (int)(a.xframe & 1);
  const uint8_t* L = a.lab + (size_t)s * a.Pp;
  uint8_t* up = (a.xhalo & 1) ? xr_halo(a.xpeer[a.xrank - 1], a, par, 1) + (size_t)s * W : nullptr;
  uint8_t* dn = (a.xhalo & 2) ? xr_halo(a.xpeer[a.xrank + 1], a, par, 0) + (size_t)s * W : nullptr;
  for (int x = threadIdx.x; x < W; x += NT) {
    if (up) up[x] = L[x];
    if (dn) dn[x] = L[(size_t)(H - 1) * W + x];
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    if (up) st_release_sys(xr_hflag(a.xpeer[a.xrank - 1], a, 1, s), (unsigned long long)a.xframe);
    if (dn) st_release_sys(xr_hflag(a.xpeer[a.xrank + 1], a, 0, s), (unsigned long long)a.xframe);
  }
}

// The median's wait for this frame's halo rows from the neighbouring ranks.
__device__ __forceinline__ void halo_wait(const Args& a, int s) {
  if (!a.xpeer) return;
  if (threadIdx.x == 0) {
    void* own = a.xpeer[a.xrank];
    if (a.xhalo & 1) wait_flag(xr_hflag(own, a, 0, s), (unsigned long long)a.xframe);
    if (a.xhalo & 2) wait_flag(xr_hflag(own, a, 1, s), (unsigned long long)a.xframe);
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// k_median: 3x3 majority vote with edge replication (pipeline.py:215-228).

static __global__ void __launch_bounds__(NT) k_median(const __grid_constant__ Args a) {
  pdl_enter();
  const int s = a.s0 + blockIdx.y;
  if (a.ctl[s].status != ST_OK) return;
  halo_wait(a, s);
  const uint8_t* L = a.lab + (size_t)s * a.Pp;
  uint8_t* M = a.mask_out + (size_t)s * a.Pp;
  const int W = a.width, H = a.height;
  for (int p = blockIdx.x * NT + threadIdx.x; p < a.P; p += gridDim.x * NT) {
    const int yy = p / W, xx = p - yy * W;
    int votes = 0;
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy) {
      const int ry = yy + dy;
      const uint8_t* row = ry < 0 ? (a.halo_top ? a.halo_top + (size_t)s * W : L)
                                  : (ry >= H ? (a.halo_bot ? a.halo_bot + (size_t)s * W : L + (size_t)(H - 1) * W)
                                             : L + (size_t)ry * W);
#pragma unroll
      for (int dx = -1; dx <= 1; ++dx) {
        const int rx = min(max(xx + dx, 0), W - 1);
        votes += row[rx];
      }
    }
    M[p] = votes >= 5 ? 1 : 0;
  }
}

// k_median4: the same filter, four pixels per thread with byte-lane SIMD
// (widths that are a multiple of 4; every BASELINE shape).  Column sums of the
// three rows are one 32-bit add (labels are 0/1, sums <= 3 per byte); the
// horizontal window adds the word shifted by one byte each way, with the
// neighbouring columns (edge-replicated) shifted in; >= 5 is __vcmpgeu4.
static __global__ void __launch_bounds__(NT) k_median4(const __grid_constant__ Args a) {
  pdl_enter();
  const int s = a.s0 + blockIdx.y;
  if (a.ctl[s].status != ST_OK) return;
  halo_wait(a, s);
  const int W = a.width, H = a.height, wq = W >> 2;
  const uint8_t* L = a.lab + (size_t)s * a.Pp;
  uint32_t* M = reinterpret_cast<uint32_t*>(a.mask_out + (size_t)s * a.Pp);
  const int nw = wq * H;
  // rows beyond the local block: a neighbour's halo row (pixel sharding), else
  // the edge row itself (edge replication)
  const uint8_t* above = a.halo_top ? a.halo_top + (size_t)s * W : L;
  const uint8_t* below = a.halo_bot ? a.halo_bot + (size_t)s * W : L + (size_t)(H - 1) * W;
  for (int q = blockIdx.x * NT + threadIdx.x; q < nw; q += gridDim.x * NT) {
    const int yy = q / wq, xq = q - yy * wq, x0 = xq << 2;
    const int xl = x0 > 0 ? x0 - 1 : 0, xr = x0 + 4 < W ? x0 + 4 : W - 1;
    const uint8_t* ra = yy > 0 ? L + (size_t)(yy - 1) * W : above;
    const uint8_t* rm = L + (size_t)yy * W;
    const uint8_t* rb = yy < H - 1 ? L + (size_t)(yy + 1) * W : below;
    const uint32_t v = __ldg(reinterpret_cast<const uint32_t*>(ra + x0)) +
                       __ldg(reinterpret_cast<const uint32_t*>(rm + x0)) +
                       __ldg(reinterpret_cast<const uint32_t*>(rb + x0));
    const uint32_t l = (uint32_t)__ldg(ra + xl) + __ldg(rm + xl) + __ldg(rb + xl);
    const uint32_t r = (uint32_t)__ldg(ra + xr) + __ldg(rm + xr) + __ldg(rb + xr);
    const uint32_t win = v + ((v << 8) | l) + ((v >> 8) | (r << 24));
    M[q] = __vcmpgeu4(win, 0x05050505u) & 0x01010101u;
  }
}

// k_median16: sixteen pixels per thread (widths that are a multiple of 16):
// three 16-byte row loads and two edge bytes per row per 16 pixels.
static __global__ void __launch_bounds__(NT) k_median16(const __grid_constant__ Args a) {
  pdl_enter();
  const int s = a.s0 + blockIdx.y;
  if (a.ctl[s].status != ST_OK) return;
  halo_wait(a, s);
  const int W = a.width, H = a.height, wq = W >> 4;
  const uint8_t* L = a.lab + (size_t)s * a.Pp;
  uint8_t* M = a.mask_out + (size_t)s * a.Pp;
  const uint8_t* above = a.halo_top ? a.halo_top + (size_t)s * W : L;
  const uint8_t* below = a.halo_bot ? a.halo_bot + (size_t)s * W : L + (size_t)(H - 1) * W;
  const int nw = wq * H;
  for (int q = blockIdx.x * NT + threadIdx.x; q < nw; q += gridDim.x * NT) {
    const int yy = q / wq, x0 = (q - yy * wq) << 4;
    const int xl = x0 > 0 ? x0 - 1 : 0, xr = x0 + 16 < W ? x0 + 16 : W - 1;
    const uint8_t* ra = yy > 0 ? L + (size_t)(yy - 1) * W : above;
    const uint8_t* rm = L + (size_t)yy * W;
    const uint8_t* rb = yy < H - 1 ? L + (size_t)(yy + 1) * W : below;
    const uint4 A = __ldg(reinterpret_cast<const uint4*>(ra + x0));
    const uint4 B = __ldg(reinterpret_cast<const uint4*>(rm + x0));
    const uint4 C = __ldg(reinterpret_cast<const uint4*>(rb + x0));
    const uint32_t v[4] = {A.x + B.x + C.x, A.y + B.y + C.y, A.z + B.z + C.z, A.w + B.w + C.w};
    const uint32_t l = (uint32_t)__ldg(ra + xl) + __ldg(rm + xl) + __ldg(rb + xl);
    const uint32_t r = (uint32_t)__ldg(ra + xr) + __ldg(rm + xr) + __ldg(rb + xr);
    uint32_t o[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t lb = i > 0 ? (v[i - 1] >> 24) : l;
      const uint32_t rb8 = i < 3 ? (v[i + 1] & 0xffu) : r;
      const uint32_t win = v[i] + ((v[i] << 8) | lb) + ((v[i] >> 8) | (rb8 << 24));
      o[i] = __vcmpgeu4(win, 0x05050505u) & 0x01010101u;
    }
    *reinterpret_cast<uint4*>(M + (size_t)yy * W + x0) = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

// ---------------------------------------------------------------------------
// Resampling shell: bilinear frame resampling with
// half-pixel centres (pipeline.py:164-193) and nearest-neighbour mask
// upsampling (pipeline.py:245-258), in fp64 with the reference's operation
// order and no FMA contraction, so results equal numpy's bit for bit.

__device__ __forceinline__ void axis_coord(int i, int n_out, int n_in, int& lo, int& hi, double& w) {
  double src = __dsub_rn(__dmul_rn((double)i + 0.5, (double)n_in / (double)n_out), 0.5);
  src = fmin(fmax(src, 0.0), (double)n_in - 1.0);
  lo = (int)floor(src);
  hi = min(lo + 1, n_in - 1);
  w = __dsub_rn(src, (double)lo);
}

template <typename TI, typename TO>
__global__ void k_resample(const TI* __restrict__ src, TO* __restrict__ dst, int C, int w_in,
                           int h_in, int w_out, int h_out, double scale) {
  const long long total = (long long)C * w_out * h_out;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i / ((long long)w_out * h_out));
    const int rem = (int)(i - (long long)c * w_out * h_out);
    const int oy = rem / w_out, ox = rem - oy * w_out;
    int x0, x1, y0, y1;
    double wx, wy;
    axis_coord(ox, w_out, w_in, x0, x1, wx);
    axis_coord(oy, h_out, h_in, y0, y1, wy);
    const TI* pl = src + (size_t)c * w_in * h_in;
    const double a00 = (double)pl[(size_t)y0 * w_in + x0] * scale, a01 = (double)pl[(size_t)y0 * w_in + x1] * scale;
    const double a10 = (double)pl[(size_t)y1 * w_in + x0] * scale, a11 = (double)pl[(size_t)y1 * w_in + x1] * scale;
    const double top = __dadd_rn(__dmul_rn(1.0 - wx, a00), __dmul_rn(wx, a01));
    const double bot = __dadd_rn(__dmul_rn(1.0 - wx, a10), __dmul_rn(wx, a11));
    dst[i] = (TO)__dadd_rn(__dmul_rn(1.0 - wy, top), __dmul_rn(wy, bot));
  }
}

static __global__ void k_upsample_mask(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, int w_in,
                                int h_in, int w_out, int h_out) {
  const long long total = (long long)w_out * h_out;
  const double fx = (double)w_in / (double)w_out, fy = (double)h_in / (double)h_out;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int oy = (int)(i / w_out), ox = (int)(i - (long long)oy * w_out);
    const int xs = min((int)__dmul_rn((double)ox + 0.5, fx), w_in - 1);
    const int ys = min((int)__dmul_rn((double)oy + 0.5, fy), h_in - 1);
    dst[i] = src[(size_t)ys * w_in + xs];
  }
}

// ---------------------------------------------------------------------------
// k_confusion: per-stream tp / fp / tn / fn of a predicted mask against a
// ground-truth frame (evaluate.py:87-106): pixels labelled outside-ROI (85) or
// unknown (170) are not scored, 255 is foreground, every other value
// background.  Integer atomics: exact and order-independent.

static __global__ void __launch_bounds__(NT) k_confusion(const uint8_t* __restrict__ mask,
                                                  const uint8_t* __restrict__ truth, int P,
                                                  long long mask_stride, unsigned long long* counts) {
  const int s = blockIdx.y;
  const uint8_t* M = mask + (size_t)s * mask_stride;
  const uint8_t* G = truth + (size_t)s * P;
  unsigned c[4] = {0u, 0u, 0u, 0u};  // tp, fp, tn, fn
  for (int p = blockIdx.x * NT + threadIdx.x; p < P; p += gridDim.x * NT) {
    const unsigned g = G[p];
    if (g == 85u || g == 170u) continue;
    const bool tfg = g == 255u, pfg = M[p] != 0;
    c[tfg ? (pfg ? 0 : 3) : (pfg ? 1 : 2)] += 1u;
  }
  __shared__ unsigned long long sc[4];
  if (threadIdx.x < 4) sc[threadIdx.x] = 0ull;
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    unsigned v = c[i];
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(&sc[i], (unsigned long long)v);
  }
  __syncthreads();
  if (threadIdx.x < 4 && sc[threadIdx.x]) atomicAdd(counts + (size_t)s * 4 + threadIdx.x, sc[threadIdx.x]);
}

// ---------------------------------------------------------------------------
// k_unpack_pnm: binary PGM / PPM payload (interleaved u8) -> channel-planar
// intensities on [0, 1] (decode_pnm, frameio.py:120-137): x / 255 in fp64
// (correctly rounded, as numpy), then the output type.

template <typename TO>
__global__ void k_unpack_pnm(const uint8_t* __restrict__ payload, int C, int P, TO* __restrict__ dst) {
  const long long total = (long long)C * P;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i / P), p = (int)(i - (long long)c * P);
    dst[i] = (TO)__ddiv_rn((double)payload[(size_t)p * C + c], 255.0);
  }
}

// ---------------------------------------------------------------------------
// k_combine3: 3-channel label = any channel's abs(r') >= delta (pipeline.py:
// 210-211) from the TMEM kernel's per-coordinate flags; streams whose frame
// was rejected keep their labels.

static __global__ void __launch_bounds__(NT) k_combine3(const __grid_constant__ Args a) {
  const int s = a.s0 + blockIdx.y;
  if (a.ctl[s].status != ST_OK) return;
  const uint32_t* F = reinterpret_cast<const uint32_t*>(a.labc + (size_t)s * a.np);
  uint32_t* L = reinterpret_cast<uint32_t*>(a.lab + (size_t)s * a.Pp);
  uint32_t* R = a.raw_out ? reinterpret_cast<uint32_t*>(a.raw_out + (size_t)s * a.Pp) : nullptr;
  const int nw = a.Pp / 4, pw = a.Pp / 4;
  for (int q = blockIdx.x * NT + threadIdx.x; q < nw; q += gridDim.x * NT) {
    const uint32_t v = F[q] | F[pw + q] | F[2 * pw + q];
    L[q] = v;
    if (R) R[q] = v;
  }
}

// ---------------------------------------------------------------------------
// k_xlogic: exchange mode — the scalar tail of phase `step` for every stream
// the phase ran for, from the cross-rank sums in xred (one warp per stream).

// XS_START: the statistics kernel once every stream is frozen — no reduction
// and so no exchange, but it still opens the frame (std, status: a frame
// after a rejected one must run)
enum XStep { XS_STATS = 0, XS_COLD, XS_PASS0, XS_ITER, XS_LSFB, XS_GRADFB, XS_GEO, XS_GRAM, XS_GEOQR, XS_START };

template <int K>
__global__ void __launch_bounds__(32) k_xlogic(const __grid_constant__ Args a, int step) {
  const int s = a.s0 + blockIdx.x;
  if (!a.xgo[s]) return;
  Ctl* c = a.ctl + s;
  __shared__ double red[KMAX * (KMAX + 1) / 2 + 8];
  const int lane = threadIdx.x;
  for (int v = lane; v < a.nvmax; v += 32) red[v] = a.xred[(size_t)s * a.nvmax + v];
  __syncwarp();
  switch (step) {
    case XS_STATS: if (lane == 0) tail_stats(c, a, s, red); break;
    case XS_COLD: tail_cold<K>(c, a, s, lane, red); break;
    case XS_PASS0: after_pass0<K>(c, a, s, lane, red); break;
    case XS_ITER: after_iter<K>(c, a, s, lane, red, c->gwin_lo); break;
    case XS_LSFB: after_lsfb(c, a, s, lane, red, c->ls_next); break;
    case XS_GRADFB: after_gradfb<K>(c, a, s, lane, red); break;
    case XS_GRAM: if (lane == 0) tail_gram(c, a, s, red); break;
    default: break;
  }
}

// ---------------------------------------------------------------------------
// k_background: clip((U y) * scale + mean, 0, 1) (jobs.py:231-239).

template <typename T, int K, int VEC>
__global__ void __launch_bounds__(NT) k_background(const __grid_constant__ Args a) {
  const int s = a.s0 + blockIdx.y;
  const Ctl* c = a.ctl + s;
  __shared__ double sy[K], sscale;
  if (threadIdx.x < K) sy[threadIdx.x] = threadIdx.x < a.k ? c->y[threadIdx.x] : 0.0;
  if (threadIdx.x == 0) sscale = c->frozen ? c->pstd : running_std(c);
  __syncthreads();
  const T scale = (T)sscale;
  const T* U = static_cast<const T*>(a.U) + (size_t)s * a.k * a.np;
  const T* M = static_cast<const T*>(a.mean) + (size_t)s * a.np;
  T* BG = static_cast<T*>(a.bg_out) + (size_t)s * a.np;
  const int ng = a.Pp / VEC;
  for (int q = blockIdx.x * NT + threadIdx.x; q < ng; q += a.chunks * NT) {
    const int pix = q * VEC;
    for (int ch = 0; ch < a.C; ++ch) {
      const size_t off = (size_t)ch * a.Pp + pix;
      T acc[VEC];
#pragma unroll
      for (int e = 0; e < VEC; ++e) acc[e] = (T)0;
#pragma unroll
      for (int j = 0; j < K; ++j) {
        if (j < a.k) {
          T u[VEC];
          VecIO<T, VEC>::ld(U + (size_t)j * a.np + off, u);
#pragma unroll
          for (int e = 0; e < VEC; ++e) acc[e] += u[e] * (T)sy[j];
        }
      }
      T mv[VEC], b[VEC];
      VecIO<T, VEC>::ld(M + off, mv);
#pragma unroll
      for (int e = 0; e < VEC; ++e) b[e] = fmin(fmax(add_rn(acc[e] * scale, mv[e]), (T)0), (T)1);
      VecIO<T, VEC>::st(BG + off, b);
    }
  }
}

// ---------------------------------------------------------------------------
// layout conversion between dense user arrays [S][C][P] and padded [S][C][Pp]

template <typename TS, typename TD>
__global__ void k_pack(const TS* __restrict__ src, TD* __restrict__ dst, int S, int C, int P,
                       int Pp, int to_padded, double scale) {
  const long long total = (long long)S * C * P;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long row = i / P;
    const int p = (int)(i - row * P);
    const long long dense = i, padded = row * Pp + p;
    if (to_padded) dst[padded] = (TD)((double)src[dense] * scale);
    else dst[dense] = (TD)((double)src[padded] * scale);
  }
}

}  // namespace prost
