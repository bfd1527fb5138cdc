// prost_logic_fast.cuh — the scalar part of the CG fit and the geodesic
// set-up (fit.py:108-153, manifold.py:130-197, tracker.py:140-143) for the
// fp32 TMEM kernel, with the reductions of a decision step fused into one
// warp butterfly.
//
// Same decisions as after_pass0 / after_iter / after_lsfb / after_gradfb in
// prost_kernels.cuh (which the fp64 parity instantiation keeps: they sum
// every dot product separately, in the order the reference's numpy code
// forms them).  Here lane j holds component j of y, d and the gradient in
// registers, and every quantity the step needs — ||g_new||^2, g_new.g_old,
// g_new.d_old, ||y_new||^2 — comes out of ONE butterfly of four doubles:
//   beta  = max(0, (||g_new||^2 - g_new.g_old) / ||g_old||^2)      fit.py:140
//   d_new = -g_new + beta d_old, slope = d_new.g_new = -||g_new||^2 + beta g_new.d_old
//   ||y|| for v = y / ||y|| and the projected-gradient norm (finish).
// Each team sum's scalar tail drops from ~5 dependent warp sums (plus the
// exp() of the step size, now taken at frame start) to one.
#pragma once

#include "prost_kernels.cuh"

#ifndef PROST_FL_SEQ
#define PROST_FL_SEQ 0
#endif
#ifndef PROST_FL_OLDFIN
#define PROST_FL_OLDFIN 0
#endif
#ifndef PROST_FL_NOMOD
#define PROST_FL_NOMOD 0
#endif

namespace prost {

// Butterfly sum of four doubles over the warp (all lanes get the totals).
__device__ __forceinline__ void warp_sum4(double& a, double& b, double& c, double& d) {
#if PROST_FL_SEQ
  a = warp_sum(a); b = warp_sum(b); c = warp_sum(c); d = warp_sum(d); return;
#endif
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, m);
    b += __shfl_xor_sync(0xffffffffu, b, m);
    c += __shfl_xor_sync(0xffffffffu, c, m);
    d += __shfl_xor_sync(0xffffffffu, d, m);
  }
}

// End of the CG loop: projected-gradient norm, geodesic scalars.  g2 =
// ||U^T eta||^2 (the last gradient), yn2 = ||y||^2, yj = y[lane]; the step
// size c->t was set at frame start.
__device__ __forceinline__ void fl_finish(Ctl* c, const Args& a, int s, int lane, double g2,
                                          double yn2, double yj) {
#if PROST_FL_OLDFIN
  __syncwarp(); finish_frame(c, a, s, lane); return;
#endif
  const double t = c->t;
  const double rn = sqrt(yn2);
  const double ln = sqrt(fmax(c->gsq - g2, 0.0));  // ||eta - U U^T eta|| (orthonormal U)
  const bool zero = (ln < NORM_FLOOR) || (rn < NORM_FLOOR) || (t == 0.0);
  if (!zero && lane < a.k) c->v[lane] = yj / rn;
  if (lane == 0) {
    c->active = 0;
    if (zero) {
      c->do_geo = 0;
      c->qr_now = 0;
    } else {
      const double phi = (ln * rn) * t;
      c->do_geo = 1;
      double sphi, cphi;
      sincos(phi, &sphi, &cphi);
      c->geo_a = cphi - 1.0;
      c->geo_s = sphi;
      c->geo_ln = ln;
      c->geo_yn = rn;
      c->since_qr += 1;
      c->qr_now = c->since_qr >= QR_EVERY ? 1 : 0;
    }
    c->frame_index += 1;
    write_info(c, a, s);
  }
  __syncwarp();
}

// Top of CG iteration `it` (fit.py:108-119) with gradient gj (lane), current
// direction dj, gn2 = ||g||^2, slope = d.g, yn2 / yj for an immediate finish.
__device__ __forceinline__ void fl_begin(Ctl* c, const Args& a, int s, int lane, int it, double gj,
                                         double dj, double gn2, double slope, double yn2, double yj) {
  if (lane == 0) {
    c->need_lsfb = 0;
    c->need_gradfb = 0;
  }
  if (it >= a.max_iters) {
    fl_finish(c, a, s, lane, gn2, yn2, yj);
    return;
  }
  const double gn = sqrt(gn2);
  if (gn <= a.grad_tol) {
    fl_finish(c, a, s, lane, gn2, yn2, yj);
    return;
  }
  if (!PROST_FL_NOMOD && it > 0 && it % a.k == 0) {  // periodic restart
    dj = -gj;
    slope = -gn2;
  }
  if (slope >= 0.0) {  // not a descent direction: steepest descent
    dj = -gj;
    slope = -gn * gn;
  }
  if (lane < a.k) c->d[lane] = dj;
  if (lane == 0) {
    c->slope = slope;
    c->gnorm = gn;
    c->active = 1;
    int lo = c->last_acc;
    lo = lo < 0 ? 0 : (lo > WC - WG ? WC - WG : lo);
    c->gwin_lo = lo;
  }
  __syncwarp();
}

// Accepted step alpha with cost fnew and coordinate-gradient sums gs[j]
// (= sum_i U_ij g_i): fit.py:137-144.
__device__ __forceinline__ void fl_complete(Ctl* c, const Args& a, int s, int lane, double alpha,
                                            double fnew, const double* gs, double gsq_new) {
  const bool own = lane < a.k;
  const double dj = own ? c->d[lane] : 0.0;
  const double gold = own ? c->grad[lane] : 0.0;
  const double gnew = own ? -gs[lane] : 0.0;
  const double yj = own ? c->y[lane] + alpha * dj : 0.0;
  const double gnorm = c->gnorm;
  const int it = c->it + 1;
  double s1 = gnew * gnew, s2 = gnew * gold, s3 = gnew * dj, s4 = yj * yj;
  warp_sum4(s1, s2, s3, s4);
  const double beta = fmax(0.0, (s1 - s2) / (gnorm * gnorm));
  const double dnew = -gnew + beta * dj;
  __syncwarp();
  if (own) {
    c->y[lane] = yj;
    c->d[lane] = dnew;
    c->grad[lane] = gnew;
  }
  if (lane == 0) {
    c->pend_alpha = alpha;
    c->f = fnew;
    c->gsq = gsq_new;
    c->cost_evals += 1;
    c->grad_evals += 1;
    c->iterations = it;
    c->it = it;
  }
  __syncwarp();
  fl_begin(c, a, s, lane, it, gnew, dnew, s1, -s1 + beta * s3, s4, yj);
}

// fit.py:133-134: no acceptable step -> leave the loop, residual unchanged.
__device__ __forceinline__ void fl_fail(Ctl* c, const Args& a, int s, int lane) {
  const bool own = lane < a.k;
  const double gj = own ? c->grad[lane] : 0.0;
  const double yj = own ? c->y[lane] : 0.0;
  double g2 = gj * gj, y2 = yj * yj, z0 = 0.0, z1 = 0.0;
  warp_sum4(g2, y2, z0, z1);
  if (lane == 0) c->pend_alpha = 0.0;
  __syncwarp();
  fl_finish(c, a, s, lane, g2, y2, yj);
}

// red: [0] cost, [1..K] sum_i U_ij g_i, [K+1] ||g||^2, [K+2] non-finite count
template <int K>
__device__ __forceinline__ void fl_after_pass0(Ctl* c, const Args& a, int s, int lane, const double* red) {
  if (red[K + 2] > 0.0) {
    mark_nonfinite(c, a, s, lane);
    return;
  }
  const bool own = lane < a.k;
  const double gj = own ? -red[1 + lane] : 0.0;  // fit.py:101: grad = -(U^T g)
  const double yj = own ? c->y[lane] : 0.0;
  if (own) {
    c->grad[lane] = gj;
    c->d[lane] = -gj;
  }
  if (lane == 0) {
    c->f = red[0];
    c->gsq = red[K + 1];
    c->it = 0;
    c->iterations = 0;
    c->cost_evals = 1;
    c->grad_evals = 1;
    c->pend_alpha = 0.0;
  }
  double g2 = gj * gj, y2 = yj * yj, z0 = 0.0, z1 = 0.0;
  warp_sum4(g2, y2, z0, z1);
  __syncwarp();
  fl_begin(c, a, s, lane, 0, gj, -gj, g2, -g2, y2, yj);
}

// red: [0..WC) trial costs, then per speculative slot mm: K gradient sums + ||g||^2
template <int K>
__device__ __forceinline__ void fl_after_iter(Ctl* c, const Args& a, int s, int lane, const double* red,
                                              int wlo) {
  const int nmax = a.max_bt < WC ? a.max_bt : WC;
  int first = -1;
  double alpha = a.step0;
  for (int m = 0; m < nmax; ++m) {
    if (red[m] <= c->f + a.c_armijo * alpha * c->slope) {  // fit.py:126-135
      first = m;
      break;
    }
    alpha *= a.shrink;
  }
  if (lane == 0) c->pend_alpha = 0.0;
  __syncwarp();
  if (first >= 0) {
    const int mm = first - wlo;
    if (lane == 0) {
      c->cost_evals += first + 1;
      c->last_acc = first;
    }
    __syncwarp();
    if (mm >= 0 && mm < WG) {
      fl_complete(c, a, s, lane, alpha, red[first], red + WC + mm * (K + 1), red[WC + mm * (K + 1) + K]);
    } else if (lane == 0) {
      c->need_gradfb = 1;
      c->acc_idx = first;
      c->acc_alpha = alpha;
      c->acc_cost = red[first];
    }
  } else {
    if (lane == 0) c->cost_evals += nmax;
    __syncwarp();
    if (nmax >= a.max_bt) {
      fl_fail(c, a, s, lane);
    } else if (lane == 0) {
      c->need_lsfb = 1;
      c->ls_next = nmax;
    }
  }
  __syncwarp();
}

// red: [0..cnt) trial costs for step indices base..base+cnt-1
__device__ __forceinline__ void fl_after_lsfb(Ctl* c, const Args& a, int s, int lane, const double* red,
                                              int base) {
  const int cnt = (a.max_bt - base) < LSW ? (a.max_bt - base) : LSW;
  const double f = c->f, slope = c->slope;
  int first = -1;
  double alpha = alpha_at(a, base);
  for (int m = 0; m < cnt; ++m) {
    if (red[m] <= f + a.c_armijo * alpha * slope) {
      first = m;
      break;
    }
    alpha *= a.shrink;
  }
  if (first >= 0) {
    if (lane == 0) {
      c->cost_evals += first + 1;
      c->need_lsfb = 0;
      c->need_gradfb = 1;
      c->last_acc = base + first;
      c->acc_idx = base + first;
      c->acc_alpha = alpha;
      c->acc_cost = red[first];
    }
  } else {
    if (lane == 0) c->cost_evals += cnt;
    __syncwarp();
    if (base + cnt >= a.max_bt) {
      if (lane == 0) c->need_lsfb = 0;
      __syncwarp();
      fl_fail(c, a, s, lane);
    } else if (lane == 0) {
      c->ls_next = base + cnt;
    }
  }
  __syncwarp();
}

// red: [0..K) gradient sums at the accepted step, [K] ||g||^2
template <int K>
__device__ __forceinline__ void fl_after_gradfb(Ctl* c, const Args& a, int s, int lane, const double* red) {
  if (lane == 0) c->need_gradfb = 0;
  __syncwarp();
  fl_complete(c, a, s, lane, c->acc_alpha, c->acc_cost, red, red[K]);
}

}  // namespace prost
