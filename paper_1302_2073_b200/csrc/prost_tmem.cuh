// prost_tmem.cuh — the TMEM-resident frame kernel (k_tmem).
//
// Same team structure as k_resident (a persistent cooperative grid split into
// T teams of G CTAs; a team owns one stream per round; the frame's dependent
// reductions are team-wide sums through double-buffered global slots and a
// release/acquire counter barrier, after which every CTA runs the scalar
// logic itself).  The difference is where a CTA keeps its slice of U: each
// thread owns QT row groups (4 rows x k values) in its lane of tensor memory
// (written once per frame with tcgen05.st, read row by row with tcgen05.ld in
// every phase), plus, when the slice is larger, row groups in shared memory.
// With 256 KB of TMEM + shared memory per SM a C3 stream (76,800 x 15 fp32 =
// 4.6 MB) fits on 13 SMs, so 11 streams are in flight at once, and U crosses
// HBM exactly once each way per frame.  Working one row (k values) at a time
// keeps the live basis registers at 16 instead of 4k.
#pragma once

#include "prost_resident.cuh"
#include "tmem_io.cuh"

namespace prost {

#ifndef PROST_TM_NT
#define PROST_TM_NT 512
#endif
#ifndef PROST_TM_CPS
#define PROST_TM_CPS 1
#endif
// threads per CTA: 4 warps per 128-column TMEM block (one per lane quarter);
// the CTA allocates TM_NT columns.  TM_CPS CTAs share an SM (their teams
// interleave: one computes while the other waits on a team barrier).
constexpr int TM_NT = PROST_TM_NT;
constexpr int TM_CPS = PROST_TM_CPS;
static_assert(TM_NT == 128 || TM_NT == 256 || TM_NT == 512, "TMEM allocation is TM_NT columns");

template <int K>
struct TmemGeom {
  // columns per row (power of two >= k: every tcgen05 access is width-aligned)
  static constexpr int RS = K <= 4 ? 4 : (K <= 8 ? 8 : 16);
  static constexpr int QW = 4 * RS;        // columns per row group
  static constexpr int QT = 128 / QW;      // row groups per thread in TMEM
};

// Dynamic shared memory of k_tmem<K> for qpc row groups per CTA.
template <int K>
__host__ __device__ constexpr size_t tmem_smem(int qpc) {
  const int qs = qpc > TmemGeom<K>::QT * TM_NT ? qpc - TmemGeom<K>::QT * TM_NT : 0;
  return (size_t)16 * TmemGeom<K>::RS * qs     // basis row groups kept in shared memory
         + (size_t)qpc * (3 * 16 + 4)           // r, u_dir, normalized frame, labels
         + (size_t)(TM_NT / 32 + 1) * RES_RNV_MAX * 8 + sizeof(Ctl) + 64;
}

template <int RS>
__device__ __forceinline__ void tmem_ld_row(unsigned taddr, float (&v)[RS]) {
  if constexpr (RS == 16) tmem_ld16(taddr, v);
  else if constexpr (RS == 8) tmem_ld8(taddr, v);
  else tmem_ld4(taddr, v);
}
template <int RS>
__device__ __forceinline__ void tmem_st_row(unsigned taddr, const float (&v)[RS]) {
  if constexpr (RS == 16) tmem_st16(taddr, v);
  else if constexpr (RS == 8) tmem_st8(taddr, v);
  else tmem_st4(taddr, v);
}

__device__ __forceinline__ void f4(float4 v, float (&o)[4]) {
  o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
}

// k-term dot product with four independent partial sums (short FMA chains)
template <int K>
__device__ __forceinline__ float dotk(const float* u, const float* v) {
  float p0 = 0.f, p1 = 0.f, p2 = 0.f, p3 = 0.f;
#pragma unroll
  for (int j = 0; j < K; j += 4) {
    p0 = fmaf(u[j], v[j], p0);
    if (j + 1 < K) p1 = fmaf(u[j + 1], v[j + 1], p1);
    if (j + 2 < K) p2 = fmaf(u[j + 2], v[j + 2], p2);
    if (j + 3 < K) p3 = fmaf(u[j + 3], v[j + 3], p3);
  }
  return (p0 + p1) + (p2 + p3);
}

template <int K, int PM>
__global__ void __launch_bounds__(TM_NT, TM_CPS)
    k_tmem(const __grid_constant__ Args a, const __grid_constant__ RArgs ra) {
  using Geo = TmemGeom<K>;
  constexpr int RS = Geo::RS, QW = Geo::QW, QT = Geo::QT;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  __shared__ unsigned s_tbase;
  __shared__ unsigned long long sprof[PROF_N];
  __shared__ float sfv[4][K];  // fp32 copies of y, d, v, grad for the per-element math
  const int G = ra.G, T = ra.T, qpc = ra.qpc;
  const int team = blockIdx.x / G, rank = blockIdx.x - team * G;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int k = a.k;
  const int nq = a.Pp / 4;
  const int q0 = rank * qpc;
  const int qcount = max(0, min(qpc, nq - q0));
  const int nslots = (qcount + TM_NT - 1) / TM_NT;  // uniform across the CTA
  const int qs = qpc > QT * TM_NT ? qpc - QT * TM_NT : 0;

  // basis rows kept in shared memory: [row e][4-column group][row group] float4,
  // so a thread reads one row with RS/4 conflict-free 16-byte loads
  float4* sU = reinterpret_cast<float4*>(smem_raw);         // [4][RS/4][qs]
  float4* sR = sU + (size_t)RS * qs;                        // [qpc] residual
  float4* sD = sR + qpc;                                    // [qpc] u_dir
  float4* sX = sD + qpc;                                    // [qpc] normalized frame
  uint32_t* sL = reinterpret_cast<uint32_t*>(sX + qpc);     // [qpc] label bytes
  const float* Mg = static_cast<const float*>(a.mean);      // running mean stays in global/L2
  double* wred = reinterpret_cast<double*>(sL + ((qpc + 1) / 2) * 2);
  double* red = wred + (size_t)(TM_NT / 32) * RES_RNV_MAX;
  Ctl* cs = reinterpret_cast<Ctl*>(red + RES_RNV_MAX);

  if (tid < PROF_N) sprof[tid] = 0;
  const unsigned long long t_start = gtimer();
  // TMEM: TM_NT columns, allocated by warp 0
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
        smem_addr(&s_tbase)), "n"(TM_NT));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  // this thread's lane and columns: lane quarter = warp % 4, column block = warp / 4
  const unsigned tbase =
      s_tbase + ((unsigned)(32 * (warp & 3)) << 16) + (unsigned)((warp >> 2) * 128);
  unsigned epoch = 0;

#define SYNC_FLOATS()                      \
  do {                                     \
    if (tid < K) {                         \
      sfv[0][tid] = (float)cs->y[tid];     \
      sfv[1][tid] = (float)cs->d[tid];     \
      sfv[2][tid] = (float)cs->v[tid];     \
      sfv[3][tid] = (float)cs->grad[tid];  \
    }                                      \
  } while (0)
#define LOGIC(call)                                                        \
  do {                                                                     \
    const unsigned long long tl0 = (ra.prof && tid == 0) ? gtimer() : 0;   \
    if (tid < 32) {                                                        \
      call;                                                                \
      __syncwarp();                                                        \
      SYNC_FLOATS();                                                       \
    }                                                                      \
    if (ra.prof && tid == 0) sprof[PROF_LOGIC] += gtimer() - tl0;          \
  } while (0)

  // One row (e) of row group `slot`: the k basis values of that coordinate.
  // TMEM rows are read by the whole warp (tcgen05 is warp-collective).
  auto load_row = [&](int slot, int e, float (&u)[RS]) {
    if (slot < QT) {
      tmem_ld_row<RS>(tbase + slot * QW + e * RS, u);
      tmem_wait_ld();
    } else {
      const int i = slot * TM_NT + tid - QT * TM_NT;
      const bool ok = slot * TM_NT + tid < qcount;
      const float4* rp = sU + (size_t)(e * (RS / 4)) * qs + i;
#pragma unroll
      for (int g4 = 0; g4 < RS / 4; ++g4) {
        const float4 t = ok ? rp[(size_t)g4 * qs] : make_float4(0.f, 0.f, 0.f, 0.f);
        u[4 * g4] = t.x; u[4 * g4 + 1] = t.y; u[4 * g4 + 2] = t.z; u[4 * g4 + 3] = t.w;
      }
    }
  };
  const float omega = a.omegaf;
  auto weights = [&](int qi, float (&w)[4]) {
    const uint32_t lb = qi < qcount ? sL[qi] : 0u;
    const int pix = (q0 + qi) * 4;
#pragma unroll
    for (int e = 0; e < 4; ++e)
      w[e] = (qi < qcount && pix + e < a.P) ? (((lb >> (8 * e)) & 0xffu) ? omega : 1.f) : 0.f;
  };
  const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);

  // Stagger the teams: rounds are near-identical in length, so without an
  // offset all teams load (and store) their slices at the same moment and the
  // HBM traffic comes in bursts.  Odd teams start half a round late (ra.stagger_ns).
  if ((team & 1) && ra.stagger_ns > 0) {
    const unsigned long long t0 = gtimer();
    while (gtimer() - t0 < (unsigned long long)ra.stagger_ns) __nanosleep(1000);
  }

  for (int s = team; s < ra.S; s += T) {
    if (ra.prof && tid == 0) sprof[PROF_ROUNDS] += 1;
    // ---- load this stream's slice: U -> TMEM / shared, frame, mean, labels ---
    {
      const unsigned long long tw0 = (ra.prof && tid == 0) ? gtimer() : 0;
      const float* U = static_cast<const float*>(a.U) + (size_t)s * k * a.np;
      for (int slot = 0; slot < nslots; ++slot) {
        const int qi = slot * TM_NT + tid;  // row group within the slice
        const bool ok = qi < qcount;
        const size_t off = (size_t)(q0 + qi) * 4;
        float4 p[K];
#pragma unroll
        for (int j = 0; j < K; ++j)
          p[j] = (ok && j < k) ? __ldcs(reinterpret_cast<const float4*>(U + (size_t)j * a.np + off)) : z4;
        if (ok) {
          sX[qi] = __ldcs(reinterpret_cast<const float4*>(static_cast<const float*>(a.x) + (size_t)s * a.np + off));
          sL[qi] = *reinterpret_cast<const uint32_t*>(a.lab + (size_t)s * a.Pp + (q0 + qi) * 4);
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float row[RS];
#pragma unroll
          for (int j = 0; j < RS; ++j) {
            const float4 t = j < K ? p[j] : z4;
            row[j] = e == 0 ? t.x : (e == 1 ? t.y : (e == 2 ? t.z : t.w));
          }
          if (slot < QT) {
            tmem_st_row<RS>(tbase + slot * QW + e * RS, row);
          } else if (ok) {
            float4* rp = sU + (size_t)(e * (RS / 4)) * qs + (qi - QT * TM_NT);
#pragma unroll
            for (int g4 = 0; g4 < RS / 4; ++g4)
              rp[(size_t)g4 * qs] = make_float4(row[4 * g4], row[4 * g4 + 1], row[4 * g4 + 2], row[4 * g4 + 3]);
          }
        }
      }
      tmem_wait_st();
      if (tid < (int)(sizeof(Ctl) / 8))
        reinterpret_cast<double*>(cs)[tid] = __ldcg(reinterpret_cast<const double*>(a.ctl + s) + tid);
      __syncthreads();
      if (tid == 0) cs->no_info = rank != 0;
      SYNC_FLOATS();
      __syncthreads();
      if (ra.prof && tid == 0) sprof[PROF_PREFETCH] += gtimer() - tw0;
    }

    unsigned long long tph = (ra.prof && tid == 0) ? gtimer() : 0;
#define PHASE_MARK(idx)                              \
  do {                                               \
    if (ra.prof && tid == 0) {                       \
      const unsigned long long tn = gtimer();        \
      sprof[idx] += tn - tph;                        \
      tph = tn;                                      \
    }                                                \
  } while (0)
    // ---- frame start: running statistics (pipeline.py:120-140) -------------
    const bool upd = a.pipeline && !cs->frozen && cs->frame_index < a.i_init;
    if (upd) {
      double s1 = 0.0, s2 = 0.0, nf = 0.0;
      for (int slot = 0; slot < nslots; ++slot) {
        const int qi = slot * TM_NT + tid;
        if (qi >= qcount) continue;
        float xv[4];
        f4(sX[qi], xv);
        const int pix = (q0 + qi) * 4;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          if (pix + e < a.P) {
            const double v = (double)xv[e];
            s1 += v;
            s2 += v * v;
            nf += isfinite(v) ? 0.0 : 1.0;
          }
        }
      }
      rstage(s1, wred, 0, 3);
      rstage(s2, wred, 1, 3);
      rstage(nf, wred, 2, 3);
      team_sum(ra, team, rank, wred, 3, red, epoch, sprof);
      if (tid == 0) {
        if (red[2] > 0.0) {
          cs->status = ST_NONFINITE;
          cs->t = step_size(a, cs->frame_index);
          write_info(cs, a, s);
        } else {
          cs->psum += red[0];
          cs->psumsq += red[1];
          cs->pcount += a.n_real;
          cs->pseen += 1;
          cs->std_cur = running_std(cs);
          cs->update_stats = 1;
          cs->status = ST_OK;
        }
      }
    } else if (tid == 0) {
      double sd = 1.0;
      if (a.pipeline) {
        sd = cs->frozen ? cs->pstd : running_std(cs);
        if (!cs->frozen) {
          cs->frozen = 1;
          cs->pstd = sd;
        }
      }
      cs->std_cur = sd;
      cs->update_stats = 0;
      cs->status = ST_OK;
    }
    __syncthreads();

    // normalize the frame in place; fold the running mean (pipeline.py:148-156)
    bool bad = false;
    if (cs->status == ST_OK) {
      const float stdv = (float)cs->std_cur, seen = (float)cs->pseen;
      for (int slot = 0; slot < nslots; ++slot) {
        const int qi = slot * TM_NT + tid;
        if (qi >= qcount) continue;
        const int pix = (q0 + qi) * 4;
        float xv[4], mv[4], xh[4];
        f4(sX[qi], xv);
        f4(a.pipeline ? *reinterpret_cast<const float4*>(Mg + (size_t)s * a.np + pix) : z4, mv);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          bad |= !isfinite(xv[e]);
          if (a.pipeline) {
            if (upd) mv[e] = __fadd_rn(mv[e], __fdiv_rn(__fsub_rn(xv[e], mv[e]), seen));
            xh[e] = __fdiv_rn(__fsub_rn(xv[e], mv[e]), stdv);
          } else {
            xh[e] = xv[e];
          }
          if (pix + e >= a.P) xh[e] = 0.f;
        }
        sX[qi] = make_float4(xh[0], xh[1], xh[2], xh[3]);
        if (upd) {
          *reinterpret_cast<float4*>(static_cast<float*>(a.mean) + (size_t)s * a.np + pix) =
              make_float4(mv[0], mv[1], mv[2], mv[3]);
        }
      }

      // ---- cold start y = U^T x (fit.py:86-87) -------------------------------
      if (cs->frame_index == 0) {
        float pk[K];
#pragma unroll
        for (int j = 0; j < K; ++j) pk[j] = 0.f;
        for (int slot = 0; slot < nslots; ++slot) {
          const int qi = slot * TM_NT + tid;
          float xh[4];
          f4(qi < qcount ? sX[qi] : z4, xh);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            float u[RS];
            load_row(slot, e, u);
#pragma unroll
            for (int j = 0; j < K; ++j) pk[j] += u[j] * xh[e];
          }
        }
        stage_floats<K>(pk, wred, K + 1, 0);
        rstage(bad ? 1.0 : 0.0, wred, K, K + 1);
        team_sum(ra, team, rank, wred, K + 1, red, epoch, sprof);
        if (tid < 32) {
          if (red[K] > 0.0) mark_nonfinite(cs, a, s, tid);
          else if (tid < k) cs->y[tid] = red[tid];
          __syncwarp();
          SYNC_FLOATS();
        }
        __syncthreads();
      }
    }

    PHASE_MARK(PROF_T_STATS);
    if (cs->status == ST_OK) {
      // ---- pass 0: r = x - U y, cost, coordinate gradient (fit.py:96-104) ---
      {
        double cost = 0.0;
        float pk[K + 1];
#pragma unroll
        for (int j = 0; j <= K; ++j) pk[j] = 0.f;
        for (int slot = 0; slot < nslots; ++slot) {
          const int qi = slot * TM_NT + tid;
          float xh[4], w[4], r[4];
          f4(qi < qcount ? sX[qi] : z4, xh);
          weights(qi, w);
          float tc = 0.f;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            float u[RS];
            load_row(slot, e, u);
            const float uy = dotk<K>(u, sfv[0]);
            r[e] = __fsub_rn(xh[e], uy);
            float tw, g;
            penalty_t<PM>(r[e], w[e], a, tw, g);
            tc += tw;
            pk[K] += g * g;
#pragma unroll
            for (int j = 0; j < K; ++j) pk[j] += u[j] * g;
          }
          cost += (double)tc;
          if (qi < qcount) sR[qi] = make_float4(r[0], r[1], r[2], r[3]);
        }
        rstage(cost, wred, 0, K + 3);
        stage_floats<K + 1>(pk, wred, K + 3, 1);
        rstage(bad ? 1.0 : 0.0, wred, K + 2, K + 3);
        team_sum(ra, team, rank, wred, K + 3, red, epoch, sprof);
        LOGIC(after_pass0<K>(cs, a, s, tid, red));
        __syncthreads();
      }
      PHASE_MARK(PROF_T_PASS0);

      // ---- CG iterations (fit.py:108-144) -----------------------------------
      while (cs->status == ST_OK && cs->active) {
        if (cs->need_lsfb) {
          const int base = cs->ls_next;
          const int cnt = (a.max_bt - base) < LSW ? (a.max_bt - base) : LSW;
          const double al0 = alpha_at(a, base);
          float cst[LSW];
#pragma unroll
          for (int m = 0; m < LSW; ++m) cst[m] = 0.f;
          for (int slot = 0; slot < nslots; ++slot) {
            const int qi = slot * TM_NT + tid;
            if (qi >= qcount) continue;
            float r[4], ud[4], w[4];
            f4(sR[qi], r);
            f4(sD[qi], ud);
            weights(qi, w);
            double al = al0;
#pragma unroll
            for (int m = 0; m < LSW; ++m) {
              if (m < cnt) {
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  float tw, g;
                  penalty_t<PM>(trial(r[e], (float)al, ud[e]), w[e], a, tw, g);
                  cst[m] += tw;
                }
              }
              al *= a.shrink;
            }
          }
#pragma unroll
          for (int m = 0; m < LSW; ++m) rstage((double)cst[m], wred, m, LSW);
          team_sum(ra, team, rank, wred, LSW, red, epoch, sprof);
          LOGIC(after_lsfb(cs, a, s, tid, red, base));
        } else if (cs->need_gradfb) {
          const float al = (float)cs->acc_alpha;
          float pk[K + 1];
#pragma unroll
          for (int j = 0; j <= K; ++j) pk[j] = 0.f;
          for (int slot = 0; slot < nslots; ++slot) {
            const int qi = slot * TM_NT + tid;
            float r[4], ud[4], w[4];
            f4(qi < qcount ? sR[qi] : z4, r);
            f4(qi < qcount ? sD[qi] : z4, ud);
            weights(qi, w);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              float u[RS];
              load_row(slot, e, u);
              float tw, g;
              penalty_t<PM>(trial(r[e], al, ud[e]), w[e], a, tw, g);
              pk[K] += g * g;
#pragma unroll
              for (int j = 0; j < K; ++j) pk[j] += u[j] * g;
            }
          }
          stage_floats<K + 1>(pk, wred, K + 1, 0);
          team_sum(ra, team, rank, wred, K + 1, red, epoch, sprof);
          LOGIC(after_gradfb<K>(cs, a, s, tid, red));
        } else {
          constexpr int NV = WC + WG * (K + 1);
          const int wlo = cs->gwin_lo;
          float al[WC];
          {
            double v = a.step0;
#pragma unroll
            for (int m = 0; m < WC; ++m) {
              al[m] = (float)v;
              v *= a.shrink;
            }
          }
          float cst[WC];
          float pk[WG * (K + 1)];
#pragma unroll
          for (int m = 0; m < WC; ++m) cst[m] = 0.f;
#pragma unroll
          for (int i = 0; i < WG * (K + 1); ++i) pk[i] = 0.f;
          for (int slot = 0; slot < nslots; ++slot) {
            const int qi = slot * TM_NT + tid;
            float r[4], w[4], ud[4];
            f4(qi < qcount ? sR[qi] : z4, r);
            weights(qi, w);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              float u[RS];
              load_row(slot, e, u);
              const float d = dotk<K>(u, sfv[1]);
              ud[e] = d;
              // trial costs for every window step; the gradient only for the
              // speculative pair (same arithmetic as penalty_t, split)
              float ts[WG], hs[WG], es[WG];
#pragma unroll
              for (int mm = 0; mm < WG; ++mm) ts[mm] = hs[mm] = es[mm] = 0.f;
#pragma unroll
              for (int m = 0; m < WC; ++m) {
                const float t = trial(r[e], al[m], d);
                if (PM == PM_HALF) {
                  const float b = fmaf(t, t, a.muf);
                  const float h = rsqrtf(b);
                  const float q = rsqrtf(h);
                  cst[m] += q * w[e];
#pragma unroll
                  for (int mm = 0; mm < WG; ++mm) {
                    const bool sel = m == wlo + mm;
                    ts[mm] = sel ? t : ts[mm];
                    hs[mm] = sel ? h : hs[mm];
                    es[mm] = sel ? q : es[mm];
                  }
                } else {
                  float tw, g;
                  penalty_t<PM>(t, w[e], a, tw, g);
                  cst[m] += tw;
#pragma unroll
                  for (int mm = 0; mm < WG; ++mm) {
                    const bool sel = m == wlo + mm;
                    ts[mm] = sel ? g : ts[mm];
                  }
                }
              }
              float gs[WG];
#pragma unroll
              for (int mm = 0; mm < WG; ++mm)
                gs[mm] = PM == PM_HALF ? 0.5f * ts[mm] * (es[mm] * w[e]) * (hs[mm] * hs[mm]) : ts[mm];
#pragma unroll
              for (int mm = 0; mm < WG; ++mm) {
                pk[mm * (K + 1) + K] += gs[mm] * gs[mm];
#pragma unroll
                for (int j = 0; j < K; ++j) pk[mm * (K + 1) + j] += u[j] * gs[mm];
              }
            }
            if (qi < qcount) sD[qi] = make_float4(ud[0], ud[1], ud[2], ud[3]);
          }
#pragma unroll
          for (int m = 0; m < WC; ++m) rstage((double)cst[m], wred, m, NV);
          stage_floats<WG * (K + 1)>(pk, wred, NV, WC);
          team_sum(ra, team, rank, wred, NV, red, epoch, sprof);
          LOGIC(after_iter<K>(cs, a, s, tid, red, wlo));
        }
        __syncthreads();
        // apply an accepted step to the residual kept in shared memory
        const float pa = (float)cs->pend_alpha;
        if (pa != 0.f) {
          for (int slot = 0; slot < nslots; ++slot) {
            const int qi = slot * TM_NT + tid;
            if (qi >= qcount) continue;
            float r[4], ud[4];
            f4(sR[qi], r);
            f4(sD[qi], ud);
#pragma unroll
            for (int e = 0; e < 4; ++e) r[e] = trial(r[e], pa, ud[e]);
            sR[qi] = make_float4(r[0], r[1], r[2], r[3]);
          }
        }
        __syncthreads();
        if (tid == 0) cs->pend_alpha = 0.0;
        __syncthreads();
      }
    }
    PHASE_MARK(PROF_T_ITER);

    if (cs->status == ST_OK) {
      // ---- geodesic step + relabel (manifold.py:116-197, tracker.py:146-147) ---
      // With a re-orthonormalization due (every 1000th step) U' is written back
      // unlabeled; the streamed k_gram / k_geo<QR> kernels that follow every
      // launch apply U' R^-1 and relabel (manifold.py:192-196).
      const bool geo = cs->do_geo != 0, qr = geo && cs->qr_now != 0;
      const float ga = (float)cs->geo_a, gsn = (float)cs->geo_s, ln = (float)cs->geo_ln;
      float* Ug = static_cast<float*>(a.U) + (size_t)s * k * a.np;
      for (int slot = 0; slot < nslots; ++slot) {
        const int qi = slot * TM_NT + tid;
        const bool ok = qi < qcount;
        const int pix = (q0 + qi) * 4;
        float r[4], w[4];
        f4(ok ? sR[qi] : z4, r);
        weights(qi, w);
        float up[4][K];  // U' rows of this row group
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float u[RS];
          load_row(slot, e, u);
          float coef = 0.f;
          if (geo) {
            float tw, g;
            penalty_t<PM>(r[e], w[e], a, tw, g);
            const float eta = -g;  // cost.py:103-112
            const float uv = dotk<K>(u, sfv[2]);
            const float ug = dotk<K>(u, sfv[3]);
            coef = ga * uv - gsn * ((eta - ug) / ln);
          }
#pragma unroll
          for (int j = 0; j < K; ++j) up[e][j] = u[j] + coef * sfv[2][j];
        }
        if (!ok) continue;
        if (geo) {
#pragma unroll
          for (int j = 0; j < K; ++j)
            if (j < k)
              __stcs(reinterpret_cast<float4*>(Ug + (size_t)j * a.np + pix),
                     make_float4(up[0][j], up[1][j], up[2][j], up[3][j]));
        }
        if (qr) continue;
        const size_t off = (size_t)s * a.np + pix;
        float xh[4], bgn[4], rr[4];
        f4(sX[qi], xh);
        uint32_t nl = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float acc = dotk<K>(up[e], sfv[0]);
          bgn[e] = acc;
          rr[e] = __fsub_rn(xh[e], acc);
          if (pix + e < a.P && fabs((double)rr[e]) >= a.delta) nl |= 1u << (8 * e);
        }
        *reinterpret_cast<uint32_t*>(a.lab + (size_t)s * a.Pp + pix) = nl;
        if (a.raw_out) *reinterpret_cast<uint32_t*>(a.raw_out + (size_t)s * a.Pp + pix) = nl;
        if (a.res_out)
          *reinterpret_cast<float4*>(static_cast<float*>(a.res_out) + off) = make_float4(rr[0], rr[1], rr[2], rr[3]);
        if (a.bg_out) {
          const float sc = (float)cs->std_cur;
          float m4[4], b[4];
          f4(a.pipeline ? *reinterpret_cast<const float4*>(Mg + off) : z4, m4);
#pragma unroll
          for (int e = 0; e < 4; ++e)
            b[e] = a.pipeline ? fminf(fmaxf(__fadd_rn(bgn[e] * sc, m4[e]), 0.f), 1.f) : bgn[e];
          *reinterpret_cast<float4*>(static_cast<float*>(a.bg_out) + off) = make_float4(b[0], b[1], b[2], b[3]);
        }
      }
    }

    // ---- commit the control block (one writer per stream) ------------------
    __syncthreads();
    PHASE_MARK(PROF_T_GEO);
#undef PHASE_MARK
    if (rank == 0 && tid < (int)(sizeof(Ctl) / 8))
      reinterpret_cast<double*>(a.ctl + s)[tid] = reinterpret_cast<const double*>(cs)[tid];
    __syncthreads();
  }
#undef LOGIC
#undef SYNC_FLOATS
  if (ra.prof && tid == 0) {
    sprof[PROF_TOTAL] = gtimer() - t_start;
    for (int i = 0; i < PROF_N; ++i) ra.prof[(size_t)blockIdx.x * PROF_N + i] = sprof[i];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_tbase), "n"(TM_NT));
}

}  // namespace prost
