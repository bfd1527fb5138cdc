// prost_resident.cuh — the register-resident frame kernel.
//
// The streamed phase kernels read U once per reduction (pass 0, every CG
// iteration, the geodesic) — 4 reads + 1 write of the n x k basis per frame.
// Here U crosses HBM exactly once in each direction per frame: a persistent,
// cooperatively launched grid is split into T teams of G CTAs (one CTA per
// SM); a team owns one stream per round, each CTA a contiguous slice of its
// rows, each thread ONE group of 4 rows whose k x 4 basis values stay in
// registers for every phase of the frame.  The chain of dependent reductions
// (statistics, pass 0, CG iterations, Armijo fallbacks, periodic Gram) runs
// as team-wide reductions: CTA partials -> global slots (double-buffered) ->
// a team barrier (release/acquire counter) -> every CTA sums the G slots in
// slot order and runs the scalar logic itself, so all CTAs of a team hold
// bit-identical control blocks without a second barrier.  While a team
// computes stream s, one thread streams the next stream's slice (U planes,
// frame, running mean) into shared memory with TMA bulk copies
// (cp.async.bulk + mbarrier complete_tx), so the HBM reads of round i+1
// overlap the reductions of round i; U' is written back from registers.
#pragma once

#include "prost_phases.cuh"

namespace prost {

struct RArgs {
  int G;            // CTAs per team
  int T;            // teams in the grid
  int qpc;          // row groups (4 rows) per CTA, multiple of 4
  int rnv;          // slot stride (doubles)
  unsigned* bar;    // [T] barrier counters, zeroed before every launch
  double* rpart;    // [2][T][rnv][G] reduction slots (value-major)
  int S;            // streams
  unsigned long long* prof;  // [gridDim][8] optional timing counters (ns), or null
  int stagger_ns;            // start delay of odd teams (k_tmem), 0 = none
  int prefetch;              // k_tmem: L2 prefetch of the slots after the first of a CTA's slice
  int alt;                   // k_tmem with 2 slot groups: alternate the groups' slice loads
  int median;                // k_tmem cluster teams: the 3x3 label median in-kernel (mask_out)
};

// Timing counters of one CTA (thread 0, %globaltimer ns): see PROF_* below.
enum {
  PROF_TOTAL = 0, PROF_BARRIER, PROF_SLOTS, PROF_LOGIC, PROF_PREFETCH, PROF_NSUMS, PROF_ROUNDS,
  PROF_T_STATS, PROF_T_PASS0, PROF_T_ITER, PROF_T_GEO,  // phase wall times (k_tmem)
  PROF_GT_TOTAL,  // kernel time in %globaltimer ns (the others count SM clocks)
  PROF_SW_OWN,    // k_tmem CG iteration sweeps: thread 0's own sweep + staging
  PROF_SW_ALL,    //   ... until every warp of the CTA has staged its partials
  PROF_LOGIC_ITER,  // k_tmem: scalar logic after the CG iteration sweeps only
  PROF_N = 16
};

// Profiling clock: SM cycles (the ~1 us tick of %globaltimer is too coarse for
// sub-microsecond phases); the host converts with PROF_TOTAL / PROF_GT_TOTAL.
__device__ __forceinline__ unsigned long long ptimer() { return clock64(); }

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

constexpr int RES_RNV_MAX = 16 * 17 / 2 + 8;  // Gram of K = 16 dominates

// --------------------------------------------------------------------------
// PTX helpers: mbarrier, TMA bulk copy, acquire/release counter

__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  unsigned done = 0;
  long long spins = 0;
  while (true) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
    if (done) break;
    if (++spins > (1LL << 26)) __trap();
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// All CTAs of a team: arrive on the counter, wait until `target` arrivals.
// (Co-residency is guaranteed by the cooperative launch; a stuck barrier
// traps instead of hanging the device.)
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void team_barrier(unsigned* ctr, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    red_release_add(ctr, 1u);
    long long spins = 0;
    while (ld_acquire(ctr) < target) {
      if (++spins > (1LL << 26)) __trap();
    }
  }
  __syncthreads();
}

// Per-CTA staged values (wred[warp][nv]) -> team sum into red[nv], identical
// in every CTA of the team.  Slots are value-major ([v][rank]) so that one
// warp reads all ranks of a value in a single coalesced round trip; the sum
// order (rank partials by lane, then a butterfly) is fixed.
__device__ __forceinline__ void team_sum(const RArgs& ra, int team, int rank, const double* wred,
                                         int nv, double* red, unsigned& epoch,
                                         unsigned long long* sprof) {
  __syncthreads();
  const bool tp = ra.prof && threadIdx.x == 0;
  unsigned long long t0 = tp ? ptimer() : 0;
  const int nwarp = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = ra.G;
  const int par = epoch & 1;
  double* area = ra.rpart + ((size_t)par * ra.T + team) * (size_t)ra.rnv * G;
  for (int v = threadIdx.x; v < nv; v += blockDim.x) {
    double acc = 0.0;
    for (int w = 0; w < nwarp; ++w) acc += wred[w * nv + v];
    area[(size_t)v * G + rank] = acc;
  }
  ++epoch;
  team_barrier(ra.bar + team, epoch * (unsigned)G);
  unsigned long long t1 = tp ? ptimer() : 0;
  for (int v0 = warp; v0 < nv; v0 += 4 * nwarp) {
    double acc[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      acc[i] = 0.0;
      const int v = v0 + i * nwarp;
      if (v < nv) {
        const double* b = area + (size_t)v * G;
#pragma unroll
        for (int c = 0; c < 5; ++c)  // G <= 160: up to 5 independent loads per lane
          if (lane + 32 * c < G) acc[i] += __ldcg(b + lane + 32 * c);
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const double t = warp_sum(acc[i]);
      const int v = v0 + i * nwarp;
      if (lane == 0 && v < nv) red[v] = t;
    }
  }
  __syncthreads();
  if (tp) {
    const unsigned long long t2 = ptimer();
    sprof[PROF_BARRIER] += t1 - t0;
    sprof[PROF_SLOTS] += t2 - t1;
    sprof[PROF_NSUMS] += 1;
  }
}

// One double per lane -> its warp sum in wred[warp][slot].
__device__ __forceinline__ void rstage(double x, double* wred, int slot, int nv) {
  x = warp_sum(x);
  if ((threadIdx.x & 31) == 0) wred[(threadIdx.x >> 5) * nv + slot] = x;
}

// 32 floats per lane -> lane L ends with the warp sum of value L (butterfly
// reduce-scatter: 31 shuffles instead of 32 x 5).
template <int OFF>
__device__ __forceinline__ void rs_step(float (&v)[32], int lane) {
  const bool up = (lane & OFF) != 0;
#pragma unroll
  for (int i = 0; i < OFF; ++i) {
    const float keep = up ? v[i + OFF] : v[i];
    const float send = up ? v[i] : v[i + OFF];
    v[i] = keep + __shfl_xor_sync(0xffffffffu, send, OFF);
  }
}
__device__ __forceinline__ float warp_reduce_scatter32(float (&v)[32]) {
  // compile-time offsets keep v[] in registers
  const int lane = threadIdx.x & 31;
  rs_step<16>(v, lane);
  rs_step<8>(v, lane);
  rs_step<4>(v, lane);
  rs_step<2>(v, lane);
  rs_step<1>(v, lane);
  return v[0];
}

// N floats per lane -> warp sums in wred[warp][base .. base+N).
template <int N>
__device__ __forceinline__ void stage_floats(const float (&v)[N], double* wred, int nv, int base) {
#pragma unroll
  for (int c0 = 0; c0 < N; c0 += 32) {
    float t[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) t[i] = (c0 + i < N) ? v[c0 + i] : 0.f;
    const float r = warp_reduce_scatter32(t);
    const int lane = threadIdx.x & 31;
    if (c0 + lane < N) wred[(threadIdx.x >> 5) * nv + base + c0 + lane] = (double)r;
  }
}

// --------------------------------------------------------------------------

// Dynamic shared memory of k_resident<K> for `qpc` row groups and `nwarp` warps:
// prefetch buffer (K basis planes + frame + mean) + current frame/mean
// + reduction staging + control block + Cholesky scratch + mbarrier.
template <int K>
__host__ __device__ constexpr size_t resident_smem(int qpc, int nwarp) {
  return (size_t)(K + 4) * qpc * 16 + (size_t)(nwarp + 1) * RES_RNV_MAX * 8 + sizeof(Ctl) +
         (size_t)2 * K * K * 8 + 16;
}

template <int K, int NTMAX, int PM>
__global__ void __launch_bounds__(NTMAX, 1) k_resident(const __grid_constant__ Args a, const __grid_constant__ RArgs ra) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  const int G = ra.G, T = ra.T, qpc = ra.qpc;
  const int team = blockIdx.x / G, rank = blockIdx.x - team * G;
  const int tid = threadIdx.x, nwarp = blockDim.x >> 5;
  const int k = a.k;
  const int nq = a.Pp / 4;
  const int q0 = rank * qpc;
  const int qcount = max(0, min(qpc, nq - q0));
  const bool own = tid < qcount;
  const int pix = (q0 + tid) * 4;  // first of this thread's 4 pixels (C == 1)

  // shared memory carve-up
  float4* pU = reinterpret_cast<float4*>(smem_raw);  // [K][qpc] prefetched basis slice
  float4* pX = pU + (size_t)K * qpc;                 // [qpc] prefetched frame slice
  float4* pM = pX + qpc;                             // [qpc] prefetched running mean
  float4* cX = pM + qpc;                             // [qpc] normalized frame of this round
  float4* cM = cX + qpc;                             // [qpc] running mean of this round
  double* wred = reinterpret_cast<double*>(cM + qpc);  // [nwarp][RES_RNV_MAX]
  double* red = wred + (size_t)nwarp * RES_RNV_MAX;    // [RES_RNV_MAX]
  Ctl* cs = reinterpret_cast<Ctl*>(red + RES_RNV_MAX);
  double* rinv = reinterpret_cast<double*>(cs + 1);  // [K*K]
  double* Rm = rinv + K * K;                          // [K*K]
  uint64_t* mbar = reinterpret_cast<uint64_t*>(Rm + K * K);

  unsigned epoch = 0;
  __shared__ unsigned long long sprof[PROF_N];
  if (tid < PROF_N) sprof[tid] = 0;
  const unsigned long long t_start = ptimer(), g_start = gtimer();
#define LOGIC(call)                                                    \
  do {                                                                 \
    const unsigned long long tl0 = (ra.prof && tid == 0) ? ptimer() : 0; \
    if (tid < 32) call;                                                \
    if (ra.prof && tid == 0) sprof[PROF_LOGIC] += ptimer() - tl0;      \
  } while (0)

  if (tid == 0) mbar_init(mbar, 1);
  __syncthreads();

  auto issue = [&](int s) {
    const unsigned row_bytes = (unsigned)qcount * 16u;
    const unsigned planes = (unsigned)k + 1u + (a.pipeline ? 1u : 0u);
    mbar_expect_tx(mbar, row_bytes * planes);
    const float* U = static_cast<const float*>(a.U) + (size_t)s * k * a.np + (size_t)q0 * 4;
    for (int j = 0; j < k; ++j) bulk_g2s(pU + (size_t)j * qpc, U + (size_t)j * a.np, row_bytes, mbar);
    bulk_g2s(pX, static_cast<const float*>(a.x) + (size_t)s * a.np + (size_t)q0 * 4, row_bytes, mbar);
    if (a.pipeline)
      bulk_g2s(pM, static_cast<const float*>(a.mean) + (size_t)s * a.np + (size_t)q0 * 4, row_bytes, mbar);
  };
  if (tid == 0 && qcount > 0 && team < ra.S) issue(team);

  int round = 0;
  for (int s = team; s < ra.S; s += T, ++round) {
    // ---- stage the prefetched slice into registers -------------------------
    {
      const unsigned long long tw0 = (ra.prof && tid == 0) ? ptimer() : 0;
      if (qcount > 0) mbar_wait(mbar, round & 1);
      if (ra.prof && tid == 0) {
        sprof[PROF_PREFETCH] += ptimer() - tw0;
        sprof[PROF_ROUNDS] += 1;
      }
    }
    float u[K][4];
    float xr[4] = {0.f, 0.f, 0.f, 0.f}, mr[4] = {0.f, 0.f, 0.f, 0.f};
    uint32_t lbits = 0;  // label bytes of the 4 pixels (1 = foreground)
    if (own) {
#pragma unroll
      for (int j = 0; j < K; ++j) {
        if (j < k) {
          const float4 t = pU[(size_t)j * qpc + tid];
          u[j][0] = t.x; u[j][1] = t.y; u[j][2] = t.z; u[j][3] = t.w;
        } else {
          u[j][0] = u[j][1] = u[j][2] = u[j][3] = 0.f;
        }
      }
      const float4 tx = pX[tid];
      xr[0] = tx.x; xr[1] = tx.y; xr[2] = tx.z; xr[3] = tx.w;
      if (a.pipeline) {
        const float4 tm = pM[tid];
        mr[0] = tm.x; mr[1] = tm.y; mr[2] = tm.z; mr[3] = tm.w;
      }
      lbits = *reinterpret_cast<const uint32_t*>(a.lab + (size_t)s * a.Pp + pix);
    } else {
#pragma unroll
      for (int j = 0; j < K; ++j) u[j][0] = u[j][1] = u[j][2] = u[j][3] = 0.f;
    }
    if (tid < (int)(sizeof(Ctl) / 8))
      reinterpret_cast<double*>(cs)[tid] = __ldcg(reinterpret_cast<const double*>(a.ctl + s) + tid);
    __syncthreads();
    if (tid == 0) cs->no_info = rank != 0;  // one FitInfo writer per stream
    __syncthreads();  // prefetch buffer consumed, control block staged
    if (tid == 0 && qcount > 0 && s + T < ra.S) {
      fence_proxy_async();
      issue(s + T);
    }
    const float omega = (float)a.omega;
    auto weight = [&](int e) -> float {
      return (own && pix + e < a.P) ? (((lbits >> (8 * e)) & 0xffu) ? omega : 1.f) : 0.f;
    };

    // ---- frame start: running statistics (pipeline.py:120-140) ------------
    const bool upd = a.pipeline && !cs->frozen && cs->frame_index < a.i_init;
    if (upd) {
      double s1 = 0.0, s2 = 0.0, nf = 0.0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (own && pix + e < a.P) {
          const double v = (double)xr[e];
          s1 += v;
          s2 += v * v;
          nf += isfinite(v) ? 0.0 : 1.0;
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

    bool bad = false;
    if (cs->status == ST_OK) {
      const float stdv = (float)cs->std_cur;
      const float seen = (float)cs->pseen;
      float xh[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        bad |= !isfinite(xr[e]);
        if (a.pipeline) {
          if (upd) mr[e] = __fadd_rn(mr[e], __fdiv_rn(__fsub_rn(xr[e], mr[e]), seen));
          xh[e] = __fdiv_rn(__fsub_rn(xr[e], mr[e]), stdv);
        } else {
          xh[e] = xr[e];
        }
        if (!(own && pix + e < a.P)) xh[e] = 0.f;
      }
      if (own) {
        cX[tid] = make_float4(xh[0], xh[1], xh[2], xh[3]);
        cM[tid] = make_float4(mr[0], mr[1], mr[2], mr[3]);
      }
      if (upd && own) {
        *reinterpret_cast<float4*>(static_cast<float*>(a.mean) + (size_t)s * a.np + pix) =
            make_float4(mr[0], mr[1], mr[2], mr[3]);
      }

      // ---- cold start y = U^T x (fit.py:86-87) ------------------------------
      if (cs->frame_index == 0) {
        float acc[K];
#pragma unroll
        for (int j = 0; j < K; ++j) {
          acc[j] = 0.f;
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[j] += u[j][e] * xh[e];
        }
        stage_floats<K>(acc, wred, K + 1, 0);
        rstage(bad ? 1.0 : 0.0, wred, K, K + 1);
        team_sum(ra, team, rank, wred, K + 1, red, epoch, sprof);
        if (tid < 32) {
          if (red[K] > 0.0) mark_nonfinite(cs, a, s, tid);
          else if (tid < k) cs->y[tid] = red[tid];
        }
        __syncthreads();
      }

      // ---- pass 0: r = x - U y, cost, coordinate gradient (fit.py:96-104) ---
      float r[4] = {0.f, 0.f, 0.f, 0.f}, ud[4] = {0.f, 0.f, 0.f, 0.f};
      if (cs->status == ST_OK) {
        double cost = 0.0;
        float g[4];
        float pk[K + 1];
        pk[K] = 0.f;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float uy = 0.f;
#pragma unroll
          for (int j = 0; j < K; ++j) uy += u[j][e] * (float)cs->y[j];
          r[e] = __fsub_rn(xh[e], uy);
          float tw;
          penalty_t<PM>(r[e], weight(e), a, tw, g[e]);
          cost += (double)tw;
          pk[K] += g[e] * g[e];
        }
#pragma unroll
        for (int j = 0; j < K; ++j) {
          pk[j] = 0.f;
#pragma unroll
          for (int e = 0; e < 4; ++e) pk[j] += u[j][e] * g[e];
        }
        rstage(cost, wred, 0, K + 3);
        stage_floats<K + 1>(pk, wred, K + 3, 1);
        rstage(bad ? 1.0 : 0.0, wred, K + 2, K + 3);
        team_sum(ra, team, rank, wred, K + 3, red, epoch, sprof);
        LOGIC(after_pass0<K>(cs, a, s, tid, red));
        __syncthreads();
      }

      // ---- CG iterations (fit.py:108-144) -----------------------------------
      while (cs->status == ST_OK && cs->active) {
        if (cs->need_lsfb) {
          const int base = cs->ls_next;
          const int cnt = (a.max_bt - base) < LSW ? (a.max_bt - base) : LSW;
          double al = alpha_at(a, base);
          for (int m = 0; m < LSW; ++m) {
            double cost = 0.0;
            if (m < cnt) {
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                float tw, g;
                penalty_t<PM>(trial(r[e], (float)al, ud[e]), weight(e), a, tw, g);
                cost += (double)tw;
              }
            }
            rstage(cost, wred, m, LSW);
            al *= a.shrink;
          }
          team_sum(ra, team, rank, wred, LSW, red, epoch, sprof);
          LOGIC(after_lsfb(cs, a, s, tid, red, base));
        } else if (cs->need_gradfb) {
          const float al = (float)cs->acc_alpha;
          float g[4], pk[K + 1];
          pk[K] = 0.f;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            float tw;
            penalty_t<PM>(trial(r[e], al, ud[e]), weight(e), a, tw, g[e]);
            pk[K] += g[e] * g[e];
          }
#pragma unroll
          for (int j = 0; j < K; ++j) {
            pk[j] = 0.f;
#pragma unroll
            for (int e = 0; e < 4; ++e) pk[j] += u[j][e] * g[e];
          }
          stage_floats<K + 1>(pk, wred, K + 1, 0);
          team_sum(ra, team, rank, wred, K + 1, red, epoch, sprof);
          LOGIC(after_gradfb<K>(cs, a, s, tid, red));
        } else {
          constexpr int NV = WC + WG * (K + 1);
          const int wlo = cs->gwin_lo;
#pragma unroll
          for (int e = 0; e < 4; ++e) ud[e] = 0.f;
#pragma unroll
          for (int j = 0; j < K; ++j) {
            const float dj = (float)cs->d[j];
#pragma unroll
            for (int e = 0; e < 4; ++e) ud[e] += u[j][e] * dj;
          }
          float gs[WG][4];
          double al = a.step0;
#pragma unroll
          for (int m = 0; m < WC; ++m) {
            double cost = 0.0;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              float tw, g;
              penalty_t<PM>(trial(r[e], (float)al, ud[e]), weight(e), a, tw, g);
              cost += (double)tw;
#pragma unroll
              for (int mm = 0; mm < WG; ++mm)
                if (m == wlo + mm) gs[mm][e] = g;
            }
            rstage(cost, wred, m, NV);
            al *= a.shrink;
          }
          float pk[WG * (K + 1)];
#pragma unroll
          for (int mm = 0; mm < WG; ++mm) {
            float gsq = 0.f;
#pragma unroll
            for (int e = 0; e < 4; ++e) gsq += gs[mm][e] * gs[mm][e];
            pk[mm * (K + 1) + K] = gsq;
#pragma unroll
            for (int j = 0; j < K; ++j) {
              float acc = 0.f;
#pragma unroll
              for (int e = 0; e < 4; ++e) acc += u[j][e] * gs[mm][e];
              pk[mm * (K + 1) + j] = acc;
            }
          }
          stage_floats<WG * (K + 1)>(pk, wred, NV, WC);
          team_sum(ra, team, rank, wred, NV, red, epoch, sprof);
          LOGIC(after_iter<K>(cs, a, s, tid, red, wlo));
        }
        __syncthreads();
        // apply an accepted step to the register-resident residual
        const float pa = (float)cs->pend_alpha;
        if (pa != 0.f) {
#pragma unroll
          for (int e = 0; e < 4; ++e) r[e] = trial(r[e], pa, ud[e]);
        }
        __syncthreads();
        if (tid == 0) cs->pend_alpha = 0.0;
        __syncthreads();
      }

      if (cs->status == ST_OK) {
        if (a.fitres_out && own)  // FitResult.residual (fit.py:50-63)
          *reinterpret_cast<float4*>(static_cast<float*>(a.fitres_out) + (size_t)s * a.np + pix) =
              make_float4(r[0], r[1], r[2], r[3]);
        // ---- geodesic step of the basis (manifold.py:116-197) ---------------
        if (cs->do_geo) {
          const float ga = (float)cs->geo_a, gsn = (float)cs->geo_s, ln = (float)cs->geo_ln;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            float tw, g;
            penalty_t<PM>(r[e], weight(e), a, tw, g);
            const float eta = -g;  // cost.py:103-112
            float uv = 0.f, ug = 0.f;
#pragma unroll
            for (int j = 0; j < K; ++j) {
              uv += u[j][e] * (float)cs->v[j];
              ug += u[j][e] * (float)cs->grad[j];
            }
            const float coef = ga * uv - gsn * ((eta - ug) / ln);
#pragma unroll
            for (int j = 0; j < K; ++j) u[j][e] += coef * (float)cs->v[j];
          }
          if (cs->qr_now) {
            // periodic re-orthonormalization: Gram, Cholesky, U R^-1 (manifold.py:192-196)
            const int npair = k * (k + 1) / 2;
            int pr = 0;
#pragma unroll
            for (int ia = 0; ia < K; ++ia) {
#pragma unroll
              for (int ib = ia; ib < K; ++ib) {
                if (ib < k) {
                  double acc = 0.0;
#pragma unroll
                  for (int e = 0; e < 4; ++e) acc += (double)u[ia][e] * (double)u[ib][e];
                  rstage(acc, wred, pr, npair);
                  ++pr;
                }
              }
            }
            team_sum(ra, team, rank, wred, npair, red, epoch, sprof);
            if (tid == 0) {
              auto Gat = [&](int i, int j) {
                if (i > j) { const int t = i; i = j; j = t; }
                return red[i * k - i * (i - 1) / 2 + (j - i)];
              };
              for (int i = 0; i < K * K; ++i) { Rm[i] = 0.0; rinv[i] = 0.0; }
              for (int j = 0; j < k; ++j) {
                double dsum = Gat(j, j);
                for (int l = 0; l < j; ++l) dsum -= Rm[l * K + j] * Rm[l * K + j];
                const double rjj = sqrt(fmax(dsum, 1e-300));
                Rm[j * K + j] = rjj;
                for (int i = j + 1; i < k; ++i) {
                  double o = Gat(j, i);
                  for (int l = 0; l < j; ++l) o -= Rm[l * K + j] * Rm[l * K + i];
                  Rm[j * K + i] = o / rjj;
                }
              }
              for (int j = 0; j < k; ++j) {
                rinv[j * K + j] = 1.0 / Rm[j * K + j];
                for (int i = j - 1; i >= 0; --i) {
                  double o = 0.0;
                  for (int l = i + 1; l <= j; ++l) o += Rm[i * K + l] * rinv[l * K + j];
                  rinv[i * K + j] = -o / Rm[i * K + i];
                }
              }
              cs->since_qr = 0;
            }
            __syncthreads();
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              float nu[K];
#pragma unroll
              for (int j = 0; j < K; ++j) {
                nu[j] = 0.f;
#pragma unroll
                for (int l = 0; l <= j; ++l) nu[j] += u[l][e] * (float)rinv[l * K + j];
              }
#pragma unroll
              for (int j = 0; j < K; ++j) u[j][e] = nu[j];
            }
          }
          if (own) {
            float* U = static_cast<float*>(a.U) + (size_t)s * k * a.np + pix;
#pragma unroll
            for (int j = 0; j < K; ++j)
              if (j < k)
                __stcs(reinterpret_cast<float4*>(U + (size_t)j * a.np),
                       make_float4(u[j][0], u[j][1], u[j][2], u[j][3]));
          }
        }

        // ---- relabel against the updated basis (tracker.py:146-147) ---------
        if (own) {
          const float4 cx = cX[tid];
          const float xh2[4] = {cx.x, cx.y, cx.z, cx.w};
          float bgn[4], rr[4];
          uint32_t nl = 0;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            float acc = 0.f;
#pragma unroll
            for (int j = 0; j < K; ++j) acc += u[j][e] * (float)cs->y[j];
            bgn[e] = acc;
            rr[e] = __fsub_rn(xh2[e], acc);
            if (pix + e < a.P && fabs((double)rr[e]) >= a.delta) nl |= 1u << (8 * e);
          }
          const size_t off = (size_t)s * a.np + pix;
          *reinterpret_cast<uint32_t*>(a.lab + (size_t)s * a.Pp + pix) = nl;
          if (a.raw_out) *reinterpret_cast<uint32_t*>(a.raw_out + (size_t)s * a.Pp + pix) = nl;
          if (a.res_out)
            *reinterpret_cast<float4*>(static_cast<float*>(a.res_out) + off) =
                make_float4(rr[0], rr[1], rr[2], rr[3]);
          if (a.bg_out) {
            const float sc = (float)cs->std_cur;
            const float4 cm = cM[tid];
            const float m4[4] = {cm.x, cm.y, cm.z, cm.w};
            float b[4];
#pragma unroll
            for (int e = 0; e < 4; ++e)
              b[e] = a.pipeline ? fminf(fmaxf(__fadd_rn(bgn[e] * sc, m4[e]), 0.f), 1.f) : bgn[e];
            *reinterpret_cast<float4*>(static_cast<float*>(a.bg_out) + off) =
                make_float4(b[0], b[1], b[2], b[3]);
          }
        }
      }
    }

    // ---- commit the control block (one writer per stream) ------------------
    __syncthreads();
    if (rank == 0 && tid < (int)(sizeof(Ctl) / 8))
      reinterpret_cast<double*>(a.ctl + s)[tid] = reinterpret_cast<const double*>(cs)[tid];
    __syncthreads();
  }
  if (ra.prof && tid == 0) {
    sprof[PROF_TOTAL] = ptimer() - t_start;
    sprof[PROF_GT_TOTAL] = gtimer() - g_start;
    for (int i = 0; i < PROF_N; ++i) ra.prof[(size_t)blockIdx.x * PROF_N + i] = sprof[i];
  }
#undef LOGIC
}

}  // namespace prost
