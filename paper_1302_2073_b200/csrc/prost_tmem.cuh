// prost_tmem.cuh — the TMEM-resident frame kernel (k_tmem).
//
// A persistent grid split into T teams of G CTAs (one CTA per SM); a team owns
// one stream per round.  The frame's dependent reductions are team-wide sums
// through double-buffered global slots and a release/acquire counter barrier,
// after which every CTA runs the scalar logic itself (prost_resident.cuh).
//
// Where the basis lives: each thread owns row groups (4 rows x k values) in
// its lane of tensor memory (written once per frame with tcgen05.st, read one
// row at a time with tcgen05.ld in every phase) and, when the slice is larger,
// row groups in shared memory.  Per CTA that is 256 KB of TMEM + ~200 KB of
// shared memory, so a C3 stream (76,800 x 15 fp32 = 4.6 MB) fits on 12 SMs and
// 12 streams are in flight; U crosses HBM exactly once each way per frame.
//
// What is kept per row group besides U: the residual r and the last u_dir = U d
// (shared memory).  The frame itself is re-read from global memory (L2) by the
// two sweeps that need it (pass 0 and the relabel), so no copy is kept on chip.
// With k < 16 the per-coordinate weight w (1, omega, or 0 for padding) rides in
// the unused 16th TMEM / shared-memory column of each row.
//
// Instruction economy: the sweeps are compile-time loops over the 4 rows of a
// row group; TMEM and shared-memory row groups are separate loop instances; the
// CG iteration sweep is instantiated per speculative-gradient window position;
// an accepted step's residual update is applied by the next sweep that reads r.
#pragma once

#include <type_traits>

#include "prost_logic_fast.cuh"
// Timing counters (RArgs.prof, the bench's counters pass) only in the PROF
// instances: the timer values live across the sweeps, and in the 128-register
// kernel they cost spills (stack 152 -> 128 B, C3 1.143 -> 1.109 ms per step)
#define TM_PROF_ON(r) (PROF && (r).prof != nullptr)
#ifndef PROST_FAST_LOGIC
#define PROST_FAST_LOGIC 1
#endif
#if PROST_FAST_LOGIC
#if PROST_OLD_PASS0
#define TM_AFTER_PASS0 after_pass0
#else
#define TM_AFTER_PASS0 fl_after_pass0
#endif
#if PROST_OLD_ITER
#define TM_AFTER_ITER after_iter
#else
#define TM_AFTER_ITER fl_after_iter
#endif
#define TM_AFTER_LSFB fl_after_lsfb
#define TM_AFTER_GRADFB fl_after_gradfb
#else
#define TM_AFTER_PASS0 after_pass0
#define TM_AFTER_ITER after_iter
#define TM_AFTER_LSFB after_lsfb
#define TM_AFTER_GRADFB after_gradfb
#endif
#include "prost_resident.cuh"
#include "tmem_io.cuh"

#ifndef PROST_TM_NT
#define PROST_TM_NT 512
#endif
#ifndef PROST_TM_CPS
#define PROST_TM_CPS 1
#endif
#ifndef PROST_DYN
#define PROST_DYN 1  // dynamic stream-to-team assignment (see the round loop)
#endif
#ifndef PROST_SKEW_PROBE
#define PROST_SKEW_PROBE 0
#endif
#ifndef PROST_RCP_STD
#define PROST_RCP_STD 1  // normalize with the reciprocal of the std (<= 1 ulp from x / std)
#endif


namespace prost {

// threads per CTA: 4 warps per 128-column TMEM block (one per lane quarter);
// the CTA allocates TM_NT columns.  TM_CPS CTAs may share an SM.
constexpr int TM_NT = PROST_TM_NT;
constexpr int TM_CPS = PROST_TM_CPS;
static_assert(TM_NT == 128 || TM_NT == 256 || TM_NT == 512, "TMEM allocation is TM_NT columns");

template <int K>
struct TmemGeom {
  // columns per row (power of two >= k: every tcgen05 access is width-aligned)
  static constexpr int RS = K <= 4 ? 4 : (K <= 8 ? 8 : (K <= 16 ? 16 : 32));
  static constexpr int QW = 4 * RS;     // columns per row group
  static constexpr int QT = 128 / QW;   // row groups per thread in TMEM
  static constexpr bool WCOL = K < RS;  // weight stored in column RS-1
  // values reduced per team sum (largest: the CG iteration sweep)
  static constexpr int NV0 = WC + WG * (K + 1);
  static constexpr int NV1 = LSW > K + 3 ? LSW : K + 3;
  static constexpr int NV = NV0 > NV1 ? NV0 : NV1;
};

// Dynamic shared memory of one slot group of k_tmem<K, PM, NG> (TM_NT / NG
// threads) for qpc row groups per CTA slice.
template <int K, int NG>
__host__ __device__ constexpr size_t tmem_group_smem(int qpc) {
  using Geo = TmemGeom<K>;
  constexpr int TG = TM_NT / NG;
  const int qs = qpc > Geo::QT * TG ? qpc - Geo::QT * TG : 0;
  const int qa = (qpc + TG - 1) / TG * TG;  // r / u_dir arrays cover whole slots
  return ((size_t)16 * Geo::RS * qs        // basis row groups kept in shared memory
          + (size_t)qa * 48                // r, u_dir, U y
          + (Geo::WCOL ? 0 : (size_t)qa * 4)  // label words
          + (size_t)(TG / 32 + 1) * Geo::NV * 8 + sizeof(Ctl) + 127) / 128 * 128;
}
template <int K, int NG = 1>
__host__ __device__ constexpr size_t tmem_smem(int qpc) {
  return NG * tmem_group_smem<K, NG>(qpc) + 64;
}

// Named barrier of one slot group (ids 1.., TG threads); NG == 1 uses the CTA barrier.
template <int NG>
__device__ __forceinline__ void group_sync(int g) {
  if constexpr (NG == 1) {
    __syncthreads();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "n"(TM_NT / NG) : "memory");
  }
}

// team_sum / rstage / stage_floats of one slot group: wred is the group's
// [TG/32][nv] staging, lt the thread within the group; the team's slots and
// barrier counter are those of virtual team vt.
// CL: the team is one thread-block cluster (one CTA per rank): the CTA sums
// stay in each CTA's shared memory, the hardware cluster barrier replaces the
// counter barrier, and every CTA reads its peers' sums over DSMEM — added in
// the same order as the global-slot path (lane = rank, then the warp
// butterfly), so both give the same bits.
constexpr int CL_NV = 64;
template <int NG, bool CL = false, bool PROF = false>
__device__ __forceinline__ void team_sum_g(const RArgs& ra, int vt, int VT, int rank, int g, int lt,
                                           const double* wred, int nv, double* red, unsigned& epoch,
                                           unsigned long long* sprof) {
  constexpr int TG = TM_NT / NG, NWG = TG / 32;
  if constexpr (CL) {
    static_assert(NG == 1, "cluster team sums: one slot group");
    __shared__ double cpart[2][CL_NV];
    __syncthreads();
    const bool tp = TM_PROF_ON(ra) && lt == 0;
    const unsigned long long t0 = tp ? ptimer() : 0;
    const int warp = lt >> 5, lane = lt & 31;
    const int par = epoch & 1;
    ++epoch;
    for (int v = lt; v < nv; v += TG) {
      double acc = 0.0;
      for (int w = 0; w < NWG; ++w) acc += wred[w * nv + v];
      cpart[par][v] = acc;
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    const unsigned long long t1 = tp ? ptimer() : 0;
    // every load in flight at once (nv <= 4 * NWG), then the butterflies
    for (int v0 = warp; v0 < nv; v0 += 4 * NWG) {
      double x[4];
      bool have[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int v = v0 + i * NWG;
        have[i] = v < nv && lane < ra.G;
        x[i] = 0.0;
        if (have[i]) {
          unsigned remote;
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_addr(&cpart[par][v])), "r"(lane));
          asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(x[i]) : "r"(remote) : "memory");
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        double acc = 0.0;
        if (have[i]) acc += x[i];
        const double t = warp_sum(acc);
        const int v = v0 + i * NWG;
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
    return;
  }
  group_sync<NG>(g);
  const bool tp = TM_PROF_ON(ra) && g == 0 && lt == 0;
  unsigned long long t0 = tp ? ptimer() : 0;
  const int warp = lt >> 5, lane = lt & 31;
  const int G = ra.G;
  const int par = epoch & 1;
  double* area = ra.rpart + ((size_t)par * VT + vt) * (size_t)ra.rnv * G;
  for (int v = lt; v < nv; v += TG) {
    double acc = 0.0;
    for (int w = 0; w < NWG; ++w) acc += wred[w * nv + v];
    area[(size_t)v * G + rank] = acc;
  }
  ++epoch;
  group_sync<NG>(g);
  if (lt == 0) {
    unsigned* ctr = ra.bar + vt;
    const unsigned target = epoch * (unsigned)G;
#if PROST_SKEW_PROBE
    // experiment build: the last CTA to arrive times the bare round trip
    // (PROF_SW_OWN / PROF_SW_ALL are repurposed)
    unsigned old;
    asm volatile("atom.release.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(ctr) : "memory");
    const bool last_in = old + 1 == target;
#else
    red_release_add(ctr, 1u);
#endif
    long long spins = 0;
    while (ld_acquire(ctr) < target) {
      if (++spins > (1LL << 26)) __trap();
    }
#if PROST_SKEW_PROBE
    if (tp && last_in) {
      sprof[PROF_SW_OWN] += ptimer() - t0;
      sprof[PROF_SW_ALL] += 1000;
    }
#endif
  }
  group_sync<NG>(g);
  unsigned long long t1 = tp ? ptimer() : 0;
  for (int v0 = warp; v0 < nv; v0 += 4 * NWG) {
    double acc[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      acc[i] = 0.0;
      const int v = v0 + i * NWG;
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
      const int v = v0 + i * NWG;
      if (lane == 0 && v < nv) red[v] = t;
    }
  }
  group_sync<NG>(g);
  if (tp) {
    const unsigned long long t2 = ptimer();
    sprof[PROF_BARRIER] += t1 - t0;
    sprof[PROF_SLOTS] += t2 - t1;
    sprof[PROF_NSUMS] += 1;
  }
}

// One double per lane -> its warp sum in wred[lwarp][slot].
__device__ __forceinline__ void rstage_g(double x, double* wred, int slot, int nv, int lt) {
  x = warp_sum(x);
  if ((lt & 31) == 0) wred[(lt >> 5) * nv + slot] = x;
}

// N floats per lane -> warp sums in wred[lwarp][base .. base+N).
template <int N>
__device__ __forceinline__ void stage_floats_g(const float (&v)[N], double* wred, int nv, int base,
                                               int lt) {
#pragma unroll
  for (int c0 = 0; c0 < N; c0 += 32) {
    float t[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) t[i] = (c0 + i < N) ? v[c0 + i] : 0.f;
    const float r = warp_reduce_scatter32(t);
    const int lane = lt & 31;
    if (c0 + lane < N) wred[(lt >> 5) * nv + base + c0 + lane] = (double)r;
  }
}

template <int RS>
__device__ __forceinline__ void tmem_ld_row(unsigned taddr, float (&v)[RS]) {
  if constexpr (RS == 32) tmem_ld32(taddr, v);
  else if constexpr (RS == 16) tmem_ld16(taddr, v);
  else if constexpr (RS == 8) tmem_ld8(taddr, v);
  else tmem_ld4(taddr, v);
}
template <int RS>
__device__ __forceinline__ void tmem_st_row(unsigned taddr, const float (&v)[RS]) {
  if constexpr (RS == 32) tmem_st32(taddr, v);
  else if constexpr (RS == 16) tmem_st16(taddr, v);
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

// Row access of one row group: TMEM (warp-collective tcgen05.ld) or shared memory.
template <int RS>
struct TmemRows {
  unsigned taddr;
  __device__ __forceinline__ void operator()(int e, float (&u)[RS]) const {
    tmem_ld_row<RS>(taddr + e * RS, u);
    tmem_wait_ld();
  }
  // write a row group back (frame blocking): K values per row, the weight
  // in column RS-1 when k < RS (pair with tmem_wait_st before the next read)
  template <int K>
  __device__ __forceinline__ void store(const float (&up)[4][K], const float (&wn)[4]) const {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float row[RS];
#pragma unroll
      for (int j = 0; j < RS; ++j) row[j] = j < K ? up[e][j] : 0.f;
      if (K < RS) row[RS - 1] = wn[e];
      tmem_st_row<RS>(taddr + e * RS, row);
    }
  }
};
template <int RS>
struct SmemRows {
  float4* base;  // row e, column group g at base[(e * RS/4 + g) * qs]
  int qs;
  bool ok;
  __device__ __forceinline__ void operator()(int e, float (&u)[RS]) const {
#pragma unroll
    for (int g4 = 0; g4 < RS / 4; ++g4) {
      const float4 t = base[(size_t)(e * (RS / 4) + g4) * qs];  // (the sweep skips rows past the slice)
      u[4 * g4] = t.x; u[4 * g4 + 1] = t.y; u[4 * g4 + 2] = t.z; u[4 * g4 + 3] = t.w;
    }
  }
  template <int K>
  __device__ __forceinline__ void store(const float (&up)[4][K], const float (&wn)[4]) const {
    if (!ok) return;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float row[RS];
#pragma unroll
      for (int j = 0; j < RS; ++j) row[j] = j < K ? up[e][j] : 0.f;
      if (K < RS) row[RS - 1] = wn[e];
#pragma unroll
      for (int g4 = 0; g4 < RS / 4; ++g4)
        base[(size_t)(e * (RS / 4) + g4) * qs] =
            make_float4(row[4 * g4], row[4 * g4 + 1], row[4 * g4 + 2], row[4 * g4 + 3]);
    }
  }
};

template <int V>
using IC = std::integral_constant<int, V>;

// Bulk prefetch of [p, p + bytes) into L2 (no destination, no completion).
__device__ __forceinline__ void prefetch_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// NG slot groups per CTA (1 or 2): group g (TG = TM_NT / NG threads, TMEM
// columns [512 g / NG, 512 (g + 1) / NG), its own share of shared memory)
// works on its own stream: CTA team t's group g is virtual team t * NG + g.
// With NG = 2 the two groups of an SM are in different phases of their
// frames, so one group's HBM traffic (slice load, U' store) and its team-sum
// latency overlap the other group's sweeps (optionally enforced: ra.alt makes
// the groups' slice loads alternate A, B, A, B, ...).
// BLK: the frame-blocking instance (prost_push_many); the single-frame
// instance compiles the blocking paths out (they cost registers).
template <int K, int PM, int NG, bool BLK, bool CL = false, bool PROF = false>
__global__ void __launch_bounds__(TM_NT, TM_CPS)
    k_tmem(const __grid_constant__ Args a, const __grid_constant__ RArgs ra) {
  using Geo = TmemGeom<K>;
  constexpr int RS = Geo::RS, QW = Geo::QW, QT = Geo::QT, NVM = Geo::NV;
  constexpr bool WCOL = Geo::WCOL;
  constexpr int TG = TM_NT / NG;  // threads per slot group
  static_assert(NG == 1 || NG == 2, "slot groups");
  extern __shared__ __align__(128) uint8_t smem_raw[];
  __shared__ unsigned s_tbase;
  __shared__ unsigned long long sprof[PROF_N];
  __shared__ float sfv_all[NG][4][K];  // fp32 copies of y, d, v, grad for the per-element math
  __shared__ volatile int s_loads[2], s_done[2];  // slice loads done per group (ra.alt)
  const int G = ra.G, T = ra.T, qpc = ra.qpc;
  const int team = blockIdx.x / G, rank = blockIdx.x - team * G;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int g = NG == 1 ? 0 : tid / TG;
  const int lt = tid - g * TG;  // thread within the slot group
  const int VT = T * NG, vt = team * NG + g;
  float (&sfv)[4][K] = sfv_all[g];
  const int k = a.k;
  // row groups over the stream's stacked coordinates: with 3 channels a slice
  // may cover parts of several planes (Pp is a multiple of 4: a row group never
  // straddles two planes); labels and padding are per pixel
  const int nq = (int)(a.np / 4);
  const int q0 = rank * qpc;
  const int qcount = max(0, min(qpc, nq - q0));
  const int nslots = (qcount + TG - 1) / TG;  // uniform across the group
  const int nst = nslots < QT ? nslots : QT;  // TMEM slots in use
  const int qs = qpc > QT * TG ? qpc - QT * TG : 0;
  const int qa = (qpc + TG - 1) / TG * TG;

  // basis rows kept in shared memory: [row e][4-column group][row group] float4,
  // so a thread reads one row with RS/4 conflict-free 16-byte loads
  float4* sU = reinterpret_cast<float4*>(smem_raw + (size_t)g * tmem_group_smem<K, NG>(qpc));  // [4][RS/4][qs]
  float4* sR = sU + (size_t)RS * qs;                    // [qa] residual
  float4* sD = sR + qa;                                 // [qa] u_dir
  // [qa] U y at the current coordinates: pass 0's dot, then every accepted
  // step adds alpha * u_dir (the residual's recurrence, fit.py:136).  The
  // geodesic sweep gets U v = U y / ||y|| and the background U'y = U y +
  // coef ||y|| from it instead of two more k-term dot products per row.
  float4* sY = sD + qa;
  uint32_t* sL = reinterpret_cast<uint32_t*>(sY + qa);  // [qa] label bytes (!WCOL)
  double* wred = reinterpret_cast<double*>(sL + (WCOL ? 0 : qa));
  double* red = wred + (size_t)(TG / 32) * NVM;
  Ctl* cs = reinterpret_cast<Ctl*>(red + NVM);
  const float* Mg = static_cast<const float*>(a.mean);
  const float* Xg = static_cast<const float*>(a.x);
  // 4 frame values at coordinate offset off: fp32, or 8-bit divided by 255
  // exactly as the conversion kernel k_pack does (u8_unit: the double product, rounded)
  auto ld_x4 = [&](size_t off, float (&xv)[4]) {
    if (a.xu8) {
      const uchar4 b = *reinterpret_cast<const uchar4*>(static_cast<const uint8_t*>(a.x) + off);
      xv[0] = u8_unit(b.x);
      xv[1] = u8_unit(b.y);
      xv[2] = u8_unit(b.z);
      xv[3] = u8_unit(b.w);
    } else {
      f4(*reinterpret_cast<const float4*>(Xg + off), xv);
    }
  };

  if constexpr (CL) pdl_enter();  // cluster teams run with programmatic dependent launch
  if (tid < PROF_N) sprof[tid] = 0;
  if (tid < 2) {
    s_loads[tid] = 0;
    s_done[tid] = NG == 1 ? 1 : 0;
  }
  const unsigned long long t_start = ptimer(), g_start = gtimer();
  // TMEM: TM_NT columns, allocated by warp 0
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_addr(&s_tbase)),
                 "n"(TM_NT));
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
    if (lt < K) {                          \
      sfv[0][lt] = (float)cs->y[lt];       \
      sfv[1][lt] = (float)cs->d[lt];       \
      sfv[2][lt] = (float)cs->v[lt];       \
      sfv[3][lt] = (float)cs->grad[lt];    \
    }                                      \
  } while (0)
#define LOGIC(call)                                                        \
  do {                                                                     \
    const unsigned long long tl0 = (TM_PROF_ON(ra) && tid == 0) ? ptimer() : 0;   \
    if (lt < 32) {                                                         \
      call;                                                                \
      __syncwarp();                                                        \
      SYNC_FLOATS();                                                       \
    }                                                                      \
    if (TM_PROF_ON(ra) && tid == 0) sprof[PROF_LOGIC] += ptimer() - tl0;          \
  } while (0)

  // Visit every row group of this thread: body(qi, rows).  TMEM row groups
  // first, then shared-memory ones (separate instances of the body).
  auto sweep = [&](auto&& body) {
    for (int slot = 0; slot < nst; ++slot)
      body(slot * TG + lt, TmemRows<RS>{tbase + (unsigned)(slot * QW)});
    for (int slot = QT; slot < nslots; ++slot) {
      // rows past qcount were never loaded and hold nothing: skipped (their
      // contributions are exact zeros — weight 0 — and nothing reads their r)
      const int qi = slot * TG + lt;
      if (qi < qcount) body(qi, SmemRows<RS>{sU + (qi - QT * TG), qs, true});
    }
  };
  const float omega = a.omegaf;
  // weights of a row group from the label words (layout without a weight column)
  auto pixel_of = [&](int coord) { return a.C == 1 ? coord : coord % a.Pp; };
  auto lab_weights = [&](int qi, float (&w)[4]) {
    const uint32_t lb = qi < qcount ? sL[qi] : 0u;
    const int pix = pixel_of((q0 + qi) * 4);
#pragma unroll
    for (int e = 0; e < 4; ++e)
      w[e] = (qi < qcount && pix + e < a.P) ? (((lb >> (8 * e)) & 0xffu) ? omega : 1.f) : 0.f;
  };
  const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);

  // Stagger the teams (optional): odd teams start ra.stagger_ns late.
  if ((team & 1) && ra.stagger_ns > 0) {
    const unsigned long long t0 = gtimer();
    while (gtimer() - t0 < (unsigned long long)ra.stagger_ns) __nanosleep(1000);
  }

  int round = 0;
#if PROST_DYN
  // Dynamic stream assignment: a team's first stream is vt, then rank 0
  // takes the next one from a global counter (ra.bar[VT]) at the start of each
  // round and publishes it (ra.bar[VT + 1 + 2 vt + parity]) before the round's first team
  // sum, whose release/acquire barrier makes it visible to the team — teams
  // that draw cheap streams take more (a stream's result does not depend on
  // its team: every team has the same geometry).
  for (int s = vt; s < ra.S; ++round) {
    if (!CL && NG == 1 && rank == 0 && lt == 0) {
      // slot by round parity: a team mate may still be reading this round's
      // stream (published last round) while rank 0 publishes the next one
      const unsigned nx = (unsigned)VT + atomicAdd(ra.bar + VT, 1u);
      asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(ra.bar + VT + 1 + 2 * vt + ((round + 1) & 1)),
                   "r"(nx)
                   : "memory");
    }
#else
  for (int s = vt; s < ra.S; s += VT, ++round) {
#endif
    if (TM_PROF_ON(ra) && tid == 0) sprof[PROF_ROUNDS] += 1;
    if (NG > 1 && ra.alt) {
      // the groups' slice loads alternate: A0 B0 A1 B1 ... (a finished group
      // no longer holds the other back)
      if (lt == 0) {
        const int o = g ^ 1, need = g == 0 ? round : round + 1;
        long long spins = 0;
        while (s_loads[o] < need && !s_done[o]) {
          __nanosleep(64);
          if (++spins > (1LL << 28)) __trap();
        }
      }
      group_sync<NG>(g);
    }
    const size_t so = (size_t)s * a.np;  // this stream's plane offset
    // ---- the stream's control block -----------------------------------------
    if (lt < (int)(sizeof(Ctl) / 8))
      reinterpret_cast<double*>(cs)[lt] = __ldcg(reinterpret_cast<const double*>(a.ctl + s) + lt);
    group_sync<NG>(g);
    if (lt == 0) {
      cs->no_info = rank != 0;
      cs->t = step_size(a, cs->frame_index);  // tracker.py:99-103, off the reductions' critical path
    }
    SYNC_FLOATS();
    group_sync<NG>(g);

    // Frame blocking (a.nframes = F > 1, one channel): the stream's next F
    // frames run while its slice stays on chip — U is loaded once and stored
    // once per block, each frame's geodesic sweep writes U' back to TMEM /
    // shared memory and runs the next frame's pass 0 on the rows it just
    // updated (r0 = x_{f+1} - U'y_f: the warm start is this frame's y), and
    // the per-frame outputs go to [f][S][...].  Every frame computes exactly
    // what one push per frame computes.
    const int F = (BLK && a.nframes > 1 && a.C == 1) ? a.nframes : 1;
    bool p0_ready = false;  // this frame's pass 0 partials came with the last geodesic sweep
    double cost_n = 0.0;
    bool bad_n = false;
    float pk_n[K + 1];
#pragma unroll
    for (int j = 0; j <= K; ++j) pk_n[j] = 0.f;
    for (int f = 0; f < F; ++f) {
    const size_t fo = (size_t)f * ra.S * a.np;  // this frame's coordinate outputs / input
    const size_t fl = (size_t)f * ra.S * a.Pp;  // this frame's label outputs
    const size_t sox = fo + so;                 // this frame's input of this stream
    if (f > 0) {
      if (lt == 0) {
        cs->t = step_size(a, cs->frame_index);
        cs->info_slot = f * ra.S;
      }
      group_sync<NG>(g);
    } else if (lt == 0) {
      cs->info_slot = 0;
    }

    unsigned long long tph = (TM_PROF_ON(ra) && tid == 0) ? ptimer() : 0;
#define PHASE_MARK(idx)                              \
  do {                                               \
    if (TM_PROF_ON(ra) && tid == 0) {                       \
      const unsigned long long tn = ptimer();        \
      sprof[idx] += tn - tph;                        \
      tph = tn;                                      \
    }                                                \
  } while (0)
    // ---- frame start: running statistics (pipeline.py:120-140) -------------
    // (reads the frame only; the normalization below needs its team sum)
    const bool upd = a.pipeline && !cs->frozen && cs->frame_index < a.i_init;
    if (upd) {
      double s1 = 0.0, s2 = 0.0, nf = 0.0;
      for (int slot = 0; slot < nslots; ++slot) {
        const int qi = slot * TG + lt;
        if (qi >= qcount) continue;
        const int coord = (q0 + qi) * 4, pix = pixel_of(coord);
        float xv[4];
        ld_x4(sox + coord, xv);
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
      rstage_g(s1, wred, 0, 3, lt);
      rstage_g(s2, wred, 1, 3, lt);
      rstage_g(nf, wred, 2, 3, lt);
      team_sum_g<NG, CL, PROF>(ra, vt, VT, rank, g, lt, wred, 3, red, epoch, sprof);
      if (lt == 0) {
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
    } else if (lt == 0) {
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
    group_sync<NG>(g);
    PHASE_MARK(PROF_T_STATS);

    // normalized frame of a row group (pipeline.py:148-156); the sweep that
    // owns this frame's running-mean update writes the mean back
    const float stdv = (float)cs->std_cur, seen = (float)cs->pseen;
    const float inv_std = (float)(1.0 / cs->std_cur);
    auto xhat = [&](int qi, bool wr, float (&xh)[4], bool& bad) {
      const bool ok = qi < qcount;
      const int coord = (q0 + qi) * 4, pix = pixel_of(coord);
      float xv[4] = {0.f, 0.f, 0.f, 0.f};
      if (ok) ld_x4(sox + coord, xv);
      if (a.pipeline) {
        float mv[4];
        f4(ok ? *reinterpret_cast<const float4*>(Mg + so + coord) : z4, mv);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          bad |= !isfinite(xv[e]);
          if (wr) mv[e] = __fadd_rn(mv[e], __fdiv_rn(__fsub_rn(xv[e], mv[e]), seen));
#if PROST_RCP_STD
          xh[e] = __fmul_rn(__fsub_rn(xv[e], mv[e]), inv_std);
#else
          xh[e] = __fdiv_rn(__fsub_rn(xv[e], mv[e]), stdv);
#endif
          if (pix + e >= a.P) xh[e] = 0.f;
        }
        if (wr && ok)
          *reinterpret_cast<float4*>(static_cast<float*>(a.mean) + so + coord) =
              make_float4(mv[0], mv[1], mv[2], mv[3]);
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          bad |= !isfinite(xv[e]);
          xh[e] = pix + e < a.P ? xv[e] : 0.f;
        }
      }
    };

    // ---- load this stream's slice: U (+ weights) -> TMEM / shared memory,
    // fused with pass 0: r = x - U y, cost, coordinate gradient (fit.py:96-104)
    // needs nothing but the row itself, so it runs on the rows as they arrive
    // from HBM (the frame and mean loads overlap the basis loads).  A
    // stream's first frame cannot fuse: its warm start y = U^T x (fit.py:86-87)
    // is a reduction over the whole slice, so pass 0 then sweeps separately.
    // A frame rejected by the statistics check (non-finite) loads nothing.
    const bool frame_ok = cs->status == ST_OK;
    const bool cold = frame_ok && cs->frame_index == 0;
    const bool fuse = frame_ok && !cold;
    const bool use_p0 = BLK && f > 0 && p0_ready && frame_ok && !upd;
    bool bad = use_p0 ? bad_n : false;
    bool mean_pending = upd;  // running-mean update not yet written this frame
    double cost = use_p0 ? cost_n : 0.0;
    float pk[K + 1];
#pragma unroll
    for (int j = 0; j <= K; ++j) pk[j] = use_p0 ? pk_n[j] : 0.f;
    p0_ready = false;
    if (frame_ok && f == 0) {
      const unsigned long long tw0 = (TM_PROF_ON(ra) && tid == 0) ? ptimer() : 0;
      const float* U = static_cast<const float*>(a.U) + (size_t)s * k * a.np;
      // The slots after the first arrive through L2: one bulk prefetch per
      // basis plane (and for the frame / mean / label bytes) of the rest of
      // this CTA's slice, issued before slot 0's loads, so HBM streams the
      // whole slice while the threads work through the slots in order.
      if (ra.prefetch && (lt >> 5) == 0 && nslots > 1) {
        const int lane = lt & 31;
        const long long c0 = (long long)(q0 + TG) * 4, c1 = (long long)(q0 + qcount) * 4;
        auto pf = [&](const void* base, long long b0, long long b1) {
          const uintptr_t p0 = ((uintptr_t)base + b0 + 15) & ~(uintptr_t)15;
          const uintptr_t p1 = ((uintptr_t)base + b1) & ~(uintptr_t)15;
          if (p1 > p0) prefetch_l2(reinterpret_cast<const void*>(p0), (unsigned)(p1 - p0));
        };
        if (lane < k) pf(U + (size_t)lane * a.np, c0 * 4, c1 * 4);
        if (lane == 31 && fuse) {
          if (a.xu8) pf(static_cast<const uint8_t*>(a.x) + sox, c0, c1);
          else pf(Xg + sox, c0 * 4, c1 * 4);
        }
        if (lane == 30 && fuse && a.pipeline) pf(Mg + so, c0 * 4, c1 * 4);
        if (lane == 29 && a.C == 1) pf(a.lab + (size_t)s * a.Pp, c0, c1);
      }
      for (int slot = 0; slot < nslots; ++slot) {
        const int qi = slot * TG + lt;  // row group within the slice
        const bool ok = qi < qcount;
        const int coord = (q0 + qi) * 4, pix = pixel_of(coord);
        float4 p[K];
        if (ok && k == K) {  // the common case: every plane, no per-plane predicate or zero fill
          const float* Uc = U + coord;
#pragma unroll
          for (int j = 0; j < K; ++j) p[j] = __ldcs(reinterpret_cast<const float4*>(Uc + (size_t)j * a.np));
        } else {
#pragma unroll
          for (int j = 0; j < K; ++j)
            p[j] = (ok && j < k) ? __ldcs(reinterpret_cast<const float4*>(U + (size_t)j * a.np + coord)) : z4;
        }
        const uint32_t lb = ok ? *reinterpret_cast<const uint32_t*>(a.lab + (size_t)s * a.Pp + pix) : 0u;
        if (!WCOL) sL[qi] = lb;
        float xh[4], w[4], r[4], uy[4];
        if (fuse) xhat(qi, mean_pending, xh, bad);
#pragma unroll
        for (int e = 0; e < 4; ++e)
          w[e] = (ok && pix + e < a.P) ? (((lb >> (8 * e)) & 0xffu) ? omega : 1.f) : 0.f;
        float tc = 0.f;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float row[RS];
#pragma unroll
          for (int j = 0; j < RS; ++j) {
            const float4 t = j < K ? p[j] : z4;
            row[j] = e == 0 ? t.x : (e == 1 ? t.y : (e == 2 ? t.z : t.w));
          }
          if (WCOL) row[RS - 1] = w[e];
          if (slot < QT) {
            tmem_st_row<RS>(tbase + slot * QW + e * RS, row);
          } else if (ok) {
            float4* rp = sU + (size_t)(e * (RS / 4)) * qs + (qi - QT * TG);
#pragma unroll
            for (int g4 = 0; g4 < RS / 4; ++g4)
              rp[(size_t)g4 * qs] = make_float4(row[4 * g4], row[4 * g4 + 1], row[4 * g4 + 2], row[4 * g4 + 3]);
          }
          if (fuse) {
            uy[e] = dotk<K>(row, sfv[0]);
            r[e] = __fsub_rn(xh[e], uy[e]);
            float tw, gg;
            penalty_t<PM>(r[e], w[e], a, tw, gg);
            tc += tw;
            pk[K] += gg * gg;
#pragma unroll
            for (int j = 0; j < K; ++j) pk[j] += row[j] * gg;
          }
        }
        if (fuse) {
          cost += (double)tc;
          sR[qi] = make_float4(r[0], r[1], r[2], r[3]);
          sD[qi] = z4;
          sY[qi] = make_float4(uy[0], uy[1], uy[2], uy[3]);
        }
      }
      tmem_wait_st();
      if (fuse) mean_pending = false;
      group_sync<NG>(g);  // shared-memory rows, r and u_dir visible to every warp
      if (TM_PROF_ON(ra) && tid == 0) sprof[PROF_PREFETCH] += ptimer() - tw0;
    }
    if (NG > 1 && lt == 0) s_loads[g] = round + 1;
    tph = (TM_PROF_ON(ra) && tid == 0) ? ptimer() : 0;

    if (frame_ok) {
      // ---- cold start y = U^T x (fit.py:86-87), then pass 0 over the slice ---
      // (also: a blocked frame whose pass 0 did not come with the geodesic
      // sweep — statistics window, or the previous frame was rejected)
      if (cold || (f > 0 && !use_p0)) {
        float pkc[K];
#pragma unroll
        for (int j = 0; j < K; ++j) pkc[j] = 0.f;
        if (cold) {
        sweep([&](int qi, const auto& rows) {
          float xh[4];
          xhat(qi, upd, xh, bad);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            float u[RS];
            rows(e, u);
#pragma unroll
            for (int j = 0; j < K; ++j) pkc[j] += u[j] * xh[e];
          }
        });
        mean_pending = false;
        stage_floats_g<K>(pkc, wred, K + 1, 0, lt);
        rstage_g(bad ? 1.0 : 0.0, wred, K, K + 1, lt);
        team_sum_g<NG, CL, PROF>(ra, vt, VT, rank, g, lt, wred, K + 1, red, epoch, sprof);
        if (lt < 32) {
          if (red[K] > 0.0) mark_nonfinite(cs, a, s, lt);
          else if (lt < k) cs->y[lt] = red[lt];
          __syncwarp();
          SYNC_FLOATS();
        }
        group_sync<NG>(g);
        }
        if (cs->status == ST_OK) {
          sweep([&](int qi, const auto& rows) {
            float xh[4], w[4], r[4], uy[4];
            xhat(qi, mean_pending, xh, bad);
            if (!WCOL) lab_weights(qi, w);
            float tc = 0.f;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              float u[RS];
              rows(e, u);
              if (WCOL) w[e] = u[RS - 1];
              uy[e] = dotk<K>(u, sfv[0]);
              r[e] = __fsub_rn(xh[e], uy[e]);
              float tw, gg;
              penalty_t<PM>(r[e], w[e], a, tw, gg);
              tc += tw;
              pk[K] += gg * gg;
#pragma unroll
              for (int j = 0; j < K; ++j) pk[j] += u[j] * gg;
            }
            cost += (double)tc;
            sR[qi] = make_float4(r[0], r[1], r[2], r[3]);
            sD[qi] = z4;
            sY[qi] = make_float4(uy[0], uy[1], uy[2], uy[3]);
          });
        }
      }
      if (cs->status == ST_OK) {
        rstage_g(cost, wred, 0, K + 3, lt);
        stage_floats_g<K + 1>(pk, wred, K + 3, 1, lt);
        rstage_g(bad ? 1.0 : 0.0, wred, K + 2, K + 3, lt);
        team_sum_g<NG, CL, PROF>(ra, vt, VT, rank, g, lt, wred, K + 3, red, epoch, sprof);
        LOGIC(TM_AFTER_PASS0<K>(cs, a, s, lt, red));
        group_sync<NG>(g);
      }
    }
    PHASE_MARK(PROF_T_PASS0);

    // ---- CG iterations (fit.py:108-144) -------------------------------------
    // pend_alpha (an accepted step not yet applied to r) is applied by the
    // next sweep that reads r: the iteration sweep or the geodesic sweep.
    while (cs->status == ST_OK && cs->active) {
      if (cs->need_lsfb) {
        const int base = cs->ls_next;
        const int cnt = (a.max_bt - base) < LSW ? (a.max_bt - base) : LSW;
        const double al0 = alpha_at(a, base);
        float cst[LSW];
#pragma unroll
        for (int m = 0; m < LSW; ++m) cst[m] = 0.f;
        sweep([&](int qi, const auto& rows) {
          float r[4], ud[4], w[4];
          f4(sR[qi], r);
          f4(sD[qi], ud);
          if (WCOL) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              float u[RS];
              rows(e, u);
              w[e] = u[RS - 1];
            }
          } else {
            lab_weights(qi, w);
          }
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
        });
#pragma unroll
        for (int m = 0; m < LSW; ++m) rstage_g((double)cst[m], wred, m, LSW, lt);
        team_sum_g<NG, CL, PROF>(ra, vt, VT, rank, g, lt, wred, LSW, red, epoch, sprof);
        LOGIC(TM_AFTER_LSFB(cs, a, s, lt, red, base));
      } else if (cs->need_gradfb) {
        const float al = (float)cs->acc_alpha;
        float pk[K + 1];
#pragma unroll
        for (int j = 0; j <= K; ++j) pk[j] = 0.f;
        sweep([&](int qi, const auto& rows) {
          float r[4], ud[4], w[4];
          f4(sR[qi], r);
          f4(sD[qi], ud);
          if (!WCOL) lab_weights(qi, w);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            float u[RS];
            rows(e, u);
            if (WCOL) w[e] = u[RS - 1];
            float tw, g;
            penalty_t<PM>(trial(r[e], al, ud[e]), w[e], a, tw, g);
            pk[K] += g * g;
#pragma unroll
            for (int j = 0; j < K; ++j) pk[j] += u[j] * g;
          }
        });
        stage_floats_g<K + 1>(pk, wred, K + 1, 0, lt);
        team_sum_g<NG, CL, PROF>(ra, vt, VT, rank, g, lt, wred, K + 1, red, epoch, sprof);
        LOGIC(TM_AFTER_GRADFB<K>(cs, a, s, lt, red));
      } else {
        constexpr int NV = WC + WG * (K + 1);
        const int wlo = cs->gwin_lo;
        const float pa = (float)cs->pend_alpha;
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
        // trial costs for every window step; the gradient only for the
        // speculative pair [wlo, wlo + WG).  One code path: every trial value
        // is computed once, and the pair is picked with a warp-uniform index
        // (separate instantiations per window position were merged by the
        // compiler into a predicated body that recomputed the trials: 12
        // instead of 8 MUFU and ~30 selects per row).
        static_assert(WC <= 4 && WG <= 2 && WC - WG <= 2, "window positions");
        const bool w1 = wlo >= 1, w2 = wlo >= 2;
        const unsigned long long tsw0 = (TM_PROF_ON(ra) && tid == 0) ? ptimer() : 0;
        sweep([&](int qi, const auto& rows) {
          float r[4], w[4], udo[4], ud[4];
          f4(sR[qi], r);
          f4(sD[qi], udo);
          if (pa != 0.f) {  // the pending accepted step moves U y too
            float y4[4];
            f4(sY[qi], y4);
#pragma unroll
            for (int e = 0; e < 4; ++e) y4[e] = fmaf(pa, udo[e], y4[e]);
            sY[qi] = make_float4(y4[0], y4[1], y4[2], y4[3]);
          }
          if (!WCOL) lab_weights(qi, w);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            float u[RS];
            rows(e, u);
            if (WCOL) w[e] = u[RS - 1];
            r[e] = trial(r[e], pa, udo[e]);  // pending accepted step (exact no-op at 0)
            const float d = dotk<K>(u, sfv[1]);
            ud[e] = d;
            float gm[WC];
#pragma unroll
            for (int m = 0; m < WC; ++m) {
              const float t = trial(r[e], al[m], d);
              if (PM == PM_HALF) {
                const float b = fmaf(t, t, a.muf);
                const float h = rsqrtf(b);
                const float q = rsqrtf(h);
                cst[m] = fmaf(q, w[e], cst[m]);
                // twice the coordinate gradient (cost.py:103-112 without its
                // factor 1/2): exactly 2x in fp32, and so are the gradient sums
                // built from it; the scalar logic halves them (exact) — one
                // multiply fewer per trial
                gm[m] = t * (q * w[e]) * (h * h);
              } else {
                float tw, gg;
                penalty_t<PM>(t, w[e], a, tw, gg);
                cst[m] += tw;
                gm[m] = 2.f * gg;
              }
            }
            float gs[WG];
            gs[0] = w2 ? gm[2 < WC ? 2 : WC - 1] : (w1 ? gm[1] : gm[0]);
            if (WG > 1) gs[WG - 1] = w2 ? gm[3 < WC ? 3 : WC - 1] : (w1 ? gm[2 < WC ? 2 : WC - 1] : gm[1]);
#pragma unroll
            for (int mm = 0; mm < WG; ++mm) {
              pk[mm * (K + 1) + K] = fmaf(gs[mm], gs[mm], pk[mm * (K + 1) + K]);
#pragma unroll
              for (int j = 0; j < K; ++j) pk[mm * (K + 1) + j] = fmaf(u[j], gs[mm], pk[mm * (K + 1) + j]);
            }
          }
          sR[qi] = make_float4(r[0], r[1], r[2], r[3]);
          sD[qi] = make_float4(ud[0], ud[1], ud[2], ud[3]);
        });
        if (lt == 0) cs->pend_alpha = 0.0;  // consumed by this sweep
#pragma unroll
        for (int m = 0; m < WC; ++m) rstage_g((double)cst[m], wred, m, NV, lt);
        stage_floats_g<WG * (K + 1)>(pk, wred, NV, WC, lt);
        if (TM_PROF_ON(ra)) {  // (uniform: every thread of the group takes the barrier)
          const unsigned long long t1 = tid == 0 ? ptimer() : 0;
          group_sync<NG>(g);
          if (tid == 0) {
#if !PROST_SKEW_PROBE
            sprof[PROF_SW_OWN] += t1 - tsw0;
            sprof[PROF_SW_ALL] += ptimer() - tsw0;
#endif
          }
        }
        team_sum_g<NG, CL, PROF>(ra, vt, VT, rank, g, lt, wred, NV, red, epoch, sprof);
        {
          const unsigned long long tli = (TM_PROF_ON(ra) && tid == 0) ? ptimer() : 0;
          if (lt < 32) {  // the sweep summed 2 g (and 4 g^2): exact halving in double
            for (int v = WC + lt; v < NV; v += 32) red[v] *= ((v - WC) % (K + 1) == K) ? 0.25 : 0.5;
            __syncwarp();
          }
          LOGIC(TM_AFTER_ITER<K>(cs, a, s, lt, red, wlo));
          if (TM_PROF_ON(ra) && tid == 0) sprof[PROF_LOGIC_ITER] += ptimer() - tli;
        }
      }
      group_sync<NG>(g);
    }
    PHASE_MARK(PROF_T_ITER);

    if (cs->status == ST_OK) {
      // ---- geodesic step + relabel (manifold.py:116-197, tracker.py:146-147) --
      // With a re-orthonormalization due (every 1000th step) U' is written back
      // unlabeled; the streamed k_gram / k_geo<QR> kernels that follow the
      // launch apply U' R^-1 and relabel (manifold.py:192-196).
      const bool geo = cs->do_geo != 0, qr = geo && cs->qr_now != 0;
      const float ga = (float)cs->geo_a, gsn = (float)cs->geo_s;
      const float inv_ln = geo ? (float)(1.0 / cs->geo_ln) : 0.f;  // s = pi(eta) / ||pi(eta)||
      const float pa = (float)cs->pend_alpha;
      float* Ug = static_cast<float*>(a.U) + (size_t)s * k * a.np;
      // r' = x - U'y (tracker.py:146) without re-reading the frame: every row
      // moves by U'_i - U_i = coef_i v^T with v = y / ||y||, so
      // U'_i y = U_i y + coef_i ||y|| and r'_i = r_i - coef_i ||y||, where r is
      // the fit residual x - U y kept on chip (fit.py's res, the same
      // recurrence of accepted steps as the reference)
      const float yn = (float)cs->geo_yn;
      const float inv_yn = geo ? (float)(1.0 / cs->geo_yn) : 0.f;
      const bool want_bg = a.bg_out != nullptr;
      // frame blocking: keep U' on chip for frame f+1 and run its pass 0 here
      // when its normalization is already fixed (frozen statistics)
      const bool resident = BLK && f + 1 < F && !qr;
      const long long nfi = cs->frame_index;  // f+1's frame index (advanced by finish)
      const bool fuse_next = resident && !(a.pipeline && !cs->frozen && nfi < a.i_init);
      const double sd_next = a.pipeline ? (cs->frozen ? cs->pstd : running_std(cs)) : 1.0;
      const float inv_std_n = (float)(1.0 / sd_next);
      const size_t sox_n = sox + (size_t)ra.S * a.np;  // frame f+1's input of this stream
      cost_n = 0.0;
      bad_n = false;
#pragma unroll
      for (int j = 0; j <= K; ++j) pk_n[j] = 0.f;
      sweep([&](int qi, const auto& rows) {
        const bool ok = qi < qcount;
        const int coord = (q0 + qi) * 4, pix = pixel_of(coord);
        const size_t off = so + coord;
        float m4[4] = {0.f, 0.f, 0.f, 0.f};  // running mean, loaded first
        if ((want_bg || fuse_next) && a.pipeline && ok && !qr) f4(*reinterpret_cast<const float4*>(Mg + off), m4);
        float x4[4] = {0.f, 0.f, 0.f, 0.f};  // frame f+1 (fused pass 0)
        if (fuse_next && ok) ld_x4(sox_n + coord, x4);
        float r[4], w[4], ud[4], uy[4];
        f4(sR[qi], r);
        f4(sD[qi], ud);
        f4(sY[qi], uy);
        if (!WCOL) lab_weights(qi, w);
        float up[4][K];  // U' rows of this row group
        float rr[4], bgn[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float u[RS];
          rows(e, u);
          if (WCOL) w[e] = u[RS - 1];
          r[e] = trial(r[e], pa, ud[e]);  // the fit residual x - U y (fit.py res)
          uy[e] = fmaf(pa, ud[e], uy[e]);  // U y at the fitted y
          float coef = 0.f;
          if (geo) {
            float tw, g;
            penalty_t<PM>(r[e], w[e], a, tw, g);
            const float eta = -g;  // cost.py:103-112
            const float uv = uy[e] * inv_yn;  // U v, v = y / ||y||
            const float ug = dotk<K>(u, sfv[3]);
            coef = ga * uv - gsn * ((eta - ug) * inv_ln);
          }
          rr[e] = fmaf(-coef, yn, r[e]);
          bgn[e] = fmaf(coef, yn, uy[e]);  // U'y = U y + coef ||y||
#pragma unroll
          for (int j = 0; j < K; ++j) up[e][j] = u[j] + coef * sfv[2][j];
        }
        if (ok && a.fitres_out)
          *reinterpret_cast<float4*>(static_cast<float*>(a.fitres_out) + fo + off) = make_float4(r[0], r[1], r[2], r[3]);
        uint32_t nl = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (pix + e < a.P && fabsf(rr[e]) >= a.deltaf) nl |= 1u << (8 * e);
        if (resident) {
          // U' (and the new weights, the next frame's) back on chip
          float wn[4];
#pragma unroll
          for (int e = 0; e < 4; ++e)
            wn[e] = (ok && pix + e < a.P) ? (((nl >> (8 * e)) & 0xffu) ? omega : 1.f) : 0.f;
          if (!WCOL && ok) sL[qi] = nl;
          rows.template store<K>(up, wn);
          if (fuse_next) {  // pass 0 of frame f+1: r0 = x - U'y_f (fit.py:96-104)
            float tc = 0.f, r0[4], uy0[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              bad_n |= !isfinite(x4[e]);
              float xh = a.pipeline ? __fmul_rn(__fsub_rn(x4[e], m4[e]), inv_std_n) : x4[e];
              if (pix + e >= a.P) xh = 0.f;
              float uu[RS];
#pragma unroll
              for (int j = 0; j < RS; ++j) uu[j] = j < K ? up[e][j] : 0.f;
              uy0[e] = dotk<K>(uu, sfv[0]);  // a fresh dot, as the next push's pass 0
              r0[e] = __fsub_rn(xh, uy0[e]);
              float tw, gg;
              penalty_t<PM>(r0[e], wn[e], a, tw, gg);
              tc += tw;
              pk_n[K] += gg * gg;
#pragma unroll
              for (int j = 0; j < K; ++j) pk_n[j] += up[e][j] * gg;
            }
            cost_n += (double)tc;
            sR[qi] = make_float4(r0[0], r0[1], r0[2], r0[3]);
            sD[qi] = z4;
            sY[qi] = make_float4(uy0[0], uy0[1], uy0[2], uy0[3]);
          }
        }
        if (!ok) return;
        if (geo && !resident) {
#pragma unroll
          for (int j = 0; j < K; ++j)
            if (j < k)
              __stcs(reinterpret_cast<float4*>(Ug + (size_t)j * a.np + coord),
                     make_float4(up[0][j], up[1][j], up[2][j], up[3][j]));
        }
        if (qr) return;
        if (a.C == 1) {
          *reinterpret_cast<uint32_t*>(a.lab + (size_t)s * a.Pp + pix) = nl;
          if (a.raw_out) *reinterpret_cast<uint32_t*>(a.raw_out + fl + (size_t)s * a.Pp + pix) = nl;
        } else {  // per-channel flags; k_combine3 takes the max over channels (pipeline.py:210-211)
          *reinterpret_cast<uint32_t*>(a.labc + off) = nl;
        }
        if (a.res_out)
          *reinterpret_cast<float4*>(static_cast<float*>(a.res_out) + fo + off) = make_float4(rr[0], rr[1], rr[2], rr[3]);
        if (want_bg) {
          const float sc = (float)cs->std_cur;
          float b[4];
#pragma unroll
          for (int e = 0; e < 4; ++e)
            b[e] = a.pipeline ? fminf(fmaxf(__fadd_rn(bgn[e] * sc, m4[e]), 0.f), 1.f) : bgn[e];
          *reinterpret_cast<float4*>(static_cast<float*>(a.bg_out) + fo + off) = make_float4(b[0], b[1], b[2], b[3]);
        }
      });
      if (resident) tmem_wait_st();
      p0_ready = fuse_next;
    }

    group_sync<NG>(g);
    PHASE_MARK(PROF_T_GEO);
    if (lt == 0) cs->pend_alpha = 0.0;
    group_sync<NG>(g);
    }  // frames of the block

    // ---- commit the control block (one writer per stream) ------------------
#undef PHASE_MARK
    if (rank == 0 && lt < (int)(sizeof(Ctl) / 8))
      reinterpret_cast<double*>(a.ctl + s)[lt] = reinterpret_cast<const double*>(cs)[lt];
    group_sync<NG>(g);

    // ---- cluster teams: the stream's 3x3 label median here (pipeline.py:
    // 215-228, edge replication) instead of in a separate kernel — after the
    // cluster barrier every label of the team's stream is written; L2 reads
    // (__ldcg), since other CTAs wrote them during this launch
    if constexpr (CL && !BLK) {
      if (ra.median) {
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        if (cs->status == ST_OK) {
          const int W = a.width, H = a.height, wq = W >> 2;
          const uint8_t* L = a.lab + (size_t)s * a.Pp;
          uint32_t* M = reinterpret_cast<uint32_t*>(a.mask_out + (size_t)s * a.Pp);
          for (int qi = lt; qi < qcount; qi += TG) {
            const int q = q0 + qi;
            if (q * 4 >= a.P) continue;
            const int yy = q / wq, x0 = (q - yy * wq) << 2;
            const int xl = x0 > 0 ? x0 - 1 : 0, xr = x0 + 4 < W ? x0 + 4 : W - 1;
            const uint8_t* ra_ = L + (size_t)(yy > 0 ? yy - 1 : 0) * W;
            const uint8_t* rm = L + (size_t)yy * W;
            const uint8_t* rb = L + (size_t)(yy < H - 1 ? yy + 1 : H - 1) * W;
            const uint32_t v = __ldcg(reinterpret_cast<const unsigned*>(ra_ + x0)) +
                               __ldcg(reinterpret_cast<const unsigned*>(rm + x0)) +
                               __ldcg(reinterpret_cast<const unsigned*>(rb + x0));
            const uint32_t l = (uint32_t)__ldcg(reinterpret_cast<const unsigned char*>(ra_ + xl)) +
                               __ldcg(reinterpret_cast<const unsigned char*>(rm + xl)) +
                               __ldcg(reinterpret_cast<const unsigned char*>(rb + xl));
            const uint32_t r = (uint32_t)__ldcg(reinterpret_cast<const unsigned char*>(ra_ + xr)) +
                               __ldcg(reinterpret_cast<const unsigned char*>(rm + xr)) +
                               __ldcg(reinterpret_cast<const unsigned char*>(rb + xr));
            const uint32_t win = v + ((v << 8) | l) + ((v >> 8) | (r << 24));
            M[q] = __vcmpgeu4(win, 0x05050505u) & 0x01010101u;
          }
        }
      }
    }
#if PROST_DYN
    if constexpr (CL || NG > 1) {
      s += VT;
    } else {
      unsigned nx;
      asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];"
                   : "=r"(nx)
                   : "l"(ra.bar + VT + 1 + 2 * vt + ((round + 1) & 1))
                   : "memory");
      s = (int)nx;
    }
#endif
  }
  if (NG > 1 && lt == 0) s_done[g] = 1;
#undef LOGIC
#undef SYNC_FLOATS
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (TM_PROF_ON(ra) && tid == 0) {
    sprof[PROF_TOTAL] = ptimer() - t_start;
    sprof[PROF_GT_TOTAL] = gtimer() - g_start;
    for (int i = 0; i < PROF_N; ++i) ra.prof[(size_t)blockIdx.x * PROF_N + i] = sprof[i];
  }
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_tbase), "n"(TM_NT));
  if constexpr (CL)  // no CTA leaves while a peer may still read its team sums
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

}  // namespace prost
