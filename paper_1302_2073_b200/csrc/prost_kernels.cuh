// prost_kernels.cuh — sm_100a kernels for the pROST per-frame step.
//
// The per-frame step (reference tracker.py:121-156) is a chain of dependent
// global reductions over the n x k basis U.  Each phase below is one kernel
// that streams U (stored as k coordinate planes of n_pad values per stream,
// so every load is a coalesced 8/16-byte vector) over a grid of
// (chunks, streams) CTAs.  Every CTA reduces its partial sums in a fixed
// order, writes them to a slot, and the last CTA to arrive for a stream sums
// the slots in slot order (deterministic, no float atomics) and runs the
// scalar part of the algorithm for that stream in one warp (lane j owns
// component j of the k-vectors), in double precision, writing the control
// block that the next phase reads.
//
// Phases (host order, per frame):
//   k_stats   running statistics of the raw frame (pipeline.py:120-140)
//   k_cold    y = U^T x on the first frame (fit.py:86-87)
//   k_pass0   r = x - U y, cost and coordinate gradient (fit.py:96-104)
//   k_iter    u_dir = U d, Armijo trial costs for a window of WC step sizes
//             and the coordinate gradient speculatively for WG of them
//             (fit.py:108-144) — one U pass per CG iteration
//   k_lsfb    remaining Armijo trials when the window held no acceptable step
//             (elementwise over stored r and u_dir: no U traffic)
//   k_gradfb  gradient at an accepted step outside the speculative window
//   k_geo     rank-one geodesic update of U with the projected gradient,
//             relabel, background and residual (manifold.py:116-197,
//             tracker.py:140-147, jobs.py:231-239)
//   k_gram / k_geo<QR>  periodic re-orthonormalization (manifold.py:192-196)
//   k_median  3x3 majority filter (pipeline.py:215-228)
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

namespace prost {

constexpr int KMAX = 32;      // largest supported subspace dimension
constexpr int NT = 256;       // threads per CTA
constexpr int NW = NT / 32;   // warps per CTA
#ifndef PROST_WC
#define PROST_WC 4
#endif
#ifndef PROST_MINB
#define PROST_MINB 2
#endif
constexpr int WC = PROST_WC;  // Armijo trial costs evaluated per U pass
#ifndef PROST_WG
#define PROST_WG 2
#endif
constexpr int WG = PROST_WG;  // speculative gradients per U pass
constexpr int LSW = 16;       // trial costs per fallback line-search pass
constexpr int MAXBT = 64;     // cap on CgOptions.max_backtracks
constexpr int QR_EVERY = 1000;        // manifold.py:40
constexpr double NORM_FLOOR = 1e-14;  // manifold.py:38
constexpr double STD_FLOOR = 1e-6;    // pipeline.py:19

enum PenaltyMode { PM_GENERAL = 0, PM_ONE = 1, PM_TWO = 2, PM_HALF = 3 };
enum StreamStatus { ST_OK = 0, ST_NONFINITE = 3 };

// Per-stream control block: everything the scalar part of the algorithm
// carries between phases (double precision throughout).
// An 8-bit intensity as the reference reads it, float(b / 255) (frameio.py:136:
// the double product b * (1/255) rounded to fp32), in four fp32 instructions:
// q = b * fl(1/255) corrected once by its exact FMA residual.  Equal to the
// double expression for all 256 values (checked exhaustively: tests/test_host.py).
__device__ __forceinline__ float u8_unit(unsigned b) {
  constexpr float R = 1.0f / 255.0f;
  const float bf = (float)b;
  const float q = __fmul_rn(bf, R);
  return fmaf(fmaf(-q, 255.0f, bf), R, q);
}

struct Ctl {
  double y[KMAX], d[KMAX], grad[KMAX], v[KMAX];
  double f;            // current cost (fit.py f_cur)
  double slope;        // d . grad of the current iteration
  double gnorm;        // ||grad|| at the start of the current iteration
  double gsq;          // ||eta||^2 at the current residual
  double pend_alpha;   // residual update r -= pend_alpha * u_dir not yet applied
  double acc_alpha, acc_cost;
  double std_cur;      // normalization scale of this frame
  double t, geo_a, geo_s, geo_ln, geo_yn;  // geo_yn = ||y|| (the relabel's U'y update)
  double psum, psumsq, pstd;
  long long pcount, pseen, frame_index, since_qr;
  int it, active, need_lsfb, need_gradfb, acc_idx, ls_next, gwin_lo, last_acc;
  int do_geo, qr_now, status, iterations, cost_evals, grad_evals, frozen, cold;
  int update_stats, no_info;  // no_info: this copy must not write FitInfo
  int info_slot;              // FitInfo row of this frame (frame-blocked pushes: f * S)
  int pad0;
  // frame-blocked streamed pushes: frame_index + 1 of the frame whose pass 0
  // already ran inside the previous frame's geodesic sweep (k_geo_tma<K,
  // true>); its statistics and pass-0 kernels then exit at once.  0: none.
  long long p0_next;
};

struct FitInfo {  // layout-identical to prost_fit_info
  double fit_cost, step;
  long long frame_index;
  int iterations, cost_evals, grad_evals, status;
};

// Kernel arguments (passed by value; identical for every phase).
struct Args {
  void* U;             // [S][k][np]
  void* r;             // [S][np] residual (lazily updated)
  void* ud;            // [S][np] u_dir = U d of the last iteration
  const void* x;       // [S][np] frame (raw intensities or normalized x)
  const void* xnext;   // frame-blocked streamed pushes: the next frame (same layout), or null
  void* mean;          // [S][np] running mean (pipeline)
  uint8_t* lab;        // [S][Pp] labels: 1 = foreground (weight omega)
  Ctl* ctl;            // [S]
  double* part;        // [S][chunks][nvmax]
  unsigned* cnt;       // [S]
  double* rinv;        // [S][KMAX][KMAX] inverse Cholesky factor (periodic QR)
  FitInfo* info;       // [S]
  FitInfo* info_next;  // frame-blocked streamed pushes: the next frame's FitInfo rows
  void* bg_out;        // [S][np] or null
  void* res_out;       // [S][np] or null
  void* fitres_out;    // [S][np] fit residual x - U y before the geodesic (FitResult.residual) or null
  uint8_t* raw_out;    // [S][Pp] or null
  uint8_t* mask_out;   // [S][Pp] or null
  // Pixel-sharded (exchange) mode: a phase kernel's last CTA leaves the
  // stream's reduced partials in xred[s] (and whether the phase ran for the
  // stream in xgo[s]) instead of running the scalar logic; the caller sums
  // xred over ranks and k_xlogic finishes the phase.  Null otherwise.
  double* xred;        // [S][nvmax]
  int* xgo;            // [S]
  const uint8_t* halo_top;  // [S][width] label row above the local rows, or null
  const uint8_t* halo_bot;  // [S][width] label row below the local rows, or null
  // In-kernel exchange over peer memory (pixel sharding after prost_xpeer_open;
  // xred = null): the last CTA of a phase kernel stores the stream's sums into
  // every rank's exchange region (NVLink peer stores), waits for every rank's
  // flag and sums the ranks' vectors in rank order itself (xpeer_exchange).
  void* const* xpeer;        // [xworld] exchange regions of all ranks (device table), or null
  unsigned long long* xseq;  // [S] exchanges so far per stream (same on every rank)
  int xrank, xworld, xS;     // this rank, ranks, streams of the handle
  int xhalo;                 // bit 0: a rank above exists; bit 1: a rank below
  long long xframe;          // frames pushed (label-row halo sequence)
  uint8_t* labc;       // [S][np] per-coordinate flags of the TMEM kernel (3 channels), or null
  int xu8;             // TMEM kernel: x holds 8-bit frames, divided by 255 on load (frameio.py:136)
  int nframes;         // TMEM kernel: consecutive frames per stream in this launch (frame blocking;
                       // x, outputs and info are [nframes][S][...]); 0 or 1: one frame
  int s0;              // first stream of this launch
  int k, C, P, Pp, width, height;
  long long np;        // padded coordinates per stream = C * Pp
  int chunks, nvmax;
  int pipeline, max_iters, max_bt, i_init, pmode, n_real;
  double p, half_p, mu, delta, omega, t_init, t_min, tau, grad_tol, step0, shrink, c_armijo;
  float pf, half_pf, muf, omegaf;  // fp32 copies for the per-element math
  float deltaf;  // smallest float >= delta: abs(r) >= deltaf <=> (double)abs(r) >= delta
};

// ---------------------------------------------------------------------------
// vector access: VEC consecutive coordinates of one plane

template <typename T, int VEC> struct VecIO;

template <> struct VecIO<float, 4> {
  static __device__ __forceinline__ void ld(const float* p, float (&o)[4]) {
    float4 a = *reinterpret_cast<const float4*>(p);
    o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w;
  }
  static __device__ __forceinline__ void ldg(const float* p, float (&o)[4]) {
    float4 a = __ldg(reinterpret_cast<const float4*>(p));
    o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w;
  }
  static __device__ __forceinline__ void st(float* p, const float (&o)[4]) {
    *reinterpret_cast<float4*>(p) = make_float4(o[0], o[1], o[2], o[3]);
  }
};
template <> struct VecIO<float, 2> {
  static __device__ __forceinline__ void ld(const float* p, float (&o)[2]) {
    float2 a = *reinterpret_cast<const float2*>(p);
    o[0] = a.x; o[1] = a.y;
  }
  static __device__ __forceinline__ void ldg(const float* p, float (&o)[2]) {
    float2 a = __ldg(reinterpret_cast<const float2*>(p));
    o[0] = a.x; o[1] = a.y;
  }
  static __device__ __forceinline__ void st(float* p, const float (&o)[2]) {
    *reinterpret_cast<float2*>(p) = make_float2(o[0], o[1]);
  }
};
template <> struct VecIO<float, 1> {
  static __device__ __forceinline__ void ld(const float* p, float (&o)[1]) { o[0] = *p; }
  static __device__ __forceinline__ void ldg(const float* p, float (&o)[1]) { o[0] = __ldg(p); }
  static __device__ __forceinline__ void st(float* p, const float (&o)[1]) { *p = o[0]; }
};
template <> struct VecIO<double, 2> {
  static __device__ __forceinline__ void ld(const double* p, double (&o)[2]) {
    double2 a = *reinterpret_cast<const double2*>(p);
    o[0] = a.x; o[1] = a.y;
  }
  static __device__ __forceinline__ void ldg(const double* p, double (&o)[2]) {
    double2 a = __ldg(reinterpret_cast<const double2*>(p));
    o[0] = a.x; o[1] = a.y;
  }
  static __device__ __forceinline__ void st(double* p, const double (&o)[2]) {
    *reinterpret_cast<double2*>(p) = make_double2(o[0], o[1]);
  }
};
template <> struct VecIO<double, 1> {
  static __device__ __forceinline__ void ld(const double* p, double (&o)[1]) { o[0] = *p; }
  static __device__ __forceinline__ void ldg(const double* p, double (&o)[1]) { o[0] = __ldg(p); }
  static __device__ __forceinline__ void st(double* p, const double (&o)[1]) { *p = o[0]; }
};

template <int VEC> __device__ __forceinline__ void ld_lab(const uint8_t* p, uint8_t (&o)[VEC]) {
  if constexpr (VEC == 4) {
    uchar4 a = *reinterpret_cast<const uchar4*>(p);
    o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w;
  } else if constexpr (VEC == 2) {
    uchar2 a = *reinterpret_cast<const uchar2*>(p);
    o[0] = a.x; o[1] = a.y;
  } else {
    o[0] = *p;
  }
}
template <int VEC> __device__ __forceinline__ void st_lab(uint8_t* p, const uint8_t (&o)[VEC]) {
  if constexpr (VEC == 4) {
    *reinterpret_cast<uchar4*>(p) = make_uchar4(o[0], o[1], o[2], o[3]);
  } else if constexpr (VEC == 2) {
    *reinterpret_cast<uchar2*>(p) = make_uchar2(o[0], o[1]);
  } else {
    *p = o[0];
  }
}

// Coordinates per thread-vector: keeps the K*VEC basis values of one vector
// group in at most ~64 registers.
template <typename T, int K> struct Vec {
  static constexpr int raw = 64 / (K * (int)(sizeof(T) / 4));
  static constexpr int value = sizeof(T) == 8 ? (raw >= 2 ? 2 : 1) : (raw >= 4 ? 4 : 2);
};

// ---------------------------------------------------------------------------
// smoothed lp penalty (cost.py:57-93): weighted term w*(r^2+mu)^(p/2) and the
// residual gradient p*r*(w*term)/base.

// PM: compile-time penalty mode, or PM_ANY for a runtime switch on a.pmode.
constexpr int PM_ANY = -1;

template <int PM>
__device__ __forceinline__ void penalty_t(float r, float w, const Args& a, float& tw, float& g) {
  const float b = fmaf(r, r, a.muf);
  const int pm = PM == PM_ANY ? a.pmode : PM;
  if (pm == PM_HALF) {  // b^(1/4) and b^(-3/4) from two MUFU.RSQ
    const float h = rsqrtf(b);
    const float e = rsqrtf(h);
    tw = e * w;
    g = 0.5f * r * tw * (h * h);
  } else if (pm == PM_ONE) {
    const float h = rsqrtf(b);
    tw = b * h * w;
    g = r * w * h;
  } else if (pm == PM_TWO) {
    tw = b * w;
    g = 2.f * r * w;
  } else {
    const float L = __log2f(b);
    tw = exp2f(a.half_pf * L) * w;
    g = a.pf * r * tw * __frcp_rn(b);
  }
}

__device__ __forceinline__ void penalty(float r, float w, const Args& a, float& tw, float& g) {
  penalty_t<PM_ANY>(r, w, a, tw, g);
}

// Double instantiation: the same operation sequence and rounding as the
// reference's numpy code (no FMA contraction), for 1e-10 parity.
__device__ __forceinline__ void penalty(double r, double w, const Args& a, double& tw, double& g) {
  const double b = __dadd_rn(__dmul_rn(r, r), a.mu);
  double term;
  if (a.pmode == PM_TWO) term = b;
  else if (a.pmode == PM_ONE) term = sqrt(b);
  else term = exp(__dmul_rn(a.half_p, log(b)));
  tw = __dmul_rn(term, w);
  g = __dmul_rn(__dmul_rn(a.p, r), __ddiv_rn(tw, b));
}

__device__ __forceinline__ float trial(float r, float al, float ud) { return fmaf(-al, ud, r); }
__device__ __forceinline__ double trial(double r, double al, double ud) {
  return __dsub_rn(r, __dmul_rn(al, ud));
}

// ---------------------------------------------------------------------------
// reductions

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) x += __shfl_xor_sync(0xffffffffu, x, m);
  return x;
}

// Reduce one per-thread value over the CTA into sm[warp][slot] (lane 0 writes).
// ---------------------------------------------------------------------------
// Exchange region of one rank (prost_xpeer_handle allocates it, peers write it):
//   sums   [2 parity][world][S][nvmax] fp64   (parity = exchange sequence & 1)
//   flags  [world][S] u64                     (last sequence number received)
//   halos  [2 parity][2: row above, row below][S][width] u8
//   hflags [2: above, below][S] u64           (last frame received)
// Sequence numbers only grow, so flags need no parity; two data parities are
// enough because a rank cannot start exchange n+2 before every rank has
// contributed to n+1, i.e. finished reading n.
__host__ __device__ inline size_t xr_sums_bytes(int world, int S, int nv) {
  return (size_t)2 * world * S * nv * sizeof(double);
}
__host__ __device__ inline size_t xr_flags_off(int world, int S, int nv) { return xr_sums_bytes(world, S, nv); }
__host__ __device__ inline size_t xr_halo_off(int world, int S, int nv) {
  return (xr_flags_off(world, S, nv) + (size_t)world * S * 8 + 15) / 16 * 16;
}
__host__ __device__ inline size_t xr_hflags_off(int world, int S, int nv, int width) {
  return (xr_halo_off(world, S, nv) + (size_t)4 * S * width + 15) / 16 * 16;
}
__host__ __device__ inline size_t xr_bytes(int world, int S, int nv, int width) {
  return xr_hflags_off(world, S, nv, width) + (size_t)2 * S * 8;
}
__device__ __forceinline__ double* xr_sums(void* base, const Args& a, int par, int q, int s) {
  return static_cast<double*>(base) + (((size_t)par * a.xworld + q) * a.xS + s) * a.nvmax;
}
__device__ __forceinline__ unsigned long long* xr_flag(void* base, const Args& a, int q, int s) {
  return reinterpret_cast<unsigned long long*>(static_cast<uint8_t*>(base) + xr_flags_off(a.xworld, a.xS, a.nvmax)) +
         (size_t)q * a.xS + s;
}
__device__ __forceinline__ uint8_t* xr_halo(void* base, const Args& a, int par, int which) {
  return static_cast<uint8_t*>(base) + xr_halo_off(a.xworld, a.xS, a.nvmax) +
         ((size_t)par * 2 + which) * a.xS * a.width;
}
__device__ __forceinline__ unsigned long long* xr_hflag(void* base, const Args& a, int which, int s) {
  return reinterpret_cast<unsigned long long*>(static_cast<uint8_t*>(base) +
                                               xr_hflags_off(a.xworld, a.xS, a.nvmax, a.width)) +
         (size_t)which * a.xS + s;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// Spin until *p >= v; a rank that never arrives (a dead peer) traps after
// ~10 s instead of hanging the GPU.
__device__ __forceinline__ void wait_flag(const unsigned long long* p, unsigned long long v) {
  const long long t0 = clock64();
  while (ld_acquire_sys(p) < v) {
    __nanosleep(32);
    if (clock64() - t0 > 20000000000LL) __trap();
  }
}

// The cross-rank sum of one phase, run by the last CTA of stream s: red[0..nv)
// holds this rank's sums on entry and the all-rank sums, added in rank order,
// on exit — the same numbers on every rank.
template <int NTH>
__device__ __noinline__ void xpeer_exchange(const Args& a, int s, int nv, double* red) {
  __shared__ unsigned long long sseq;
  if (threadIdx.x == 0) {
    sseq = a.xseq[s] + 1;
    a.xseq[s] = sseq;
  }
  __syncthreads();
  const unsigned long long seq = sseq;
  const int par = (int)(seq & 1ull);
  for (int i = threadIdx.x; i < a.xworld * nv; i += NTH) {
    const int q = i / nv, v = i - q * nv;
    xr_sums(a.xpeer[q], a, par, a.xrank, s)[v] = red[v];  // peer store (NVLink)
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x < a.xworld) {
    __threadfence_system();
    st_release_sys(xr_flag(a.xpeer[threadIdx.x], a, a.xrank, s), seq);
    wait_flag(xr_flag(a.xpeer[a.xrank], a, threadIdx.x, s), seq);
  }
  __syncthreads();
  void* own = a.xpeer[a.xrank];
  for (int v = threadIdx.x; v < nv; v += NTH) {
    double acc = 0.0;
    for (int q = 0; q < a.xworld; ++q) acc += __ldcv(xr_sums(own, a, par, q, s) + v);
    red[v] = acc;
  }
  __syncthreads();
}

// Programmatic dependent launch: a phase kernel launched with programmatic
// stream serialization may be scheduled while its predecessor drains; it
// waits here for the predecessor's completion and memory, then allows its own
// successor to be scheduled.  Both are no-ops for an ordinary launch.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// NTH: threads of the CTA (the TMA-fed streamed kernels run 512).
template <int NTH = NT>
__device__ __forceinline__ void cta_stage(double x, double* sm, int slot, int nv) {
  x = warp_sum(x);
  if ((threadIdx.x & 31) == 0) sm[(threadIdx.x >> 5) * nv + slot] = x;
}

// Finish the CTA reduction: sum warps in order into this CTA's partial slot,
// then arrive; returns true in the last CTA of the stream, whose `red` holds
// the stream-wide sums (slots summed in slot order).
template <int NTH = NT>
__device__ __forceinline__ bool cta_finish(const Args& a, int s, double* sm, int nv, double* red) {
  constexpr int NWL = NTH / 32;
  __shared__ int last;
  double* slot = a.part + ((size_t)s * a.chunks + blockIdx.x) * a.nvmax;
  __syncthreads();
  for (int v = threadIdx.x; v < nv; v += NTH) {
    double acc = 0.0;
    for (int w = 0; w < NWL; ++w) acc += sm[w * nv + v];
    slot[v] = acc;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned prev = atomicAdd(a.cnt + s, 1u);
    last = (prev == (unsigned)(a.chunks - 1));
    if (last) a.cnt[s] = 0u;
  }
  __syncthreads();
  if (!last) return false;
  __threadfence();
  // Sum the chunk slots in a fixed order with the whole CTA: lane = value
  // (32 at a time), warp w = chunks w, w + NW, ... (four independent loads in
  // flight per lane), then the NW warp sums in warp order.
  const double* base = a.part + (size_t)s * a.chunks * a.nvmax;
  __shared__ double wsum[NWL][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int v0 = 0; v0 < nv; v0 += 32) {
    const int v = v0 + lane;
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
    if (v < nv) {
      int c = warp;
      for (; c + 3 * NWL < a.chunks; c += 4 * NWL) {
        acc0 += __ldcg(base + (size_t)c * a.nvmax + v);
        acc1 += __ldcg(base + (size_t)(c + NWL) * a.nvmax + v);
        acc2 += __ldcg(base + (size_t)(c + 2 * NWL) * a.nvmax + v);
        acc3 += __ldcg(base + (size_t)(c + 3 * NWL) * a.nvmax + v);
      }
      for (; c < a.chunks; c += NWL) acc0 += __ldcg(base + (size_t)c * a.nvmax + v);
    }
    wsum[warp][lane] = (acc0 + acc1) + (acc2 + acc3);
    __syncthreads();
    if (warp == 0 && v < nv) {
      double acc = 0.0;
      for (int w = 0; w < NWL; ++w) acc += wsum[w][lane];
      red[v] = acc;
      if (a.xred) a.xred[(size_t)s * a.nvmax + v] = acc;  // exchange mode: k_xlogic finishes
    }
    __syncthreads();
  }
  if (a.xpeer) xpeer_exchange<NTH>(a, s, nv, red);
  return a.xred == nullptr;
}

// Exchange mode: record whether this phase runs for stream s (block 0 only).
__device__ __forceinline__ void mark_go(const Args& a, int s, int go) {
  if (a.xgo && blockIdx.x == 0 && threadIdx.x == 0) a.xgo[s] = go;
}

// ---------------------------------------------------------------------------
// scalar part of the algorithm (warp 0 of the last CTA; lane j owns j)

__device__ __forceinline__ double step_size(const Args& a, long long i) {
  // tracker.py:99-103
  return fmax(exp(-a.tau * (double)i) * a.t_init, a.t_min);
}

__device__ __forceinline__ double alpha_at(const Args& a, int m) {
  // fit.py:124,134: alpha *= shrink, starting from initial_step
  double al = a.step0;
  for (int i = 0; i < m; ++i) al *= a.shrink;
  return al;
}

static_assert(sizeof(Ctl) % 8 == 0, "Ctl is copied as 8-byte words");

// Linkage of the scalar decision functions below (PROST_LOGIC=__forceinline__
// inlines them into every kernel).
#ifndef PROST_LOGIC
#define PROST_LOGIC __forceinline__
#endif

__device__ PROST_LOGIC void write_info(Ctl* c, const Args& a, int s) {
  if (!a.info || c->no_info) return;
  FitInfo fi;
  fi.fit_cost = c->f;
  fi.step = c->t;
  fi.frame_index = c->frame_index;
  fi.iterations = c->iterations;
  fi.cost_evals = c->cost_evals;
  fi.grad_evals = c->grad_evals;
  fi.status = c->status;
  a.info[s + c->info_slot] = fi;
}

// End of the CG loop: projected-gradient norm, geodesic scalars
// (manifold.py:130-197, tracker.py:140-143).
__device__ PROST_LOGIC void finish_frame(Ctl* c, const Args& a, int s, int lane) {
  const double t = step_size(a, c->frame_index);
  const double gj = lane < a.k ? c->grad[lane] : 0.0;  // = U^T eta
  const double yj = lane < a.k ? c->y[lane] : 0.0;
  const double g2 = warp_sum(gj * gj);
  const double rn = sqrt(warp_sum(yj * yj));
  // ||eta - U U^T eta||^2 = ||eta||^2 - ||U^T eta||^2 for orthonormal U
  const double ln = sqrt(fmax(c->gsq - g2, 0.0));
  const bool zero = (ln < NORM_FLOOR) || (rn < NORM_FLOOR) || (t == 0.0);
  if (!zero && lane < a.k) c->v[lane] = yj / rn;
  __syncwarp();
  if (lane == 0) {
    c->active = 0;
    c->t = t;
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

// Top of CG iteration c->it (fit.py:108-119).
__device__ PROST_LOGIC void begin_iteration(Ctl* c, const Args& a, int s, int lane) {
  if (lane == 0) {
    c->need_lsfb = 0;
    c->need_gradfb = 0;
  }
  __syncwarp();
  if (c->it >= a.max_iters) { finish_frame(c, a, s, lane); return; }
  const double gj = lane < a.k ? c->grad[lane] : 0.0;
  const double gn = sqrt(warp_sum(gj * gj));
  if (gn <= a.grad_tol) { finish_frame(c, a, s, lane); return; }
  double dj = lane < a.k ? c->d[lane] : 0.0;
  if (c->it > 0 && c->it % a.k == 0) dj = -gj;
  double slope = warp_sum(dj * gj);
  if (slope >= 0.0) {
    dj = -gj;
    slope = -gn * gn;
  }
  __syncwarp();
  if (lane < a.k) c->d[lane] = dj;
  __syncwarp();
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
__device__ PROST_LOGIC void complete_iteration(Ctl* c, const Args& a, int s, int lane, double alpha,
                                   double fnew, const double* gs, double gsq_new) {
  const double dj = lane < a.k ? c->d[lane] : 0.0;
  const double gold = lane < a.k ? c->grad[lane] : 0.0;
  const double gnew = lane < a.k ? -gs[lane] : 0.0;
  const double num = warp_sum(gnew * (gnew - gold));
  const double beta = fmax(0.0, num / (c->gnorm * c->gnorm));
  __syncwarp();
  if (lane < a.k) {
    c->y[lane] = c->y[lane] + alpha * dj;
    c->d[lane] = -gnew + beta * dj;
    c->grad[lane] = gnew;
  }
  __syncwarp();
  if (lane == 0) {
    c->pend_alpha = alpha;
    c->f = fnew;
    c->gsq = gsq_new;
    c->cost_evals += 1;
    c->grad_evals += 1;
    c->iterations = c->it + 1;
    c->it += 1;
  }
  __syncwarp();
  begin_iteration(c, a, s, lane);
}

__device__ PROST_LOGIC void fail_iteration(Ctl* c, const Args& a, int s, int lane) {
  // fit.py:133-134: no acceptable step -> leave the loop, residual unchanged
  if (lane == 0) c->pend_alpha = 0.0;
  __syncwarp();
  finish_frame(c, a, s, lane);
}

__device__ __forceinline__ void mark_nonfinite(Ctl* c, const Args& a, int s, int lane) {
  if (lane == 0) {
    c->p0_next = 0;
    c->status = ST_NONFINITE;
    c->active = 0;
    c->t = step_size(a, c->frame_index);
    write_info(c, a, s);
  }
  __syncwarp();
}

// ---------------------------------------------------------------------------
// Decisions after each reduction (warp 0; every lane sees the same `red`).
// Shared by the streamed phase kernels and the resident frame kernel.

// red: [0] cost, [1..K] sum_i U_ij g_i, [K+1] ||g||^2, [K+2] non-finite count
template <int K>
__device__ PROST_LOGIC void after_pass0(Ctl* c, const Args& a, int s, int lane, const double* red) {
  if (red[K + 2] > 0.0) { mark_nonfinite(c, a, s, lane); return; }
  if (lane < a.k) {
    const double gj = -red[1 + lane];  // fit.py:101: grad = -(U^T g)
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
  __syncwarp();
  begin_iteration(c, a, s, lane);
}

// red: [0..WC) trial costs, then per speculative slot mm: K gradient sums + ||g||^2
template <int K>
__device__ PROST_LOGIC void after_iter(Ctl* c, const Args& a, int s, int lane, const double* red, int wlo) {
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
      complete_iteration(c, a, s, lane, alpha, red[first], red + WC + mm * (K + 1),
                         red[WC + mm * (K + 1) + K]);
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
      fail_iteration(c, a, s, lane);
    } else if (lane == 0) {
      c->need_lsfb = 1;
      c->ls_next = nmax;
    }
  }
  __syncwarp();
}

// red: [0..cnt) trial costs for step indices base..base+cnt-1
__device__ PROST_LOGIC void after_lsfb(Ctl* c, const Args& a, int s, int lane, const double* red, int base) {
  const int cnt = (a.max_bt - base) < LSW ? (a.max_bt - base) : LSW;
  int first = -1;
  double alpha = alpha_at(a, base);
  for (int m = 0; m < cnt; ++m) {
    if (red[m] <= c->f + a.c_armijo * alpha * c->slope) {
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
      fail_iteration(c, a, s, lane);
    } else if (lane == 0) {
      c->ls_next = base + cnt;
    }
  }
  __syncwarp();
}

// red: [0..K) gradient sums at the accepted step, [K] ||g||^2
template <int K>
__device__ PROST_LOGIC void after_gradfb(Ctl* c, const Args& a, int s, int lane, const double* red) {
  if (lane == 0) c->need_gradfb = 0;
  __syncwarp();
  complete_iteration(c, a, s, lane, c->acc_alpha, c->acc_cost, red, red[K]);
}

}  // namespace prost
