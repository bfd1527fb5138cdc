// prost_stream_tma.cuh — TMA-fed streamed phase kernels (fp32, one channel,
// k > 20: BASELINE C4, whose 8.3M x 30 basis, 1 GB, cannot stay on chip).
//
// The plain streamed kernels (prost_phases.cuh) load every basis value and
// per-coordinate input with per-thread loads and compute on them as they
// arrive; at k = 30 they hold 60-90 values per thread, spill, and stall on
// the load scoreboard (ncu on C4's k_iter: 52% of the DRAM peak, half of the
// warp samples on long_sb).  Here each CTA (512 threads, one per SM — the
// tile ring takes most of shared memory) walks tiles of TT = 512 coordinates:
// thread 0 keeps NSTG tiles in flight, each tile one mbarrier and
//   - the basis: two 2-D tensor copies (cp.async.bulk.tensor) of
//     [k planes x 256 coordinates] from the [S*k][np] basis tensor map,
//   - the per-coordinate inputs of the phase (residual, u_dir, frame, mean,
//     labels): 1-D bulk copies (cp.async.bulk) of the tile's span,
// and every thread handles one coordinate of the tile already in shared
// memory.  The geodesic update writes U' over its own tile in shared memory
// and thread 0 stores it back with 2-D tensor stores (bulk groups).
// Same arithmetic per coordinate as k_pass0 / k_iter / k_gradfb / k_geo
// (fit.py:96-141, manifold.py:130-197, pipeline.py:158-175); only the order
// of the per-CTA partial sums differs (CTAs own contiguous tiles).
//
// Requirements (checked by the host, prost_b200.cu setup_tma / frame):
// C == 1, fp32, Pp % 16 == 0 (1-D bulk copies move multiples of 16 bytes),
// 16-byte aligned frame pointer.
#pragma once

#include <cuda.h>

#include "prost_phases.cuh"

namespace prost {

#ifndef PROST_TMA_ALT
#define PROST_TMA_ALT 1  // alternate the tile order of consecutive U passes (ring_geometry)
#endif

constexpr int TT = 512;       // threads per CTA = coordinates per tile
constexpr int TBOX = 256;     // tensor-map box width (box dims are <= 256)
constexpr int NSTG = 3;       // tiles in flight per CTA
constexpr int TSIDE = TT * 4; // bytes of one fp32 per-coordinate input per tile

__device__ __forceinline__ unsigned tma_smem(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

// Stage of a tile: basis [2 boxes][K][TBOX] fp32, NS fp32 side inputs, labels.
template <int K, int NS>
struct TStage {
  static constexpr size_t U_BYTES = (size_t)K * TT * 4;
  static constexpr size_t BYTES = U_BYTES + (size_t)NS * TSIDE + TT;
  static constexpr size_t SMEM = NSTG * BYTES + 64;
  static_assert(BYTES % 16 == 0, "stage alignment");
};

// Dynamic shared memory of the four kernels (host: cudaFuncSetAttribute).
template <int K>
__host__ __device__ constexpr size_t tma_smem_small() { return TStage<K, 2>::SMEM; }
template <int K>
__host__ __device__ constexpr size_t tma_smem_geo() { return TStage<K, 4>::SMEM; }
template <int K>
__host__ __device__ constexpr size_t tma_smem_geo_next() { return TStage<K, 5>::SMEM; }

// The tile ring of one CTA over tiles blockIdx.x, blockIdx.x + chunks, ...
// of stream s (rows s*k .. s*k+k-1 of the tensor map).
template <int K, int NS>
struct Ring {
  using St = TStage<K, NS>;
  uint8_t* base;
  uint64_t* bar;
  const CUtensorMap* map;
  const uint8_t* side[NS];  // per-stream base of each side input (null: not loaded)
  int side_es[NS];          // its element size (1 or 4)
  const uint8_t* lab;
  int k, row0, Pp, first, stride, ntiles;
  bool rev;  // walk this CTA's tiles last to first (see ring_geometry)

  __device__ __forceinline__ int tile_of(int i) const { return first + (rev ? ntiles - 1 - i : i) * stride; }
  __device__ __forceinline__ uint8_t* stage(int st) const { return base + (size_t)st * St::BYTES; }
  // basis value j of tile coordinate c (box c / TBOX lands as [k][TBOX])
  __device__ __forceinline__ float* urow(int st, int j, int c) const {
    return reinterpret_cast<float*>(stage(st)) + (size_t)(c / TBOX) * K * TBOX + (size_t)j * TBOX + (c % TBOX);
  }
  __device__ __forceinline__ const float* sidef(int st, int q) const {
    return reinterpret_cast<const float*>(stage(st) + St::U_BYTES + (size_t)q * TSIDE);
  }
  __device__ __forceinline__ const uint8_t* sideb(int st, int q) const {
    return stage(st) + St::U_BYTES + (size_t)q * TSIDE;
  }
  __device__ __forceinline__ const uint8_t* labs(int st) const {
    return stage(st) + St::U_BYTES + (size_t)NS * TSIDE;
  }

  __device__ __forceinline__ void issue(int i) const {
    const int st = i % NSTG, b = tile_of(i) * TT;
    const int n = min(TT, Pp - b);  // multiple of 16 (Pp % 16 == 0)
    const int nbox = n > TBOX ? 2 : 1;
    unsigned bytes = (unsigned)(nbox * k * TBOX * 4) + (unsigned)n;
#pragma unroll
    for (int q = 0; q < NS; ++q)
      if (side[q]) bytes += (unsigned)(n * side_es[q]);
    const unsigned mb = tma_smem(bar + st);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
    for (int h = 0; h < nbox; ++h)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3}], [%4];" ::"r"(tma_smem(urow(st, 0, h * TBOX))),
          "l"(map), "r"(b + h * TBOX), "r"(row0), "r"(mb)
          : "memory");
#pragma unroll
    for (int q = 0; q < NS; ++q)
      if (side[q])
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                tma_smem(sideb(st, q))),
            "l"(side[q] + (size_t)b * side_es[q]), "r"(n * side_es[q]), "r"(mb)
            : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            tma_smem(labs(st))),
        "l"(lab + b), "r"(n), "r"(mb)
        : "memory");
  }

  __device__ __forceinline__ void wait(int i) const {
    const unsigned mb = tma_smem(bar + i % NSTG);
    const unsigned par = (unsigned)(i / NSTG) & 1u;
    unsigned done = 0;
    long long spins = 0;
    for (;;) {
      asm volatile(
          "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
          " selp.u32 %0, 1, 0, p;\n}\n"
          : "=r"(done)
          : "r"(mb), "r"(par)
          : "memory");
      if (done) break;
      if (++spins > (1LL << 28)) __trap();  // a lost copy must not hang the GPU
    }
  }

  // barriers initialised, the first NSTG tiles in flight
  __device__ __forceinline__ void start(uint8_t* smem) {
    base = smem;
    bar = reinterpret_cast<uint64_t*>(smem + NSTG * St::BYTES);
    // rows k..K-1 of every box stay zero (the copies fill k rows), so the
    // unrolled K-row loops need no k guard: u = 0 there, as in the plain
    // kernels (and the direction / coefficient entries are 0 too)
    const int pad = (K - k) * TBOX;
    for (int e = threadIdx.x; e < NSTG * 2 * pad; e += blockDim.x) {
      const int st = e / (2 * pad), h = (e / pad) % 2, o = e % pad;
      urow(st, k, h * TBOX)[o] = 0.f;
    }
    if (threadIdx.x == 0) {
      for (int q = 0; q < NSTG; ++q)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tma_smem(bar + q)) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int q = 0; q < NSTG && q < ntiles; ++q) issue(q);
  }

  // every thread is done reading tile i: refill its stage with tile i + NSTG
  __device__ __forceinline__ void release(int i) const {
    __syncthreads();
    if (threadIdx.x == 0 && i + NSTG < ntiles) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(i + NSTG);
    }
  }
};

// Tile order: the chip walks the stream in bands of `chunks` tiles (band i =
// every CTA's i-th tile).  Consecutive U passes alternate direction — pass 0
// forward, CG iteration `it` backward when it is even, the plain geodesic
// sweep backward, so with two iterations the passes run F, R, F, R and the
// next frame's pass 0 F again — so each pass starts on the bands the previous
// one finished with, which are still in L2 (126 MB against a 1 GB basis at
// C4).  Passes with a reduction keep a fixed direction per pass (the partial
// sums' order, and so the bits, do not depend on the previous pass).
template <int K, int NS>
__device__ __forceinline__ void ring_geometry(Ring<K, NS>& R, const Args& a, int s, const CUtensorMap* map,
                                              bool rev = false) {
  R.rev = rev;
  R.map = map;
  R.k = a.k;
  R.row0 = s * a.k;
  R.Pp = a.Pp;
  const int nt = (a.Pp + TT - 1) / TT;
  R.first = blockIdx.x;
  R.stride = a.chunks;
  R.ntiles = nt > R.first ? (nt - R.first + R.stride - 1) / R.stride : 0;
  R.lab = a.lab + (size_t)s * a.Pp;
#pragma unroll
  for (int q = 0; q < NS; ++q) {
    R.side[q] = nullptr;
    R.side_es[q] = 4;
  }
}

// weight of coordinate pix from its label (load_weights, VEC = 1)
__device__ __forceinline__ float tile_weight(const Args& a, int pix, uint8_t l) {
  return pix < a.P ? (l ? (float)a.omega : 1.f) : 0.f;
}

// normalized() (VEC = 1) on the staged frame / mean values
__device__ __forceinline__ float tile_xhat(const Args& a, const uint8_t* xs, const float* ms, int c,
                                           float* M, int pix, bool upd, float seen, float stdv,
                                           bool& bad) {
  const float xv = a.xu8 ? u8_unit(xs[c]) : reinterpret_cast<const float*>(xs)[c];
  bad |= !isfinite(xv);
  if (!a.pipeline) return xv;
  float mv = ms[c];
  if (upd) {
    mv = add_rn(mv, norm_div(sub_rn(xv, mv), seen));
    M[pix] = mv;
  }
  return norm_div(sub_rn(xv, mv), stdv);
}

// ---------------------------------------------------------------------------
// pass 0 (fit.py:96-104): r = x - U y, cost, coordinate gradient
template <int K>
__global__ void __launch_bounds__(TT, 1) k_pass0_tma(const __grid_constant__ Args a,
                                                     const __grid_constant__ CUtensorMap map) {
  pdl_enter();
  extern __shared__ __align__(128) uint8_t tsm[];
  const int s = a.s0 + blockIdx.y;
  Ctl* c = a.ctl + s;
  __shared__ int go, upd;
  __shared__ double sstd, sseen;
  __shared__ float sy[K];
  if (threadIdx.x == 0) {
    go = c->status == ST_OK && c->p0_next != c->frame_index + 1;
    upd = c->update_stats;
    sstd = c->std_cur;
    sseen = (double)c->pseen;
  }
  if (threadIdx.x < K) sy[threadIdx.x] = threadIdx.x < a.k ? (float)c->y[threadIdx.x] : 0.f;
  __syncthreads();
  mark_go(a, s, go);
  if (!go) return;
  constexpr int NV = K + 3;
  __shared__ double sm[(TT / 32) * NV];
  __shared__ double red[NV];
  Ring<K, 2> R;
  ring_geometry(R, a, s, &map);
  R.side[0] = static_cast<const uint8_t*>(a.x) + (size_t)s * a.np * (a.xu8 ? 1 : 4);
  R.side_es[0] = a.xu8 ? 1 : 4;
  if (a.pipeline) R.side[1] = static_cast<const uint8_t*>(a.mean) + (size_t)s * a.np * 4;
  R.start(tsm);
  float acc[K];
#pragma unroll
  for (int j = 0; j < K; ++j) acc[j] = 0.f;
  double cost = 0.0;
  float gsq = 0.f;
  bool bad = false;
  const float seen = (float)sseen, stdv = (float)sstd;
  float* RR = static_cast<float*>(a.r) + (size_t)s * a.np;
  float* M = static_cast<float*>(a.mean) + (size_t)s * a.np;
  const int t = threadIdx.x;
  for (int i = 0; i < R.ntiles; ++i) {
    R.wait(i);
    const int st = i % NSTG, pix = R.tile_of(i) * TT + t;
    if (pix < a.Pp) {
      const float w = tile_weight(a, pix, R.labs(st)[t]);
      const float xh = tile_xhat(a, R.sideb(st, 0), R.sidef(st, 1), t, M, pix, upd, seen, stdv, bad);
      float uy = 0.f;
#pragma unroll
      for (int j = 0; j < K; ++j)
        uy += *R.urow(st, j, t) * sy[j];
      const float r = sub_rn(xh, uy);
      float tw, g;
      penalty(r, w, a, tw, g);
      cost += (double)tw;
      gsq += g * g;
#pragma unroll
      for (int j = 0; j < K; ++j)
        acc[j] += *R.urow(st, j, t) * g;
      RR[pix] = r;
    }
    R.release(i);
  }
  cta_stage<TT>(cost, sm, 0, NV);
#pragma unroll
  for (int j = 0; j < K; ++j) cta_stage<TT>((double)acc[j], sm, 1 + j, NV);
  cta_stage<TT>((double)gsq, sm, K + 1, NV);
  cta_stage<TT>(bad ? 1.0 : 0.0, sm, K + 2, NV);
  if (!cta_finish<TT>(a, s, sm, NV, red)) return;
  if (threadIdx.x < 32) after_pass0<K>(c, a, s, threadIdx.x, red);
}

// ---------------------------------------------------------------------------
// one CG iteration's U pass (fit.py:108-141): u_dir = U d, the window's trial
// costs, the speculative gradients
template <int K>
__global__ void __launch_bounds__(TT, 1) k_iter_tma(const __grid_constant__ Args a,
                                                    const __grid_constant__ CUtensorMap map) {
  pdl_enter();
  extern __shared__ __align__(128) uint8_t tsm[];
  const int s = a.s0 + blockIdx.y;
  Ctl* c = a.ctl + s;
  __shared__ int go, lo, back;
  __shared__ double spend;
  __shared__ __align__(16) float sd[K];
  if (threadIdx.x == 0) {
    go = c->status == ST_OK && c->active;
    lo = c->gwin_lo;
    spend = c->pend_alpha;
    back = PROST_TMA_ALT && (c->it % 2 == 0);
  }
  if (threadIdx.x < K) sd[threadIdx.x] = threadIdx.x < a.k ? (float)c->d[threadIdx.x] : 0.f;
  __syncthreads();
  mark_go(a, s, go);
  if (!go) return;
  constexpr int NV = WC + WG * (K + 1);
  __shared__ double sm[(TT / 32) * NV];
  __shared__ double red[NV];
  Ring<K, 2> R;
  ring_geometry(R, a, s, &map, back != 0);
  R.side[0] = static_cast<const uint8_t*>(a.r) + (size_t)s * a.np * 4;
  if (spend != 0.0) R.side[1] = static_cast<const uint8_t*>(a.ud) + (size_t)s * a.np * 4;
  R.start(tsm);
  float al[WC];
  {
    double v = a.step0;
#pragma unroll
    for (int m = 0; m < WC; ++m) {
      al[m] = (float)v;
      v *= a.shrink;
    }
  }
  const float pend = (float)spend;
  const bool moved = spend != 0.0;
  const int wlo = lo;
  double cost[WC];
#pragma unroll
  for (int m = 0; m < WC; ++m) cost[m] = 0.0;
  float gacc[WG][K], gsq[WG];
#pragma unroll
  for (int mm = 0; mm < WG; ++mm) {
    gsq[mm] = 0.f;
#pragma unroll
    for (int j = 0; j < K; ++j) gacc[mm][j] = 0.f;
  }
  float* RR = static_cast<float*>(a.r) + (size_t)s * a.np;
  float* UD = static_cast<float*>(a.ud) + (size_t)s * a.np;
  const int t = threadIdx.x;
  for (int i = 0; i < R.ntiles; ++i) {
    R.wait(i);
    const int st = i % NSTG, pix = R.tile_of(i) * TT + t;
    if (pix < a.Pp) {
      const float w = tile_weight(a, pix, R.labs(st)[t]);
      float r = R.sidef(st, 0)[t];
      if (moved) {
        r = trial(r, pend, R.sidef(st, 1)[t]);
        RR[pix] = r;
      }
      float ud = 0.f;
#pragma unroll
      for (int j = 0; j < K; ++j)
        ud += *R.urow(st, j, t) * sd[j];
      UD[pix] = ud;
      float gs[WG];
#pragma unroll
      for (int mm = 0; mm < WG; ++mm) gs[mm] = 0.f;
#pragma unroll
      for (int m = 0; m < WC; ++m) {
        float tw, g;
        penalty(trial(r, al[m], ud), w, a, tw, g);
        cost[m] += (double)tw;
#pragma unroll
        for (int mm = 0; mm < WG; ++mm)
          if (m == wlo + mm) gs[mm] = g;
      }
#pragma unroll
      for (int j = 0; j < K; ++j) {
        const float u = *R.urow(st, j, t);
#pragma unroll
        for (int mm = 0; mm < WG; ++mm) gacc[mm][j] += u * gs[mm];
      }
#pragma unroll
      for (int mm = 0; mm < WG; ++mm) gsq[mm] += gs[mm] * gs[mm];
    }
    R.release(i);
  }
#pragma unroll
  for (int m = 0; m < WC; ++m) cta_stage<TT>(cost[m], sm, m, NV);
#pragma unroll
  for (int mm = 0; mm < WG; ++mm) {
#pragma unroll
    for (int j = 0; j < K; ++j) cta_stage<TT>((double)gacc[mm][j], sm, WC + mm * (K + 1) + j, NV);
    cta_stage<TT>((double)gsq[mm], sm, WC + mm * (K + 1) + K, NV);
  }
  if (!cta_finish<TT>(a, s, sm, NV, red)) return;
  if (threadIdx.x < 32) after_iter<K>(c, a, s, threadIdx.x, red, wlo);
}

// ---------------------------------------------------------------------------
// the gradient at an accepted step outside the window (fit.py:137-141)
template <int K>
__global__ void __launch_bounds__(TT, 1) k_gradfb_tma(const __grid_constant__ Args a,
                                                      const __grid_constant__ CUtensorMap map) {
  pdl_enter();
  extern __shared__ __align__(128) uint8_t tsm[];
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
  __shared__ double sm[(TT / 32) * NV];
  __shared__ double red[NV];
  Ring<K, 2> R;
  ring_geometry(R, a, s, &map);
  R.side[0] = static_cast<const uint8_t*>(a.r) + (size_t)s * a.np * 4;
  R.side[1] = static_cast<const uint8_t*>(a.ud) + (size_t)s * a.np * 4;
  R.start(tsm);
  const float alpha = (float)salpha;
  float acc[K];
#pragma unroll
  for (int j = 0; j < K; ++j) acc[j] = 0.f;
  float gsq = 0.f;
  const int t = threadIdx.x;
  for (int i = 0; i < R.ntiles; ++i) {
    R.wait(i);
    const int st = i % NSTG, pix = R.tile_of(i) * TT + t;
    if (pix < a.Pp) {
      const float w = tile_weight(a, pix, R.labs(st)[t]);
      float tw, g;
      penalty(trial(R.sidef(st, 0)[t], alpha, R.sidef(st, 1)[t]), w, a, tw, g);
      gsq += g * g;
#pragma unroll
      for (int j = 0; j < K; ++j)
        acc[j] += *R.urow(st, j, t) * g;
    }
    R.release(i);
  }
#pragma unroll
  for (int j = 0; j < K; ++j) cta_stage<TT>((double)acc[j], sm, j, NV);
  cta_stage<TT>((double)gsq, sm, K, NV);
  if (!cta_finish<TT>(a, s, sm, NV, red)) return;
  if (threadIdx.x < 32) after_gradfb<K>(c, a, s, threadIdx.x, red);
}

// ---------------------------------------------------------------------------
// rank-one geodesic step of U (manifold.py:130-197) and the relabel /
// background / residual epilogue (pipeline.py:158-175) — k_geo<float, K, 1,
// false> with the basis tile updated in shared memory and stored back by TMA.
//
// NEXT (frame-blocked pushes, a.xnext = the next frame): pass 0 of the next
// frame runs in the same sweep, on U' while it is in shared memory, with the
// labels just computed as its weights and this frame's y as its warm start —
// r0 = x_{f+1}/std - U'y is the relabel's U'y (same operation order as
// k_pass0_tma, so the same bits), saving one pass over U per frame.  Only when
// the next frame does not update the running statistics (its normalization is
// then known here) and no periodic QR follows this frame; the last CTA does
// the next frame's start (what k_stats does for a frozen stream) and
// after_pass0, and marks the frame (Ctl::p0_next) so its own statistics and
// pass-0 kernels exit at once.  A non-finite next frame is left to its own
// pass 0 (which reports it).
template <int K, bool NEXT = false>
__global__ void __launch_bounds__(TT, 1) k_geo_tma(const __grid_constant__ Args a,
                                                   const __grid_constant__ CUtensorMap map) {
  pdl_enter();
  extern __shared__ __align__(128) uint8_t tsm[];
  const int s = a.s0 + blockIdx.y;
  Ctl* c = a.ctl + s;
  __shared__ int go, dogeo, relabel, fuse;
  __shared__ double sc[6];
  __shared__ __align__(16) float sv[K], sg[K], sy[K];
  if (threadIdx.x == 0) {
    go = c->status == ST_OK;
    dogeo = c->do_geo;
    relabel = !c->qr_now;
    sc[0] = c->geo_a;
    sc[1] = c->geo_s;
    sc[2] = c->geo_ln;
    sc[3] = c->pend_alpha;
    sc[4] = c->std_cur;
    int fu = 0;
    if (NEXT && a.xnext && go && relabel) {
      // the next frame (frame_index was advanced by this frame's finish)
      const bool upd1 = a.pipeline && !c->frozen && c->frame_index < a.i_init;
      fu = !upd1;
      sc[5] = !a.pipeline ? 1.0 : (c->frozen ? c->pstd : running_std(c));
    }
    fuse = fu;
  }
  if (threadIdx.x < K) {
    const int j = threadIdx.x;
    sv[j] = j < a.k ? (float)c->v[j] : 0.f;
    sg[j] = j < a.k ? (float)c->grad[j] : 0.f;
    sy[j] = j < a.k ? (float)c->y[j] : 0.f;
  }
  __syncthreads();
  if (!go) return;
  const float ga = (float)sc[0], gsn = (float)sc[1], ln = (float)sc[2], pend = (float)sc[3],
              stdv = (float)sc[4];
  const bool moved = sc[3] != 0.0;
  const bool do_geo = dogeo, do_lab = relabel, fu = NEXT && fuse;
  float* FRES = a.fitres_out ? static_cast<float*>(a.fitres_out) + (size_t)s * a.np : nullptr;
  float* RES = a.res_out ? static_cast<float*>(a.res_out) + (size_t)s * a.np : nullptr;
  float* BG = a.bg_out ? static_cast<float*>(a.bg_out) + (size_t)s * a.np : nullptr;
  float* RR = static_cast<float*>(a.r) + (size_t)s * a.np;
  uint8_t* L = a.lab + (size_t)s * a.Pp;
  uint8_t* RAW = a.raw_out ? a.raw_out + (size_t)s * a.Pp : nullptr;
  const bool need_r = FRES || do_geo;
  constexpr int NS = NEXT ? 5 : 4;
  Ring<K, NS> R;
  // backward, except when the next frame's pass 0 (a reduction) rides along:
  // it keeps k_pass0_tma's forward order, bit for bit
  ring_geometry(R, a, s, &map, PROST_TMA_ALT && !(NEXT && fu));
  if (need_r) R.side[0] = static_cast<const uint8_t*>(a.r) + (size_t)s * a.np * 4;
  if (need_r && moved) R.side[1] = static_cast<const uint8_t*>(a.ud) + (size_t)s * a.np * 4;
  if (do_lab) {
    R.side[2] = static_cast<const uint8_t*>(a.x) + (size_t)s * a.np * (a.xu8 ? 1 : 4);
    R.side_es[2] = a.xu8 ? 1 : 4;
    if (a.pipeline) R.side[3] = static_cast<const uint8_t*>(a.mean) + (size_t)s * a.np * 4;
  }
  if constexpr (NEXT) {
    if (fu) {
      R.side[4] = static_cast<const uint8_t*>(a.xnext) + (size_t)s * a.np * (a.xu8 ? 1 : 4);
      R.side_es[4] = a.xu8 ? 1 : 4;
    }
  }
  R.start(tsm);
  // next frame's pass 0 (NEXT): cost, coordinate gradient, ||g||^2, non-finite
  constexpr int KN = NEXT ? K : 1;
  float acc1[KN];
#pragma unroll
  for (int j = 0; j < KN; ++j) acc1[j] = 0.f;
  double cost1 = 0.0;
  float gsq1 = 0.f;
  bool bad1 = false;
  const float std1 = NEXT ? (float)sc[5] : 1.f;
  const int t = threadIdx.x;
  for (int i = 0; i < R.ntiles; ++i) {
    R.wait(i);
    const int st = i % NSTG, b = R.tile_of(i) * TT, pix = b + t;
    if (pix < a.Pp) {
      const float w = tile_weight(a, pix, R.labs(st)[t]);
      if (need_r) {
        float r = R.sidef(st, 0)[t];
        if (moved) r = trial(r, pend, R.sidef(st, 1)[t]);
        if (FRES) FRES[pix] = r;  // FitResult.residual (fit.py:50-63)
        if (do_geo) {
          float tw, g;
          penalty(r, w, a, tw, g);
          const float eta = -g;  // cost.py:103-112
          float uv = 0.f, ug = 0.f;
#pragma unroll
          for (int j = 0; j < K; ++j) {
            const float u = *R.urow(st, j, t);
            uv += u * sv[j];
            ug += u * sg[j];
          }
          const float proj = eta - ug;  // manifold.py:127
          const float coef = ga * uv - gsn * (proj / ln);
#pragma unroll
          for (int j = 0; j < K; ++j) {
            float* up = R.urow(st, j, t);
            *up = *up + coef * sv[j];
          }
        }
      }
      if (do_lab) {
        bool bad = false;
        const float xh = tile_xhat(a, R.sideb(st, 2), R.sidef(st, 3), t, nullptr, pix, false, 1.f, stdv, bad);
        float acc = 0.f;
#pragma unroll
        for (int j = 0; j < K; ++j) acc += *R.urow(st, j, t) * sy[j];
        const float rr = sub_rn(xh, acc);
        const float mx = fmaxf(0.f, fabsf(rr));
        if (RES) RES[pix] = rr;
        if (BG) BG[pix] = a.pipeline ? fminf(fmaxf(add_rn(acc * stdv, R.sidef(st, 3)[t]), 0.f), 1.f) : acc;
        const uint8_t lb = (pix < a.P && (double)mx >= a.delta) ? 1 : 0;
        L[pix] = lb;
        if (RAW) RAW[pix] = lb;
        if constexpr (NEXT) {
          if (fu) {  // pass 0 of the next frame (k_pass0_tma's operations)
            const float w1 = tile_weight(a, pix, lb);
            const float xh1 = tile_xhat(a, R.sideb(st, 4), R.sidef(st, 3), t, nullptr, pix, false, 1.f, std1, bad1);
            const float r0 = sub_rn(xh1, acc);
            float tw, g;
            penalty(r0, w1, a, tw, g);
            cost1 += (double)tw;
            gsq1 += g * g;
#pragma unroll
            for (int j = 0; j < K; ++j) acc1[j] += *R.urow(st, j, t) * g;
            RR[pix] = r0;
          }
        }
      }
    }
    if (do_geo) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // U' visible to the store
    __syncthreads();
    if (threadIdx.x == 0) {
      if (do_geo) {
        const int nbox = (a.Pp - b) > TBOX ? 2 : 1;
        for (int h = 0; h < nbox; ++h)
          asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&map),
                       "r"(b + h * TBOX), "r"(R.row0), "r"(tma_smem(R.urow(st, 0, h * TBOX)))
                       : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      // refill the stage of tile i - 1 once its store has read shared memory
      // (tile i's store is still running): NSTG - 1 tiles stay in flight
      if (i >= 1 && i - 1 + NSTG < R.ntiles) {
        if (do_geo) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        R.issue(i - 1 + NSTG);
      }
    }
  }
  if (threadIdx.x == 0 && do_geo) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  if constexpr (NEXT) {
    if (!fu) return;
    constexpr int NV = K + 3;
    __shared__ double sm[(TT / 32) * NV];
    __shared__ double red[NV];
    cta_stage<TT>(cost1, sm, 0, NV);
#pragma unroll
    for (int j = 0; j < K; ++j) cta_stage<TT>((double)acc1[j], sm, 1 + j, NV);
    cta_stage<TT>((double)gsq1, sm, K + 1, NV);
    cta_stage<TT>(bad1 ? 1.0 : 0.0, sm, K + 2, NV);
    if (!cta_finish<TT>(a, s, sm, NV, red)) return;
    if (threadIdx.x < 32 && red[K + 2] == 0.0) {
      if (threadIdx.x == 0) {  // the next frame's start (k_stats, frozen stream)
        if (a.pipeline && !c->frozen) {
          c->frozen = 1;
          c->pstd = sc[5];
        }
        c->std_cur = sc[5];
        c->update_stats = 0;
        c->status = ST_OK;
        c->p0_next = c->frame_index + 1;
      }
      __syncwarp();
      Args an = a;  // the next frame's FitInfo rows (a fit that ends at pass 0 reports there)
      an.info = a.info_next;
      after_pass0<K>(c, an, s, threadIdx.x, red);
    }
  }
}

}  // namespace prost
