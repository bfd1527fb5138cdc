// prost_b200.cu — host side of the C-ABI declared in include/prost_b200.h.
//
// A handle owns the device state of n_streams trackers (basis planes, labels,
// running statistics, control blocks) and enqueues one frame as a fixed
// sequence of phase kernels (prost_phases.cuh) on the caller's CUDA stream.
// Data-dependent control flow (Armijo fallbacks, periodic QR, first-frame
// cold start) is decided on the device: kernels whose condition is false for
// a stream exit immediately, so the host never synchronizes inside a frame.

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "../../include/prost_b200.h"
#include "prost_phases.cuh"
#include "prost_resident.cuh"
#include "prost_tmem.cuh"
#include "prost_stream_tma.cuh"
#include "kernel_ops.h"

using namespace prost;
using namespace prost_ops;

static_assert(sizeof(FitInfo) == sizeof(prost_fit_info), "FitInfo layout");

namespace {

struct Ops {
  void (*frame)(prost_handle*, Args&, cudaStream_t, int sw);
  void (*background)(prost_handle*, Args&, cudaStream_t, int sw);
  void (*qr)(prost_handle*, Args&, cudaStream_t, int sw);  // periodic QR pair only
  // exchange (pixel-sharded) mode: one phase kernel / the logic of a phase
  void (*step)(prost_handle*, Args&, cudaStream_t, int sw, int xs);
  void (*xlogic)(prost_handle*, Args&, cudaStream_t, int sw, int xs);
  int K, VEC;
};

}  // namespace

struct prost_handle {
  prost_params prm;
  int S = 0;
  uint32_t flags = 0;
  int device = 0;
  bool fp64 = false, pipeline = false;
  int k = 0, C = 1, P = 0, Pp = 0;
  long long np = 0;
  size_t esz = 4;
  int chunks = 1, nvmax = 0, wave = 0, n_ls = 0, sms = 148;
  Ops ops{};
  // resident modes (k_resident / k_tmem): team geometry and its scratch
  bool resident = false;
  bool tmem = false;
  int rG = 0, rT = 0, rqpc = 0, rnt = 0;
  int rng = 1;  // k_tmem slot groups per CTA
  bool tm_cl = false;  // k_tmem teams as thread-block clusters (team sums over DSMEM)
  bool pdl = false;    // streamed phase kernels with programmatic dependent launch (PROST_PDL)
  size_t rsmem = 0;
  unsigned* rbar = nullptr;
  double* rpart = nullptr;
  unsigned long long* rprof = nullptr;
  int resident_ops_K = 0;
  // streamed fp32 one-channel k > 20 (BASELINE C4): pass 0 / iteration /
  // gradient passes fed by tensor copies of U (prost_stream_tma.cuh)
  bool tma = false;
  bool tma_next = false;  // k_geo_tma<K, true> (next frame's pass 0 fused) fits shared memory
  int tma_chunks = 0;
  CUtensorMap umap{};
  // device state
  void* U = nullptr;
  void* r = nullptr;
  void* ud = nullptr;
  void* x = nullptr;
  void* mean = nullptr;
  uint8_t* lab = nullptr;
  uint8_t* labc = nullptr;  // 3-channel TMEM path: per-coordinate label flags
  Ctl* ctl = nullptr;
  double* part = nullptr;
  unsigned* cnt = nullptr;
  double* rinv = nullptr;
  FitInfo* info = nullptr;
  FitInfo* info_h = nullptr;  // pinned
  // non-blocking look at the FitInfo of the last push without a readback
  // (fit == nullptr): decides when the cold-start kernel can be skipped
  FitInfo* info_peek = nullptr;  // pinned
  cudaEvent_t ev_peek = nullptr;
  bool peek_pending = false;
  // lazily allocated
  void* bgbuf = nullptr;
  void* resbuf = nullptr;
  void* fresbuf = nullptr;  // fit residual (FitResult.residual) when it cannot be written in place
  // frame-blocked pushes (prost_push_many): [F][S][...] staging
  void* xblk = nullptr;
  size_t xblk_bytes = 0;
  void* oblk[3] = {nullptr, nullptr, nullptr};  // background, residual, fit residual
  size_t oblk_bytes = 0;
  uint8_t* rawblk = nullptr;
  uint8_t* maskblk = nullptr;
  size_t lblk_bytes = 0;
  FitInfo* infoblk = nullptr;
  int infoblk_n = 0;
  uint8_t* maskbuf = nullptr;
  // conversion staging: uploads (frames) and downloads (outputs) have their
  // own buffers, so a pipelined push's upload of frame N+1 on s_in never
  // overwrites frame N's outputs still being converted / copied out on s_out
  void* stage[2] = {nullptr, nullptr};
  size_t stage_bytes[2] = {0, 0};
  long long launches = 0;
  bool maybe_cold = true;
  // every stream is known (from a FitInfo readback or peek) to be past its
  // statistics window: the exchange program drops the statistics phase
  bool stats_over = false;
  // upper bound on every stream's steps-since-QR before the next push: the
  // periodic re-orthonormalization kernels are launched only when it can be due
  long long qr_bound = 0;
  bool qr_due = true;
  // exchange (pixel-sharded) mode: prost_xbegin / xnext / xapply / xfinish
  bool xmode = false;
  double* xred = nullptr;  // [S][nvmax] partial sums, summed over ranks by the caller
  int* xgo = nullptr;      // [S]
  long long n_real_glob = 0;
  long long frames_pushed = 0;
  std::vector<int> xprog;  // phase program of the frame in flight
  size_t xpc = 0;
  int xlast = -1;          // phase whose partials are in xred
  Args xa;
  prost_outputs xo{};
  bool xactive = false;
  // in-kernel exchange over peer memory (prost_xpeer_handle / prost_xpeer_open):
  // the frame runs as in single-GPU mode, the phase kernels exchange their sums
  // through every rank's exchange region themselves
  void* xp_region = nullptr;  // this rank's exchange region (cudaMalloc, exported by IPC)
  int xp_world = 0;           // world size the region was sized for
  std::vector<void*> xp_opened;  // peers' regions mapped through IPC
  void** xp_table = nullptr;  // device [world]: every rank's region
  unsigned long long* xseq = nullptr;  // device [S]
  int xrank = 0, xworld = 0;
  bool xpeer_on = false;
  long long xframe = 0;
  // pipelined host I/O (prost_push with host frames and host outputs): upload
  // on s_in, kernels on s_comp, download on s_out, double-buffered, so the
  // copies of one frame overlap the kernels of the next
  cudaStream_t s_in = nullptr, s_comp = nullptr, s_out = nullptr;
  cudaEvent_t ev_user = nullptr, ev_in[2] = {}, ev_comp[2] = {}, ev_out[2] = {};
  void* io_x[2] = {};
  void* io_bg[2] = {};
  void* io_res[2] = {};
  uint8_t* io_mask[2] = {};
  uint8_t* io_raw[2] = {};   // raw labels written by the kernels (pipelined host I/O)
  FitInfo* io_info[2] = {};  // per-slot FitInfo written by the kernels (fit_async)
  int io_slot = 0, io_last = 0;
  bool io_pending = false;
  // optional per-phase timing (prost_profile)
  bool prof = false;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> prof_ev;
  std::vector<cudaEvent_t> ev_pool;
  double prof_ms[PROST_N_PHASES] = {0};
  long long prof_n[PROST_N_PHASES] = {0};
  std::string err;
};

namespace {

int fail(prost_handle* h, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (h) h->err = buf;
  return code;
}

#define CK(call)                                                                      \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess)                                                            \
      return fail(h, PROST_ERR_CUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                                \
  } while (0)

inline int blocks_for(long long n, int t = NT) {
  long long b = (n + t - 1) / t;
  return (int)std::min<long long>(std::max<long long>(b, 1), 148LL * 16);
}

Args make_args(prost_handle* h, int s0) {
  Args a;
  std::memset(&a, 0, sizeof a);
  a.U = h->U;
  a.r = h->r;
  a.ud = h->ud;
  a.x = h->x;
  a.mean = h->mean;
  a.lab = h->lab;
  a.labc = h->labc;
  a.ctl = h->ctl;
  a.part = h->part;
  a.cnt = h->cnt;
  a.rinv = h->rinv;
  a.info = h->info;
  a.s0 = s0;
  a.k = h->k;
  a.C = h->C;
  a.P = h->P;
  a.Pp = h->Pp;
  a.width = h->prm.width;
  a.height = h->prm.height;
  a.np = h->np;
  a.chunks = h->chunks;
  a.nvmax = h->nvmax;
  a.pipeline = h->pipeline ? 1 : 0;
  a.max_iters = h->prm.cg_max_iters;
  a.max_bt = h->prm.max_backtracks;
  a.i_init = h->prm.i_init;
  const double p = h->prm.p;
  a.pmode = p == 2.0 ? PM_TWO : (p == 1.0 ? PM_ONE : ((p == 0.5 && !h->fp64) ? PM_HALF : PM_GENERAL));
  a.n_real = h->xmode ? h->n_real_glob : (long long)h->C * h->P;
  if (h->xmode && !h->xpeer_on) {
    a.xred = h->xred;
    a.xgo = h->xgo;
  }
  if (h->xpeer_on) {
    a.xpeer = h->xp_table;
    a.xseq = h->xseq;
    a.xrank = h->xrank;
    a.xworld = h->xworld;
    a.xS = h->S;
    a.xhalo = (h->xrank > 0 ? 1 : 0) | (h->xrank < h->xworld - 1 ? 2 : 0);
    a.xframe = h->xframe;
    const int par = (int)(h->xframe & 1);
    uint8_t* hb = static_cast<uint8_t*>(h->xp_region) + xr_halo_off(h->xworld, h->S, h->nvmax);
    if (a.xhalo & 1) a.halo_top = hb + (size_t)(par * 2 + 0) * h->S * h->prm.width;
    if (a.xhalo & 2) a.halo_bot = hb + (size_t)(par * 2 + 1) * h->S * h->prm.width;
  }
  a.p = p;
  a.half_p = 0.5 * p;
  a.mu = h->prm.mu;
  a.delta = h->prm.delta;
  a.omega = h->prm.omega;
  a.t_init = h->prm.t_init;
  a.t_min = h->prm.t_min;
  a.tau = h->prm.tau;
  a.grad_tol = h->prm.grad_tol;
  a.step0 = h->prm.initial_step;
  a.shrink = h->prm.shrink;
  a.c_armijo = h->prm.sufficient_decrease;
  a.pf = (float)a.p;
  a.half_pf = (float)a.half_p;
  a.muf = (float)a.mu;
  a.omegaf = (float)a.omega;
  a.deltaf = (float)a.delta;
  if ((double)a.deltaf < a.delta) a.deltaf = std::nextafter(a.deltaf, INFINITY);
  return a;
}

cudaEvent_t take_event(prost_handle* h) {
  if (!h->ev_pool.empty()) {
    cudaEvent_t e = h->ev_pool.back();
    h->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

// Records a CUDA event pair around one kernel launch when profiling is on.
struct PhaseTimer {
  prost_handle* h;
  cudaStream_t st;
  int phase;
  cudaEvent_t e0 = nullptr;
  PhaseTimer(prost_handle* h_, cudaStream_t st_, int ph) : h(h_), st(st_), phase(ph) {
    if (h->prof) {
      e0 = take_event(h);
      cudaEventRecord(e0, st);
    }
  }
  ~PhaseTimer() {
    if (h->prof) {
      cudaEvent_t e1 = take_event(h);
      cudaEventRecord(e1, st);
      h->prof_ev.push_back({phase, {e0, e1}});
    }
  }
};

// 3x3 majority filter of the raw labels into a.mask_out (pipeline.py:215-228)
// Launch a phase kernel; pdl: with programmatic stream serialization (the
// kernel starts with pdl_enter, prost_kernels.cuh), so its launch and ramp
// overlap the predecessor's drain.
template <typename... P, typename... A>
void launchk(bool pdl, void (*k)(P...), dim3 g, dim3 b, size_t sm, cudaStream_t st, A&&... args) {
  if (!pdl) {
    k<<<g, b, sm, st>>>(std::forward<A>(args)...);
    return;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = g;
  cfg.blockDim = b;
  cfg.dynamicSmemBytes = sm;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, std::forward<A>(args)...);
}

void launch_median(prost_handle* h, const Args& a, cudaStream_t st, int sw, bool pdl = false) {
  const uintptr_t al = (uintptr_t)a.mask_out | (uintptr_t)a.halo_top | (uintptr_t)a.halo_bot;
  // CTAs per stream: at most 128, or ~8 per SM over the launch when there
  // are few streams (one 3840x2160 stream: 1184 CTAs, not 128 latency-bound
  // ones looping 16 times; 19 -> ~5 us per frame)
  const int cap = std::max(128, 8 * h->sms / std::max(1, sw));
  if (h->prm.width % 16 == 0 && (al & 15) == 0 && h->Pp % 16 == 0) {
    const int nw = h->P / 16;
    const dim3 mg(std::max(1, std::min((nw + NT - 1) / NT, cap)), sw);
    launchk(pdl, k_median16, mg, dim3(NT), 0, st, a);
  } else if (h->prm.width % 4 == 0 && ((uintptr_t)a.mask_out & 3) == 0) {
    const int nw = h->P / 4;
    const dim3 mg(std::max(1, std::min((nw + NT - 1) / NT, cap)), sw);
    launchk(pdl, k_median4, mg, dim3(NT), 0, st, a);
  } else {
    const dim3 mg(std::max(1, std::min((h->P + NT - 1) / NT, std::max(64, cap))), sw);
    launchk(pdl, k_median, mg, dim3(NT), 0, st, a);
  }
}

#define LAUNCH(phase, ...)                  \
  do {                                      \
    PhaseTimer pt_(h, st, phase);           \
    __VA_ARGS__;                            \
    ++n;                                    \
  } while (0)

template <typename T, int K>
struct Impl {
  static constexpr int VEC = Vec<T, K>::value;

  static void frame(prost_handle* h, Args& a, cudaStream_t st, int sw) {
    const dim3 grid(h->chunks, sw);
    long long n = 0;
    LAUNCH(PROST_PH_STATS, (launchk(h->pdl, k_stats<T, VEC>, grid, dim3(NT), 0, st, a)));
    if (h->maybe_cold) LAUNCH(PROST_PH_COLD, (launchk(h->pdl, k_cold<T, K, VEC>, grid, dim3(NT), 0, st, a)));
    // tensor-copy-fed U passes (prost_stream_tma.cuh): frame pointer aligned
    // for the 1-D bulk copies
    bool fed = false;
    if constexpr (std::is_same<T, float>::value && K > 20) {
      if (h->tma && ((uintptr_t)a.x & 15) == 0) {
        fed = true;
        Args at = a;
        at.chunks = h->tma_chunks;
        const dim3 tg(h->tma_chunks, sw);
        constexpr size_t sm = tma_smem_small<K>(), sg = tma_smem_geo<K>();
        LAUNCH(PROST_PH_PASS0, (launchk(h->pdl, k_pass0_tma<K>, tg, dim3(TT), sm, st, at, h->umap)));
        for (int it = 0; it < h->prm.cg_max_iters; ++it) {
          LAUNCH(PROST_PH_ITER, (launchk(h->pdl, k_iter_tma<K>, tg, dim3(TT), sm, st, at, h->umap)));
          for (int l = 0; l < h->n_ls; ++l) LAUNCH(PROST_PH_LSFB, (launchk(h->pdl, k_lsfb<T, VEC>, grid, dim3(NT), 0, st, a)));
          LAUNCH(PROST_PH_GRADFB, (launchk(h->pdl, k_gradfb_tma<K>, tg, dim3(TT), sm, st, at, h->umap)));
        }
        if (a.xnext && h->tma_next && ((uintptr_t)a.xnext & 15) == 0)
          LAUNCH(PROST_PH_GEO, (launchk(h->pdl, k_geo_tma<K, true>, tg, dim3(TT), tma_smem_geo_next<K>(), st, at, h->umap)));
        else
          LAUNCH(PROST_PH_GEO, (launchk(h->pdl, k_geo_tma<K>, tg, dim3(TT), sg, st, at, h->umap)));
      }
    }
    if (!fed) {
      LAUNCH(PROST_PH_PASS0, (launchk(h->pdl, k_pass0<T, K, VEC>, grid, dim3(NT), 0, st, a)));
      for (int it = 0; it < h->prm.cg_max_iters; ++it) {
        LAUNCH(PROST_PH_ITER, (launchk(h->pdl, k_iter<T, K, VEC>, grid, dim3(NT), 0, st, a)));
        for (int l = 0; l < h->n_ls; ++l) LAUNCH(PROST_PH_LSFB, (launchk(h->pdl, k_lsfb<T, VEC>, grid, dim3(NT), 0, st, a)));
        LAUNCH(PROST_PH_GRADFB, (launchk(h->pdl, k_gradfb<T, K, VEC>, grid, dim3(NT), 0, st, a)));
      }
      LAUNCH(PROST_PH_GEO, (launchk(h->pdl, k_geo<T, K, VEC, false>, grid, dim3(NT), 0, st, a)));
    }
    if (h->qr_due) {
      LAUNCH(PROST_PH_QR, (launchk(h->pdl, k_gram<T, K, VEC>, grid, dim3(NT), 0, st, a)));
      LAUNCH(PROST_PH_QR, (launchk(h->pdl, k_geo<T, K, VEC, true>, grid, dim3(NT), 0, st, a)));
    }
    if (a.mask_out) {
      if (a.xpeer && a.xhalo) LAUNCH(PROST_PH_MEDIAN, (launchk(h->pdl, k_halo_push, dim3(1, sw), dim3(NT), 0, st, a)));
      LAUNCH(PROST_PH_MEDIAN, launch_median(h, a, st, sw, h->pdl));
    }
    h->launches += n;
  }

  static void qr(prost_handle* h, Args& a, cudaStream_t st, int sw) {
    const dim3 grid(h->chunks, sw);
    long long n = 0;
    LAUNCH(PROST_PH_QR, (k_gram<T, K, VEC><<<grid, NT, 0, st>>>(a)));
    LAUNCH(PROST_PH_QR, (k_geo<T, K, VEC, true><<<grid, NT, 0, st>>>(a)));
    h->launches += n;
  }

  static void background(prost_handle* h, Args& a, cudaStream_t st, int sw) {
    k_background<T, K, VEC><<<dim3(h->chunks, sw), NT, 0, st>>>(a);
    h->launches += 1;
  }

  static void step(prost_handle* h, Args& a, cudaStream_t st, int sw, int xs) {
    const dim3 grid(h->chunks, sw);
    long long n = 0;
    if constexpr (std::is_same<T, float>::value && K > 20) {
      if (h->tma && ((uintptr_t)a.x & 15) == 0 &&
          (xs == XS_PASS0 || xs == XS_ITER || xs == XS_GRADFB || xs == XS_GEO)) {
        Args at = a;
        at.chunks = h->tma_chunks;
        const dim3 tg(h->tma_chunks, sw);
        constexpr size_t sm = tma_smem_small<K>(), sg = tma_smem_geo<K>();
        switch (xs) {
          case XS_PASS0: LAUNCH(PROST_PH_PASS0, (k_pass0_tma<K><<<tg, TT, sm, st>>>(at, h->umap))); break;
          case XS_ITER: LAUNCH(PROST_PH_ITER, (k_iter_tma<K><<<tg, TT, sm, st>>>(at, h->umap))); break;
          case XS_GRADFB: LAUNCH(PROST_PH_GRADFB, (k_gradfb_tma<K><<<tg, TT, sm, st>>>(at, h->umap))); break;
          default: LAUNCH(PROST_PH_GEO, (k_geo_tma<K><<<tg, TT, sg, st>>>(at, h->umap))); break;
        }
        h->launches += n;
        return;
      }
    }
    switch (xs) {
      case XS_STATS:
      case XS_START: LAUNCH(PROST_PH_STATS, (k_stats<T, VEC><<<grid, NT, 0, st>>>(a))); break;
      case XS_COLD: LAUNCH(PROST_PH_COLD, (k_cold<T, K, VEC><<<grid, NT, 0, st>>>(a))); break;
      case XS_PASS0: LAUNCH(PROST_PH_PASS0, (k_pass0<T, K, VEC><<<grid, NT, 0, st>>>(a))); break;
      case XS_ITER: LAUNCH(PROST_PH_ITER, (k_iter<T, K, VEC><<<grid, NT, 0, st>>>(a))); break;
      case XS_LSFB: LAUNCH(PROST_PH_LSFB, (k_lsfb<T, VEC><<<grid, NT, 0, st>>>(a))); break;
      case XS_GRADFB: LAUNCH(PROST_PH_GRADFB, (k_gradfb<T, K, VEC><<<grid, NT, 0, st>>>(a))); break;
      case XS_GEO: LAUNCH(PROST_PH_GEO, (k_geo<T, K, VEC, false><<<grid, NT, 0, st>>>(a))); break;
      case XS_GRAM: LAUNCH(PROST_PH_QR, (k_gram<T, K, VEC><<<grid, NT, 0, st>>>(a))); break;
      case XS_GEOQR: LAUNCH(PROST_PH_QR, (k_geo<T, K, VEC, true><<<grid, NT, 0, st>>>(a))); break;
      default: break;
    }
    h->launches += n;
  }

  static void xlogic(prost_handle* h, Args& a, cudaStream_t st, int sw, int xs) {
    k_xlogic<K><<<sw, 32, 0, st>>>(a, xs);
    h->launches += 1;
  }
};

// Tensor map of the basis planes, [S*k rows][np coordinates] fp32, read in
// boxes of k rows x TBOX coordinates (prost_stream_tma.cuh).  The driver entry
// point is looked up at run time (no -lcuda).  PROST_TMA=0 keeps the plain
// streamed kernels.
typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int K>
bool tma_attrs() {
  const int sm = (int)tma_smem_small<K>(), sg = (int)tma_smem_geo<K>();
  return cudaFuncSetAttribute(k_pass0_tma<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm) == cudaSuccess &&
         cudaFuncSetAttribute(k_iter_tma<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm) == cudaSuccess &&
         cudaFuncSetAttribute(k_gradfb_tma<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm) == cudaSuccess &&
         cudaFuncSetAttribute(k_geo_tma<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, sg) == cudaSuccess;
}

template <int K>
bool tma_attr_next() {
  return cudaFuncSetAttribute(k_geo_tma<K, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)tma_smem_geo_next<K>()) == cudaSuccess;
}

void setup_tma(prost_handle* h, int sms) {
  const char* env = getenv("PROST_TMA");
  if ((env && env[0] == '0') || h->Pp % 16 != 0) return;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !fn) {
    cudaGetLastError();
    return;
  }
  const cuuint64_t dims[2] = {(cuuint64_t)h->np, (cuuint64_t)h->S * h->k};
  const cuuint64_t strides[1] = {(cuuint64_t)h->np * 4};
  const cuuint32_t box[2] = {(cuuint32_t)TBOX, (cuuint32_t)h->k};
  const cuuint32_t estr[2] = {1, 1};
  if (reinterpret_cast<EncodeTiled>(fn)(&h->umap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, h->U, dims, strides, box, estr,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return;
  const bool ok = h->ops.K == 30 ? tma_attrs<30>() : h->ops.K == 32 ? tma_attrs<32>() : false;
  if (!ok) {
    cudaGetLastError();
    return;
  }
  // the geodesic sweep with the next frame's pass 0 (frame-blocked pushes):
  // one more staged input per tile; used only if its shared memory fits
  h->tma_next = h->ops.K == 30 ? tma_attr_next<30>() : h->ops.K == 32 ? tma_attr_next<32>() : false;
  cudaGetLastError();
  // one CTA per SM (the tile ring takes most of shared memory), at most the
  // part slots the plain kernels use, at least one tile per CTA
  const long long tiles = (h->Pp + TT - 1) / TT;
  const long long per = std::max<long long>(1, (long long)sms / h->S);
  h->tma_chunks = (int)std::max<long long>(1, std::min<long long>({per, tiles, (long long)h->chunks}));
  h->tma = true;
}

template <typename T>
Ops pick(int k) {
#define PROST_K(KK) \
  if (k <= KK) \
    return Ops{&Impl<T, KK>::frame, &Impl<T, KK>::background, &Impl<T, KK>::qr, &Impl<T, KK>::step, \
               &Impl<T, KK>::xlogic, KK, Impl<T, KK>::VEC};
  PROST_K(4)
  PROST_K(8)
  PROST_K(15)
  PROST_K(16)
  PROST_K(20)
  PROST_K(30)
  PROST_K(32)
#undef PROST_K
  return Ops{nullptr, nullptr, nullptr, nullptr, nullptr, 0, 0};
}

int validate(prost_handle* h, const prost_params* p, int n_streams) {
  // The reference's own checks (tracker.py:64-76, cost.py:41-45, fit.py:35-47)
  // plus the limits of this implementation.
  if (p->k < 1) return fail(h, PROST_ERR_CONFIG, "subspace dimension must be >= 1, got %d", p->k);
  if (!(p->p > 0.0 && p->p <= 2.0)) return fail(h, PROST_ERR_CONFIG, "p must be in (0, 2], got %g", p->p);
  if (!(p->mu > 0.0)) return fail(h, PROST_ERR_CONFIG, "mu must be > 0, got %g", p->mu);
  if (!(p->delta > 0.0)) return fail(h, PROST_ERR_CONFIG, "delta must be > 0, got %g", p->delta);
  if (!(p->omega > 0.0 && p->omega <= 1.0))
    return fail(h, PROST_ERR_CONFIG, "omega must be in (0, 1], got %g", p->omega);
  if (!(p->t_min > 0.0 && p->t_min <= p->t_init))
    return fail(h, PROST_ERR_CONFIG, "need 0 < t_min <= t_init, got t_min=%g, t_init=%g", p->t_min, p->t_init);
  if (!(p->tau >= 0.0)) return fail(h, PROST_ERR_CONFIG, "tau must be >= 0, got %g", p->tau);
  if (p->cg_max_iters < 1) return fail(h, PROST_ERR_CONFIG, "max_iters must be >= 1, got %d", p->cg_max_iters);
  if (!(p->grad_tol >= 0.0)) return fail(h, PROST_ERR_CONFIG, "grad_tol must be >= 0, got %g", p->grad_tol);
  if (!(p->shrink > 0.0 && p->shrink < 1.0)) return fail(h, PROST_ERR_CONFIG, "shrink must be in (0, 1), got %g", p->shrink);
  if (!(p->sufficient_decrease > 0.0 && p->sufficient_decrease <= 0.5))
    return fail(h, PROST_ERR_CONFIG, "sufficient_decrease must be in (0, 0.5], got %g", p->sufficient_decrease);
  if (p->max_backtracks < 1) return fail(h, PROST_ERR_CONFIG, "max_backtracks must be >= 1, got %d", p->max_backtracks);
  if (p->max_backtracks > MAXBT) return fail(h, PROST_ERR_CONFIG, "max_backtracks > %d is not supported", MAXBT);
  if (!(p->initial_step > 0.0)) return fail(h, PROST_ERR_CONFIG, "initial_step must be > 0");
  if (p->i_init < 1) return fail(h, PROST_ERR_CONFIG, "i_init must be >= 1, got %d", p->i_init);
  if (p->channels != 1 && p->channels != 3)
    return fail(h, PROST_ERR_DIMENSION, "channels must be 1 or 3, got %d", p->channels);
  if (p->width < 1 || p->height < 1) return fail(h, PROST_ERR_DIMENSION, "bad dimensions %dx%d", p->width, p->height);
  const long long n = (long long)p->width * p->height * p->channels;
  if (!(p->k < n)) return fail(h, PROST_ERR_DIMENSION, "need 1 <= k < m, got m=%lld, k=%d", n, p->k);
  if (p->k > KMAX) return fail(h, PROST_ERR_CONFIG, "k=%d exceeds the supported maximum %d", p->k, KMAX);
  if (n_streams < 1) return fail(h, PROST_ERR_CONFIG, "n_streams must be >= 1");
  if ((long long)p->width * p->height >= (1LL << 30)) return fail(h, PROST_ERR_DIMENSION, "frame too large");
  return PROST_OK;
}

void* dev_alloc(size_t bytes, cudaError_t* e) {
  void* p = nullptr;
  *e = cudaMalloc(&p, std::max<size_t>(bytes, 16));
  if (*e == cudaSuccess) *e = cudaMemset(p, 0, std::max<size_t>(bytes, 16));
  return p;
}

enum { STAGE_IN = 0, STAGE_OUT = 1 };
int ensure_stage(prost_handle* h, int which, size_t bytes) {
  if (h->stage_bytes[which] >= bytes) return PROST_OK;
  if (h->stage[which]) cudaFree(h->stage[which]);
  h->stage[which] = nullptr;
  h->stage_bytes[which] = 0;
  CK(cudaMalloc(&h->stage[which], bytes));
  h->stage_bytes[which] = bytes;
  return PROST_OK;
}

size_t dtype_size(int dt) { return dt == PROST_F64 ? 8 : (dt == PROST_U8 ? 1 : 4); }

// Copy a dense [S][C][P] array of dtype `dt` (host or device) into a padded
// device array of the handle's element type.
int upload_dense(prost_handle* h, const void* src, int dt, int on_device, void* dst, int rows,
                 cudaStream_t st) {
  const int P = h->P, Pp = h->Pp;
  const size_t dsz = dtype_size(dt);
  const bool same = (dt == PROST_F64) == h->fp64 && dt != PROST_U8;
  if (same) {
    CK(cudaMemcpy2DAsync(dst, (size_t)Pp * h->esz, src, (size_t)P * dsz, (size_t)P * dsz, rows,
                         on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
    return PROST_OK;
  }
  const void* dsrc = src;
  if (!on_device) {
    int rc = ensure_stage(h, STAGE_IN, (size_t)rows * P * dsz);
    if (rc) return rc;
    CK(cudaMemcpyAsync(h->stage[STAGE_IN], src, (size_t)rows * P * dsz, cudaMemcpyHostToDevice, st));
    dsrc = h->stage[STAGE_IN];
  }
  const int nb = blocks_for((long long)rows * P);
  const double sc = dt == PROST_U8 ? 1.0 / 255.0 : 1.0;
  if (h->fp64) {
    if (dt == PROST_F32) k_pack<float, double><<<nb, NT, 0, st>>>((const float*)dsrc, (double*)dst, rows, 1, P, Pp, 1, sc);
    else k_pack<uint8_t, double><<<nb, NT, 0, st>>>((const uint8_t*)dsrc, (double*)dst, rows, 1, P, Pp, 1, sc);
  } else {
    if (dt == PROST_F64) k_pack<double, float><<<nb, NT, 0, st>>>((const double*)dsrc, (float*)dst, rows, 1, P, Pp, 1, sc);
    else k_pack<uint8_t, float><<<nb, NT, 0, st>>>((const uint8_t*)dsrc, (float*)dst, rows, 1, P, Pp, 1, sc);
  }
  h->launches += 1;
  CK(cudaGetLastError());
  return PROST_OK;
}

// Copy a padded device array of the handle's element type into a dense user
// array [rows][P] of dtype dt (host or device).
int download_dense(prost_handle* h, const void* src, void* dst, int dt, int on_device, int rows,
                   cudaStream_t st) {
  const int P = h->P, Pp = h->Pp;
  const size_t dsz = dtype_size(dt);
  const bool same = (dt == PROST_F64) == h->fp64 && dt != PROST_U8;
  if (same) {
    CK(cudaMemcpy2DAsync(dst, (size_t)P * dsz, src, (size_t)Pp * h->esz, (size_t)P * dsz, rows,
                         on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
    return PROST_OK;
  }
  if (dt == PROST_U8) return fail(h, PROST_ERR_CONFIG, "u8 is an input-only dtype");
  void* ddst = dst;
  if (!on_device) {
    int rc = ensure_stage(h, STAGE_OUT, (size_t)rows * P * dsz);
    if (rc) return rc;
    ddst = h->stage[STAGE_OUT];
  }
  const int nb = blocks_for((long long)rows * P);
  if (h->fp64) k_pack<double, float><<<nb, NT, 0, st>>>((const double*)src, (float*)ddst, rows, 1, P, Pp, 0, 1.0);
  else k_pack<float, double><<<nb, NT, 0, st>>>((const float*)src, (double*)ddst, rows, 1, P, Pp, 0, 1.0);
  h->launches += 1;
  CK(cudaGetLastError());
  if (!on_device) CK(cudaMemcpyAsync(dst, ddst, (size_t)rows * P * dsz, cudaMemcpyDeviceToHost, st));
  return PROST_OK;
}

int copy_labels(prost_handle* h, const uint8_t* src, uint8_t* dst, int on_device, cudaStream_t st) {
  CK(cudaMemcpy2DAsync(dst, h->P, src, h->Pp, h->P, h->S,
                       on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
  return PROST_OK;
}

// Retire a finished non-blocking FitInfo peek (see push_outputs).
void retire_peek(prost_handle* h) {
  if (!h->peek_pending || cudaEventQuery(h->ev_peek) != cudaSuccess) return;
  bool cold = false, over = true;
  for (int s = 0; s < h->S; ++s) {
    cold |= h->info_peek[s].frame_index == 0;
    over &= h->info_peek[s].frame_index > h->prm.i_init;  // frozen (pipeline.py:142-146)
  }
  h->maybe_cold = cold;
  h->stats_over = h->stats_over || over;
  h->peek_pending = false;
}

int check_stream(prost_handle* h, int s) {
  if (!h) return PROST_ERR_CONFIG;
  if (s < 0 || s >= h->S) return fail(h, PROST_ERR_DIMENSION, "stream %d out of range [0, %d)", s, h->S);
  return PROST_OK;
}

template <typename T>
void rows_to_planes(const double* U, int n_rows_dense, int k, int C, int P, int Pp, std::vector<T>& out) {
  // U row-major [C*P][k] -> planes [k][C*Pp]
  const size_t np = (size_t)C * Pp;
  out.assign((size_t)k * np, (T)0);
  for (int c = 0; c < C; ++c)
    for (int p = 0; p < P; ++p) {
      const size_t row = (size_t)c * P + p;
      for (int j = 0; j < k; ++j) out[(size_t)j * np + (size_t)c * Pp + p] = (T)U[row * k + j];
    }
  (void)n_rows_dense;
}

}  // namespace

// prost_push, first half: validation, QR due-check, frame upload, output
// routing.  Fills *ap / *op for the kernels and push_outputs.
int push_setup(prost_handle* h, const void* frames, int32_t dtype, int32_t on_device,
               const prost_outputs* out, cudaStream_t st, Args* ap, prost_outputs* op) {
  if (!h) return PROST_ERR_CONFIG;
  if (!frames) return fail(h, PROST_ERR_DIMENSION, "frames is NULL");
  if (dtype != PROST_F32 && dtype != PROST_F64 && dtype != PROST_U8)
    return fail(h, PROST_ERR_CONFIG, "unknown frame dtype %d", dtype);
  CK(cudaSetDevice(h->device));
  retire_peek(h);
  // A QR is due in this push only for a stream whose steps-since-QR is already
  // QR_EVERY - 1 (manifold.py:192).  Near that bound, refresh it from the
  // device (one small synchronous read every ~QR_EVERY frames).
  if (h->qr_bound >= QR_EVERY - 1) {
    std::vector<Ctl> cs(h->S);
    CK(cudaDeviceSynchronize());  // every stream (also the pipelined-I/O ones) is done with ctl
    CK(cudaMemcpy(cs.data(), h->ctl, (size_t)h->S * sizeof(Ctl), cudaMemcpyDeviceToHost));
    long long mx = 0;
    for (const Ctl& c : cs) mx = std::max(mx, c.since_qr);
    h->qr_bound = mx;
  }
  h->qr_due = h->qr_bound >= QR_EVERY - 1;
  h->qr_bound += 1;
  if (h->xpeer_on) h->xframe += 1;
  const bool same = (dtype == PROST_F64) == h->fp64 && dtype != PROST_U8;
  const bool dense = h->P == h->Pp;
  const void* xdev = h->x;
  // 8-bit frames go to the TMEM kernel as they are (1 byte per coordinate in
  // HBM and over PCIe) and are divided by 255 on load; the other kernels read
  // a converted copy (k_pack)
  const bool x8 = dtype == PROST_U8 && (h->tmem || h->tma) && dense;
  if (x8) {
    if (on_device) xdev = frames;
    else CK(cudaMemcpyAsync(h->x, frames, (size_t)h->S * h->C * h->P, cudaMemcpyHostToDevice, st));
  } else if (on_device && same && dense) {
    xdev = frames;  // zero-copy: kernels read the caller's device frames
  } else {
    int rc = upload_dense(h, frames, dtype, on_device, h->x, h->S * h->C, st);
    if (rc) return rc;
  }
  prost_outputs o{};
  if (out) o = *out;
  const int odt = o.dtype == PROST_F64 ? PROST_F64 : PROST_F32;
  const bool osame = (odt == PROST_F64) == h->fp64;
  const size_t fbytes = (size_t)h->S * h->np * h->esz;
  cudaError_t e = cudaSuccess;
  Args a = make_args(h, 0);
  a.x = xdev;
  a.xu8 = x8 ? 1 : 0;
  if (o.fit_residual) {
    if (o.on_device && osame && dense) a.fitres_out = o.fit_residual;
    else {
      if (!h->fresbuf) h->fresbuf = dev_alloc(fbytes, &e);
      if (e != cudaSuccess) return fail(h, PROST_ERR_CUDA, "fit residual buffer: %s", cudaGetErrorString(e));
      a.fitres_out = h->fresbuf;
    }
  }
  if (o.background) {
    if (o.on_device && osame && dense) a.bg_out = o.background;
    else {
      if (!h->bgbuf) h->bgbuf = dev_alloc(fbytes, &e);
      if (e != cudaSuccess) return fail(h, PROST_ERR_CUDA, "bg buffer: %s", cudaGetErrorString(e));
      a.bg_out = h->bgbuf;
    }
  }
  if (o.residual) {
    if (o.on_device && osame && dense) a.res_out = o.residual;
    else {
      if (!h->resbuf) h->resbuf = dev_alloc(fbytes, &e);
      if (e != cudaSuccess) return fail(h, PROST_ERR_CUDA, "residual buffer: %s", cudaGetErrorString(e));
      a.res_out = h->resbuf;
    }
  }
  if (o.mask) {
    if (o.on_device && dense) a.mask_out = o.mask;
    else {
      if (!h->maskbuf) h->maskbuf = (uint8_t*)dev_alloc((size_t)h->S * h->Pp, &e);
      if (e != cudaSuccess) return fail(h, PROST_ERR_CUDA, "mask buffer: %s", cudaGetErrorString(e));
      a.mask_out = h->maskbuf;
    }
  }
  if (o.raw_mask && o.on_device && dense) a.raw_out = o.raw_mask;
  *ap = a;
  *op = o;
  return PROST_OK;
}

// prost_push, second half: outputs the kernels could not write in place, and
// the FitInfo readback (raises NonFiniteError for a rejected frame).
int push_outputs(prost_handle* h, const Args& a, const prost_outputs& o, cudaStream_t st) {
  const int odt = o.dtype == PROST_F64 ? PROST_F64 : PROST_F32;
  CK(cudaGetLastError());
  // outputs the kernels could not write in place
  int rc = PROST_OK;
  if (o.background && a.bg_out == h->bgbuf)
    rc = download_dense(h, h->bgbuf, o.background, odt, o.on_device, h->S * h->C, st);
  if (!rc && o.residual && a.res_out == h->resbuf)
    rc = download_dense(h, h->resbuf, o.residual, odt, o.on_device, h->S * h->C, st);
  if (!rc && o.fit_residual && a.fitres_out == h->fresbuf)
    rc = download_dense(h, h->fresbuf, o.fit_residual, odt, o.on_device, h->S * h->C, st);
  if (!rc && o.mask && a.mask_out == h->maskbuf) rc = copy_labels(h, h->maskbuf, o.mask, o.on_device, st);
  if (!rc && o.raw_mask && a.raw_out == nullptr) rc = copy_labels(h, h->lab, o.raw_mask, o.on_device, st);
  if (!rc && o.raw_mask && a.raw_out != nullptr && a.raw_out != o.raw_mask)
    rc = copy_labels(h, a.raw_out, o.raw_mask, o.on_device, st);  // a pipelined slot's raw labels
  if (rc) return rc;
  if (o.fit && o.fit_async) {
    // stream-ordered copy into the caller's (pinned) array; statuses are the
    // caller's to check once the push is joined
    CK(cudaMemcpyAsync(o.fit, a.info, (size_t)h->S * sizeof(FitInfo), cudaMemcpyDeviceToHost, st));
  }
  if (o.fit && !o.fit_async) {
    CK(cudaMemcpyAsync(h->info_h, h->info, (size_t)h->S * sizeof(FitInfo), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    std::memcpy(o.fit, h->info_h, (size_t)h->S * sizeof(FitInfo));
    int first_bad = PROST_OK;
    bool cold = false, over = true;
    for (int s = 0; s < h->S; ++s) {
      if (h->info_h[s].status != PROST_OK && first_bad == PROST_OK) first_bad = h->info_h[s].status;
      cold |= h->info_h[s].frame_index == 0;  // rejected at its first frame: still cold
      over &= h->info_h[s].frame_index > h->prm.i_init;
    }
    h->maybe_cold = cold;
    h->stats_over = h->stats_over || over;
    h->peek_pending = false;
    if (first_bad != PROST_OK) return fail(h, first_bad, "frame contains non-finite values");
  } else if ((h->maybe_cold || (h->xmode && h->pipeline && !h->stats_over)) && !h->peek_pending) {
    // no readback requested: peek at the frame indices asynchronously and
    // keep launching the cold-start kernel until every stream is past frame 0
    // (a stream whose first frame was rejected stays cold, fit.py:86-87)
    CK(cudaMemcpyAsync(h->info_peek, a.info, (size_t)h->S * sizeof(FitInfo), cudaMemcpyDeviceToHost, st));
    CK(cudaEventRecord(h->ev_peek, st));
    h->peek_pending = true;
  }
  return PROST_OK;
}

// The kernels of one frame for every stream on stream `st`.
int launch_frame(prost_handle* h, Args& a, cudaStream_t st) {
  if (h->resident || h->tmem) {
    // one cooperative launch for the whole frame of every stream, then the median
    const char* stg = getenv("PROST_STAGGER_NS");
    // k_tmem: L2 bulk prefetch of the rest of a CTA's slice at the start of its
    // load (PROST_PREFETCH=0 turns it off; within +-0.3% on C3: the load phase
    // gains what the other teams' reductions lose)
    const char* pfe = getenv("PROST_PREFETCH");
    const char* alt = getenv("PROST_ALT");       // 0: slot groups load independently
    RArgs ra{h->rG, h->rT, h->rqpc, RES_RNV_MAX, h->rbar, h->rpart, h->S,
             h->prof ? h->rprof : nullptr, stg ? atoi(stg) : 0, pfe ? atoi(pfe) : 1,
             alt ? atoi(alt) : 1};
    // team barrier counters, the stream counter and the teams' next streams
    if (!h->tm_cl) CK(cudaMemsetAsync(h->rbar, 0, (size_t)(3 * h->rT * h->rng + 1) * sizeof(unsigned), st));
    // cluster teams filter the labels themselves (one channel, 4-pixel words)
    // (not when the periodic QR may run after the kernel: it relabels)
    const bool med_in =
        h->tm_cl && h->C == 1 && h->prm.width % 4 == 0 && h->P == h->Pp && a.mask_out && !h->qr_due;
    ra.median = med_in ? 1 : 0;
    long long n = 0;
    {
      PhaseTimer pt_(h, st, PROST_PH_FRAME);
      if (h->tmem)
        CK(pick_tmem(h->resident_ops_K, h->prm.p == 0.5, h->rng, false, h->tm_cl).launch(a, ra, h->rsmem, st));
      else
        CK(pick_resident(h->resident_ops_K, h->prm.p == 0.5).launch(a, ra, h->rnt, h->rsmem, st));
      ++n;
    }
    if (h->tmem && h->C == 3) {  // labels: any channel over the threshold
      const dim3 cg(std::max(1, std::min((h->Pp / 4 + NT - 1) / NT, 64)), h->S);
      k_combine3<<<cg, NT, 0, st>>>(a);
      ++n;
    }
    if (h->tmem && h->qr_due) h->ops.qr(h, a, st, h->S);  // per stream: exits unless due
    if (a.mask_out && !med_in) {
      PhaseTimer pt_(h, st, PROST_PH_MEDIAN);
      launch_median(h, a, st, h->S);
      ++n;
    }
    h->launches += n;
  } else {
    const int wave = std::max(1, std::min(h->wave, h->S));
    for (int s0 = 0; s0 < h->S; s0 += wave) {
      a.s0 = s0;
      h->ops.frame(h, a, st, std::min(wave, h->S - s0));
    }
  }
  CK(cudaGetLastError());
  return PROST_OK;
}

// Wait for pipelined host-I/O pushes still in flight (before any direct state access).
int io_drain(prost_handle* h) {
  if (!h->io_pending) return PROST_OK;
  CK(cudaStreamSynchronize(h->s_in));
  CK(cudaStreamSynchronize(h->s_comp));
  CK(cudaStreamSynchronize(h->s_out));
  h->io_pending = false;
  return PROST_OK;
}

// prost_push with host frames and host outputs: H2D of this frame overlaps the
// kernels of the previous one, whose D2H overlaps both.  Ordered after the
// caller's stream `st` at entry; prost_join / prost_synchronize wait for it.
int push_pipelined(prost_handle* h, const void* frames, int32_t dtype, const prost_outputs* out,
                   cudaStream_t st) {
  CK(cudaSetDevice(h->device));
  if (!h->s_in) {
    CK(cudaStreamCreateWithFlags(&h->s_in, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&h->s_comp, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&h->s_out, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&h->ev_user, cudaEventDisableTiming));
    for (int i = 0; i < 2; ++i) {
      CK(cudaEventCreateWithFlags(&h->ev_in[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&h->ev_comp[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&h->ev_out[i], cudaEventDisableTiming));
      cudaError_t e = cudaSuccess;
      const size_t fbytes = (size_t)h->S * h->np * h->esz;
      if (i == 0) {  // lazily allocated single buffers are superseded by the slots
        if (h->bgbuf) cudaFree(h->bgbuf);
        if (h->resbuf) cudaFree(h->resbuf);
        if (h->maskbuf) cudaFree(h->maskbuf);
        h->bgbuf = h->resbuf = nullptr;
        h->maskbuf = nullptr;
      }
      h->io_x[i] = i == 0 ? h->x : dev_alloc(fbytes, &e);
      if (e == cudaSuccess) h->io_bg[i] = dev_alloc(fbytes, &e);
      if (e == cudaSuccess) h->io_res[i] = dev_alloc(fbytes, &e);
      if (e == cudaSuccess) h->io_mask[i] = (uint8_t*)dev_alloc((size_t)h->S * h->Pp, &e);
      if (e == cudaSuccess) h->io_raw[i] = (uint8_t*)dev_alloc((size_t)h->S * h->Pp, &e);
      if (e == cudaSuccess) h->io_info[i] = (FitInfo*)dev_alloc((size_t)h->S * sizeof(FitInfo), &e);
      if (e != cudaSuccess) return fail(h, PROST_ERR_CUDA, "I/O buffers: %s", cudaGetErrorString(e));
    }
  }
  const int sl = h->io_slot;
  // this slot's buffers were last read by the kernels / copies of two frames ago
  h->x = h->io_x[sl];
  h->bgbuf = h->io_bg[sl];
  h->resbuf = h->io_res[sl];
  h->maskbuf = h->io_mask[sl];
  CK(cudaEventRecord(h->ev_user, st));
  CK(cudaStreamWaitEvent(h->s_in, h->ev_user, 0));
  CK(cudaStreamWaitEvent(h->s_in, h->ev_comp[sl], 0));
  Args a;
  prost_outputs o{};
  int rc = push_setup(h, frames, dtype, 0, out, h->s_in, &a, &o);
  if (rc) return rc;
  // raw labels and FitInfo go to this slot's own buffers: the next frame's
  // kernels overwrite the label state and the handle's FitInfo
  if (o.raw_mask) a.raw_out = h->io_raw[sl];
  if (o.fit) a.info = h->io_info[sl];
  CK(cudaEventRecord(h->ev_in[sl], h->s_in));
  CK(cudaStreamWaitEvent(h->s_comp, h->ev_in[sl], 0));
  CK(cudaStreamWaitEvent(h->s_comp, h->ev_out[sl], 0));
  if (h->io_pending) CK(cudaStreamWaitEvent(h->s_comp, h->ev_comp[h->io_last], 0));
  rc = launch_frame(h, a, h->s_comp);
  if (rc) return rc;
  CK(cudaEventRecord(h->ev_comp[sl], h->s_comp));
  CK(cudaStreamWaitEvent(h->s_out, h->ev_comp[sl], 0));
  rc = push_outputs(h, a, o, h->s_out);
  if (rc) return rc;
  CK(cudaEventRecord(h->ev_out[sl], h->s_out));
  h->io_last = sl;
  h->io_slot = sl ^ 1;
  h->io_pending = true;
  return PROST_OK;
}

// ===========================================================================
// C ABI

extern "C" {

int prost_abi_version(void) { return PROST_ABI_VERSION; }

int prost_create(const prost_params* params, int32_t n_streams, uint32_t flags, int32_t device,
                 prost_handle** out) {
  if (!params || !out) return PROST_ERR_CONFIG;
  *out = nullptr;
  prost_handle* h = new prost_handle();
  int rc = validate(h, params, n_streams);
  if (rc) {
    // keep the handle so the caller can read the message, then destroy it
    *out = h;
    return rc;
  }
  h->prm = *params;
  h->S = n_streams;
  h->flags = flags;
  h->device = device;
  h->fp64 = (flags & PROST_FLAG_FP64) != 0;
  h->pipeline = (flags & PROST_FLAG_PIPELINE) != 0;
  h->k = params->k;
  h->C = params->channels;
  h->P = params->width * params->height;
  h->Pp = (h->P + 3) / 4 * 4;
  h->np = (long long)h->C * h->Pp;
  h->esz = h->fp64 ? 8 : 4;
  h->ops = h->fp64 ? pick<double>(h->k) : pick<float>(h->k);
  {
    const char* pe = getenv("PROST_PDL");
    h->pdl = pe ? pe[0] == '1' : true;  // C4: 0.966 -> 0.942 ms per frame
  }
  *out = h;
  if (!h->ops.frame) return fail(h, PROST_ERR_CONFIG, "no kernel instance for k=%d", h->k);
  const int K = h->ops.K;
  h->nvmax = std::max({K + 3, WC + WG * (K + 1), LSW, K * (K + 1) / 2, 3});
  h->n_ls = params->max_backtracks > WC ? (params->max_backtracks - WC + LSW - 1) / LSW : 0;
  CK(cudaSetDevice(device));
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  h->sms = sms;
  const long long groups = (h->Pp / h->ops.VEC + NT - 1) / NT;
  // Streamed phase kernels: CTAs per stream.  Many streams: ~16 CTAs per SM
  // in total (waves keep the HBM queues full); few large streams: one wave of
  // resident CTAs (the phase kernels are limited to 2 per SM by registers)
  // with grid-stride loops, so the last CTA sums few partial slots.
  const long long target = (long long)sms * (h->S >= sms ? 16 : 2);
  h->chunks = (int)std::max<long long>(1, std::min<long long>(groups, (target + h->S - 1) / h->S));
  h->wave = h->S;
  cudaError_t e = cudaSuccess;
  const size_t S = h->S, np = h->np, esz = h->esz;
#define ALLOC(field, bytes)                                                             \
  do {                                                                                  \
    h->field = (decltype(h->field))dev_alloc((bytes), &e);                              \
    if (e != cudaSuccess)                                                               \
      return fail(h, PROST_ERR_CUDA, "cudaMalloc(%s, %zu): %s", #field, (size_t)(bytes), \
                  cudaGetErrorString(e));                                               \
  } while (0)
  ALLOC(U, S * h->k * np * esz);
  ALLOC(r, S * np * esz);
  ALLOC(ud, S * np * esz);
  ALLOC(x, S * np * esz);
  ALLOC(mean, S * np * esz);
  ALLOC(lab, S * h->Pp);
  ALLOC(ctl, S * sizeof(Ctl));
  ALLOC(part, S * h->chunks * h->nvmax * sizeof(double));
  ALLOC(cnt, S * sizeof(unsigned));
  ALLOC(rinv, S * KMAX * KMAX * sizeof(double));
  ALLOC(info, S * sizeof(FitInfo));
  CK(cudaMallocHost(&h->info_h, S * sizeof(FitInfo)));
  CK(cudaMallocHost(&h->info_peek, S * sizeof(FitInfo)));
  CK(cudaEventCreateWithFlags(&h->ev_peek, cudaEventDisableTiming));
  if (!h->fp64 && h->C == 1 && K > 20) setup_tma(h, sms);
  // Resident frame kernel: fp32, one channel, k <= 16, and a team that fits the
  // chip.  The geometry depends on the stream shape only (not on n_streams), so
  // a stream's reduction order — and its result — is the same in any batch.
  // Kernel path: PROST_KERNEL = streamed | resident | tmem (PROST_RESIDENT=1 is
  // an alias of resident; PROST_NO_RESIDENT=1 forces streamed).
  const char* want_res = getenv("PROST_RESIDENT");
  const char* no_res = getenv("PROST_NO_RESIDENT");
  const char* kenv = getenv("PROST_KERNEL");
  std::string kpath = kenv ? kenv : (want_res && want_res[0] == '1' ? "resident" : "tmem");
  if (no_res && no_res[0] == '1') kpath = "streamed";
  const bool eligible = !h->fp64 && K <= 20;
  // slot groups per CTA (prost_tmem.cuh): 1; PROST_TM_GROUPS=2 (two streams
  // per CTA in parallel warp groups) is kept as an experiment switch and
  // falls back to 1 when that instance is not built (measured slower)
  const char* ngenv = getenv("PROST_TM_GROUPS");
  int ng = ngenv ? atoi(ngenv) : 1;
  if (ng != 1 && ng != 2) ng = 1;
  const char* genv = getenv("PROST_TM_G");  // force the team size (experiments)
  const int force_G = genv ? atoi(genv) : 0;
  for (int attempt = 0; attempt < 2 && !h->tmem; ++attempt, ng = 1) {
  const TmOps to = pick_tmem(K, params->p == 0.5, ng);
  if (eligible && kpath == "tmem" && to.launch) {
    if (getenv("PROST_DEBUG")) to.describe();
    // Team size: among the slices that fit TMEM + shared memory, the one with
    // the most stream frames per unit time, teams / round time, with the round
    // time modelled as a fixed part (reduction latency, ~1.5 slot sweeps as
    // measured on C3) plus one part per row-group slot a thread walks (every
    // thread of a group walks the same number of slots, so a slice just over a
    // slot boundary costs a whole extra slot).  Depends on the stream shape
    // and the chip only (not on n_streams): per-stream results do not depend
    // on the batch.
    const int nq = (int)(h->np / 4);  // row groups over all channel planes
    const int tg = TM_NT / ng;         // threads per slot group
    int bestG = 0;
    double best_cost = 0;
    for (int G = 1; G <= sms; ++G) {
      const int qpc = ((nq + G - 1) / G + 3) / 4 * 4;
      if ((nq + qpc - 1) / qpc != G) continue;
      const size_t sm = to.smem(qpc);
      if (sm > (size_t)227 * 1024) continue;
      if (force_G > 0 && G != force_G) continue;
      const int slots = (qpc + tg - 1) / tg;
      // throughput: virtual teams / round time; latency (PROST_FLAG_LATENCY):
      // the round time of one stream, slots per thread plus a small per-CTA
      // barrier cost
      const double cost = (flags & PROST_FLAG_LATENCY) ? slots + 0.05 * G
                                                       : (1.5 + slots) / (double)(sms * TM_CPS / G * ng);
      if (bestG == 0 || cost < best_cost) {
        bestG = G;
        best_cost = cost;
      }
    }
    for (int G = bestG > 0 ? bestG : sms + 1; G <= sms; ++G) {
      const int qpc = ((nq + G - 1) / G + 3) / 4 * 4;
      if ((nq + qpc - 1) / qpc != G) continue;
      const size_t sm = to.smem(qpc);
      if (sm > (size_t)227 * 1024) continue;
      const TmOps tb = pick_tmem(K, params->p == 0.5, ng, true);  // frame-blocking instance
      const bool set = to.prepare(sm) == cudaSuccess && (!tb.prepare || tb.prepare(sm) == cudaSuccess);
      const bool fits = set && (TM_CPS == 1 ? to.occupancy(sm) >= 1
                                            : (size_t)TM_CPS * (sm + 2048) <= (size_t)228 * 1024);
      if (!fits) {
        if (getenv("PROST_DEBUG"))
          fprintf(stderr, "prost: tmem G=%d qpc=%d smem=%zu rejected (%s, occupancy %d)\n", G, qpc, sm,
                  cudaGetErrorString(cudaGetLastError()), to.occupancy(sm));
        cudaGetLastError();
        continue;  // TM_CPS CTAs of this size do not fit an SM: larger team
      }
      {
        h->tmem = true;
        h->rng = ng;
        h->rqpc = qpc;
        h->rnt = TM_NT;
        h->rsmem = sm;
        h->rG = G;
        // enough teams for every stream to have a slot group, at most the chip
        h->rT = std::min((h->S + ng - 1) / ng, sms * TM_CPS / G);
        if (const char* tenv = getenv("PROST_TM_T"))  // cap the teams (experiments)
          if (atoi(tenv) > 0) h->rT = std::min(h->rT, atoi(tenv));
        h->resident_ops_K = K;
        if (h->C == 3) ALLOC(labc, S * np);
        ALLOC(rbar, (size_t)sms * TM_CPS * 2 * sizeof(unsigned));
        ALLOC(rpart, (size_t)2 * sms * TM_CPS * 2 * RES_RNV_MAX * sizeof(double));
        ALLOC(rprof, (size_t)sms * TM_CPS * PROF_N * sizeof(unsigned long long));
        // A team that fits one thread-block cluster (<= 16 CTAs), with every
        // team's cluster resident at once (the one-stream latency layout: C0),
        // sums over DSMEM with the hardware cluster barrier instead of global
        // slots and a counter barrier.  (C3's 13-CTA teams: only 7 such
        // clusters fit the chip, against 11 teams of plain CTAs.)
        const char* clenv = getenv("PROST_CLUSTER");
        if (G <= 16 && !(clenv && clenv[0] == '0')) {
          const TmOps tc = pick_tmem(K, params->p == 0.5, ng, false, true);
          if (tc.launch && tc.prepare(sm) == cudaSuccess && tc.clusters(sm, G) >= h->rT) h->tm_cl = true;
          cudaGetLastError();
        }
        if (getenv("PROST_DEBUG"))
          fprintf(stderr, "prost: tmem NG=%d G=%d T=%d qpc=%d smem=%zu cluster=%d\n", ng, G, h->rT, qpc, sm,
                  (int)h->tm_cl);
      }
      cudaGetLastError();
      break;
    }
  }
  }
  const ResOps ro = pick_resident(K, params->p == 0.5);
  if (eligible && h->C == 1 && ro.launch && kpath == "resident") {
    const int nq = h->Pp / 4;
    int best_used = 0, best_qpc = 0;
    for (int qpc = ro.ntmax / 4 * 4; qpc >= 32; qpc -= 4) {
      const int G = (nq + qpc - 1) / qpc;
      if (G > sms) break;
      const int used = (sms / G) * G;
      const int nt = (qpc + 31) / 32 * 32;
      if (ro.smem(qpc, nt / 32) > 227 * 1024) continue;
      // prefer full-chip use; among near-equal choices, the largest slice (fewest CTAs per team)
      if (used > best_used * 1.03) {
        best_used = used;
        best_qpc = qpc;
      }
    }
    if (best_qpc > 0) {
      const int qpc = best_qpc;
      const int nt = (qpc + 31) / 32 * 32;
      const size_t sm = ro.smem(qpc, nt / 32);
      if (ro.prepare(sm) == cudaSuccess && ro.occupancy(nt, sm) >= 1) {
        h->resident = true;
        h->rqpc = qpc;
        h->rnt = nt;
        h->rsmem = sm;
        h->rG = (nq + qpc - 1) / qpc;
        h->rT = std::min(h->S, sms / h->rG);
        h->resident_ops_K = K;
        ALLOC(rbar, (size_t)sms * sizeof(unsigned));
        ALLOC(rpart, (size_t)2 * sms * RES_RNV_MAX * sizeof(double));
        ALLOC(rprof, (size_t)sms * PROF_N * sizeof(unsigned long long));
      }
      cudaGetLastError();
    }
  }
#undef ALLOC
  // U = first k unit vectors until the caller installs the numpy-drawn basis
  if (h->fp64) {
    std::vector<double> eye;
    std::vector<double> Ud((size_t)h->C * h->P * h->k, 0.0);
    for (int j = 0; j < h->k; ++j) Ud[(size_t)j * h->k + j] = 1.0;
    rows_to_planes<double>(Ud.data(), 0, h->k, h->C, h->P, h->Pp, eye);
    for (size_t s = 0; s < S; ++s)
      CK(cudaMemcpy((char*)h->U + s * h->k * np * esz, eye.data(), eye.size() * esz, cudaMemcpyHostToDevice));
  } else {
    std::vector<float> eye;
    std::vector<double> Ud((size_t)h->C * h->P * h->k, 0.0);
    for (int j = 0; j < h->k; ++j) Ud[(size_t)j * h->k + j] = 1.0;
    rows_to_planes<float>(Ud.data(), 0, h->k, h->C, h->P, h->Pp, eye);
    for (size_t s = 0; s < S; ++s)
      CK(cudaMemcpy((char*)h->U + s * h->k * np * esz, eye.data(), eye.size() * esz, cudaMemcpyHostToDevice));
  }
  CK(cudaDeviceSynchronize());
  return PROST_OK;
}

void prost_destroy(prost_handle* h) {
  if (!h) return;
  void* bufs[] = {h->U, h->r, h->ud, h->x, h->mean, h->lab, h->ctl, h->part, h->cnt,
                  h->rinv, h->info, h->bgbuf, h->resbuf, h->fresbuf, h->maskbuf, h->stage[0], h->stage[1],
                  h->xblk, h->oblk[0], h->oblk[1], h->oblk[2], h->rawblk, h->maskblk, h->infoblk,
                  h->rbar, h->rpart, h->rprof, h->xred, h->xgo, h->labc};
  for (void* b : bufs)
    if (b) cudaFree(b);
  for (void* pr : h->xp_opened) cudaIpcCloseMemHandle(pr);
  if (h->xp_table) cudaFree(h->xp_table);
  if (h->xseq) cudaFree(h->xseq);
  if (h->xp_region) cudaFree(h->xp_region);
  // pipelined-I/O slot buffers (slot 0's frame buffer is h->x's allocation,
  // and h->x / bgbuf / resbuf / maskbuf may point at slot buffers)
  if (h->s_in) {
    cudaDeviceSynchronize();
    void* own[] = {h->io_x[1], h->io_bg[0], h->io_bg[1], h->io_res[0], h->io_res[1], h->io_mask[0],
                   h->io_mask[1], h->io_raw[0], h->io_raw[1], h->io_info[0], h->io_info[1]};
    for (void* b : own)
      if (b && b != h->x && b != h->bgbuf && b != h->resbuf && b != h->maskbuf) cudaFree(b);
    if (h->io_x[0] != h->x) cudaFree(h->io_x[0]);
    cudaStreamDestroy(h->s_in);
    cudaStreamDestroy(h->s_comp);
    cudaStreamDestroy(h->s_out);
    cudaEventDestroy(h->ev_user);
    for (int i = 0; i < 2; ++i) {
      cudaEventDestroy(h->ev_in[i]);
      cudaEventDestroy(h->ev_comp[i]);
      cudaEventDestroy(h->ev_out[i]);
    }
  }
  if (h->info_h) cudaFreeHost(h->info_h);
  if (h->info_peek) cudaFreeHost(h->info_peek);
  if (h->ev_peek) cudaEventDestroy(h->ev_peek);
  for (auto& pe : h->prof_ev) {
    cudaEventDestroy(pe.second.first);
    cudaEventDestroy(pe.second.second);
  }
  for (cudaEvent_t e : h->ev_pool) cudaEventDestroy(e);
  delete h;
}

int prost_set_core_state(prost_handle* h, int32_t stream, const double* U, const double* y,
                         const double* weights, int64_t frame_index, int64_t steps_since_qr) {
  if (h) {
    int drc = io_drain(h);
    if (drc) return drc;
  }
  int rc = check_stream(h, stream);
  if (rc) return rc;
  CK(cudaSetDevice(h->device));
  const int k = h->k, C = h->C, P = h->P, Pp = h->Pp;
  const size_t np = h->np;
  if (U) {
    if (h->fp64) {
      std::vector<double> pl;
      rows_to_planes<double>(U, 0, k, C, P, Pp, pl);
      CK(cudaMemcpy((char*)h->U + (size_t)stream * k * np * h->esz, pl.data(), pl.size() * 8, cudaMemcpyHostToDevice));
    } else {
      std::vector<float> pl;
      rows_to_planes<float>(U, 0, k, C, P, Pp, pl);
      CK(cudaMemcpy((char*)h->U + (size_t)stream * k * np * h->esz, pl.data(), pl.size() * 4, cudaMemcpyHostToDevice));
    }
  }
  if (weights) {
    std::vector<uint8_t> lb(Pp, 0);
    for (int p = 0; p < P; ++p) {
      for (int c = 0; c < C; ++c) {
        const double w = weights[(size_t)c * P + p];
        const uint8_t l = (w == 1.0) ? 0 : 1;
        if (w != 1.0 && w != h->prm.omega)
          return fail(h, PROST_ERR_CONFIG, "weights must be 1 or omega (%g), got %g", h->prm.omega, w);
        if (c == 0) lb[p] = l;
        else if (lb[p] != l)
          return fail(h, PROST_ERR_CONFIG, "channel weights of pixel %d disagree", p);
      }
    }
    CK(cudaMemcpy(h->lab + (size_t)stream * Pp, lb.data(), Pp, cudaMemcpyHostToDevice));
  }
  Ctl c;
  CK(cudaMemcpy(&c, h->ctl + stream, sizeof c, cudaMemcpyDeviceToHost));
  if (y)
    for (int j = 0; j < k; ++j) c.y[j] = y[j];
  c.frame_index = frame_index;
  c.p0_next = 0;
  c.since_qr = steps_since_qr;
  h->qr_bound = std::max<long long>(h->qr_bound, steps_since_qr);
  c.status = ST_OK;
  c.active = 0;
  CK(cudaMemcpy(h->ctl + stream, &c, sizeof c, cudaMemcpyHostToDevice));
  if (frame_index == 0) {
    h->maybe_cold = true;
  }
  h->stats_over = false;
  h->peek_pending = false;  // an older peek predates this state
  return PROST_OK;
}

int prost_get_core_state(prost_handle* h, int32_t stream, double* U, double* y, double* weights,
                         int64_t* frame_index, int64_t* steps_since_qr) {
  if (h) {
    int drc = io_drain(h);
    if (drc) return drc;
  }
  int rc = check_stream(h, stream);
  if (rc) return rc;
  CK(cudaSetDevice(h->device));
  CK(cudaDeviceSynchronize());
  const int k = h->k, C = h->C, P = h->P, Pp = h->Pp;
  const size_t np = h->np;
  if (U) {
    std::vector<char> raw((size_t)k * np * h->esz);
    CK(cudaMemcpy(raw.data(), (char*)h->U + (size_t)stream * k * np * h->esz, raw.size(), cudaMemcpyDeviceToHost));
    for (int c = 0; c < C; ++c)
      for (int p = 0; p < P; ++p)
        for (int j = 0; j < k; ++j) {
          const size_t src = (size_t)j * np + (size_t)c * Pp + p;
          U[((size_t)c * P + p) * k + j] =
              h->fp64 ? ((const double*)raw.data())[src] : (double)((const float*)raw.data())[src];
        }
  }
  if (weights) {
    std::vector<uint8_t> lb(Pp);
    CK(cudaMemcpy(lb.data(), h->lab + (size_t)stream * Pp, Pp, cudaMemcpyDeviceToHost));
    for (int c = 0; c < C; ++c)
      for (int p = 0; p < P; ++p) weights[(size_t)c * P + p] = lb[p] ? h->prm.omega : 1.0;
  }
  Ctl c;
  CK(cudaMemcpy(&c, h->ctl + stream, sizeof c, cudaMemcpyDeviceToHost));
  if (y)
    for (int j = 0; j < k; ++j) y[j] = c.y[j];
  if (frame_index) *frame_index = c.frame_index;
  if (steps_since_qr) *steps_since_qr = c.since_qr;
  return PROST_OK;
}

int prost_set_preproc(prost_handle* h, int32_t stream, const double* mean, const double* sc) {
  if (h) {
    int drc = io_drain(h);
    if (drc) return drc;
  }
  int rc = check_stream(h, stream);
  if (rc) return rc;
  CK(cudaSetDevice(h->device));
  if (mean) {
    rc = upload_dense(h, mean, PROST_F64, 0, (char*)h->mean + (size_t)stream * h->np * h->esz, h->C, 0);
    if (rc) return rc;
    CK(cudaDeviceSynchronize());
  }
  if (sc) {
    Ctl c;
    CK(cudaMemcpy(&c, h->ctl + stream, sizeof c, cudaMemcpyDeviceToHost));
    c.psum = sc[0];
    c.psumsq = sc[1];
    c.pcount = (long long)sc[2];
    c.pseen = (long long)sc[3];
    c.frozen = sc[4] != 0.0;
    c.pstd = sc[5];
    CK(cudaMemcpy(h->ctl + stream, &c, sizeof c, cudaMemcpyHostToDevice));
    h->stats_over = false;
    h->peek_pending = false;
  }
  return PROST_OK;
}

int prost_get_preproc(prost_handle* h, int32_t stream, double* mean, double* sc) {
  if (h) {
    int drc = io_drain(h);
    if (drc) return drc;
  }
  int rc = check_stream(h, stream);
  if (rc) return rc;
  CK(cudaSetDevice(h->device));
  CK(cudaDeviceSynchronize());
  if (mean) {
    rc = download_dense(h, (char*)h->mean + (size_t)stream * h->np * h->esz, mean, PROST_F64, 0, h->C, 0);
    if (rc) return rc;
    CK(cudaDeviceSynchronize());
  }
  if (sc) {
    Ctl c;
    CK(cudaMemcpy(&c, h->ctl + stream, sizeof c, cudaMemcpyDeviceToHost));
    sc[0] = c.psum;
    sc[1] = c.psumsq;
    sc[2] = (double)c.pcount;
    sc[3] = (double)c.pseen;
    sc[4] = c.frozen ? 1.0 : 0.0;
    sc[5] = c.pstd;
  }
  return PROST_OK;
}

// Grow-only device scratch for frame-blocked pushes.
int grow(prost_handle* h, void** p, size_t* have, size_t need) {
  if (*have >= need && *p) return PROST_OK;
  if (*p) cudaFree(*p);
  *p = nullptr;
  cudaError_t e = cudaMalloc(p, need);
  if (e != cudaSuccess) return fail(h, PROST_ERR_CUDA, "block buffer: %s", cudaGetErrorString(e));
  *have = need;
  return PROST_OK;
}

int prost_push(prost_handle* h, const void* frames, int32_t dtype, int32_t on_device,
               const prost_outputs* out, void* cuda_stream);

// F consecutive frames of every stream in one launch (frame blocking, see
// prost_tmem.cuh): frames [F][S][C*P], outputs [F][S][...], fit [F][S].
// Where the TMEM kernel cannot block (fp64, 3 channels, padded planes, the
// periodic QR possibly inside the block) it runs F single-frame pushes.
// prost_push_many on a TMA-fed streamed handle: the frames of the block run
// in order with the device frames [F][S][n] and outputs [F][S][...] in place;
// frame f's geodesic sweep also runs frame f+1's pass 0 (k_geo_tma<K, true>).
int push_many_streamed(prost_handle* h, const void* frames, int nframes, int dtype, int on_device,
                       const prost_outputs& o, cudaStream_t st) {
  const int S = h->S;
  const size_t n = (size_t)h->C * h->P;
  const size_t fsz = dtype_size(dtype);
  CK(cudaSetDevice(h->device));
  {
    int drc = io_drain(h);
    if (drc) return drc;
  }
  retire_peek(h);
  h->qr_due = false;
  h->qr_bound += nframes;
  const char* xdev = static_cast<const char*>(frames);
  if (!on_device) {
    const size_t bytes = (size_t)nframes * S * n * fsz;
    int rc = grow(h, &h->xblk, &h->xblk_bytes, bytes);
    if (rc) return rc;
    CK(cudaMemcpyAsync(h->xblk, frames, bytes, cudaMemcpyHostToDevice, st));
    xdev = static_cast<const char*>(h->xblk);
  }
  const size_t obytes = (size_t)nframes * S * n * 4;
  void* ouser[3] = {o.background, o.residual, o.fit_residual};
  void* odev[3] = {nullptr, nullptr, nullptr};
  for (int i = 0; i < 3; ++i) {
    if (!ouser[i]) continue;
    if (o.on_device) {
      odev[i] = ouser[i];
    } else {
      if (h->oblk_bytes < obytes) {
        for (int j = 0; j < 3; ++j) {
          if (h->oblk[j]) cudaFree(h->oblk[j]);
          h->oblk[j] = nullptr;
        }
        h->oblk_bytes = obytes;
      }
      if (!h->oblk[i]) CK(cudaMalloc(&h->oblk[i], h->oblk_bytes));
      odev[i] = h->oblk[i];
    }
  }
  const size_t lbytes = (size_t)nframes * S * h->Pp;
  if (o.mask || o.raw_mask) {
    if (h->lblk_bytes < lbytes) {
      if (h->rawblk) cudaFree(h->rawblk);
      if (h->maskblk) cudaFree(h->maskblk);
      h->rawblk = h->maskblk = nullptr;
      h->lblk_bytes = lbytes;
    }
    if (!h->rawblk) CK(cudaMalloc(&h->rawblk, h->lblk_bytes));
    if (!h->maskblk) CK(cudaMalloc(&h->maskblk, h->lblk_bytes));
  }
  uint8_t* raw_d = (o.raw_mask && o.on_device) ? o.raw_mask : h->rawblk;
  uint8_t* mask_d = (o.mask && o.on_device) ? o.mask : h->maskblk;
  if (h->infoblk_n < (nframes + 1) * S) {
    if (h->infoblk) cudaFree(h->infoblk);
    h->infoblk = nullptr;
    CK(cudaMalloc(&h->infoblk, (size_t)(nframes + 1) * S * sizeof(FitInfo)));
    h->infoblk_n = (nframes + 1) * S;
  }
  const Args a0 = make_args(h, 0);
  for (int f = 0; f < nframes; ++f) {
    Args a = a0;
    a.x = xdev + (size_t)f * S * n * fsz;
    a.xu8 = dtype == PROST_U8 ? 1 : 0;
    a.xnext = f + 1 < nframes ? xdev + (size_t)(f + 1) * S * n * fsz : nullptr;
    a.info = h->infoblk + (size_t)f * S;
    a.info_next = h->infoblk + (size_t)(f + 1) * S;
    void** oarg[3] = {&a.bg_out, &a.res_out, &a.fitres_out};
    for (int i = 0; i < 3; ++i)
      if (odev[i]) *oarg[i] = static_cast<char*>(odev[i]) + (size_t)f * S * n * 4;
    if (o.mask || o.raw_mask) a.raw_out = raw_d + (size_t)f * S * h->Pp;
    if (o.mask) a.mask_out = mask_d + (size_t)f * S * h->Pp;
    int rc = launch_frame(h, a, st);
    if (rc) return rc;
  }
  if (!o.on_device) {
    for (int i = 0; i < 3; ++i)
      if (ouser[i]) CK(cudaMemcpyAsync(ouser[i], odev[i], obytes, cudaMemcpyDeviceToHost, st));
    if (o.mask) CK(cudaMemcpyAsync(o.mask, h->maskblk, lbytes, cudaMemcpyDeviceToHost, st));
    if (o.raw_mask) CK(cudaMemcpyAsync(o.raw_mask, h->rawblk, lbytes, cudaMemcpyDeviceToHost, st));
  }
  if (o.fit) {
    CK(cudaMemcpyAsync(o.fit, h->infoblk, (size_t)nframes * S * sizeof(FitInfo), cudaMemcpyDeviceToHost, st));
    if (!o.fit_async) {
      CK(cudaStreamSynchronize(st));
      bool cold = false;
      for (int i = 0; i < nframes * S; ++i)
        if (o.fit[i].status != PROST_OK) return fail(h, o.fit[i].status, "frame contains non-finite values");
      for (int i = 0; i < S; ++i) cold |= o.fit[(size_t)(nframes - 1) * S + i].frame_index == 0;
      h->maybe_cold = cold;
    }
  }
  return PROST_OK;
}

int prost_push_many(prost_handle* h, const void* frames, int32_t nframes, int32_t dtype,
                    int32_t on_device, const prost_outputs* out, void* cuda_stream) {
  if (!h) return PROST_ERR_CONFIG;
  if (nframes < 1) return fail(h, PROST_ERR_DIMENSION, "nframes must be >= 1, got %d", nframes);
  if (h->xmode) return fail(h, PROST_ERR_CONFIG, "exchange-mode handle: use prost_xbegin");
  if (dtype != PROST_F32 && dtype != PROST_F64 && dtype != PROST_U8)
    return fail(h, PROST_ERR_CONFIG, "unknown frame dtype %d", dtype);
  cudaStream_t st = (cudaStream_t)cuda_stream;
  prost_outputs o{};
  if (out) o = *out;
  const int S = h->S, P = h->P;
  const size_t n = (size_t)h->C * P;
  const size_t fsz = dtype_size(dtype);
  const int odt = o.dtype == PROST_F64 ? PROST_F64 : PROST_F32;
  const size_t osz = dtype_size(odt);
  const bool dense = h->P == h->Pp;
  const bool blockable = nframes > 1 && h->tmem && h->C == 1 && dense && dtype != PROST_F64 &&
                         odt == PROST_F32 && h->qr_bound + nframes < QR_EVERY - 1;
  // TMA-fed streamed handles (k > 20): the frames run one after another, each
  // geodesic sweep carrying the next frame's pass 0 (one U pass fewer per frame)
  const bool sblockable = nframes > 1 && !h->tmem && h->tma && h->tma_next && h->C == 1 && dense &&
                          dtype != PROST_F64 && odt == PROST_F32 && h->qr_bound + nframes < QR_EVERY - 1;
  if (sblockable) return push_many_streamed(h, frames, nframes, dtype, on_device, o, st);
  if (!blockable) {
    for (int f = 0; f < nframes; ++f) {
      prost_outputs of = o;
      auto at = [&](void* base, size_t per) { return base ? (void*)((char*)base + (size_t)f * S * per) : nullptr; };
      of.background = at(o.background, n * osz);
      of.residual = at(o.residual, n * osz);
      of.fit_residual = at(o.fit_residual, n * osz);
      of.mask = (uint8_t*)at(o.mask, P);
      of.raw_mask = (uint8_t*)at(o.raw_mask, P);
      of.fit = o.fit ? o.fit + (size_t)f * S : nullptr;
      const int rc = prost_push(h, (const char*)frames + (size_t)f * S * n * fsz, dtype, on_device, &of, st);
      if (rc) return rc;
    }
    return PROST_OK;
  }
  CK(cudaSetDevice(h->device));
  {
    int drc = io_drain(h);  // order after pipelined single-frame pushes
    if (drc) return drc;
  }
  retire_peek(h);
  h->qr_due = false;
  h->qr_bound += nframes;
  // frames: used in place on the device, else uploaded as they are (u8 stays u8)
  const void* xdev = frames;
  if (!on_device) {
    const size_t bytes = (size_t)nframes * S * n * fsz;
    int rc = grow(h, &h->xblk, &h->xblk_bytes, bytes);
    if (rc) return rc;
    CK(cudaMemcpyAsync(h->xblk, frames, bytes, cudaMemcpyHostToDevice, st));
    xdev = h->xblk;
  }
  Args a = make_args(h, 0);
  a.x = xdev;
  a.xu8 = dtype == PROST_U8 ? 1 : 0;
  a.nframes = nframes;
  const size_t obytes = (size_t)nframes * S * n * 4;
  void* ouser[3] = {o.background, o.residual, o.fit_residual};
  void** oarg[3] = {&a.bg_out, &a.res_out, &a.fitres_out};
  for (int i = 0; i < 3; ++i) {
    if (!ouser[i]) continue;
    if (o.on_device) {
      *oarg[i] = ouser[i];
    } else {
      if (h->oblk_bytes < obytes) {
        for (int j = 0; j < 3; ++j) {
          if (h->oblk[j]) cudaFree(h->oblk[j]);
          h->oblk[j] = nullptr;
        }
        h->oblk_bytes = obytes;
      }
      if (!h->oblk[i]) CK(cudaMalloc(&h->oblk[i], h->oblk_bytes));
      *oarg[i] = h->oblk[i];
    }
  }
  // raw labels of every frame (the median reads them); the filtered masks
  const size_t lbytes = (size_t)nframes * S * h->Pp;
  if (o.mask || o.raw_mask) {
    if (h->lblk_bytes < lbytes) {
      if (h->rawblk) cudaFree(h->rawblk);
      if (h->maskblk) cudaFree(h->maskblk);
      h->rawblk = h->maskblk = nullptr;
      h->lblk_bytes = lbytes;
    }
    if (!h->rawblk) CK(cudaMalloc(&h->rawblk, h->lblk_bytes));
    if (!h->maskblk) CK(cudaMalloc(&h->maskblk, h->lblk_bytes));
    a.raw_out = (o.raw_mask && o.on_device) ? o.raw_mask : h->rawblk;
  }
  if (h->infoblk_n < nframes * S) {
    if (h->infoblk) cudaFree(h->infoblk);
    h->infoblk = nullptr;
    CK(cudaMalloc(&h->infoblk, (size_t)nframes * S * sizeof(FitInfo)));
    h->infoblk_n = nframes * S;
  }
  a.info = h->infoblk;
  const char* stg = getenv("PROST_STAGGER_NS");
  RArgs ra{h->rG, h->rT, h->rqpc, RES_RNV_MAX, h->rbar, h->rpart, h->S,
           h->prof ? h->rprof : nullptr, stg ? atoi(stg) : 0, 0, 1};
  CK(cudaMemsetAsync(h->rbar, 0, (size_t)(3 * h->rT * h->rng + 1) * sizeof(unsigned), st));
  {
    PhaseTimer pt_(h, st, PROST_PH_FRAME);
    CK(pick_tmem(h->resident_ops_K, h->prm.p == 0.5, h->rng, true).launch(a, ra, h->rsmem, st));
  }
  h->launches += 1;
  if (o.mask) {
    PhaseTimer pt_(h, st, PROST_PH_MEDIAN);
    for (int f = 0; f < nframes; ++f) {
      Args am = a;
      am.lab = a.raw_out + (size_t)f * S * h->Pp;
      am.mask_out = (o.on_device ? o.mask : h->maskblk) + (size_t)f * S * h->Pp;
      launch_median(h, am, st, S);
      h->launches += 1;
    }
  }
  CK(cudaGetLastError());
  // host outputs
  if (!o.on_device) {
    for (int i = 0; i < 3; ++i)
      if (ouser[i]) CK(cudaMemcpyAsync(ouser[i], *oarg[i], obytes, cudaMemcpyDeviceToHost, st));
    if (o.mask) CK(cudaMemcpyAsync(o.mask, h->maskblk, lbytes, cudaMemcpyDeviceToHost, st));
    if (o.raw_mask) CK(cudaMemcpyAsync(o.raw_mask, h->rawblk, lbytes, cudaMemcpyDeviceToHost, st));
  }
  if (o.fit) {
    CK(cudaMemcpyAsync(o.fit, h->infoblk, (size_t)nframes * S * sizeof(FitInfo), cudaMemcpyDeviceToHost, st));
    if (!o.fit_async) {
      CK(cudaStreamSynchronize(st));
      for (int i = 0; i < nframes * S; ++i)
        if (o.fit[i].status != PROST_OK) return fail(h, o.fit[i].status, "frame contains non-finite values");
    }
  }
  h->maybe_cold = false;  // every stream ran its first frame at f = 0 (a rejected one stays at 0)
  if (o.fit && !o.fit_async)
    for (int i = 0; i < S; ++i) h->maybe_cold |= o.fit[(size_t)(nframes - 1) * S + i].frame_index == 0;
  return PROST_OK;
}

int prost_push(prost_handle* h, const void* frames, int32_t dtype, int32_t on_device,
               const prost_outputs* out, void* cuda_stream) {
  if (!h) return PROST_ERR_CONFIG;
  if (h->xmode && !h->xpeer_on)
    return fail(h, PROST_ERR_CONFIG, "exchange-mode handle: use prost_xbegin (or prost_xpeer_open)");
  cudaStream_t st = (cudaStream_t)cuda_stream;
  Args a;
  prost_outputs o{};
  const char* nopipe = getenv("PROST_NO_PIPE");
  // (raw labels and an asynchronous FitInfo go through per-slot buffers; a
  // synchronous FitInfo readback or the fit residual disable pipelining)
  if (!on_device && out && !out->on_device && (!out->fit || out->fit_async) && !out->fit_residual &&
      !h->prof &&
      !(nopipe && nopipe[0] == '1'))
    return push_pipelined(h, frames, dtype, out, st);
  if (h->io_pending) {  // order after the pipelined pushes before this one
    CK(cudaStreamWaitEvent(st, h->ev_comp[h->io_last], 0));
    CK(cudaStreamWaitEvent(st, h->ev_out[h->io_last], 0));
    h->io_pending = false;
  }
  int rc0 = push_setup(h, frames, dtype, on_device, out, st, &a, &o);
  if (rc0) return rc0;
  rc0 = launch_frame(h, a, st);
  if (rc0) return rc0;
  return push_outputs(h, a, o, st);
}

// ---------------------------------------------------------------------------
// Exchange (pixel-sharded) mode: every rank holds a block of
// image rows of the same stream(s); after each phase kernel the caller sums
// the partials in the exchange buffer over ranks (NCCL all-reduce), then the
// phase's scalar logic runs identically on every rank.

int prost_set_exchange(prost_handle* h, int64_t n_real_global) {
  if (!h) return PROST_ERR_CONFIG;
  if (n_real_global < (int64_t)h->C * h->P)
    return fail(h, PROST_ERR_DIMENSION, "global coordinate count %lld is below the local %lld",
                (long long)n_real_global, (long long)h->C * h->P);
  CK(cudaSetDevice(h->device));
  if (!h->xred) {
    cudaError_t e = cudaSuccess;
    h->xred = (double*)dev_alloc((size_t)h->S * h->nvmax * sizeof(double), &e);
    if (e != cudaSuccess) return fail(h, PROST_ERR_CUDA, "exchange buffer: %s", cudaGetErrorString(e));
    h->xgo = (int*)dev_alloc((size_t)h->S * sizeof(int), &e);
    if (e != cudaSuccess) return fail(h, PROST_ERR_CUDA, "exchange flags: %s", cudaGetErrorString(e));
  }
  h->xmode = true;
  h->tmem = false;  // the phase-kernel (streamed) path is the one with exchange points
  h->resident = false;
  h->n_real_glob = n_real_global;
  return PROST_OK;
}

int prost_xbuffer(prost_handle* h, double** xred, int64_t* count) {
  if (!h || !xred || !count) return PROST_ERR_CONFIG;
  if (!h->xmode) return fail(h, PROST_ERR_CONFIG, "not an exchange-mode handle");
  *xred = h->xred;
  *count = (int64_t)h->S * h->nvmax;
  return PROST_OK;
}

int prost_xbegin(prost_handle* h, const void* frames, int32_t dtype, int32_t on_device,
                 const prost_outputs* out, void* cuda_stream) {
  if (!h) return PROST_ERR_CONFIG;
  if (!h->xmode) return fail(h, PROST_ERR_CONFIG, "not an exchange-mode handle");
  cudaStream_t st = (cudaStream_t)cuda_stream;
  int rc = push_setup(h, frames, dtype, on_device, out, st, &h->xa, &h->xo);
  if (rc) return rc;
  std::vector<int>& pg = h->xprog;
  pg.clear();
  // The statistics phase is a no-op once every stream is frozen, but its
  // exchange is not: drop it once a FitInfo peek has shown every stream past
  // the window.  While that is open the peek is retired synchronously, so all
  // ranks (same stream, same frame indices) build the same program.
  if (h->pipeline && !h->stats_over && h->peek_pending) {
    CK(cudaEventSynchronize(h->ev_peek));
    retire_peek(h);
  }
  // once every stream is frozen (or without the pipeline) the statistics
  // kernel only opens the frame: no reduction, no exchange
  pg.push_back(h->pipeline && !h->stats_over ? XS_STATS : XS_START);
  if (h->maybe_cold) pg.push_back(XS_COLD);
  pg.push_back(XS_PASS0);
  for (int it = 0; it < h->prm.cg_max_iters; ++it) {
    pg.push_back(XS_ITER);
    for (int l = 0; l < h->n_ls; ++l) pg.push_back(XS_LSFB);
    pg.push_back(XS_GRADFB);
  }
  pg.push_back(XS_GEO);
  if (h->qr_due) {
    pg.push_back(XS_GRAM);
    pg.push_back(XS_GEOQR);
  }
  h->xpc = 0;
  h->xlast = -1;
  h->xactive = true;
  return PROST_OK;
}

int prost_xnext(prost_handle* h, int32_t* exchange, void* cuda_stream) {
  if (!h || !exchange) return PROST_ERR_CONFIG;
  if (!h->xactive) return fail(h, PROST_ERR_SEQUENCE, "no frame in flight (prost_xbegin)");
  CK(cudaSetDevice(h->device));
  cudaStream_t st = (cudaStream_t)cuda_stream;
  *exchange = 0;
  while (h->xpc < h->xprog.size()) {
    const int xs = h->xprog[h->xpc++];
    h->ops.step(h, h->xa, st, h->S, xs);
    CK(cudaGetLastError());
    if (xs != XS_GEO && xs != XS_GEOQR && xs != XS_START) {
      h->xlast = xs;
      *exchange = 1;
      return PROST_OK;
    }
  }
  return PROST_OK;
}

int prost_xapply(prost_handle* h, void* cuda_stream) {
  if (!h) return PROST_ERR_CONFIG;
  if (!h->xactive || h->xlast < 0) return fail(h, PROST_ERR_SEQUENCE, "no exchange pending");
  CK(cudaSetDevice(h->device));
  h->ops.xlogic(h, h->xa, (cudaStream_t)cuda_stream, h->S, h->xlast);
  h->xlast = -1;
  CK(cudaGetLastError());
  return PROST_OK;
}

int prost_xedges(prost_handle* h, uint8_t* top, uint8_t* bottom, void* cuda_stream) {
  if (!h) return PROST_ERR_CONFIG;
  CK(cudaSetDevice(h->device));
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const int W = h->prm.width, H = h->prm.height;
  if (top) CK(cudaMemcpy2DAsync(top, W, h->lab, h->Pp, W, h->S, cudaMemcpyDeviceToDevice, st));
  if (bottom)
    CK(cudaMemcpy2DAsync(bottom, W, h->lab + (size_t)(H - 1) * W, h->Pp, W, h->S,
                         cudaMemcpyDeviceToDevice, st));
  return PROST_OK;
}

int prost_xfinish(prost_handle* h, const uint8_t* halo_top, const uint8_t* halo_bottom,
                  void* cuda_stream) {
  if (!h) return PROST_ERR_CONFIG;
  if (!h->xactive || h->xpc < h->xprog.size() || h->xlast >= 0)
    return fail(h, PROST_ERR_SEQUENCE, "frame program not finished");
  CK(cudaSetDevice(h->device));
  cudaStream_t st = (cudaStream_t)cuda_stream;
  h->xactive = false;
  Args a = h->xa;
  a.halo_top = halo_top;
  a.halo_bot = halo_bottom;
  if (a.mask_out) {
    if (h->prm.width % 4 != 0 || ((uintptr_t)a.mask_out & 3) || ((uintptr_t)halo_top & 3) ||
        ((uintptr_t)halo_bottom & 3)) {
      const dim3 mg(std::max(1, std::min((h->P + NT - 1) / NT, 64)), h->S);
      k_median<<<mg, NT, 0, st>>>(a);
    } else {
      launch_median(h, a, st, h->S);
    }
    h->launches += 1;
  }
  return push_outputs(h, a, h->xo, st);
}

// In-kernel exchange over peer memory.  Every rank allocates its exchange
// region (prost_xpeer_handle), the caller all-gathers the IPC handles (64 bytes
// each, any transport) and hands them to prost_xpeer_open; from then on
// prost_push runs the whole frame on the device with the phase kernels'
// cross-rank sums done in-kernel (xpeer_exchange) — only the phases that
// actually run exchange, and no host round trip per phase.
int prost_xpeer_handle(prost_handle* h, int32_t world, void* ipc_handle) {
  if (!h || !ipc_handle) return PROST_ERR_CONFIG;
  if (!h->xmode) return fail(h, PROST_ERR_CONFIG, "not an exchange-mode handle (prost_set_exchange)");
  if (world < 1 || world > 64) return fail(h, PROST_ERR_CONFIG, "world size %d outside [1, 64]", world);
  CK(cudaSetDevice(h->device));
  if (h->xp_region && h->xp_world != world)
    return fail(h, PROST_ERR_SEQUENCE, "exchange region already sized for %d ranks", h->xp_world);
  if (!h->xp_region) {
    const size_t bytes = xr_bytes(world, h->S, h->nvmax, h->prm.width);
    CK(cudaMalloc(&h->xp_region, bytes));  // plain cudaMalloc: exportable through IPC
    CK(cudaMemset(h->xp_region, 0, bytes));
    h->xp_world = world;
  }
  cudaIpcMemHandle_t ih;
  CK(cudaIpcGetMemHandle(&ih, h->xp_region));
  static_assert(sizeof(cudaIpcMemHandle_t) == PROST_IPC_HANDLE_BYTES, "IPC handle size");
  std::memcpy(ipc_handle, &ih, sizeof ih);
  return PROST_OK;
}

int prost_xpeer_open(prost_handle* h, int32_t rank, int32_t world, const void* ipc_handles) {
  if (!h || !ipc_handles) return PROST_ERR_CONFIG;
  if (!h->xp_region || h->xp_world != world)
    return fail(h, PROST_ERR_SEQUENCE, "call prost_xpeer_handle with the same world size first");
  if (rank < 0 || rank >= world) return fail(h, PROST_ERR_CONFIG, "rank %d outside world %d", rank, world);
  if (h->xpeer_on) return fail(h, PROST_ERR_SEQUENCE, "peer exchange already open");
  CK(cudaSetDevice(h->device));
  std::vector<void*> bases(world, nullptr);
  for (int q = 0; q < world; ++q) {
    if (q == rank) {
      bases[q] = h->xp_region;
      continue;
    }
    cudaIpcMemHandle_t ih;
    std::memcpy(&ih, static_cast<const uint8_t*>(ipc_handles) + (size_t)q * PROST_IPC_HANDLE_BYTES, sizeof ih);
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, ih, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      for (void* o : h->xp_opened) cudaIpcCloseMemHandle(o);
      h->xp_opened.clear();
      return fail(h, PROST_ERR_CUDA, "cudaIpcOpenMemHandle(rank %d): %s", q, cudaGetErrorString(e));
    }
    h->xp_opened.push_back(p);
    bases[q] = p;
  }
  CK(cudaMalloc(&h->xp_table, (size_t)world * sizeof(void*)));
  CK(cudaMemcpy(h->xp_table, bases.data(), (size_t)world * sizeof(void*), cudaMemcpyHostToDevice));
  CK(cudaMalloc(&h->xseq, (size_t)h->S * sizeof(unsigned long long)));
  CK(cudaMemset(h->xseq, 0, (size_t)h->S * sizeof(unsigned long long)));
  h->xrank = rank;
  h->xworld = world;
  h->xframe = 0;
  h->xpeer_on = true;
  return PROST_OK;
}

int prost_background(prost_handle* h, void* out, int32_t dtype, int32_t on_device, void* cuda_stream) {
  if (!h) return PROST_ERR_CONFIG;
  if (!out) return fail(h, PROST_ERR_DIMENSION, "out is NULL");
  if (!h->pipeline) return fail(h, PROST_ERR_CONFIG, "background_frame needs a pipeline handle");
  {
    int drc = io_drain(h);
    if (drc) return drc;
  }
  CK(cudaSetDevice(h->device));
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const int odt = dtype == PROST_F64 ? PROST_F64 : PROST_F32;
  const bool osame = (odt == PROST_F64) == h->fp64;
  cudaError_t e = cudaSuccess;
  Args a = make_args(h, 0);
  if (on_device && osame && h->P == h->Pp) a.bg_out = out;
  else {
    if (!h->bgbuf) h->bgbuf = dev_alloc((size_t)h->S * h->np * h->esz, &e);
    if (e != cudaSuccess) return fail(h, PROST_ERR_CUDA, "bg buffer: %s", cudaGetErrorString(e));
    a.bg_out = h->bgbuf;
  }
  h->ops.background(h, a, st, h->S);
  CK(cudaGetLastError());
  if (a.bg_out == h->bgbuf) {
    int rc = download_dense(h, h->bgbuf, out, odt, on_device, h->S * h->C, st);
    if (rc) return rc;
  }
  if (!on_device) CK(cudaStreamSynchronize(st));
  return PROST_OK;
}

int prost_join(prost_handle* h, void* cuda_stream) {
  if (!h) return PROST_ERR_CONFIG;
  if (!h->io_pending) return PROST_OK;
  CK(cudaSetDevice(h->device));
  cudaStream_t st = (cudaStream_t)cuda_stream;
  CK(cudaStreamWaitEvent(st, h->ev_comp[h->io_last], 0));
  CK(cudaStreamWaitEvent(st, h->ev_out[h->io_last], 0));
  return PROST_OK;
}

// Resampling shell: device buffers, no handle (pipeline.py:164-193, 245-258).
int prost_resample(const void* src, int32_t dtype_in, int32_t channels, int32_t w_in, int32_t h_in,
                   void* dst, int32_t dtype_out, int32_t w_out, int32_t h_out, void* cuda_stream) {
  if (!src || !dst) return PROST_ERR_DIMENSION;
  if (w_in < 1 || h_in < 1 || w_out < 1 || h_out < 1 || (channels != 1 && channels != 3))
    return PROST_ERR_DIMENSION;
  if (dtype_out == PROST_U8) return PROST_ERR_CONFIG;
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const long long total = (long long)channels * w_out * h_out;
  const int nb = (int)std::min<long long>((total + 255) / 256, 148LL * 16);
  const double sc = dtype_in == PROST_U8 ? 1.0 / 255.0 : 1.0;
#define RS_LAUNCH(TI, TO) \
  k_resample<TI, TO><<<nb, 256, 0, st>>>((const TI*)src, (TO*)dst, channels, w_in, h_in, w_out, h_out, sc)
  if (dtype_in == PROST_F64 && dtype_out == PROST_F64) RS_LAUNCH(double, double);
  else if (dtype_in == PROST_F64) RS_LAUNCH(double, float);
  else if (dtype_in == PROST_F32 && dtype_out == PROST_F64) RS_LAUNCH(float, double);
  else if (dtype_in == PROST_F32) RS_LAUNCH(float, float);
  else if (dtype_out == PROST_F64) RS_LAUNCH(uint8_t, double);
  else RS_LAUNCH(uint8_t, float);
#undef RS_LAUNCH
  return cudaGetLastError() == cudaSuccess ? PROST_OK : PROST_ERR_CUDA;
}

int prost_upsample_mask(const uint8_t* src, int32_t w_in, int32_t h_in, uint8_t* dst, int32_t w_out,
                        int32_t h_out, void* cuda_stream) {
  if (!src || !dst) return PROST_ERR_DIMENSION;
  if (w_in < 1 || h_in < 1 || w_out < 1 || h_out < 1) return PROST_ERR_DIMENSION;
  const long long total = (long long)w_out * h_out;
  const int nb = (int)std::min<long long>((total + 255) / 256, 148LL * 16);
  k_upsample_mask<<<nb, 256, 0, (cudaStream_t)cuda_stream>>>(src, dst, w_in, h_in, w_out, h_out);
  return cudaGetLastError() == cudaSuccess ? PROST_OK : PROST_ERR_CUDA;
}

// Confusion counts (evaluate.py:87-106), accumulated into counts[S][4] =
// {tp, fp, tn, fn} (int64, device).  mask: [S] rows of mask_stride bytes
// (>= pixels; a handle's padded masks or dense ones), truth: dense [S][pixels].
int prost_confusion(const uint8_t* mask, int64_t mask_stride, const uint8_t* truth, int32_t n_streams,
                    int32_t pixels, int64_t* counts, void* cuda_stream) {
  if (!mask || !truth || !counts) return PROST_ERR_DIMENSION;
  if (n_streams < 1 || pixels < 1 || mask_stride < pixels) return PROST_ERR_DIMENSION;
  const dim3 grid(std::max(1, std::min((pixels + NT - 1) / NT, 64)), n_streams);
  k_confusion<<<grid, NT, 0, (cudaStream_t)cuda_stream>>>(mask, truth, pixels, mask_stride,
                                                         (unsigned long long*)counts);
  return cudaGetLastError() == cudaSuccess ? PROST_OK : PROST_ERR_CUDA;
}

// Netpbm payload unpack (frameio.py:120-137): device payload of pixels x
// channels interleaved bytes -> planar f32 / f64 on [0, 1].
int prost_unpack_pnm(const uint8_t* payload, int32_t channels, int32_t pixels, void* dst,
                     int32_t dtype_out, void* cuda_stream) {
  if (!payload || !dst || pixels < 1 || (channels != 1 && channels != 3)) return PROST_ERR_DIMENSION;
  if (dtype_out != PROST_F32 && dtype_out != PROST_F64) return PROST_ERR_CONFIG;
  const long long total = (long long)channels * pixels;
  const int nb = (int)std::min<long long>((total + 255) / 256, 148LL * 16);
  cudaStream_t st = (cudaStream_t)cuda_stream;
  if (dtype_out == PROST_F64) k_unpack_pnm<double><<<nb, 256, 0, st>>>(payload, channels, pixels, (double*)dst);
  else k_unpack_pnm<float><<<nb, 256, 0, st>>>(payload, channels, pixels, (float*)dst);
  return cudaGetLastError() == cudaSuccess ? PROST_OK : PROST_ERR_CUDA;
}

int prost_synchronize(prost_handle* h) {
  if (!h) return PROST_ERR_CONFIG;
  CK(cudaSetDevice(h->device));
  CK(cudaDeviceSynchronize());
  h->io_pending = false;
  CK(cudaMemcpy(h->info_h, h->info, (size_t)h->S * sizeof(FitInfo), cudaMemcpyDeviceToHost));
  for (int s = 0; s < h->S; ++s) {
    if (h->info_h[s].status != PROST_OK) {
      if (h->info_h[s].frame_index == 0) h->maybe_cold = true;
      return fail(h, h->info_h[s].status, "stream %d: frame contains non-finite values", s);
    }
  }
  return PROST_OK;
}

int prost_last_error(prost_handle* h, char* buf, int32_t len) {
  if (!h || !buf || len <= 0) return 0;
  const int n = (int)std::min<size_t>(h->err.size(), (size_t)len - 1);
  std::memcpy(buf, h->err.data(), n);
  buf[n] = 0;
  return n;
}

int prost_query(prost_handle* h, int32_t what, int64_t* value) {
  if (!h || !value) return PROST_ERR_CONFIG;
  switch (what) {
    case PROST_Q_LAUNCHES: *value = h->launches; break;
    case PROST_Q_WAVE: *value = h->wave; break;
    case PROST_Q_BYTES_U: *value = (int64_t)h->k * h->np * (int64_t)h->esz; break;
    case PROST_Q_CHUNKS: *value = h->chunks; break;
    case PROST_Q_INSTANCE_K: *value = h->ops.K; break;
    case PROST_Q_RESIDENT: *value = h->tmem ? 2 : (h->resident ? 1 : 0); break;
    case PROST_Q_CLUSTER: *value = h->tm_cl ? 1 : 0; break;
    case PROST_Q_TMA: *value = h->tma ? h->tma_chunks : 0; break;
    case PROST_Q_TEAM: *value = h->rG; break;
    case PROST_Q_TEAMS: *value = h->rT; break;
    case PROST_Q_GROUPS: *value = h->rng; break;
    case PROST_Q_QPC: *value = h->rqpc; break;
    case PROST_Q_EXCHANGES: {  // in-kernel exchanges of stream 0 so far (synchronous read)
      unsigned long long v = 0;
      if (h->xseq) {
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(&v, h->xseq, sizeof v, cudaMemcpyDeviceToHost));
      }
      *value = (int64_t)v;
      break;
    }
    default: return fail(h, PROST_ERR_CONFIG, "unknown query %d", what);
  }
  return PROST_OK;
}

int prost_profile(prost_handle* h, int32_t enable) {
  if (!h) return PROST_ERR_CONFIG;
  h->prof = enable != 0;
  return PROST_OK;
}

int prost_profile_read(prost_handle* h, double* ms, int64_t* launches, int32_t n_phases) {
  if (!h) return PROST_ERR_CONFIG;
  CK(cudaSetDevice(h->device));
  for (auto& pe : h->prof_ev) {
    CK(cudaEventSynchronize(pe.second.second));
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, pe.second.first, pe.second.second));
    h->prof_ms[pe.first] += t;
    h->prof_n[pe.first] += 1;
    h->ev_pool.push_back(pe.second.first);
    h->ev_pool.push_back(pe.second.second);
  }
  h->prof_ev.clear();
  for (int i = 0; i < n_phases && i < PROST_N_PHASES; ++i) {
    if (ms) ms[i] = h->prof_ms[i];
    if (launches) launches[i] = h->prof_n[i];
    h->prof_ms[i] = 0.0;
    h->prof_n[i] = 0;
  }
  return PROST_OK;
}

int prost_resident_counters(prost_handle* h, int64_t* out, int32_t n) {
  if (!h || !out) return PROST_ERR_CONFIG;
  for (int i = 0; i < n; ++i) out[i] = 0;
  if (!h->resident && !h->tmem) return PROST_OK;
  CK(cudaSetDevice(h->device));
  CK(cudaDeviceSynchronize());
  const int ctas = h->rT * h->rG;
  std::vector<unsigned long long> v((size_t)ctas * PROF_N);
  CK(cudaMemcpy(v.data(), h->rprof, v.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  // per-CTA means of the counters of the last profiled launch (time counters
  // converted from SM clocks to ns with the CTA's own clock rate), then the
  // max kernel time
  const bool is_time[PROF_N] = {true, true, true, true, true, false, false,
                                true, true, true, true, false, true, true, true};
  std::vector<double> acc(PROF_N, 0.0);
  unsigned long long mx = 0;
  for (int c = 0; c < ctas; ++c) {
    const unsigned long long* cv = v.data() + (size_t)c * PROF_N;
    const double ns_per_clk = cv[PROF_TOTAL] ? (double)cv[PROF_GT_TOTAL] / (double)cv[PROF_TOTAL] : 0.0;
    for (int i = 0; i < PROF_N; ++i) acc[i] += is_time[i] ? cv[i] * ns_per_clk : (double)cv[i];
    mx = std::max(mx, cv[PROF_GT_TOTAL]);
  }
  for (int i = 0; i < PROF_N && i < n; ++i) out[i] = (int64_t)(acc[i] / ctas);
  if (n >= PROF_N) out[PROF_N - 1] = (int64_t)mx;
  return PROST_OK;
}

int prost_set_wave(prost_handle* h, int32_t streams_per_wave) {
  if (!h) return PROST_ERR_CONFIG;
  if (streams_per_wave < 0) return fail(h, PROST_ERR_CONFIG, "negative wave size");
  h->wave = streams_per_wave == 0 ? h->S : streams_per_wave;
  return PROST_OK;
}

}  // extern "C"
