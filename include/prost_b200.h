/*
 * prost_b200.h — C-ABI of the B200-native pROST per-frame step.
 *
 * One shared library (paper_1302_2073_b200/_lib/libprost_b200.so) exports
 * exactly these symbols.  No C++ or torch types cross the boundary: plain
 * pointers, sizes and POD structs.  The reference is pure Python (no FFI of
 * its own); each entry point below names the reference interface it
 * replaces, paths relative to /root/reference/pkg/src/prost/.
 *
 *   prost_create / prost_destroy
 *       StreamTracker(RunConfig) construction, jobs.py:161-171, and
 *       bootstrap(), tracker.py:106-118 (the basis itself is drawn on the
 *       host with numpy exactly as manifold.py:100-113 and handed over with
 *       prost_set_core_state, so U0 is bit-identical to the reference's).
 *   prost_push
 *       StreamTracker.push(FrameBuffer) -> FrameRecord, jobs.py:186-229
 *       (PROST_FLAG_PIPELINE), or process_frame(state, x, params),
 *       tracker.py:121-156 (no PIPELINE flag: x is already normalized, the
 *       residual against U' is returned and weights stay per coordinate).
 *   prost_background
 *       StreamTracker.background_frame(), jobs.py:231-239.
 *   prost_set_core_state / prost_get_core_state
 *       TrackerState(basis, y, weights, frame_index) of tracker.py:79-87
 *       and SubspaceBasis.steps_since_qr, manifold.py:49-78.
 *   prost_set_preproc / prost_get_preproc
 *       PreprocStats, pipeline.py:99-161 (and the snapshot fields of
 *       tracker.py:184-209).
 *
 * Status codes map one-to-one onto the reference's error classes
 * (errors.py:14-39); the Python host raises the matching class.
 *
 * Threading: a handle is single-owner (tracker.py:10-11, jobs.py:157-158);
 * calls are enqueued on the caller's CUDA stream (NULL = legacy default).
 */
#ifndef PROST_B200_H
#define PROST_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PROST_ABI_VERSION 2

/* status codes (errors.py:14-39) */
#define PROST_OK 0
#define PROST_ERR_CONFIG 1      /* ConfigError    */
#define PROST_ERR_DIMENSION 2   /* DimensionError */
#define PROST_ERR_NONFINITE 3   /* NonFiniteError */
#define PROST_ERR_SEQUENCE 4    /* SequenceError  */
#define PROST_ERR_CUDA 5        /* device / driver failure (no reference analogue) */

/* element types of frame / output buffers */
#define PROST_F32 0
#define PROST_F64 1
#define PROST_U8 2   /* 8-bit intensities, divided by 255 on load (frameio.py:136) */

/* handle flags */
#define PROST_FLAG_PIPELINE 1u  /* StreamTracker semantics: running-stats normalization,
                                   threshold (segment), 3x3 median, per-pixel weights */
#define PROST_FLAG_LATENCY 4u   /* lay the resident kernel out for the latency of one frame of a
                                   few streams (more CTAs per stream) instead of the throughput
                                   of many; per-stream results do not depend on the batch within
                                   either layout */
#define PROST_FLAG_FP64 2u      /* double-precision state and per-element arithmetic
                                   (parity instantiation); default is fp32 */

/* Tracker tunables: ProstParams (tracker.py:45-76) + LpConfig (cost.py:29-45)
 * + CgOptions (fit.py:24-47) + the RunConfig fields the pipeline needs
 * (jobs.py:74-120).  mu and tau must already be resolved. */
typedef struct prost_params {
  int32_t k;              /* subspace dimension, 1 <= k <= 32, k < n */
  int32_t width;          /* pixels per row */
  int32_t height;         /* rows */
  int32_t channels;       /* 1 or 3, channel-planar (pipeline.py:1-6) */
  int32_t cg_max_iters;   /* CgOptions.max_iters (>= 1) */
  int32_t max_backtracks; /* CgOptions.max_backtracks (1..64) */
  int32_t i_init;         /* statistics window (jobs.py:71) */
  int32_t reserved;
  double p, mu, delta, omega, t_init, t_min, tau;
  double grad_tol, initial_step, shrink, sufficient_decrease;
} prost_params;

/* FitResult (fit.py:50-63) + FrameRecord scalars (jobs.py:142-151). */
typedef struct prost_fit_info {
  double fit_cost;        /* FitResult.cost / FrameRecord.fit_cost */
  double step;            /* step_size(frame_index) used by this frame */
  int64_t frame_index;    /* after the step (FrameRecord.frame_index) */
  int32_t iterations, cost_evals, grad_evals;
  int32_t status;         /* PROST_OK or PROST_ERR_NONFINITE for this stream */
} prost_fit_info;

/* Per-push outputs; every pointer may be NULL.  Arrays are stream-major:
 * background/residual [n_streams][n], masks [n_streams][width*height]. */
typedef struct prost_outputs {
  void* background;       /* clip(U'y*std + mean, 0, 1): background_frame() after the push */
  void* residual;         /* x - U'y in the normalized domain (FrameRecord.residual) */
  uint8_t* mask;          /* median3x3(raw_mask) (FrameRecord.mask) */
  uint8_t* raw_mask;      /* segment(residual) (FrameRecord.raw_mask) */
  prost_fit_info* fit;    /* HOST array [n_streams]; non-NULL makes the call synchronous */
  int32_t dtype;          /* PROST_F32 or PROST_F64 for background/residual */
  int32_t on_device;      /* 1: the array pointers above are device pointers */
  void* fit_residual;     /* x - U y after the fit, before the geodesic (FitResult.residual,
                             fit.py:50-63); same dtype / placement as background */
  int32_t fit_async;      /* 1: `fit` is filled asynchronously (stream-ordered, pinned host
                             memory; valid after prost_join / prost_synchronize) instead of
                             making the call synchronous; a rejected (non-finite) frame then
                             shows as its stream's status instead of the return code */
} prost_outputs;

typedef struct prost_handle prost_handle;

int prost_abi_version(void);

/* n_streams independent trackers sharing one parameter set, batched in every
 * launch.  device: CUDA ordinal.  Bases start as the first k unit vectors;
 * call prost_set_core_state per stream with the numpy-drawn basis. */
int prost_create(const prost_params* params, int32_t n_streams, uint32_t flags,
                 int32_t device, prost_handle** out);
void prost_destroy(prost_handle* h);

/* U: host [n][k] row-major f64 (SubspaceBasis.data), y: [k], weights: [n]
 * with values in {1, omega} (per coordinate; in pipeline mode all channels of
 * a pixel must agree).  Any pointer may be NULL to leave that field. */
int prost_set_core_state(prost_handle* h, int32_t stream, const double* U, const double* y,
                         const double* weights, int64_t frame_index, int64_t steps_since_qr);
int prost_get_core_state(prost_handle* h, int32_t stream, double* U, double* y,
                         double* weights, int64_t* frame_index, int64_t* steps_since_qr);

/* mean: [n]; scalars: [value_sum, value_sumsq, value_count, frames_seen, frozen, std]
 * (pipeline.py:99-118). */
int prost_set_preproc(prost_handle* h, int32_t stream, const double* mean, const double* scalars);
int prost_get_preproc(prost_handle* h, int32_t stream, double* mean, double* scalars);

/* One frame for every stream: frames [n_streams][n] of `dtype`, host or
 * device memory.  Pipeline mode: raw intensities in [0,1] (or u8).  Core mode:
 * the already-normalized vector x of process_frame. */
int prost_push(prost_handle* h, const void* frames, int32_t dtype, int32_t on_device,
               const prost_outputs* out, void* cuda_stream);

/* F consecutive frames of every stream in one call (frame blocking: each
 * stream's slice stays on chip across its F frames, U crosses HBM once per
 * block).  frames [F][n_streams][n]; outputs [F][n_streams][...] (masks
 * unpadded, [F][n_streams][width*height]); out->fit [F][n_streams].  Results
 * equal F calls of prost_push.  Blocks on the TMEM kernel for fp32,
 * one-channel, width*height % 4 == 0, fp32 outputs; otherwise it runs F
 * single-frame pushes.  (No reference counterpart: StreamTracker.push
 * called F times, jobs.py:186-229.) */
int prost_push_many(prost_handle* h, const void* frames, int32_t nframes, int32_t dtype,
                    int32_t on_device, const prost_outputs* out, void* cuda_stream);

/* background_frame() for every stream into out [n_streams][n] (pipeline mode). */
int prost_background(prost_handle* h, void* out, int32_t dtype, int32_t on_device,
                     void* cuda_stream);

/* Wait for all work enqueued by this handle; returns the first per-stream
 * status of the last push (PROST_ERR_NONFINITE if a frame was rejected). */
int prost_synchronize(prost_handle* h);
/* Make `cuda_stream` wait for pushes still in flight on the handle's own
 * streams (a push with host frames and host outputs and no fit info runs
 * pipelined: upload, kernels and download of consecutive frames overlap). */
int prost_join(prost_handle* h, void* cuda_stream);

/* Copy the last error message into buf (NUL-terminated); returns its length. */
int prost_last_error(prost_handle* h, char* buf, int32_t len);

/* Introspection: PROST_Q_LAUNCHES (kernel launches so far), PROST_Q_WAVE
 * (streams per launch wave), PROST_Q_BYTES_U (bytes of U per stream),
 * PROST_Q_CHUNKS (CTAs per stream per launch). */
#define PROST_Q_LAUNCHES 0
#define PROST_Q_WAVE 1
#define PROST_Q_BYTES_U 2
#define PROST_Q_CHUNKS 3
#define PROST_Q_INSTANCE_K 4
#define PROST_Q_RESIDENT 5   /* 0 streamed, 1 register-resident, 2 TMEM-resident kernel */
#define PROST_Q_TEAM 6       /* CTAs per team (resident mode) */
#define PROST_Q_TEAMS 7      /* teams (resident mode) */
#define PROST_Q_GROUPS 8     /* slot groups per CTA of the TMEM kernel: streams per team in flight */
#define PROST_Q_QPC 9        /* row groups (4 coordinates) per CTA slice (resident modes) */
#define PROST_Q_EXCHANGES 10 /* in-kernel cross-rank exchanges of stream 0 so far (peer mode) */
#define PROST_Q_CLUSTER 11   /* 1: TMEM kernel teams run as thread-block clusters (DSMEM team sums) */
#define PROST_Q_TMA 12       /* CTAs per stream of the TMA-fed streamed kernels (k > 20), 0: not used */
int prost_query(prost_handle* h, int32_t what, int64_t* value);

/* Per-phase device timing (CUDA events around every launch, on the launch
 * stream).  prost_profile_read returns and resets the accumulated milliseconds
 * and launch counts per phase, indexed by PROST_PH_*. */
#define PROST_PH_STATS 0
#define PROST_PH_COLD 1
#define PROST_PH_PASS0 2
#define PROST_PH_ITER 3
#define PROST_PH_LSFB 4
#define PROST_PH_GRADFB 5
#define PROST_PH_GEO 6
#define PROST_PH_QR 7
#define PROST_PH_MEDIAN 8
#define PROST_PH_FRAME 9   /* the register-resident whole-frame kernel */
#define PROST_N_PHASES 10
int prost_profile(prost_handle* h, int32_t enable);
/* With profiling on, the TMEM-resident frame kernel runs its counter instance
 * (same results bit for bit; the counter-free instance that runs otherwise is
 * ~3% faster).  Resident-kernel timing of the last launch made with profiling on, as
 * per-CTA means (%globaltimer ns): [0] kernel, [1] team-barrier waits,
 * [2] slot reads, [3] scalar logic, [4] prefetch waits, [5] team reductions,
 * [6] rounds, [7] unused, [8] (if n > 8) the slowest CTA's kernel time. */
int prost_resident_counters(prost_handle* h, int64_t* out, int32_t n);
int prost_profile_read(prost_handle* h, double* ms, int64_t* launches, int32_t n_phases);

/* Tuning knob: streams per launch wave (0 = automatic, sized to L2). */
int prost_set_wave(prost_handle* h, int32_t streams_per_wave);

/* ---- Resampling shell -------------------------------
 * Device buffers, enqueued on cuda_stream; no handle.
 *   prost_resample: bilinear, half-pixel centres, per channel plane
 *     (resample, pipeline.py:164-193); u8 input is divided by 255 first.
 *   prost_upsample_mask: nearest neighbour on categorical labels
 *     (upsample_mask, pipeline.py:245-258). */
int prost_resample(const void* src, int32_t dtype_in, int32_t channels, int32_t w_in, int32_t h_in,
                   void* dst, int32_t dtype_out, int32_t w_out, int32_t h_out, void* cuda_stream);
int prost_upsample_mask(const uint8_t* src, int32_t w_in, int32_t h_in, uint8_t* dst, int32_t w_out,
                        int32_t h_out, void* cuda_stream);

/* Binary PGM / PPM payload (after the header, parsed on the host) to a
 * channel-planar frame on [0, 1] (decode_pnm, frameio.py:120-137). */
int prost_unpack_pnm(const uint8_t* payload, int32_t channels, int32_t pixels, void* dst,
                     int32_t dtype_out, void* cuda_stream);

/* Confusion counts of predicted masks against ground-truth frames
 * (accumulate, evaluate.py:87-106): counts[S][4] =
 * {tp, fp, tn, fn} (int64, device) are incremented; ground-truth gray levels
 * 85 (outside ROI) and 170 (unknown) are not scored, 255 is foreground. */
int prost_confusion(const uint8_t* mask, int64_t mask_stride, const uint8_t* truth, int32_t n_streams,
                    int32_t pixels, int64_t* counts, void* cuda_stream);

/* ---- Exchange (pixel-sharded) mode, SURVEY.md §8(e) ------------------------
 * One stream too large for one GPU (BASELINE config C4) is split by image
 * rows: rank g's handle is created for its block of rows (params.height =
 * local rows) and switched to exchange mode with the stream's global
 * coordinate count.  A frame then runs as a phase program; after each phase
 * with a reduction the caller sums the exchange buffer over ranks (NCCL
 * all-reduce, in place, on the same CUDA stream) and lets the phase's scalar
 * logic run — identically on every rank, so the basis row blocks stay one
 * basis.  The 3x3 median needs the label row above and below the block from
 * the neighbouring ranks (prost_xedges / prost_xfinish).  Replaces, for one
 * sharded stream, the same reference seam as prost_push
 * (StreamTracker.push, jobs.py:186-229, over process_frame, tracker.py:121-156):
 *
 *   prost_xbegin(frame)
 *   while (prost_xnext(&x), x) { allreduce_sum(xred, count); prost_xapply(); }
 *   prost_xedges(top, bottom); exchange rows with the neighbours
 *   prost_xfinish(row above or NULL at the image top, row below or NULL)
 */
int prost_set_exchange(prost_handle* h, int64_t n_real_global);
int prost_xbuffer(prost_handle* h, double** xred, int64_t* count);  /* device, [S][nvmax] f64 */
int prost_xbegin(prost_handle* h, const void* frames, int32_t dtype, int32_t on_device,
                 const prost_outputs* out, void* cuda_stream);
int prost_xnext(prost_handle* h, int32_t* exchange, void* cuda_stream);
int prost_xapply(prost_handle* h, void* cuda_stream);
int prost_xedges(prost_handle* h, uint8_t* top, uint8_t* bottom, void* cuda_stream);  /* [S][width] */
int prost_xfinish(prost_handle* h, const uint8_t* halo_top, const uint8_t* halo_bottom,
                  void* cuda_stream);

/* Pixel sharding with the exchange inside the kernels (the
 * compute step and its collective fused over NVLink peer memory).  Instead of
 * the host-driven program above, every rank of an exchange-mode handle
 *
 *   prost_xpeer_handle(h, world, handle)          64-byte IPC handle of its exchange region
 *   (all-gather the handles over the ranks, e.g. torch.distributed)
 *   prost_xpeer_open(h, rank, world, handles)     map every rank's region
 *
 * after which prost_push(h, this rank's row block, ...) runs the whole frame:
 * the last CTA of each phase kernel stores the stream's sums into every rank's
 * region, waits for every rank's flag and sums them in rank order; phases that
 * do not run for the stream (fallbacks, statistics after the window) exchange
 * nothing.  The median takes its halo rows from the neighbours' stores.  Every
 * rank must push every frame (the kernels wait for each other). */
#define PROST_IPC_HANDLE_BYTES 64
int prost_xpeer_handle(prost_handle* h, int32_t world, void* ipc_handle);
int prost_xpeer_open(prost_handle* h, int32_t rank, int32_t world, const void* ipc_handles);

#ifdef __cplusplus
}
#endif

#endif /* PROST_B200_H */
