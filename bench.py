"""Benchmark: batched pROST per-frame update on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl ours|reference]

One step = one frame for every stream of the workload (the BASELINE config
named by --config; default C3: 256 independent 320x240 grayscale streams,
k=15, p=0.5, mu=1e-4, 2 CG iterations).  Streams shard across ranks with no
collective (weak scaling: every rank runs its own `--streams` streams).  Rank 0
prints one JSON line.

`value`: stream-frames/s over all ranks, frames already resident in HBM,
device-timed with CUDA events (max over ranks).  `e2e`: the same through the
public API with pinned HOST frames in and host mask + background out, copies
inside the timed region.  `roofline`: algorithmic bytes of the frame update
(B_alg = 8nk + 12n + 3P per stream-frame) over the measured
step time against MEASURED_PEAKS.json's HBM copy bandwidth.  `cpu_baseline`:
the numpy oracle port of the reference path on this host's cores.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

PHASE_BYTES_NOTE = "per-phase algorithmic bytes per stream-frame launch"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="C3")
    ap.add_argument("--streams", type=int, default=None, help="streams per rank")
    ap.add_argument("--frames", type=int, default=0,
                    help="distinct frames staged per stream and cycled (0: every step gets the "
                         "stream's next consecutive frame, generated on the device)")
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"])
    ap.add_argument("--cpu-frames", type=int, default=12, help="oracle frames per CPU worker")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-port", action="store_true",
                    help="also time the numpy port beside the reference package (their ratio)")
    ap.add_argument("--e2e-background", action="store_true",
                    help="the end-to-end leg also downloads every stream's background frame")
    ap.add_argument("--e2e-f32", action="store_true",
                    help="end-to-end leg with fp32 frames instead of 8-bit camera frames")
    ap.add_argument("--wave", type=int, default=0)
    ap.add_argument("--block", type=int, default=8,
                    help="also time frame-blocked pushes (push_many) of this many frames per "
                         "stream per call; 0 or 1: skip")
    ap.add_argument("--exchange", choices=["peer", "program"], default="peer",
                    help="pixel sharding: in-kernel exchange over peer memory (peer) or the "
                         "host-driven all-reduce program (program)")
    ap.add_argument("--pixel-shard", action="store_true",
                    help="shard one stream's pixel rows over the ranks (default for C4 with N > 1)")
    ap.add_argument("--preroll", type=int, default=None,
                    help="untimed frames before warm-up (default: i_init, i.e. past the statistics window)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# workload


def workload(name, streams):
    from paper_1302_2073_b200.synth import CONFIGS

    c = CONFIGS[name]
    S = streams if streams is not None else c["streams"]
    t = dict(c["tracker"])
    return c, S, t


def gen_frames(name, stream_ids, n_frames, dtype=np.float32):
    from paper_1302_2073_b200.synth import SceneStream, config_spec

    out = None
    for i, sid in enumerate(stream_ids):
        f = SceneStream(config_spec(name, sid), dtype=dtype).next_frames(n_frames)
        if out is None:
            out = np.empty((n_frames, len(stream_ids), f.shape[1]), dtype=dtype)
        out[:, i] = f
    return out


def b_alg(n, k, P):
    """U read+write + x + mean + background + 3 label bytes."""
    return 8 * n * k + 12 * n + 3 * P


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)


class Clocks:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.gpu)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # the sampler's first line can take a while on a fresh box: start
            # the timed region only once it is producing samples
            t0 = time.time()
            while not self.lines and time.time() - t0 < 10.0 and self.proc.poll() is None:
                time.sleep(0.02)
        except Exception:
            self.proc = None

    def mark(self):
        """Samples so far (call at the start of the timed region)."""
        return len(self.lines)

    def wait_one_more(self, n0, limit=1.0):
        """Wait (bounded) for a sample taken after the timed region started, so
        a short region still has one sample at or after its end."""
        t0 = time.time()
        while len(self.lines) <= n0 and time.time() - t0 < limit and self.proc is not None:
            time.sleep(0.01)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.t:
            self.t.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU baseline: the reference's own StreamTracker (baseline/_ref, the unmodified
# package installed offline) — or, when that install is absent, the numpy port
# of its path (oracle/, pinned bit-exact to it) — one stream per worker process,
# timed on the same steady-state frame window as the GPU arm (after the i_init
# statistics window, which is pushed untimed first).

REF_DIR = ROOT / "baseline" / "_ref"


def _reference_tracker(tracker, i_init, kind):
    """A StreamTracker-like object with push(vec) for the CPU arm."""
    W, H = tracker["target_width"], tracker["target_height"]
    ch = 1 if tracker["grayscale"] else 3
    if kind == "reference":
        if str(REF_DIR) not in sys.path:
            sys.path.insert(0, str(REF_DIR))
        from prost import jobs, pipeline  # the reference package itself

        tr = jobs.StreamTracker(jobs.RunConfig(**tracker), i_init=i_init)
        return lambda v: tr.push(pipeline.FrameBuffer(W, H, ch, v))
    from oracle import prost_oracle as orc
    from paper_1302_2073_b200.params import RunConfig

    prm = RunConfig(**tracker).params(i_init)
    ref = orc.PipelineOracle(W, H, ch, orc.OracleParams(
        k=prm.k, p=prm.cfg.p, mu=prm.cfg.mu, delta=prm.delta, omega=prm.omega,
        t_init=prm.t_init, t_min=prm.t_min, tau=prm.tau, max_iters=prm.cg.max_iters),
        i_init=i_init, seed=RunConfig(**tracker).seed)

    def push(v):
        ref.push(v)
        ref.background()
    return push


def _cpu_worker(job):
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    name, sid, n_frames, tracker, kind, preroll = job
    sys.path.insert(0, str(ROOT))
    frames = gen_frames(name, [sid], preroll + n_frames, dtype=np.float64)[:, 0]
    push = _reference_tracker(tracker, 100, kind)
    for f in frames[:preroll]:  # the statistics window, untimed (the GPU arm's pre-roll)
        push(f)
    t0 = time.perf_counter()
    for f in frames[preroll:]:
        push(f)
    return n_frames, time.perf_counter() - t0


def reference_kind():
    return "reference" if (REF_DIR / "prost" / "jobs.py").exists() else "port"


def cpu_plan(tracker, n_frames, cores, preroll=100):
    """Bound the CPU sample: the reference costs ~4.5e-8 s per coordinate x k
    per frame on one core (11 s per C4 frame) and holds
    a few fp64 copies of the n x k basis, so very large streams (C4) run on
    fewer workers, pre-roll 1 frame instead of the statistics window and time
    2 frames; the sample text says so."""
    n = tracker["target_width"] * tracker["target_height"] * (1 if tracker["grayscale"] else 3)
    k = tracker["subspace_dim"]
    t_frame = 4.5e-8 * n * k
    cores = max(1, min(cores, int(24e9 // (n * k * 32))))
    if (preroll + n_frames) * t_frame > 60.0:
        preroll = 1
        n_frames = max(2, min(n_frames, int(30.0 / t_frame)))
    return n_frames, cores, preroll


def cpu_rate(name, tracker, n_frames, cores=None, kind=None, preroll=100):
    import multiprocessing as mp

    cores = cores or len(os.sched_getaffinity(0))
    n_frames, cores, preroll = cpu_plan(tracker, n_frames, cores, preroll)
    kind = kind or reference_kind()
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    ctx = mp.get_context("spawn")
    jobs = [(name, sid, n_frames, tracker, kind, preroll) for sid in range(cores)]
    t0 = time.perf_counter()
    with ctx.Pool(cores) as pool:
        res = pool.map(_cpu_worker, jobs)
    wall = time.perf_counter() - t0
    frames = sum(r[0] for r in res)
    slowest = max(r[1] for r in res)
    cpu_rate.last_preroll = preroll
    return frames / slowest, cores, frames, wall, kind


def _window_note(name):
    pre = getattr(cpu_rate, "last_preroll", 100)
    return (f"{name} stream after the 100-frame statistics window" if pre >= 100 else
            f"{name} stream after a {pre}-frame pre-roll (bounded sample: the full statistics "
            "window would take minutes per worker at this size)")


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---------------------------------------------------------------------------


def shard_streams(rank, per_rank):
    """Weak scaling by stream: rank r owns global streams
    [r*per_rank, (r+1)*per_rank), each seeded by its global index; no data-path
    collective."""
    return list(range(rank * per_rank, (rank + 1) * per_rank))


def reduce_max(value, world, device=None):
    """Max over ranks of a per-rank device time (outside the timed region)."""
    if world == 1:
        return value
    import torch
    import torch.distributed as dist

    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def run_reference(args):
    ws, rank, _ = dist_env()
    c, S, tracker = workload(args.config, args.streams)
    if rank != 0:
        return 0
    cores = len(os.sched_getaffinity(0))
    # each step: one frame for `cores` streams (one worker process each), on
    # the GPU arm's steady-state window (the statistics window is pre-rolled)
    n_frames = args.warmup + args.steps
    rate, cores, frames, wall, kind = cpu_rate(args.config, tracker, n_frames, cores)
    n_frames = frames // cores
    W, H = tracker["target_width"], tracker["target_height"]
    P = W * H
    line = {
        "impl": "reference", "metric": "frames/s", "value": rate, "unit": "stream-frames/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * cores / rate, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, SURVEY.md §8(d) model)",
        "config": {"workload": f"{args.config}: {W}x{H} gray, k={tracker['subspace_dim']}, "
                               f"p={tracker['p']}, mu={tracker['mu']}, cg={tracker['cg_max_iters']}",
                   "streams_per_step": cores},
        "mpix_per_s": rate * P / 1e6,
        "cpu_baseline": {"value": rate, "unit": "stream-frames/s", "cores": cores,
                         "kind": kind, "cpu": cpu_model(),
                         "sample": f"{cores} worker processes x {n_frames} frames of their own "
                                   f"{_window_note(args.config)} "
                                   f"({'the reference package prost.jobs.StreamTracker.push' if kind == 'reference' else 'numpy port of the reference path'}, "
                                   "OPENBLAS_NUM_THREADS=1)"},
        "e2e": {"value": rate, "unit": "stream-frames/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch

    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist

        if os.environ.get("PROST_BENCH_SHARE_GPU") == "1":
            # test of the multi-rank code path on a box with fewer GPUs than
            # ranks: ranks share devices (their kernels never wait on each
            # other — stream sharding has no data-path collective), gloo for
            # the timing reductions (NCCL refuses two ranks on one device)
            local = local % torch.cuda.device_count()
            torch.cuda.set_device(local)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()

    import paper_1302_2073_b200 as pkg

    c, S, tracker = workload(args.config, args.streams)
    cfg = pkg.RunConfig(i_init=100, **tracker)
    W, H = cfg.target_width, cfg.target_height
    ch = 1 if cfg.grayscale else 3
    P = W * H
    n = P * ch
    k = cfg.subspace_dim
    # C3-style configs shard independent streams over ranks (weak scaling);
    # one very large stream (C4) shards its pixel rows (strong scaling, NCCL
    # all-reduce of the phase partials)
    pixel = args.pixel_shard or (ws > 1 and c.get("shard") == "pixel")
    if pixel:
        S = 1
    stream_ids = [0] if pixel else shard_streams(rank, S)

    preroll = cfg.i_init if args.preroll is None else args.preroll
    run_frames = c["frames"]  # frames per stream of the BASELINE run
    # staged frames: every step a new frame, up to what fits comfortably in HBM
    # (long runs cycle through the staged window after the pre-roll — a scene
    # cut, which the tracker handles like any other frame); the e2e leg cycles
    # through at most 64 pinned host frames
    e2e_frames = 0 if args.no_e2e else min(max(2, args.warmup) + args.steps, 64)
    nblock = 0 if args.block <= 1 else args.block * (max(1, min(args.steps // args.block, 12)) + 2)
    need = preroll + args.warmup + args.steps + 3 + e2e_frames + nblock
    frame_bytes = len(stream_ids) * n * 4
    need_full = need
    need = min(need, max(preroll + args.warmup + 3 * max(args.block, 1) + 16,
                         int(0.3 * torch.cuda.mem_get_info(dev)[0] / frame_bytes)))
    t_gen = time.perf_counter()
    if args.frames > 0:
        # a few distinct frames, cycled (numpy generator, bit-identical to the tests' streams)
        host = gen_frames(args.config, stream_ids, args.frames)  # [F, S, n] float32
        frames_dev = torch.from_numpy(host).to(f"cuda:{dev}")
        data_note = (f"synthetic (seeded SURVEY.md §8(d) generator, {args.frames} distinct frames "
                     "per stream staged in HBM and cycled)")
    else:
        # every step is the next consecutive frame of every stream (a cycled
        # clip would restart the scene every few frames and distort the line
        # search); the scene model runs on the device
        from paper_1302_2073_b200.synth import DeviceScenes, config_spec

        specs = [config_spec(args.config, sid) for sid in stream_ids]
        host = None
        if any(sp.jitter for sp in specs):
            # camera jitter (C2) is generated on the host (numpy), then staged
            frames_dev = torch.from_numpy(gen_frames(args.config, stream_ids, need)).to(f"cuda:{dev}")
            data_note = (f"synthetic (seeded SURVEY.md §8(d) generator on the host: {need} "
                         "consecutive frames per stream staged in HBM, a new frame every step)")
        else:
            # a pixel-sharded stream is the same stream on every rank
            scenes = DeviceScenes(specs, f"cuda:{dev}", seed=1000 + (0 if pixel else rank))
            frames_dev = scenes.next_frames(need)
            del scenes
            data_note = (f"synthetic (seeded SURVEY.md §8(d) scene model run on the device: {need} "
                         "consecutive frames per stream staged in HBM, a new frame every step)")
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t_gen
    F = frames_dev.shape[0]
    if host is None and F < need_full:
        data_note += f" (a {need_full}-frame run: cycled through frames {preroll}..{F - 1} after that)"

    def frame_at(i):
        """Frame i of the run: the staged window, cycled after the pre-roll."""
        if i < F:
            return i
        return i % F if F <= preroll + 1 else preroll + (i - preroll) % (F - preroll)
    from paper_1302_2073_b200 import _native as nat

    if pixel:
        from paper_1302_2073_b200.shard import ShardedTracker

        st = ShardedTracker(cfg, precision=args.precision, device=dev, exchange=args.exchange)
        native = st.native
        W_, r0, r1 = W, st.row0, st.row1
        # this rank's row block of every staged frame
        frames_dev = torch.cat([frames_dev[:, 0, c_ * P + r0 * W_: c_ * P + r1 * W_]
                                for c_ in range(ch)], dim=1).contiguous()[:, None, :]
        P_loc, n_loc = (r1 - r0) * W, (r1 - r0) * W * ch

        def do_push(frame, background, mask):
            st.push(frame[0], background=background[0], mask=mask[0])
    else:
        # one stream per GPU: lay the resident kernel out for latency
        bt = pkg.BatchTracker(cfg, S, precision=args.precision, device=dev, latency=S == 1)
        if args.wave:
            bt.native.set_wave(args.wave)
        native = bt.native
        P_loc, n_loc = P, n

        def do_push(frame, background, mask):
            bt.push(frame, background=background, mask=mask)

    mode = native.query(nat.Q_RESIDENT)
    if pixel:
        kernel_path = (f"pixel-sharded: rows {r0}-{r1} of {H} on rank {rank}, streamed phase "
                       + ("kernels exchanging their partials in-kernel over peer memory"
                          if args.exchange == "peer" else
                          "kernels, NCCL all-reduce of the phase partials (host-driven program)"))
    elif mode:
        cl = native.query(nat.Q_CLUSTER)
        kernel_path = (f"{'tmem' if mode == 2 else 'register'}-resident: "
                       f"{native.query(nat.Q_TEAMS)} teams x "
                       f"{native.query(nat.Q_TEAM)} CTAs x {native.query(nat.Q_GROUPS)} slot groups, "
                       + ("each team one thread-block cluster (DSMEM team sums), one launch per step"
                          if cl else "one cooperative launch per step"))
    else:
        tma = native.query(nat.Q_TMA)
        kernel_path = (f"streamed, TMA-fed: {tma} CTAs x 512 threads per stream per U pass "
                       "(tensor-map tiles + bulk copies)" if tma else
                       f"streamed: {native.query(nat.Q_CHUNKS)} CTAs per stream per phase kernel")
    mask = torch.empty((S, P_loc), dtype=torch.uint8, device=f"cuda:{dev}")
    bg = torch.empty((S, n_loc), dtype=torch.float32 if args.precision == "fp32" else torch.float64,
                     device=f"cuda:{dev}")

    def barrier():
        if ws > 1:
            import torch.distributed as dist

            dist.barrier()

    def max_over_ranks(v):
        return reduce_max(v, ws, f"cuda:{dev}")

    step = 0
    torch.cuda.synchronize()
    t_pre = time.perf_counter()
    p0 = torch.cuda.Event(enable_timing=True)
    p1 = torch.cuda.Event(enable_timing=True)
    for i in range(preroll):
        if i == 1:
            p0.record()
        do_push(frames_dev[frame_at(step)], bg, mask)
        step += 1
    p1.record()
    torch.cuda.synchronize()
    t_pre = time.perf_counter() - t_pre
    # the i_init window (running statistics), device-timed over frames
    # 1..preroll-1 of every stream (frame 0, the cold start and the first
    # launch of the process, stays out)
    ms_pre = max_over_ranks(p0.elapsed_time(p1)) if preroll > 1 else 0.0
    for _ in range(args.warmup):
        do_push(frames_dev[frame_at(step)], bg, mask)
        step += 1
    torch.cuda.synchronize()
    native.synchronize()

    clocks = Clocks(int(os.environ.get("CUDA_VISIBLE_DEVICES", str(dev)).split(",")[0])
                    if os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",")[0].isdigit() else dev)
    clocks.start()
    launches0 = native.launches
    def exchanges_so_far():
        if not pixel:
            return 0
        return st.peer_exchanges() if args.exchange == "peer" else st.exchanges

    ex0 = exchanges_so_far()
    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    n_clk0 = clocks.mark()
    e0.record()
    for _ in range(args.steps):
        do_push(frames_dev[frame_at(step)], bg, mask)
        step += 1
    e1.record()
    torch.cuda.synchronize()
    barrier()
    ms = e0.elapsed_time(e1)
    launches = native.launches - launches0
    ex_timed = (exchanges_so_far() - ex0) / args.steps if pixel else None
    clocks.wait_one_more(n_clk0)
    clk = clocks.stop()
    ms = max_over_ranks(ms)
    ms_step = ms / args.steps
    units = S if pixel else ws * S  # stream-frames of the whole job
    value = units * args.steps / (ms / 1000.0)

    # frame blocking (BatchTracker.push_many): the same streams continue, F
    # consecutive frames per stream per call, each stream's slice kept on chip
    # across its F frames — the same per-frame results (tested bit-identical)
    blocked = None
    FB = args.block if (not pixel and args.block and args.block > 1 and host is None) else 0
    if FB:
        bg_b = torch.empty((FB,) + tuple(bg.shape), dtype=bg.dtype, device=bg.device)
        mask_b = torch.empty((FB,) + tuple(mask.shape), dtype=mask.dtype, device=mask.device)
        reps = max(1, min(args.steps // FB, 12))

        def block_at(i):  # F consecutive staged frames from i (or from the window start)
            i = frame_at(i)
            return i if i + FB <= F else preroll

        s0 = block_at(step)
        bt.push_many(frames_dev[s0:s0 + FB], background=bg_b, mask=mask_b)
        step = s0 + FB
        blocks = []
        for _ in range(reps):
            blocks.append(block_at(step))
            step = blocks[-1] + FB
        torch.cuda.synchronize()
        barrier()
        e0.record()
        for b0 in blocks:
            bt.push_many(frames_dev[b0:b0 + FB], background=bg_b, mask=mask_b)
        e1.record()
        torch.cuda.synchronize()
        barrier()
        ms_b = max_over_ranks(e0.elapsed_time(e1)) / (reps * FB)
        # per-phase split of one blocked call (separate, untimed)
        native.profile(True)
        s0 = block_at(step)
        bt.push_many(frames_dev[s0:s0 + FB], background=bg_b, mask=mask_b)
        step = s0 + FB
        torch.cuda.synchronize()
        ph_b = native.profile_read()
        native.profile(False)
        tmem_blk = native.query(nat.Q_RESIDENT) == 2
        blocked = {"frames_per_call": FB, "value": units / (ms_b / 1000.0), "unit": "stream-frames/s",
                   "ms_per_frame_step": ms_b, "steps": reps * FB,
                   "hbm_bytes_per_stream_frame": (8 * n_loc * k / FB + 12 * n_loc + 3 * P_loc) if tmem_blk
                   else (4 * 4 * n_loc * k + 24 * n_loc + 3 * P_loc),
                   "phases_us_per_frame": {nm: 1000.0 * v[0] / FB for nm, v in ph_b.items() if v[1]},
                   "note": ("BatchTracker.push_many: U crosses HBM once per block of F frames"
                            if tmem_blk else
                            "BatchTracker.push_many on the TMA-fed streamed kernels: each geodesic "
                            "sweep also runs the next frame's pass 0 (4 passes over U per frame "
                            "instead of 5)") +
                           " (per-frame results identical to push; tests/test_gpu_parity.py)"}

    # per-phase breakdown (separate, untimed pass with events around launches)
    native.profile(True)
    for _ in range(3):
        do_push(frames_dev[frame_at(step)], bg, mask)
        step += 1
    torch.cuda.synchronize()
    phases = native.profile_read()
    resident_counters = native.resident_counters() if native.query(nat.Q_RESIDENT) else None
    native.profile(False)

    # end to end through the public API (BatchTracker.push, the StreamTracker
    # seam batched): pinned HOST frames in — 8-bit camera frames, divided by
    # 255 on the device like frameio.py:136 — and, per stream-frame, the
    # FrameRecord fields out (jobs.py:142-151): mask, raw_mask and the
    # FitInfo (fit_cost, step, frame_index, status; delivered asynchronously),
    # plus the background frame with --e2e-background.  Host copies inside the
    # timed region, pipelined against the kernels on the handle's streams.
    e2e = None
    if not args.no_e2e:
        from paper_1302_2073_b200.tracker import FitInfoBuffer

        u8 = not args.e2e_f32 and not pixel
        if host is not None:
            src = torch.from_numpy(host)
            e2e0, HF = 0, src.shape[0]
        else:
            # the e2e frames continue the streams: stage them in pinned host memory
            e2e0, HF = step, e2e_frames
            src = frames_dev[[frame_at(e2e0 + i) for i in range(HF)]]
        if u8:
            host_pinned = torch.empty(tuple(src.shape), dtype=torch.uint8, pin_memory=True)
            host_pinned.copy_(torch.clamp(torch.round(src.float() * 255.0), 0, 255).to(torch.uint8))
        else:
            host_pinned = torch.empty(tuple(src.shape), dtype=src.dtype, pin_memory=True)
            host_pinned.copy_(src)
        want_bg = args.e2e_background or pixel or args.e2e_f32
        mask_h = torch.empty((S, P_loc), dtype=torch.uint8).pin_memory()
        raw_h = torch.empty((S, P_loc), dtype=torch.uint8).pin_memory()
        bg_h = torch.empty((S, n_loc), dtype=bg.dtype).pin_memory() if want_bg else None
        fit_h = FitInfoBuffer(S)

        def push_e2e(frame):
            if pixel:
                do_push(frame, bg_h, mask_h)
            else:
                bt.push(frame, background=bg_h, mask=mask_h, raw_mask=raw_h, fit_out=fit_h)

        for _ in range(max(2, args.warmup)):  # untimed: the host-I/O path's own warm-up
            push_e2e(host_pinned[(step - e2e0) % HF])
            step += 1
        torch.cuda.synchronize()
        native.synchronize()
        barrier()
        e0.record()
        for _ in range(args.steps):
            push_e2e(host_pinned[(step - e2e0) % HF])
            step += 1
        native.join(torch.cuda.current_stream().cuda_stream)  # the last step's copies too
        e1.record()
        torch.cuda.synchronize()
        barrier()
        ms_e2e = max_over_ranks(e0.elapsed_time(e1))
        d2h = S * P_loc + (0 if pixel else S * P_loc + fit_h.nbytes) + (
            S * n_loc * bg_h.element_size() if want_bg else 0)
        e2e = {"value": units * args.steps / (ms_e2e / 1000.0), "unit": "stream-frames/s",
               "h2d_bytes_per_step": S * n_loc * host_pinned.element_size(),
               "d2h_bytes_per_step": d2h,
               "ms_per_step": ms_e2e / args.steps,
               "frames": "u8 (frame/255 on the device)" if u8 else str(host_pinned.dtype),
               "outputs": ("mask, raw_mask, FitInfo" if not pixel else "mask") +
                          (", background" if want_bg else "")}
        if not pixel:
            e2e["fit_cost_finite"] = bool(np.all(np.isfinite(fit_h.fit_costs())))
    native.synchronize()

    # roofline of the frame update (per GPU)
    peaks_path = ROOT / "MEASURED_PEAKS.json"
    if peaks_path.exists():
        peak = float(json.loads(peaks_path.read_text())["hbm_gbs"])
        peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)"
    else:
        peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    ba = b_alg(n_loc, k, P_loc)  # per GPU: its own streams, or its row block
    achieved = S * ba / (ms_step / 1000.0) / 1e9
    bu = 8 * n_loc * k
    traffic = None
    tpath = ROOT / "profiles" / "traffic.json"
    if tpath.exists():
        try:
            tj = json.loads(tpath.read_text())
            if tj.get("config") == args.config and tj.get("streams") == S:
                traffic = tj.get("bytes_per_step")
        except Exception:
            traffic = None
    tot_ms = sum(v[0] for v in phases.values()) or 1.0
    phase_out = {nm: {"ms_per_step": v[0] / 3, "launches_per_step": v[1] / 3,
                      "share": v[0] / tot_ms} for nm, v in phases.items() if v[1]}
    dom = max(phase_out, key=lambda nm: phase_out[nm]["ms_per_step"]) if phase_out else None

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        try:
            rate, cores, frames, wall, kind = cpu_rate(args.config, tracker, args.cpu_frames)
            cpu = {"value": rate, "unit": "stream-frames/s", "cores": cores, "kind": kind,
                   "cpu": cpu_model(),
                   "sample": f"{cores} worker processes x {frames // cores} frames of their own "
                             f"{_window_note(args.config)} "
                             f"({'prost.jobs.StreamTracker.push, the reference package' if kind == 'reference' else 'numpy port of the reference path'}, "
                             f"OPENBLAS_NUM_THREADS=1; {wall:.1f} s wall)"}
            if kind == "reference" and args.cpu_port:
                prate, _, _, pwall, _ = cpu_rate(args.config, tracker, args.cpu_frames, cores,
                                                 kind="port")
                cpu["port_value"] = prate
                cpu["reference_over_port"] = rate / prate
        except Exception as exc:  # the baseline is reported, never required
            cpu = {"value": None, "unit": "stream-frames/s", "cores": None, "kind": reference_kind(),
                   "sample": f"failed: {exc!r}"}

    if rank == 0:
        line = {
            "metric": "frames/s", "value": value, "unit": "stream-frames/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong" if pixel else "weak", "vs_baseline": None,
            "dtype": "f32" if args.precision == "fp32" else "f64",
            "data": data_note,
            "config": {"workload": f"{args.config}: {S} streams/GPU x {W}x{H}x{ch}, k={k}, "
                                   f"p={cfg.p}, mu={cfg.mu}, cg_max_iters={cfg.cg_max_iters}",
                       "streams_per_gpu": S, "n": n, "k": k, "precision": args.precision,
                       "l2": "inputs larger than L2 (U alone is %.2f GB per GPU)" % (S * 4 * n * k / 1e9),
                       "parallelism": f"pixel-row-sharded x{ws}" if pixel else f"stream-sharded x{ws}",
                       "kernel_path": kernel_path},
            "mpix_per_s": value * P / 1e6,
            "gpu_launches": launches,
            "roofline": {"bound": "hbm", "kernel": "frame update (all phase kernels of one step)",
                         "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "frac_nominal_8000": achieved / 8000.0,
                         "traffic": traffic, "peak_source": peak_src,
                         "bytes_per_stream_frame": ba, "b_u_frac": (S * bu / (ms_step / 1e3) / 1e9) / peak,
                         "dominant_phase": dom},
            "phases": phase_out,
            "resident_counters": resident_counters,
            "clocks": clk,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "gen_seconds": t_gen,
            "exchanges_per_frame": ex_timed,
            "blocked": blocked,
            "preroll": {"frames": preroll, "seconds": t_pre,
                        "ms_per_step": ms_pre / (preroll - 1) if preroll > 1 else None,
                        "value": units * (preroll - 1) / (ms_pre / 1e3) if preroll > 1 else None,
                        "note": "frames through the i_init statistics window before warm-up, device-timed "
                                "(frames 1..preroll-1); the timed steps are the steady-state frames"},
            "full_run": ({"frames": run_frames,
                          "value": units * run_frames / ((ms_pre / (preroll - 1) * preroll
                                                          + (run_frames - preroll) * ms_step) / 1e3),
                          "unit": "stream-frames/s",
                          "note": f"the whole {run_frames}-frame BASELINE run: the i_init window at its "
                                  "measured step time, the rest at the timed steady-state step time"}
                         if preroll > 1 and run_frames > preroll else None),
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
