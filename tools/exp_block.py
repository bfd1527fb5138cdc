"""Frame blocking on C3: stream-frames/s of push (one frame per call) vs
push_many (F frames per call), frames resident in HBM, CUDA events."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1302_2073_b200 as pkg  # noqa: E402
from paper_1302_2073_b200.synth import CONFIGS, DeviceScenes, config_spec  # noqa: E402

S = 256
cfg = pkg.RunConfig(i_init=100, **CONFIGS["C3"]["tracker"])
n = cfg.target_width * cfg.target_height
scenes = DeviceScenes([config_spec("C3", s) for s in range(S)], "cuda:0", seed=1000)
Fmax = int(sys.argv[1]) if len(sys.argv) > 1 else 8
frames = scenes.next_frames(100 + 4 * 16 + 4 * Fmax + 8)  # [T, S, n]
bt = pkg.BatchTracker(cfg, S, seeds=[0] * S, init_bases=False)
mask = torch.empty((Fmax, S, n), dtype=torch.uint8, device="cuda")
bg = torch.empty((Fmax, S, n), dtype=torch.float32, device="cuda")
t = 0
for _ in range(100):
    bt.push(frames[t], background=bg[0], mask=mask[0])
    t += 1
torch.cuda.synchronize()
for F in [1, 2, 4, Fmax]:
    reps = max(1, 16 // F)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    bt.push_many(frames[t:t + F], background=bg[:F], mask=mask[:F])
    t += F
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        bt.push_many(frames[t:t + F], background=bg[:F], mask=mask[:F])
        t += F
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / (reps * F)
    print(f"F={F}: {ms:.4f} ms per frame-step, {S / ms * 1e3:.0f} stream-frames/s", flush=True)
