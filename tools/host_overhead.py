"""Host cost of one push (Python + ctypes + launches) against the device time,
for the small single-stream configs (C0) where the host can bound the rate.

    python tools/host_overhead.py [C0] [n]
"""
import cProfile
import pstats
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1302_2073_b200 as pkg  # noqa: E402
from paper_1302_2073_b200.synth import CONFIGS, DeviceScenes, config_spec  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C0"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 300
cfg = pkg.RunConfig(i_init=100, **CONFIGS[name]["tracker"])
bt = pkg.BatchTracker(cfg, 1, latency=True)
frames = DeviceScenes([config_spec(name, 0)], "cuda:0", seed=1000).next_frames(n + 110)
P = cfg.target_width * cfg.target_height
ch = 1 if cfg.grayscale else 3
mask = torch.empty((1, P), dtype=torch.uint8, device="cuda")
bg = torch.empty((1, P * ch), dtype=torch.float32, device="cuda")
for i in range(110):
    bt.push(frames[i], background=bg, mask=mask)
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(n):
    bt.push(frames[110 + (i % n)], background=bg, mask=mask)
t_issue = time.perf_counter() - t0
torch.cuda.synchronize()
t_all = time.perf_counter() - t0
print(f"{name}: host issue {1e6 * t_issue / n:.1f} us/push, wall {1e6 * t_all / n:.1f} us/push")
pr = cProfile.Profile()
pr.enable()
for i in range(n):
    bt.push(frames[110 + (i % n)], background=bg, mask=mask)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
