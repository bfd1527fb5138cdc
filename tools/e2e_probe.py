"""Where the C3 end-to-end step goes: PCIe copy rates on this box and the
pipelined push with growing output sets (u8 pinned host frames in).

    python tools/e2e_probe.py [steps]
"""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1302_2073_b200 as pkg  # noqa: E402
from paper_1302_2073_b200.synth import CONFIGS, DeviceScenes, config_spec  # noqa: E402
from paper_1302_2073_b200.tracker import FitInfoBuffer  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
S, P = 256, 320 * 240
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def rate(fn, n=steps):
    fn()
    torch.cuda.synchronize()
    a, b = ev(), ev()
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


h8 = torch.empty((S, P), dtype=torch.uint8, pin_memory=True)
d8 = torch.empty((S, P), dtype=torch.uint8, device="cuda")
for name, fn, nb in (("H2D 19.7 MB", lambda: d8.copy_(h8, non_blocking=True), S * P),
                     ("D2H 19.7 MB", lambda: h8.copy_(d8, non_blocking=True), S * P)):
    ms = rate(fn)
    print(f"{name}: {ms:.3f} ms = {nb / ms / 1e6:.1f} GB/s")

cfg = pkg.RunConfig(i_init=100, **CONFIGS["C3"]["tracker"])
bt = pkg.BatchTracker(cfg, S)
frames = DeviceScenes([config_spec("C3", s) for s in range(S)], "cuda:0", seed=1000).next_frames(130)
mask_d = torch.empty((S, P), dtype=torch.uint8, device="cuda")
for f in range(100):
    bt.push(frames[f], mask=mask_d)
host = torch.empty((30, S, P), dtype=torch.uint8, pin_memory=True)
host.copy_(torch.clamp(torch.round(frames[100:130].float() * 255), 0, 255).to(torch.uint8))
mask_h = torch.empty((S, P), dtype=torch.uint8).pin_memory()
raw_h = torch.empty((S, P), dtype=torch.uint8).pin_memory()
fit_h = FitInfoBuffer(S)
i = [0]


def nxt():
    i[0] += 1
    return host[i[0] % 30]


def nxt_dev(src):
    i[0] += 1
    return src[i[0] % 30]


print(f"device frames, device mask: {rate(lambda: bt.push(nxt_dev(frames[100:130]), mask=mask_d)):.3f} ms")
dev8 = host.cuda()
print(f"device u8 frames, device mask: {rate(lambda: bt.push(nxt_dev(dev8), mask=mask_d)):.3f} ms")
for label, kw in (("u8 in, nothing out", {}),
                  ("u8 in, mask", dict(mask=mask_h)),
                  ("u8 in, mask + raw", dict(mask=mask_h, raw_mask=raw_h)),
                  ("u8 in, mask + raw + FitInfo", dict(mask=mask_h, raw_mask=raw_h, fit_out=fit_h))):
    def fn(kw=kw):
        bt.push(nxt(), **kw)
    t0 = time.perf_counter()
    ms = rate(fn)
    bt.join(torch.cuda.current_stream().cuda_stream)
    print(f"{label}: {ms:.3f} ms/step (host {1e3 * (time.perf_counter() - t0) / (steps + 1):.3f} ms/step)")
