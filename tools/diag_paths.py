"""Diagnostic: tmem vs streamed kernel paths on a small C3-shaped batch,
frame by frame (fit cost, iterations, cost evaluations, bg difference)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, '.')
import paper_1302_2073_b200 as pkg
from paper_1302_2073_b200.synth import SceneSpec, SceneStream


def c0_stream(n_frames, width, height, seed):
    spec = SceneSpec(width=width, height=height, channels=1, rank=5, noise=0.02, seed=seed)
    return SceneStream(spec).next_frames(n_frames)

W, H, S, F = 320, 240, 6, 8
cfg = pkg.RunConfig(subspace_dim=15, p=0.5, mu=1e-4, cg_max_iters=2, target_width=W,
                    target_height=H, grayscale=True, i_init=4, seed=0)
data = [c0_stream(F, W, H, seed=s) for s in range(S)]
res = {}
for path in ("tmem", "streamed"):
    os.environ["PROST_KERNEL"] = path
    bt = pkg.BatchTracker(cfg, S, seeds=list(range(S)))
    bg = torch.empty((S, W * H), dtype=torch.float32, device="cuda")
    mask = torch.empty((S, W * H), dtype=torch.uint8, device="cuda")
    rows = []
    for f in range(F):
        fr = torch.from_numpy(np.stack([d[f] for d in data]).astype(np.float32)).cuda()
        info = bt.push(fr, background=bg, mask=mask, fit=True)
        rows.append(([(i.fit_cost, i.iterations, i.cost_evals) for i in info], bg.cpu().numpy().copy(),
                     mask.cpu().numpy().copy()))
    res[path] = rows
for f in range(F):
    a, b = res["tmem"][f], res["streamed"][f]
    for s in range(S):
        ca, cb = a[0][s], b[0][s]
        rel = np.linalg.norm(a[1][s] - b[1][s]) / np.linalg.norm(b[1][s])
        mk = np.mean(a[2][s] != b[2][s])
        flag = "" if (ca[1:] == cb[1:] and rel < 1e-6) else "  <--"
        print(f"f{f} s{s} cost {ca[0]:.6f} vs {cb[0]:.6f}  it/evals {ca[1:]} vs {cb[1:]}  bg rel {rel:.2e} mask {mk:.5f}{flag}")
