"""Outputs of one library build on a C3-shaped batch (24 streams, 8 frames):
masks, backgrounds and three streams' bases, saved to an .npz — run it once
per build (PROST_LIB=path/to/variant.so) and compare the files to check that a
change is bit-identical.

    PROST_LIB=$PWD/_lib/exp/a.so python tools/bitcmp.py /tmp/a.npz
"""
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_1302_2073_b200 as pkg
from paper_1302_2073_b200.synth import DeviceScenes, config_spec
S, F = 24, 8
cfg = pkg.RunConfig(subspace_dim=15, p=0.5, mu=1e-4, cg_max_iters=2, target_width=320, target_height=240, grayscale=True, i_init=3, seed=0)
fr = DeviceScenes([config_spec("C3", s) for s in range(S)], "cuda:0", seed=3).next_frames(F)
bt = pkg.BatchTracker(cfg, S, seeds=list(range(S)))
m = torch.empty((S, 76800), dtype=torch.uint8, device="cuda"); b = torch.empty((S, 76800), device="cuda")
outs = []
for f in range(F):
    bt.push(fr[f], background=b, mask=m)
    outs.append(m.cpu().numpy().copy()); outs.append(b.cpu().numpy().copy())
outs.append(np.stack([bt.native.get_core_state(s)[0] for s in (0, 11, 23)]))
np.savez(sys.argv[1], *outs)
