"""Diagnostic: Armijo trial statistics of the GPU tracker vs the CPU oracle on
C3-shaped streams (cost_evals per frame = 1 + sum over iterations of
(accepted trial index + 2))."""
import collections, sys, time
import numpy as np, torch
sys.path.insert(0, '.')
import paper_1302_2073_b200 as pkg
from paper_1302_2073_b200.synth import SceneStream, config_spec
from oracle import prost_oracle as orc

S = int(sys.argv[1]) if len(sys.argv) > 1 else 16
F = int(sys.argv[2]) if len(sys.argv) > 2 else 130
cyc = int(sys.argv[3]) if len(sys.argv) > 3 else 0
W, H = 320, 240
frames = np.stack([SceneStream(config_spec('C3', s)).next_frames(cyc or F) for s in range(S)], 1)
cfg = pkg.RunConfig(subspace_dim=15, p=0.5, mu=1e-4, cg_max_iters=2, target_width=W, target_height=H,
                    grayscale=True, i_init=100, seed=0)
bt = pkg.BatchTracker(cfg, S)
dev = torch.from_numpy(frames.astype(np.float32)).cuda()
hist = collections.defaultdict(collections.Counter)
gpu_costs = []
for t in range(F):
    info = bt.push(dev[t % dev.shape[0]], fit=True)
    ph = 'f<100' if t < 100 else 'f>=100'
    for s in range(S):
        hist[ph][(info[s].iterations, info[s].cost_evals)] += 1
    gpu_costs.append(info[0].fit_cost)
for ph, c in hist.items():
    print(ph, sorted(c.items(), key=lambda kv: -kv[1])[:12])
# oracle on stream 0
prm = cfg.params(100)
ref = orc.PipelineOracle(W, H, 1, orc.OracleParams(k=15, p=0.5, mu=1e-4, delta=0.35, omega=5e-5,
      t_init=5e-3, t_min=1e-4, tau=prm.tau, max_iters=2), i_init=100, seed=0)
oh = collections.Counter()
for t in range(F):
    r = ref.push(frames[t % frames.shape[0], 0].astype(np.float64))
    if t >= 100: oh[(r.fit.iterations, r.fit.cost_evals)] += 1
    if t in (0, 1, 50, 99, 100, F - 1):
        print('frame', t, 'cost gpu', gpu_costs[t], 'oracle', r.fit_cost)
print('oracle stream0 f>=100', sorted(oh.items(), key=lambda kv: -kv[1]))
U = bt.native.get_core_state(0)[0]
print('stream0 sine vs oracle', orc.subspace_sine(U, ref.state.U))
