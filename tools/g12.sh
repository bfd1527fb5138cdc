mkdir -p gpurun_out
python - <<'PY'
import os, sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1302_2073_b200 as pkg
from paper_1302_2073_b200 import _native as nat
from paper_1302_2073_b200.synth import SceneSpec, SceneStream
W, H, S, F = 640, 480, 2, 8
cfg = pkg.RunConfig(subspace_dim=20, p=0.5, mu=1e-4, cg_max_iters=2, target_width=W, target_height=H, grayscale=True, i_init=4, seed=0)
data = [SceneStream(SceneSpec(width=W, height=H, channels=1, rank=6, noise=0.03, seed=s)).next_frames(F) for s in range(S)]
out = {}
for path in ("tmem", "streamed"):
    os.environ["PROST_KERNEL"] = path
    bt = pkg.BatchTracker(cfg, S, seeds=list(range(S)))
    print(path, "mode", bt.native.query(nat.Q_RESIDENT), "teams", bt.native.query(nat.Q_TEAMS), "G", bt.native.query(nat.Q_TEAM))
    mask = torch.empty((S, W*H), dtype=torch.uint8, device="cuda"); bg = torch.empty((S, W*H), dtype=torch.float32, device="cuda")
    for f in range(F):
        info = bt.push(torch.from_numpy(np.stack([d[f] for d in data]).astype(np.float32)).cuda(), background=bg, mask=mask, fit=True)
    out[path] = (mask.cpu().numpy(), bg.cpu().numpy(), [info[s].fit_cost for s in range(S)])
(m1,b1,c1),(m2,b2,c2) = out["tmem"], out["streamed"]
print("mask dis", np.mean(m1!=m2), "bg rel", np.linalg.norm(b1-b2)/np.linalg.norm(b2), "costs", c1, c2)
PY
timeout 600 python bench.py --config C2 --no-cpu --steps 10 --warmup 3 > gpurun_out/b_C2.log 2>&1; echo "C2 rc=$?"
tail -1 gpurun_out/b_C2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms/step %.4f  value %.1f  frac %.3f e2e %.1f' % (d['ms_per_step'], d['value'], d['roofline']['frac'], d['e2e']['value'])); print(d['config'].get('kernel_path'), d.get('resident_counters'))"
