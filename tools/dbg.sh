PROST_DEBUG=1 PROST_LIB=$PWD/paper_1302_2073_b200/_lib/exp/b_nt256.so python -c "
import paper_1302_2073_b200 as pkg, numpy as np
from paper_1302_2073_b200.tracker import BatchTracker
cfg = pkg.RunConfig(subspace_dim=15, p=0.5, mu=1e-4, cg_max_iters=2, target_width=320, target_height=240, grayscale=True)
bt = BatchTracker(cfg, 256, init_bases=False)
" 2>&1 | grep -v rejected | head
