"""C4b subset-DP batch (for ncu): python tools/prof_dp_c4b.py [n_scen]"""
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2309_01172_b200 import configs as CF, engine  # noqa: E402
from paper_2309_01172_b200.tensorize import build_host  # noqa: E402

n_scen = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
rng = np.random.default_rng(7)
models = {L: CF.encoder_stages(4096, L, 32000, 4, 1024, cells="layer") for L in range(24, 37)}
hosts = []
for _ in range(n_scen):
    L = int(rng.integers(24, 37))
    p = int(rng.integers(5, 9))
    peers = CF.hetero_peers(p, int(rng.integers(1 << 30)), lam=(0.3, 1.0))
    fl = CF.load(CF.fleet_doc(peers, float(rng.uniform(0, 1e-2)), float(10 ** rng.uniform(-1, 1))))
    hosts.append(build_host(models[L], fl, True))
batch = engine.device_batch(hosts)
n_max = max(h.n for h in hosts)
for _ in range(2):
    engine.subset_dp(batch, n_max, 8)
torch.cuda.synchronize()
