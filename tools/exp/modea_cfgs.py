"""Mode A stream: time every DM_MODEA_CFG on C1 and C2 (same populations as
bench.mode_a_measure): python tools/exp/modea_cfgs.py [c1|c2] [cfg ...]"""
import math
import os
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2309_01172_b200 import configs as CF, engine  # noqa: E402
from paper_2309_01172_b200.tensorize import build_host  # noqa: E402

dev = torch.device("cuda", 0)
which = sys.argv[1] if len(sys.argv) > 1 else "c1"
cfgs = sys.argv[2:] or [None]
if which == "c1":
    st = CF.model_stages("gpt2-small"); fl = CF.load(CF.c1_fleet_doc(10.0, 1e-3)); n, p = 26, 4
    total = engine.bruteforce_total(n, p)
    base = engine.materialize(n, p, "bruteforce", 0, total, device=dev)
    N = 1 << 27
    own = base.repeat(math.ceil(N / total), 1)[:N].contiguous()
    del base
else:
    st = CF.model_stages("llama2-7b-layers"); fl = CF.load(CF.c2_fleet_doc(0)); n, p = 34, 32
    N = 1 << 28
    own = engine.materialize(n, p, "splits", engine.splits_total(n, p) // 2 - N // 2, N, device=dev)
batch = engine.device_batch([build_host(st, fl)], device=dev)
out = (torch.empty(N, dtype=torch.float64, device=dev), torch.empty(N, dtype=torch.uint8, device=dev))
bufs = engine.WinnerBuffers(dev)
peak = bench._hbm_peak()[0]
for cfg in cfgs:
    if cfg:
        os.environ["DM_MODEA_CFG"] = cfg
    else:
        os.environ.pop("DM_MODEA_CFG", None)
    ms = bench._time_ms(lambda: engine.eval_owner_argmin(batch, own, 0, bufs, out), steps=5)
    gbs = N * (n + 9) / (ms / 1e3) / 1e9
    print(which, cfg, f"ms {ms:.3f} cand/s {N / (ms / 1e3):.3e} GB/s {gbs:.0f} frac {gbs / peak:.3f}",
          bufs.read(), flush=True)
