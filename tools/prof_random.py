"""One C5 random-placement pass (for ncu): python tools/prof_random.py [N]"""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_2309_01172_b200 import configs as CF, engine, rng as R
from paper_2309_01172_b200.tensorize import build_host
st = CF.model_stages("opt-175b"); fl = CF.load(CF.c5_fleet_doc(0)); _, on = CF.c5_churn(1024, 0.1, 0)
host = build_host(st, fl)
batch = engine.device_batch([host])
online = torch.tensor([host.index_of[i] for i in on], dtype=torch.int32, device="cuda")
N = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
engine.enum(batch, "random", 0, min(N, 1 << 20), online=online, seed=20260).read()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
bufs = engine.enum(batch, "random", 0, N, online=online, seed=20260)
b.record(); b.synchronize()
print(bufs.read(), "ms", a.elapsed_time(b), "cand/s", N / (a.elapsed_time(b) / 1e3))
