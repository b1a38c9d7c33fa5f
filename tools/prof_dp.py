"""C1 link-grid DP batch (for ncu): python tools/prof_dp.py"""
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2309_01172_b200 import configs as CF, engine  # noqa: E402
from paper_2309_01172_b200.tensorize import build_host  # noqa: E402

stages = CF.model_stages("gpt2-small")
bws, alphas = CF.c1_link_grid()
fleets = [CF.load(CF.c1_fleet_doc(bw, al)) for bw in bws for al in alphas]
batch = engine.device_batch([build_host(stages, f, True) for f in fleets])
for _ in range(3):
    engine.subset_dp(batch, 26, 4)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20):
    engine.subset_dp(batch, 26, 4)
b.record()
b.synchronize()
print(f"subset_dp x1024 C1 fleets: {a.elapsed_time(b) / 20:.3f} ms per call")
