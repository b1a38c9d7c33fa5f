"""Where does one public-API schedule() call (C1) spend its time?  cProfile
with CUDA syncs attributed to the caller, plus a torch profiler kernel list."""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import torch

from paper_2309_01172_b200 import configs as CF
from paper_2309_01172_b200 import scheduling as S

stages = CF.model_stages("gpt2-small")
fleet = CF.load(CF.c1_fleet_doc(10.0, 1e-3))
for _ in range(3):
    S.schedule(stages, fleet)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    S.schedule(stages, fleet)
print("ms/call", (time.perf_counter() - t0) / 10 * 1e3, "links", len(fleet.links))
cProfile.run("for _ in range(10): S.schedule(stages, fleet)", "/tmp/api.prof")
pstats.Stats("/tmp/api.prof").sort_stats("cumtime").print_stats(25)
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA, torch.profiler.ProfilerActivity.CPU]) as prof:
    S.schedule(stages, fleet)
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=15))
