"""cProfile of one public schedule() call on C3 (256 workers, 32,640 links):
python tools/exp/sched_c3_prof.py"""
import cProfile
import pathlib
import pstats
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2309_01172_b200 import configs as CF, engine, scheduling as S  # noqa: E402

engine.warmup()
stages = CF.model_stages("llama2-70b")
fleet = CF.load(CF.c3_fleet_doc(0))
for _ in range(5):
    S.schedule(stages, fleet)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(50):
    S.schedule(stages, fleet)
print("ms per call", (time.perf_counter() - t) / 50 * 1e3)
pr = cProfile.Profile()
pr.enable()
for _ in range(50):
    S.schedule(stages, fleet)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
