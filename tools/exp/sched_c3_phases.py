"""Phase times of one public schedule() call on C3: tensorise, device
(H2D + kernels + D2H + sync), report assembly: python tools/exp/sched_c3_phases.py"""
import pathlib
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402

from paper_2309_01172_b200 import configs as CF, engine, scheduling as S  # noqa: E402
from paper_2309_01172_b200.tensorize import build_host  # noqa: E402

engine.warmup()
stages = CF.model_stages("llama2-70b")
fleet = CF.load(CF.c3_fleet_doc(0))
workers = fleet.worker_ids()
n, p = len(stages), len(workers)
pairs = [(q - 1, q) for q in range(1, min(n, p))]
t = {"worker_ids": [], "build_host": [], "device": [], "report": [], "total": []}
for it in range(60):
    t0 = time.perf_counter()
    w = fleet.worker_ids()
    t1 = time.perf_counter()
    host = build_host(stages, fleet, True, link_pairs=pairs, workers=w)
    t2 = time.perf_counter()
    out = engine.schedule_slot().schedule(host, False, False)
    t3 = time.perf_counter()
    b, pe = out["bounds"], out["peers"]
    runs = tuple((w[int(pe[q])], tuple(range(int(b[q]), int(b[q + 1])))) for q in range(out["n_runs"]))
    r = out["n_runs"]
    res = dict(cand_ptr=np.array([0, r]), code=np.array([out["code"]]), code_run=np.array([out["bad_run"]]),
               compute=out["compute"], read=out["read"], makespan=np.array([out["makespan"]]))
    S._report(stages, fleet, runs, True, ("x",), res, 0, host)
    t4 = time.perf_counter()
    S.schedule(stages, fleet)
    t5 = time.perf_counter()
    if it >= 10:
        for k, v in zip(t, (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4)):
            t[k].append(v * 1e3)
print({k: round(float(np.median(v)), 3) for k, v in t.items()})
