"""DP timings (C1 grid, C4b) with the warp or CTA kernel: DM_DP_CTA=0|1 python tools/exp/dp_time.py"""
import json
import os
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2309_01172_b200 import engine  # noqa: E402

dev = torch.device("cuda", 0)
r = bench.dp_measure(dev, engine.fp64_peak())
r.pop("roofline", None)
print(os.environ.get("DM_DP_CTA"), "c1", json.dumps({k: r[k] for k in ("ms", "value", "oracle_spot_check")}))
r = bench.dp_c4b_measure(dev)
print(os.environ.get("DM_DP_CTA"), "c4b", json.dumps({k: r[k] for k in ("ms", "value", "oracle_spot_check")}))
r = bench.api_latency_measure(dev)
print("api c1 ms", r["c1"]["ms_per_call"], r["c1"]["same_report"])
