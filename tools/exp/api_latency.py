"""schedule() latency through the public API vs the reference's own, C1 and C3:
python tools/exp/api_latency.py"""
import json
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402

print(json.dumps(bench.api_latency_measure(torch.device("cuda", 0)), indent=1))
