"""schedule() over C4 scenarios (prop_hill + epilogue): python tools/exp/c4_time.py [n_scen]"""
import json
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2309_01172_b200 import engine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10 ** 6
r = bench.c4_measure(torch.device("cuda", 0), engine.fp64_peak(), n_scen=n)
r.pop("roofline", None)
print(json.dumps(r))
