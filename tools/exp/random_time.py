"""Random-placement timings (C5, C3) through bench.random_measure:
python tools/exp/random_time.py [c5] [c3]"""
import json
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402

dev = torch.device("cuda", 0)
for which in sys.argv[1:] or ["c5", "c3"]:
    r = bench.random_measure(dev, which)
    print(which, json.dumps(r), flush=True)
