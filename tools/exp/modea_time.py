"""Mode A stream timings (C1, C2) through bench.mode_a_measure:
python tools/exp/modea_time.py [c1] [c2]"""
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402

dev = torch.device("cuda", 0)
for which in sys.argv[1:] or ["c1", "c2"]:
    r = bench.mode_a_measure(dev, which)
    print(which, f"ms {r['ms']:.3f} cand/s {r['value']:.3e} frac {r['roofline']['frac']:.3f}",
          r["winner"], r.get("matches_mode_b"), flush=True)
