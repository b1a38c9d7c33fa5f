"""C4b subset-DP batch timing through bench.dp_c4b_measure: python tools/exp/dp_c4b_time.py"""
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402

r = bench.dp_c4b_measure(torch.device("cuda", 0))
print({k: r[k] for k in ("ms", "value", "oracle_spot_check")}, flush=True)
