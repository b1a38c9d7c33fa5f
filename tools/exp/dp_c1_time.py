"""C1 link-grid subset-DP timing through bench.dp_measure: python tools/exp/dp_c1_time.py"""
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402

r = bench.dp_measure(torch.device("cuda", 0), 1.85e13)
print({k: r[k] for k in ("ms", "per_python_call_ms", "value", "oracle_spot_check")}, flush=True)
