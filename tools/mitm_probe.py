"""Probe the whole-population split sweep on one generated instance (debug aid):
python tools/mitm_probe.py N P [dag] — prints the MITM and memo-kernel records."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
from gen import big_instance  # noqa: E402
from paper_2309_01172_b200 import engine  # noqa: E402
from paper_2309_01172_b200.tensorize import build_host  # noqa: E402

n, p = int(sys.argv[1]), int(sys.argv[2])
dag = len(sys.argv) > 3 and sys.argv[3] == "dag"
rng = np.random.default_rng(12)
st, fleet = big_instance(rng, n, p, dag=dag, pressure=(0.2, 0.9))
batch = engine.device_batch([build_host(st, fleet)])
total = engine.splits_total(n, p)
print("mitm", engine.enum(batch, "splits", 0, total).read(), flush=True)
os.environ["DM_DISABLE_MITM"] = "1"
print("memo", engine.enum(batch, "splits", 0, total).read(), flush=True)
