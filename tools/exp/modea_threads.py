"""A/B of the Mode A triangular stream kernel: 1024 threads without the
violation-code table vs 512 threads with it (DM_STREAM_TRI_THREADS=512)."""
import json
import os
import sys

sys.path.insert(0, ".")
import torch

import bench

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
r = bench.mode_a_measure(dev, "c2")
print(json.dumps({"tri_threads": os.environ.get("DM_STREAM_TRI_THREADS", "1024"), "ms": r["ms"], "value": r["value"],
                  "winner": r["winner"]}))
