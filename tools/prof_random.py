"""One random-placement launch of 2^24 candidates (for ncu: the first
launch is the profiled one): python tools/prof_random.py [c5|c3] [N]"""
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2309_01172_b200 import configs as CF, engine  # noqa: E402
from paper_2309_01172_b200.tensorize import build_host  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c5"
N = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 24
if which == "c5":
    st, fl = CF.model_stages("opt-175b"), CF.load(CF.c5_fleet_doc(0))
    on = CF.c5_churn(1024, 0.1, 0)[1]
else:
    st, fl = CF.model_stages("llama2-70b"), CF.load(CF.c3_fleet_doc(0))
    on = list(fl.worker_ids())
host = build_host(st, fl)
batch = engine.device_batch([host])
online = torch.tensor([host.index_of[i] for i in on], dtype=torch.int32, device="cuda")
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
bufs = engine.enum(batch, "random", 0, N, online=online, seed=20260)
b.record()
b.synchronize()
print(bufs.read(), "ms", a.elapsed_time(b), "cand/s", N / (a.elapsed_time(b) / 1e3))
