"""One Mode A stream pass (for ncu): python tools/prof_modea.py c1|c2"""
import sys, pathlib, math
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import torch
from paper_2309_01172_b200 import configs as CF, engine
from paper_2309_01172_b200.tensorize import build_host
which = sys.argv[1] if len(sys.argv) > 1 else "c1"
if which == "c1":
    st = CF.model_stages("gpt2-small"); fl = CF.load(CF.c1_fleet_doc(10.0, 1e-3)); n, p = 26, 4
    total = engine.bruteforce_total(n, p)
    base = engine.materialize(n, p, "bruteforce", 0, total)
    own = base.repeat(math.ceil((1 << 25) / total), 1)[: 1 << 25].contiguous()
else:
    st = CF.model_stages("llama2-7b-layers"); fl = CF.load(CF.c2_fleet_doc(0)); n, p = 34, 32
    own = engine.materialize(n, p, "splits", 4_000_000_000, 1 << 25)
batch = engine.device_batch([build_host(st, fl)])
(mk, code), bufs = engine.eval_owner_argmin(batch, own)
print(bufs.read())
torch.cuda.synchronize()
