"""One C2 exhaustive split sweep (for ncu): python tools/prof_splits.py [k1]"""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import torch
from paper_2309_01172_b200 import configs as CF, engine
from paper_2309_01172_b200.tensorize import build_host
st = CF.model_stages("llama2-7b-layers"); fl = CF.load(CF.c2_fleet_doc(0))
batch = engine.device_batch([build_host(st, fl)])
total = engine.splits_total(34, 32)
k1 = int(sys.argv[1]) if len(sys.argv) > 1 else total
print(engine.enum(batch, "splits", 0, k1).read())
torch.cuda.synchronize()
