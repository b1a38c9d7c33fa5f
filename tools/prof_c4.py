"""One C4 schedule batch (for ncu): python tools/prof_c4.py [n_scen]"""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import torch
from paper_2309_01172_b200 import batch as B, engine
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 18
sb = B.c4_batch(n, seed=0, device=torch.device("cuda", 0))
for _ in range(2):
    owner, _, _ = engine.prop_hill(sb, sb.n_max)
    engine.epilogue(sb, sb.n_max, owner, 512, 4)
torch.cuda.synchronize()
