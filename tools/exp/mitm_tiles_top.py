import ctypes as C, pathlib, sys
ROOT = pathlib.Path('/root/repo'); sys.path.insert(0, str(ROOT))
import numpy as np, torch
from paper_2309_01172_b200 import _lib, configs as CF, engine
from paper_2309_01172_b200.tensorize import build_host
st = CF.model_stages("llama2-7b-layers"); fl = CF.load(CF.c2_fleet_doc(0))
batch = engine.device_batch([build_host(st, fl)]); total = engine.splits_total(34, 32)
bufs = engine.WinnerBuffers(batch.dev_buf.device)
for _ in range(3): engine.enum(batch, "splits", 0, total, bufs)
torch.cuda.synchronize()
lib = _lib.load(); buf = (C.c_uint * ((1 << 16) * 4))(); lib.dm_debug_mitm_tiles(buf)
a = np.frombuffer(buf, dtype=np.uint32).reshape(-1, 4).astype(np.int64)[:5850]
order = np.argsort(-a[:, 1])
print("top tiles: g blk clocks_us nx ny")
for g in order[:25]: print(g, a[g,0], round(a[g,1]/1965,1), a[g,2], a[g,3])
print("first 30 tiles us:", [round(v/1965,1) for v in a[:30,1]])
print("tiles 296..326 us:", [round(v/1965,1) for v in a[296:326,1]])
