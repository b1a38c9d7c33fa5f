"""Per-tile clocks of the split sweep (debug build with -DDM_MITM_TIMING):
python tools/exp/mitm_tiles.py — tile durations vs the planner's estimate."""
import ctypes as C
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2309_01172_b200 import _lib, configs as CF, engine  # noqa: E402
from paper_2309_01172_b200.tensorize import build_host  # noqa: E402

st = CF.model_stages("llama2-7b-layers")
fl = CF.load(CF.c2_fleet_doc(0))
batch = engine.device_batch([build_host(st, fl)])
total = engine.splits_total(34, 32)
bufs = engine.WinnerBuffers(batch.dev_buf.device)
for _ in range(3):
    engine.enum(batch, "splits", 0, total, bufs)
torch.cuda.synchronize()
lib = _lib.load()
buf = (C.c_uint * ((1 << 16) * 4))()
lib.dm_debug_mitm_tiles(buf)
a = np.frombuffer(buf, dtype=np.uint32).reshape(-1, 4).astype(np.int64)
nt = int((a[:, 1] > 0).sum())
a = a[:nt]
clk, nx, ny = a[:, 1], a[:, 2], a[:, 3]
est = nx * ny + 256 * (nx + ny)
thin = ny < 256
print(f"tiles {nt}; thin {thin.sum()}")
for nm, msk in (("normal", ~thin), ("thin", thin)):
    c, e = clk[msk], est[msk]
    if len(c) == 0:
        continue
    r = c / e
    print(f"{nm:7s} clocks/est-unit: median {np.median(r):.4f} p10 {np.percentile(r, 10):.4f} p90 {np.percentile(r, 90):.4f}"
          f"  total clocks {c.sum():.4g} ({c.sum() / clk.sum() * 100:.1f}%)  median tile {np.median(c) / 1965:.1f} us")
# fit clocks ~ a*pairs + b*elements + c per tile
X = np.stack([nx * ny, nx + ny, np.ones_like(nx)], 1).astype(float)
for nm, msk in (("normal", ~thin), ("thin", thin)):
    coef, *_ = np.linalg.lstsq(X[msk], clk[msk].astype(float), rcond=None)
    print(f"{nm:7s} fit clocks = {coef[0]:.4f}*pairs + {coef[1]:.2f}*elements + {coef[2]:.0f}")
print("last 20 tiles (queue order): us", [round(float(v) / 1965, 1) for v in clk[-20:]])
print("largest 10 tiles us", [round(float(v) / 1965, 1) for v in np.sort(clk)[-10:]])
