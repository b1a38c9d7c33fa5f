"""Phase timing of the split sweep (debug build with -DDM_MITM_TIMING):
python tools/exp/mitm_phases.py — per-phase min/median/max over CTAs (us)."""
import ctypes as C
import pathlib
import statistics
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
buf = (C.c_ulonglong * (1024 * 12))()
lib.dm_debug_mitm_times(buf)
a = np.frombuffer(buf, dtype=np.uint64).reshape(1024, 12).astype(np.int64)
a = a[a[:, 0] > 0]
a[:, 4:6] = a[:, 4:6]
t0 = a[:, 0].min()
names = ["T load", "plan", "tiles"]
for i, nm in enumerate(names):
    d = (a[:, i + 1] - a[:, i]) / 1e3
    print(f"{nm:12s} min {d.min():8.1f} med {statistics.median(d):8.1f} max {d.max():8.1f} us")
print(f"pairs processed: normal tiles {a[:, 4].sum():.4g}, thin tiles {a[:, 5].sum():.4g}")
print(f"sweep kernel (first start -> last end) {(a[:, 3].max() - t0) / 1e3:.1f} us; CTAs {len(a)}")
tot = a[:, 8].astype(float)
print(f"clock share (thread 0): elements+barrier {a[:, 6].sum() / tot.sum():.3f}  cross {a[:, 7].sum() / tot.sum():.3f}  "
      f"rest {(tot.sum() - a[:, 6].sum() - a[:, 7].sum()) / tot.sum():.3f}")
print(f"tiles {a[:, 9].sum()} (thin {a[:, 10].sum()}), per CTA min {a[:, 9].min()} max {a[:, 9].max()}")
end = np.sort((a[:, 3] - t0) / 1e3)
print("CTA end times (us) percentiles 0/10/50/90/95/99/100:",
      [round(float(np.percentile(end, q)), 1) for q in (0, 10, 50, 90, 95, 99, 100)])
print("last 12 CTAs end:", [round(float(v), 1) for v in end[-12:]])
