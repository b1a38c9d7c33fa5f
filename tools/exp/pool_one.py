"""Pooled-sweep kernel variant on ONE GPU (world = 1: every load local, the
queue local) against the normal sweep of the same C2 scenario, with phase
times (dm_sweep_timing): separates the POOL kernel's own cost from
multi-GPU effects."""
import ctypes as C
import json
import pathlib
import sys

import numpy as np
import torch

ROOT = pathlib.Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from paper_2309_01172_b200 import _lib, configs as CF, engine  # noqa: E402
from paper_2309_01172_b200.tensorize import build_host  # noqa: E402


def main():
    lib = _lib.load()
    engine.warmup()
    stages = CF.model_stages("llama2-7b-layers")
    batch = engine.device_batch([build_host(stages, CF.load(CF.c2_fleet_doc(0, *CF.C2_LINKS[0])), True)])
    total = engine.splits_total(len(stages), 32)
    nbytes = engine.splits_workspace_bytes(batch)
    ws = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
    bufs = engine.WinnerBuffers(ws.device)
    out = {}
    for name, fn in (("normal", lambda: engine.enum(batch, "splits", 0, total, bufs=bufs)),
                     ("pooled_world1", lambda: engine.splits_pooled(batch, 0, 1, [ws.data_ptr()], nbytes, bufs))):
        fn()
        lib.dm_sweep_timing(1, None, None)
        acc = []
        for _ in range(7):
            fn()
            a, b = C.c_float(0), C.c_float(0)
            _lib.check(lib.dm_sweep_timing(-1, C.byref(a), C.byref(b)))
            acc.append((a.value, b.value))
        lib.dm_sweep_timing(0, None, None)
        out[name] = {"tables_ms": float(np.median([x[0] for x in acc])),
                     "plan_sweep_ms": float(np.median([x[1] for x in acc])), "winner": bufs.read()}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
