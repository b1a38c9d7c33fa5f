"""Pooled split sweep (dm_enum_splits_pooled): one population swept by
`world` ranks sharing their side tables through device memory.

On one GPU the ranks run on separate streams with plain device workspaces (the
same kernels, barriers and cross-workspace loads as the multi-process pool,
where the peers' workspaces are CUDA IPC mappings over NVLink; the
multi-process form is tools/exp/pool_dist.py under torchrun).  The merged
records of the ranks must equal the single-GPU sweep bit for bit —
winner makespan, rank, evaluated / feasible counts and checksum — for every
world size, over consecutive sweeps of different instances on the same pool
(a rank reading a peer's stale slice would change the checksum)."""

import json
import pathlib

import numpy as np
import pytest

from gen import big_instance

pytestmark = pytest.mark.gpu
GOLD = json.loads((pathlib.Path(__file__).resolve().parent / "golden" / "full_size.json").read_text())
KEYS = ("makespan", "rank", "n_evaluated", "n_feasible", "checksum")


def _pooled(engine, batch, world, wss, nbytes, order=None):
    import torch
    from paper_2309_01172_b200 import dist as D
    streams = [torch.cuda.Stream() for _ in range(world)]
    bufs = [engine.WinnerBuffers(batch.dev_buf.device) for _ in range(world)]
    torch.cuda.synchronize()
    for q in order or range(world):
        with torch.cuda.stream(streams[q]):
            engine.splits_pooled(batch, q, world, wss, nbytes, bufs[q])
    torch.cuda.synchronize()
    for w in wss:
        assert engine.pool_status(w) == 0
    raw = np.concatenate([b.out.cpu().numpy() for b in bufs])
    return D.merge_records(raw), [b.read() for b in bufs]


def test_pooled_sweep_equals_single_sweep(engine_ready):
    import torch
    from paper_2309_01172_b200 import engine
    from paper_2309_01172_b200.tensorize import build_host
    rng = np.random.default_rng(1172)
    insts = []
    for n, p, dag, links, pr in [(12, 5, False, False, (0.05, 0.9)), (26, 12, True, False, (0.2, 0.9)),
                                 (30, 24, False, True, (0.1, 0.6)), (34, 32, False, False, (0.3, 1.2)),
                                 (34, 32, False, False, (0.1, 0.5))]:
        st, fleet = big_instance(rng, n, p, dag=dag, links=links, pressure=pr)
        insts.append(engine.device_batch([build_host(st, fleet)]))
    for world in (1, 2, 3, 4, 8):
        # one pool per shape, reused across consecutive sweeps
        pools = {}
        for rep in range(2):
            for i, batch in enumerate(insts):
                st = batch.struct(0)
                total = engine.splits_total(st.n, st.p)
                want = engine.enum(batch, "splits", 0, total).read()
                nbytes = engine.splits_workspace_bytes(batch)
                assert nbytes > 0, (st.n, st.p)
                key = (st.n, st.p)
                if key not in pools:
                    pools[key] = [torch.zeros(nbytes, dtype=torch.uint8, device="cuda") for _ in range(world)]
                wss = [w.data_ptr() for w in pools[key]]
                order = list(range(world))[::-1] if rep else None
                got, per_rank = _pooled(engine, batch, world, wss, nbytes, order)
                assert got == want, (world, i, rep)
                assert sum(r["n_evaluated"] for r in per_rank) == total


def test_pooled_sweep_c2_scenarios(engine_ready):
    """The bench's C2 scenarios (8,589,934,558 splits each) swept by a pool
    of 2 and 4 ranks equal the pinned full-size goldens."""
    import torch
    from paper_2309_01172_b200 import configs as CF, engine
    from paper_2309_01172_b200.tensorize import build_host
    stages = CF.model_stages("llama2-7b-layers")
    for world in (2, 4):
        wss = None
        for scen in sorted(GOLD["c2"], key=int)[:3]:
            a, bw = CF.C2_LINKS[int(scen)]
            batch = engine.device_batch([build_host(stages, CF.load(CF.c2_fleet_doc(0, a, bw)), True)])
            nbytes = engine.splits_workspace_bytes(batch)
            if wss is None:
                bufs = [torch.zeros(nbytes, dtype=torch.uint8, device="cuda") for _ in range(world)]
                wss = [b.data_ptr() for b in bufs]
            got, _ = _pooled(engine, batch, world, wss, nbytes)
            assert got == {k: GOLD["c2"][scen][k] for k in KEYS}, (world, scen)


def test_pooled_sweep_arguments(engine_ready):
    """Bad rank/world or a short workspace fail with DM_E_ARG, before any launch."""
    import torch
    from paper_2309_01172_b200 import _lib, engine
    from paper_2309_01172_b200.tensorize import build_host
    rng = np.random.default_rng(5)
    st, fleet = big_instance(rng, 10, 4)
    batch = engine.device_batch([build_host(st, fleet)])
    nbytes = engine.splits_workspace_bytes(batch)
    ws = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
    for rank, world, nb in ((2, 2, nbytes), (0, 9, nbytes), (0, 1, nbytes - 1), (-1, 1, nbytes)):
        with pytest.raises(_lib.EngineError):
            engine.splits_pooled(batch, rank, world, [ws.data_ptr()] * max(world, 1), nb)


def test_pool_ipc_alloc_roundtrip(engine_ready):
    """dm_pool_alloc returns zeroed memory and a 64-byte IPC handle."""
    import torch
    from paper_2309_01172_b200 import engine
    ptr, handle = engine.pool_alloc(1 << 20)
    try:
        assert len(handle) == 64
        assert engine.pool_status(ptr) == 0
    finally:
        engine.pool_free(ptr)
    torch.cuda.synchronize()
