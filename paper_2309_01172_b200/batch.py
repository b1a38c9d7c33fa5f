"""Vectorised construction of large scenario batches (config C4: 10^6
independent schedule() problems).

A scenario = one of a few distinct stage tables (the 196 (L, h) models of C4)
+ its own fleet (p workers drawn from GPU_TABLE with lambda, a default link).
Stage tables are packed once per model; the per-scenario peer columns are
built with numpy in one shot (the same IEEE float64 products parse_fleet
performs: tflops * 1e12, gpu_gb * 2^30, peak * lambda) and the dm_tables
records are filled column-wise, so 10^6 scenarios tensorise in about a
second instead of a Python loop per scenario.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .refapi import GPU_TABLE
from .tensorize import TABLES_DTYPE, HostTables

_KINDS = tuple(GPU_TABLE)


class ScenarioBatch:
    """Device-resident batch of scenarios sharing a small set of models."""

    def __init__(self, models: list[HostTables], scen_model, scen_p, scen_kind, scen_lam, scen_alpha, scen_beta,
                 include_comm=True, device="cuda", compute_column="tensor"):
        import torch

        scen_model = np.asarray(scen_model, np.int64)
        scen_p = np.asarray(scen_p, np.int64)
        ns = scen_model.size
        self.n_scen = ns
        self.models = models
        self.scen_model = scen_model
        self.scen_p = scen_p
        # ---- model segments, packed once
        sizes = [m.packed_size() for m in models]
        mbuf = np.zeros(sum(sizes) + 256, np.uint8)
        moffs, base = [], 0
        for m, sz in zip(models, sizes):
            moffs.append(m.pack_into(mbuf, base))
            base += sz
        # ---- peer columns for every scenario (flat, offsets by cumsum of p)
        poff = np.zeros(ns + 1, np.int64)
        np.cumsum(scen_p, out=poff[1:])
        kinds = np.asarray(scen_kind, np.int64)
        lam = np.asarray(scen_lam, np.float64)
        tfl = np.array([getattr(GPU_TABLE[k], f"tflops_{compute_column}") for k in _KINDS], np.float64)
        mem = np.array([float(GPU_TABLE[k].memory_gb) for k in _KINDS], np.float64)
        peak = tfl[kinds] * 1e12
        speed = peak * lam
        capg = mem[kinds] * float(2 ** 30)
        capc = np.full(speed.size, 16.0 * 2 ** 30)
        capd = np.full(speed.size, 64.0 * 2 ** 30)
        P_total = speed.size
        seg = (P_total * 8 + 255) // 256 * 256
        total = base + 4 * seg + 256
        self.host_buf = torch.empty(total, dtype=torch.uint8, pin_memory=True)
        hb = self.host_buf.numpy()
        hb[:base] = mbuf[:base]
        for j, col in enumerate((speed, capg, capc, capd)):
            hb[base + j * seg: base + j * seg + col.nbytes] = col.view(np.uint8)
        self.dev_buf = torch.empty(total, dtype=torch.uint8, device=device)
        self.dev_buf.copy_(self.host_buf, non_blocking=True)
        d0 = int(self.dev_buf.data_ptr())
        # ---- records
        recs = np.zeros(ns, dtype=TABLES_DTYPE)
        mrec = np.zeros(len(models), dtype=TABLES_DTYPE)
        for i, (m, o) in enumerate(zip(models, moffs)):
            mrec[i] = m.struct_record(o, d0)
        r = mrec[scen_model]
        for name in ("n", "n_edges", "flops", "gpu", "cpu", "disk", "pre_flops", "pre_gpu", "pre_cpu",
                     "pre_disk", "edge_ptr", "edge_src", "edge_m"):
            recs[name] = r[name]
        recs["p"] = scen_p
        recs["P"] = scen_p
        mflags = r["flags"] & ~np.uint32(_lib.DM_F_PAIR_LINKS | _lib.DM_F_INCLUDE_COMM)
        recs["flags"] = mflags | (np.uint32(_lib.DM_F_INCLUDE_COMM) if include_comm else np.uint32(0))
        recs["def_alpha"] = np.asarray(scen_alpha, np.float64)
        recs["def_beta"] = np.asarray(scen_beta, np.float64)
        for j, name in enumerate(("speed", "cap_gpu", "cap_cpu", "cap_disk")):
            recs[name] = d0 + base + j * seg + 8 * poff[:-1]
        self.records = recs
        self.records_host = torch.from_numpy(recs.view(np.uint8).copy()).pin_memory()
        self.structs_dev = torch.empty(recs.nbytes, dtype=torch.uint8, device=device)
        self.structs_dev.copy_(self.records_host, non_blocking=True)
        self.n_max = int(max(m.n for m in models))
        self.p_max = int(scen_p.max()) if ns else 0
        self.speed, self.capg, self.capc, self.capd, self.poff = speed, capg, capc, capd, poff
        self.h2d_bytes = total + recs.nbytes
        self.hosts = [None] * ns  # len() used by engine helpers

    def struct_ptr(self) -> int:
        return int(self.structs_dev.data_ptr())

    def reupload(self):
        """H2D copy of the whole batch (used by the end-to-end timing)."""
        self.dev_buf.copy_(self.host_buf, non_blocking=True)
        self.structs_dev.copy_(self.records_host, non_blocking=True)


def c4_batch(n_scen: int, seed: int = 0, device="cuda", vocab: int = 32000, batch: int = 4, seq: int = 1024,
             lo: int = 0, hi: int | None = None):
    """Config C4: n_scen independent scenarios, L ~ U{32..80}, h in
    {2048, 4096, 5120, 8192} (196 distinct models), p ~ U{8..64} workers from
    GPU_TABLE, lambda ~ U[.3, 1], alpha ~ U[0, 10 ms], bandwidth ~ LogU[.1, 10]
    Gbit/s.  Every draw is made for all n_scen scenarios (so a slice is
    identical on any rank); the batch holds scenarios [lo, hi)."""
    from .configs import C4_HIDDEN, c4_params, encoder_stages
    from .refapi import Fleet, Peer
    from .tensorize import build_host

    hi = n_scen if hi is None else hi
    P = c4_params(n_scen, seed)
    layers, hid, p, alpha, bw = P["layers"], P["hid"], P["p"], P["alpha"], P["bw"]
    kinds, lam, poff = P["kinds"], P["lam"], P["poff"]
    a, b = int(poff[lo]), int(poff[hi])
    layers, hid, p, alpha, bw = layers[lo:hi], hid[lo:hi], p[lo:hi], alpha[lo:hi], bw[lo:hi]
    kinds, lam = kinds[a:b], lam[a:b]
    beta = 8.0 / (bw * 1e9)
    keys = sorted(set(zip(layers.tolist(), hid.tolist())))
    index = {k: i for i, k in enumerate(keys)}
    dummy = Fleet(peers={"1": Peer("1")})
    models = [build_host(encoder_stages(C4_HIDDEN[h], L, vocab, batch, seq), dummy, True) for L, h in keys]
    scen_model = np.array([index[(L, h)] for L, h in zip(layers.tolist(), hid.tolist())], np.int64)
    sb = ScenarioBatch(models, scen_model, p, kinds, lam, alpha, beta, device=device)
    sb.params = dict(layers=layers, hid=hid, p=p, alpha=alpha, bw=bw, kinds=kinds, lam=lam, keys=keys, lo=lo)
    return sb


def scenario_instance(sb: ScenarioBatch, s: int):
    """Rebuild scenario s (batch-local index) as (stages, Fleet) with the reference types — the exact
    values parse_fleet would produce for the scenario's fleet document."""
    from .configs import C4_HIDDEN, encoder_stages
    from .refapi import Fleet, Link, Peer

    L, h = sb.params["keys"][int(sb.scen_model[s])]
    stages = encoder_stages(C4_HIDDEN[h], L, 32000, 4, 1024)
    a, b = int(sb.poff[s]), int(sb.poff[s + 1])
    peers = {}
    for j in range(a, b):
        k = _KINDS[int(sb.params["kinds"][j])]
        peers[str(j - a + 1)] = Peer(str(j - a + 1), peak_flops=getattr(GPU_TABLE[k], "tflops_tensor") * 1e12,
                                     lam=float(sb.params["lam"][j]), gpu_bytes=float(GPU_TABLE[k].memory_gb) * 2 ** 30,
                                     cpu_bytes=16.0 * 2 ** 30, disk_bytes=64.0 * 2 ** 30)
    fleet = Fleet(peers=peers, default_link=Link(float(sb.params["alpha"][s]), 8.0 / (float(sb.params["bw"][s]) * 1e9)))
    return stages, fleet
