"""Synthetic workloads of BASELINE.json's configs, in the reference's schemas.

Jobs are encoder chains laid out like pkg/src/dagmesh/pipeline.py:85-118
(tokens -> embed -> L x (attention_block, ffn_block) -> head), emitted as
reference-schema job dicts, and their stage tables are produced in closed form
here (the "tensoriser fast path for build_stages"):

* FLOPs from the catalog's MAC rules (ops.py:416-419, 483-486, 272-274):
  attention 8bsh^2 + 4bs^2h, ffn 4bshm, head 2bsh^2, embedding 0;
* memory_footprint (hardware.py:235-259): gpu = 4(params + activations),
  disk = 4 params, cpu = len(json.dumps(desc rows, sort_keys=True)) + 4 params
  — the desc rows are rebuilt with the same keys so the JSON quirk matches;
* one (src = i-1, 4bsh bytes) in-edge per stage after the first
  (build_stages :123-139, message_bytes hardware.py:157-158).

tests/test_host_cpu.py::test_closed_form_stages_match_reference_digests pins
every model used here against the reference's own parse_job_definition +
build_stages (sha256 digests in tests/golden/stage_digests.json).

Fleets are reference-schema fleet documents (hardware.py:265-354) loaded with
the reference's own parse_fleet.
"""

from __future__ import annotations

import functools
import json

import numpy as np

from .refapi import GPU_TABLE, Stage, parse_fleet

ELEMENT_BYTES = 4


# ------------------------------------------------------------------- jobs
def _block_names(layers: int, width: int = 2):
    out = []
    for i in range(1, layers + 1):
        out.append(f"l{i:0{width}d}_att")
        out.append(f"l{i:0{width}d}_ffn")
    return out


def encoder_job(hidden: int, layers: int, vocab: int, batch: int, seq: int, inner: int | None = None,
                cells: str = "block"):
    """(job dict in the reference schema, cell partition).

    cells='block': (tokens, embed), one cell per att/ffn block, (head,) -> 2L+2
    cells='layer': (tokens, embed), one (att, ffn) cell per layer, (head,) -> L+2
    """
    names = _block_names(layers)
    nodes = [{"name": "tokens", "type": "placeholder", "shape": [batch, seq], "users": ["embed"]},
             {"name": "embed", "type": "parametric", "op_class": "embedding",
              "kwargs": {"num_embeddings": vocab, "embedding_dim": hidden}, "args": ["tokens"],
              "users": [names[0]]}]
    prev = "embed"
    for j, nm in enumerate(names):
        op = "attention_block" if nm.endswith("att") else "ffn_block"
        nxt = names[j + 1] if j + 1 < len(names) else "head"
        row = {"name": nm, "type": "parametric", "op_class": op, "args": [prev], "users": [nxt]}
        if op == "ffn_block" and inner is not None:
            row["kwargs"] = {"inner_features": inner}
        nodes.append(row)
        prev = nm
    nodes.append({"name": "head", "type": "parametric", "op_class": "linear", "kwargs": {"out_features": hidden},
                  "args": [prev], "users": []})
    meta = {"batch_size": batch, "sequence_length": seq,
            "data": {"per_node": {"tokens": {"kind": "ids", "high": vocab}}}}
    if cells == "block":
        cl = [("tokens", "embed")] + [(nm,) for nm in names] + [("head",)]
    elif cells == "layer":
        cl = [("tokens", "embed")] + [(names[2 * i], names[2 * i + 1]) for i in range(layers)] + [("head",)]
    else:
        raise ValueError(cells)
    return {"meta": meta, "nodes": nodes}, cl


def encoder_stages(hidden: int, layers: int, vocab: int, batch: int, seq: int, inner: int | None = None,
                   cells: str = "block") -> list:
    """Closed-form build_stages of encoder_job(...) (memoised: Stage is a
    frozen dataclass, so the cached tuple is shared safely)."""
    return list(_encoder_stages(hidden, layers, vocab, batch, seq, inner, cells))


@functools.lru_cache(maxsize=512)
def _encoder_stages(hidden, layers, vocab, batch, seq, inner, cells) -> tuple:
    job, cl = encoder_job(hidden, layers, vocab, batch, seq, inner, cells)
    b, s, h = batch, seq, hidden
    m = inner if inner is not None else 4 * h
    bsh = b * s * h
    info = {}
    for row in job["nodes"]:
        nm, op = row["name"], row.get("op_class")
        kw = dict(row.get("kwargs") or {})
        if row["type"] == "placeholder":
            params, act, flops, shape, kind = 0, b * s, 0, [b, s], "placeholder"
        elif op == "embedding":
            params, act, flops, shape, kind = vocab * h, bsh + b * s, 0, [b, s, h], "parametric"
        elif op == "attention_block":
            params, act, flops, shape, kind = 4 * h * h, 2 * bsh, 8 * b * s * h * h + 4 * b * s * s * h, [b, s, h], "parametric"
        elif op == "ffn_block":
            params, act, flops, shape, kind = 2 * h * m, 2 * bsh, 4 * b * s * h * m, [b, s, h], "parametric"
        else:  # head: linear h -> h
            params, act, flops, shape, kind = h * h + h, 2 * bsh, 2 * b * s * h * h, [b, s, h], "parametric"
        desc = {"name": nm, "type": kind, "op_class": op, "args": list(row.get("args", [])),
                "users": list(row.get("users", [])), "kwargs": kw, "shape": shape}
        info[nm] = (params, act, flops, desc)
    stages = []
    for idx, cell in enumerate(cl):
        params = sum(info[nm][0] for nm in cell)
        act = sum(info[nm][1] for nm in cell)
        flops = float(sum(info[nm][2] for nm in cell))
        desc_bytes = len(json.dumps([info[nm][3] for nm in cell], sort_keys=True).encode("utf-8"))
        edges = () if idx == 0 else ((idx - 1, ELEMENT_BYTES * bsh),)
        label = cell[0] if len(cell) == 1 else f"{cell[0]}..{cell[-1]}"
        stages.append(Stage(idx, label, flops, ELEMENT_BYTES * (params + act),
                            desc_bytes + ELEMENT_BYTES * params, ELEMENT_BYTES * params, edges))
    return tuple(stages)


def encoder_params(graph, cells):
    """Parameters (hidden, layers, vocab, batch, seq, inner, cells) when the
    job graph and cell partition are exactly an encoder chain of the
    pipeline._encoder_model layout (pipeline.py:85-118) — node names, op
    classes, kwargs, wiring and output shapes — else None.  Those are the
    instances encoder_stages() builds in closed form."""
    try:
        names = list(graph.topo_order)
        nodes = graph.nodes
        if len(names) < 4 or names[0] != "tokens" or names[1] != "embed" or names[-1] != "head":
            return None
        tok, emb, head = nodes["tokens"], nodes["embed"], nodes["head"]
        if tok.kind.value != "placeholder" or len(tok.out_shape) != 2 or tok.users != ("embed",):
            return None
        b, s = (int(x) for x in tok.out_shape)
        if emb.op_class != "embedding" or emb.args != ("tokens",):
            return None
        vocab, h = int(emb.kwargs["num_embeddings"]), int(emb.kwargs["embedding_dim"])
        if set(emb.kwargs) != {"num_embeddings", "embedding_dim"}:
            return None
        blocks = names[2:-1]
        if len(blocks) % 2 or len(blocks) // 2 > 99:
            return None
        layers = len(blocks) // 2
        if blocks != _block_names(layers):
            return None
        inner = None
        prev = "embed"
        for j, nm in enumerate(blocks):
            nd = nodes[nm]
            nxt = blocks[j + 1] if j + 1 < len(blocks) else "head"
            want = "attention_block" if nm.endswith("att") else "ffn_block"
            if nd.op_class != want or nd.args != (prev,) or nd.users != (nxt,) or tuple(nd.out_shape) != (b, s, h):
                return None
            if want == "attention_block" and nd.kwargs:
                return None
            if want == "ffn_block":
                kw = dict(nd.kwargs)
                m = kw.pop("inner_features", None)
                if kw or (j > 1 and m != inner):
                    return None
                inner = m
            prev = nm
        if head.op_class != "linear" or head.args != (prev,) or head.users or dict(head.kwargs) != {"out_features": h}:
            return None
        cl = [tuple(c) for c in cells]
        for kind in ("block", "layer"):
            if cl == encoder_job(h, layers, vocab, b, s, inner, kind)[1]:
                return dict(hidden=h, layers=layers, vocab=vocab, batch=b, seq=s, inner=inner, cells=kind)
    except (AttributeError, KeyError, TypeError, ValueError):
        return None
    return None


def stages_for(graph, cells) -> list:
    """build_stages (scheduling.py:107-145) with the tensoriser fast path:
    encoder chains in closed form (encoder_stages), anything else through the
    reference's own builder."""
    prm = encoder_params(graph, cells)
    if prm is not None:
        return encoder_stages(**prm)
    from dagmesh import scheduling as ref_sched
    return ref_sched.build_stages(graph, cells)


# named models of BASELINE.json configs
MODELS = {
    "gpt2-small": dict(hidden=768, layers=12, vocab=50257, batch=8, seq=1024),                      # C1, n=26
    "llama2-7b-layers": dict(hidden=4096, layers=32, vocab=32000, batch=8, seq=4096, inner=16512,
                             cells="layer"),                                                          # C2, n=34
    "llama2-70b": dict(hidden=8192, layers=80, vocab=32000, batch=8, seq=4096, inner=43008),         # C3, n=162
    "opt-175b": dict(hidden=12288, layers=96, vocab=50272, batch=8, seq=2048),                       # C5, n=194
}


def model_stages(name: str) -> list:
    return encoder_stages(**MODELS[name])


# ----------------------------------------------------------------- fleets
def fleet_doc(peers, default_alpha=0.0, bandwidth_gbps=None, overrides=(), backup_pool=(), name="fleet",
              msg_ratio=1.0):
    links = {"default_alpha_s": default_alpha}
    if bandwidth_gbps is not None:
        links["bandwidth_gbps"] = bandwidth_gbps
    if overrides:
        links["overrides"] = list(overrides)
    doc = {"name": name, "peers": list(peers), "links": links, "msg_ratio": msg_ratio}
    if backup_pool:
        doc["backup_pool"] = list(backup_pool)
    return doc


def c1_fleet_doc(bandwidth_gbps: float = 1.0, alpha_s: float = 5e-3):
    """4 mixed consumer GPUs: rtx4090 .9, rtx4080 .8, rtx3080 .7 x2."""
    peers = [{"id": "1", "gpu": "rtx4090", "lambda": 0.9}, {"id": "2", "gpu": "rtx4080", "lambda": 0.8},
             {"id": "3", "gpu": "rtx3080", "lambda": 0.7}, {"id": "4", "gpu": "rtx3080", "lambda": 0.7}]
    return fleet_doc(peers, alpha_s, bandwidth_gbps, name="c1-mixed4")


def c1_link_grid(nb: int = 32, na: int = 32):
    bws = [float(x) for x in np.logspace(-1, 2, nb)]
    alphas = [float(x) for x in np.linspace(0.0, 1e-2, na)]
    return bws, alphas


def hetero_peers(p: int, seed: int, kinds=("rtx4090", "rtx4080", "rtx3080", "a100"), lam=(0.4, 1.0),
                 start_id: int = 1):
    rng = np.random.default_rng(seed)
    gi = rng.integers(0, len(kinds), p)
    lm = rng.uniform(lam[0], lam[1], p)
    return [{"id": str(start_id + i), "gpu": kinds[int(gi[i])], "lambda": float(lm[i])} for i in range(p)]


def c2_fleet_doc(seed: int = 0, alpha_s: float = 5e-3, bandwidth_gbps: float = 10.0):
    """32 heterogeneous workers, default link 5 ms / 10 Gbit/s."""
    return fleet_doc(hetero_peers(32, seed), alpha_s, bandwidth_gbps, name="c2-hetero32")


# The C2 fleet under 16 network conditions (default-link latency s, bandwidth
# Gbit/s): the base 5 ms / 10 Gbit/s first, then the rest of a what-if grid
# {5, 2, 1, 0.5} ms x {10, 1, 25, 100} Gbit/s.  The bench's step sweeps all 16
# (one scenario batch, sharded across the GPUs: 2 per GPU at N = 8).
C2_LINKS = tuple((a, bw) for a in (5e-3, 2e-3, 1e-3, 5e-4) for bw in (10.0, 1.0, 25.0, 100.0))


def c3_fleet_doc(seed: int = 0, p: int = 256):
    """256 workers (GPU_TABLE mix) with p(p-1)/2 randomised pairwise links."""
    rng = np.random.default_rng(seed + 1)
    peers = hetero_peers(p, seed, kinds=tuple(GPU_TABLE), lam=(0.4, 1.0))
    ov = []
    for a in range(1, p + 1):
        for b in range(a + 1, p + 1):
            bw = float(10 ** rng.uniform(-1, 2))
            ov.append({"src": str(a), "dst": str(b), "alpha_s": float(rng.uniform(0, 0.02)), "bandwidth_gbps": bw})
    return fleet_doc(peers, 5e-3, 10.0, overrides=ov, name="c3-rand256")


def c5_fleet_doc(seed: int = 0, p: int = 1024):
    return fleet_doc(hetero_peers(p, seed, kinds=tuple(GPU_TABLE), lam=(0.4, 1.0)), 5e-3, 10.0,
                     name="c5-1024")


def c5_churn(p: int = 1024, quit_frac: float = 0.1, seed: int = 0):
    """Scenario-file style join/quit script (sim/loop.py:77-95 schema) and the
    resulting online worker ids (the only thing the hot path consumes)."""
    rng = np.random.default_rng(seed + 7)
    quits = sorted(rng.choice(np.arange(1, p + 1), int(round(p * quit_frac)), replace=False).tolist())
    events = [{"time_s": 0.0, "action": "join", "peer_id": str(i)} for i in range(1, p + 1)]
    events += [{"time_s": 0.25 + 0.01 * k, "action": "quit", "peer_id": str(q)} for k, q in enumerate(quits)]
    online = [str(i) for i in range(1, p + 1) if i not in set(quits)]
    return events, online


def load(doc, compute_column: str = "tensor"):
    return parse_fleet(doc, compute_column)


# ------------------------------------------------------- C4 scenario sampler
C4_HIDDEN = (2048, 4096, 5120, 8192)


def c4_params(n_scen: int, seed: int = 0) -> dict:
    """Every draw of config C4, made for all n_scen scenarios in
    one fixed order so any slice is identical on any rank: L ~ U{32..80},
    h index, p ~ U{8..64}, alpha ~ U[0, 10 ms], bandwidth ~ LogU[.1, 10]
    Gbit/s, then per worker a GPU_TABLE kind and lambda ~ U[.3, 1]."""
    rng = np.random.default_rng(seed)
    layers = rng.integers(32, 81, n_scen)
    hid = rng.integers(0, len(C4_HIDDEN), n_scen)
    p = rng.integers(8, 65, n_scen)
    alpha = rng.uniform(0.0, 1e-2, n_scen)
    bw = 10.0 ** rng.uniform(-1.0, 1.0, n_scen)
    kinds = rng.integers(0, len(GPU_TABLE), int(p.sum()))
    lam = rng.uniform(0.3, 1.0, int(p.sum()))
    poff = np.concatenate([[0], np.cumsum(p)])
    return dict(layers=layers, hid=hid, p=p, alpha=alpha, bw=bw, kinds=kinds, lam=lam, poff=poff)


def c4_instance(P: dict, s: int):
    """Scenario s of c4_params as the reference's objects: closed-form stages
    (== build_stages) and the scenario's fleet document through parse_fleet."""
    L, h = int(P["layers"][s]), C4_HIDDEN[int(P["hid"][s])]
    a, b = int(P["poff"][s]), int(P["poff"][s + 1])
    kinds = tuple(GPU_TABLE)
    peers = [{"id": str(j - a + 1), "gpu": kinds[int(P["kinds"][j])], "lambda": float(P["lam"][j])}
             for j in range(a, b)]
    return (encoder_stages(h, L, 32000, 4, 1024),
            load(fleet_doc(peers, float(P["alpha"][s]), float(P["bw"][s]), name="c4")))
