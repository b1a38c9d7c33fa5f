"""Oracle restatement of op_time / subgraph_time against the reference's own
outputs (tests/golden/opcost_cases.json)."""

import ctypes as C

import numpy as np

from golden_io import load_fleet
from opcost_util import load
from paper_2309_01172_b200 import refapi as M


def _csr(lists):
    ptr = np.zeros(len(lists) + 1, np.int32)
    flat = []
    for i, l in enumerate(lists):
        flat.extend(l)
        ptr[i + 1] = len(flat)
    return ptr, np.array(flat or [0], np.int32)


def test_oracle_op_costs_match_reference(oracle_mod):
    data = load()
    tab = data["table"]
    names = tab["names"]
    n = len(names)
    aptr, aidx = _csr(tab["args"])
    uptr, uidx = _csr(tab["users"])
    flops = np.array(tab["flops"], np.float64)
    L = oracle_mod.lib()
    L.or_op_costs.argtypes = [C.c_void_p, C.c_int] + [C.c_void_p] * 9 + [C.c_int, C.c_void_p, C.c_void_p]
    L.or_subgraph.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    checked = 0
    for fcase in data["fleets"]:
        fl = load_fleet(fcase["fleet"], M)
        inst = oracle_mod.Instance([], fl)
        mb = np.array([float(int(round(e * 4 * fl.msg_ratio))) for e in tab["out_elements"]], np.float64)
        wb = np.array([float(fl.peers[p].write_bandwidth) for p in inst.order], np.float64)
        isnp = lambda v: type(v) not in (int, float, bool)
        wnp = np.array([isnp(fl.peers[p].write_bandwidth) for p in inst.order], np.uint8)
        np_links = int(any(isnp(v) for lk in [fl.default_link, *fl.links.values()] for v in (lk.alpha, lk.beta)))
        onp = np.zeros(n, np.uint8)
        for pl, want_ops, want_sub in zip(data["placements"], fcase["ops"], fcase["subgraphs"]):
            place = np.array([inst.idx[str(pl[nm])] for nm in names], np.int32)
            out = np.zeros(3 * n)
            L.or_op_costs(C.byref(inst.t), n, flops.ctypes.data, mb.ctypes.data, aptr.ctypes.data,
                          aidx.ctypes.data, uptr.ctypes.data, uidx.ctypes.data, wb.ctypes.data,
                          place.ctypes.data, out.ctypes.data, np_links, wnp.ctypes.data, onp.ctypes.data)
            assert out.reshape(n, 3).tolist() == want_ops
            for cell, want in zip(data["cells"], want_sub):
                idx = np.array([names.index(x) for x in cell], np.int32)
                o3 = np.zeros(3)
                L.or_subgraph(len(cell), idx.ctypes.data, out.ctypes.data, onp.ctypes.data, o3.ctypes.data)
                assert o3.tolist() == want
                checked += 1
    assert checked == len(data["fleets"]) * 13 * 4 and len(data["fleets"]) == 4
