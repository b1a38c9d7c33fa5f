"""Shared helpers for the op-cost parity tests: a duck-typed graph over the
golden op table (the engine reads graphs by attribute) and the table's
`op_flops` (the golden FLOPs, produced by the reference's ir.op_flops)."""

import json
import pathlib

GOLD = pathlib.Path(__file__).resolve().parent / "golden"


def load():
    return json.loads((GOLD / "opcost_cases.json").read_text())


class _Node:
    def __init__(self, g, i):
        self.name = g.names[i]
        self.args = tuple(g.names[a] for a in g.table["args"][i])
        self.users = tuple(g.names[u] for u in g.table["users"][i])
        self.out_elements = g.table["out_elements"][i]
        self.flops = g.table["flops"][i]


class TableGraph:
    def __init__(self, table):
        self.table = table
        self.names = list(table["names"])
        self.nodes = {n: _Node(self, i) for i, n in enumerate(self.names)}

    def node(self, name):
        return self.nodes[name]


def op_flops(node):
    return node.flops
