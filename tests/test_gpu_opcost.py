"""GPU op_time / subgraph_time (dm_op_costs, dm_subgraph_times) against the
reference's own outputs (tests/golden/opcost_cases.json, produced by
hardware.op_time / subgraph_time on the demo job, hardware.py:190-226)."""

import pytest

from golden_io import load_fleet
from opcost_util import TableGraph, load
from paper_2309_01172_b200 import refapi as M
from paper_2309_01172_b200 import opcost as O

pytestmark = pytest.mark.gpu


def test_op_costs_and_subgraphs_bitwise(engine_ready):
    data = load()
    g = TableGraph(data["table"])
    table = O.op_table_from_graph(g)
    for fcase in data["fleets"]:
        fl = load_fleet(fcase["fleet"], M)
        got = O.op_costs(table, fl, data["placements"])
        assert got.tolist() == fcase["ops"]
        sub = O.subgraph_costs(table, fl, data["placements"], data["cells"])
        assert sub.tolist() == fcase["subgraphs"]


def test_op_time_api(engine_ready):
    data = load()
    g = TableGraph(data["table"])
    fl = load_fleet(data["fleets"][0]["fleet"], M)
    pl = data["placements"][0]
    for i, name in enumerate(g.names):
        c = O.op_time(g, name, fl, pl)
        assert list(c) == data["fleets"][0]["ops"][0][i]
        assert c.total_s == c.read_s + c.compute_s + c.write_s
    t = O.subgraph_time(g, ("TensorA", "Multiply"), fl, pl)
    assert list(t) == data["fleets"][0]["subgraphs"][0][0]
    assert O.subgraph_time(g, (), fl, {}) == (0.0, 0.0, 0.0)
    with pytest.raises(M.FleetError):
        O.op_time(g, "Conv", fl, dict(pl, Conv="99"))
