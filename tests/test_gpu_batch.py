"""Config C4 (batched schedule() over independent scenarios): the vectorised
scenario batch (batch.py) + prop/hill + epilogue kernels against the oracle
run scenario by scenario on instances rebuilt from the same draws."""

import numpy as np
import pytest

from paper_2309_01172_b200 import batch as B
from paper_2309_01172_b200 import engine

pytestmark = pytest.mark.gpu


def test_c4_batch_matches_oracle(oracle_mod, engine_ready):
    sb = B.c4_batch(3000, seed=1)
    owner, score, moves = engine.prop_hill(sb, sb.n_max)
    epi = engine.epilogue(sb, sb.n_max, owner, 512, 4).cpu().numpy()
    owner = owner.cpu().numpy()
    rng = np.random.default_rng(0)
    for s in rng.choice(3000, 40, replace=False):
        st, fl = B.scenario_instance(sb, int(s))
        inst = oracle_mod.Instance(st, fl)
        path, own = inst.schedule()
        assert owner[s, :len(st)].tolist() == own.tolist(), s
        runs = inst.owner_to_runs(own)
        mk, code, _, _, comp, read = inst.eval_runs(runs)
        assert epi[s, 0] == mk and int(epi[s, 5]) == code
        assert tuple(epi[s, 1:5]) == oracle_mod.epilogue(comp, read, 512, 4)


def test_c4_hill_moves_match_oracle(oracle_mod, engine_ready):
    """Scenarios whose hill climb accepts moves (one or several, across
    rounds): the warp-parallel move scoring takes the same first improving
    move in the reference's order every time."""
    sb = B.c4_batch(6000, seed=3)
    owner, score, moves = engine.prop_hill(sb, sb.n_max)
    owner, moves = owner.cpu().numpy(), moves.cpu().numpy()
    picked = list(np.flatnonzero(moves >= 3)[:20]) + list(np.flatnonzero(moves == 1)[:20]) + \
        list(np.flatnonzero(moves == 2)[:10])
    assert len(picked) >= 30 and moves.max() >= 3
    for s in picked:
        st, fl = B.scenario_instance(sb, int(s))
        _, own = oracle_mod.Instance(st, fl).schedule()
        assert owner[s, :len(st)].tolist() == own.tolist(), (s, int(moves[s]))
