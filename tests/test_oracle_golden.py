"""Pin the C oracle (oracle/mdr_oracle.c) against the reference's own outputs.

The golden fixtures were produced by the real reference package
(tests/golden/make_golden.py); bit-exact means `==` on every field
(-0.0 == +0.0, as numpy compares).
"""
import numpy as np
import pytest

import golden_io as G
from oracle import oracle as O

OPS = range(6)


KEY_FIELDS = ("r1", "r2", "p1", "p2", "len1", "len2", "rev1", "rev2", "depot", "mode")


def _cm(cands):
    return np.stack([np.asarray(cands[f]).astype(np.int64) for f in G.FIELDS])


def _key(cands, i):
    """Move.key() without the op (moves.py:66-70)."""
    return [int(cands[f][i]) for f in KEY_FIELDS]


@pytest.mark.parametrize("case", G.cases("small"), ids=lambda c: c.tag)
def test_oracle_ops_small_bit_exact(case):
    oi = O.OracleInstance(case.inst, case.consts, case.nbr)
    for op in OPS:
        ref = case.op_full(op)
        got = O.enumerate_op(oi, case.sol, op)
        cands, deltas = ref
        assert np.array_equal(_cm(got), _cm(cands)), f"op {op}: candidate set/order differs"
        d = O.evaluate(oi, case.sol, op, got, case.lam)
        for f in G.DFIELDS + ("fleet_neutral",):
            assert np.array_equal(d[f], deltas[f]), f"op {op} field {f}"
        rec = case.meta["ops"][str(op)]
        best, fol = O.leader_followers(got, d, True)
        if rec["leader"] is None:
            assert best < 0
        else:
            key = _key(got, best)
            assert key == rec["leader"][1:]
            assert rec["n_followers"] == len(fol)
            fk = [_key(got, i) for i in fol[:256]]
            assert fk == [k[1:] for k in rec["followers"]]
    tot = O.totals(oi, case.sol)
    assert [x.hex() for x in tot] == case.meta["totals"]


@pytest.mark.parametrize("case", G.cases("medium"), ids=lambda c: c.tag)
def test_oracle_ops_medium_sha(case):
    oi = O.OracleInstance(case.inst, case.consts, case.nbr)
    for op in OPS:
        rec = case.meta["ops"][str(op)]
        got = O.enumerate_op(oi, case.sol, op)
        assert len(got["r1"]) == rec["n"]
        d = O.evaluate(oi, case.sol, op, got, case.lam)
        dm = np.stack([d[f] for f in G.DFIELDS])
        assert G.canon_sha(_cm(got), dm, d["fleet_neutral"].astype(np.uint8)) == rec["sha"], f"op {op}"


@pytest.mark.parametrize("case", G.cases("traj"), ids=lambda c: c.tag)
def test_oracle_local_search_trajectory(case):
    oi = O.OracleInstance(case.inst, case.consts, case.nbr)
    m = case.meta
    perms = case.S[f"{case.tag}_perms"]
    routes, lam, st, tr = O.local_search(oi, case.sol, case.lam, m["depth"], m["multi_move"], 0.5,
                                         0.01, 1e4, perms, trace_cap=m["depth"] + 1)
    assert routes == case.final_routes()
    assert [x.hex() for x in lam] == m["final_lam"]
    assert st["passes"] == m["passes"] and st["accepted"] == m["accepted"]
    assert np.array_equal(tr["op"], case.S[f"{case.tag}_tr_op"])
    assert np.array_equal(tr["n_moves"], case.S[f"{case.tag}_tr_nmoves"])
    assert np.array_equal(tr["lam"], case.S[f"{case.tag}_tr_lam"])
    feasD = case.S[f"{case.tag}_feasD"]
    assert np.array_equal(tr["D"][tr["feasible"]], feasD)
