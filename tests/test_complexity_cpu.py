"""Table I complexity model (dbp_complexity, P566-595) against SPEC's worked
values and hand-evaluated cells (tests/golden/table1_examples.json), plus the
model's structural invariants.  Host-only: runs without a GPU."""
import json
import os

import pytest

from paper_1702_04458_b200 import dbp

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "table1_examples.json")))


@pytest.mark.parametrize("case", GOLD["cases"], ids=lambda c: f"{c['algo']}-{c['mode']}-{c['metric']}-{c['field']}")
def test_table1_golden(case):
    got = dbp.complexity(case["algo"], case["mode"], case["metric"], case["U"], case["S"], case["C"], case["T"])
    assert got[case["field"]] == case["value"], case["cite"]


@pytest.mark.parametrize("algo,mode", [("admm_dl", "SxS"), ("admm_dl", "UxU"), ("admm_ul", "SxS"),
                                       ("admm_ul", "UxU"), ("cg_ul", None)])
def test_table1_invariants(algo, mode):
    for U, S, C in [(4, 16, 2), (16, 32, 32), (32, 32, 128), (5, 7, 3)]:
        tm = [dbp.complexity(algo, mode, "TM", U, S, C, T) for T in (1, 2, 5)]
        ar = [dbp.complexity(algo, mode, "AR", U, S, C, T) for T in (1, 2, 5)]
        for rep in tm + ar:
            assert min(rep.values()) >= 0
        for T, rep in zip((1, 2, 5), tm):
            assert rep["total"] == rep["pre"] + rep["first"] + (T - 1) * rep["next"]
        # AR counts every cluster's PE: never below the single-PE timing count, and equal to it at C = 1
        for a, t in zip(ar, tm):
            assert a["pre"] >= t["pre"] and a["total"] >= t["total"] - 4 * U * 5
        one_t = dbp.complexity(algo, mode, "TM", U, S, 1, 3)
        one_a = dbp.complexity(algo, mode, "AR", U, S, 1, 3)
        assert one_a["pre"] == one_t["pre"]
        # preprocessing AR scales linearly in C (all decentralized rows)
        assert dbp.complexity(algo, mode, "AR", U, S, 2 * C, 1)["pre"] - 2 * ar[0]["pre"] in (0, -2 * U)


def test_modes_coincide_at_s_equals_u():
    for U in (4, 16, 32):
        for algo in ("admm_dl", "admm_ul"):
            a = dbp.complexity(algo, "SxS", "TM", U, U, 4, 5)
            b = dbp.complexity(algo, "UxU", "TM", U, U, 4, 5)
            assert a["pre"] == b["pre"]        # Table I: the two modes' preprocessing agree at S = U


def test_centralized_cubic_in_u():
    a = dbp.complexity("mmse_ul", None, "TM", 8, 32, 32, 1)["total"]
    b = dbp.complexity("mmse_ul", None, "TM", 16, 32, 32, 1)["total"]
    assert 3.5 < b / a < 8.5                  # 6CSU^2 dominates: ~4x per doubling of U


def test_invalid_arguments():
    for bad in [("admm_ul", "UxU", "TM", 0, 4, 4, 1), ("admm_ul", "UxU", "TM", 4, 4, 4, 0)]:
        with pytest.raises(dbp.DbpError):
            dbp.complexity(*bad)
