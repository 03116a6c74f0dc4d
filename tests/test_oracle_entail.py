"""CPU: the entailment oracle (oracle/entailment.py) against golden vectors
produced by the REFERENCE run_rule (tests/golden/make_golden_entail.py):
stage indices, both hash tables, conclusions and report counts."""

import numpy as np
import pytest

from helpers import VocabDictionary, entail_store, load_golden_entail, table_pairs
from oracle import entailment as oe

CASES, ARR = load_golden_entail()


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c['dataset']}-r{c['rule']}-d{int(c['deduplicate'])}")
def test_oracle_matches_reference(case):
    rows = ARR[f"{case['dataset']}/rows"]
    d = VocabDictionary(case["max_id"], case["vocab"])
    idx1, t1, idx2, t2, concl, res1, res2 = oe.run_rule(case["rule"], entail_store(rows, case["chunk_triples"]), d,
                                                        deduplicate=case["deduplicate"])
    np.testing.assert_array_equal(idx1, ARR[case["idx1"]])
    np.testing.assert_array_equal(idx2, ARR[case["idx2"]])
    np.testing.assert_array_equal(table_pairs(t1, 2), ARR[case["table1"]])
    width = 1 + len(oe.RULES[case["rule"]].value_slots)
    np.testing.assert_array_equal(table_pairs(t2, width), ARR[case["table2"]])
    np.testing.assert_array_equal(np.array(sorted(concl), dtype=np.int64).reshape(-1, 3), ARR[case["conclusions"]])
    sum2 = sum(len(v) for v in t2.values())
    assert [res1, len(t1), res2, sum2, len(concl)] == case["counts"]
    assert {k: v for k, v in d.vocab.items() if k not in case["vocab"]} == case["encoded"]


def test_rule11_known_answer():
    """SPEC.md/PAPER.md Rule-11 example: conclusions {(76,84,77),(76,84,78)}"""
    case = next(c for c in CASES if c["dataset"] == "rule11" and c["rule"] == 11 and c["deduplicate"])
    assert case["counts"] == [4, 3, 2, 2, 2]
    np.testing.assert_array_equal(ARR[case["conclusions"]], [[76, 84, 77], [76, 84, 78]])
