"""GPU: entailment run_rule (paper_1807_01409_b200.entailment) — §8f row 2.
Stage indices, hash tables, conclusions, report counts and the dictionary's
encoded conclusion predicate equal the REFERENCE run_rule's golden vectors;
larger RDFS-shaped stores (resident, chunked, .tid path) equal the oracle."""

import numpy as np
import pytest

from helpers import VocabDictionary, entail_store, load_golden_entail, table_pairs
from oracle import entailment as oe
from paper_1807_01409_b200 import entailment as E
from paper_1807_01409_b200.store import DeviceStore, TripleChunk, write_tid

pytestmark = pytest.mark.gpu
CASES, ARR = load_golden_entail()


def check(run, case):
    np.testing.assert_array_equal(run.stage1_indices, ARR[case["idx1"]])
    np.testing.assert_array_equal(run.stage2_indices, ARR[case["idx2"]])
    np.testing.assert_array_equal(table_pairs(run.stage1_table, 2), ARR[case["table1"]])
    width = 1 + len(E.RULES[case["rule"]].value_slots)
    np.testing.assert_array_equal(table_pairs(run.stage2_table, width), ARR[case["table2"]])
    np.testing.assert_array_equal(np.array(sorted(run.conclusions), dtype=np.int64).reshape(-1, 3),
                                  ARR[case["conclusions"]])
    assert list(E.report_counts(run)) == case["counts"]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c['dataset']}-r{c['rule']}-d{int(c['deduplicate'])}")
def test_run_rule_matches_reference(gpu, case):
    rows = ARR[f"{case['dataset']}/rows"]
    d = VocabDictionary(case["max_id"], case["vocab"])
    run = E.run_rule(case["rule"], entail_store(rows, case["chunk_triples"]), d,
                     deduplicate=case["deduplicate"])
    check(run, case)
    assert {k: v for k, v in d.vocab.items() if k not in case["vocab"]} == case["encoded"]
    if len(rows):  # the resident store gives the same run
        d2 = VocabDictionary(case["max_id"], case["vocab"])
        check(E.run_rule(case["rule"], DeviceStore.upload(TripleChunk(rows.reshape(-1).copy(), 0)), d2,
                         deduplicate=case["deduplicate"]), case)


def _big_store(seed, n):
    rng = np.random.default_rng(seed)
    n_props, n_classes, n_ent = 300, 500, 200_000
    props = 10 + np.arange(n_props)
    classes = 10 + n_props + np.arange(n_classes)
    ents = 10 + n_props + n_classes + np.arange(n_ent)
    kind = rng.choice(6, size=n, p=[0.002, 0.002, 0.002, 0.7, 0.2, 0.094])
    s = rng.choice(ents, size=n)
    p = rng.choice(props, size=n)
    o = rng.choice(ents, size=n)
    sch = kind < 3
    s[sch] = rng.choice(props, size=int(sch.sum()))
    p[sch] = 2 + kind[sch]
    o[kind == 0] = rng.choice(classes, size=int((kind == 0).sum()))
    o[kind == 1] = rng.choice(classes, size=int((kind == 1).sum()))
    o[kind == 2] = rng.choice(props, size=int((kind == 2).sum()))
    typ = kind == 4
    p[typ] = 1
    o[typ] = rng.choice(classes, size=int(typ.sum()))
    sub = kind == 5
    s[sub] = rng.choice(classes, size=int(sub.sum()))
    p[sub] = 5
    o[sub] = rng.choice(classes, size=int(sub.sum()))
    rows = np.stack([s, p, o], axis=1).astype(np.uint32)
    vocab = {E.RDF_TYPE: 1, E.RDFS_DOMAIN: 2, E.RDFS_RANGE: 3, E.RDFS_SUBPROPERTY: 4, E.RDFS_SUBCLASS: 5}
    return rows, vocab, int(ents[-1])


@pytest.mark.parametrize("rule", sorted(E.RULES))
def test_run_rule_large_vs_oracle(gpu, tmp_path, rule):
    rows, vocab, max_id = _big_store(rule, 400_000)
    chunk = TripleChunk(rows.reshape(-1).copy(), 0)
    want = oe.run_rule(rule, chunk, VocabDictionary(max_id, vocab))
    p = tmp_path / "rdfs.tid"
    write_tid(rows, p)
    for store in (DeviceStore.upload(chunk), str(p), entail_store(rows, 99_991)):
        for dedup in (True, False):
            run = E.run_rule(rule, store, VocabDictionary(max_id, vocab), deduplicate=dedup)
            np.testing.assert_array_equal(run.stage1_indices, want[0])
            np.testing.assert_array_equal(run.stage2_indices, want[2])
            assert run.stage1_table == want[1] and run.stage2_table == want[3]
            assert run.conclusions == want[4]
            assert run.res1 == want[5]
            if dedup:
                assert run.res2 == want[6]
    w = oe.run_rule(rule, chunk, VocabDictionary(max_id, vocab), deduplicate=False)
    assert E.run_rule(rule, chunk, VocabDictionary(max_id, vocab), deduplicate=False).res2 == w[6]


def test_run_rule_errors(gpu):
    rows, vocab, max_id = _big_store(1, 1000)
    with pytest.raises(ValueError):
        E.run_rule(9, TripleChunk(rows.reshape(-1).copy(), 0), VocabDictionary(max_id, vocab), workers=0)
    # unknown stage-1 predicate: empty run, no search (and no ValueError)
    run = E.run_rule(9, TripleChunk(rows.reshape(-1).copy(), 0), VocabDictionary(max_id, {}), workers=0)
    assert run.conclusions == set() and E.report_counts(run) == (0, 0, 0, 0, 0)
