"""Golden vectors for the entailment two-stage rules, produced by running the
REFERENCE ``tripleid.entailment.run_rule`` (entailment.py:175-255) itself.

    python tests/golden/make_golden_entail.py      # build container only

Writes golden_entail.json + golden_entail.npz (committed).  Datasets: the
SPEC Rule-11 example and seeded random
RDFS-shaped stores (schema triples over property/class IDs, instance, type
and subclass triples); every rule in {2, 3, 5, 7, 9, 11} with
deduplicate in {True, False}, whole-chunk and chunked stores.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, "/root/reference/pkg/src")

from tripleid import entailment as E  # noqa: E402
from tripleid.store import TripleChunk  # noqa: E402

from helpers import (RDF_TYPE, RDFS_DOMAIN, RDFS_RANGE, RDFS_SUBCLASS,  # noqa: E402
                     RDFS_SUBPROPERTY, VocabDictionary)

meta: dict = {"cases": []}
arrays: dict[str, np.ndarray] = {}


def put(name, a):
    arrays[name] = np.ascontiguousarray(a)
    return name


def pairs(table: dict, width: int) -> np.ndarray:
    out = []
    for k in sorted(table):
        for v in sorted(table[k]):
            out.append([int(k)] + (list(map(int, v)) if isinstance(v, tuple) else [int(v)]))
    return np.array(out, dtype=np.int64).reshape(-1, width)


def record(name, rows, vocab, max_id, chunk_triples=None):
    put(f"{name}/rows", rows)
    for rule in sorted(E.RULES):
        for dedup in (True, False):
            d = VocabDictionary(max_id, vocab)
            if chunk_triples:
                flat = rows.reshape(-1)
                store = [TripleChunk(flat[3 * lo:3 * min(len(rows), lo + chunk_triples)].copy(), lo)
                         for lo in range(0, len(rows), chunk_triples)]
            else:
                store = TripleChunk(rows.reshape(-1).copy(), 0)
            run = E.run_rule(rule, store, d, workers=1, deduplicate=dedup)
            key = f"{name}/r{rule}/{int(dedup)}"
            meta["cases"].append({
                "dataset": name, "rule": rule, "deduplicate": dedup, "chunk_triples": chunk_triples,
                "max_id": max_id, "vocab": vocab,
                "idx1": put(key + "/idx1", run.stage1_indices),
                "idx2": put(key + "/idx2", run.stage2_indices),
                "table1": put(key + "/table1", pairs(run.stage1_table, 2)),
                "table2": put(key + "/table2", pairs(run.stage2_table, 1 + len(E.RULES[rule].value_slots))),
                "conclusions": put(key + "/conclusions", np.array(sorted(run.conclusions), dtype=np.int64).reshape(-1, 3)),
                "counts": list(map(int, E.report_counts(run))),
                "encoded": {k: v for k, v in d.vocab.items() if k not in vocab},
            })


# SPEC Rule-11 example: 84 = rdfs:subClassOf, 83 another predicate
rule11 = np.array([[76, 84, 56], [31, 84, 77], [56, 84, 78], [56, 84, 77], [44, 83, 2]], dtype=np.uint32)
record("rule11", rule11, {RDFS_SUBCLASS: 84}, 100)

rng = np.random.default_rng(1807)
VOCAB = {RDF_TYPE: 1, RDFS_DOMAIN: 2, RDFS_RANGE: 3, RDFS_SUBPROPERTY: 4, RDFS_SUBCLASS: 5}


def rdfs_store(rng, n, n_props, n_classes, n_ent, vocab_present=True):
    props = 10 + np.arange(n_props)
    classes = 10 + n_props + np.arange(n_classes)
    ents = 10 + n_props + n_classes + np.arange(n_ent)
    kinds = rng.choice(6, size=n, p=[0.05, 0.05, 0.05, 0.55, 0.2, 0.1])
    rows = np.empty((n, 3), dtype=np.uint32)
    for i, k in enumerate(kinds):
        if k == 0:  # p domain C
            rows[i] = (rng.choice(props), 2, rng.choice(classes))
        elif k == 1:  # p range C
            rows[i] = (rng.choice(props), 3, rng.choice(classes))
        elif k == 2:  # p subPropertyOf q
            rows[i] = (rng.choice(props), 4, rng.choice(props))
        elif k == 3:  # instance s p o
            rows[i] = (rng.choice(ents), rng.choice(props), rng.choice(ents))
        elif k == 4:  # s type C
            rows[i] = (rng.choice(ents), 1, rng.choice(classes))
        else:  # C subClassOf D
            rows[i] = (rng.choice(classes), 5, rng.choice(classes))
    max_id = int(10 + n_props + n_classes + n_ent)
    vocab = dict(VOCAB)
    if not vocab_present:  # rdf:type unknown: R2/R3/R9 stage 1 or the conclusion predicate
        del vocab[RDF_TYPE]
        rows = rows[rows[:, 1] != 1]
    return rows, vocab, max_id


for i, (n, np_, nc, ne) in enumerate([(40, 3, 3, 10), (500, 6, 8, 50), (3000, 12, 20, 300),
                                      (20000, 25, 40, 2000)]):
    rows, vocab, max_id = rdfs_store(rng, n, np_, nc, ne)
    record(f"rdfs{i}", rows, vocab, max_id, chunk_triples=None)
rows, vocab, max_id = rdfs_store(rng, 5000, 10, 12, 400)
record("rdfs_chunked", rows, vocab, max_id, chunk_triples=777)
rows, vocab, max_id = rdfs_store(rng, 3000, 8, 10, 200, vocab_present=False)
record("rdfs_no_type", rows, vocab, max_id)
record("empty", np.empty((0, 3), np.uint32), dict(VOCAB), 50)

json.dump(meta, open(os.path.join(HERE, "golden_entail.json"), "w"), indent=0)
np.savez_compressed(os.path.join(HERE, "golden_entail.npz"), **arrays)
print(f"{len(meta['cases'])} entailment cases")
