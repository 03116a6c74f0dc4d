"""Shared test helpers: dictionary shims and plan (de)serialisation."""

from __future__ import annotations

import json
import os

import numpy as np

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


class IdDictionary:
    """Dictionary shim over a dense ID space: lexical(id) = <http://x.org/{id}>."""

    def __init__(self, max_id: int):
        self.max_id = int(max_id)

    def decode_lexical(self, ident: int) -> str:
        ident = int(ident)
        if ident <= 0 or ident > self.max_id:
            raise KeyError(ident)
        return f"<http://x.org/{ident}>"

    def lookup(self, lexical: str):
        pre = "<http://x.org/"
        if lexical.startswith(pre) and lexical.endswith(">") and lexical[len(pre):-1].isdigit():
            k = int(lexical[len(pre):-1])
            return k if 1 <= k <= self.max_id else None
        return None


RDF_TYPE = "<http://www.w3.org/1999/02/22-rdf-syntax-ns#type>"
RDFS_DOMAIN = "<http://www.w3.org/2000/01/rdf-schema#domain>"
RDFS_RANGE = "<http://www.w3.org/2000/01/rdf-schema#range>"
RDFS_SUBPROPERTY = "<http://www.w3.org/2000/01/rdf-schema#subPropertyOf>"
RDFS_SUBCLASS = "<http://www.w3.org/2000/01/rdf-schema#subClassOf>"


class VocabDictionary(IdDictionary):
    """IdDictionary plus fixed IDs for the RDF/RDFS vocabulary terms and the
    reference Dictionary's encode_lexical (assigns max_id + 1 to new terms,
    dictionary.py:68-78) — the duck type entailment.run_rule needs."""

    def __init__(self, max_id: int, vocab: dict):
        super().__init__(max_id)
        self.vocab = {k: int(v) for k, v in vocab.items()}
        self.by_id = {v: k for k, v in self.vocab.items()}

    def lookup(self, lexical: str):
        if lexical in self.vocab:
            return self.vocab[lexical]
        k = super().lookup(lexical)
        return None if k in self.by_id else k

    def decode_lexical(self, ident: int) -> str:
        return self.by_id.get(int(ident)) or super().decode_lexical(ident)

    def encode_lexical(self, lexical: str, role) -> int:
        k = self.lookup(lexical)
        if k is None:
            self.max_id += 1
            k = self.max_id
            self.vocab[lexical] = k
            self.by_id[k] = lexical
        return k


def plan_to_json(compiled) -> dict:
    """Serialise a compiled query (reference or ours) by attribute access."""

    def slot(x):
        return {"var": x.name} if hasattr(x, "name") else {"term": x.lexical}

    return {
        "distinct": bool(compiled.distinct),
        "projection": None if compiled.projection is None else list(compiled.projection),
        "output_columns": list(compiled.output_columns),
        "groups": [
            {
                "patterns": [[slot(x) for x in p.slots] for p in g.patterns],
                "filters": [[f.variable, f.regex] for f in g.filters],
                "keys": [[k.subj, k.pred, k.obj] for k in g.keys],
                "satisfiable": bool(g.satisfiable),
            }
            for g in compiled.groups
        ],
    }


def plan_from_json(d: dict):
    """Rebuild a CompiledQuery with the package's plan types."""
    from paper_1807_01409_b200 import plan
    from paper_1807_01409_b200.kernel import PatternKey

    groups = []
    for g in d["groups"]:
        pats = [plan.TriplePattern(*[plan.Var(x["var"]) if "var" in x else plan.Term(x["term"])
                                     for x in p]) for p in g["patterns"]]
        groups.append(plan.CompiledGroup(
            patterns=pats,
            filters=[plan.Filter(v, rx) for v, rx in g["filters"]],
            keys=[PatternKey(*k) for k in g["keys"]],
            var_slots=[p.var_slots() for p in pats],
            satisfiable=g["satisfiable"],
            variables=plan.Group(pats, []).variables(),
        ))
    return plan.CompiledQuery(groups, d["distinct"], d["projection"], d["output_columns"])


def load_golden():
    meta = json.load(open(os.path.join(GOLDEN_DIR, "golden.json")))
    arrays = np.load(os.path.join(GOLDEN_DIR, "golden.npz"))
    return meta, arrays


def table_rows(table) -> np.ndarray:
    """(n, ncols) uint32 rows of a BindingTable-like object in column order."""
    if not table.columns:
        return np.empty((0, 0), dtype=np.uint32)
    return np.stack([np.asarray(table.data[c], dtype=np.uint32) for c in table.columns], axis=1)


def sorted_rows(rows: np.ndarray) -> np.ndarray:
    if rows.size == 0:
        return rows
    return rows[np.lexsort(rows.T[::-1])]


def load_golden_entail():
    meta = json.load(open(os.path.join(GOLDEN_DIR, "golden_entail.json")))
    arrays = np.load(os.path.join(GOLDEN_DIR, "golden_entail.npz"))
    return meta["cases"], arrays


def entail_store(rows: np.ndarray, chunk_triples):
    """The golden case's store: one TripleChunk, or a list of chunks."""
    from paper_1807_01409_b200.store import TripleChunk

    if not chunk_triples:
        return TripleChunk(rows.reshape(-1).copy(), 0)
    flat = rows.reshape(-1)
    return [TripleChunk(flat[3 * lo:3 * min(len(rows), lo + chunk_triples)].copy(), lo)
            for lo in range(0, len(rows), chunk_triples)]


def table_pairs(table: dict, width: int) -> np.ndarray:
    out = []
    for k in sorted(table):
        for v in sorted(table[k]):
            out.append([int(k)] + (list(map(int, v)) if isinstance(v, tuple) else [int(v)]))
    return np.array(out, dtype=np.int64).reshape(-1, width)
