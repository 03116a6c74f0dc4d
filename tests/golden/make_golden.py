"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports ``tripleid`` from /root/reference/pkg/src and records, for seeded
inputs, the reference's own outputs of search_chunk / search_multi /
merge_join / analyze_relationships / evaluate_query (queries parsed and
compiled by the reference's own SPARQL front-end).  The fixtures
(golden.json + golden.npz) are committed; the GPU box never reads
/root/reference.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, "/root/reference/pkg/src")

from tripleid import kernel as K  # noqa: E402
from tripleid import query_ops as Q  # noqa: E402
from tripleid import sparql as SP  # noqa: E402
from tripleid.store import TripleChunk  # noqa: E402

from helpers import IdDictionary, plan_to_json  # noqa: E402
from oracle import synth as osynth  # noqa: E402
from paper_1807_01409_b200.synth import SynthDictionary, zipf_cdf_table  # noqa: E402

meta: dict = {"scan": [], "chunk": [], "merge_join": [], "query": [], "relationships": []}
arrays: dict[str, np.ndarray] = {}


def put(name: str, a: np.ndarray) -> str:
    arrays[name] = np.ascontiguousarray(a)
    return name


# ---------------------------------------------------------------- scan cases
rng = np.random.default_rng(20181807)


def random_keys(rng, rows, k):
    keys = []
    for _ in range(k):
        mask = int(rng.integers(0, 8))
        if len(rows) and rng.random() < 0.8:
            t = rows[int(rng.integers(0, len(rows)))]
        else:
            t = rng.integers(1, 40, size=3)
        keys.append(K.PatternKey(*(int(t[i]) if mask & (4 >> i) else 0 for i in range(3))))
    return keys


scan_specs = []
# SPEC Rule-11 dataset
rule11 = np.array([[76, 84, 56], [31, 84, 77], [56, 84, 78], [56, 84, 77], [44, 83, 2]], dtype=np.uint32)
scan_specs.append(("rule11", rule11, 0, [[K.PatternKey(0, 84, 0)], [K.PatternKey(44, 83, 2)],
                                         [K.PatternKey(0, 84, 0), K.PatternKey(56, 0, 0)]]))
scan_specs.append(("empty", np.empty((0, 3), np.uint32), 0, [[K.PatternKey(0, 84, 0)], [K.PatternKey()]]))
for i in range(48):
    n = int(rng.choice([1, 7, 100, 997, 4095, 4096, 4097, 9000, 20000]))
    hi = int(rng.choice([3, 10, 40, 1000]))
    rows = rng.integers(1, hi + 1, size=(n, 3), dtype=np.uint32)
    if i % 12 == 5:  # raw chunk with zero IDs (not a valid store, but the API accepts it)
        rows[rng.random(size=rows.shape) < 0.1] = 0
    base = int(rng.choice([0, 5, 1 << 33]))
    ks = [random_keys(rng, rows, int(rng.choice([1, 1, 2, 3, 5, 8, 32]))) for _ in range(3)]
    scan_specs.append((f"rand{i}", rows, base, ks))

for name, rows, base, keysets in scan_specs:
    chunk = TripleChunk(rows.reshape(-1).copy(), base)
    data_name = put(f"scan/{name}/data", rows)
    for j, keys in enumerate(keysets):
        res = K.search_multi(chunk, keys)
        meta["scan"].append({
            "name": f"{name}/{j}", "data": data_name, "base": base,
            "keys": [[k.subj, k.pred, k.obj] for k in keys],
            "indices": put(f"scan/{name}/{j}/idx", res.indices),
            "marks": put(f"scan/{name}/{j}/marks", res.values),
        })
        key = keys[0]
        rc = K.search_chunk(chunk, key)
        meta["chunk"].append({
            "name": f"{name}/{j}", "data": data_name, "base": base,
            "key": [key.subj, key.pred, key.obj],
            "indices": put(f"chunk/{name}/{j}/idx", rc.indices),
            "bits": put(f"chunk/{name}/{j}/bits", rc.values),
        })

# truth table: all 8 masks x 8 match combos via match_bits/accepts
tt = []
for mask in range(8):
    key = K.PatternKey(*(10 + i if mask & (4 >> i) else 0 for i in range(3)))
    for combo in range(8):
        triple = tuple((10 + i) if combo & (4 >> i) else (20 + i) for i in range(3))
        bits = K.match_bits(triple, key)
        tt.append([mask, combo, bits, int(K.accepts(bits, key))])
meta["truth_table"] = tt

# ---------------------------------------------------------------- merge_join
for i in range(30):
    nl = int(rng.choice([0, 1, 5, 100, 1000]))
    nr = int(rng.choice([0, 1, 7, 300, 1000]))
    hi = int(rng.choice([2, 20, 500]))
    lk = rng.integers(1, hi + 1, size=nl, dtype=np.uint32)
    rk = rng.integers(1, hi + 1, size=nr, dtype=np.uint32)
    pairs = Q.merge_join(lk, rk)
    meta["merge_join"].append({"name": f"mj{i}", "left": put(f"mj/{i}/l", lk),
                               "right": put(f"mj/{i}/r", rk), "pairs": put(f"mj/{i}/pairs", pairs)})

# ---------------------------------------------------------------- datasets
N_A, P_A, E_A, SEED_A = 20000, 50, 2000, 7
data_a = osynth.generate(N_A, seed=SEED_A, n_p=P_A, n_e=E_A, cdf=zipf_cdf_table(P_A))
meta["dataset_a"] = {"n": N_A, "n_p": P_A, "n_e": E_A, "seed": SEED_A, "data": put("data/a", data_a)}
dict_a = SynthDictionary(P_A, E_A)

N_B, MAX_B = 3000, 30
data_b = np.random.default_rng(99).integers(1, MAX_B + 1, size=(N_B, 3), dtype=np.uint32)
meta["dataset_b"] = {"n": N_B, "max_id": MAX_B, "data": put("data/b", data_b)}
dict_b = IdDictionary(MAX_B)

PRE_A = "PREFIX p: <http://example.org/p/> PREFIX e: <http://example.org/e/> "
PRE_B = "PREFIX x: <http://x.org/> "
queries_a = {
    "single_pp": "SELECT * WHERE { ?s p:3 ?o . }",
    "single_proj": "SELECT ?o WHERE { ?s p:1 ?o . }",
    "union4_distinct": "SELECT DISTINCT ?s WHERE { { ?s p:2 ?o . } UNION { ?s p:3 ?o . } UNION { ?s p:4 ?o . } UNION { ?s p:5 ?o . } }",
    "union4_bag": "SELECT ?s WHERE { { ?s p:2 ?o . } UNION { ?s p:3 ?o . } UNION { ?s p:4 ?o . } UNION { ?s p:5 ?o . } }",
    "union8_distinct_so": "SELECT DISTINCT ?s ?o WHERE { { ?s p:2 ?o . } UNION { ?s p:3 ?o . } UNION { ?s p:4 ?o . } UNION { ?s p:5 ?o . } UNION { ?s p:6 ?o . } UNION { ?s p:7 ?o . } UNION { ?s p:8 ?o . } UNION { ?s p:9 ?o . } }",
    "union_unbound": "SELECT * WHERE { { ?a p:2 ?b . } UNION { ?c p:3 ?a . } }",
    "star3": "SELECT * WHERE { ?s p:1 ?o1 . ?s p:2 ?o2 . ?s p:3 ?o3 . }",
    "star4_filter": "SELECT * WHERE { ?s p:3 ?o1 . ?s p:5 ?o2 . ?s p:7 ?o3 . ?s p:11 ?o4 . FILTER(regex(str(?o1), \"7$\")) . }",
    "chain3": "SELECT * WHERE { ?x p:1 ?y . ?y p:2 ?z . ?z p:3 ?w . }",
    "chain2_filter": "SELECT * WHERE { ?x p:3 ?y . ?y p:5 ?z . FILTER(regex(str(?y), \"7$\")) . }",
    "filter_single": "SELECT * WHERE { ?s p:1 ?o . FILTER(regex(str(?o), \"e/1\")) . }",
    "filter_two": "SELECT * WHERE { ?s p:1 ?o . FILTER(regex(str(?o), \"1\")) FILTER(regex(str(?s), \"2\")) . }",
    "filter_shared": "SELECT * WHERE { ?s p:1 ?o1 . ?s p:2 ?o2 . FILTER(regex(str(?s), \"3\")) . }",
    "repeated_var": "SELECT * WHERE { ?x ?p ?x . }",
    "pos_bound_o": "SELECT ?s WHERE { ?s p:1 e:5 . }",
    "s_bound": "SELECT * WHERE { e:17 ?p ?o . }",
    "triangle": "SELECT * WHERE { ?a p:1 ?b . ?b p:2 ?c . ?a p:3 ?c . }",
    "unsat_branch": "SELECT * WHERE { { ?s p:1 ?o . } UNION { ?s <http://nope/> ?o . } }",
    "all_free_join": "SELECT * WHERE { ?s ?p e:10 . ?s ?q ?o . }",
    "os_join": "SELECT * WHERE { ?s p:1 ?o . ?o p:1 ?o2 . }",
    "pp_join": "SELECT * WHERE { e:5 ?p ?o . e:6 ?p ?o2 . }",
    "filter_pred": "SELECT * WHERE { e:5 ?p ?o . FILTER(regex(str(?p), \"p/1\")) . }",
    "distinct_star": "SELECT DISTINCT ?s WHERE { ?s p:1 ?o1 . ?s p:2 ?o2 . }",
    "spo_exact": "SELECT * WHERE { ?s ?p ?o . FILTER(regex(str(?p), \"p/4$\")) . }",
}
rel_types = ["SS", "OO", "PP", "OP", "OS", "PS", "PO", "SP", "SO"]
queries_b = {}
for t in rel_types:
    def pat(slot_letter, var, bound_ids):
        slots = []
        for i, letter in enumerate("SPO"):
            if letter == slot_letter:
                slots.append(f"?{var}")
            else:
                slots.append(f"x:{bound_ids[i]}" if bound_ids[i] else f"?{var}_{letter.lower()}")
        return " ".join(slots)
    p1 = pat(t[0], "j", [0, 3, 0] if t[0] != "P" else [0, 0, 0])
    p2 = pat(t[1], "j", [0, 5, 0] if t[1] != "P" else [7, 0, 0])
    p2 = p2.replace("?j_", "?k_")
    queries_b[f"rel_{t}"] = f"SELECT * WHERE {{ {p1} . {p2} . }}"
queries_b["star_b"] = "SELECT * WHERE { ?s x:1 ?a . ?s x:2 ?b . ?s x:3 ?c . }"
queries_b["chain_b"] = "SELECT * WHERE { ?a x:1 ?b . ?b x:2 ?c . ?c x:3 ?d . }"
queries_b["two_shared"] = "SELECT * WHERE { ?a ?p ?b . ?a x:4 ?b . }"
queries_b["repeat_sp"] = "SELECT * WHERE { ?x ?x ?y . }"
queries_b["repeat_po"] = "SELECT * WHERE { ?y ?x ?x . }"
queries_b["repeat_all"] = "SELECT * WHERE { ?x ?x ?x . }"
queries_b["distinct_union_b"] = "SELECT DISTINCT ?a WHERE { { ?a x:1 ?b . } UNION { ?b x:2 ?a . } UNION { ?a ?p x:3 . } }"


def record_query(ds, name, text, dictionary, chunk, row_cap=None):
    ast = SP.parse_query(text)
    compiled = SP.compile_keys(ast, dictionary)
    entry = {"dataset": ds, "name": name, "text": text, "plan": plan_to_json(compiled),
             "row_cap": row_cap}
    try:
        table = Q.evaluate_query(compiled, chunk, dictionary, row_cap=row_cap)
        entry["columns"] = list(table.columns)
        entry["result"] = put(f"q/{ds}/{name}", np.stack(
            [np.asarray(table.data[c], dtype=np.uint32) for c in table.columns], axis=1)
            if table.columns else np.empty((0, 0), np.uint32))
        entry["n_rows"] = int(table.n_rows)
    except Exception as exc:  # record the reference's error class
        entry["error"] = type(exc).__name__
    meta["query"].append(entry)


chunk_a = TripleChunk(data_a.reshape(-1).copy(), 0)
chunk_b = TripleChunk(data_b.reshape(-1).copy(), 0)
for name, text in queries_a.items():
    record_query("a", name, PRE_A + text, dict_a, chunk_a)
for name, text in queries_b.items():
    record_query("b", name, PRE_B + text, dict_b, chunk_b)
record_query("a", "row_cap_hit", PRE_A + "SELECT * WHERE { ?s p:1 ?o1 . ?s p:1 ?o2 . }", dict_a, chunk_a,
             row_cap=100)
record_query("a", "row_cap_ok", PRE_A + "SELECT * WHERE { ?s p:1 ?o1 . ?s p:1 ?o2 . }", dict_a, chunk_a,
             row_cap=10_000_000)
# ResourceLimit on UNREDUCED pair counts (query_ops.py:321-324): subject 10
# has 200 x:1 and 200 x:2 triples but no x:3 triple, so the first merge_join
# of the star yields 40,000+ pairs although the group's result is small
c_rows = [[10, 1, 100 + k] for k in range(200)] + [[10, 2, 400 + k] for k in range(200)]
for s_ in range(11, 41):
    for p_ in (1, 2, 3):
        c_rows += [[s_, p_, 700 + (s_ * 7 + p_ * 3 + j) % 250] for j in range(2)]
data_c = np.array(c_rows, dtype=np.uint32)[np.random.default_rng(5).permutation(len(c_rows))]
meta["dataset_c"] = {"n": len(data_c), "max_id": 1000, "data": put("data/c", data_c)}
dict_c = IdDictionary(1000)
chunk_c = TripleChunk(data_c.reshape(-1).copy(), 0)
STAR_C = PRE_B + "SELECT * WHERE { ?s x:1 ?a . ?s x:2 ?b . ?s x:3 ?c . }"
record_query("c", "star_cap_unreduced_hit", STAR_C, dict_c, chunk_c, row_cap=30_000)
record_query("c", "star_cap_unreduced_ok", STAR_C, dict_c, chunk_c, row_cap=50_000)
record_query("c", "star_cap_none", STAR_C, dict_c, chunk_c, row_cap=None)
record_query("c", "star_cap_default", STAR_C, dict_c, chunk_c, row_cap=10_000_000)
record_query("c", "star_cap_boundary_hit", STAR_C, dict_c, chunk_c, row_cap=40_119)
record_query("c", "star_cap_boundary_ok", STAR_C, dict_c, chunk_c, row_cap=40_120)

# more than 8 output columns through a join and a DISTINCT (9 variables)
data_d = np.random.default_rng(77).integers(1, 41, size=(150, 3), dtype=np.uint32)
meta["dataset_d"] = {"n": len(data_d), "max_id": 40, "data": put("data/d", data_d)}
dict_d = IdDictionary(40)
chunk_d = TripleChunk(data_d.reshape(-1).copy(), 0)
CHAIN9 = "?a ?p1 ?b . ?b ?p2 ?c . ?c ?p3 ?d . ?d ?p4 ?e ."
record_query("d", "chain9", PRE_B + "SELECT * WHERE { " + CHAIN9 + " }", dict_d, chunk_d)
record_query("d", "chain9_distinct_union", PRE_B + "SELECT DISTINCT ?e ?p4 ?d ?p3 ?c ?p2 ?b ?p1 ?a WHERE { { "
             + CHAIN9 + " } UNION { " + CHAIN9 + " } }", dict_d, chunk_d)
record_query("d", "chain9_distinct_proj", PRE_B + "SELECT DISTINCT ?a ?b ?c ?d ?e ?p1 ?p2 ?p3 ?p4 WHERE { "
             + CHAIN9 + " }", dict_d, chunk_d)
record_query("d", "chain10_filter", PRE_B + "SELECT * WHERE { " + CHAIN9 + " ?e ?p5 ?f . FILTER(regex(str(?f), \"1\")) . }",
             dict_d, chunk_d)

# build_relation / prepare_for_join / merge_join on relations (query_ops.py:94-177)
meta["relation"] = []
for i, (qname, slot_pat) in enumerate([("r_so", "?s x:3 ?o"), ("r_sp", "?s ?p x:2"), ("r_po", "x:5 ?p ?o"),
                                        ("r_spo", "?s ?p ?o")]):
    ast = SP.parse_query(PRE_B + f"SELECT * WHERE {{ {slot_pat} . }}")
    pat = ast.groups[0].patterns[0]
    cq = SP.compile_keys(ast, dict_b)
    res = K.search_multi(chunk_b, cq.groups[0].keys)
    rows = data_b[res.indices]
    for join_slot in "SPO":
        entry = {"name": f"{qname}/{join_slot}", "pattern": plan_to_json(cq)["groups"][0]["patterns"][0],
                 "rows": put(f"rel/{qname}/rows", rows), "join_slot": join_slot}
        try:
            rel = Q.build_relation(rows, pat, join_slot)
            entry["key"] = put(f"rel/{qname}/{join_slot}/key", rel.key)
            entry["values"] = {k: put(f"rel/{qname}/{join_slot}/v{k}", v) for k, v in rel.values.items()}
            prep = rel.prepare_for_join()
            entry["sorted_key"] = put(f"rel/{qname}/{join_slot}/skey", prep.key)
            entry["sorted_values"] = {k: put(f"rel/{qname}/{join_slot}/sv{k}", v) for k, v in prep.values.items()}
            if len(rows) <= 1000:
                entry["self_pairs"] = put(f"rel/{qname}/{join_slot}/pairs", Q.merge_join(rel, prep))
        except Exception as exc:
            entry["error"] = type(exc).__name__
        meta["relation"].append(entry)

# evaluate_group (query_ops.py:345-356) on AST groups, compiled by the reference
meta["group"] = []
for gname, text, cap in [("star", "SELECT * WHERE { ?s x:1 ?a . ?s x:2 ?b . }", None),
                         ("filter_chain", "SELECT * WHERE { ?a x:1 ?b . ?b x:2 ?c . FILTER(regex(str(?c), \"1\")) . }", None),
                         ("capped", "SELECT * WHERE { ?s x:1 ?a . ?s x:2 ?b . }", 10),
                         ("unsat", "SELECT * WHERE { ?s <http://nope/> ?a . }", None)]:
    ast = SP.parse_query(PRE_B + text)
    cq = SP.compile_keys(ast, dict_b)
    entry = {"name": gname, "text": PRE_B + text, "plan": plan_to_json(cq), "row_cap": cap}
    try:
        t = Q.evaluate_group(ast.groups[0], chunk_b, dict_b, row_cap=cap)
        entry["columns"] = list(t.columns)
        entry["result"] = put(f"group/{gname}", np.stack([t.data[c] for c in t.columns], axis=1)
                              if t.columns else np.empty((0, 0), np.uint32))
    except Exception as exc:
        entry["error"] = type(exc).__name__
    meta["group"].append(entry)

# BASELINE configs[0] (C1): the 1M-triple synthetic store (seed 1,
# n_p 10^4, n_e 10^5) and the single pattern ?s P_10 ?o, run by the
# reference's own evaluate_query; plus the C2-C5 query shapes at C1 size
# (UNION x4/x8 bag and DISTINCT, star/chain x2-x4 with FILTER) as bit-exact
# anchors for every operator.  The store is NOT committed: the tests
# regenerate it (numpy twin on CPU, the device generator on the GPU).
C1 = dict(n=1_000_000, n_p=10_000, n_e=100_000, seed=1)
data_c1 = osynth.generate(C1["n"], seed=C1["seed"], n_p=C1["n_p"], n_e=C1["n_e"], cdf=zipf_cdf_table(C1["n_p"]))
meta["dataset_C1"] = dict(C1, generated=True,
                          rows_sha256=__import__("hashlib").sha256(data_c1.tobytes()).hexdigest())
dict_c1 = SynthDictionary(C1["n_p"], C1["n_e"])
chunk_c1 = TripleChunk(data_c1.reshape(-1).copy(), 0)


def _u(ranks, proj="*", distinct=False):
    body = " UNION ".join(f"{{ ?s p:{r} ?o . }}" for r in ranks)
    return f"SELECT {'DISTINCT ' if distinct else ''}{proj} WHERE {{ {body} }}"


def _star(ranks, flt=False):
    pats = " ".join(f"?s p:{r} ?o{i + 1} ." for i, r in enumerate(ranks))
    return "SELECT * WHERE { " + pats + (' FILTER(regex(str(?o1), "7$")) .' if flt else "") + " }"


def _chain(ranks, flt=False):
    v = ["x", "y", "z", "w", "v"]
    pats = " ".join(f"?{v[i]} p:{r} ?{v[i + 1]} ." for i, r in enumerate(ranks))
    return "SELECT * WHERE { " + pats + (' FILTER(regex(str(?y), "7$")) .' if flt else "") + " }"


queries_c1 = {"c1_scan_p10": "SELECT * WHERE { ?s p:10 ?o . }",
              "c1_scan_p1": "SELECT * WHERE { ?s p:1 ?o . }",
              "c1_scan_p1000_o": "SELECT ?o WHERE { ?s p:1000 ?o . }",
              "c1_union4_bag": _u(range(2, 6)), "c1_union8_bag": _u(range(2, 10)),
              "c1_union4_distinct_s": _u(range(2, 6), "?s", True),
              "c1_union8_distinct_s": _u(range(2, 10), "?s", True),
              "c1_union8_distinct_so": _u(range(2, 10), "?s ?o", True)}
for k in (2, 3, 4):
    rk = [3, 5, 7, 11][:k]
    queries_c1[f"c1_star{k}"] = _star(rk)
    queries_c1[f"c1_star{k}_filter"] = _star(rk, True)
    queries_c1[f"c1_chain{k}"] = _chain(rk)
    queries_c1[f"c1_chain{k}_filter"] = _chain(rk, True)
queries_c1["c1_star3_c5ranks"] = _star([5, 7, 11])
queries_c1["c1_chain3_c5ranks"] = _chain([5, 7, 11])
n_query_before_c1 = len(meta["query"])
for name, text in queries_c1.items():
    record_query("C1", name, PRE_A + text, dict_c1, chunk_c1, row_cap=10_000_000)
meta["c1"] = meta["query"][n_query_before_c1:]
del meta["query"][n_query_before_c1:]

record_query("a", "disconnected",PRE_A + "SELECT * WHERE { ?s p:1 ?o1 . ?x p:2 ?y . }", dict_a, chunk_a)

for name, text in list(queries_a.items())[:10]:
    ast = SP.parse_query(PRE_A + text)
    for gi, g in enumerate(ast.groups):
        if len(g.patterns) >= 2:
            rels = Q.analyze_relationships(g.patterns)
            meta["relationships"].append({"query": name, "group": gi,
                                          "rels": [[r.i, r.j, r.rel_type, r.variable] for r in rels]})

json.dump(meta, open(os.path.join(HERE, "golden.json"), "w"), indent=0)
np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
print(f"wrote {len(meta['scan'])} scan, {len(meta['chunk'])} chunk, {len(meta['merge_join'])} merge_join, "
      f"{len(meta['query'])} query cases; {sum(a.nbytes for a in arrays.values()) / 1e6:.2f} MB raw")
