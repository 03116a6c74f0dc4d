"""GPU: the reference package itself, rebound onto libtidq.

The unmodified reference (``tripleid``, installed by tools/install_reference.sh
into baseline/_ref — a git-ignored copy that travels with the repo snapshot;
the test is skipped where it is absent) converts an N-Triples dataset with
its own CLI, then ``tripleid.cli.main(["query", ...])`` and
``main(["entail", ...])`` run twice: once stock (numpy), once after
``paper_1807_01409_b200.integrate.install()``.  stdout must be byte-identical
(TSV rows in the reference's order; conclusions), and the result-count lines
of stderr equal.  Nothing here reads /root/reference."""

import contextlib
import io
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")

RDF = "<http://www.w3.org/1999/02/22-rdf-syntax-ns#type>"
RDFS = "<http://www.w3.org/2000/01/rdf-schema#{}>"


@pytest.fixture(scope="module")
def tripleid():
    if not os.path.isdir(os.path.join(REF, "tripleid")):
        pytest.skip("reference not installed under baseline/_ref (tools/install_reference.sh)")
    sys.path.insert(0, REF)
    try:
        import tripleid.cli  # noqa: F401
    finally:
        sys.path.remove(REF)
    import tripleid

    return tripleid


def _nt_dataset(path, n=60_000, seed=3):
    """Entities shared by subject and object positions (chains join), 40
    predicates, literals with language tags / datatypes, blank nodes, comment
    and blank lines, one malformed line (lenient convert skips it), and an
    RDFS schema so every entailment rule has conclusions."""
    rng = np.random.default_rng(seed)
    ent = lambda i: f"<http://ex.org/e/{i}>"  # noqa: E731
    pred = lambda i: f"<http://ex.org/p/{i}>"  # noqa: E731
    lines = ["# synthetic dataset", ""]
    s = rng.integers(0, 3000, n)
    p = np.minimum(rng.zipf(1.6, n), 40) - 1
    o = rng.integers(0, 3000, n)
    kind = rng.integers(0, 20, n)
    for k in range(n):
        if kind[k] == 0:
            obj = f'"label {o[k]}"@en'
        elif kind[k] == 1:
            obj = f'"{o[k]}"^^<http://www.w3.org/2001/XMLSchema#integer>'
        elif kind[k] == 2:
            obj = f"_:b{o[k] % 50}"
        else:
            obj = ent(o[k])
        subj = f"_:b{s[k] % 50}" if kind[k] == 3 else ent(s[k])
        lines.append(f"{subj} {pred(p[k])} {obj} .")
    lines.append("<http://ex.org/bad> not-a-term .")
    for c in range(30):
        lines.append(f"<http://ex.org/C{c}> {RDFS.format('subClassOf')} <http://ex.org/C{(c * 7 + 3) % 30}> .")
        lines.append(f"{ent(c)} {RDF} <http://ex.org/C{c % 30}> .")
    for i in range(10):
        lines.append(f"{pred(i)} {RDFS.format('domain')} <http://ex.org/C{i}> .")
        lines.append(f"{pred(i)} {RDFS.format('range')} <http://ex.org/C{i + 10}> .")
        lines.append(f"{pred(i)} {RDFS.format('subPropertyOf')} {pred((i * 3 + 1) % 12)} .")
    path.write_text("\n".join(lines) + "\n", encoding="utf-8")


QUERIES = {
    "single": "SELECT * WHERE { ?s <http://ex.org/p/0> ?o . }",
    "star3": "SELECT * WHERE { ?s <http://ex.org/p/0> ?a . ?s <http://ex.org/p/1> ?b . ?s <http://ex.org/p/2> ?c . }",
    "chain3": "SELECT * WHERE { ?x <http://ex.org/p/0> ?y . ?y <http://ex.org/p/1> ?z . ?z <http://ex.org/p/3> ?w . }",
    "filter": 'SELECT ?s ?o WHERE { ?s <http://ex.org/p/1> ?o . FILTER(regex(str(?o), "7$")) . }',
    "filter_literal": 'SELECT * WHERE { ?s ?p ?o . FILTER(regex(str(?o), "^label 1")) . }',
    "union_distinct": "SELECT DISTINCT ?s WHERE { { ?s <http://ex.org/p/4> ?o . } UNION { ?o <http://ex.org/p/5> ?s . } }",
    "union_unbound": "SELECT * WHERE { { ?a <http://ex.org/p/6> ?b . } UNION { ?c <http://ex.org/p/7> ?a . } }",
    "unknown_term": "SELECT * WHERE { ?s <http://ex.org/nope> ?o . }",
    "bound_object": "SELECT ?s WHERE { ?s ?p <http://ex.org/e/17> . }",
    "repeated": "SELECT * WHERE { ?x ?p ?x . }",
}


def _run(main, argv):
    out, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
        rc = main(argv)
    return rc, out.getvalue(), err.getvalue()


def test_reference_cli_rebound_byte_identical(gpu, tripleid, tmp_path):
    from paper_1807_01409_b200 import integrate

    main = tripleid.cli.main
    nt_path = tmp_path / "d.nt"
    _nt_dataset(nt_path)
    base = str(tmp_path / "d")
    rc, _, err = _run(main, ["convert", str(nt_path), "--out", base])
    assert rc == 0, err
    with integrate.install():  # the native converter behind the reference CLI
        rc, _, err2 = _run(main, ["convert", str(nt_path), "--out", base + "_native"])
    assert rc == 0, err2
    for s in (".tid", ".sid", ".pid", ".oid"):
        assert open(base + s, "rb").read() == open(base + "_native" + s, "rb").read(), s
    assert err.splitlines()[:6] == err2.splitlines()[:6]  # triples, distinct s/p/o, skipped, errors
    for name, text in QUERIES.items():
        q = tmp_path / f"{name}.rq"
        q.write_text("PREFIX rdfs: <http://www.w3.org/2000/01/rdf-schema#> " + text, encoding="utf-8")
        for chunk in (None, "997"):
            argv = ["query", base, str(q), "--workers", "4"] + (["--chunk-triples", chunk] if chunk else [])
            rc0, want, _ = _run(main, argv)
            with integrate.install() as inst:
                assert tripleid.query_ops.evaluate_query.__module__.startswith("paper_1807_01409_b200")
                rc1, got, _ = _run(main, argv)
            assert not inst.saved
            assert rc0 == rc1 == 0, name
            assert got == want, f"{name} chunk={chunk}: stdout differs"
            assert want.count("\n") >= 1
    for rule in (2, 3, 5, 7, 9, 11):
        argv = ["entail", base, "--rule", str(rule), "--workers", "4"]
        rc0, want, err0 = _run(main, argv)
        with integrate.install():
            rc1, got, err1 = _run(main, argv)
        assert rc0 == rc1 == 0
        assert got == want, f"rule {rule}: conclusions differ"
        assert err0.splitlines()[-1] == err1.splitlines()[-1], f"rule {rule}: res1/dist1/res2/dist2 differ"
        assert want, f"rule {rule} has no conclusions on the test dataset"
    # the stock functions are back
    assert tripleid.query_ops.evaluate_query.__module__ == "tripleid.query_ops"
