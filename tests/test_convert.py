"""Native N-Triples -> TripleID conversion against the
reference's own cmd_convert outputs (tests/golden/golden_nt.json, recorded by
tests/golden/make_golden_nt.py): byte-identical .tid/.sid/.pid/.oid files,
the same counts, the same lenient error list (line, byte, message) and the
same strict-mode error, for 1 and many host threads.  Host-only code: runs
on CPU."""

import contextlib
import hashlib
import io
import json
import os
from types import SimpleNamespace

import pytest

from nt_cases import CASES
from paper_1807_01409_b200 import convert
from paper_1807_01409_b200.errors import ParseError

GOLD = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_nt.json")))


@pytest.mark.parametrize("threads", [1, 0, 7])
@pytest.mark.parametrize("name", sorted(CASES))
def test_convert_matches_reference(tmp_path, name, threads):
    want = GOLD[name]
    src = tmp_path / "in.nt"
    src.write_bytes(CASES[name]())
    base = tmp_path / "out"
    res = convert.convert_nt(src, base, threads=threads)
    for suffix, f in want["files"].items():
        b = (tmp_path / ("out" + suffix)).read_bytes()
        assert len(b) == f["bytes"] and hashlib.sha256(b).hexdigest() == f["sha256"], (name, suffix)
    c = want["counts"]
    assert res.triples == c["triples"]
    assert res.distinct == (c["distinct_subjects"], c["distinct_predicates"], c["distinct_objects"])
    assert res.skipped == c["skipped_lines"] and res.error_count == c["parse_errors"]
    assert [[e.line_number, e.offset, e.message] for e in res.errors] == want["errors"]
    assert not list(tmp_path.glob("*.tmp*"))
    if want["strict_rc"] == 0:
        convert.convert_nt(src, tmp_path / "strict", strict=True, threads=threads)
    else:
        with pytest.raises(ParseError) as ei:
            convert.convert_nt(src, tmp_path / "strict", strict=True, threads=threads)
        assert want["strict"] == f"parse error: {ei.value}"
        assert not list(tmp_path.glob("strict*"))


def test_cmd_convert_diagnostics_and_exit_codes(tmp_path):
    src = tmp_path / "in.nt"
    src.write_bytes(CASES["rand_crlf_errors"]())
    err = io.StringIO()
    with contextlib.redirect_stderr(err):
        rc = convert.cmd_convert(SimpleNamespace(input=str(src), out=str(tmp_path / "d"), strict=False))
    assert rc == 0
    lines = dict(x.split("\t", 1) for x in err.getvalue().splitlines() if x.count("\t") == 1)
    c = GOLD["rand_crlf_errors"]["counts"]
    for k, v in c.items():
        assert int(lines[k]) == v
    assert "bytes\td.tid\t" + str(GOLD["rand_crlf_errors"]["files"][".tid"]["bytes"]) in err.getvalue()
    err = io.StringIO()
    with contextlib.redirect_stderr(err):
        rc = convert.cmd_convert(SimpleNamespace(input=str(src), out=str(tmp_path / "s"), strict=True))
    assert rc == convert.EXIT_PARSE and err.getvalue().strip() == GOLD["rand_crlf_errors"]["strict"]
    err = io.StringIO()
    with contextlib.redirect_stderr(err):
        rc = convert.cmd_convert(SimpleNamespace(input=str(tmp_path / "missing.nt"), out=str(tmp_path / "m"),
                                                 strict=False))
    assert rc == convert.EXIT_IO
    assert err.getvalue().startswith("I/O error: [Errno 2] No such file or directory:")
    err = io.StringIO()
    with contextlib.redirect_stderr(err):
        rc = convert.cmd_convert(SimpleNamespace(input=str(src), out=str(tmp_path / "nodir" / "x"), strict=False))
    assert rc == convert.EXIT_IO and "I/O error: [Errno 2]" in err.getvalue()
    assert not list(tmp_path.glob("nodir*"))


REF = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference sources not present (build container only)")
def test_convert_live_reference_random(tmp_path):
    """Build container: a fresh random input converted by the reference and
    natively; the four files are byte-identical."""
    import sys

    sys.path.insert(0, REF)
    try:
        from tripleid import cli
    finally:
        sys.path.remove(REF)
    from nt_cases import random_file

    src = tmp_path / "r.nt"
    src.write_bytes(random_file(50_000, 99, crlf=True, errors_every=501))
    with contextlib.redirect_stderr(io.StringIO()):
        assert cli.main(["convert", str(src), "--out", str(tmp_path / "ref")]) == 0
    convert.convert_nt(src, tmp_path / "ours", threads=5)
    for s in (".tid", ".sid", ".pid", ".oid"):
        assert (tmp_path / ("ref" + s)).read_bytes() == (tmp_path / ("ours" + s)).read_bytes(), s
