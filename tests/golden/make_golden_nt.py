"""Record the REFERENCE's N-Triples conversion of tests/nt_cases.py inputs.

Run in the build container (imports tripleid from /root/reference/pkg/src):

    python tests/golden/make_golden_nt.py

For each case: the reference's cmd_convert (cli.py:64-114) in lenient mode —
SHA-256 and size of the four output files, its stderr counts — the lenient
ParseReport errors (line, byte offset, message) from nt.parse_stream, and the
strict-mode outcome (the first ParseError's text, or ok)."""

from __future__ import annotations

import contextlib
import hashlib
import io
import json
import os
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, "/root/reference/pkg/src")

from tripleid import cli, nt  # noqa: E402

from nt_cases import CASES  # noqa: E402

SUFFIXES = (".tid", ".sid", ".pid", ".oid")


def main():
    out = {}
    with tempfile.TemporaryDirectory() as td:
        for name, make in CASES.items():
            src = os.path.join(td, name + ".nt")
            with open(src, "wb") as f:
                f.write(make())
            base = os.path.join(td, name)
            err = io.StringIO()
            with contextlib.redirect_stderr(err):
                rc = cli.main(["convert", src, "--out", base])
            assert rc == 0, err.getvalue()
            files = {}
            for s in SUFFIXES:
                b = open(base + s, "rb").read()
                files[s] = {"sha256": hashlib.sha256(b).hexdigest(), "bytes": len(b)}
            counts = dict(line.split("\t", 1) for line in err.getvalue().splitlines()
                          if line.split("\t")[0] in ("triples", "distinct_subjects", "distinct_predicates",
                                                     "distinct_objects", "skipped_lines", "parse_errors"))
            rep = nt.ParseReport()
            with open(src, "rb") as f:
                for _ in nt.parse_stream(f, report=rep):
                    pass
            errors = [[e.line_number, e.offset, e.message] for e in rep.errors]
            err2 = io.StringIO()
            with contextlib.redirect_stderr(err2):
                rc2 = cli.main(["convert", src, "--out", base + "_strict", "--strict"])
            strict = "ok" if rc2 == 0 else err2.getvalue().strip()
            out[name] = {"files": files, "counts": {k: int(v) for k, v in counts.items()},
                         "errors": errors, "strict_rc": rc2, "strict": strict}
    json.dump(out, open(os.path.join(HERE, "golden_nt.json"), "w"), indent=1)
    print({k: (v["counts"]["triples"], len(v["errors"]), v["strict_rc"]) for k, v in out.items()})


if __name__ == "__main__":
    main()
