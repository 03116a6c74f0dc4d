"""Deterministic N-Triples inputs for the converter parity tests (the
reference's cmd_convert outputs for them are recorded by
tests/golden/make_golden_nt.py).  Covers nt.py's grammar and every error
branch, Python's strict UTF-8 decoder errors, CRLF, N-Quads contexts,
language tags with non-ASCII letters, and files large enough to be split
over many host threads."""

from __future__ import annotations

import numpy as np

EDGE_LINES = [
    b'<http://a/s> <http://a/p> <http://a/o> .',
    b'<http://a/s> <http://a/p> "plain" .',
    b'  \t<http://a/s>\t<http://a/p>   "tabs and spaces"   .   ',
    b'<http://a/s> <http://a/p> "esc \\" quote \\\\ back" .',
    b'<http://a/s> <http://a/p> "lang"@en-GB .',
    b'<http://a/s> <http://a/p> "unicode lang"@\xe6\x97\xa5\xe6\x9c\xac .',  # @日本 (isalnum)
    b'<http://a/s> <http://a/p> "typed"^^<http://www.w3.org/2001/XMLSchema#string> .',
    b'<http://a/s> <http://a/p> "caf\xc3\xa9 \xf0\x9f\x98\x80" .',
    b'_:b1 <http://a/p> _:b2.',
    b'_:b1 <http://a/p> _:b2 <http://graph/g1> .',
    b'<http://a/s> <http://a/p> <http://a/o> _:ctx .',
    b'<http://a/s> <http://a/p> <http://a/o> . # trailing comment',
    b'# a comment line',
    b'',
    b'   ',
    b'<http://a/s> <http://a/p> <http://a/o> .\r',
    b'<http://a/s2> <http://a/p> "x\\\xc3\xa9y" .',  # backslash before a 2-byte char
    # ---- malformed (lenient: skipped and reported) ----
    b'<http://a/s <http://a/p> <http://a/o> .',
    b'<http://a/s> <http://a/p> "unterminated .',
    b'<http://a/s> <http://a/p> "x"^^<http://unterminated .',
    b'<http://a/s> <http://a/p> "x"@ .',
    b'_x <http://a/p> <http://a/o> .',
    b'_: <http://a/p> <http://a/o> .',
    b'abc <http://a/p> <http://a/o> .',
    b"'q' <http://a/p> <http://a/o> .",
    b'\\ <http://a/p> <http://a/o> .',
    b'\x01 <http://a/p> <http://a/o> .',
    b'\xe2\x80\x8b <http://a/p> <http://a/o> .',  # U+200B (not printable)
    b'\xc3\xa9 <http://a/p> <http://a/o> .',
    b'<http://a/s> <http://a/p> <http://a/o>',
    b'<http://a/s> <http://a/p> <http://a/o> <http://c> <http://d> .',
    b'<http://a/s> <http://a/p> <http://a/o> . junk',
    b'<http://a/s> <http://a/p> .',
    b'<http://a/s> "lit" <http://a/o> .',
    b'"lit" <http://a/p> <http://a/o> .',
    b'<http://a/s> <http://a/p> <http://a/o> "ctx" .',
    b'<http://a/s> <http://a/p> "\xff" .',
    b'<http://a/s> <http://a/p> "\xc3\x28" .',
    b'<http://a/s> <http://a/p> "\xe0\x80\x80" .',
    b'<http://a/s> <http://a/p> "\xed\xa0\x80" .',
    b'<http://a/s> <http://a/p> "\xf4\x90\x80\x80" .',
    b'<http://a/s> <http://a/p> "\xf0\x9f\x98',  # truncated at end of line
    b'<http://a/s> <http://a/p> "\xe2\x82',
    b'\t.',
    b'.',
]


def edge_file() -> bytes:
    return b"\n".join(EDGE_LINES) + b"\n"


def random_file(n: int, seed: int, crlf: bool = False, errors_every: int = 0) -> bytes:
    """n statements over shared entity/predicate pools with literals, blank
    nodes, language tags and contexts; optionally CRLF and malformed lines."""
    rng = np.random.default_rng(seed)
    s = rng.integers(0, max(2, n // 5), n)
    p = np.minimum(rng.zipf(1.5, n), 200)
    o = rng.integers(0, max(2, n // 3), n)
    kind = rng.integers(0, 16, n)
    eol = b"\r\n" if crlf else b"\n"
    out = []
    for k in range(n):
        subj = b"_:n%d" % (s[k] % 97) if kind[k] == 1 else b"<http://e.org/r/%d>" % s[k]
        if kind[k] == 2:
            obj = b'"label %d"@en' % o[k]
        elif kind[k] == 3:
            obj = b'"%d"^^<http://www.w3.org/2001/XMLSchema#integer>' % o[k]
        elif kind[k] == 4:
            obj = '"café %d"@fr-CA'.encode() % o[k]
        else:
            obj = b"<http://e.org/r/%d>" % o[k]
        line = subj + b" <http://e.org/p/%d> " % p[k] + obj + (b" <http://g/%d>" % (k % 3) if kind[k] == 5 else b"") + b" ."
        if kind[k] == 6:
            line = b"# comment %d" % k
        if errors_every and k % errors_every == errors_every - 1:
            line = line[: len(line) // 2]
        out.append(line)
    return eol.join(out) + (eol if n % 2 == 0 else b"")


CASES = {
    "edge": edge_file,
    "empty": lambda: b"",
    "comments_only": lambda: b"# one\n\n# two",
    "no_final_newline": lambda: b"<a> <b> <c> .\n<a> <b> <d> .",
    "single": lambda: b"<a> <b> <c> .\n",
    "rand_small": lambda: random_file(2000, 1),
    "rand_crlf_errors": lambda: random_file(30_000, 2, crlf=True, errors_every=97),
    "rand_large": lambda: random_file(120_000, 3),  # > 1 MB: split over host threads
}
