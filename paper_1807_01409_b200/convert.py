"""N-Triples -> TripleID conversion on the host cores.

The reference converts with a pure-Python loop (cli.py:64-114:
``nt.parse_stream`` -> ``Dictionary.encode`` per term -> ``write_tid`` +
``write_id_files``).  Here the same work runs natively and in parallel
(``tidq_convert_nt``, csrc/convert.cpp): every host thread parses a
line-aligned slice of the input with nt.py's exact grammar and error rules,
a sequential merge assigns IDs in the reference's first-occurrence order, and
the four output files are byte-identical to the reference's.  String <-> ID
work stays on the host, as the north star prescribes; no GPU is needed.

``cmd_convert`` mirrors cli.cmd_convert (same stderr diagnostics, exit codes
and temporary-file/rename protocol), so the reference CLI can be rebound to it
(paper_1807_01409_b200.integrate).
"""

from __future__ import annotations

import ctypes
import os
import sys
from dataclasses import dataclass, field
from pathlib import Path
from time import perf_counter

from . import _lib
from .errors import ParseError

ROLE_SUFFIXES = (".sid", ".pid", ".oid")
EXIT_PARSE = 1
EXIT_IO = 2


@dataclass
class ConvertResult:
    """Counts of one conversion (cli.py:100-111 prints them)."""

    triples: int
    distinct: tuple  # Dictionary.role_counts(): subjects, predicates, objects
    terms: int       # dictionary size = largest ID
    skipped: int     # ParseReport.skipped: blank and comment lines
    errors: list = field(default_factory=list)  # ParseError per malformed line (lenient mode)
    file_bytes: tuple = ()

    @property
    def error_count(self) -> int:
        return len(self.errors)


def _tmp_paths(out_base: Path):
    tid = out_base.with_name(out_base.name + ".tid.tmp")
    dict_base = out_base.with_name(out_base.name + ".tmp")
    return tid, [dict_base.with_name(dict_base.name + s) for s in ROLE_SUFFIXES]


def convert_nt(input_path, out, strict: bool = False, threads: int = 0) -> ConvertResult:
    """Convert an N-Triples file into ``<out>.tid`` + ``<out>.{sid,pid,oid}``.

    strict: the first malformed line raises ParseError (nt.py:26-33) and
    nothing is written.  Lenient: malformed lines are skipped and returned in
    ``errors``.  I/O failures raise OSError; partial temporary files are
    removed as cli.py:92-98 does."""
    with open(input_path, "rb"):  # OSError exactly as cli.py:71 raises it
        pass
    out_base = Path(out)
    rep = _lib.ConvertReport()
    errs = ctypes.c_void_p()
    tmp_tid, tmp_ids = _tmp_paths(out_base)
    rc = _lib.lib().tidq_convert_nt(os.fsencode(input_path), os.fsencode(out_base), int(strict), int(threads),
                                    ctypes.byref(rep), ctypes.byref(errs))
    try:
        if rc == _lib.E_IO and rep.io_errno:
            raise OSError(rep.io_errno, os.strerror(rep.io_errno), rep.io_path.decode("utf-8", "replace"))
        _lib.check(rc)
        errors = []
        if errs.value:
            text = ctypes.string_at(errs.value).decode("utf-8", "replace")
            for rec in text.splitlines():
                ln, off, msg = rec.split("\t", 2)
                errors.append(ParseError(msg, int(ln), int(off)))
        os.replace(tmp_tid, out_base.with_name(out_base.name + ".tid"))
        for tmp, suffix in zip(tmp_ids, ROLE_SUFFIXES):
            os.replace(tmp, out_base.with_name(out_base.name + suffix))
    except OSError:
        for leftover in [tmp_tid, *tmp_ids]:
            try:
                os.unlink(leftover)
            except OSError:
                pass
        raise
    finally:
        if errs.value:
            _lib.lib().tidq_convert_free(errs)
    return ConvertResult(int(rep.triples), tuple(int(x) for x in rep.distinct), int(rep.terms),
                         int(rep.skipped_lines), errors, tuple(int(x) for x in rep.file_bytes))


def cmd_convert(args) -> int:
    """cli.cmd_convert (cli.py:64-114) on the native converter: same
    diagnostics on stderr, same exit codes."""
    t0 = perf_counter()
    try:
        res = convert_nt(args.input, args.out, strict=args.strict)
    except ParseError as err:
        print(f"parse error: {err}", file=sys.stderr)
        return EXIT_PARSE
    except OSError as err:
        print(f"I/O error: {err}", file=sys.stderr)
        return EXIT_IO
    elapsed = perf_counter() - t0
    base = Path(args.out)
    paths = [base.with_name(base.name + ".tid")] + [base.with_name(base.name + s) for s in ROLE_SUFFIXES]
    diag = lambda *p: print(*p, file=sys.stderr)  # noqa: E731
    diag(f"triples\t{res.triples}")
    diag(f"distinct_subjects\t{res.distinct[0]}")
    diag(f"distinct_predicates\t{res.distinct[1]}")
    diag(f"distinct_objects\t{res.distinct[2]}")
    diag(f"skipped_lines\t{res.skipped}")
    diag(f"parse_errors\t{res.error_count}")
    for path in paths:
        diag(f"bytes\t{path.name}\t{path.stat().st_size}")
    diag(f"elapsed_seconds\t{elapsed:.3f}")
    return 0
