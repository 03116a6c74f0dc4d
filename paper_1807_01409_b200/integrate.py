"""Rebinding of the reference package ``tripleid`` onto libtidq.

The reference has no FFI or plugin registry: its callers reach the hot path
through module attributes (``query_ops.scan_patterns`` -> ``search_multi``,
query_ops.py:278; ``entailment._search_rows``, entailment.py:147;
``cli.cmd_query`` -> ``query_ops.evaluate_query``, cli.py:142;
``cli.cmd_entail`` -> ``entailment.run_rule``, cli.py:163; ``cli.main`` looks
``cmd_convert`` up when it builds its parser, cli.py:277), so the drop-in is
an import-time rebinding with no reference source change.  ``install()``
performs exactly the rebinding INTEGRATION.md documents and returns a handle
whose ``restore()`` puts the reference's own functions back.

    import tripleid
    from paper_1807_01409_b200 import integrate
    with integrate.install():
        tripleid.cli.main(["query", "data/base", "q.rq"])   # runs on the B200
"""

from __future__ import annotations

import importlib

# (reference module, attribute, our module, our attribute)
BINDINGS = [
    ("kernel", "search_chunk", "kernel", "search_chunk"),        # kernel.py:148
    ("kernel", "search_multi", "kernel", "search_multi"),        # kernel.py:182
    ("kernel", "search_file", "kernel", "search_file"),          # kernel.py:230
    ("kernel", "gather_rows", "kernel", "gather_rows"),          # kernel.py:257
    ("query_ops", "search_multi", "kernel", "search_multi"),     # bound at query_ops.py import
    ("query_ops", "merge_join", "query_ops", "merge_join"),      # query_ops.py:144
    ("query_ops", "scan_patterns", "query_ops", "scan_patterns"),  # query_ops.py:263
    ("query_ops", "evaluate_union", "query_ops", "evaluate_union"),  # query_ops.py:359
    ("query_ops", "project_distinct", "query_ops", "project_distinct"),  # query_ops.py:379
    ("query_ops", "evaluate_query", "query_ops", "evaluate_query"),  # query_ops.py:432
    ("entailment", "search_multi", "kernel", "search_multi"),    # bound at entailment.py import
    ("entailment", "run_rule", "entailment", "run_rule"),        # entailment.py:175
    ("cli", "cmd_convert", "convert", "cmd_convert"),            # cli.py:64 (native N-Triples converter)
]


class Installed:
    """The saved reference attributes; ``restore()`` (or leaving the
    ``with`` block) puts them back."""

    def __init__(self, saved):
        self.saved = saved

    def restore(self) -> None:
        for mod, name, value in reversed(self.saved):
            setattr(mod, name, value)
        self.saved = []

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.restore()


def install(package: str = "tripleid") -> Installed:
    """Rebind the reference package's hot-path attributes to this library."""
    saved = []
    for ref_mod, ref_name, our_mod, our_name in BINDINGS:
        rm = importlib.import_module(f"{package}.{ref_mod}")
        om = importlib.import_module(f"{__package__}.{our_mod}")
        if not hasattr(rm, ref_name):
            continue  # a name the reference module does not bind (nothing calls it there)
        saved.append((rm, ref_name, getattr(rm, ref_name)))
        setattr(rm, ref_name, getattr(om, our_name))
    return Installed(saved)
