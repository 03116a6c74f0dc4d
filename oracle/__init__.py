"""CPU oracle for the TripleID-Q query path — TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference's algorithm for the hot path
(``/root/reference/pkg/src/tripleid/kernel.py`` and ``query_ops.py``), every
function citing the reference file:line it follows.  It is the parity checker
and the CPU baseline ("kind": "port"), nothing else: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl
reference`` legs may import it.  The product package never imports it and has
no CPU fallback.

Parity pinning: the oracle is checked (tests/test_oracle.py, CPU suite)
against golden vectors produced by running the REFERENCE ITSELF in the build
container (``tests/golden/make_golden.py`` imports ``/root/reference/pkg/src``)
and against the SPEC.md known-answer examples.  So parity is pinned to the
reference's own outputs, not to this restatement.

Modules
- ``scan``   search_chunk / search_multi / scan_patterns   (kernel.py:148-227,
             query_ops.py:263-295)
- ``query``  pattern_table, apply_filter, analyze_relationships, merge_join,
             join_group, evaluate_union, project_distinct, evaluate_query
             (query_ops.py:63-455)
- ``synth``  numpy twin of the device generator
- ``entailment`` run_rule of the six two-stage RDFS rules (entailment.py:46-255)
"""
