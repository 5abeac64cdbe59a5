"""ORACLE — TEST INFRASTRUCTURE ONLY.

CPU restatements of the reference's algorithms for the hot path, used as
the checker in ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py``.  Nothing in
``paper_1601_07613_b200`` imports this package; the product path never
routes through it.

Pinning: every integer restatement here is checked against the golden
fixtures in ``tests/golden/`` that ``tests/golden/make_golden.py`` produced
by running the reference (/root/reference/pkg/src/meshchroma) itself.
The floating-point DG restatement (``dg_oracle``) has no reference
counterpart — the reference puts DG out of scope — so its
parity is "unpinned by the reference" and is anchored instead on
independent known-answer properties (free-stream preservation,
conservation, the integer bridge to ``sweep_sequential``, p+1 convergence);
see DESIGN.md §Oracle.
"""
