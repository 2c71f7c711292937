"""CPU ORACLE for FAST-GED (arXiv 2605.00830) — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import anything under ``oracle/``.  The product
package ``paper_2605_00830_b200`` never imports it and shares no code with it.

* ``oracle.oracle``      — ctypes binding of ``fastged_oracle.c`` (plain C K-Best, Alg. 1)
* ``oracle.bruteforce``  — numpy enumeration of all partial injections (exact GED)

Parity status: every function is pinned by ``tests/test_oracle_pins.py``
(worked examples of SPEC.md, closed forms, brute force); see DESIGN.md §4.
"""
