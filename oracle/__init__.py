"""CPU oracle for the knob-tuner search step — TEST INFRASTRUCTURE ONLY.

This package restates, in plain numpy, the reference algorithms that the
B200 engine replaces (reference: ``/root/reference/pkg/src/knobtuner``).  It
exists to *check* the CUDA path, never to be it:

* only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
  ``cpu_baseline`` / ``--impl reference`` legs may import it;
* the product package ``paper_1905_12799_b200`` must never import it (a test
  enforces this), and fails loudly when its CUDA library is missing.

Parity pinning: every function here is checked bit-for-bit against golden
vectors produced by running the reference itself (``tests/golden/make_golden.py``,
run in the build container where ``/root/reference`` is importable) plus the
reference's own known-answer tests restated in ``tests/test_oracle.py``.

Every function operates on arrays (knob-index matrices, packed trees, ...)
rather than the reference's Python objects, and cites the reference lines it
restates.  Floating-point reduction orders follow numpy exactly (numpy's
pairwise summation for contiguous 1-D/last-axis sums, sequential for
axis-0 sums), because the reference's results depend on them.
"""
