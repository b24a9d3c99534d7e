"""CPU oracle for the EP N-particle hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import anything in this package.  The product
(``paper_1510_03816_b200``) never imports it and has no CPU fallback.

Two restatements of the reference algorithm (``/root/reference/pkg/src/geoshoot``):

* ``oracle.restate`` — numpy, line-for-line semantics of ``particles.py``,
  ``integrator.py`` and the momentum branch of ``shooting.py`` (row-blocked so
  it reaches N beyond the reference's ~30k memory wall).
* ``oracle/gs_oracle.c`` (``oracle.native``) — plain C + OpenMP, the same
  equations in the direct-difference form Σ_j c_ij (q_i − q_j), dense and
  cell-list (truncated at the KD-1 support radius), used for large-N parity
  and as the timed CPU baseline ("port").

Pinning: both are checked against the golden fixtures in ``tests/golden/``,
which were produced by running the unmodified reference in the build
container (``tests/golden/make_golden.py``), including the reference test
suite's independent sympy N=2 oracle (``test_particles.py:22-71``).
"""
