"""CPU oracle for the monitored-free-fermion trajectory step (arXiv 2508.18468).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import anything
under ``oracle/``.  The product path (``paper_2508_18468_b200``) never imports it
and shares no code with it: no kernels, helpers, constant tables or generators.

The oracle is plain, slow and written to be checked against the paper by eye.
Every floating-point quantity is float64 / complex128.  Citations ``P:NNN`` are
lines of ``/root/reference/PAPER.md`` (section / equation named alongside);
readings of ambiguous passages are the ``Q*`` items listed in ``DESIGN.md``.

Modules
-------
philox     Philox4x32-10 counter-based RNG in NumPy uint64 arithmetic (Q8, Q9).
lattice    hopping matrix H~, propagator K = exp(-i H~ dt), Neel state.
gaussian   C = U U^dagger, D = <c_i^dagger c_j>, entanglement entropy,
           mutual information, Householder orthonormalisation.
protocols  homodyne / QSD step (Eq. A3) and projective step
           (Eq. A1, A2), sequential and block forms.
trajectory one trajectory driven step by step with sampled observables.

Parity status: every function is pinned by a ``-m "not gpu"`` test in
``tests/test_oracle_*.py`` (closed forms, invariants, Fock-space brute force,
published Philox known-answer vectors).  The Eq. (A3) drift and noise
coefficients of ``protocols.homodyne_factor`` / ``protocols.qsd_generator`` are
pinned without re-using their formulas by ``tests/test_oracle_drift_pins.py``
(Born-rule martingale E[n'] = n + O(dt^2) and the Lindblad dephasing rate
-gamma, both by exact Gauss-Hermite quadrature over the noise; wrong
coefficients are shown to fail).  Nothing here is "parity unpinned".
"""
