"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the fine-propagator hot path.

This package is a numpy restatement of the reference solver
(``/root/reference/pkg/src/parakin``) restricted to the 1D-x / 1D-v case, with
the same elementwise operation order and the same (numpy pairwise / sequential
cumsum) reduction order, so that it reproduces the reference bit for bit.  It
additionally carries the spatially varying eps(x) extension, which
reduces bitwise to the reference when eps is constant.

Parity pinning: ``tests/golden/make_golden.py`` runs the real reference (in the
build container, where ``/root/reference`` exists) and stores golden vectors
under ``tests/golden/``; ``tests/test_oracle_golden.py`` checks this oracle
against them bitwise.

Who may import this: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s CPU-baseline / ``--impl reference`` leg.  The product package
``paper_2511_13386_b200`` never imports it.
"""

from .restate import *  # noqa: F401,F403
