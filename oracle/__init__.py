"""CPU oracle for the Safhire server hot path — TEST INFRASTRUCTURE ONLY.

This package is a plain numpy restatement of the reference's server-side
algorithm (``/root/reference/pkg/src/sfhr``), written independently from its
published behaviour, plus the client half (keygen / encrypt / decrypt) needed
to build message-level checks.  Every function cites the reference file:line
it restates.

Who may use it: ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs — only as the checker or as the
timed CPU baseline.  The product package ``paper_2509_01253_b200`` never
imports anything from here and has no CPU fallback.

Parity pin: ``tests/golden/make_golden.py`` imports the real reference in the
build container and records fixtures under ``tests/golden/``; the CPU tests
(``tests/test_oracle_golden.py``) check this oracle bit-for-bit against them.
"""

from . import scheme, keyswitch, pack, lowering, protocol  # noqa: F401
