"""CPU oracle for the StripedHyena 2 convolution hot path — TEST INFRASTRUCTURE ONLY.

This package is a numpy restatement of the reference ``convhybrid`` algorithms
(/root/reference/pkg/src/convhybrid, cited per function). It exists to check the
CUDA path, never to be it: only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import it. The
product package ``paper_2503_01868_b200`` must never import anything from here.

Parity pinning: the restatement is checked against golden vectors produced by
the reference itself (``tests/golden/make_golden.py`` imports the read-only
reference and writes ``tests/golden/*.npz``) and against the reference's own
known-answer tests (``tests/test_oracle_golden.py``).
"""

from .ref import *  # noqa: F401,F403
from . import cpsim  # noqa: F401
