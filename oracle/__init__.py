"""CPU oracle for the SPED hot path — TEST INFRASTRUCTURE ONLY.

This package is a plain numpy/scipy restatement of the reference
``specgap`` package's hot path (graph canonicalisation, Laplacian CSR,
dilation-polynomial apply, edge-minibatch oracle, mu-EigenGame / Oja steps).
Every function cites the reference ``file:line`` it follows
(paths relative to ``/root/reference/pkg/src/specgap/``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import it, and there only as
the checker / the timed CPU baseline.  The product package
``paper_2207_14589_b200`` never imports it.

Parity pinning: the restatement is checked against golden vectors produced by
running the reference itself in the build container
(``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``), see
``tests/test_oracle_golden.py``.  The per-term edge-minibatch polynomial has no
reference implementation; that composition is "restated" and is pinned only by
the identity-oracle goldens plus Monte-Carlo unbiasedness.
"""

from .specgap_oracle import *  # noqa: F401,F403
from .specgap_oracle import __all__  # noqa: F401
