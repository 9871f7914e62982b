"""CPU oracle for the fracodec encoder search -- TEST INFRASTRUCTURE ONLY.

This package restates, on the CPU, the reference algorithm of the encoder hot
path (arXiv 1502.00324 reference ``fracodec`` under ``/root/reference/pkg``)
so the B200 implementation can be checked against it.  It is *not* part of
the product: only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import it,
and only as the checker or the timed CPU baseline.  The product package
``paper_1502_00324_b200`` never imports it and has no CPU fallback.

Pinning: ``tests/test_oracle_golden.py`` checks this restatement against the
golden vectors in ``tests/golden/`` that ``tools/make_golden.py`` produced by
importing the reference package itself in the build container.
"""

from .fracodec_oracle import *  # noqa: F401,F403
