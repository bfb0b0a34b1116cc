"""ORACLE — test infrastructure, not product.

CPU restatement of the EDGC reference's data-parallel hot path
(/root/reference/pkg/src/edgc).  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s CPU-baseline / ``--impl reference`` leg may import this
package, and only as the checker or the timed CPU baseline.  The product
package ``paper_2511_10333_b200`` never imports it and has no CPU fallback.

Pinning: every function here is checked against the live reference (in the
build container) through the committed golden fixtures in ``tests/golden``
(generator: ``tests/golden/make_golden.py``).  The NumPy index rule
(``npchoice.c``) is additionally checked bit-for-bit against NumPy 2.3.5.
"""

from .oracle import *  # noqa: F401,F403
