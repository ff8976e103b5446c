"""CPU oracle for the seisopt FWI/LSRTM hot path.

TEST INFRASTRUCTURE ONLY.  Nothing under ``paper_2008_11778_b200/`` imports this
package.  The only permitted callers are ``tests/``, ``__graft_entry__.smoke()``
(as the checker) and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``).  The oracle is pinned against golden vectors produced by
the unmodified reference (``tests/golden/make_golden.py``).
"""

from .seisopt_oracle import *  # noqa: F401,F403
