"""CPU oracle for the online polarized-traces solve -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this package, and only
as the checker or the timed CPU baseline -- never as the product path.

Parity pinning: the oracle is checked (tests/test_oracle.py) against golden
vectors produced by running the reference package itself
(tools/make_cases.py -> tests/golden/*.ptc): its operator applies, sweeps
and GMRES results on the reference's own offline data.
"""

from .ref_port import *  # noqa: F401,F403
