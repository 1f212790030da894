"""CPU oracle for the jvp/vjp derivative path -- TEST INFRASTRUCTURE ONLY.

This package is a from-scratch NumPy (+ one small C file) restatement of the
reference implementation's algorithm (``conegrad`` 0.1.0, the CPU companion
of arXiv 2508.17522).  Each function cites the reference ``file:line`` it
follows; paths are relative to ``/root/reference/pkg/src/conegrad``.

It exists for exactly three consumers and must never be imported by the
product package ``paper_2508_17522_b200``:

* ``tests/``                   -- the checker the CUDA path is compared with;
* ``__graft_entry__.smoke()``  -- one small parity check on ``cuda:0``;
* ``bench.py``                 -- the ``cpu_baseline`` leg and ``--impl reference``.

Parity of the oracle itself is pinned against fixtures produced by running
the real reference in the build container (``tests/golden/make_fixtures.py``)
and against the reference's own committed golden files
(``pkg/tests/golden/*.json``, converted into ``tests/golden/*.npz``).
"""

from oracle import cones, qcp, gen  # noqa: F401
