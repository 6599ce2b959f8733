"""CPU oracle for the SiDA serving hot path -- TEST INFRASTRUCTURE ONLY.

This package is a plain-numpy restatement of the reference algorithm
(`/root/reference/pkg/src/sida/`, arxiv 2310.18859 desk-scale package) for
exactly the functions on the B200 hot path.
Every function cites the reference file:line it restates.

Who may import this package:
  * ``tests/``                       -- as the parity checker;
  * ``__graft_entry__.smoke()``      -- as the checker of one small GPU call;
  * ``bench.py`` ``cpu_baseline`` leg and ``--impl reference`` arm -- as the
    timed CPU implementation (``kind: "port"``).
The product package ``paper_2310_18859_b200`` never imports it; the product
path has no CPU fallback and fails loudly without the CUDA library.

Pinning: ``tests/golden/make_golden.py`` imports the real reference (in the
build container, where ``/root/reference`` exists), runs it on seeded inputs
and commits the outputs as ``tests/golden/*.npz`` / ``*.json``;
``tests/test_oracle_golden.py`` checks this oracle against those fixtures on
every CPU test run. Permutation order (A13) has no reference test or fixture:
it is pinned by its restatement (stable argsort) and the fixture generated
from numpy's own stable argsort on the reference's hash-table ids.
"""

from . import numkit, moe, predictor, permute, offload  # noqa: F401
