"""ORACLE — TEST INFRASTRUCTURE ONLY.

A CPU restatement of the reference (``mpkrylov``, /root/reference/pkg) solve
path, used as the *checker* for the B200 product path and as the CPU baseline
arm of ``bench.py``.  Nothing in ``paper_2105_07544_b200`` may import, load or
call anything in this directory; the product fails loudly when its CUDA
library is missing instead of falling back here.

Allowed importers: ``tests/``, ``__graft_entry__.smoke()`` (as the checker),
``bench.py`` (``cpu_baseline`` leg and ``--impl reference``).

Pinning: ``tests/test_oracle_golden.py`` checks this restatement against the
golden vectors in ``tests/golden/`` that ``tests/golden/make_golden.py``
produced by importing the unmodified reference in the survey container.
"""
