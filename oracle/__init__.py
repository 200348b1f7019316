"""TEST INFRASTRUCTURE ONLY — CPU oracle for the spaQR hot path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
arms (``cpu_baseline`` / ``--impl reference``) may import this package, and
only as the checker or the timed CPU reference — never as part of the
shipped B200 path (``paper_2010_06807_b200`` never imports it and fails
loudly when its CUDA library is missing).

``spaqr_oracle`` restates, in numpy, the reference package's algorithm
(`/root/reference/pkg/src/nestqr/factor.py`, `kernels/*.py`); every function
cites the reference lines it follows.  Parity of the restatement itself is
PINNED against the real reference: ``tests/golden/make_golden.py`` imported
the reference in the build container and wrote golden vectors (kernel
known-answer cases, per-level ranks/stats, R blocks, GMRES histories) that
``tests/test_oracle.py`` checks on every CPU run.
"""
