"""TEST INFRASTRUCTURE ONLY — CPU restatement of the wavevid decode path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this package, and only as the checker / the timed CPU
reference.  The product decode path (``paper_2208_10859_b200``) never
imports it.  Parity of this restatement is pinned by fixtures produced by
running the real reference (``tests/golden/make_golden.py``).
"""
