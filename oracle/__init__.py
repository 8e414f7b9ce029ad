"""CPU oracle for the CaPGNN halo-exchange + aggregation hot path.

TEST INFRASTRUCTURE ONLY. Nothing under ``oracle/`` is part of the product:
only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it, and only as the
checker (or the timed CPU baseline), never as the thing measured or shipped.

Two halves:

* ``halo_port``  -- a numpy / pure-Python restatement of the reference
  ``halopart`` integer algorithms on the path (CSR build, k-hop halos,
  partition stats, influence scores, Algorithm-1 capacities, the two-level
  JACA/FIFO/LRU cache and the simulator's round-robin epoch loop).  It is
  PINNED against golden vectors produced by the reference itself
  (``tests/golden/make_golden.py`` imports ``halopart`` from
  ``/root/reference`` and writes the fixtures).
* ``model_port`` -- a float64 numpy restatement of partitioned full-batch
  GCN / GraphSAGE-mean training over those integer outputs, with the
  staleness / caching semantics pinned in DESIGN.md §3.  The reference has no
  float code, so this half is "parity unpinned" against the reference; it is
  self-checked against a plain full-graph model (capacity 0 or s = 0 must
  equal full-graph training).
"""
