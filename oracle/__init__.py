"""CPU oracle for the HierMoE dedup dispatch/combine + expert-swap hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_2508_09591_b200`` imports this
package; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may use it, and only as the
checker (or the timed CPU baseline), never as the product path.

* :mod:`oracle.hiera` restates the reference ``hiera2a`` 0.1.0 decision path
  (``pkg/src/hiera2a/{topology,routing,traffic,swap}.py``) in numpy.  It is
  pinned against golden vectors produced by the reference itself
  (``tests/golden/make_golden.py``) and the reference's own known-answer
  tests.
* :mod:`oracle.moe` restates the MoE layer math the reference omits
  (softmax top-K gating, expert SwiGLU FFN, gate-weighted combine, and the
  per-rank dedup dispatch/combine decomposition) from ``PAPER.md:110-117``.
  The reference has no implementation of it: **parity unpinned** for layer
  outputs/gradients (the dedup copy lists it emits are pinned through
  :mod:`oracle.hiera`).
"""
