"""CPU oracle for the walkvec hot path -- TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference algorithm (/root/reference/pkg/src/walkvec,
each function cites the file:line it follows), used as the checker in
tests/, by __graft_entry__.smoke() and as bench.py's cpu_baseline leg /
``--impl reference`` arm.  Nothing in the product package imports it.

Pinned against the reference itself: tests/golden/make_golden.py runs the
reference (imported read-only from /root/reference in the build container)
and commits its outputs as fixtures; tests/test_oracle.py checks this
restatement against every fixture, and the reference's own analytic
known-answer values (6 ln 2 zero-state loss, scalar Adam recurrence).
Third-party arithmetic (numpy's SeedSequence / PCG64 / Philox streams,
numpy 2.3.x) is restated in oracle/rng.py and checked against numpy.
"""
