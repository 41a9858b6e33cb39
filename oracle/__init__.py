"""TEST INFRASTRUCTURE ONLY — CPU restatement of the reference SCFA path.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import anything under oracle/.  The product (paper_2306_01160_b200)
never does; it has no CPU fallback.

Pinned against the reference package itself: tests/golden/make_golden.py
imports /root/reference/pkg/src/scfa in the build container and writes the
fixtures that tests/test_oracle.py checks this restatement against.
"""
