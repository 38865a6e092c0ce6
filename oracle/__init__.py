"""TEST INFRASTRUCTURE ONLY — the CPU parity checkers.

``oracle.port``: ctypes bindings of the plain-C restatement (oracle/mf_oracle.c).
``oracle.ref``:  ctypes bindings of the reference's own translation units
                 compiled in place (oracle/_ref/libmfref.so, oracle/Makefile).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this package; the product
(paper_2605_26137_b200, libmfbake.so) never does.
"""
