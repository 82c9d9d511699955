"""Test oracle (NOT product code). Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package, and only as the checker or
the timed CPU baseline.

* ``oracle.ref``    -- the compiled, unmodified reference host library (oracle/_ref/libsbref.so,
                       built from /root/reference by oracle/Makefile) bound with the same
                       marshalling as the product (prefix ``sbref_``).
* ``oracle.device`` -- CPU restatement (fp64, C) of the device half: block scorer, top-k
                       selector, coverage profile, sparse attention fwd/bwd. The reference has
                       no implementation of these: parity of the device half is
                       "unpinned" by the reference and pinned instead by the golden vectors in
                       tests/golden (see DESIGN.md section Oracle).
"""
