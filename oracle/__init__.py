"""CPU oracle for the flow-analysis hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package, and only as the checker or the
timed CPU baseline; the product (paper_1108_1785_b200) never does.

* ``Oracle``    — ctypes wrapper of lib/liborc.so, the plain-C restatement
                  (gnm_oracle.c) of the reference's algorithm.
* ``Reference`` — ctypes wrapper of _ref/libflowmon_ref.so, the UNMODIFIED
                  reference sources compiled in place (oracle/Makefile `ref`),
                  present wherever it was built (it travels with the repo
                  snapshot; /root/reference itself does not).
"""
from .oracle import Oracle, Reference, reference_available  # noqa: F401
