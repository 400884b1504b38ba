"""TEST INFRASTRUCTURE ONLY (checkers for the device engine).

- ``oracle.ref``   ctypes access to the unmodified reference library built into ``oracle/_ref``.
- ``oracle.port``  ctypes access to ``liboracle.so``, the plain-C restatement in ``ttutv_oracle.c``.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may use this package.
"""
