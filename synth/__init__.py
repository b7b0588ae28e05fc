"""Seeded synthetic inputs shared by the oracle-side tests and the CUDA-side tests/bench.

This package holds input GENERATORS only -- none of the method's arithmetic (no T-CSR,
no cut search, no selection, no gather).  Both sides of every parity check consume the
same arrays produced here.  ``tiny`` builds small random graphs with numpy; ``configs``
builds the five paper-shaped workloads C1-C5 with integer-only torch ops
so the same bits come out on CPU and GPU.
"""
