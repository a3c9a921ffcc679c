"""CPU oracle for parity tests and the CPU baseline — test infrastructure only.

Importable only from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  See oracle/hotpath.py for the
reference anchors and pinning.
"""
