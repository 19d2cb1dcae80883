"""ORACLE / TEST INFRASTRUCTURE ONLY: CPU restatement of the reference ChFSI algorithm.

Importable only from tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg,
as the checker / timed CPU baseline; never on the product path.
"""
