"""ORACLE -- TEST INFRASTRUCTURE ONLY.

CPU restatement of the reference path (restate.py + loops.c).  Importable
only by tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs;
the product package never imports it.
"""
