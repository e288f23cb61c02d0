"""CPU oracle for parity tests -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference
arm may import this package. The product package (paper_2212_02197_b200)
never does. See oracle/Makefile for what is built where.
"""
