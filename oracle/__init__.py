"""CPU oracle for the ensemble-SSA hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may use
this package.  See ssa_oracle.c for the definitions and their citations.
"""
