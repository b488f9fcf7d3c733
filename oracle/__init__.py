"""CPU oracle -- TEST INFRASTRUCTURE ONLY (see hm_oracle.py header).

Importable from tests/, __graft_entry__.smoke() and bench.py's CPU-baseline
leg only; never from the shipped package.
"""
