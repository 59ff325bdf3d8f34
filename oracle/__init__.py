"""CPU oracle — TEST INFRASTRUCTURE ONLY (see abm_oracle.py header).

May be imported by tests/, __graft_entry__.smoke() and bench.py's reference /
cpu_baseline legs only; the product package never imports it.
"""
