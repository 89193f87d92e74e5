"""CPU oracle of the reference csrk path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this package; the product never does.  See oracle.py.
"""
