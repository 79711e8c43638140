"""CPU oracle for the mvamg solve path -- TEST INFRASTRUCTURE ONLY.

Importable only from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg, where it is the checker or the timed
CPU baseline -- never the product path.
"""
