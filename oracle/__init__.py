"""CPU oracles for the q8p parity tests -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` leg may import this package, and only as the checker or
the timed CPU reference; the product (paper_2402_04396_b200/) never does.
"""
