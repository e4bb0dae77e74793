"""CPU oracle of the adaptive s-step CG hot path -- TEST INFRASTRUCTURE ONLY.

Imported only by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs, always as the checker or the CPU baseline, never as the
thing measured or shipped.  See sscg_oracle.py.
"""
