"""CPU oracle for the HBS compress-from-samples path -- TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline leg may
import this package, and only as the checker / the timed CPU reference.  The
product path (`paper_2205_02990_b200`) never imports it.
"""
