"""Float64 CPU oracle for the SpecPrefill hot path -- TEST INFRASTRUCTURE ONLY.

Importable only from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  Shares no code with the CUDA path.
"""
