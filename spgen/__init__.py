"""Seeded synthetic input generators shared by the oracle side and the CUDA side.

This package holds NO arithmetic of the method (no softmax, no aggregation, no
selection).  It only produces inputs: bf16 K caches, bf16 look-ahead query rows
and int32 token ids, from a counter-based integer generator.  The same
generator is implemented twice, bit-identically:

* ``spgen.gen``      -- numpy (used by the oracle side and by tests), any slice;
* ``spgen/gen.cu``   -- CUDA fill kernels in ``libspgen.so`` (used to fill
  multi-GiB device buffers for the parity tests and the bench).

See DESIGN.md "Input recipe" for the distributions and the paper passages the
structure imitates (attention sinks / proximity bias P:115, needles P:291).
"""
from .gen import Workload, CONFIGS, needle_spans, gen_K, gen_Q, gen_tokens  # noqa: F401
