"""Per-rank time of the sequence-sharded single pass (sp_score_peer) as P
virtual ranks on one GPU (dev tool): P co-scheduled launches each capped at
SMs/P CTAs on its own K shard; the P launches share the GPU's HBM, so the
span of one call approximates P x one real rank's kernel (each rank on its own
GPU streams its shard with every SM).  Reports span/P as the per-rank estimate.

  python tools/peer_time.py C4 8 [C3 8 ...]
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from tools import peer_virtual  # noqa: E402
from spgen import gen  # noqa: E402

args = sys.argv[1:]
for i in range(0, len(args), 2):
    name, P = args[i], int(args[i + 1])
    w = gen.CONFIGS[name]
    plan, res, ms, (Q, K) = peer_virtual.run(w, P, iters=12)
    span = float(np.min(ms[2:]))
    kb = w.k_bytes / 1e9
    print(f"{name} P={P}: call span {span:.3f} ms (min of {len(ms) - 2}), per-rank estimate {span / P:.4f} ms "
          f"({kb / P / (span / P) :.0f} GB/s per rank of its 1/P shard); plan {plan}", flush=True)
    del Q, K, res
    torch.cuda.empty_cache()
