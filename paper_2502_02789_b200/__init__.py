"""B200-native (sm_100a) SpecPrefill hot path: speculator-side token importance
scoring and chunked top-k selection (arXiv 2502.02789).

The compute lives in libspecprefill.so (C ABI: include/specprefill.h); this
package is a thin binding plus the multi-GPU orchestration.
"""
from .api import (gather, kept_chunks, make_geom, score, score_chunks, score_e4m3, score_e4m3_plan, score_paged, select_ragged, score_lookahead, score_tune, score_e4m3_tune, select, specprefill,  # noqa: F401
                  check_device_error, run_host, run_workspace_bytes, score_plan, workspace,
                  score_stats, stats_combine, score_finish, score_acc, acc_importance,
                  score_peer, score_peer_buffer_bytes, score_peer_plan, score_peer_workspace_bytes,
                  seq_candidate_count, seq_edges, seq_candidates, seq_merge, score_select)
from ._lib import LIB_PATH, SIGNATURES, SpError, lib  # noqa: F401
