"""B200-native speculative expert-prefetch MoE decode path (arXiv 2603.19289).

The product is libsmoe_b200.so (paper_2603_19289_b200/csrc, C ABI in
include/smoe.h); this package only binds it.
"""
from .engine import (EXPORTS, GATING, MODE, PRED, CopyEvent, Event, ModelConfig, Session,
                     SmoeError, breakdown, hybrid_map_json, layer_hit_rates, load_library, recall_at_k,
                     select_hybrid_map, simulate, xp_pack, xp_unpack)

__all__ = ["EXPORTS", "GATING", "MODE", "PRED", "CopyEvent", "Event", "ModelConfig", "Session",
           "SmoeError", "breakdown", "hybrid_map_json", "layer_hit_rates", "load_library", "recall_at_k",
           "select_hybrid_map", "simulate", "xp_pack", "xp_unpack"]
