from .beam import (beam_search, beam_search_batch, shared_encoder_kv, topk_global,
                   topk_precut)
from .cache import TtlCache
from .engine import ServeResult, ServingConfig, ServingEngine, SnapshotStore
from .schedule import (BeamSchedule, TrafficSignal, capacity_slack, resolve_dbw,
                       scale_schedule, tabs_adjust)

__all__ = ["beam_search", "beam_search_batch", "shared_encoder_kv", "topk_global",
           "topk_precut", "TtlCache", "ServeResult", "ServingConfig", "ServingEngine",
           "SnapshotStore", "BeamSchedule", "TrafficSignal", "capacity_slack",
           "resolve_dbw", "scale_schedule", "tabs_adjust"]
