from .decoder import (DecoderConfig, DecoderModel, ForwardTrace, Param, context_process,
                      lazy_forward, load_checkpoint, save_checkpoint, sequence_log_prob)
from .layers import LN_EPS, LayerCallCounter

__all__ = ["DecoderConfig", "DecoderModel", "ForwardTrace", "Param", "context_process",
           "lazy_forward", "sequence_log_prob",
           "load_checkpoint", "save_checkpoint", "LayerCallCounter", "LN_EPS"]
