from .decoder import (DecoderConfig, DecoderModel, Param, context_process,
                      load_checkpoint, save_checkpoint)
from .layers import LN_EPS, LayerCallCounter

__all__ = ["DecoderConfig", "DecoderModel", "Param", "context_process",
           "load_checkpoint", "save_checkpoint", "LayerCallCounter", "LN_EPS"]
