"""B200-native LazyAR beam serving for GR4AD (arxiv 2602.22732).

Drop-in for the reference ``adrec`` serving hot path: ``model`` mirrors
``adrec.model`` (config, params, checkpoint I/O), ``serving`` mirrors
``adrec.serving`` (beam_search, schedule, engine, cache), ``quantizer``
keeps the SemanticId / SidIndex types.  All decode arithmetic runs in
``libgr4ad.so`` (hand-written sm_100a CUDA behind a C ABI, include/gr4ad.h);
importing the serving path without it raises -- there is no CPU fallback.
"""

__version__ = "0.1.0"
