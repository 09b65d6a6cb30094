"""Model container and configuration, mirroring ``adrec.model.decoder``
(pkg/src/adrec/model/decoder.py).

Inference-only: parameters are host float64 arrays (the reference's
``DecoderModel.params``), uploaded to the GPU once per snapshot as fp32 by
:mod:`paper_2602_22732_b200.device`.  Training-only parts of the reference
(trunk logits, MTP, autodiff) are out of scope.
"""

from __future__ import annotations

import io
import json
from dataclasses import dataclass

import numpy as np

_FORMAT_VERSION = 1  # decoder.py:29


class Param:
    """Minimal stand-in for the reference ``autodiff.Tensor`` on the
    inference path: a float64 ndarray under ``.data`` (autodiff.py:51-67)."""

    __slots__ = ("data",)

    def __init__(self, data):
        self.data = np.asarray(data, dtype=np.float64)

    @property
    def shape(self):
        return self.data.shape

    @property
    def ndim(self):
        return self.data.ndim

    def __repr__(self):
        return f"Param(shape={self.data.shape})"


@dataclass(frozen=True)
class DecoderConfig:
    """decoder.py:32-51 (same fields, same validation)."""

    feat_dim: int
    d: int
    d_ff: int
    n_layers: int
    trunk_depth: int
    level_vocab_sizes: tuple
    n_value_buckets: int
    seed: int = 0

    def __post_init__(self):
        if not 0 <= self.trunk_depth < self.n_layers:
            raise ValueError("trunk_depth must satisfy 0 <= K < n_layers")
        if not self.level_vocab_sizes or any(v < 1 for v in self.level_vocab_sizes):
            raise ValueError("level_vocab_sizes must be positive")

    @property
    def n_levels(self):
        return len(self.level_vocab_sizes)


_LAYER_PARAMS = (  # decoder.py:54-61, in draw order
    ("ln1.g", "one"), ("ln1.b", "zero"),
    ("cross.Wq", "dd"), ("cross.Wk", "dd"), ("cross.Wv", "dd"), ("cross.Wo", "dd"),
    ("ln2.g", "one"), ("ln2.b", "zero"),
    ("self.Wq", "dd"), ("self.Wk", "dd"), ("self.Wv", "dd"), ("self.Wo", "dd"),
    ("ln3.g", "one"), ("ln3.b", "zero"),
    ("ffn.W1", "d_ff"), ("ffn.b1", "zero_ff"), ("ffn.W2", "ff_d"), ("ffn.b2", "zero"),
)


def _init_params(cfg):
    """Seeded uniform(+-1/sqrt(fan_in)) init drawn in the reference's order
    (decoder.py:71-107), so ``DecoderModel(cfg)`` is bit-identical to the
    reference's for the same config and seed."""
    rng = np.random.default_rng(cfg.seed)
    d, dff = cfg.d, cfg.d_ff

    def draw(shape, fan_in):
        s = 1.0 / np.sqrt(fan_in)
        return Param(rng.uniform(-s, s, size=shape))

    p = {"ctx.W": draw((cfg.feat_dim, d), cfg.feat_dim), "ctx.b": Param(np.zeros(d)),
         "pos": draw((cfg.n_levels + 1, d), d), "bos": draw((d,), d)}
    for t, v in enumerate(cfg.level_vocab_sizes):
        p[f"emb.{t}"] = draw((v, d), d)
    fill = {"one": lambda: Param(np.ones(d)), "zero": lambda: Param(np.zeros(d)),
            "zero_ff": lambda: Param(np.zeros(dff)), "dd": lambda: draw((d, d), d),
            "d_ff": lambda: draw((d, dff), d), "ff_d": lambda: draw((dff, d), dff)}
    for i in range(cfg.n_layers):
        for name, kind in _LAYER_PARAMS:
            p[f"layer{i}.{name}"] = fill[kind]()
    p["fuse.Wg"] = draw((d, d), d)
    p["fuse.Wf"] = draw((2 * d, d), 2 * d)
    for t, v in enumerate(cfg.level_vocab_sizes):
        p[f"head.{t}"] = draw((d, v), d)
    p["head.value"] = draw((d, cfg.n_value_buckets), d)
    return p


class DecoderModel:
    """Parameter container (decoder.py:64-123)."""

    def __init__(self, config, params=None):
        self.config = config
        self.params = params if params is not None else _init_params(config)

    def clone(self):
        """Deep copy (copy-on-publish snapshots, decoder.py:113-117)."""
        return DecoderModel(self.config, {k: Param(np.array(getattr(v, "data", v), copy=True))
                                          for k, v in self.params.items()})

    def head_layer_names(self):
        k = self.config.trunk_depth
        return [n for n in self.params
                if n.startswith("layer") and int(n[5:n.index(".")]) >= k]


def param_array(v):
    return np.asarray(getattr(v, "data", v), dtype=np.float64)


def context_process(features, params):
    """X = F W_c + b_c (decoder.py:134-140), computed on the GPU.

    Returns a :class:`~paper_2602_22732_b200.device.DeviceContext` that keeps
    the fp32 result resident for ``beam_search`` and exposes ``.data``
    (float64 host copy) like the reference's Tensor."""
    from paper_2602_22732_b200.device import context_process_gpu
    return context_process_gpu(features, params)


@dataclass
class ForwardTrace:
    """decoder.py:126-131.  Trunk logits feed training losses only and are
    not computed on the serving path (None)."""

    head_logits: list
    trunk_logits: object = None
    value_logits: object = None
    states: object = None


def lazy_forward(model, context, tokens, trunk_depth=None, include_value_step=True,
                 counter=None):
    """Teacher-forced forward of one token sequence on the GPU
    (decoder.py:162-198): per-level head logits and the value-bucket logits."""
    from paper_2602_22732_b200.decode import score_sequences
    cfg = model.config
    k = cfg.trunk_depth if trunk_depth is None else trunk_depth
    if not 0 <= k < cfg.n_layers:
        raise ValueError("trunk_depth must satisfy 0 <= K < n_layers")
    if len(tokens) != cfg.n_levels:
        raise ValueError(f"expected {cfg.n_levels} tokens, got {len(tokens)}")
    ctx = getattr(context, "tensor", None)
    ctx = ctx.double().cpu().numpy() if ctx is not None else getattr(context, "data", context)
    res = score_sequences(model, [0], [list(tokens)], contexts=[ctx], trunk_depth=k,
                          include_value_step=include_value_step, return_logits=True)
    n_pos = cfg.n_levels + (1 if include_value_step else 0)
    if counter is not None:  # layers.py:79-80 via decoder.py:184-186
        for _ in range(cfg.n_layers):
            counter.add_layer_calls(n_pos)
    if include_value_step:
        _, vl, heads = res
        value = Param(vl[0])
    else:
        _, heads = res
        value = None
    return ForwardTrace([Param(h[0]) for h in heads], None, value)


def sequence_log_prob(trace, tokens):
    """Total log-probability of the sequence under the trace (decoder.py:213-219)."""
    total = 0.0
    for t, tok in enumerate(tokens):
        lg = param_array(trace.head_logits[t])
        mx = lg.max()
        total += float((lg[int(tok)] - mx) - np.log(np.exp(lg - mx).sum()))
    return total


def save_checkpoint(model, path, step=0, extra_arrays=None, meta=None):
    """Reference-compatible npz + JSON header (decoder.py:222-247)."""
    c = model.config
    header = {"format_version": _FORMAT_VERSION,
              "config": {"feat_dim": c.feat_dim, "d": c.d, "d_ff": c.d_ff,
                         "n_layers": c.n_layers, "trunk_depth": c.trunk_depth,
                         "level_vocab_sizes": list(c.level_vocab_sizes),
                         "n_value_buckets": c.n_value_buckets, "seed": c.seed},
              "step": step, "meta": meta or {},
              "extra_keys": sorted(extra_arrays) if extra_arrays else []}
    arrays = {f"param::{k}": param_array(v) for k, v in model.params.items()}
    if extra_arrays:
        arrays.update({f"extra::{k}": np.asarray(v) for k, v in extra_arrays.items()})
    buf = io.BytesIO()
    np.savez(buf, header=np.frombuffer(json.dumps(header).encode(), dtype=np.uint8), **arrays)
    with open(path, "wb") as fh:
        fh.write(buf.getvalue())


def load_checkpoint(path):
    """Returns ``(model, step, extra_arrays, meta)`` (decoder.py:250-263);
    reads checkpoints written by the reference."""
    with np.load(path) as data:
        header = json.loads(bytes(data["header"]).decode())
        if header["format_version"] != _FORMAT_VERSION:
            raise ValueError(f"unsupported checkpoint format {header['format_version']}")
        cfg_d = dict(header["config"])
        cfg_d["level_vocab_sizes"] = tuple(cfg_d["level_vocab_sizes"])
        cfg = DecoderConfig(**cfg_d)
        params = {k[len("param::"):]: Param(data[k]) for k in data.files
                  if k.startswith("param::")}
        extra = {k[len("extra::"):]: data[k] for k in data.files if k.startswith("extra::")}
    return DecoderModel(cfg, params), header["step"], extra, header["meta"]
