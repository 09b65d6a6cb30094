"""The SID value type returned by beam search (quantizer/residual.py:44-59
in the reference).  Quantizer fitting itself is offline tokenization and
out of scope for the serving path.

``SemanticId(tokens, level_vocab_sizes)`` validates exactly as the
reference's frozen dataclass (same ValueErrors) and exposes the same
surface: ``.tokens``, ``.level_vocab_sizes``, ``len()``, equality and
hashing by (tokens, level_vocab_sizes), immutability.  It is a tuple of the
tokens underneath (one subclass per vocabulary), so the decode API can
materialise hundreds of thousands of them straight from a token array
(:func:`sids_from_rows`, C-level construction, one vectorised range check)
instead of running the per-token Python validation for every result.
"""

from __future__ import annotations

import threading

import numpy as np


class SemanticId(tuple):
    """A per-level token sequence with its per-level vocabulary sizes."""

    __slots__ = ()
    level_vocab_sizes = ()

    def __new__(cls, tokens, level_vocab_sizes):
        tokens = tuple(tokens)
        level_vocab_sizes = tuple(level_vocab_sizes)
        if len(tokens) != len(level_vocab_sizes) or not tokens:
            raise ValueError("tokens and level_vocab_sizes must be equal, nonzero length")
        for t, (tok, size) in enumerate(zip(tokens, level_vocab_sizes)):
            if not 0 <= tok < size:
                raise ValueError(f"token {tok} out of range [0, {size}) at level {t}")
        return tuple.__new__(sid_type(level_vocab_sizes), tokens)

    @property
    def tokens(self):
        return tuple(self)

    def __len__(self):
        return tuple.__len__(self)

    def __eq__(self, other):
        if not isinstance(other, SemanticId):
            return False  # (not NotImplemented: a plain tuple would then compare equal)
        return (self.level_vocab_sizes == other.level_vocab_sizes
                and tuple.__eq__(self, other))

    def __ne__(self, other):
        return not self.__eq__(other)

    __hash__ = tuple.__hash__

    def __repr__(self):
        return (f"SemanticId(tokens={tuple(self)!r}, "
                f"level_vocab_sizes={self.level_vocab_sizes!r})")

    def __reduce__(self):
        return (SemanticId, (tuple(self), self.level_vocab_sizes))

    def __setattr__(self, name, value):  # frozen, like the reference dataclass
        raise AttributeError(f"cannot assign to field {name!r}")


_TYPES = {}
_TYPES_LOCK = threading.Lock()


def sid_type(level_vocab_sizes):
    """The SemanticId subclass of one vocabulary (instances are plain tuples
    of the tokens; the vocabulary is a class attribute)."""
    vocab = tuple(int(v) for v in level_vocab_sizes)
    cls = _TYPES.get(vocab)
    if cls is None:
        with _TYPES_LOCK:
            cls = _TYPES.get(vocab)
            if cls is None:
                # __new__ = tuple.__new__: sid_type(v)(row) builds from an
                # iterable of tokens at C speed (no per-token validation)
                cls = type("SemanticId", (SemanticId,),
                           {"__slots__": (), "level_vocab_sizes": vocab,
                            "__new__": tuple.__new__, "__module__": __name__,
                            "__qualname__": "SemanticId"})
                _TYPES[vocab] = cls
    return cls


def check_token_range(tokens, level_vocab_sizes):
    """Vectorised form of SemanticId's range check over a (..., T) integer
    array (the same ValueError for the first offending token)."""
    arr = np.asarray(tokens)
    vocab = np.asarray(level_vocab_sizes, dtype=np.int64)
    if arr.size == 0:
        return
    if arr.shape[-1] != vocab.size:
        raise ValueError("tokens and level_vocab_sizes must be equal, nonzero length")
    bad = (arr < 0) | (arr >= vocab)
    if bad.any():
        idx = np.argwhere(bad)[0]
        t = int(idx[-1])
        raise ValueError(f"token {int(arr[tuple(idx)])} out of range [0, {int(vocab[t])}) "
                         f"at level {t}")


def sids_from_rows(rows, level_vocab_sizes):
    """SemanticIds from already range-checked token rows (lists / tuples)."""
    return list(map(sid_type(level_vocab_sizes), rows))
