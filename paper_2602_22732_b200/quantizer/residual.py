"""The SID value type returned by beam search (quantizer/residual.py:44-59
in the reference).  Quantizer fitting itself is offline tokenization and
out of scope for the serving path."""

from dataclasses import dataclass


@dataclass(frozen=True)
class SemanticId:
    """A per-level token sequence with its per-level vocabulary sizes."""

    tokens: tuple
    level_vocab_sizes: tuple

    def __post_init__(self):
        if len(self.tokens) != len(self.level_vocab_sizes) or not self.tokens:
            raise ValueError("tokens and level_vocab_sizes must be equal, nonzero length")
        for t, (tok, size) in enumerate(zip(self.tokens, self.level_vocab_sizes)):
            if not 0 <= tok < size:
                raise ValueError(f"token {tok} out of range [0, {size}) at level {t}")

    def __len__(self):
        return len(self.tokens)
