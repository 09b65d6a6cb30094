from .index import SidIndex
from .residual import SemanticId

__all__ = ["SemanticId", "SidIndex"]
