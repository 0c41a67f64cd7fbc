"""The six benchmark host programs of PAPER.md §V-B (L838-891)."""
from .vec_bs import BlackScholes, Vec

PROGRAMS = {"vec": Vec, "bs": BlackScholes}

__all__ = ["PROGRAMS", "Vec", "BlackScholes"]
