"""The six benchmark host programs of PAPER.md §V-B (L838-891)."""
from .hits_dl import DeepLearning, Hits
from .img_ml import Images, MLEnsemble
from .vec_bs import BlackScholes, Vec

PROGRAMS = {"vec": Vec, "bs": BlackScholes, "img": Images, "ml": MLEnsemble, "hits": Hits,
            "dl": DeepLearning}

__all__ = ["PROGRAMS", "Vec", "BlackScholes", "Images", "MLEnsemble", "Hits", "DeepLearning"]
