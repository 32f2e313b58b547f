"""B200-native (sm_100a) coarsening level of arXiv 2605.20497.

The product is libhgp.so (C-ABI in include/hgp.h); ``hgp`` is its thin Python
binding. Import is lazy so that CPU-only environments can load the package
metadata; any compute call without the built extension or a GPU raises.
"""
import importlib

__all__ = ["hgp"]


def __getattr__(name):
    if name == "hgp":
        return importlib.import_module(__name__ + ".hgp")
    raise AttributeError(name)
