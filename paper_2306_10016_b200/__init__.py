"""paper_2306_10016_b200 -- hybrid-dealiased convolution (arXiv 2306.10016) on B200.

The compute path is libhdconv.so (CUDA, sm_100a) behind the C ABI in
include/hdconv.h; `paper_2306_10016_b200.hdconv` is its ctypes binding.  Importing
`hdconv` without the built library raises: there is no CPU fallback.
"""
import importlib

__all__ = ["hdconv", "build"]


def __getattr__(name):
    if name in ("hdconv", "build"):
        return importlib.import_module(f"{__name__}.{name}")
    raise AttributeError(name)
