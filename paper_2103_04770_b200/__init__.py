"""paper_2103_04770_b200 -- B200-native (sm_100a, FP64) hot path of the staggered FFT solver for
implicit-gradient ductile damage (Magri et al., arXiv 2103.04770).

The product is libfgd.so (C ABI, include/fgd.h, sources in csrc/).  `api.Context` and `_fgd`
are its thin Python binding.  Importing the package does not load the library (so that
`python -m paper_2103_04770_b200.build` works on a fresh tree); touching `Context`,
`FgdError` or `Material` loads it and fails loudly if it is missing -- there is no CPU fallback.
"""
__all__ = ["Context", "FgdError", "Material", "nccl_id", "loopback_id"]


def __getattr__(name):
    if name in __all__:
        from . import api
        return getattr(api, name)
    raise AttributeError(name)
