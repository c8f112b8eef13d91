"""korch-b200: B200-native kernel-orchestrated primitive-graph executor (Korch, arXiv 2406.09465).

The hot path lives in libkorch.so (C ABI in include/korch.h) and the sm_100a
kernels it generates; this package is the thin Python binding plus the
host-side BLP selection.  The binding is imported on first use, so
`paper_2406_09465_b200.build` works before the library exists; every other entry
point fails loudly (ImportError) when libkorch.so is missing.
"""
_API = ("Context", "KorchGraph", "torch_inputs")
_SELECT = ("INF", "operator_aligned", "singletons", "solve_blp")
_MODULES = ("tunedb", "select", "dist")
__all__ = list(_API + _SELECT)


def __getattr__(name):
    if name in _API:
        from . import api
        return getattr(api, name)
    if name in _MODULES:
        import importlib
        return importlib.import_module(f"{__name__}.{name}")
    if name in _SELECT:
        from . import select
        return getattr(select, name)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
