"""B200-native fused RK4 finite-difference stencil library (arXiv:1410.1764's hot path).

``capi`` is the ctypes binding of include/chemora.h (same names as the C entry points);
``grid`` holds the torch-backed convenience handles.  Importing either fails loudly when
the CUDA library has not been built -- there is no CPU fallback on the product path.
(The package itself imports lazily so that ``python -m paper_1410_1764_b200.build`` can
run before the library exists.)
"""

__all__ = ["capi", "grid", "Grid", "LocalSlabs", "ChemoraError"]


def __getattr__(name):
    import importlib
    if name in ("capi", "grid"):
        return importlib.import_module(f"{__name__}.{name}")
    if name in ("Grid", "LocalSlabs"):
        return getattr(importlib.import_module(f"{__name__}.grid"), name)
    if name == "ChemoraError":
        return importlib.import_module(f"{__name__}.capi").ChemoraError
    raise AttributeError(name)
