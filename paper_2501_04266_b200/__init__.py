"""paper_2501_04266_b200: B200-native hierarchical ZeRO++ data-parallel hot path.

  hz      ctypes binding of libhz.so (include/hz.h) — the product path; importing
          it without the built library raises ImportError (no CPU fallback).
  synth   seeded synthetic inputs (no method arithmetic).
  build   nvcc build of libhz.so for sm_100a.
"""

__all__ = ["hz", "synth", "build"]


def __getattr__(name):
    if name in __all__:
        import importlib
        return importlib.import_module(f"{__name__}.{name}")
    raise AttributeError(name)
