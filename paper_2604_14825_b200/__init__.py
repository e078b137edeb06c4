"""B200-native backend and runtime for the Nautilus (tilecc) MA-tile path.

Public API (mirrors the reference seams):
  execute_ma(module, inputs, device=None, precision=None, ...)   ~ tilecc.ma.interp.interpret_ma
  run_pipeline(ma, inputs, device=None, precision=None)          ~ tilecc.pipeline.run_pipeline
  recognize(module)                                               MA kernels -> KernelSpecs
"""

__version__ = "0.1.0"

from .recognize import AttentionSpec, GemmChainSpec, recognize  # noqa: F401


def __getattr__(name):
    # torch-dependent entry points are imported lazily
    if name in ("execute_ma", "run_pipeline", "ExecReport"):
        from . import executor
        return getattr(executor, name)
    raise AttributeError(name)
