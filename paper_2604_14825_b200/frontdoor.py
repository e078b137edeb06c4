"""Front door: the reference's own upstream pipeline, unchanged.

The B200 backend keeps the reference's Python API surface for everything
upstream of the MA-tile IR: ``.te`` text ->
``frontend`` (tilecc/pipeline.py:37-43) -> ``run_autoscheduler``
(tilecc/autosched/scheduler.py:73) -> ``lower_seed`` (tilecc/pipeline.py:46-55)
-> MA module.  Only the executor behind it changes.  ``tilecc`` is imported
from the normal path or from ``baseline/_ref`` (the offline reference install).
"""

from __future__ import annotations

import os
import sys
from dataclasses import replace
from typing import Optional

from . import ma_ir
from .programs import PROGRAMS

_REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_REF_PATHS = (os.path.join(_REPO, "baseline", "_ref"), "/root/reference/pkg/src")


def import_tilecc():
    """Import the reference package (``tilecc``) or raise ImportError."""
    try:
        import tilecc  # noqa: F401
        return tilecc
    except ImportError:
        pass
    for p in _REF_PATHS:
        if os.path.isdir(os.path.join(p, "tilecc")) and p not in sys.path:
            sys.path.append(p)
            try:
                import tilecc  # noqa: F401
                return tilecc
            except ImportError:
                sys.path.remove(p)
    raise ImportError("tilecc (the reference front end) is not importable; install it into baseline/_ref")


def device_profile(**overrides):
    """The reference VirtualDevice with overrides (e.g. max_tile_elems=10**6)."""
    import_tilecc()
    from tilecc.ma.device import DEFAULT_DEVICE
    return replace(DEFAULT_DEVICE, **overrides) if overrides else DEFAULT_DEVICE


def compile_program(program: str, binding: dict, device=None, seed_index: int = 0,
                    assignment: Optional[dict] = None, options=None):
    """Run the reference pipeline; return (mirrored MA module, tilecc LoweredSeed, seeds).

    ``program`` is ``.te`` text or a key of ``programs.PROGRAMS``.
    """
    import_tilecc()
    from tilecc.autosched.scheduler import SchedulerOptions, run_autoscheduler
    from tilecc.pipeline import frontend, lower_seed

    text = PROGRAMS.get(program, program)
    device = device or device_profile()
    bound, base = frontend(text, binding)
    seeds = run_autoscheduler(base, device, options or SchedulerOptions())
    if not seeds:
        from .errors import UnsupportedMA
        raise UnsupportedMA("the auto-scheduler found no viable seeds")
    lw = lower_seed(base, seeds[seed_index].schedule, device, assignment)
    return ma_ir.from_tilecc(lw.ma), lw, seeds
