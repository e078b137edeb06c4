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


B200_PROFILE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "b200.device")
B200_BACKENDS = ("sm100a",)


def b200_device(**overrides):
    """The B200 ``VirtualDevice``: ``b200.device`` parsed by the reference's own
    ``load_device`` (tilecc/ma/device.py:59-100), with optional overrides."""
    import_tilecc()
    from tilecc.ma.device import load_device
    dev = load_device(B200_PROFILE)
    return replace(dev, **overrides) if overrides else dev


def b200_options(**kw):
    """``SchedulerOptions`` restricted to the sm100a backend (tilecc/autosched/scheduler.py:35-40, 79):
    a profile file can add a backend but not drop the defaults, so the seed fan-out
    is cut here (6 seeds -> 2)."""
    import_tilecc()
    from tilecc.autosched.scheduler import SchedulerOptions
    return SchedulerOptions(backends=B200_BACKENDS, **kw)


def resolve_device(device):
    """None -> the reference default profile; "b200" -> ``b200_device()``; a path -> that
    profile file; a VirtualDevice -> itself.  Returns (device, default SchedulerOptions)."""
    import_tilecc()
    from tilecc.autosched.scheduler import SchedulerOptions
    if device is None or device == "default":
        return device_profile(), SchedulerOptions()
    if device == "b200":
        return b200_device(), b200_options()
    if isinstance(device, str):
        from tilecc.ma.device import load_device
        return load_device(device), SchedulerOptions()
    return device, SchedulerOptions()


def device_profile(**overrides):
    """The reference VirtualDevice with overrides (e.g. max_tile_elems=10**6)."""
    import_tilecc()
    from tilecc.ma.device import DEFAULT_DEVICE
    return replace(DEFAULT_DEVICE, **overrides) if overrides else DEFAULT_DEVICE


def compile_program(program: str, binding: dict, device=None, seed_index: int = 0,
                    assignment: Optional[dict] = None, options=None, upstream_fixes: bool = False):
    """Run the reference pipeline; return (mirrored MA module, tilecc LoweredSeed, seeds).

    ``program`` is ``.te`` text or a key of ``programs.PROGRAMS``; ``device`` is
    None (reference default), ``"b200"`` (``b200.device`` + sm100a-only options),
    a profile path or a VirtualDevice; ``upstream_fixes`` schedules with
    ``upstream.apply()`` (scale / mask after the sum).
    """
    import_tilecc()
    from tilecc.autosched.scheduler import SchedulerOptions, run_autoscheduler
    from tilecc.pipeline import frontend, lower_seed

    text = PROGRAMS.get(program, program)
    device, default_opts = resolve_device(device)
    bound, base = frontend(text, binding)
    if upstream_fixes:
        from . import upstream
        with upstream.fixed():
            seeds = run_autoscheduler(base, device, options or default_opts)
    else:
        seeds = run_autoscheduler(base, device, options or default_opts)
    if not seeds:
        from .errors import UnsupportedMA
        raise UnsupportedMA("the auto-scheduler found no viable seeds")
    lw = lower_seed(base, seeds[seed_index].schedule, device, assignment)
    return ma_ir.from_tilecc(lw.ma), lw, seeds
