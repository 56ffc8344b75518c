"""Route an existing ``megores`` installation's hot path through the B200 kernels.

    import megores
    from paper_2109_13504_b200 import shim
    shim.install(megores)        # megores.megopolis(...) now runs on the GPU

``megores`` binds its public names at import (M/__init__.py:12-28) while
``make_resampler`` resolves ``metropolis``/``megopolis``/... from
``megores.resample`` globals at call time (M/resample.py:441-454), so both
namespaces are patched.  Host inputs keep returning ``np.int64`` ancestors.
``traffic=True`` also routes the transaction model (``comparison_indices``,
``trace_algorithm``, ``traffic_report``, ``count_transactions``) in every module that bound
it: ``megores``, ``megores.resample``, ``megores.warpsim`` and ``megores.bench``.
"""

from __future__ import annotations

from . import metrics as _metrics
from . import resample as _r

PATCHED = {
    "metropolis": _r.metropolis,
    "metropolis_c1": _r.metropolis_c1,
    "metropolis_c2": _r.metropolis_c2,
    "megopolis": _r.megopolis,
    "multinomial": _r.multinomial,
    "systematic_improved": _r.systematic_improved,
}


def install(megores_module, offspring: bool = False, traffic: bool = False):
    """Patch ``megores`` and its submodules in place; returns the originals."""
    import importlib

    mods = [megores_module, importlib.import_module(megores_module.__name__ + ".resample")]
    saved = {}
    names = dict(PATCHED)
    if offspring:
        names["ancestors_to_offspring"] = _r.ancestors_to_offspring
        names["apply_ancestors"] = _r.apply_ancestors
    if traffic:
        from . import warpsim as _w

        names.update(comparison_indices=_r.comparison_indices, trace_algorithm=_w.trace_algorithm,
                     traffic_report=_w.traffic_report, count_transactions=_w.count_transactions)
        for sub in (".warpsim", ".bench"):
            try:
                mods.append(importlib.import_module(megores_module.__name__ + sub))
            except ImportError:
                pass
    for name, fn in names.items():
        for mod in mods:
            if hasattr(mod, name):
                saved[(mod.__name__, name)] = getattr(mod, name)
                setattr(mod, name, fn)
    return saved


def uninstall(megores_module, saved) -> None:
    import sys

    for (modname, name), fn in saved.items():
        setattr(sys.modules[modname], name, fn)


__all__ = ["install", "uninstall", "PATCHED", "_metrics"]
