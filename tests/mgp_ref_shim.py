"""pytest plugin: run the reference's own, unmodified test files with the B200 shim active.

Loaded with ``-p mgp_ref_shim`` by tests/test_reference_unmodified_gpu.py, in a child
pytest whose rootdir is the unmodified reference test directory (baseline/_ref/tests) and
whose ``megores`` is the unmodified reference package (baseline/_ref/megores).  At
configure time -- before the reference test modules import anything -- it calls
``shim.install(megores, offspring=True)``: megores' resamplers (M/__init__.py:12-28,
M/resample.py:431-455), ``ancestors_to_offspring`` and ``apply_ancestors`` then run the
B200 kernels.  Every routed call is counted; at session end the counts, the reference
package's path and the shared objects mapped into the process are written to
``$MGP_REF_SHIM_REPORT`` (JSON), which the parent test asserts on.
"""

from __future__ import annotations

import functools
import json
import os

_COUNTS: dict = {}


def _counting(name, fn):
    @functools.wraps(fn)
    def wrapper(*a, **k):
        _COUNTS[name] = _COUNTS.get(name, 0) + 1
        return fn(*a, **k)

    return wrapper


def pytest_configure(config):
    import megores

    from paper_2109_13504_b200 import _lib, shim

    _lib.lib()  # fail loudly here if the CUDA library is missing
    saved = shim.install(megores, offspring=True)
    # wrap what was installed so the parent can see the routed calls
    import importlib
    import sys

    for (modname, name) in saved:
        mod = sys.modules[modname]
        setattr(mod, name, _counting(name, getattr(mod, name)))
    config._mgp_ref = {"megores": os.path.dirname(megores.__file__),
                       "patched": sorted({n for (_, n) in saved})}
    importlib.invalidate_caches()


def pytest_unconfigure(config):
    out = os.environ.get("MGP_REF_SHIM_REPORT")
    if not out:
        return
    maps = []
    try:
        with open("/proc/self/maps") as f:
            maps = sorted({ln.split()[-1] for ln in f if ln.rstrip().endswith(".so")})
    except OSError:
        pass
    rep = dict(getattr(config, "_mgp_ref", {}))
    rep["calls"] = _COUNTS
    rep["libmgp_mapped"] = [m for m in maps if m.endswith("libmgp.so")]
    with open(out, "w") as f:
        json.dump(rep, f)
