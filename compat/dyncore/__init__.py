"""`dyncore` -> paper_1701_03980_b200 alias.

Put `compat/` ahead of the reference core on PYTHONPATH and the reference's
own scripting frontend (pkg/frontend/src/dyngraph/__init__.py, which does
`import dyncore` / `from dyncore import ops`) runs unchanged on the B200
backend:

    PYTHONPATH=/root/repo/compat:<reference>/pkg/frontend/src python my_script.py

The alias makes `dyncore` *be* the package (same module object), and
registers its submodules under the reference's names (dyncore.ops,
dyncore.graph, ...), so `isinstance` checks and module-level state are shared.
"""

import importlib
import os
import sys

_ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if _ROOT not in sys.path:
    sys.path.insert(0, _ROOT)

_pkg = importlib.import_module("paper_1701_03980_b200")
for _sub in ("arena", "builders", "errors", "graph", "ops", "parallel", "params", "tensor", "trainers"):
    sys.modules[f"dyncore.{_sub}"] = importlib.import_module(f"paper_1701_03980_b200.{_sub}")
sys.modules[__name__] = _pkg
