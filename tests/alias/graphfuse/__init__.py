"""Alias package `graphfuse` -> paper_2411_16127_b200 (test infrastructure).

The reference's own Python tests (proj/python/tests/test_smoke.py) do
`import graphfuse as gf`; putting tests/alias on sys.path makes that import
resolve to this repo's drop-in, exactly the one-line backend switch
INTEGRATION.md §2 describes for proj/python/graphfuse/__init__.py.
"""
import sys as _sys

import paper_2411_16127_b200 as _impl
from paper_2411_16127_b200 import *  # noqa: F401,F403
from paper_2411_16127_b200 import _core  # noqa: F401

_sys.modules[__name__ + "._core"] = _impl._core
__all__ = list(_impl.__all__)
