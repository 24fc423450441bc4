"""pipeplan.ordering → paper_2204_10562_b200.ordering (see pipeplan/__init__.py)."""
import sys as _sys

from paper_2204_10562_b200 import ordering as _m

_sys.modules[__name__] = _m
