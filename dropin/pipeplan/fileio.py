"""pipeplan.fileio → paper_2204_10562_b200.fileio (see pipeplan/__init__.py)."""
import sys as _sys

from paper_2204_10562_b200 import fileio as _m

_sys.modules[__name__] = _m
