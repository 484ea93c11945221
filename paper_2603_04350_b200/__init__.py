"""B200-native Exp-ParaDiag hot path (arXiv 2603.04350).

libexpd.so (csrc/, C-ABI include/expd.h) holds every kernel; expd.py is the ctypes
binding.  See DESIGN.md.
"""
from .expd import EXPORTS, Comm, ExpdError, HostComm, Plan, Problem, a2a_schedule, layout, load_library  # noqa: F401

__all__ = ["Plan", "Problem", "Comm", "HostComm", "ExpdError", "load_library", "layout", "a2a_schedule", "EXPORTS"]
