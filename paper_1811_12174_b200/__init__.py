"""paper_1811_12174_b200 -- PowerAI DDL's topology-aware gradient all-reduce (arXiv
1811.12174 §2.1), B200-native: libddl.so (hand-written sm_100a kernels, C ABI in
include/ddl.h) plus a thin ctypes binding (ddl.py).  No CPU fallback."""
from . import ddl  # noqa: F401
from .ddl import Comm, Loopback, init, local_reduce, parse_dims, DDLError  # noqa: F401
