import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def _ensure_built():
    """Build libddl.so (nvcc, sm_100a; no GPU needed) if this checkout has not built it yet."""
    import subprocess
    lib = os.path.join(ROOT, "paper_1811_12174_b200", "libddl.so")
    src = os.path.join(ROOT, "paper_1811_12174_b200", "csrc")
    newest = max(os.path.getmtime(os.path.join(src, f)) for f in os.listdir(src))
    newest = max(newest, os.path.getmtime(os.path.join(ROOT, "include", "ddl.h")))
    if not os.path.exists(lib) or os.path.getmtime(lib) < newest:
        subprocess.run(["bash", os.path.join(ROOT, "build.sh")], check=True, cwd=ROOT,
                       stdout=subprocess.DEVNULL)


def pytest_configure(config):
    _ensure_built()
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: longer CPU test")
