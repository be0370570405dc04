"""B200-native FFTrainer state-backup / failover-recovery path.

The product is libffx.so (sm_100a kernels + the C ABI in include/ffx.h) and
the C++ facade over it (facade/, the reference's ftsim API).  `ffx` is the
ctypes binding used by tests and bench.py; importing it without the built
library raises ImportError -- there is no CPU fallback.
"""
import os

PACKAGE_DIR = os.path.dirname(os.path.abspath(__file__))
REPO_ROOT = os.path.dirname(PACKAGE_DIR)
LIB_PATH = os.path.join(PACKAGE_DIR, "libffx.so")

__all__ = ["PACKAGE_DIR", "REPO_ROOT", "LIB_PATH"]
