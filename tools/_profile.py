"""Point the package at the profiling build (tools/libternkit_b200_profile.so,
compiled with -DTK_PROFILE so the TK_CONV_* / TK_GEMM_* experiment knobs and
in-kernel timestamps exist).  Import this before anything loads the library;
the product library itself has no knobs and no override."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_2008_05101_b200 import _lib, build  # noqa: E402

_lib.LIB_PATH = build.build(profile=True)
