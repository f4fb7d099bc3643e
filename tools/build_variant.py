#!/usr/bin/env python
"""Compile-time A/B builds: libhps_b200.<name>.so with extra -D defines, loaded
by the package when HPSB_LIB_VARIANT=<name> (then tools/ab.sh compares them on
one box).

  python tools/build_variant.py <name> [DEFINE[=VALUE] ...]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2210_08804_b200 import _build  # noqa: E402

if __name__ == "__main__":
    print(_build.build(verbose=False, variant=sys.argv[1], defines=tuple(sys.argv[2:])))
