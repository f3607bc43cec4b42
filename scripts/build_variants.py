#!/usr/bin/env python
"""A/B builds of libbbot.so with extra nvcc flags (own object dir + library under
paper_2209_00315_b200/variants/, git-ignored, shipped to the GPU box by gpurun); select one
at run time with BBOT_LIB=<path>.

    python scripts/build_variants.py minb6=-DBBOT_LAP_MINB=6 minb7=-DBBOT_LAP_MINB=7
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "paper_2209_00315_b200"))
import _build  # noqa: E402

VDIR = os.path.join(ROOT, "paper_2209_00315_b200", "variants")
for arg in sys.argv[1:]:
    name, flags = arg.split("=", 1)
    lib = os.path.join(VDIR, f"libbbot_{name}.so")
    _build.build(lib=lib, build_dir=os.path.join(VDIR, "build_" + name), extra=flags.split(","))
    print(lib)
