"""Build an A/B variant of libgvt.so with extra nvcc flags into ab/lib<name>.so (its objects under
ab/_build_<name>), for scripts/ab_matvec.py "lib=ab/lib<name>.so".
usage: python scripts/build_variant.py <name> -DS16_SCALE_ROWS=1 [...]"""
import importlib.util
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
spec = importlib.util.spec_from_file_location("_gvt_build", os.path.join(ROOT, "paper_2009_01054_b200", "build.py"))
b = importlib.util.module_from_spec(spec)
spec.loader.exec_module(b)
name, flags = sys.argv[1], sys.argv[2:]
os.makedirs(os.path.join(ROOT, "ab"), exist_ok=True)
print(b.build(extra_flags=flags, lib=os.path.join(ROOT, "ab", f"lib{name}.so"),
              build_dir=os.path.join(ROOT, "ab", f"_build_{name}")))
