"""Run bench.py against an experiment build: python tools/run_variant.py <tag> <bench args...>
(LIB_PATH -> paper_2010_03660_b200/libsten_<tag>.so; tag 'base' = the product library)."""
import os
import runpy
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2010_03660_b200 as sten  # noqa: E402

tag = sys.argv[1]
if tag != "base":
    sten.LIB_PATH = os.path.join(ROOT, "paper_2010_03660_b200", f"libsten_{tag}.so")
sys.argv = ["bench.py"] + sys.argv[2:]
os.chdir(ROOT)
runpy.run_path(os.path.join(ROOT, "bench.py"), run_name="__main__")
