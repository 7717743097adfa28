"""Build experiment variants of libsten.so (compile-time switches) as
paper_2010_03660_b200/libsten_<tag>.so, then rebuild the product library.  Usage:
  python tools/build_variants.py tag1='-DX=1 -DY=2' tag2='-DX=2' ...
Run them with tools/run_variant.py (the bench with LIB_PATH pointed at a variant)."""
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2010_03660_b200 import build as b  # noqa: E402

for arg in sys.argv[1:]:
    tag, flags = arg.split("=", 1)
    os.environ["STEN_NVCC_EXTRA"] = flags
    b.FLAGS[:] = [f for f in b.FLAGS if not f.startswith("-DSTEN_")] + flags.split()
    b.build(force=True)
    shutil.copy(b.LIB, os.path.join(ROOT, "paper_2010_03660_b200", f"libsten_{tag}.so"))
    print("built", tag, flags)
b.FLAGS[:] = [f for f in b.FLAGS if not f.startswith("-DSTEN_")]
os.environ["STEN_NVCC_EXTRA"] = ""
b.build(force=True)
print("product library rebuilt")
