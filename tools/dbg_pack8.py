import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2010_03660_b200 as sten
from test_gpu_sr import _sweep_case
got, dots, ref, rh = _sweep_case(sten, sys.argv[1], (37, 19, 5), tiling=(16, 3, 2, 5, 8), seed=4)
print("ok")
