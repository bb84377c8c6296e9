"""Does TMA (tensor-map) streaming work from the mapped pinned-host arena?
Runs the hot-shape parity with TTKV_SLOW_TC=1 (host arena) in a child
process so a fault cannot poison other work."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["TTKV_SLOW_TC"] = "1"
import test_gpu_parity as P
import paper_2604_19769_b200 as T
w = P.run_parity(T, S=3, G=4, d=128, B=128, l_fast=512, ctx=5000, steps=4)
print("host-arena TMA slow TC parity ok, worst rel err", w)
