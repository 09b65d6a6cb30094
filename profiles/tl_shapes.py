"""tc_timeline.py's run() on level-sized products: pair tiles vs 128-wide
single-CTA tiles (A/B for the wave-quantisation tail at M = 16384)."""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.argv = ["x"]
exec(open(os.path.join(HERE, "tc_timeline.py")).read().split("for shape in")[0])
for shape in [(16384, 1024, 1024), (16384, 1024, 2048), (32768, 1024, 1024), (16384, 2048, 1024)]:
    for few in (0, 1):
        run(*shape, few=few)
