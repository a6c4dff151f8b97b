"""One persistent 2-D launch of config 2 (fp32), for ncu: python tools/p2prof.py [steps]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from paper_1406_7042_b200 import prep
from paper_1406_7042_b200.fdtd import Sim
from synth import scenario
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
scn = scenario(2, precision=32)
prob, _ = prep.build_problem(scn, precision=32)
sim = Sim(prob, precision=32)
sim.step(n)
sim.sync()
print("paths", sim.path())
sim.close()
