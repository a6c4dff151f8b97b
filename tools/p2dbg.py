import os, sys
sys.path.insert(0, os.getcwd())
os.environ["FDTD_P2DBG"] = "1"
from synth import scenario
from paper_1406_7042_b200 import prep
from paper_1406_7042_b200.fdtd import Sim
scn = scenario(2, precision=32); prob, info = prep.build_problem(scn, precision=32)
sim = Sim(prob, precision=32)
sim.step(200); sim.sync()
sim.step(200); sim.sync()
sim.close()
