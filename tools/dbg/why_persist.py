import os, sys
sys.path.insert(0, os.getcwd())
os.environ["FDTD_VERBOSE"]="1"
from synth import scenario
from paper_1406_7042_b200 import prep
from paper_1406_7042_b200.fdtd import Sim
scn=scenario(2, precision=32); prob,info=prep.build_problem(scn, precision=32)
import numpy as np
itf=prob["interface"]; rp=np.asarray(itf["rowptr"]); print("max terms", np.diff(rp).max(), "n rows", len(rp)-1)
sim=Sim(prob, precision=32); sim.step(10); sim.sync(); print("launches", sim.launch_count()); sim.close()
