"""Phase timeline of the persistent 2-D kernel (FDTD_P2DBG=1: globaltimer
stamps of tile 0, an interface tile and reduced CTA 0 for steps 100-107,
printed by the library to stderr)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
os.environ["FDTD_P2DBG"] = "1"
from paper_1406_7042_b200 import prep
from paper_1406_7042_b200.fdtd import Sim
from synth import scenario
scn = scenario(2, precision=32)
prob, _ = prep.build_problem(scn, precision=32)
sim = Sim(prob, precision=32)
sim.step(200)
sim.sync()
sim.close()
