"""Debug helper: one step from a random state, TMA stencil vs the cp.async one,
repeated; reports mismatching unknowns (i, j, k)."""
import os
import sys
sys.path.insert(0, os.getcwd())
import numpy as np
from synth import scenario
from paper_1406_7042_b200 import prep
from paper_1406_7042_b200.fdtd import Sim

name = sys.argv[1]
trials = int(sys.argv[2])
nsteps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
scn = scenario(name, precision=64)
prob, info = prep.build_problem(scn, precision=64)
prob["init"] = {}
nx, ny, nz = prob["n"]
rng = np.random.default_rng(0)


def run(no_tma, state):
    if no_tma:
        os.environ["FDTD_NO_TMA"] = "1"
    else:
        os.environ.pop("FDTD_NO_TMA", None)
    sim = Sim(prob, precision=64, graph_steps=0)
    for c in range(6):
        sim.set_state(c, state[c])
    sim.step(nsteps)
    sim.sync()
    out = [sim.get_state(c) for c in range(6)]
    sim.close()
    return out


S = (nx + 1) * (ny + 1) * (nz + 1)
tot = 0
for t in range(trials):
    state = [rng.standard_normal((1, S)) for _ in range(6)]
    a = run(True, state)
    b = run(False, state)
    for c in range(6):
        d = np.nonzero(a[c][0] != b[c][0])[0]
        if len(d):
            tot += 1
            i = d % (nx + 1); j = (d // (nx + 1)) % (ny + 1); k = d // ((nx + 1) * (ny + 1))
            print("trial", t, "comp", c, "n", len(d), "first", list(zip(i[:12].tolist(), j[:12].tolist(), k[:12].tolist())),
                  "maxdiff", float(np.abs(a[c][0] - b[c][0]).max()), flush=True)
print("trials with mismatch:", tot)
