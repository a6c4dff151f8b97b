"""Debug helper: run a prepared scenario several times on the GPU, report
bitwise repeatability and the error against the oracle."""
import os
import sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, "tests")
import numpy as np
from synth import scenario
from paper_1406_7042_b200 import prep

name = sys.argv[1]
n = int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
gs = int(os.environ.get("GRAPH_STEPS", "32"))
scn = scenario(name, precision=64)
if os.environ.get("NBOX"):
    scn["boxes"] = scn["boxes"][:int(os.environ["NBOX"])]
prob, info = prep.build_problem(scn, precision=64)
from parity import run_gpu, run_oracle, compare
outs = []
for r in range(reps):
    g = run_gpu(prob, n, precision=64, graph_steps=gs)
    outs.append(g)
    print("rep", r, "checksum", [float(np.abs(g["state"][c]).sum()) for c in sorted(g["state"])], flush=True)
for r in range(1, reps):
    same = all(np.array_equal(outs[0]["state"][c], outs[r]["state"][c]) for c in outs[0]["state"])
    print("rep", r, "bitwise equal to rep 0:", same)
if os.environ.get("ORACLE", "1") == "1":
    o = run_oracle(prob, n)
    for r in range(reps):
        print("rep", r, "err", compare(prob, outs[r], o))
