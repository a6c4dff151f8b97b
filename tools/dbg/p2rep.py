import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, "tests")
import numpy as np
from synth import scenario
from paper_1406_7042_b200 import prep
from parity import run_gpu
name = sys.argv[1]; prec = int(sys.argv[2]); n = int(sys.argv[3]); reps = int(sys.argv[4])
scn = scenario(name, precision=prec); prob, info = prep.build_problem(scn, precision=prec)
os.environ["FDTD_PERSIST"] = "0"
ref = run_gpu(prob, n, precision=prec)
del os.environ["FDTD_PERSIST"]
bad = 0
for r in range(reps):
    b = run_gpu(prob, n, precision=prec)
    d = max(float(np.abs(ref["state"][c] - b["state"][c]).max()) for c in ref["state"])
    bad += d > 0
    print("rep", r, "maxdiff", d, flush=True)
print("mismatching reps", bad, "of", reps)
