import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, "tests")
import numpy as np
from synth import scenario
from paper_1406_7042_b200 import prep
from parity import run_gpu
name = sys.argv[1] if len(sys.argv) > 1 else "tiny2d_B"
prec = int(sys.argv[2]) if len(sys.argv) > 2 else 32
n = int(sys.argv[3]) if len(sys.argv) > 3 else 5
scn = scenario(name, precision=prec); prob, info = prep.build_problem(scn, precision=prec)
os.environ["FDTD_PERSIST"] = "0"
a = run_gpu(prob, n, precision=prec)
del os.environ["FDTD_PERSIST"]
os.environ["FDTD_VERBOSE"] = "1"
b = run_gpu(prob, n, precision=prec)
print("launches", a["launches"], b["launches"])
nx, ny = prob["n"][:2]
for c in a["state"]:
    d = np.abs(a["state"][c] - b["state"][c])[0]
    k = np.argsort(-d)[:5]
    print(c, d.max(), [(int(q % (nx + 1)), int(q // (nx + 1)), float(d[q])) for q in k])
print("red", np.abs(a["red_e"] - b["red_e"]).max(), np.abs(a["red_h"] - b["red_h"]).max())
itf = prob["interface"]; print("itf unknown sample", [(int(u % ((nx+1)*(ny+1))) % (nx+1), int(u % ((nx+1)*(ny+1))) // (nx+1)) for u in np.asarray(itf["unknown"])[:4]])
src = prob["sources"]; S = (nx+1)*(ny+1); print("src", [(int(u % S) % (nx+1), int(u % S)//(nx+1)) for u in np.asarray(src["unknown"])])
