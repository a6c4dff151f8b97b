"""Small runs of every kernel family for compute-sanitizer (racecheck /
synccheck / memcheck): the persistent 2-D kernel with its fp32 LL exchange
(tiny2d_B; and the temporal-blocking variant), the TMA tile stencil
(config3_small), the batched tile stencil + leap-frog GEMMs + the tcgen05 GEMM
(tiny4, B = 16), the fused cluster GEMM (tiny5 with N >= 4 columns via 2
instances x 2 members is not available -> tiny4 fused, B = 4)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np  # noqa: E402

from paper_1406_7042_b200 import prep  # noqa: E402
from paper_1406_7042_b200.fdtd import Sim  # noqa: E402
from synth import scenario  # noqa: E402


def run(name, prec, n, **kw):
    scn = scenario(name, precision=prec)
    prob, _ = prep.build_problem(scn, precision=prec)
    batch16 = kw.pop("batch16", False)
    if batch16:
        w = np.asarray(prob["sources"]["wave"])
        amp = np.linspace(1.0, -1.3, 16)
        prob = dict(prob, sources=dict(prob["sources"], wave=w[:, :, :1] * amp[None, None, :]), batch=16)
    sim = Sim(prob, precision=prec, **kw)
    for c, a in (prob.get("init") or {}).items():
        sim.set_state(int(c), a)
    sim.step(n)
    sim.sync()
    p = sim.probe()
    print(name, prec, kw, "paths", sim.path(), "probe norm", float(np.linalg.norm(p)), flush=True)
    sim.close()


which = sys.argv[1] if len(sys.argv) > 1 else "all"
if which in ("all", "p2d"):
    run("tiny2d_B", 32, 24)
    os.environ["FDTD_P2K"] = "2"
    run("tiny2d_B", 32, 24)
    os.environ.pop("FDTD_P2K")
    run("tiny2d_B", 64, 12)
if which in ("all", "3d"):
    run("config3_small", 32, 6)
    os.environ["FDTD_FORCE_SKINNY"] = "1"      # the tcgen05 S_E h~ GEMM on the small guide
    run("tiny4", 32, 6, batch16=True, reduced_form="leapfrog")
    os.environ.pop("FDTD_FORCE_SKINNY")
    run("tiny4", 32, 6, reduced_form="fused")
    run("tiny5", 64, 6)
