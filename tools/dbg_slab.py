import sys, os, traceback
sys.path.insert(0, '.')
from synth import scenario
from paper_1406_7042_b200 import prep
from paper_1406_7042_b200.dist import SlabSim
for which, prec, slabs, cuts in (("lossy3d", 64, 3, None), ("lossy3d_b16", 32, 2, (0, 6, 9))):
    scn = scenario(which, precision=prec)
    prob, _ = prep.build_problem(scn, precision=prec)
    try:
        sl = SlabSim(prob, n_slabs=slabs, precision=prec, cuts=cuts)
        for s in range(5):
            for r, sim in sl.sims.items():
                sim.step(1); sim.sync(); print(which, "step", s, "rank", r, "ok", flush=True)
            for r in sl.sims:
                for nb, k_send, _ in sl.plan.faces(r):
                    sl._pack(r, nb, k_send, False); sl.sims[r].sync(); print(which, "pack", r, nb, k_send, "ok", flush=True)
            for r in sl.sims:
                for nb, _, _ in sl.plan.faces(r):
                    sl.buf[(r, nb, "recv")].copy_(sl.buf[(nb, r, "send")])
            for r in sl.sims:
                for nb, _, k_ghost in sl.plan.faces(r):
                    sl._pack(r, nb, k_ghost, True); sl.sims[r].sync(); print(which, "unpack", r, nb, k_ghost, "ok", flush=True)
    except Exception:
        traceback.print_exc()
