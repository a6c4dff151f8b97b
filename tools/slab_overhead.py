#!/usr/bin/env python
"""Cost of the per-step halo exchange on ONE GPU: config 3's grid (256^3, fp32)
advanced as 1 handle (graphs of 32 steps), as 1 handle stepped one step per call
(what SlabSim does), and as 2 / 4 slabs with the plane copies on the stream."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(steps=200):
    import torch
    from paper_1406_7042_b200 import prep
    from paper_1406_7042_b200.dist import SlabSim
    from paper_1406_7042_b200.fdtd import Sim
    from synth import scenario
    scn = scenario(3, precision=32)
    prob, _ = prep.build_problem(scn, precision=32)
    cells = 256 ** 3

    def timed(fn):
        fn(20); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(steps); e1.record(); torch.cuda.synchronize()
        return e0.elapsed_time(e1) / steps * 1e3

    out = {}
    s = Sim(prob, precision=32)
    for c, a in prob["init"].items():
        s.set_state(int(c), a)
    out["one handle, 32-step graphs"] = timed(s.step)
    out["one handle, one step per call"] = timed(lambda n: [s.step(1) for _ in range(n)])
    s.close()
    for n_slabs in (2, 4):
        sl = SlabSim(prob, n_slabs=n_slabs, precision=32)
        out[f"{n_slabs} slabs on one GPU (2-cell overlap, Hx/Hy planes copied every step)"] = timed(sl.step)
        sl.close()
    for k, v in out.items():
        print(f"{k}: {v:.1f} us per step, {cells / v / 1e3:.1f} Gcell/s")
    print(json.dumps(out))


if __name__ == "__main__":
    main()
