"""Slab decomposition along z with a per-step halo exchange (SURVEY §8(e),
NEXT-4; paper_1406_7042_b200/dist.py SlabSim, fdtd_plane_device of the C ABI)
on ONE GPU: the slabs are separate handles stepped one after the other, their
face planes copied on the stream.  Every owned unknown is updated by the same
kernel arithmetic from the same values, so the decomposed run equals the
undecomposed one bit for bit (states and probe series)."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

pytestmark = pytest.mark.gpu

from synth import scenario  # noqa: E402


@pytest.mark.parametrize("which,prec,slabs,cuts", [
    ("config3_small", 32, 2, None), ("config3_small", 64, 3, None), ("lossy3d", 32, 2, (0, 6, 19)),
    ("lossy3d", 64, 3, None), ("lossy3d_b16", 32, 2, (0, 6, 9))])
def test_slab_run_bitwise_equals_single_domain(which, prec, slabs, cuts):
    from paper_1406_7042_b200 import prep
    from paper_1406_7042_b200.dist import SlabSim
    from paper_1406_7042_b200.fdtd import Sim
    scn = scenario(which, precision=prec)
    prob, _ = prep.build_problem(scn, precision=prec)
    n = 45
    ref = Sim(prob, precision=prec, graph_steps=0)
    for c, a in (prob.get("init") or {}).items():
        ref.set_state(int(c), a)
    ref.step(n); ref.sync()
    want = [ref.get_state(c) for c in range(6)]
    want_p = ref.probe()
    ref.close()
    sl = SlabSim(prob, n_slabs=slabs, precision=prec, cuts=cuts)
    sl.step(n); sl.sync()
    for c in range(6):
        got = sl.get_state(c)
        assert np.linalg.norm(want[c]) > 0 or c >= 3 or which != "config3_small"
        assert np.array_equal(got, want[c]), (c, np.abs(got - want[c]).max())
    if want_p.size:
        assert np.array_equal(sl.probe(), want_p)
    sl.close()


def test_plane_device_argument_checks():
    from paper_1406_7042_b200 import prep
    from paper_1406_7042_b200.fdtd import FdtdError, Sim
    import torch
    scn = scenario("config3_small", precision=32)
    prob, _ = prep.build_problem(scn, precision=32)
    sim = Sim(prob, precision=32)
    buf = torch.zeros((prob["n"][1] + 1) * (prob["n"][0] + 1), dtype=torch.float32, device="cuda")
    with pytest.raises(FdtdError):
        sim.plane_device(6, 0, buf.data_ptr(), False)
    with pytest.raises(FdtdError):
        sim.plane_device(3, prob["n"][2] + 1, buf.data_ptr(), False)
    # round trip of one plane
    src = torch.arange(buf.numel(), dtype=torch.float32, device="cuda")
    sim.plane_device(4, 7, src.data_ptr(), True)
    sim.plane_device(4, 7, buf.data_ptr(), False)
    sim.sync()
    assert torch.equal(buf, src)
    sim.close()
