"""Which comparison of the TB jitter test differs, and where."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np
from parity import run_gpu
from sampled_state import random_state
from synth import scenario
from paper_1406_7042_b200 import prep
K = sys.argv[1] if len(sys.argv) > 1 else "2"
os.environ["FDTD_P2K"] = K
prob, _ = prep.build_problem(scenario("tiny2d_B", precision=32), precision=32)
prob = dict(prob, init={})
arrays, red_e, red_h = random_state(prob, seed=99)
start = dict(arrays=arrays, red_e=red_e, red_h=red_h, step=3)
n = 90
for chunks in ([30, 1, 59], [90], [1] * 10):
    nn = sum(chunks)
    os.environ.pop("FDTD_JITTER", None)
    ref = run_gpu(prob, nn, precision=32, chunks=chunks, start=start)
    for jit in ("0", "0", "700", "3000"):
        if jit != "0":
            os.environ["FDTD_JITTER"] = jit
        else:
            os.environ.pop("FDTD_JITTER", None)
        b = run_gpu(prob, nn, precision=32, chunks=chunks, start=start)
        diffs = {c: float(np.max(np.abs(ref["state"][c] - b["state"][c]))) for c in ref["state"]}
        de = float(np.max(np.abs(ref["red_e"] - b["red_e"])))
        dp = float(np.max(np.abs(ref["probes"] - b["probes"])))
        bad = {c: int(np.argmax(np.abs(ref["state"][c] - b["state"][c]))) for c in ref["state"] if diffs[c] > 0}
        print(f"K={K} chunks={chunks} jitter={jit}: state {diffs} red {de} probes {dp} first-bad-idx {bad}", flush=True)
