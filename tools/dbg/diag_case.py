"""Debug helper: per-part GPU-vs-oracle errors for a prepared scenario."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
sys.path.insert(0, "tests")
from parity import run_gpu, run_oracle, reduced_member, block_shapes
from synth import scenario
from paper_1406_7042_b200 import prep

name = sys.argv[1]
form = sys.argv[2] if len(sys.argv) > 2 else None
scn = scenario(name, precision=64)
if os.environ.get("NBOX"):
    scn["boxes"] = scn["boxes"][:int(os.environ["NBOX"])]
if os.environ.get("NOSHEETS"):
    scn["pec_sheets"] = []
prob, info = prep.build_problem(scn, precision=64)
if os.environ.get("SPLIT"):
    sys.path.insert(0, "tools/dbg")
    from split_inst import split_instances
    prob = split_instances(prob)
print("blocks", [(b["qe"], b["qh"], b["n_inst"], len(b.get("if_rows", b.get("interface", [])) or [])) for b in prob["blocks"]])
print("sources", len(prob["sources"]["unknown"]), "probes", len(prob["probes"]))
STEPS = [int(x) for x in os.environ.get("DIAG_STEPS", "1,2,3,5,20").split(",")]
for n in STEPS:
    kw = {} if form is None else dict(reduced_form=form)
    g = run_gpu(prob, n, precision=64, **kw)
    o = run_oracle(prob, n)
    rec = o["rec"]
    S = rec.S
    for lab, ids, vec in (("E", rec.e_ids, o["E"][:len(rec.e_ids)]), ("H", rec.h_ids, o["H"][:len(rec.h_ids)])):
        comp, pos = ids // S, ids % S
        gg = np.empty(len(ids))
        for c in np.unique(comp):
            m = comp == c
            gg[m] = g["state"][int(c)][0][pos[m]]
        d = np.abs(gg - vec)
        k = int(np.argmax(d))
        print(n, lab, "err", d.max(), "scale", np.abs(vec).max(), "at comp", comp[k], "pos", pos[k],
              "n_bad", int((d > 1e-10 * max(np.abs(vec).max(), 1e-300)).sum()))
        if d.max() > 1e-10 * np.abs(vec).max():
            bad = np.argsort(-d)[:8]
            nx, ny, nz = prob["n"]
            itf_u = set(np.asarray(prob["interface"]["unknown"]).tolist()) if prob.get("interface") else set()
            src_u = set(np.asarray(prob["sources"]["unknown"]).tolist())
            for b in bad:
                ps_ = int(pos[b]); i = ps_ % (nx + 1); j = (ps_ // (nx + 1)) % (ny + 1); k = ps_ // ((nx + 1) * (ny + 1))
                u = int(comp[b]) * S + ps_
                print("    comp", comp[b], "ijk", (i, j, k), "gpu", gg[b], "ora", vec[b], "itf" if u in itf_u else "",
                      "src" if u in src_u else "", "mat", int(np.asarray(prob["mat_id"]).ravel()[ps_]))
    sh = block_shapes(prob)
    for side, ref in (("e", o["red_e"]), ("h", o["red_h"])):
        gr = reduced_member(g["red_" + side], sh, 1, 0, side)
        print(n, "red", side, np.abs(gr - ref).max(), np.abs(ref).max())
    if g["probes"] is not None and len(g["probes"]):
        print(n, "probes", np.abs(g["probes"][:, :, 0] - o["probes"]).max(), np.abs(o["probes"]).max())
