"""Debug helper: rewrite a problem so every instance is its own block."""
import copy
import numpy as np


def split_instances(prob):
    p = copy.deepcopy(prob)
    newb, base = [], []
    for b in prob["blocks"]:
        base.append(len(newb))
        for i in range(int(b["n_inst"])):
            nb = dict(b)
            nb["n_inst"] = 1
            newb.append(nb)
    p["blocks"] = newb
    itf = p["interface"]
    blk = np.asarray(itf["block"]); ins = np.asarray(itf["inst"])
    itf["block"] = np.array([base[b] + i for b, i in zip(blk, ins)], dtype=np.asarray(itf["block"]).dtype)
    itf["inst"] = np.zeros_like(ins)
    for pr in p["probes"]:
        if pr.get("kind", 0) in (1, 2):
            pr["block"] = base[pr["block"]] + pr.get("inst", 0)
            pr["inst"] = 0
    return p
