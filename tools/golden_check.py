#!/usr/bin/env python
"""Print the per-subset errors of a full-length GPU run against its oracle
golden (tests/test_gpu_golden.golden_report), e.g. under different
FDTD_* environment switches:  python tools/golden_check.py 2 32 [--golden-prec 32] [--form leapfrog]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

from test_gpu_golden import golden_report  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config", type=int)
ap.add_argument("prec", type=int)
ap.add_argument("--members", default="0")
ap.add_argument("--golden-prec", type=int, default=None)
ap.add_argument("--form", default="auto")
ap.add_argument("--tag", default="")
a = ap.parse_args()
rep, paths, n = golden_report(a.config, a.prec, tuple(int(m) for m in a.members.split(",")),
                              golden_prec=a.golden_prec, reduced_form=a.form)
print(json.dumps(dict(tag=a.tag, config=a.config, prec=a.prec, steps=n, paths=paths,
                      report={k: [float(f"{v[0]:.3e}"), float(f"{v[1]:.3e}")] for k, v in rep.items()})), flush=True)
