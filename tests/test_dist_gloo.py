"""The multi-rank host logic of bench.py (replicas, max-over-ranks timing,
unit sums) on world size 2 with the gloo backend, on CPU."""
import os
import socket
import subprocess
import sys
import textwrap

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run_torchrun(script, nproc=2, timeout=240):
    path = os.path.join(ROOT, "gpurun_out", f"_gloo_{os.getpid()}.py")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    with open(path, "w") as f:
        f.write(textwrap.dedent(script))
    env = dict(os.environ, PYTHONPATH=ROOT, CUDA_VISIBLE_DEVICES="")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), path]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, env=env, cwd=ROOT)
    os.remove(path)
    return r


def test_reduce_max_sum_and_replicas_world2():
    r = _run_torchrun("""
        import os
        from paper_1406_7042_b200 import dist
        rank, world, local = dist.init(backend="gloo")
        assert world == 2
        t = dist.reduce_max(1.0 + rank)
        u = dist.reduce_sum(10.0 * (rank + 1))
        dist.barrier()
        if rank == 0:
            print("RESULT", t, u, dist.replica_scale(0), dist.replica_scale(1))
        dist.finalize()
    """)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [l for l in r.stdout.splitlines() if l.startswith("RESULT")][0]
    _, t, u, s0, s1 = line.split()
    assert float(t) == 2.0 and float(u) == 30.0
    assert float(s0) == 1.0 and float(s1) == 1.125


def test_bench_reference_arm_world2_rank0_only():
    # --impl reference under torchrun: rank 0 alone times the oracle and prints
    r = _run_torchrun("""
        import sys
        sys.argv = ["bench.py", "--impl", "reference", "--config", "3", "--steps", "1", "--warmup", "0",
                    "--ref-steps", "1"]
        sys.path.insert(0, ".")
        import bench
        from synth import scenario
        # shrink the workload for the CPU test: monkeypatch the config builder
        orig = bench.build_workload
        def small(config, precision, rank=0):
            from paper_1406_7042_b200 import prep
            scn = scenario("tiny3d", precision=32, n_steps=4)
            prob, info = prep.build_problem(scn, cache=False)
            return scn, prob, info
        bench.build_workload = small
        sys.exit(bench.main(sys.argv[1:]))
    """, timeout=400)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    import json
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["cores"] == 1
