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


def test_slab_plan_and_halo_exchange_world2():
    # NEXT-4 host logic on two gloo ranks: each rank builds its slab from the
    # SlabPlan, advances it one step at a time (the oracle's recursion stands in
    # for the kernels on CPU) and swaps its face planes with halo_exchange; the
    # gathered state equals the undecomposed oracle run
    r = _run_torchrun("""
        import sys
        import numpy as np
        import torch
        import torch.distributed as td
        sys.path.insert(0, ".")
        from paper_1406_7042_b200 import dist, prep
        from oracle import problem_step as ps
        from synth import scenario
        rank, world, local = dist.init(backend="gloo")
        scn = scenario("lossy3d", precision=64)
        prob, _ = prep.build_problem(scn, cache=False)
        plan = dist.SlabPlan(prob, world, cuts=(0, 6, 19))      # the source plane (k = 9) stays out of the overlap
        lp = plan.local_problem(rank)
        rec = ps.build(lp)
        E, H = ps.initial_state(rec, lp)
        Sl, plane = rec.S, plan.plane
        hc, hpos = rec.h_ids // Sl, rec.h_ids % Sl
        def sel(c, k):
            m = (hc == c) & (hpos // plane == k)
            return np.nonzero(m)[0], hpos[m] % plane
        faces = plan.faces(rank)
        n = 30
        for s in range(n):
            E, H, _, _ = ps.run(lp, 1, state=(E, H), start_step=s, rec=rec)
            send, recv = {}, {}
            for nb, k_send, k_ghost in faces:
                t = torch.zeros(len(dist.EXCHANGED) * plane, dtype=torch.float64)
                for q, c in enumerate(dist.EXCHANGED):
                    idx, pos = sel(c, k_send)
                    t[q * plane + torch.as_tensor(pos)] = torch.as_tensor(H[idx])
                send[nb], recv[nb] = t, torch.zeros_like(t)
            dist.halo_exchange(rank, faces, send, recv)
            for nb, k_send, k_ghost in faces:
                for q, c in enumerate(dist.EXCHANGED):
                    idx, pos = sel(c, k_ghost)
                    H[idx] = recv[nb][q * plane + torch.as_tensor(pos)].numpy()
        st, _, _ = ps.to_storage(rec, E, H)
        worst = 0.0
        Eg, Hg, _, recg = ps.run(prob, n)
        stg, _, _ = ps.to_storage(recg, Eg, Hg)
        for c in range(6):
            mine = plan.gather({rank: st.get(c, np.zeros(Sl))[None, :]})[0]
            k0, k1 = plan.own_lo[rank], plan.own_hi[rank]
            ref = stg.get(c, np.zeros(plan.S))
            d = np.abs(mine[k0 * plane:k1 * plane] - ref[k0 * plane:k1 * plane]).max()
            worst = max(worst, d / max(np.abs(ref).max(), 1e-300))
        t = torch.tensor([worst]); td.all_reduce(t, op=td.ReduceOp.MAX)
        if rank == 0:
            print("RESULT", float(t), plan.cuts)
        dist.finalize()
    """, timeout=400)
    assert r.returncode == 0, r.stderr[-3000:]
    line = [l for l in r.stdout.splitlines() if l.startswith("RESULT")][0]
    assert float(line.split()[1]) <= 1e-13
