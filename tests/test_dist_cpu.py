"""N > 1 host logic on CPU with torch.distributed (gloo, world_size 2): the slab halo plan
exported by libmhd (mhd_halo_plan, the same function mhd_step uses to post its NCCL
send/recv) is executed with gloo point-to-point on numpy slabs in libmhd's storage layout
[z + 2][f][y][x]; every ghost plane must equal the neighbour's interior plane bitwise, i.e.
the decomposition reproduces the periodic (or outflow-edge) ghost fill of the global array
(SPEC.md:102-110 halo_exchange examples).  Also: the 128-byte NCCL unique
id of rank 0 reaches every rank through the torch.distributed broadcast (bench.py's path)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, nz_glob, periodic, ghost, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2510_24175_b200 import mhd
        nv, ny, nx = 9, 4, 5
        rng = np.random.default_rng(1234)
        G = rng.standard_normal((nz_glob, nv, ny, nx))  # global interior, storage order [z][f][y][x]
        nz = nz_glob // world
        z0 = rank * nz
        g = ghost
        S = np.full((nz + 2 * g, nv, ny, nx), np.nan)
        S[g:nz + g] = G[z0:z0 + nz]
        plan = mhd.halo_plan(rank, world, nz_glob, periodic, ghost)
        reqs = []
        for peer, kind, first, count in plan:  # posting order of the plan
            if peer < 0:
                continue
            buf = torch.from_numpy(S[first:first + count])
            if kind == 0:
                reqs.append(dist.isend(buf.contiguous(), dst=peer))
            else:
                reqs.append((dist.irecv(buf, src=peer), buf))
        for r in reqs:
            if isinstance(r, tuple):
                r[0].wait()
            else:
                r.wait()
        ok = True
        pairs = [(m, z0 - g + m) for m in range(g)] + [(nz + g + m, z0 + nz + m) for m in range(g)]
        for sp, zglob in pairs:
            if 0 <= zglob < nz_glob or periodic:
                if not np.array_equal(S[sp], G[zglob % nz_glob]):
                    ok = False
            else:
                ok = ok and np.isnan(S[sp]).all()  # domain edge: filled locally (outflow copy)
        ids = [mhd.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(ids, src=0)
        q.put((rank, ok, ids[0]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("periodic,ghost", [(True, 2), (False, 2), (True, 3)])
def test_two_rank_halo_plan_with_gloo(periodic, ghost):
    from paper_2510_24175_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, 12, periodic, ghost, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _ in res), res
    assert res[0][2] == res[1][2] and len(res[0][2]) == 128


def test_halo_plan_shapes():
    from paper_2510_24175_b200 import build, mhd
    build.build()
    # P = 1: no peers; P = 4 periodic: ring neighbours; P = 4 outflow: no wrap at the ends
    assert all(r[0] == -1 for r in mhd.halo_plan(0, 1, 64))
    assert [r[0] for r in mhd.halo_plan(0, 4, 64)] == [1, 3, 3, 1]
    assert [r[0] for r in mhd.halo_plan(0, 4, 64, False)] == [1, -1, -1, 1]
    assert [r[0] for r in mhd.halo_plan(3, 4, 64, False)] == [-1, 2, 2, -1]
    assert mhd.halo_plan(1, 4, 64)[0] == (2, 0, 16, 2) and mhd.halo_plan(1, 4, 64)[3] == (2, 1, 18, 2)
    with pytest.raises(mhd.MhdError):
        mhd.halo_plan(0, 3, 64)  # 3 does not divide 64
    assert mhd.halo_plan(1, 4, 64, True, 3)[0] == (2, 0, 16, 3) and mhd.halo_plan(1, 4, 64, True, 3)[3] == (2, 1, 19, 3)
    with pytest.raises(mhd.MhdError):
        mhd.halo_plan(0, 32, 64, True, 3)  # slab of 2 planes < ghost width 3


def test_reference_arm_under_torchrun_two_ranks():
    """bench.py --impl reference launched the driver's way (torchrun, 2 ranks, 127.0.0.1): rank 0
    alone prints one JSON line with impl "reference", the other rank exits 0 without work."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--impl", "reference",
           "--gpus", "2", "--steps", "1", "--warmup", "0"]
    r = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["e2e"]["h2d_bytes_per_step"] == 0


def _simulate_plans(world, nz_glob, periodic, ghost):
    """Execute every rank's halo plan with NCCL's pairing rule (the k-th send from a to b meets
    the k-th receive on b from a) on numpy slabs; return the slabs and the global array."""
    from paper_2510_24175_b200 import mhd
    rng = np.random.default_rng(world * 100 + nz_glob + ghost)
    G = rng.standard_normal((nz_glob, 3, 2, 2))
    nz = nz_glob // world
    S = []
    for r in range(world):
        s = np.full((nz + 2 * ghost, 3, 2, 2), np.nan)
        s[ghost:ghost + nz] = G[r * nz:(r + 1) * nz]
        S.append(s)
    sends, recvs = {}, {}
    for r in range(world):
        for peer, kind, first, count in mhd.halo_plan(r, world, nz_glob, periodic, ghost):
            if peer < 0:
                continue
            key = (r, peer) if kind == 0 else (peer, r)
            (sends if kind == 0 else recvs).setdefault(key, []).append((r, first, count))
    assert sends.keys() == recvs.keys()
    for key in sends:
        assert len(sends[key]) == len(recvs[key]), key
        for (src, f0, c0), (dst, f1, c1) in zip(sends[key], recvs[key]):
            assert c0 == c1
            S[dst][f1:f1 + c1] = S[src][f0:f0 + c0]
    return S, G, nz


@pytest.mark.parametrize("world", [1, 2, 3, 4, 5, 8])
@pytest.mark.parametrize("ghost", [2, 3, 4])
@pytest.mark.parametrize("periodic", [True, False])
def test_halo_plan_all_rank_counts(world, ghost, periodic):
    """Up to the 8 ranks of one node, every ghost depth the stages use (2 PLM, 3 WENO-Z, 4 CT with
    WENO-Z): executing all plans together fills every ghost plane with the global neighbour plane
    (periodic wrap) or leaves it to the local outflow copy at the domain ends."""
    from paper_2510_24175_b200 import build
    build.build()
    nz_glob = world * max(ghost, 4)
    S, G, nz = _simulate_plans(world, nz_glob, periodic, ghost)
    for r in range(world):
        z0 = r * nz
        for m in range(ghost):
            for sp, zg in ((m, z0 - ghost + m), (nz + ghost + m, z0 + nz + m)):
                if world > 1 and (periodic or 0 <= zg < nz_glob):
                    assert np.array_equal(S[r][sp], G[zg % nz_glob]), (r, sp, zg)
                elif world > 1:
                    assert np.isnan(S[r][sp]).all()


def test_nccl_bench_script_runs_on_gloo(tmp_path):
    """tools/nccl_bench.py's halo / allreduce schedule, run with the gloo backend on 2 CPU ranks."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", "29541",
                        os.path.join(root, "tools", "nccl_bench.py"), "--backend", "gloo", "--sizes", "32", "--iters", "3",
                        "--warmup", "1"], capture_output=True, text=True, timeout=300, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][0])
    assert d["world"] == 2 and d["halo"][0]["message_MB"] == 2 * 9 * 32 * 32 * 8 / 1e6 and d["allreduce_16B"]["us"] > 0
