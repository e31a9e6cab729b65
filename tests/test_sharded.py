"""Sharded lane: vertices 1-D partitioned over ranks, the
policy slices exchanged after every improvement pass, the rest replicated.

CPU (gloo, world size 2): the exchange step of TorchComm -- in-place
chunked all-gather of the policy arrays and max-reduction of the region
flags -- on CPU tensors, in two processes.
GPU: W shards driven in one process (LocalComm) reproduce the unsharded
solve bit for bit (policy, keys, iteration counts), including ranks that own
no vertex; TorchComm over NCCL runs the same loop at world size 1.
"""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1111_0627_b200 as P
from helpers import case_arrays, golden_cases

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, n, chunk, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1111_0627_b200.sharded import TorchComm
    comm = TorchComm()
    full = chunk * world
    policy = [torch.full((full,), -1, dtype=torch.int32) for _ in range(2)]
    policy.append(torch.full((full,), -1.0, dtype=torch.float64))
    lo = rank * chunk
    for k, t in enumerate(policy):
        t[lo:lo + chunk] = torch.arange(lo, lo + chunk) * (k + 1) + rank
    flags = [torch.zeros(5, dtype=torch.int32), torch.zeros(5, dtype=torch.int32)]
    flags[0][rank] = 1
    flags[1][4] = rank + 7
    comm.exchange_arrays(policy, flags, chunk)
    out_q.put((rank, [t.tolist() for t in policy], [f.tolist() for f in flags]))
    dist.destroy_process_group()


def test_torchcomm_exchange_gloo_cpu():
    world, chunk = 2, 6
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, chunk * world, chunk, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict((r, (pol, fl)) for r, pol, fl in (q.get(timeout=120) for _ in procs))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        pol, fl = res[r]
        for k in range(3):
            want = [float(i * (k + 1) + i // chunk) if k == 2 else i * (k + 1) + i // chunk
                    for i in range(chunk * world)]
            assert pol[k] == want
        assert fl[0] == [1, 1, 0, 0, 0]
        assert fl[1] == [0, 0, 0, 0, 8]


def _single(source, objective):
    g = source if isinstance(source, P.Graph) else None
    s = P.Session(g, P.SolveOptions(objective=objective)) if g else \
        P.Session.generated(source, P.SolveOptions(objective=objective))
    return s.solve(), s.values()


def _sharded(source, objective, world):
    from paper_1111_0627_b200.sharded import LocalComm, ShardSession, solve_sharded
    shards = [ShardSession(source, P.SolveOptions(objective=objective), r, world)
              for r in range(world)]
    sols = solve_sharded(shards, LocalComm())
    return sols, [sh.values() for sh in shards]


def _same(a, va, b, vb):
    assert a.has_cycle == b.has_cycle
    if not a.has_cycle:
        return
    assert (a.mu_exact, a.mu, a.cycle_vertices) == (b.mu_exact, b.mu, b.cycle_vertices)
    assert (a.stats.outer_iters, a.stats.spf_passes) == (b.stats.outer_iters, b.stats.spf_passes)
    for k in ("key_num", "lam_num", "lam_den", "fval", "succ_vertex"):
        assert np.array_equal(va[k], vb[k]), k


SOURCES = {
    "uniform": lambda: P.Generator("uniform", n=100_000, deg=8, seed=17),
    "powerlaw": lambda: P.Generator("powerlaw", n=60_000, deg=4, dmax=30_000, seed=18),
    "server10": lambda: P.generate_model(P.server_scenario(), 10),
}


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(SOURCES))
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("objective", ["min", "max"])
def test_local_shards_match_single(name, world, objective):
    src = SOURCES[name]()
    a, va = _single(src, objective)
    sols, vals = _sharded(src, objective, world)
    for b, vb in zip(sols, vals):
        _same(a, va, b, vb)


@pytest.mark.gpu
def test_local_shards_golden_cases():
    # tiny graphs: most ranks own nothing; float weights included
    for case in golden_cases()[::7]:
        s, d, w = case_arrays(case)
        g = P.build_graph(case["n"], (s, d, w))
        if len(w) and np.abs(w).max() >= 2 ** 31:
            # 64-bit weights: the sharded lanes refuse loudly (wide lane is 1-GPU)
            with pytest.raises(P.UnsupportedError, match="sharded"):
                _sharded(g, "min", 2)
            continue
        for objective in ("min", "max"):
            a, va = _single(g, objective)
            sols, vals = _sharded(g, objective, 4)
            for b, vb in zip(sols, vals):
                _same(a, va, b, vb)


NCCL_WORLD1 = r"""
import os, sys, torch, torch.distributed as dist
sys.path.insert(0, sys.argv[1])
import paper_1111_0627_b200 as P
from paper_1111_0627_b200.sharded import ShardSession, TorchComm, solve_sharded
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=sys.argv[2])
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1)
spec = P.Generator("uniform", n=50_000, deg=8, seed=5)
sh = ShardSession(spec, P.SolveOptions(), 0, 1)
(sol,) = solve_sharded([sh], TorchComm())
ref = P.Session.generated(spec).solve()
assert (sol.mu_exact, sol.cycle_vertices, sol.stats.spf_passes) == \
    (ref.mu_exact, ref.cycle_vertices, ref.stats.spf_passes)
dist.destroy_process_group()
print("ok", sol.mu_exact, sol.stats.launches)
"""


@pytest.mark.gpu
def test_torchcomm_nccl_world1():
    r = subprocess.run([sys.executable, "-c", NCCL_WORLD1, ROOT, str(_free_port())],
                       capture_output=True, text=True, timeout=300)
    if r.returncode != 0:
        tail = [l for l in r.stderr.splitlines() if "Error" in l or "error" in l][-5:]
        raise AssertionError("\n".join(tail) + "\n" + r.stderr[-1500:])
    assert r.stdout.strip().splitlines()[-1].startswith("ok"), r.stdout


def _gloo_gpu_worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1111_0627_b200.sharded import ShardSession, TorchComm, solve_sharded
    try:
        res = []
        for spec in (P.Generator("uniform", n=40_000, deg=8, seed=23),
                     P.Generator("powerlaw", n=30_000, deg=4, dmax=20_000, seed=24)):
            for objective in ("min", "max"):
                sh = ShardSession(spec, P.SolveOptions(objective=objective), rank, world)
                (sol,) = solve_sharded([sh], TorchComm())
                vals = sh.values()
                ref = P.Session.generated(spec, P.SolveOptions(objective=objective))
                rs = ref.solve()
                rv = ref.values()
                same = (sol.mu_exact == rs.mu_exact and sol.cycle_vertices == rs.cycle_vertices
                        and sol.stats.spf_passes == rs.stats.spf_passes
                        and all(np.array_equal(vals[k], rv[k]) for k in ("key_num", "succ_vertex")))
                res.append((str(spec.kind), objective, same, str(sol.mu_exact)))
        out_q.put((rank, res, None))
    except Exception as e:  # reported by the parent
        out_q.put((rank, None, repr(e)))
    dist.destroy_process_group()


@pytest.mark.gpu
def test_torchcomm_two_processes_one_gpu():
    """Two ranks (processes) share the one GPU of this box and exchange over
    gloo: the full multi-process sharded loop, with real device kernels."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_gpu_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
    for rank, res, err in got:
        assert err is None, (rank, err)
        assert all(same for _, _, same, _ in res), (rank, res)


def _fused(source, objective, world, solves=2):
    from paper_1111_0627_b200.sharded import ShardSession, connect_local, solve_fused
    shards = [ShardSession(source, P.SolveOptions(objective=objective), r, world)
              for r in range(world)]
    connect_local(shards)
    out = None
    for _ in range(solves):  # re-solving exercises the persistent barrier epochs
        out = solve_fused(shards)
    return out, [sh.values() for sh in shards]


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(SOURCES))
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("objective", ["min", "max"])
def test_fused_shards_match_single(name, world, objective, monkeypatch):
    """The fused lane (policy pushed into peer replicas inside the kernel,
    cross-rank barriers on system-scope atomics): `world` ranks as concurrent
    cooperative kernels sharing this box's GPU, each on 1/world of the SMs,
    reproduce the unsharded solve bit for bit."""
    src = SOURCES[name]()
    a, va = _single(src, objective)
    monkeypatch.setenv("OCM_GRID", str(148 * 4 // world))
    sols, vals = _fused(src, objective, world)
    for b, vb in zip(sols, vals):
        _same(a, va, b, vb)
        assert b.stats.launches == 1  # the whole sharded solve in one launch per rank


def _fused_ipc_worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                      OCM_GRID=str(148 * 4 // world))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1111_0627_b200.sharded import ShardSession, connect_torch, solve_fused
    try:
        res = []
        for spec in (P.Generator("uniform", n=40_000, deg=8, seed=23),
                     P.Generator("powerlaw", n=30_000, deg=4, dmax=20_000, seed=24)):
            for objective in ("min", "max"):
                sh = ShardSession(spec, P.SolveOptions(objective=objective), rank, world)
                connect_torch(sh)  # descriptors over torch.distributed, buffers via CUDA IPC
                dist.barrier()
                (sol,) = solve_fused([sh])
                ref = P.Session.generated(spec, P.SolveOptions(objective=objective))
                rs = ref.solve()
                same = (sol.mu_exact == rs.mu_exact and sol.cycle_vertices == rs.cycle_vertices
                        and sol.stats.spf_passes == rs.stats.spf_passes
                        and np.array_equal(sh.values()["key_num"], ref.values()["key_num"]))
                res.append((str(spec.kind), objective, same))
                dist.barrier()  # peers unmap before the next shard frees its buffers
                del sh
        out_q.put((rank, res, None))
    except Exception as e:  # reported by the parent
        out_q.put((rank, None, repr(e)))
    dist.destroy_process_group()


@pytest.mark.gpu
def test_fused_two_processes_ipc():
    """The fused lane across processes, as on a multi-GPU box: each rank maps
    its peers' replicas through CUDA IPC handles exchanged over
    torch.distributed, and the two kernels meet at system-scope barriers.
    Here both processes share the box's one GPU."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fused_ipc_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
    for rank, res, err in got:
        assert err is None, (rank, err)
        assert res and all(same for _, _, same in res), (rank, res)


@pytest.mark.gpu
@pytest.mark.parametrize("objective", ["min", "max"])
def test_fused_shards_with_tma_staged_pass(objective, monkeypatch):
    """The fused lane's per-rank improvement range through the staged pass."""
    src = P.Generator("uniform", n=50_000, deg=8, seed=21)
    a, va = _single(src, objective)
    monkeypatch.setenv("OCM_STAGED", "1")
    monkeypatch.setenv("OCM_GRID", str(148 * 4 // 2))
    sols, vals = _fused(src, objective, 2)
    for b, vb in zip(sols, vals):
        _same(a, va, b, vb)


@pytest.mark.gpu
@pytest.mark.parametrize("objective", ["min", "max"])
def test_fused_and_sharded_with_connected_bitmap(objective, monkeypatch):
    """The replicated keep/attach phases of both sharded lanes with the
    connected-vertex bitmap forced on (by default only from 2^24 vertices)."""
    src = P.Generator("powerlaw", n=50_000, deg=2, dmax=5000, wlo=-50, whi=50, seed=22)
    a, va = _single(src, objective)
    monkeypatch.setenv("OCM_CBITS_MIN_N", "0")
    monkeypatch.setenv("OCM_GRID", str(148 * 4 // 2))
    sols, vals = _fused(src, objective, 2)
    for b, vb in zip(sols, vals):
        _same(a, va, b, vb)
    sols, vals = _sharded(src, objective, 3)
    for b, vb in zip(sols, vals):
        _same(a, va, b, vb)
