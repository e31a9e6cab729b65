"""Benchmark: policy-iteration throughput of the B200 optimal-cycle-mean solver.

One step = one full time-to-OCM solve (policy iteration from the initial
policy until no policy edge changes) for the minimum AND the maximum cycle
mean of the workload graph, resident in HBM.

metric: edges/s per policy iteration = intra-region edges x improvement
passes / device time, summed over ranks (weak scaling: every rank solves its
own seeded instance -- round 1 runs replicas).

Workloads (--config, BASELINE.json "configs", 1-based):
  1  uniform 10^4 vertices, out-degree 4 (the reference's CPU-runnable case)
  2  uniform 10^6 vertices, out-degree 8 -- the default (the metric's config)
  3  client/server state space, 19 clients (1.05*10^7 states, 2.0*10^8 edges;
     the reference's generate_model scenario beyond its 5*10^6-state bound)
  4  power-law out-degree graph, 6.4*10^7 vertices, ~1.0*10^9 edges
  5  uniform 2.5*10^8 vertices, out-degree 8 (2*10^9 edges)
Graphs 1, 2, 4, 5 are generated directly in HBM (bit-identical to the host
generator the checkers use); 3 is generated on the host and uploaded.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--config C]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "policy-iteration edges/s (time-to-OCM, min+max cycle mean)"
UNIT = "edges/s"
L2_FLUSH_BYTES = 512 << 20  # > 126 MB L2
SEED = 1111_0627

CONFIGS = {
    1: dict(kind="uniform", n=10_000, deg=4, desc="uniform random digraph n=10^4 out-degree 4 weights "
                                                 "1..100 (BASELINE configs[0])"),
    2: dict(kind="uniform", n=1_000_000, deg=8, desc="uniform random digraph n=10^6 out-degree 8 "
                                                     "weights 1..100 (BASELINE configs[1])"),
    3: dict(kind="model", clients=19, desc="client/server state space (reference server scenario, "
                                           "19 clients, BFS-numbered; BASELINE configs[2])"),
    4: dict(kind="powerlaw-hubs", n=64_000_000, deg=8, dmax=1 << 20,
            desc="power-law degree digraph n=6.4*10^7: out-degree min(2^20, floor(8/sqrt(u))), "
                 "in-degree tail exponent 3 too (hub targets), ~1.0*10^9 edges, weights 1..100 "
                 "(BASELINE configs[3])"),
    5: dict(kind="uniform", n=250_000_000, deg=8, desc="uniform random digraph n=2.5*10^8 "
                                                       "out-degree 8 weights 1..100 (BASELINE configs[4])"),
}
# The reference arm and cpu_baseline solve the workload graph itself; for the
# two configs whose graph the reference cannot hold or solve in minutes on the
# host (10^9 and 2*10^9 edges) they solve the same generator at n = 10^6,
# and say so in "config" / "sample".
REF_SAMPLE = {4: dict(n=1_000_000), 5: dict(n=1_000_000)}

def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=None, choices=sorted(CONFIGS),
                    help="BASELINE config (default: 2 on one GPU, 4 -- the 10^9-edge power-law "
                         "graph north_star shards -- on several)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-single-baseline", action="store_true",
                    help="N > 1: skip rank 0's single-GPU run of the same graph after the timed region")
    ap.add_argument("--lane", default=None, choices=["replicas", "sharded", "fused"],
                    help="replicas: every rank solves its own graph (weak scaling, the driver's "
                         "run); sharded: all ranks solve one graph, vertices 1-D partitioned, "
                         "policy all-gathered by NCCL between launches; fused: the same inside one "
                         "launch per rank, policy pushed into peer memory (strong scaling, "
                         "DESIGN.md §7). Default: fused when several GPUs are used")
    return ap.parse_args()


def resolve_defaults(a, world):
    if a.config is None:
        a.config = 2 if world == 1 else 4
    if a.lane is None:
        a.lane = "replicas" if world == 1 else "fused"
    return a


def self_launch(a):
    """`bench.py --gpus N` without a torchrun environment: start N ranks on
    this node with torch.distributed.run (127.0.0.1 rendezvous) and return
    their exit status. Refuses N beyond the visible GPUs unless
    OCM_BENCH_SHARE_GPU=1 maps several ranks onto one device (tests)."""
    n = a.gpus
    if a.impl == "b200" and os.environ.get("OCM_BENCH_SHARE_GPU") != "1":
        import torch
        have = torch.cuda.device_count()
        if have < n:
            sys.stderr.write(f"bench.py: --gpus {n} but only {have} GPU(s) are visible\n")
            return 2
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node",
           str(n), "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def config(a, world):
    c = CONFIGS[a.config]
    out = {"workload": c["desc"] + ", min+max cycle mean per step", "config_index": a.config,
           "weights": [1, 100], "seed": SEED, "objectives": ["min", "max"],
           "parallelism": f"replicas x{world}" if world > 1 else "1 gpu",
           "l2": "flushed between steps (512 MiB write)"}
    out.update({k: v for k, v in c.items() if k not in ("desc",)})
    return out


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region
    (B200_PROFILING.md clocks line): NVML polled every 2 ms from a thread
    (the timed region of config 2 is ~100 ms, shorter than nvidia-smi's
    start-up), falling back to `nvidia-smi -lms 50` where NVML is missing."""

    HW = 0x8        # nvmlClocksEventReasonHwSlowdown
    HW_THERMAL = 0x40
    SW_THERMAL = 0x20
    SW_POWER = 0x4

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []
        self.samples = []  # (sm_mhz, reasons bitmask)
        self.max_mhz = None
        self.nvml = None
        self.stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.nvml = (pynvml, h)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.nvml = None
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.3)  # let nvidia-smi start before the timed region
        except OSError:
            self.proc = None
        return self

    def _poll(self):
        pynvml, h = self.nvml
        while not self.stop.is_set():
            try:
                mhz = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                try:
                    rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                except AttributeError:
                    rs = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                self.samples.append((mhz, rs))
            except Exception:
                pass
            time.sleep(0.002)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        self.stop.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        elif self.nvml:
            self.t.join(timeout=1)

    def summary(self):
        sm, mx, reasons = [], 0, set()
        if self.nvml:
            for mhz, rs in self.samples:
                sm.append(float(mhz))
                for bit, nm in ((self.HW, "hw_slowdown"), (self.HW_THERMAL, "hw_thermal_slowdown"),
                                (self.SW_THERMAL, "sw_thermal_slowdown"),
                                (self.SW_POWER, "sw_power_cap")):
                    if rs & bit:
                        reasons.add(nm)
            mx = float(self.max_mhz or 0)
            src = "nvml (2 ms polling)"
        else:
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            for ln in self.lines:
                parts = [p.strip() for p in ln.split(",")]
                if len(parts) < 6:
                    continue
                try:
                    sm.append(float(parts[0]))
                    mx = max(mx, float(parts[1]))
                except ValueError:
                    continue
                for nm, val in zip(names, parts[2:]):
                    if val.lower() == "active":
                        reasons.add(nm)
            src = "nvidia-smi -lms 50"
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm), "source": src}


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def gather_peak(n):
    """Measured random 8-byte gather throughput (scripts/micro/gather.cu on
    this pool's B200, profiles/micro_gather_r01.log): ~210 G/s while the
    gathered array is L2-resident (<= 64 MB), ~40 G/s once it is HBM-resident
    (>= 1 GB); linear in between is not claimed, so 256 MB-class arrays use
    the measured 70 G/s point."""
    b = 8 * n
    if b <= (126 << 20):  # fits the 126 MB L2 (measured at 8-64 MB)
        return 2.1e11, "measured: L2-resident random gather, 8 MB-64 MB arrays"
    if b <= (256 << 20):
        return 7.0e10, "measured: random gather, 256 MB array"
    return 4.0e10, "measured: HBM-resident random gather, 1-8 GB arrays"


def ncu_traffic(cfg):
    """DRAM bytes per k_solve launch from the committed ncu --set full summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "solve_traffic.json")) as f:
            return json.load(f).get(str(cfg), {}).get("dram_bytes_per_launch")
    except Exception:
        return None


def algorithmic_bytes(stats):
    """Algorithmic bytes of one solve: every improvement pass
    streams each intra-region edge's 8 B {target, weight} record and gathers
    its head's 8 B key (16 B/edge) and touches 28 B per vertex (row 4,
    region 4, incumbent edge/head/weight 12, key 8); every policy iteration
    then reads each vertex's policy head and weight (8 B) and writes its key
    (8 B) to determine the values (16 B/vertex)."""
    imp = 16 * stats.m_solved + 28 * stats.n_solved
    return stats.spf_passes * imp + stats.outer_iters * 16 * stats.n_solved, imp


def build_graph_host(a, P):
    c = CONFIGS[a.config]
    if c["kind"] == "model":
        return P.generate_model(P.server_scenario(), c["clients"], max_states=1 << 31)
    return P.generate(P.Generator(c["kind"], n=c["n"], deg=c["deg"], dmax=c.get("dmax", 0),
                                  wlo=1, whi=100, seed=SEED))


def reference_workload(cfg):
    """(spec, sampled): the graph the reference solves for config `cfg`."""
    c = dict(CONFIGS[cfg])
    sampled = cfg in REF_SAMPLE
    c.update(REF_SAMPLE.get(cfg, {}))
    return c, sampled


def oracle_graph(c):
    """The workload graph from the checkers' bit-identical generators
    (oracle/, test infrastructure) -- the reference arm never imports the
    product package."""
    import oracle as O
    if c["kind"] == "model":
        return O.generate_model("server", c["clients"])
    if c["kind"] == "uniform":
        s, d, w = O.generate_uniform(c["n"], c["deg"], 1, 100, SEED)
    else:
        s, d, w = O.generate_powerlaw(c["n"], c["deg"], c["dmax"], 1, 100, SEED,
                                      hubs={"powerlaw": 0, "powerlaw-hubs": 1, "powerlaw-web": 3}[c["kind"]])
    return c["n"], s, d, w


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def reference_solves(cfg, steps, warmup, threads):
    """The reference's CPU solver (oracle/_ref: the unmodified proj/src
    compiled in place, lane `howard` = run_howard_seq, proj/src/solve.cpp:43,
    the reference CLI's default) on the workload graph, one min + one max
    solve per step. The graph is built once (ocm::build_graph); the solves of
    all steps run concurrently on `threads` host threads (ctypes releases the
    GIL; ocm::solve only reads the graph), so the value is the reference's
    throughput with the host's cores in use; time-to-OCM is the mean wall time
    of one ocm::solve call among them. Edges are counted as on the device:
    intra-region edges x improvement passes."""
    from concurrent.futures import ThreadPoolExecutor

    import oracle as O
    c, sampled = reference_workload(cfg)
    n, s, d, w = oracle_graph(c)
    intra = _intra_edges(n, s, d)
    g = O.RefGraph(n, s, d, w)
    m = len(s)
    del s, d, w
    # each concurrent solve holds O(n + m) state of its own: bound the
    # concurrency for the 10^8-edge graphs
    threads = max(1, min(threads, 2 * max(1, steps), 4 if m > 50_000_000 else threads))
    objs = ("min", "max")
    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(lambda o: g.solve("howard", o), [o for _ in range(warmup) for o in objs]))
        t0 = time.perf_counter()
        res = list(ex.map(lambda o: g.solve("howard", o), [o for _ in range(steps) for o in objs]))
        wall = time.perf_counter() - t0
    edges = sum(intra * r.spf_passes for r in res)
    per = {o: [r for r, oo in zip(res, objs * steps) if oo == o] for o in objs}
    what = (f"server scenario {c['clients']} clients" if c["kind"] == "model"
            else f"{c['kind']} n={c['n']} deg={c['deg']}")
    if sampled:
        what += f" (the config's generator at n={c['n']}: the full graph does not fit the host)"
    else:
        what += " (the full workload graph)"
    return {
        "value": edges / wall, "wall_s": wall, "cores": threads, "m_intra": intra,
        "time_to_ocm_s": {o: sum(r.solve_ms for r in per[o]) / len(per[o]) / 1e3 for o in objs},
        "policy_iterations": {o: per[o][0].spf_passes for o in objs},
        "mu": {o: f"{per[o][0].mu_num}/{per[o][0].mu_den}" for o in objs},
        "config": dict(c, sampled=sampled),
        "sample": f"{what}, {steps} step(s) of min+max (2*{steps} ocm::solve calls of the "
                  f"reference's default lane 'howard', run_howard_seq, proj/src/solve.cpp:43) on "
                  f"{threads} concurrent host threads; value = intra-region edges x passes / wall "
                  f"time of those calls (graph built once beforehand)",
    }


_INTRA = {}


def _intra_edges(n, s, d):
    """Edges inside non-trivial SCCs (what an improvement pass streams)."""
    key = (n, len(s))
    if key not in _INTRA:
        import numpy as np
        from scipy.sparse import csr_matrix
        from scipy.sparse.csgraph import connected_components
        g = csr_matrix((np.ones(len(s), np.int8), (s.astype(np.int64), d.astype(np.int64))),
                       shape=(n, n))
        _, lab = connected_components(g, directed=True, connection="strong")
        size = np.bincount(lab)
        self_loop = np.zeros(n, bool)
        self_loop[s[s == d]] = True
        nontriv = (size[lab] > 1) | self_loop
        _INTRA[key] = int(np.count_nonzero((lab[s] == lab[d]) & nontriv[s]))
    return _INTRA[key]


def run_reference(a, world, rank):
    """--impl reference: rank 0 alone times the reference's CPU solver on
    this arm's config; other ranks exit without work."""
    if rank != 0:
        return
    r = reference_solves(a.config, a.steps, a.warmup, host_threads())
    cfg = config(a, 1)
    if r["config"]["sampled"]:
        cfg.update(n=r["config"]["n"], sampled_from_n=CONFIGS[a.config]["n"],
                   workload=cfg["workload"] + f" -- SAMPLE: the same generator at "
                                              f"n={r['config']['n']}")
    cfg["parallelism"] = f"{r['cores']} host threads (concurrent solves)"
    line = {"impl": "reference", "metric": METRIC, "value": r["value"], "unit": UNIT,
            "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": r["wall_s"] * 1e3 / a.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic (seeded generator, oracle/ copy bit-identical to the product's)",
            "config": cfg, "time_to_ocm_s": r["time_to_ocm_s"],
            "policy_iterations": r["policy_iterations"], "mu": r["mu"],
            "cpu_baseline": {"value": r["value"], "unit": UNIT, "cores": r["cores"],
                             "kind": "reference", "sample": r["sample"]},
            "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def make_sessions(a, P, rank, local):
    c = CONFIGS[a.config]
    opts = {o: P.SolveOptions(objective=o, device=local) for o in ("min", "max")}
    if c["kind"] == "model":
        g = build_graph_host(a, P)
        return g, {o: P.Session(g, opts[o]) for o in opts}
    spec = P.Generator(c["kind"], n=c["n"], deg=c["deg"], dmax=c.get("dmax", 0), wlo=1, whi=100,
                       seed=SEED + rank)
    return spec, {o: P.Session.generated(spec, opts[o]) for o in opts}


def single_gpu_same_config(a, P, local, flush, steps=2):
    """Rank 0 alone: the single-GPU session lane on the sharded run's graph,
    one warm-up and `steps` timed min+max steps (CUDA events, L2 flushed)."""
    import torch
    c = CONFIGS[a.config]
    if c["kind"] == "model":
        g = build_graph_host(a, P)
        sess = {o: P.Session(g, P.SolveOptions(objective=o, device=local)) for o in ("min", "max")}
    else:
        spec = P.Generator(c["kind"], n=c["n"], deg=c["deg"], dmax=c.get("dmax", 0), wlo=1,
                           whi=100, seed=SEED)
        sess = {o: P.Session.generated(spec, P.SolveOptions(objective=o, device=local))
                for o in ("min", "max")}
    ms, edges = 0.0, 0
    for i in range(steps + 1):
        for o in ("min", "max"):
            flush.fill_(1)
            torch.cuda.synchronize()
            sol = sess[o].solve()
            if i:
                ms += sol.stats.device_ms
                edges += sol.stats.m_solved * sol.stats.spf_passes
    return {"value": edges / (ms / 1e3), "unit": UNIT, "ms_per_step": ms / steps, "steps": steps,
            "note": "rank 0's GPU alone, single-GPU session lane, same graph, device time per solve"}


def run_sharded(a, world, rank, local):
    """Strong scaling: one graph, every rank improves its vertex slice, the
    policy slices are all-gathered over NCCL each iteration."""
    import torch
    import torch.distributed as dist

    import paper_1111_0627_b200 as P
    from paper_1111_0627_b200.sharded import (ShardSession, TorchComm, connect_torch, solve_fused,
                                              solve_sharded)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29511")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    comm = TorchComm()
    c = CONFIGS[a.config]
    if c["kind"] == "model":
        src = build_graph_host(a, P)
    else:
        src = P.Generator(c["kind"], n=c["n"], deg=c["deg"], dmax=c.get("dmax", 0), wlo=1,
                          whi=100, seed=SEED)  # the same graph on every rank
    shards = {o: ShardSession(src, P.SolveOptions(objective=o, device=local), rank, world)
              for o in ("min", "max")}
    fused = a.lane == "fused"
    if fused:
        for o in shards:
            connect_torch(shards[o])
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
    streams = {o: torch.cuda.ExternalStream(int(P._lib.ocm_session_stream(shards[o]._h)), device=dev)
               for o in shards}

    def step():
        out, ms = {}, {}
        for o in ("min", "max"):
            flush.fill_(1)
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(streams[o])
            if fused:
                (out[o],) = solve_fused([shards[o]])
            else:
                (out[o],) = solve_sharded([shards[o]], comm)
            e1.record(streams[o])
            e1.synchronize()
            ms[o] = e0.elapsed_time(e1)
        return out, ms

    for _ in range(a.warmup):
        step()
    sols, tot = [], {"min": 0.0, "max": 0.0}
    with ClockSampler(local) as clocks:
        for _ in range(a.steps):
            out, ms = step()
            sols.append(out)
            for o in ms:
                tot[o] += ms[o]
    # per objective, max over ranks (a step's time is the sum of the two maxima)
    t = torch.tensor([tot["min"], tot["max"]], dtype=torch.float64,
                     device=dev if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_obj = {"min": float(t[0].item()), "max": float(t[1].item())}
    ms_max = ms_obj["min"] + ms_obj["max"]
    # (the shard sessions stay alive: their memory is mapped by the peers)
    dist.barrier()
    single = None
    if rank == 0 and not a.no_single_baseline:
        single = single_gpu_same_config(a, P, local, flush)
    dist.barrier()
    edges = sum(s[o].stats.m_solved * s[o].stats.spf_passes for s in sols for o in s)
    launches = sum(s[o].stats.launches for s in sols for o in s)
    if rank == 0:
        line = {
            "metric": METRIC, "value": edges / (ms_max / 1e3), "unit": UNIT, "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_max / a.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic (seeded generator)",
            "config": dict(config(a, world), parallelism=(
                f"fused x{world} (1-D vertex partition, policy pushed into peer memory inside one "
                f"launch per rank)" if fused else
                f"sharded x{world} (1-D vertex partition, policy all-gather per iteration)")),
            "time_to_ocm_s": {o: ms_obj[o] / a.steps / 1e3 for o in ("min", "max")},
            "policy_iterations": {o: sols[0][o].stats.spf_passes for o in ("min", "max")},
            "mu": {o: str(sols[0][o].mu_exact) for o in ("min", "max")},
            "gpu_launches": int(launches), "clocks": clocks.summary(),
            # the same graph on rank 0's GPU alone (the single-GPU lane,
            # after the timed region): the strong-scaling reference point --
            # the N=1 bench line measures config 2, not this config
            "single_gpu_same_config": single,
            # the graph is generated in HBM on every rank (10^9 edges): no
            # host-to-device leg to time at N > 1
            "e2e": None,
            "note": ("device time = CUDA events on the session stream around each solve (one "
                     "persistent launch per rank, exchange inside the kernel), max over ranks"
                     if fused else
                     "device time = CUDA events on the session stream around each sharded solve "
                     "(launches + NCCL exchanges), max over ranks"),
        }
        print(json.dumps(line), flush=True)


def main():
    a = parse()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(a))
    world, rank, local = dist_env()
    if world != a.gpus and "WORLD_SIZE" in os.environ:
        sys.stderr.write(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={world}\n")
        sys.exit(2)
    resolve_defaults(a, world)
    share = a.impl == "b200" and os.environ.get("OCM_BENCH_SHARE_GPU") == "1" and world > 1
    if share:
        # test mode: several ranks on one GPU -- NCCL refuses duplicate
        # devices, so the plumbing goes over gloo, and each rank's persistent
        # grid takes 1/world of the SMs so the ranks' kernels are co-resident
        import torch
        local = local % max(1, torch.cuda.device_count())
        os.environ.setdefault("OCM_GRID", str(148 * 4 // world))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist
        if a.impl == "b200" and not share:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            if a.impl == "b200":
                torch.cuda.set_device(local)
            dist.init_process_group("gloo")
    if a.impl == "reference":
        run_reference(a, world, rank)
        if dist:
            dist.destroy_process_group()
        return
    if a.lane in ("sharded", "fused"):
        run_sharded(a, world, rank, local)
        import torch.distributed as tdist
        if tdist.is_initialized():
            tdist.destroy_process_group()
        return

    import torch

    import paper_1111_0627_b200 as P
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)

    src_desc, sess = make_sessions(a, P, rank, local)

    def step():
        out = {}
        for o in ("min", "max"):
            flush.fill_(1)
            torch.cuda.synchronize()
            out[o] = sess[o].solve()
        return out

    for _ in range(a.warmup):
        step()

    def barrier():
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    sols = []
    with ClockSampler(local) as clocks:
        barrier()
        for _ in range(a.steps):
            sols.append(step())
        barrier()
    dev_ms = sum(s[o].stats.device_ms for s in sols for o in s)
    imp_ms = sum(s[o].stats.improve_ms for s in sols for o in s)
    passes = sum(s[o].stats.spf_passes for s in sols for o in s)
    launches = sum(s[o].stats.launches for s in sols for o in s)
    edges = sum(s[o].stats.m_solved * s[o].stats.spf_passes for s in sols for o in s)
    alg = sum(algorithmic_bytes(s[o].stats)[0] for s in sols for o in s)
    # the roofline is quoted on the min-objective launches: the ncu capture
    # (profiles/solve_traffic.json) is of a min launch, so achieved and
    # traffic describe the same launch
    alg_min = sum(algorithmic_bytes(s["min"].stats)[0] for s in sols)
    ms_min = sum(s["min"].stats.device_ms for s in sols)
    imp_bytes = sum(algorithmic_bytes(s[o].stats)[1] * s[o].stats.spf_passes for s in sols for o in s)
    st0 = sols[0]["min"].stats
    for s in sols:
        for o in s:
            assert s[o].has_cycle and s[o].stats.launches >= 1, "device lane did not run"
    # outside the timed region: the device optimality certificate of the last
    # solves (Bellman optimality on every edge + the anchor cycle of mean mu)
    certified = {}
    for o in ("min", "max"):
        if sols[-1][o].exact:
            c = sess[o].certify()
            certified[o] = (c["key_violations"] == 0 and c["policy_violations"] == 0
                            and c["cycle_violations"] == 0)

    # end to end through the drop-in boundary: every step hands the host graph
    # -- the reference's own CSR arrays (ocm::Graph fwd_index / fwd_target /
    # fwd_weight, graph.hpp:38-41) in ordinary pageable memory, as the
    # reference holds a loaded graph -- to ocm_solve_csr, once per objective:
    # staged upload, device validation, region split, policy iteration,
    # result read-back. Nothing is pinned or kept on the device between calls
    # (INTEGRATION.md §1 is exactly this call).
    e2e = None
    if not a.no_e2e:
        import numpy as np
        g = src_desc if isinstance(src_desc, P.Graph) else P.generate(src_desc)
        # the graph's own CSR arrays, zero-copy (the reference's EdgeId
        # offsets are 32-bit: one small conversion of n+1 entries)
        idx64, hd, hw = g.csr()
        hidx = idx64.astype(np.uint32)
        gn = g.n
        for _ in range(max(1, a.warmup)):  # untimed: grows the memory pool, staging ring
            for o in ("min", "max"):
                P.solve_csr(gn, hidx, hd, hw, P.SolveOptions(objective=o, device=local))
        e2e_s, e2e_edges, h2d, d2h = 0.0, 0, 0, 0
        e2e_steps = max(1, a.steps)
        torch.cuda.synchronize()
        for _ in range(e2e_steps):
            t0 = time.perf_counter()
            for o in ("min", "max"):
                s = P.solve_csr(gn, hidx, hd, hw, P.SolveOptions(objective=o, device=local))
                e2e_edges += s.stats.m_solved * s.stats.spf_passes
                h2d += s.stats.h2d_bytes
                d2h += s.stats.d2h_bytes
                if os.environ.get("OCM_BENCH_E2E_TRACE"):
                    sys.stderr.write(f"e2e {o}: {1e3 * (time.perf_counter() - t0):.3f} ms "
                                     f"device {s.stats.device_ms:.3f} prep {s.stats.host_prep_ms:.3f}\n")
            e2e_s += time.perf_counter() - t0
        e2e = (e2e_s, e2e_edges, h2d // e2e_steps, d2h // e2e_steps)
        del hidx, hd, hw, idx64, g

    vals = [dev_ms, e2e[0] if e2e else 0.0]
    tots = [float(edges), float(e2e[1] if e2e else 0), float(launches)]
    if dist:
        rdev = dev if dist.get_backend() == "nccl" else "cpu"
        t = torch.tensor(vals, dtype=torch.float64, device=rdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot = torch.tensor(tots, dtype=torch.float64, device=rdev)
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
        vals, tots = t.tolist(), tot.tolist()
    dev_ms_max, e2e_max = vals
    edges_all, e2e_edges_all, launches_all = tots

    if rank == 0:
        peak, peak_src = measured_peak()
        achieved = alg_min / (ms_min / 1e3) / 1e9
        imp_achieved = imp_bytes / (imp_ms / 1e3) / 1e9 if imp_ms else None
        line = {
            "metric": METRIC, "value": edges_all / (dev_ms_max / 1e3), "unit": UNIT,
            "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": dev_ms_max / a.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int64", "data": "synthetic (seeded generator)",
            "config": config(a, world),
            "graph": {"n_solved": st0.n_solved, "m_solved": st0.m_solved,
                      "regions": st0.regions, "trivial_regions": st0.trivial_regions},
            "time_to_ocm_s": {o: sum(s[o].stats.device_ms for s in sols) / a.steps / 1e3
                              for o in ("min", "max")},
            "policy_iterations": {o: sols[0][o].stats.spf_passes for o in ("min", "max")},
            "mu": {o: str(sols[0][o].mu_exact) for o in ("min", "max")},
            "certified": certified,
            "improve_share": imp_ms / dev_ms,
            "roofline": {
                "bound": "hbm", "kernel": "k_solve (persistent: one cooperative launch per solve)",
                "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": ncu_traffic(a.config),
                "bytes_per_launch": alg_min / a.steps, "avg_launch_ms": ms_min / a.steps,
                "launches": "min-objective k_solve launches (the ncu-captured one)",
                "all_launches": {"achieved": alg / (dev_ms / 1e3) / 1e9,
                                 "bytes_per_launch": alg / (2 * a.steps),
                                 "avg_launch_ms": dev_ms / (2 * a.steps)},
                "peak_source": peak_src,
                "improve_phase": {"achieved": imp_achieved,
                                  "frac": imp_achieved / peak if imp_achieved else None,
                                  "bytes_per_pass": imp_bytes / passes,
                                  "avg_pass_ms": imp_ms / passes,
                                  # the pass is bound by random 8-byte key gathers (one per
                                  # edge), whose measured B200 ceiling depends on whether the
                                  # key array stays in L2 (profiles/micro_gather_r01.log)
                                  "gathers_per_s": st0.m_solved / (imp_ms / passes / 1e3) if imp_ms else None,
                                  "gather_peak_per_s": gather_peak(st0.n_solved)[0],
                                  "gather_frac": (st0.m_solved / (imp_ms / passes / 1e3)
                                                  / gather_peak(st0.n_solved)[0]) if imp_ms else None,
                                  "gather_peak_source": gather_peak(st0.n_solved)[1]},
                "note": "achieved = algorithmic bytes (DESIGN.md §5) / CUDA-event time of the "
                        "launch on the session stream; improve_phase timed by SM clock share "
                        "between the phase's grid barriers",
            },
            "gpu_launches": int(launches_all),
            "clocks": clocks.summary(),
        }
        if e2e:
            line["e2e"] = {"value": e2e_edges_all / e2e_max, "unit": UNIT,
                           "h2d_bytes_per_step": e2e[2], "d2h_bytes_per_step": e2e[3],
                           "ms_per_step": e2e_max * 1e3 / max(1, a.steps),
                           "path": "ocm_solve_csr per objective on pageable host CSR arrays "
                                   "(upload, validation, region split, solve, read-back)"}
        if world == 1 and not a.no_cpu_baseline:
            # one min + one max solve of the reference on the same graph,
            # concurrently on two host threads (~20-30 s of CPU work)
            r = reference_solves(a.config, 1, 0, 2)
            line["cpu_baseline"] = {"value": r["value"], "unit": UNIT, "cores": r["cores"],
                                    "kind": "reference", "sample": r["sample"],
                                    "time_to_ocm_s": r["time_to_ocm_s"], "mu": r["mu"]}
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
