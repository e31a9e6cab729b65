"""Benchmark: policy-iteration throughput of the B200 optimal-cycle-mean solver.

Workload (BASELINE.json configs[1]): random sparse digraph, 10^6 vertices,
out-degree 8, integer weights 1..100, min AND max cycle mean. One step = one
full time-to-OCM solve for each objective on the graph resident in HBM
(policy iteration from the initial policy until no policy edge changes).

metric: edges/s per policy iteration = intra-region edges x improvement passes
/ device time, summed over ranks (weak scaling: every rank solves its own
seeded instance; the path's per-iteration work is independent per graph).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--deg", type=int, default=8)
    ap.add_argument("--seed", type=int, default=1111_0627)
    ap.add_argument("--cpu-sample-n", type=int, default=250_000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def config(a, world):
    return {"workload": f"uniform random digraph n={a.n} out-degree {a.deg} weights 1..100 "
                        f"(BASELINE configs[1]), min+max cycle mean per step",
            "n": a.n, "out_degree": a.deg, "weights": [1, 100], "seed": a.seed,
            "objectives": ["min", "max"], "parallelism": f"replicas x{world}" if world > 1 else "1 gpu",
            "l2": "flushed between steps (512 MiB write)"}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0, set()
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
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic():
    """dram bytes per k_improve launch from the committed ncu --set full summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "improve_traffic.json")) as f:
            return json.load(f).get("dram_bytes_per_launch")
    except Exception:
        return None


def improve_bytes(n_solved, m_solved):
    """Algorithmic bytes of one k_improve launch (kernel 1): per edge an
    8 B {target, weight} record and an 8 B key gather; per vertex row (4 B),
    region id (4 B), incumbent edge/target/weight (12 B) and its key (8 B)."""
    return 16 * m_solved + 28 * n_solved


def cpu_sample(a, steps=1):
    """Reference CPU solver on a bounded sample (same generator, smaller n)."""
    import oracle as O
    n = a.cpu_sample_n
    s, d, w = O.generate_uniform(n, a.deg, 1, 100, a.seed)
    use_ref = O.ref_available()
    tot_ms, edges = 0.0, 0
    for _ in range(steps):
        for objective in ("min", "max"):
            if use_ref:
                r = O.ref_solve(n, s, d, w, "howard", objective, "tarjan")
                tot_ms += r.solve_ms
            else:
                t0 = time.perf_counter()
                r = O.oracle_solve(n, s, d, w, objective)
                tot_ms += (time.perf_counter() - t0) * 1e3
                r.extra["spf_passes_seq"] = r.extra.get("spf_passes_seq", r.spf_passes)
            passes = r.spf_passes if use_ref else r.extra["spf_passes_seq"]
            edges += len(s) * passes
    return {"value": edges / (tot_ms / 1e3), "unit": UNIT, "cores": 1,
            "kind": "reference" if use_ref else "port",
            "sample": f"uniform n={n} deg={a.deg} weights 1..100, min+max, reference lane "
                      f"'howard' (proj/src/solve.cpp run_howard_seq, single thread; the default "
                      f"CLI lane and the fastest reference lane on this workload), "
                      f"{steps} step(s), solve time only",
            "ms": tot_ms}


def run_reference(a, world, rank):
    if rank != 0:
        return
    steps = []
    for i in range(a.warmup + a.steps):
        r = cpu_sample(a, 1)
        if i >= a.warmup:
            steps.append(r)
    tot_ms = sum(r["ms"] for r in steps)
    val = sum(r["value"] * r["ms"] for r in steps) / tot_ms
    base = steps[0]
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": tot_ms / a.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic (seeded uniform digraph)", "config": config(a, 1),
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": base["cores"],
                             "kind": base["kind"], "sample": base["sample"]},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    a = parse()
    world, rank, local = dist_env()
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl" if a.impl == "b200" else "gloo")
    if a.impl == "reference":
        run_reference(a, world, rank)
        if dist:
            dist.destroy_process_group()
        return

    import torch

    import paper_1111_0627_b200 as P
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)

    g = P.generate_uniform(a.n, a.deg, 1, 100, a.seed + rank)
    sess = {o: P.Session(g, P.SolveOptions(objective=o, device=local)) for o in ("min", "max")}

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
    m_solved = sols[0]["min"].stats.m_solved
    n_solved = sols[0]["min"].stats.n_solved
    edges = m_solved * passes

    # end-to-end through the public API: the host graph (CSR in pinned host
    # memory, built and pinned once outside the timed region, as a user's
    # loaded graph would be) goes through ocm_solve every step: upload, device
    # region split, policy iteration, result read-back.
    src, dst, w = g.edges()
    gg = P.build_graph(a.n, (src, dst, w))
    P.solve(gg, P.SolveOptions(objective="min", device=local))  # pins the host arrays
    e2e_s, e2e_edges, h2d, d2h = 0.0, 0, 0, 0
    e2e_steps = max(1, a.steps)
    torch.cuda.synchronize()
    for i in range(e2e_steps):
        t0 = time.perf_counter()
        for o in ("min", "max"):
            s = P.solve(gg, P.SolveOptions(objective=o, device=local))
            e2e_edges += s.stats.m_solved * s.stats.spf_passes
            h2d += s.stats.h2d_bytes
            d2h += s.stats.d2h_bytes
        e2e_s += time.perf_counter() - t0

    if dist:
        t = torch.tensor([dev_ms, e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot = torch.tensor([float(edges), float(e2e_edges), float(launches)], dtype=torch.float64,
                           device=dev)
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
        dev_ms_max, e2e_max = t.tolist()
        edges_all, e2e_edges_all, launches_all = tot.tolist()
    else:
        dev_ms_max, e2e_max = dev_ms, e2e_s
        edges_all, e2e_edges_all, launches_all = edges, e2e_edges, launches

    if rank == 0:
        peak, peak_src = measured_peak()
        per_launch_ms = imp_ms / passes
        bytes_launch = improve_bytes(n_solved, m_solved)
        achieved = bytes_launch / (per_launch_ms / 1e3) / 1e9
        traffic = ncu_traffic()
        line = {
            "metric": METRIC, "value": edges_all / (dev_ms_max / 1e3), "unit": UNIT,
            "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": dev_ms_max / a.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int64", "data": "synthetic (seeded uniform digraph)",
            "config": config(a, world),
            "time_to_ocm_s": {o: sum(s[o].stats.device_ms for s in sols) / a.steps / 1e3
                              for o in ("min", "max")},
            "policy_iterations": {o: sols[0][o].stats.spf_passes for o in ("min", "max")},
            "mu": {o: str(sols[0][o].mu_exact) for o in ("min", "max")},
            "improve_share": imp_ms / dev_ms,
            "roofline": {"bound": "hbm", "kernel": "k_improve", "achieved": achieved,
                         "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "bytes_per_launch": bytes_launch,
                         "avg_launch_ms": per_launch_ms, "peak_source": peak_src,
                         "note": "working set (64 MB edges + 8 MB keys) fits the 126 MB L2; "
                                 "passes after the first read edges from L2"},
            "e2e": {"value": e2e_edges_all / e2e_max, "unit": UNIT,
                    "h2d_bytes_per_step": h2d // e2e_steps, "d2h_bytes_per_step": d2h // e2e_steps},
            "gpu_launches": int(launches_all),
            "clocks": clocks.summary(),
        }
        if world == 1 and not a.no_cpu_baseline:
            cb = cpu_sample(a, 1)
            cb.pop("ms")
            line["cpu_baseline"] = cb
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
