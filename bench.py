"""Throughput benchmark: batched quasi-static equilibrium solves/s on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--impl ours|reference]
                    [--dist-backend nccl|gloo] [--chunk C]

One step = `Engine.solve_static_batch` (run_static of the reference,
engine.py:267-283) over a batch of B independent cfg4 scenarios (100-element
robot in the lumen mesh, ~20 contacts; tensions / load scale / insertion
sampled per scenario).  With N GPUs (torchrun, one process per
GPU) every rank solves its own B-scenario shard of the 65,536-scenario table:
weak scaling, no data-path collective (the scenarios are independent); the
process group carries only the barriers, the max-over-ranks step time and the
final result gather.  `--chunk C` replaces the static shards by a dynamic
cross-rank queue of C-scenario chunks over the process group's store (one
launch per chunk); `--dist-backend gloo` lets several ranks share one GPU
(NCCL refuses two ranks on one device).

Timing: W untimed warm-up steps; then K steps, each timed with CUDA events on
the launching stream, an L2 flush (512 MiB write) between steps outside the
events; value = scenarios of all ranks / max-over-ranks mean step time.
`e2e` repeats the measurement through the host-buffer C-ABI path
(accfem_solve_batch_host: H2D of the inputs, solve, D2H of every output).

--impl reference times the reference's own CPU implementation on all host
cores, rank 0 only: the unmodified `cablefem` package from baseline/_ref
(oracle/reference_runner.py, kind "reference") when it is installed, else the
numpy restatement (oracle/accfem_oracle.py, kind "port").
"""

from __future__ import annotations

import argparse
import hashlib
import json
import multiprocessing as mp
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "quasi-static equilibrium solves/sec (batched)"
UNIT = "solves/s"
WORKLOAD = ("cfg4: batch of 100-element robots in a lumen mesh (3780 triangles), ~20 contacts, per-scenario "
            "cable tensions / load scale / insertion offset")


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--batch", type=int, default=8192, help="scenarios per GPU per step")
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--cpu-sample", type=int, default=32, help="scenarios in the CPU baseline sample")
    p.add_argument("--cpu-kind", default="auto", choices=["auto", "reference", "port"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"])
    p.add_argument("--chunk", type=int, default=0, help="dynamic cross-rank chunks of C scenarios (0: static shards)")
    return p.parse_args()


# ----------------------------------------------------------------------------
# CPU arms: one process per host core
# ----------------------------------------------------------------------------

_KIND = "port"


def _cpu_one(i):
    """One run_static of cfg4 scenario i on the CPU (scene cached per process)."""
    from paper_2503_06922_b200 import scenarios
    w = scenarios.cfg4(1, start=i)
    if _KIND == "reference":
        from oracle import reference_runner
        return reference_runner.run_static(w, 0)
    from oracle import accfem_oracle as O
    return O.solve_workload(w)[0]["status"]


def cpu_kind(requested):
    from oracle import reference_runner
    if requested == "auto":
        return "reference" if reference_runner.available() else "port"
    if requested == "reference" and not reference_runner.available():
        raise SystemExit("baseline/_ref is not installed (see oracle/reference_runner.py)")
    return requested


def cpu_rate(indices, cores, kind):
    """solves/s over `indices` on `cores` processes (one warm-up task per worker)."""
    global _KIND
    _KIND = kind
    os.environ.update({"OMP_NUM_THREADS": "1", "OPENBLAS_NUM_THREADS": "1", "MKL_NUM_THREADS": "1"})
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        pool.map(_cpu_one, list(indices[:cores]))  # warm-up: imports, scipy paging
        t0 = time.perf_counter()
        status = pool.map(_cpu_one, list(indices), chunksize=1)
        dt = time.perf_counter() - t0
    return len(indices) / dt, dt, status


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ----------------------------------------------------------------------------
# clocks during the timed region
# ----------------------------------------------------------------------------

class ClockSampler:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        self.thread.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for nm, v in zip(names, r[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


# ----------------------------------------------------------------------------
# FLOP model from per-frame device traces of a sample
# ----------------------------------------------------------------------------

def flops_per_solve(eng, w, sample=256):
    """Average algorithmic FLOP per solve over the first `sample` scenarios:
    (F+1)(3000E + 100N) + F_c N (7900+650) + F_0 N 2200 + sum_f I_f (250N + 30 m_f)
    + 250 N K + 80 P + 1300 N R, with K = sum_f [min(I_f, 8) + floor(I_f / 25)],
    P the broad-phase (node, triangle) pairs and R the polish rounds, both counted
    on the device per frame (ACCFEM_TRACE_STATS columns 12 and 13)."""
    from paper_2503_06922_b200 import _lib
    s = min(sample, w.size)
    N = w.model.node_count
    E = N - 1
    res = eng.solve_static_batch(np.ascontiguousarray(w.x0[:s]), np.ascontiguousarray(w.tensions[:s]),
                                 np.ascontiguousarray(w.applied[:s]), tol=w.tol, max_frames=w.max_frames,
                                 trace_frames=w.max_frames)
    nf = len(eng._rows)
    tot, pairs, rounds = 0.0, 0.0, 0.0
    for i in range(s):
        F = int(res.frames[i])
        st = res.trace_stats[i, :F]
        its, nc = st[:, 5], st[:, 6]
        Fc = int((nc > 0).sum())
        F0 = F - Fc
        K = float(np.sum(np.minimum(its, 8) + np.floor(its / 25)))
        P = float(st[:, 12].sum())
        R = float(st[:, 13].sum())
        pairs += P
        rounds += R
        tot += ((F + 1) * (3000 * E + 100 * N) + Fc * N * (7900 + 650) + F0 * N * 2200
                + float(np.sum(its * (250 * N + 30 * (nf + nc)))) + 250 * N * K + 80 * P + 1300 * N * R)
    assert _lib.TRACE_STATS == 14
    return tot / s, pairs / s, rounds / s


def fp64_peak_tflops(dev):
    """Measured cuBLAS DGEMM throughput (8192^3, best of 5) as the FP64 peak."""
    import torch
    a = torch.randn(8192, 8192, dtype=torch.float64, device=dev)
    b = torch.randn(8192, 8192, dtype=torch.float64, device=dev)
    best = 0.0
    for _ in range(6):
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        torch.matmul(a, b)
        s1.record()
        s1.synchronize()
        best = max(best, 2 * 8192 ** 3 / (s0.elapsed_time(s1) * 1e-3) / 1e12)
    del a, b
    return best


def library_sha():
    """Identity of the library build: sha256 of its sources and nvcc flags
    (build.sources(), build.FLAGS) -- the binary itself embeds nvcc temp-file
    names, so its bytes differ between otherwise identical builds."""
    from paper_2503_06922_b200 import build
    h = hashlib.sha256(" ".join(build.FLAGS).encode())
    for p in sorted(build.sources()):
        with open(p, "rb") as fh:
            h.update(os.path.basename(p).encode() + fh.read())
    return h.hexdigest()[:16]


def ncu_profile(sha):
    """DRAM bytes and FP64-pipe utilisation of k_solve per solve from the committed
    ncu capture (profiles/k_solve_ncu.json) -- used only if it was taken of this
    very library build (same source sha256 prefix, library_sha()), else reported
    as stale."""
    p = os.path.join(ROOT, "profiles", "k_solve_ncu.json")
    if not os.path.exists(p):
        return None
    with open(p) as fh:
        d = json.load(fh)
    return d if d.get("library_source_sha256_16") == sha else {"stale": True, "source": d.get("source")}


def load_balance(ts):
    """Per-team load-balance record of one launch (4 int64 per team: scenarios, busy ns,
    start ns, end ns): the idle tail after the median team finished, as a fraction of
    the launch span, and the busy fraction of all teams."""
    if ts is None or not len(ts):
        return None
    ts = np.asarray(ts, dtype=np.float64)
    start, end = ts[:, 2].min(), ts[:, 3].max()
    span = max(end - start, 1.0)
    return {"teams": int(len(ts)), "tail_frac": float((end - np.median(ts[:, 3])) / span),
            "busy_frac": float(ts[:, 1].sum() / (span * len(ts))),
            "scenarios_per_team": [int(ts[:, 0].min()), int(ts[:, 0].max())]}


# ----------------------------------------------------------------------------

def run_reference(args, rank, world):
    if rank != 0:
        return
    cores = host_cores()
    kind = cpu_kind(args.cpu_kind)
    n = max(args.cpu_sample, cores)
    vals = []
    for step in range(args.warmup + args.steps):
        idx = list(range(step * n, (step + 1) * n))
        rate, dt, _ = cpu_rate(idx, cores, kind)
        if step >= args.warmup:
            vals.append(rate)
    v = statistics.mean(vals)
    what = ("the unmodified reference package (cablefem from baseline/_ref, Engine.run_static)" if kind == "reference"
            else "the numpy/scipy restatement of the reference (oracle/accfem_oracle.py)")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": n / v * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "scenarios_per_step": n,
                       "note": f"CPU: {what} on all host cores ({cpu_model()})"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": kind,
                             "sample": f"{n} cfg4 scenarios per step, one process per core"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch
    import torch.distributed as dist

    gloo = args.dist_backend == "gloo"
    dev_index = local % max(torch.cuda.device_count(), 1) if gloo else local
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if gloo:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    red_dev = torch.device("cpu") if gloo else dev
    pg = dist if world > 1 else None
    from paper_2503_06922_b200 import _lib, scenarios, shard
    from paper_2503_06922_b200.engine import Engine

    B = args.batch
    dynamic = args.chunk > 0 and world > 1
    if dynamic:
        # every rank holds the whole B x world table; chunks are claimed from the store
        w = scenarios.cfg4(B * world, start=0)
    else:
        start, _ = shard.shard_range(rank, world, B, scenarios.CFG4_TOTAL)
        w = scenarios.cfg4(B, start=start)
    eng = Engine(**w.engine_kwargs(), device=dev_index)
    x0 = torch.tensor(w.x0, device=dev)
    ten = torch.tensor(w.tensions, device=dev)
    app = torch.tensor(w.applied, device=dev)
    out = eng.allocate_batch(w.size)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    team_cap = 4096
    team_stats = torch.zeros((team_cap, 4), dtype=torch.int64, device=dev)
    store = dist.distributed_c10d._get_default_store() if dynamic else None
    mine = np.zeros(w.size, bool)

    def launch(a, b, stats=None):
        sl = slice(a, b)
        o = type(out)(**{f: (getattr(out, f)[sl] if getattr(out, f) is not None else None)
                         for f in out.__dataclass_fields__})
        eng.solve_static_batch(x0[sl], ten[sl], app[sl], tol=w.tol, max_frames=w.max_frames, out=o, stream=stream)

    step_no = [0]

    def step(record=False):
        if dynamic:
            q = shard.ChunkQueue(store, f"bench_step_{step_no[0]}", w.size, args.chunk)
            step_no[0] += 1
            while True:
                r = q.next()
                if r is None:
                    break
                launch(*r)
                mine[r[0]:r[1]] = True
        else:
            eng.solve_static_batch(x0, ten, app, tol=w.tol, max_frames=w.max_frames, out=out, stream=stream,
                                   team_stats=team_stats if record else None)
            mine[:] = True

    for _ in range(args.warmup):
        step()
        flush.zero_()
    torch.cuda.synchronize()
    clocks = ClockSampler(dev_index)
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = eng.launches
    times = []
    for k in range(args.steps):
        mine[:] = False
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step(record=(k == args.steps - 1))
        e1.record(stream)
        flush.zero_()
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = eng.launches - launches0
    clk = clocks.stop()
    ms = shard.max_over_ranks(statistics.mean(times), pg, red_dev)
    total = B * world
    value = total / (ms * 1e-3)
    lb = None
    if not dynamic:
        teams = min(eng._lib.accfem_last_launch_teams(eng._h), team_cap)
        lb = load_balance(team_stats[:teams].cpu().numpy())
    # results of every rank (outside the timed region): status / frames of all scenarios
    st_local = np.where(mine, out.status.cpu().numpy(), -1).astype(np.int64)
    fr_local = np.where(mine, out.frames.cpu().numpy(), -1).astype(np.int64)
    if dynamic:
        st_all = shard.all_max([st_local], pg)[0]
        fr_all = shard.all_max([fr_local], pg)[0]
    else:
        st_all, fr_all = shard.gather_results([st_local, fr_local], pg, red_dev)
    status, frames = np.asarray(st_all), np.asarray(fr_all)
    assert status.size == total and (status >= 0).all(), "a scenario was not solved"

    # e2e through the host-buffer C-ABI path (copies inside the timed region)
    e2e = None
    if not args.no_e2e and not dynamic:
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
        hx0, hten, happ = pin(w.x0), pin(w.tensions), pin(w.applied)
        hout = eng.allocate_batch(B, host=True)
        for f in ("coords", "status", "frames", "converged", "residual", "n_contacts", "contact_node",
                  "contact_triangle", "contact_gap", "contact_multiplier", "contact_force", "contact_normal",
                  "contact_point"):
            setattr(hout, f, pin(getattr(hout, f)))
        eng.solve_static_batch(hx0, hten, happ, tol=w.tol, max_frames=w.max_frames, out=hout)  # warm
        if world > 1:
            dist.barrier()
        et = []
        for _ in range(max(1, args.steps)):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            eng.solve_static_batch(hx0, hten, happ, tol=w.tol, max_frames=w.max_frames, out=hout)
            et.append((time.perf_counter() - t0) * 1e3)
            flush.zero_()
        ems = shard.max_over_ranks(statistics.mean(et), pg, red_dev)
        h2d = hx0.nbytes + hten.nbytes + happ.nbytes
        d2h = sum(getattr(hout, f).nbytes for f in ("coords", "status", "frames", "converged", "residual",
                                                      "n_contacts", "contact_node", "contact_triangle",
                                                      "contact_gap", "contact_multiplier", "contact_force",
                                                      "contact_normal", "contact_point"))
        e2e = {"value": B * world / (ems * 1e-3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": ems,
               "path": "Engine.solve_static_batch(numpy) -> accfem_solve_batch_host: H2D from pinned host "
                       "buffers, solve, D2H of every output"}

    # p50 single-solve latency (batch = 1, wall clock incl. launch and sync)
    lat = {}
    if rank == 0:
        for tag, wl in (("cfg4_s0", scenarios.cfg4(1)), ("cfg3p", scenarios.cfg3p(1))):
            e1 = Engine(**wl.engine_kwargs(), device=dev_index)
            a = [None if v is None else torch.tensor(v, device=dev) for v in (wl.x0, wl.tensions, wl.applied)]
            o1 = e1.allocate_batch(1)
            ts = []
            for rep in range(12):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                e1.solve_static_batch(a[0], a[1], a[2], tol=wl.tol, max_frames=wl.max_frames, out=o1)
                torch.cuda.synchronize()
                if rep >= 2:
                    ts.append((time.perf_counter() - t0) * 1e3)
            lat[tag] = {"p50_ms": statistics.median(ts), "frames": int(o1.frames[0].item()),
                        "kernel": "k_solve<8, cyclic reduction> (one CTA per scenario)"}

    line = None
    if rank == 0:
        sha = library_sha()
        prof = ncu_profile(sha)
        fl, pairs, rounds = flops_per_solve(eng, w)
        peak = fp64_peak_tflops(dev)
        achieved = fl * B / (ms * 1e-3) / 1e12  # per GPU
        traffic = prof["dram_bytes_per_solve"] * B if prof and "dram_bytes_per_solve" in prof else None
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cores = host_cores()
            kind = cpu_kind(args.cpu_kind)
            n = max(args.cpu_sample, cores)
            rate, dt, _ = cpu_rate(list(range(n)), cores, kind)
            cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": kind,
                   "sample": f"first {n} cfg4 scenarios, one process per core ({cpu_model()}), {dt:.1f} s"}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "scenarios_per_gpu_per_step": B, "global_batch": total, "tol": w.tol,
                       "max_frames": w.max_frames,
                       "parallelism": (f"dp{world} (dynamic {args.chunk}-scenario chunks)" if dynamic
                                       else f"dp{world} (scenario shards)"),
                       "dist_backend": args.dist_backend if world > 1 else None,
                       "l2": "512 MiB flush between timed steps (outside the events)",
                       "status_counts": {str(k): int(v) for k, v in zip(*np.unique(status, return_counts=True))},
                       "mean_frames": float(frames.mean())},
            "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "traffic_source": None if not prof or prof.get("stale") else prof.get("source"),
                         "fp64_pipe_pct_ncu": None if not prof or prof.get("stale") else prof.get("fp64_pipe_pct"),
                         "peak_source": "cuBLAS DGEMM 8192^3 measured in this run (no FP64 entry in "
                                        "MEASURED_PEAKS.json)",
                         "flop_per_solve": fl, "pairs_per_solve": pairs, "polish_rounds_per_solve": rounds,
                         "library_source_sha256_16": sha,
                         "kernel": "k_solve<2> (persistent, one 2-warp CTA per scenario, "
                                   f"{eng._lib.accfem_teams_resident(eng._h)} resident)"},
            "load_balance": lb,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches), "clocks": clk,
            "latency": {"batch": 1, "wall_clock": "solve_static_batch + cudaDeviceSynchronize", **lat},
        }
        print(json.dumps(line), flush=True)
        assert _lib.TRACE_STATS == 14
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
