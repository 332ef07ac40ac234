"""Throughput benchmark: batched quasi-static equilibrium solves/s on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--impl ours|reference]

One step = `Engine.solve_static_batch` (run_static of the reference,
engine.py:267-283) over a batch of B independent cfg4 scenarios (100-element
robot in the lumen mesh, ~20 contacts; tensions / load scale / insertion
sampled per scenario).  With N GPUs (torchrun, one process per
GPU) every rank solves its own B-scenario shard of the 65,536-scenario table:
weak scaling, no data-path collective (the scenarios are independent); NCCL
is used only for the barrier and the max-over-ranks step time.

Timing: W untimed warm-up steps; then K steps, each timed with CUDA events on
the launching stream, an L2 flush (512 MiB write) between steps outside the
events; value = scenarios of all ranks / max-over-ranks mean step time.
`e2e` repeats the measurement through the host-buffer C-ABI path
(accfem_solve_batch_host: H2D of the inputs, solve, D2H of every output).

--impl reference times the CPU oracle (the numpy/scipy restatement of the
reference algorithm, oracle/accfem_oracle.py) on all host cores, rank 0 only.
"""

from __future__ import annotations

import argparse
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


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--batch", type=int, default=8192, help="scenarios per GPU per step")
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--cpu-sample", type=int, default=32, help="scenarios in the CPU baseline sample")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    return p.parse_args()


# ----------------------------------------------------------------------------
# CPU oracle (reference arm / cpu_baseline): one process per host core
# ----------------------------------------------------------------------------

def _oracle_one(i):
    """One run_static of cfg4 scenario i with the CPU oracle (scene cached per process)."""
    from oracle import accfem_oracle as O
    from paper_2503_06922_b200 import scenarios
    w = scenarios.cfg4(1, start=i)
    return O.solve_workload(w)[0]["status"]


def cpu_oracle_rate(indices, cores):
    """solves/s of the oracle over `indices` on `cores` processes (1 warm-up task each)."""
    env = {"OMP_NUM_THREADS": "1", "OPENBLAS_NUM_THREADS": "1", "MKL_NUM_THREADS": "1"}
    os.environ.update(env)
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        pool.map(_oracle_one, list(indices[:cores]))  # warm-up: imports, scipy paging
        t0 = time.perf_counter()
        status = pool.map(_oracle_one, list(indices), chunksize=1)
        dt = time.perf_counter() - t0
    return len(indices) / dt, dt, status


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


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
# FLOP model from per-frame traces of a sample
# ----------------------------------------------------------------------------

def flops_per_solve(eng, w, sample=256):
    """Average algorithmic FLOP per solve over the first `sample` scenarios:
    (F+1)(3000E + 100N) + F_c N (7900+650) + F_0 N 2200 + sum_f I_f (250N + 30 m_f)
    + 250 N K + 80 P + 1300 N R, with K = sum_f [min(I_f, 8) + floor(I_f / 25)],
    P ~ 18 candidate pairs per node per frame, R ~ 3 polish rounds per contact
    frame (oracle statistics of cfg3)."""
    import ctypes

    from paper_2503_06922_b200 import _lib
    s = min(sample, w.size)
    N, n = w.model.node_count, w.model.dof_count
    E = N - 1
    cap = w.max_frames
    H = dict(x0=np.ascontiguousarray(w.x0[:s]), tensions=np.ascontiguousarray(w.tensions[:s]),
             applied=np.ascontiguousarray(w.applied[:s]), coords=np.zeros((s, n)), status=np.zeros(s, np.int32),
             frames=np.zeros(s, np.int32), converged=np.zeros(s, np.int32), residual=np.zeros(s),
             n_contacts=np.zeros(s, np.int32), contact_node=np.zeros((s, N), np.int32),
             contact_triangle=np.zeros((s, N), np.int32), contact_gap=np.zeros((s, N)),
             contact_multiplier=np.zeros((s, N)), contact_force=np.zeros((s, N, 3)),
             contact_normal=np.zeros((s, N, 3)), contact_point=np.zeros((s, N, 3)),
             trace_stats=np.zeros((s, cap, _lib.TRACE_STATS)))
    d = _lib.BatchDesc()
    d.S = s
    for name, _ in _lib.BATCH_FIELDS:
        if name in H:
            setattr(d, name, _lib.ptr(H[name]))
    d.trace_cap, d.max_frames, d.stop_on_tol, d.tol, d.fail_on_limit = cap, w.max_frames, 1, w.tol, 1
    eng._check(eng._lib.accfem_solve_batch_host(eng._h, ctypes.byref(d), None))
    nf = len(eng._rows)
    tot = 0.0
    for i in range(s):
        F = int(H["frames"][i])
        st = H["trace_stats"][i, :F]
        its = st[:, 5]
        nc = st[:, 6]
        Fc = int((nc > 0).sum())
        F0 = F - Fc
        K = float(np.sum(np.minimum(its, 8) + np.floor(its / 25)))
        P = 18.0 * N * F
        R = 3.0 * Fc
        tot += ((F + 1) * (3000 * E + 100 * N) + Fc * N * (7900 + 650) + F0 * N * 2200
                + float(np.sum(its * (250 * N + 30 * (nf + nc)))) + 250 * N * K + 80 * P + 1300 * N * R)
    return tot / s


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


# ----------------------------------------------------------------------------

def run_reference(args, rank, world):
    if rank != 0:
        return
    cores = host_cores()
    n = max(args.cpu_sample, cores)
    base = args.batch * 0
    vals = []
    for step in range(args.warmup + args.steps):
        idx = list(range(base + step * n, base + (step + 1) * n))
        rate, dt, _ = cpu_oracle_rate(idx, cores)
        if step >= args.warmup:
            vals.append(rate)
    v = statistics.mean(vals)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": n / v * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "cfg4: 100-element robot in lumen mesh (3780 tri), ~20 contacts, "
                                   "per-scenario tensions/load/insertion", "scenarios_per_step": n,
                       "note": "CPU oracle (numpy/scipy restatement of the reference) on all host cores"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
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

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=dev)
    from paper_2503_06922_b200 import scenarios
    from paper_2503_06922_b200.engine import Engine

    from paper_2503_06922_b200 import shard

    B = args.batch
    start, _ = shard.shard_range(rank, world, B, scenarios.CFG4_TOTAL)
    w = scenarios.cfg4(B, start=start)
    eng = Engine(**w.engine_kwargs(), device=local)
    x0 = torch.tensor(w.x0, device=dev)
    ten = torch.tensor(w.tensions, device=dev)
    app = torch.tensor(w.applied, device=dev)
    out = eng.allocate_batch(B)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        eng.solve_static_batch(x0, ten, app, tol=w.tol, max_frames=w.max_frames, out=out, stream=stream)

    for _ in range(args.warmup):
        step()
        flush.zero_()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = eng.launches
    times = []
    for _ in range(args.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        flush.zero_()
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = eng.launches - launches0
    clk = clocks.stop()
    ms = shard.max_over_ranks(statistics.mean(times), dist if world > 1 else None, dev)
    value = B * world / (ms * 1e-3)
    status = out.status.cpu().numpy()
    frames = out.frames.cpu().numpy()

    # e2e through the host-buffer C-ABI path (copies inside the timed region)
    e2e = None
    if not args.no_e2e:
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
        ems = shard.max_over_ranks(statistics.mean(et), dist if world > 1 else None, dev)
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
        for tag, wl in (("cfg4_s0", scenarios.cfg4(1, start=start)), ("cfg3p", scenarios.cfg3p(1))):
            e1 = eng if tag == "cfg4_s0" else Engine(**wl.engine_kwargs(), device=local)
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
            lat[tag] = {"p50_ms": statistics.median(ts), "frames": int(o1.frames[0].item())}

    line = None
    if rank == 0:
        # DRAM bytes per launch of k_solve: dram__bytes_read + write per solve from the committed ncu
        # --set full capture (profiles/k_solve_dram.json), times the scenarios of this launch
        traffic, traffic_src = None, None
        tf = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "k_solve_dram.json")
        if os.path.exists(tf):
            with open(tf) as fh:
                td = json.load(fh)
            traffic = td["dram_bytes_per_solve"] * B
            traffic_src = td["source"]
        fl = flops_per_solve(eng, w)
        peak = fp64_peak_tflops(dev)
        achieved = fl * B / (ms * 1e-3) / 1e12
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cores = host_cores()
            n = max(args.cpu_sample, cores)
            rate, dt, _ = cpu_oracle_rate(list(range(n)), cores)
            cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "port",
                   "sample": f"first {n} cfg4 scenarios, one oracle process per core, {dt:.1f} s"}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "cfg4: batch of 100-element robots in a lumen mesh (3780 triangles), "
                                   "~20 contacts, per-scenario cable tensions / load scale / insertion offset",
                       "scenarios_per_gpu_per_step": B, "global_batch": B * world, "tol": w.tol,
                       "max_frames": w.max_frames, "parallelism": f"dp{world} (scenario shards)",
                       "l2": "512 MiB flush between timed steps (outside the events)",
                       "status_counts": {str(k): int(v) for k, v in zip(*np.unique(status, return_counts=True))},
                       "mean_frames": float(frames.mean())},
            "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                         "peak_source": "cuBLAS DGEMM 8192^3 measured in this run (no FP64 entry in "
                                        "MEASURED_PEAKS.json)",
                         "flop_per_solve": fl, "kernel": "k_solve (persistent, one 2-warp CTA per scenario, 3 CTAs/SM)"},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches), "clocks": clk,
            "latency": {"batch": 1, "wall_clock": "solve_static_batch + cudaDeviceSynchronize", **lat},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
