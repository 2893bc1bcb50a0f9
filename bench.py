#!/usr/bin/env python
"""Benchmark: repetend candidates evaluated/s and time-to-optimal of the
schedule search (BASELINE.json metric) on BASELINE.json configs[1]: the
X-shape (Chimera-style) placement, 8 devices, 8 micro-batches (max_nr=8),
GPT-style fwd:bwd 1:2.  The search ends at the load bound
t_R = 6 in N_R = 5 after 10.6 M candidates; every step is checked
bit-exactly against the reference's golden result for the same call
(tests/golden/search_C2_8.json, ~1 h of the reference's CPU search).

A step = one full ``completion.search()`` (repetend phase over all
candidates + warmup/cooldown completion).

  value  candidates / s of the whole search step (wall time, device
         synchronised, max over ranks) with the engine resident: placement
         and frontier count tables already in HBM.  The engine-kernel device
         time is reported beside it (engine_kernel_s_per_step, roofline).
  e2e    the same metric through the public API from host objects:
         search(PlacementSpec) -> Schedule with a fresh engine per step, all
         host<->device traffic inside the timed region;
         e2e.time_to_optimal_s is its per-step wall time.

Multi-GPU (``--gpus N``; started under torch.distributed.run by the driver,
or by this script itself when no rank environment is present): the search
is SHARDED — every candidate window is split by rank prefix across the
GPUs, each GPU scans its share with no collective inside the scan, and per
window one all-gather of first-SAT rows plus one broadcast of rank 0's
replay decisions keep every rank on the same bound (parallel.py).  Total
work is fixed (scaling "strong"); value = candidates / max-over-ranks time.

``--impl reference`` times the reference's own CPU search (oracle/_ref, the
unmodified reference package built here; else the oracle port) on the host.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
os.environ.setdefault("TESSEL_BUDGET_SECS", "1e9")

BASE = json.loads((ROOT / "BASELINE.json").read_text())
METRIC = BASE["metric"]
UNIT = "candidates/s"
DEFAULT_WORKLOAD = "C2@8"
GOLDEN = {"C2@8": "C2_8", "C2@4": "C2_4", "C2@3": "C2_3", "C1": "C1", "C3@9": "C3_9", "C5@2": "C5_2",
          "C5@3": "C5_3", "C4b": "C4b", "C3@12": "C3_12", "C4a@3": "C4a_3", "C4a@4": "C4a_4",
          "C5@4": "C5_4", "C5@5": "C5_5"}


def _env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0, period=None):
        self.index = index
        self.period = float(os.environ.get("BENCH_CLOCK_PERIOD", "0.2")) if period is None else period
        self.rows, self._stop = [], threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _nvml(self):
        """In-process NVML sampler (same fields as the nvidia-smi query): a
        fresh nvidia-smi process every period initialises NVML each time and
        measurably stalled the e2e leg's CUDA allocation calls."""
        try:
            import pynvml as nv

            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            get = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                nv.nvmlDeviceGetCurrentClocksThrottleReasons
            bits = (0x8, 0x40, 0x20, 0x4)  # hw_slowdown, hw_thermal, sw_thermal, sw_power_cap

            def sample():
                r = get(h)
                return [str(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)), str(mx)] + \
                    ["Active" if r & b else "Not Active" for b in bits]
            sample()
            return sample
        except Exception:
            return None

    def _run(self):
        if self.period <= 0:  # diagnosis only: no sampling
            self.source = "off"
            return
        sample = self._nvml()
        self.source = "nvml (in-process)" if sample is not None else "nvidia-smi"
        while not self._stop.is_set():
            try:
                if sample is not None:
                    self.rows.append(sample())
                else:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                                          "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits"], capture_output=True,
                                         text=True, timeout=5).stdout.strip()
                    if out:
                        self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(self.period)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 2 + i and r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows), "sampler": getattr(self, "source", None)}


def _flush_l2(torch, dev):
    buf = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    buf.fill_(1)
    torch.cuda.synchronize(dev)


def _golden(workload):
    name = GOLDEN.get(workload)
    path = ROOT / "tests" / "golden" / f"search_{name}.json"
    return json.loads(path.read_text()) if name and path.exists() else None


def _matches(res, doc):
    if doc is None:
        return None
    s = res.schedule
    return (res.report.best_t_r == doc["best_t_r"]
            and [[list(a), t] for a, t in res.report.improvements] == doc["improvements"]
            and len(res.report.candidates) == doc["n_candidates"]
            and sorted([b.stage, b.mb, t] for b, t in s.entries.items())
            == doc["schedule"]["entries"]
            and s.makespan() == doc["schedule"]["makespan"])


def reference_search(p, cap, max_nr, budget, jobs):
    """The reference's own CPU search (oracle/_ref) or, if absent, the oracle
    port.  Returns (kind, candidates, wall, timed_out)."""
    import oracle

    ref = oracle.load_reference()
    if ref is not None:
        from repsched import completion as RC
        from repsched import placement as RP

        from paper_2311_15269_b200.placement import placement_to_dict

        rp = RP.placement_from_dict(placement_to_dict(p))
        t0 = time.perf_counter()
        res = RC.search(rp, cap, max_nr=max_nr, budget=budget, jobs=jobs)
        wall = time.perf_counter() - t0
        return "reference", len(res.report.candidates), wall, res.report.timed_out
    from oracle import search_port

    res = search_port.search(p, cap, max_nr, time_limit=budget)
    return "port", res.n_candidates, res.wall, res.schedule is None


def run_reference_arm(args):
    """The reference's own CPU search on the host: every step times a
    bounded sample with jobs=1 (the reference default) and jobs=nproc (its
    process-pool fan-out) and keeps the better rate."""
    rank, world, _ = _env_rank()
    if rank != 0:
        return
    from paper_2311_15269_b200.workloads import WORKLOADS

    w = WORKLOADS[args.workload]
    p = w.placement()
    nproc = os.cpu_count() or 1
    vals, walls, kinds, per_jobs = [], [], set(), {1: [], nproc: []}
    for i in range(args.warmup + args.steps):
        best = None
        for jobs in sorted(per_jobs):
            kind, n, wall, _ = reference_search(p, w.mem_capacity, w.max_nr, args.ref_sample_secs,
                                                jobs)
            kinds.add(kind)
            if i >= args.warmup:
                per_jobs[jobs].append(n / wall)
            if best is None or n / wall > best[0]:
                best = (n / wall, wall, jobs)
        if i >= args.warmup:
            vals.append(best[0])
            walls.append(best[1])
    v = statistics.mean(vals)
    rates = {f"jobs={j}": statistics.mean(r) for j, r in per_jobs.items() if r}
    best_jobs = max(rates, key=rates.get)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * statistics.mean(walls), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": {"workload": f"{args.workload}: {w.note}", "max_nr": w.max_nr,
                   "mem_capacity": w.mem_capacity,
                   "sample": f"search() with budget={args.ref_sample_secs}s per step and "
                             f"jobs setting, better of jobs=1 / jobs={nproc}"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": int(best_jobs.split("=")[1]),
                         "kind": kinds.pop(), "rates": rates,
                         "sample": f"reference completion.search on the host, wall budget "
                                   f"{args.ref_sample_secs}s per step, better of jobs=1 and "
                                   f"jobs={nproc} (BASELINE.md §3.4)"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _roofline(kernel_ms: dict, steps: int, workload: str):
    """Issue roofline of the dominant kernel (largest live CUDA-event time).

    achieved = warp instructions the kernel issues per step (deterministic
    for a given workload; counted once with ncu smsp__inst_executed.sum over a
    full search, committed in profiles/inst_counts.json) ÷ the kernel's live
    per-step time measured here with CUDA events on the engine stream.
    peak = 148 SMs x 4 warp-schedulers x 1 instr/clk x sm_max_mhz."""
    peaks = {}
    mp = ROOT / "MEASURED_PEAKS.json"
    if mp.exists():
        peaks = json.loads(mp.read_text())
    mhz = peaks.get("sm_max_mhz", 1965.0)
    hbm = peaks.get("hbm_gbs", 6457.4)
    peak = 148 * 4 * mhz * 1e6
    kern = max(kernel_ms, key=kernel_ms.get)
    out = {"bound": "issue", "unit": "warp-inst/s", "peak": peak, "kernel": kern,
           "kernel_ms_per_step": {k: v / steps for k, v in kernel_ms.items()},
           "peak_basis": f"148 SMs x 4 issue/clk x {mhz} MHz (MEASURED_PEAKS sm_max_mhz)",
           "achieved": None, "frac": None, "traffic": None}
    ip = ROOT / "profiles" / "r02_int_peak.json"
    if ip.exists():  # INT32 lane throughput measured on the box (scripts/int_peak.cu)
        d = json.loads(ip.read_text())
        out["int32_measured"] = {
            "lop3_lanes_per_sm_clk": d["lop3_lanes_per_sm_clk"],
            "iadd3_lanes_per_sm_clk": d["iadd_lanes_per_sm_clk"],
            "alu_warp_inst_peak_per_s": d["lop3_ops_per_s"] / 32,
            "basis": "scripts/int_peak.cu on a B200 (profiles/r02_int_peak.json): the ALU "
                     "pipe retires 64 int32 lanes/SM/clk = half the warp-issue peak"}
    prof = ROOT / "profiles" / "inst_counts.json"
    if prof.exists():
        d = json.loads(prof.read_text())
        ps = d.get("per_step", {}) if d.get("workload") == workload else {}
        k = ps.get(kern)
        if k and kernel_ms[kern] > 0:
            ach = k["warp_inst"] / (kernel_ms[kern] / steps / 1e3)
            out.update(achieved=ach, frac=ach / peak, traffic=k.get("dram_bytes"),
                       traffic_basis="ncu dram__bytes_read+write per step for this kernel",
                       basis=d.get("basis"))
        # every timed kernel against the same issue peak (and its HBM bytes)
        out["kernels"] = {
            name: {"ms_per_step": ms / steps,
                   "warp_inst_per_step": ps[name]["warp_inst"],
                   "issue_frac": ps[name]["warp_inst"] / (ms / steps / 1e3) / peak,
                   "dram_bytes_per_step": ps[name]["dram_bytes"],
                   "hbm_frac": ps[name]["dram_bytes"] / (ms / steps / 1e3) / (hbm * 1e9)}
            for name, ms in kernel_ms.items() if name in ps and ms > 0}
    return out


def _device_sync(torch, dev):
    if dev.type == "cuda":
        torch.cuda.synchronize(dev)


def run_b200_arm(args):
    import torch

    rank, world, local = _env_rank()
    cuda = torch.cuda.is_available()
    dev = torch.device("cuda", local) if cuda else torch.device("cpu")
    dist = None
    if world > 1:
        import torch.distributed as dist

        if cuda:
            dist.init_process_group("nccl", device_id=dev)
        else:  # CPU protocol check (tests/test_bench.py): gloo, engine patched by the test
            dist.init_process_group("gloo")
    if cuda:
        torch.cuda.set_device(local)

    from paper_2311_15269_b200 import _native
    from paper_2311_15269_b200.completion import search
    from paper_2311_15269_b200.engine import BatchedRepetendSearch
    from paper_2311_15269_b200.workloads import WORKLOADS

    _native.build()
    if cuda:
        _native.lib().tsl_set_device(local)
    w = WORKLOADS[args.workload]
    p = w.placement()
    golden = _golden(args.workload)

    comm = None
    if world > 1:
        from paper_2311_15269_b200.parallel import Comm

        comm = Comm(device=dev)
    eng = BatchedRepetendSearch(p, local)      # placement tables resident in HBM
    for _ in range(args.warmup):
        res = search(p, w.mem_capacity, max_nr=w.max_nr, engine=eng, comm=comm)
    parity = _matches(res, golden) if args.warmup else None
    if args.warmup:  # the e2e leg's path (fresh engine per call) warmed once too
        parity = parity and _matches(
            search(p, w.mem_capacity, max_nr=w.max_nr, device=local, comm=comm), golden)

    per_kernel = {"k_root": 0.0, "k_resolve_warp": 0.0, "k_verify_warp": 0.0, "k_stage": 0.0}
    cands = 0
    walls, e2e_walls = [], []
    stats = {"probes": 0, "nodes": 0, "capped": 0, "root_refuted": 0, "levels": 0,
             "dj_nodes": 0, "verified": 0}
    phase = {"repetend": 0.0, "warmup": 0.0, "cooldown": 0.0}
    c = eng.counters
    sp0 = _native.sp_stats()  # subtree-parallel completion decides (host-timed rounds)

    def check(res):
        nonlocal parity
        ok = _matches(res, golden)
        parity = ok if parity is None else (parity and ok)

    # the cyclic GC stays off over both timed legs (search() pauses it
    # itself; between steps a full collection over the results still held
    # added 0.3-0.7 s to single e2e steps, profiles/r02l_bench_line.json)
    gc.collect()
    gc.disable()
    with ClockSampler(local) as clk:
        # (1) value: the whole search step with the engine resident (its
        # placement tables and frontier count tables already in HBM)
        if dist:
            dist.barrier()
        _device_sync(torch, dev)
        c0 = _native.counters()
        for _ in range(args.steps):
            if cuda:
                _flush_l2(torch, dev)           # L2 flushed between timed steps
            k0 = (c.root_ms, c.probe_ms + c.resolve_ms, c.verify_ms, c.stage_ms)
            n0 = {k: getattr(c, k) for k in stats}
            _device_sync(torch, dev)
            t0 = time.perf_counter()
            res = search(p, w.mem_capacity, max_nr=w.max_nr, engine=eng, comm=comm)
            _device_sync(torch, dev)
            walls.append(time.perf_counter() - t0)
            per_kernel["k_root"] += c.root_ms - k0[0]
            per_kernel["k_resolve_warp"] += c.probe_ms + c.resolve_ms - k0[1]
            per_kernel["k_verify_warp"] += c.verify_ms - k0[2]
            per_kernel["k_stage"] += c.stage_ms - k0[3]
            cands += len(res.report.candidates)
            for k in stats:
                stats[k] += getattr(c, k) - n0[k]
            for k in phase:
                phase[k] += res.report.phase_secs[k]
            check(res)
        c1 = _native.counters()
        sp1 = _native.sp_stats()
        # (2) e2e: the public API from host objects — PlacementSpec in,
        # Schedule out, a fresh engine per step (placement tables uploaded,
        # count tables built), every host<->device copy inside the timed region
        for _ in range(args.steps):
            if cuda:
                _flush_l2(torch, dev)
            _device_sync(torch, dev)
            t0 = time.perf_counter()
            res = search(p, w.mem_capacity, max_nr=w.max_nr, device=local, comm=comm)
            _device_sync(torch, dev)
            e2e_walls.append(time.perf_counter() - t0)
            check(res)
        c2 = _native.counters()
        if dist:
            dist.barrier()
    gc.enable()
    launches = c1["launches"] - c0["launches"]
    wall, e2e_wall = sum(walls), sum(e2e_walls)
    if dist:
        t = torch.tensor([wall, e2e_wall, float(not parity)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        wall, e2e_wall, parity = float(t[0]), float(t[1]), not bool(t[2])
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    clocks = clk.summary()
    kernel_s = sum(per_kernel.values()) / 1e3
    per_step = {k: v // args.steps for k, v in stats.items()}
    line = {
        "metric": METRIC,
        "value": cands / wall,
        "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * wall / args.steps, "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": {"workload": f"{args.workload}: {w.note}", "max_nr": w.max_nr,
                   "mem_capacity": w.mem_capacity, "candidates_per_step": cands // args.steps,
                   "parallelism": f"sharded{world} (rank-prefix windows)" if world > 1
                   else "single",
                   "l2": "flushed between timed steps (256 MiB write)"},
        "value_basis": "candidates / wall time of the whole search step (repetend scan, "
                       "replay, completion) with the engine resident; max over ranks",
        "time_to_optimal_s": wall / args.steps,
        "parity_vs_reference": parity,
        "e2e": {"value": cands / e2e_wall, "unit": UNIT,
                "time_to_optimal_s": e2e_wall / args.steps,
                "h2d_bytes_per_step": (c2["h2d_bytes"] - c1["h2d_bytes"]) // args.steps,
                "d2h_bytes_per_step": (c2["d2h_bytes"] - c1["d2h_bytes"]) // args.steps,
                "basis": "search(PlacementSpec) -> Schedule through the public API, fresh "
                         "engine per step",
                "step_walls_s": [round(x, 4) for x in e2e_walls]},
        "step_walls_s": [round(x, 4) for x in walls],
        "gpu_launches": launches,
        "work_per_step": per_step,
        "rates": {"candidates_per_s": cands / wall,
                  "probes_per_s": stats["probes"] / wall,
                  "dfs_nodes_per_s": stats["nodes"] / wall,
                  "dj_nodes_per_s": stats["dj_nodes"] / wall},
        "phase_s_per_step": {k: v / args.steps for k, v in phase.items()},
        "engine_kernel_s_per_step": kernel_s / args.steps,
        "completion_sp_per_step": {
            k: (sp1.get(k, 0) - sp0.get(k, 0)) / args.steps
            for k in ("master_ms", "task_ms", "master_nodes", "tasks", "rounds")},
        "clocks": clocks,
        "roofline": _roofline(per_kernel, args.steps, args.workload),
    }
    if not args.no_cpu_baseline:
        kind, n, cwall, _ = reference_search(p, w.mem_capacity, w.max_nr, args.ref_sample_secs, 1)
        line["cpu_baseline"] = {"value": n / cwall, "unit": UNIT, "cores": 1, "kind": kind,
                                "sample": f"{args.workload} search(jobs=1) on the host, wall "
                                          f"budget {args.ref_sample_secs}s ({n} candidates)"}
        if golden:
            line["cpu_baseline"]["reference_time_to_optimal_s_container"] = golden["ref_wall_secs"]
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def launch_ranks(args) -> int:
    """`--gpus N` without a torch.distributed environment: start one rank per
    GPU under torch.distributed.run (127.0.0.1 rendezvous) and return its
    exit code; rank 0 prints the JSON line."""
    import socket

    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           str(ROOT / "bench.py"), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD)
    ap.add_argument("--ref-sample-secs", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(launch_ranks(args))
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_b200_arm(args)


if __name__ == "__main__":
    main()
