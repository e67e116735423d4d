#!/usr/bin/env python3
"""Benchmark: simulated queries/s over the PARIS x ELSA scenario grid.

Workload (BASELINE.json configs[4], "C5" — the grid the metric names): 10^4 scenarios
x 10^6 expected queries. 75 cells = 3 model presets (MobileNet / ResNet-50 / BERT-base)
x 5 plans (the model's 8-GPU PARIS plan and homogeneous 1g/2g/3g/7g fleets of 56
GPCs: 8..56 partitions) x 5 loads (30..90 % of the plan's nominal capacity), ELSA,
lognormal(1,1) batches over 1..32, SLA = 1.5 x latency(7g, 32); scenario i = cell
i mod 75 with seed 1 + i // 75. One step = the whole grid: device trace generation
(sample_trace), simulation (run), exact p95/p99 selection (tail_latency).

N > 1 GPUs (torchrun, one process per GPU): strong scaling — the same grid is cut
into cost-balanced contiguous shards (distributed.shard_bounds), each rank simulates
its shard with no data-path collective; the end-to-end leg then all-gathers the
fixed-size per-scenario results (NCCL) and every rank takes the PARIS argmin (best plan
per model and load by mean p99).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c5|c2] [--scenarios S] [--queries Q]
"""
from __future__ import annotations

import argparse
import hashlib
import json
import math
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "simulated queries/sec over PARIS×ELSA scenario grid at 1/2/4/8 B200 vs CPU"
UNIT = "queries/s"
SIM_BYTES_PER_QUERY = 20  # arrival f64 + batch i32 read, measured latency f64 written
TAILS = (0.95, 0.99)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c5", choices=["c5", "c2"])
    ap.add_argument("--scenarios", type=int, default=10_000, help="C5: scenarios in the grid")
    ap.add_argument("--seeds", type=int, default=1024, help="C2: seeds per load level")
    ap.add_argument("--queries", type=float, default=None, help="expected queries per scenario")
    ap.add_argument("--cpu-seconds", type=float, default=20.0, help="CPU baseline sample budget (s)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    a = ap.parse_args()
    if a.queries is None:
        a.queries = 1e6 if a.workload == "c5" else 1e5
    return a


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), \
        int(os.environ.get("LOCAL_RANK", "0"))


def workload(args, reference: bool = False):
    """The scenario list (whole grid). The reference arm builds it from oracle/_ref alone
    (tests/ref_workloads.py), so that process never maps the product library."""
    if reference:
        from tests import ref_workloads as W
    else:
        from paper_2202_13481_b200 import workloads as W
    if args.workload == "c5":
        return W.c5(n_scenarios=args.scenarios, queries=args.queries)
    return W.c2(seeds=args.seeds, queries=args.queries)


def config(args, world, specs):
    if args.workload == "c5":
        name = ("C5: large Monte-Carlo grid, %d scenarios x %.0e queries (3 models x {PARIS 8-GPU, "
                "homogeneous 1g/2g/3g/7g} plans of 8-56 partitions x loads 0.3-0.9 x seeds), ELSA"
                % (args.scenarios, args.queries))
    else:
        name = "C2: BERT-base, 8-GPU PARIS plan (23 partitions), ELSA, load 10-100%% of peak, %d seeds" % args.seeds
    return {"workload": name, "scenarios": len(specs), "queries_per_scenario": args.queries, "n_gpus": world,
            "sharding": "strong: cost-balanced contiguous shards of one grid" if world > 1 else "single GPU",
            "l2": "inputs larger than L2 (traces ~12 B/query resident in HBM, >10 GB per step)",
            "trace": "generated on device every step (MT19937-64 + glibc-log1p transcription)"}


class ClockSampler:
    """SM clocks and throttle reasons sampled during the timed region, in process through
    NVML (an nvidia-smi process every 200 ms measurably perturbed the timed loop); falls
    back to nvidia-smi when NVML is unavailable."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index: int, interval: float = 0.25):
        self.index = index
        self.interval = interval
        self.rows: list[tuple[float, float, set]] = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._nvml = None
        try:
            import pynvml as nv
            nv.nvmlInit()
            # the process's CUDA ordinal -> NVML handle (honours CUDA_VISIBLE_DEVICES)
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            ordinal = int(vis.split(",")[index]) if vis and vis.split(",")[index].isdigit() else index
            self._h = nv.nvmlDeviceGetHandleByIndex(ordinal)
            self._bits = {nv.nvmlClocksEventReasonHwSlowdown: "hw_slowdown",
                          nv.nvmlClocksEventReasonHwThermalSlowdown: "hw_thermal_slowdown",
                          nv.nvmlClocksEventReasonSwThermalSlowdown: "sw_thermal_slowdown",
                          nv.nvmlClocksEventReasonSwPowerCap: "sw_power_cap"}
            self._nvml = nv
        except Exception:
            self._nvml = None

    def _sample(self):
        nv = self._nvml
        if nv is not None:
            sm = float(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
            mx = float(nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM))
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            return [(sm, mx, {name for bit, name in self._bits.items() if r & bit})]
        out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
        rows = []
        for line in out.stdout.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 6 and f[0].replace(".", "").isdigit():
                rows.append((float(f[0]), float(f[1]), {self.NAMES[i] for i in range(4) if f[2 + i] == "Active"}))
        return rows

    def _run(self):
        while not self._stop.is_set():
            try:
                self.rows += self._sample()
            except Exception:
                pass
            self._stop.wait(self.interval)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        return {"sm_mhz": float(np.median([r[0] for r in self.rows])), "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": sorted(set().union(*(r[2] for r in self.rows))), "samples": len(self.rows),
                "source": "nvml" if self._nvml is not None else "nvidia-smi"}


def host_cores() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)


def cpu_sample(specs, budget_s: float, start: int = 0):
    """The reference's own CPU path (oracle/_ref: sample_trace -> run -> tail_latency) on
    every host core (one std::thread per core pulling scenarios), over a bounded sample:
    the `n` consecutive scenarios from `start` (C5 interleaves its 75 cells, so a run of
    consecutive scenarios covers every plan and load), n sized from a one-scenario probe
    so the sample is about `budget_s` of wall time."""
    from tests import oracle_py as O
    ora = O.best_oracle()
    cores = host_cores()
    t0 = time.perf_counter()
    ora.run_grid([specs[start % len(specs)]], TAILS, threads=1)
    per = max(time.perf_counter() - t0, 1e-3)
    n = int(max(cores, min(len(specs), budget_s * cores / per)))
    idx = [(start + j) % len(specs) for j in range(n)]
    sample = [specs[i] for i in idx]
    t0 = time.perf_counter()
    r = ora.run_grid(sample, TAILS, threads=cores)
    dt = time.perf_counter() - t0
    q = int(r["total"].sum())
    return {"value": q / dt, "unit": UNIT, "cores": cores, "kind": ora.kind,
            "sample": f"{len(sample)} consecutive scenarios of the grid from index {start} (every plan and load), "
                      f"{q} simulated queries, {dt:.1f} s wall on {cores} threads"}, r, idx


def run_reference(args):
    """--impl reference: the compiled reference (oracle/_ref) on the box's host cores, on
    this arm's config and metric; each step a bounded sample of the same grid."""
    rank, world, _ = dist_env()
    if world > 1 and rank != 0:
        return
    specs = workload(args, reference=True)
    vals, base, start = [], None, 0
    for i in range(args.warmup + args.steps):
        b, _, idx = cpu_sample(specs, max(args.cpu_seconds / 4.0, 4.0), start)
        start = (idx[-1] + 1) % len(specs)
        if i >= args.warmup:
            vals.append(b["value"])
            base = b
    val = float(np.median(vals))
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config(args, args.gpus, specs),
            "cpu_baseline": {**base, "value": val},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(finite(line), allow_nan=False), flush=True)


def finite(x):
    """The JSON line carries null, never NaN / inf (strict parsers reject them)."""
    if isinstance(x, float) and not math.isfinite(x):
        return None
    if isinstance(x, dict):
        return {k: finite(v) for k, v in x.items()}
    if isinstance(x, (list, tuple)):
        return [finite(v) for v in x]
    return x


def profile_summary(kernel_sources):
    """Per-launch DRAM traffic / instruction mix of K2 from the newest committed ncu summary,
    used only if it was captured from the kernel sources built now (sha256 match) — a stale
    capture is reported as such, never silently."""
    want = hashlib.sha256(b"".join(p.read_bytes() for p in kernel_sources)).hexdigest()
    for sp in sorted((ROOT / "profiles").glob("r*/summary.json"), reverse=True):
        try:
            js = json.loads(sp.read_text())
        except Exception:
            continue
        if "K2 sim_warp_kernel" not in js.get("kernels", {}):
            continue
        fresh = js.get("kernel_sources_sha256") == want
        return js, str(sp.relative_to(ROOT)), fresh
    return None, None, False


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    rank, world, local = dist_env()
    import torch
    import torch.distributed as td
    # one process per GPU; MSV_DIST_BACKEND=gloo exercises the multi-rank logic on a box
    # with fewer GPUs than ranks (ranks share devices; the only collectives are the
    # result exchange and the timing reductions, never inside the timed kernels)
    backend = os.environ.get("MSV_DIST_BACKEND", "nccl")
    dev = local % max(1, torch.cuda.device_count())
    coll = "cuda" if backend == "nccl" else "cpu"
    if world > 1:
        torch.cuda.set_device(dev)
        if backend == "nccl":
            td.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            td.init_process_group(backend)
    from paper_2202_13481_b200 import Engine
    from paper_2202_13481_b200 import distributed as D
    eng = Engine(dev)
    specs = workload(args)
    bounds = D.shard_bounds(specs, world)
    lo, hi = bounds[rank]
    mine = specs[lo:hi]

    def reduce(vals, op):
        t = torch.tensor(vals, dtype=torch.float64, device=coll if world > 1 else "cpu")
        if world > 1:
            td.all_reduce(t, op=op)
        return t.cpu().numpy()

    # ---- device-resident throughput (value): this rank's shard, traces regenerated per step ----
    grid = eng.grid(mine, TAILS)
    grid.set_usage(False)  # the metric needs counts and tails, not per-partition usage
    for _ in range(args.warmup):
        grid.launch()
    eng.synchronize()
    queries = grid.queries()
    launches0 = eng.kernel_launches()
    if world > 1:
        td.barrier()
    eng.synchronize()
    with ClockSampler(dev) as clk:
        eng.event_record(0)
        for _ in range(args.steps):
            grid.launch()
        eng.event_record(1)
        dev_ms = eng.event_elapsed_ms(0, 1)
    eng.synchronize()
    launches = eng.kernel_launches() - launches0
    res = grid.results()
    # per-stage timing of one more launch, stages back to back (events on the library stream)
    grid.set_overlap(False)
    grid.launch()
    stage = grid.timing()
    grid.set_overlap(True)
    grid.close()
    dev_ms_max = float(reduce([dev_ms], D_MAX(td))[0])
    total_q = float(reduce([float(queries)], D_SUM(td))[0])
    total_launches = int(reduce([float(launches)], D_SUM(td))[0])
    value = total_q * args.steps / (dev_ms_max / 1000.0)

    # ---- end to end through the public API with host buffers (e2e) ----
    # every step: msv_run_grid on this rank's shard (scenario descriptors H2D, trace/sim/
    # tails on the device, per-scenario results D2H into host buffers), the all-gather of
    # every rank's results (NCCL) and the PARIS argmin per model and load on every rank
    prepared = eng.prepare(mine)
    eng.run_grid(prepared, TAILS)  # untimed: sizes the context's reusable buffers
    h0, d0 = eng.transfer_bytes()
    labels = None
    if args.workload == "c5":
        from paper_2202_13481_b200 import workloads as W
        labels = W.c5_labels(len(specs))
    e2e_steps = max(1, min(args.steps, 3))
    if world > 1:
        td.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        full = D.run_sharded(specs, lambda sub: eng.run_grid(prepared, TAILS), rank, world,
                             device=coll if world > 1 else None)
        decision = D.grouped_argmin(full["tail"][:, 1], *labels) if labels else None
    e2e_s = time.perf_counter() - t0
    h1, d1 = eng.transfer_bytes()
    e2e_max = float(reduce([e2e_s], D_MAX(td))[0])
    e2e_value = total_q * e2e_steps / e2e_max
    assert np.array_equal(full["placement_hash"][lo:hi], res["placement_hash"]), \
        "e2e and device-resident runs disagree"

    if rank == 0:
        sim_s = stage["sim_ms"] / 1000.0
        peaks = {}
        try:
            peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        except Exception:
            pass
        peak = float(peaks.get("hbm_gbs", peaks.get("hbm_GBps", 6650.0)))
        csrc = ROOT / "paper_2202_13481_b200" / "csrc"
        prof, prof_src, fresh = profile_summary([csrc / "msv_sim_warp.cu", csrc / "msv_sim.cu"])
        sim_launches = max(1, round(launches / args.steps / 3))  # K1/K2/K3 once per chunk
        q_launch = queries / sim_launches
        # K2's per-query counters: the one-slot class (the bulk of the grid's queries)
        k2 = None
        if prof:
            cls = prof.get("k2_classes_standalone", {})
            one = next((v for kname, v in cls.items() if kname.startswith("one slot")), None)
            k2 = ({"warp_instructions_per_query": one["warp_instructions_per_query"],
                   "traffic_bytes_per_query": one["dram_bytes_per_query"]} if one
                  else prof["kernels"].get("K2 sim_warp_kernel"))
        traffic = k2["traffic_bytes_per_query"] * q_launch if (k2 and fresh and k2.get("traffic_bytes_per_query")) else None
        # K2's time in the timed (overlapped) step: its share of the launch list of this very
        # command (ncu, fresh capture) times the measured step time; the serialised stage
        # timing (stage_ms) is the fallback
        share = None
        if prof and fresh:
            share = (prof.get("launch_shares_bench", {}).get("K2 sim_warp_kernel") or {}).get("share")
        k2_s = (share * dev_ms_max / args.steps / 1000.0) if share else sim_s
        achieved = queries * SIM_BYTES_PER_QUERY / k2_s / 1e9
        clk_mhz = clk.summary().get("sm_mhz") or 1965.0
        issue = None
        if k2 and k2.get("warp_instructions_per_query"):
            sms = torch.cuda.get_device_properties(dev).multi_processor_count
            pk = sms * 4 * clk_mhz * 1e6  # one warp-instruction per scheduler per clock
            wk2 = k2["warp_instructions_per_query"]

            def per_q(name):
                v = (prof["kernels"].get(name) or {}).get("warp_instructions_per_query")
                return v if isinstance(v, (int, float)) and math.isfinite(v) else None
            # the whole step's mix (every K2 class, K1, K3) when the step capture has K2's counters
            step_k2 = per_q("K2 sim_warp_kernel")
            wi = (step_k2 if step_k2 is not None else wk2) + sum(
                per_q(kname) or 0.0 for kname in prof["kernels"] if kname.startswith(("K1", "K3")))
            issue = {"warp_inst_per_query_k2": wk2, "k2_basis": "one-slot K2 class (P <= 32), ncu source page",
                     "step_warp_inst_per_query": wi,
                     "step_basis": ("K1 + K2 (all classes) + K3 of the step capture" if step_k2 is not None
                                    else "one-slot K2 class + K1 + K3"),
                     "step_frac": wi * total_q * args.steps / (dev_ms_max / 1000.0) / world / pk,
                     "peak_warp_inst_per_s": pk, "source": prof_src, "fresh": fresh}
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": dev_ms_max / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic", "config": config(args, world, specs),
                "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": (h1 - h0) // e2e_steps,
                        "d2h_bytes_per_step": (d1 - d0) // e2e_steps,
                        "includes": "msv_run_grid with host buffers + all-gather + PARIS argmin"},
                "gpu_launches": total_launches,
                "stage_ms": {k: round(v, 3) for k, v in stage.items()},
                "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                             "frac": achieved / peak, "traffic": traffic,
                             "traffic_unit": "DRAM bytes per K2 launch (ncu, %d queries per launch)" % q_launch,
                             "traffic_source": (prof_src if fresh else f"stale capture {prof_src}: null")
                             if prof else None,
                             "algorithmic_bytes_per_launch": SIM_BYTES_PER_QUERY * q_launch,
                             "k2_time_s": k2_s, "k2_time_basis": ("K2 share %.4f of the ncu launch list x step time" % share)
                             if share else "serialised stage timing",
                             "kernel": "sim_warp_kernel (K2)", "issue": issue,
                             "note": "K2 is issue-bound (dependent FP64 state machine): 'issue' is the binding "
                                     "roof; HBM fraction is small by construction (DESIGN.md §4)"},
                "clocks": clk.summary()}
        if decision is not None:
            line["paris_decision"] = {f"{g[0]}@{g[1]}": best for g, (best, _) in sorted(decision.items())}
        if not args.no_cpu_baseline and world == 1:  # the CPU reference is timed at N=1 only
            b, ref, idx = cpu_sample(specs, args.cpu_seconds)
            line["cpu_baseline"] = b
            # the CPU sample doubles as a full-size parity check of the timed device run
            line["parity"] = {
                "scenarios_checked": len(idx), "queries_checked": int(ref["total"].sum()),
                "placement_hash_equal": bool(np.array_equal(res["placement_hash"][idx], ref["placement_hash"])),
                "tails_equal": bool(np.array_equal(res["tail"][idx], ref["tail"], equal_nan=True)),
                "counts_equal": bool(all(np.array_equal(res[k][idx], ref[k]) for k in
                                         ("total", "violations", "measured", "measured_violations"))),
                "against": b["kind"]}
        print(json.dumps(finite(line), allow_nan=False), flush=True)
    if world > 1:
        td.destroy_process_group()


def D_MAX(td):
    return td.ReduceOp.MAX


def D_SUM(td):
    return td.ReduceOp.SUM


if __name__ == "__main__":
    main()
