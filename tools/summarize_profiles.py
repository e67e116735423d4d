#!/usr/bin/env python3
"""Summarise ncu captures of the bench command into profiles/<round>/.

    python tools/summarize_profiles.py r01 gpurun_out/r01/full.ncu-rep [more.ncu-rep ...] \
        --launches gpurun_out/r01/launches.csv --bench gpurun_out/r01/bench.log \
        --reference gpurun_out/r01/bench_ref.log

The first report holds every kernel of ONE bench step (all chunks); each kernel's
launches are summed (time, warp instructions, DRAM bytes) and divided by the step's
simulated queries. Writes <kernel>_raw.csv (ncu --page raw, one row per launch),
sim_opcodes.csv (SASS opcode histogram of one K2 launch, from a report holding only
that launch: --opcodes), launches_bench.csv and summary.json, plus each kernel's share
of the launch list. Times under ncu are serialised and cold-cache: the shares, not the
absolutes, compare with bench.py.
"""
from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import re
import shutil
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
SHORT = {"trace_gen_kernel": "K1 trace_gen_kernel", "trace_group_kernel": "K1 trace_group_kernel",
         "sim_warp_kernel": "K2 sim_warp_kernel",
         "sim_kernel": "K2 sim_kernel (segmented)", "tail_kernel": "K3 tail_kernel", "paris_kernel": "K4 paris_kernel"}
METRICS = {
    "duration_ms": "gpu__time_duration.sum",
    "warp_instructions": "smsp__inst_executed.sum",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "registers": "launch__registers_per_thread",
    "warps_active_per_sm": "sm__warps_active.avg.per_cycle_active",
    "grid": "launch__grid_size",
    "threads_per_instruction": "smsp__thread_inst_executed_per_inst_executed.ratio",
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ms": 1, "us": 1e-3, "ns": 1e-6}


def ncu_csv(rep: Path, *args) -> list[list[str]]:
    out = subprocess.run(["ncu", "-i", str(rep), *args, "--csv"], capture_output=True, text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def short(name: str) -> str:
    for k, v in SHORT.items():
        if re.search(rf"\b{k}\b", name):
            return v
    return name


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("round")
    ap.add_argument("reps", nargs="+", type=Path)
    ap.add_argument("--launches", type=Path)
    ap.add_argument("--bench", type=Path)
    ap.add_argument("--reference", type=Path)
    ap.add_argument("--opcodes", type=Path, default=None, help="report holding one K2 launch (source page)")
    ap.add_argument("--note", default=None, help="what the capture is (command, grid)")
    ap.add_argument("--queries-per-step", type=float, default=None,
                    help="simulated queries of the captured step (default: from the bench line)")
    ap.add_argument("--k2-class", action="append", default=[], metavar="LABEL@REPORT:QUERIES:WHAT",
                    help="standalone capture of one K2 launch (tools/prof_k2.py, MSV_MAX_CHUNKS=1) and "
                         "the queries it simulated")
    a = ap.parse_args()
    out = ROOT / "profiles" / a.round
    out.mkdir(parents=True, exist_ok=True)
    bench = None
    if a.bench and a.bench.exists():
        lines = [l for l in a.bench.read_text().splitlines() if l.startswith("{")]
        bench = json.loads(lines[-1]) if lines else None
        if bench:
            (out / "bench_line.json").write_text(json.dumps(bench, indent=1) + "\n")
    if a.reference and a.reference.exists():
        lines = [l for l in a.reference.read_text().splitlines() if l.startswith("{")]
        if lines:
            (out / "bench_reference_line.json").write_text(json.dumps(json.loads(lines[-1]), indent=1) + "\n")
    qps = a.queries_per_step
    if qps is None and bench:
        cfg = bench["config"]
        qps = cfg.get("scenarios", cfg.get("scenarios_per_gpu")) * cfg["queries_per_scenario"]
    ADD = ("duration_ms", "warp_instructions", "dram_read", "dram_write")
    kernels, raw = {}, collections.defaultdict(list)
    # the first report holds the step; a later report (e.g. one kernel captured alone, when
    # kernel replay returned no counters for it inside the step) replaces that kernel's rows
    reports, seen = [], set()
    for rep in reversed(a.reps):
        rr = ncu_csv(rep, "--page", "raw")
        h = rr[0]
        keep = [r for r in rr[2:] if short(r[h.index("Kernel Name")]) not in seen]
        seen |= {short(r[h.index("Kernel Name")]) for r in rr[2:]}
        reports.append((h, rr[1], keep))
    for head, units, body in reports:
        for r in body:
            name = short(r[head.index("Kernel Name")])
            vals = {}
            for key, m in METRICS.items():
                if m not in head:
                    continue
                i = head.index(m)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                if key.startswith("dram"):
                    v *= UNIT.get(units[i], 1)
                elif key == "duration_ms":
                    v *= UNIT.get(units[i], 1) if units[i] != "ms" else 1
                vals[key] = v
            raw[name].append((head, units, r))
            k = kernels.setdefault(name, {"kernel": r[head.index("Kernel Name")], "launches": 0,
                                          **{x: 0.0 for x in ADD}, "_w": {}})
            k["launches"] += 1
            for x in ADD:
                k[x] += vals.get(x, 0.0)
            # duration-weighted means of the rates, instruction-weighted lane occupancy
            for x, wkey in (("issue_active_pct", "duration_ms"), ("warps_active_per_sm", "duration_ms"),
                            ("threads_per_instruction", "warp_instructions")):
                if x in vals:
                    acc = k["_w"].setdefault(x, [0.0, 0.0])
                    acc[0] += vals[x] * vals.get(wkey, 0.0)
                    acc[1] += vals.get(wkey, 0.0)
            for x in ("registers", "grid"):
                if x in vals:
                    k.setdefault(x + "_per_launch", []).append(vals[x])
    for name, k in kernels.items():
        for x, (num, den) in k.pop("_w").items():
            k[x] = num / den if den else None
        k["traffic_bytes_per_step"] = k["dram_read"] + k["dram_write"]
        if qps:
            samples = 0.9 if name.startswith("K3") else 1.0  # K3 reads the measured (post-warm-up) latencies
            k["warp_instructions_per_query"] = k["warp_instructions"] / qps
            k["traffic_bytes_per_query"] = k["traffic_bytes_per_step"] / (qps * samples)
        with open(out / f"{name.split()[0].lower()}_{name.split()[1]}_raw.csv", "w", newline="") as f:
            h, u = raw[name][0][0], raw[name][0][1]
            csv.writer(f).writerows([h, u, *[r for _, _, r in raw[name]]])
    if a.opcodes and a.opcodes.exists():
        src = ncu_csv(a.opcodes, "--page", "source", "--print-source", "cuda,sass")
        ops, tot = collections.Counter(), 0
        for r in src:
            if len(r) > 8 and r[0] == "" and r[2].startswith("0x"):
                try:
                    n = int(r[7])
                except ValueError:
                    continue
                t = re.sub(r"^@!?U?P\w+\s+", "", r[3].strip())
                ops[t.split()[0] if t else "?"] += n
                tot += n
        with open(out / "sim_opcodes.csv", "w", newline="") as f:
            w = csv.writer(f)
            w.writerow(["opcode", "warp_instructions", "share"])
            for o, n in ops.most_common():
                w.writerow([o, n, round(n / tot, 5)])
    shares = {}
    if a.launches and a.launches.exists():
        shutil.copy(a.launches, out / "launches_bench.csv")
        tot = collections.defaultdict(float)
        cnt = collections.Counter()
        for r in csv.reader(open(a.launches)):
            if len(r) > 10 and r[0].isdigit() and r[-3] == "gpu__time_duration.sum":
                k = short(r[4])
                tot[k] += float(r[-1].replace(",", ""))
                cnt[k] += 1
        s = sum(tot.values())
        shares = {k: {"launches": cnt[k], "total_ms": round(v / 1e6, 3), "share": round(v / s, 4)}
                  for k, v in tot.items()}
    import hashlib
    csrc = ROOT / "paper_2202_13481_b200" / "csrc"
    sha = hashlib.sha256(b"".join(p.read_bytes() for p in (csrc / "msv_sim_warp.cu", csrc / "msv_sim.cu"))).hexdigest()
    summary = {
        "note": a.note or ("ncu --set full --clock-control none capture of every kernel of one bench step on one "
                           "B200; per kernel: its launches in the step summed, per-query figures over the step's "
                           "queries. ncu times are serialised / cold-cache: compare shares, not absolutes."),
        "kernel_sources_sha256": sha,
        "queries_per_step": qps,
        "issue_peak_warp_inst_per_s": "148 SMs x 4 schedulers x SM clock (1 warp-instruction / scheduler / clk)",
        "kernels": kernels,
        "launch_shares_bench": shares,
    }
    if a.k2_class:
        classes = {}
        for spec in a.k2_class:
            label, rest = spec.split("@", 1)
            rep, queries, what = rest.split(":", 2)
            rows = ncu_csv(Path(rep), "--page", "raw")
            head, units = rows[0], rows[1]
            r = rows[2]
            val = lambda m: float(r[head.index(m)].replace(",", ""))
            q = float(queries)
            dram = (val(METRICS["dram_read"]) * UNIT.get(units[head.index(METRICS["dram_read"])], 1) +
                    val(METRICS["dram_write"]) * UNIT.get(units[head.index(METRICS["dram_write"])], 1))
            classes[label] = {"capture": what, "queries": q,
                              "warp_instructions_per_query": val(METRICS["warp_instructions"]) / q,
                              "threads_per_instruction": val(METRICS["threads_per_instruction"]),
                              "dram_bytes_per_query": dram / q,
                              "duration_ms": val(METRICS["duration_ms"]),
                              "issue_active_pct": val(METRICS["issue_active_pct"]),
                              "warps_active_per_sm": val(METRICS["warps_active_per_sm"]),
                              "registers": val(METRICS["registers"])}
        summary["k2_classes_standalone"] = classes
    def finite(x):  # counters ncu could not collect are NaN: null in the JSON
        if isinstance(x, float) and x != x:
            return None
        if isinstance(x, dict):
            return {k: finite(v) for k, v in x.items()}
        if isinstance(x, list):
            return [finite(v) for v in x]
        return x
    summary = finite(summary)
    (out / "summary.json").write_text(json.dumps(summary, indent=1) + "\n")
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
