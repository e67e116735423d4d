"""LBT / GPU(max) search time: device lockstep drivers vs the compiled reference drivers."""
import sys, time
sys.path.insert(0, "/root/repo")
from paper_2202_13481_b200 import Engine
from paper_2202_13481_b200 import search as S
from paper_2202_13481_b200 import workloads as W
from tests import oracle_py as O
eng = Engine(0)
ref = O.Oracle("reference")
m = W.model("resnet50")
opt = S.LbtOptions(duration_ms=20000.0, seeds=(1, 2, 3))
from paper_2202_13481_b200 import homogeneous_plan
designs = [S.Design(plan, sched, m.table, m.dist, m.sla, opt)
           for plan in (W.paris(m, 1), homogeneous_plan(7, 7, 1, 7), homogeneous_plan(3, 7, 1, 7))
           for sched in ("elsa", "fifs")]
S.latency_bounded_throughput(eng, designs)
t0 = time.perf_counter(); got = S.latency_bounded_throughput(eng, designs); dt = time.perf_counter() - t0
t0 = time.perf_counter(); want = [ref.lbt(d.plan, d.scheduler, m.table, m.sla, m.dist, opt) for d in designs]; ct = time.perf_counter() - t0
print(f"LBT 3 plans x elsa/fifs, 20 s x 3 seeds: device {dt:.2f} s, reference {ct:.2f} s, "
      f"equal {[ (g.qps, g.infeasible_at_min, g.sims_run) for g in got] == want} {want}", flush=True)
t0 = time.perf_counter(); k, plan, r = S.best_homogeneous(eng, m.table, m.dist, m.sla, 7, 1, 7, opt); dt = time.perf_counter() - t0
t0 = time.perf_counter(); kr = ref.best_homogeneous(m.table, m.dist, m.sla, 7, 1, 7, opt.duration_ms, opt.seeds); ct = time.perf_counter() - t0
print(f"GPU(max) 1 GPU: device {dt:.2f} s, reference {ct:.2f} s, device {(k, r.qps, r.sims_run)} reference {kr}", flush=True)
