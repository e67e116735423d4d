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

# paper scale: 8 GPUs (56 GPCs), BERT, every homogeneous design + PARIS, ELSA and FIFS
from concurrent.futures import ThreadPoolExecutor
m = W.model("bert_base")
designs = [S.Design(plan, sched, m.table, m.dist, m.sla, opt)
           for plan in [W.paris(m, 8)] + [homogeneous_plan(k, 56, 8, 7) for k in (1, 2, 3, 7)]
           for sched in ("elsa", "fifs")]
S.latency_bounded_throughput(eng, designs[:1])
t0 = time.perf_counter(); got = S.latency_bounded_throughput(eng, designs); dt = time.perf_counter() - t0
with ThreadPoolExecutor(len(designs)) as ex:  # the reference drivers, one design per thread
    t0 = time.perf_counter()
    want = list(ex.map(lambda d: ref.lbt(d.plan, d.scheduler, m.table, m.sla, m.dist, opt), designs))
    ct = time.perf_counter() - t0
sims = sum(g.sims_run for g in got)
print(f"LBT 8 GPUs, PARIS + 4 homogeneous x elsa/fifs ({sims} simulations of 20 s): device {dt:.2f} s, "
      f"reference {ct:.2f} s on {len(designs)} threads, equal {[(g.qps, g.infeasible_at_min, g.sims_run) for g in got] == want}",
      flush=True)
print("  qps:", [round(g.qps, 3) for g in got], flush=True)
