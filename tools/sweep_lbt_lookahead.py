import sys, time
sys.path.insert(0, "/root/repo")
from paper_2202_13481_b200 import Engine, homogeneous_plan
from paper_2202_13481_b200 import search as S
from paper_2202_13481_b200 import workloads as W
eng = Engine(0)
opt = S.LbtOptions(duration_ms=20000.0, seeds=(1, 2, 3))
m = W.model("bert_base")
designs = [S.Design(plan, sched, m.table, m.dist, m.sla, opt)
           for plan in [W.paris(m, 8)] + [homogeneous_plan(k, 56, 8, 7) for k in (1, 2, 3, 7)]
           for sched in ("elsa", "fifs")]
S.latency_bounded_throughput(eng, designs[:2])
base = None
for L in (1, 2, 3, 4, 5, 6):
    t0 = time.perf_counter(); got = S.latency_bounded_throughput(eng, designs, lookahead=L); dt = time.perf_counter() - t0
    key = [(g.qps, g.infeasible_at_min, g.sims_run) for g in got]
    base = base or key
    print(f"lookahead {L}: {dt:.3f} s, same as L=1: {key == base}", flush=True)
