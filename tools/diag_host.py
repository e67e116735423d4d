"""Host-side share of an end-to-end grid call (C4: 6,870 small scenarios): marshalling
(Engine.prepare), the whole run_grid on prepared vs unprepared specs, and the library's
per-phase host timings (MSV_HOST_TIMING=1 prints them on stderr)."""
import sys
import time
sys.path.insert(0, "/root/repo")
from paper_2202_13481_b200 import Engine
from paper_2202_13481_b200 import workloads as W
eng = Engine(0)
specs, _ = W.c4()
eng.run_grid(specs)
for _ in range(3):
    t0 = time.perf_counter(); prep = eng.prepare(specs); t1 = time.perf_counter()
    eng.run_grid(prep); t2 = time.perf_counter()
    eng.run_grid(specs); t3 = time.perf_counter()
    print(f"prepare {1e3*(t1-t0):.1f} ms, run_grid(prepared) {1e3*(t2-t1):.1f} ms, run_grid(specs) {1e3*(t3-t2):.1f} ms", flush=True)
g = eng.grid(specs); g.set_usage(False); g.launch(); eng.synchronize()
t0 = time.perf_counter(); g.launch(); eng.synchronize(); t1 = time.perf_counter()
print(f"device-resident launch {1e3*(t1-t0):.1f} ms, timing {g.timing()}")
