MSV_INPUT_REGIONS=3 MSV_TEST_WAVE_MB=60 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "multi_wave" 2>&1 | tail -1
for rep in 1 2; do for cfg in "MSV_INPUT_REGIONS=2" "MSV_INPUT_REGIONS=3" "MSV_INPUT_REGIONS=3 MSV_WAVE_PCT=80"; do env $cfg MSV_HOST_TIMING=1 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/b.log 2>&1; echo -n "$cfg: "; grep -m1 "wave(s)" gpurun_out/b.log | cut -c20-60 | tr '\n' ' '; tail -1 gpurun_out/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e9,3), round(d['e2e']['value']/1e9,3), round(d['ms_per_step'],2))"; done; done
MSV_INPUT_REGIONS=3 MSV_WAVE_PCT=80 MSV_TIMELINE=1 timeout 900 python -c "
import sys; sys.path.insert(0,'.')
from paper_2202_13481_b200 import Engine
from paper_2202_13481_b200 import workloads as W
eng=Engine(0); specs=W.c5()
g=eng.grid(specs); g.set_usage(False)
g.launch(); eng.synchronize()
g.launch(); eng.synchronize()
" > gpurun_out/timeline3.log 2>&1; grep timeline gpurun_out/timeline3.log | tail -14
