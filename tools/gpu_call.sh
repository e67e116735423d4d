P=gpurun_out/r02/wave
mkdir -p $P
for rep in 1 2; do for cfg in "MSV_WAVE_PCT=70" "MSV_WAVE_PCT=86 MSV_WAVE_CAP_GIB=160"; do env $cfg MSV_HOST_TIMING=1 timeout 900 python bench.py --no-cpu-baseline > $P/b.log 2>&1; echo -n "$cfg: "; grep -m1 "wave(s)" $P/b.log | cut -c20-90; tail -1 $P/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e9,3), round(d['e2e']['value']/1e9,3), round(d['ms_per_step'],2), d['stage_ms'])"; done; done
