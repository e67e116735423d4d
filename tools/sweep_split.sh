run() { python bench.py --no-cpu-baseline --steps 5 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e9,3), round(d['ms_per_step'],2))"; }
for sp in "3,1" "2,1,1" "3,1,1" "4,2,1" "2,1,1,1" "3,2,1,1" "6,2,1,1"; do echo -n "split=$sp "; MSV_LIB=${LIBV:-paper_2202_13481_b200/libmsv.so} MSV_CHUNK_SPLIT=$sp run; done
