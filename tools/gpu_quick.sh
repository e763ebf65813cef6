mkdir -p gpurun_out
for a in tc_pipe tc_sp; do for w in cfg2 cfg2_packed; do timeout 300 python bench.py --workload $w --algo $a --steps 300 --warmup 10 --no-cpu-baseline --e2e-steps 2 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('$a $w', round(d['ms_per_step']*1e3,2))" >> gpurun_out/quick.txt; done; done
