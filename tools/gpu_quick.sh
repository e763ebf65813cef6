mkdir -p gpurun_out
timeout 300 python tools/kbench.py --workload shape:262144,592,563,256 --algos tc --only encode --iters 10 >> gpurun_out/quick.txt 2>&1
for w in cfg2_packed cfg3_c128; do timeout 300 python bench.py --workload $w --steps 200 --warmup 10 --no-cpu-baseline --e2e-steps 2 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('$w', round(d['ms_per_step']*1e3,2), [(k['kernel'][:8], round(k['ms']*1e3,1)) for k in d['roofline']['kernels']])" >> gpurun_out/quick.txt; done
for w in cfg5 cfg4_c64 cfg4_c256; do timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('$w', round(d['ms_per_step']*1e3,2))" >> gpurun_out/quick.txt; done
