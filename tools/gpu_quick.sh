mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_split_packed.py -q -m gpu --timeout 120 -x -k "tc" > gpurun_out/pw8_tests.txt 2>&1; tail -1 gpurun_out/pw8_tests.txt
for e in "ITLUMM_TC_PW=4" "X=0" "ITLUMM_TC_PW=4" "X=0"; do for w in cfg2 cfg3_c128 cfg5; do env $e timeout 300 python tools/kbench.py --workload $w --algos tc --only acc --iters 20 | sed "s/^/$e /" >> gpurun_out/quick.txt; done; done
for e in "ITLUMM_TC_PW=4" "X=0"; do for w in cfg2 cfg2_packed; do env $e timeout 300 python bench.py --workload $w --steps 300 --warmup 10 --no-cpu-baseline --e2e-steps 2 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('$e $w', round(d['ms_per_step']*1e3,2))" >> gpurun_out/quick.txt; done; done
