mkdir -p gpurun_out
for w in cfg2 cfg3_c128 cfg5; do timeout 600 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/rt_$w.json 2>gpurun_out/rt_$w.err; done
