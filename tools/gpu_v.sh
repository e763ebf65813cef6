mkdir -p gpurun_out
for c in 16 64 256; do timeout 900 python bench.py --workload cfg4_c$c --steps 20 --warmup 3 --e2e-steps 3 > gpurun_out/bench_v_c$c.json 2> gpurun_out/bench_v_c$c.err; echo rc=$? >> gpurun_out/bench_v_c$c.err; done
