#!/bin/bash
# Round-end evidence (part 1): GPU tests, bench lines (cfg2 headline + the other configs) and the
# ncu launch list of the bench command (one ncu per gpurun call; part 2 = tools/gpu_final_full.sh).
mkdir -p gpurun_out/final
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 240 > gpurun_out/final/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/final/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/final/bench_cfg2.json 2> gpurun_out/final/bench_cfg2.err
for w in cfg1 cfg3_c64 cfg3_c128 cfg2_packed cfg3_c64_packed cfg3_c128_packed; do timeout 600 python bench.py --workload $w --steps 200 --warmup 5 --e2e-steps 3 > gpurun_out/final/bench_$w.json 2> gpurun_out/final/bench_$w.err; done
for w in cfg5 cfg5_packed; do timeout 900 python bench.py --workload $w --steps 20 --warmup 3 --e2e-steps 3 > gpurun_out/final/bench_$w.json 2> gpurun_out/final/bench_$w.err; done
for w in cfg4_c16 cfg4_c64 cfg4_c256; do timeout 900 python bench.py --workload $w --steps 10 --warmup 3 --e2e-steps 2 > gpurun_out/final/bench_$w.json 2> gpurun_out/final/bench_$w.err; done
CMD="python bench.py --steps 20 --warmup 3 --e2e-steps 3 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/final/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/final/launches.csv $CMD > gpurun_out/final/ncu_launches.log 2>&1
echo rc=$? >> gpurun_out/final/ncu_launches.log
