#!/bin/bash
# Bench lines of every workload (builder-run), under gpurun_out/<dir>/.
O=gpurun_out/${1:-sweep}
mkdir -p $O
timeout 900 python bench.py > $O/bench_cfg5.json 2> $O/bench_cfg5.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference_cfg5.json 2> $O/bench_reference_cfg5.err
for w in cfg5_packed; do timeout 900 python bench.py --workload $w > $O/bench_$w.json 2> $O/bench_$w.err; done
for w in cfg2 cfg2_packed cfg1 cfg3_c64 cfg3_c128 cfg3_c64_packed cfg3_c128_packed; do timeout 600 python bench.py --workload $w --steps 200 --warmup 5 --e2e-steps 3 > $O/bench_$w.json 2> $O/bench_$w.err; done
for w in cfg4_c16 cfg4_c64 cfg4_c256; do timeout 900 python bench.py --workload $w --steps 10 --warmup 3 --e2e-steps 2 > $O/bench_$w.json 2> $O/bench_$w.err; done
