#!/bin/bash
# Last check of the round: smoke, the GPU suite, the default bench line and the cfg3 / packed lines.
O=gpurun_out/last
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -rs > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_cfg5.json 2> $O/bench_cfg5.err
timeout 900 python bench.py --workload cfg5_packed --steps 20 --warmup 3 --e2e-steps 3 > $O/bench_cfg5_packed.json 2> $O/bench_cfg5_packed.err
for w in cfg3_c64 cfg3_c128 cfg3_c64_packed cfg3_c128_packed; do
  timeout 600 python bench.py --workload $w --steps 200 --warmup 5 --e2e-steps 3 > $O/bench_$w.json 2> $O/bench_$w.err
done
for w in cfg4_c64 cfg4_c256; do
  timeout 900 python bench.py --workload $w --steps 10 --warmup 3 --e2e-steps 2 > $O/bench_$w.json 2> $O/bench_$w.err
done
tail -n 2 $O/smoke.log $O/pytest_gpu.log; cat $O/bench_*.json | cut -c1-230
