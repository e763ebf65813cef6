#!/bin/bash
# k_tcp: L2 eviction policy of the output tensor stores (ITLUMM_OUT_HINT: 0 default, 1 evict_first,
# 3 / 4 fractional evict_first) so that the 4.3 GB output stream does not evict codes and LUT.
O=gpurun_out/outhint
mkdir -p $O
L=$O/kbench.log
for rep in 1 2; do
for h in 0 1 3 4; do
  for w in cfg5 cfg3_c128; do
    echo "out_hint=$h $w" >> $L
    ITLUMM_OUT_HINT=$h timeout 300 python tools/kbench.py --workload $w --algos tc_pipe_dense --only acc --iters 10 >> $L 2>&1
  done
done
done
for h in 0 1; do
  echo "out_hint=$h bench cfg5" >> $L
  ITLUMM_OUT_HINT=$h timeout 600 python bench.py --steps 20 --warmup 3 --e2e-steps 2 --no-cpu-baseline 2>$O/bench_h$h.err | cut -c1-260 >> $L
done
grep -v "^\s*$" $L | cut -c1-260 | paste - -
