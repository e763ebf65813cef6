#!/bin/bash
# (the ITLUMM_TCP_FAST / ITLUMM_TCP_POLL switches exist only in commit b39554f; removed afterwards)
# k_tcp streamlined dense producer (ITLUMM_TCP_FAST 0 generic / 1 ALU one-hot / 2 table): parity of
# the streamed-LUT shapes under each, then the accumulate at cfg5 / cfg3 (kbench, one box).
O=gpurun_out/tcpfast
mkdir -p $O
for f in 1 2; do
  ITLUMM_TCP_FAST=$f timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider --timeout 600 -x \
    -k "benched_streamed or parity_small or mlp_cfg4 or edge_strides or strided_rows" > $O/pytest_fast$f.log 2>&1; echo rc=$? >> $O/pytest_fast$f.log
  tail -3 $O/pytest_fast$f.log
done
L=$O/kbench.log
for rep in 1 2; do
for f in 0 1 2; do
  for w in cfg5 cfg3_c128 cfg3_c64; do
    echo "fast=$f $w" >> $L
    ITLUMM_TCP_FAST=$f timeout 300 python tools/kbench.py --workload $w --algos tc_pipe_dense --only acc --iters 10 >> $L 2>&1
  done
done
done
for f in 0 1 2; do
  echo "fast=$f bench cfg5" >> $L
  ITLUMM_TCP_FAST=$f timeout 600 python bench.py --steps 20 --warmup 3 --e2e-steps 2 --no-cpu-baseline >> $L 2>$O/bench_fast$f.err
done
grep -v "^\s*$" $L | cut -c1-300
