#!/bin/bash
# (ITLUMM_TCP_SD existed only for this probe; not in the tree)
# k_tcp: two staging boxes per epilogue warp (ITLUMM_TCP_SD=2; the ring then has 2 slots of 2 K-blocks
# or 5 of 1) against one (3 slots of 2): accumulate only (kbench) and streamed-shape parity.
O=gpurun_out/tcpsd
mkdir -p $O
L=$O/kbench.log
for rep in 1 2; do
for cfg in "1 2" "2 2" "2 1" "1 1"; do
  set -- $cfg
  for w in cfg5 cfg3_c128 cfg3_c64; do
    echo "sd=$1 ss=$2 $w" >> $L
    ITLUMM_TCP_SD=$1 ITLUMM_TCP_SS=$2 timeout 300 python tools/kbench.py --workload $w --algos tc_pipe_dense --only acc --iters 10 >> $L 2>&1
  done
done
done
ITLUMM_TCP_SD=2 timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider --timeout 600 -x \
    -k "benched_streamed or parity_small or mlp_cfg4 or edge_strides or strided_rows" > $O/pytest_sd2.log 2>&1; echo rc=$? >> $O/pytest_sd2.log
tail -n 3 $O/pytest_sd2.log
grep -v "^\s*$" $L | cut -c1-200 | paste - -
