#!/bin/bash
# A/B of two builds of the library on one box (ITLUMM_DEV_LIB = lib/libitlumm_ref.so vs the in-tree
# build), alternating, on the workloads given; then the GPU parity subset with the in-tree build.
TAG=${1:-ab}
shift
WL=${@:-cfg2 cfg2p cfg1}
mkdir -p gpurun_out
L=gpurun_out/ablib_$TAG.log
timeout 900 python -m pytest tests/test_parity_gpu.py -q -m gpu -p no:cacheprovider -k "${PYK:-small or cfg1 or cfg2 or edge or mlp}" > gpurun_out/pytest_$TAG.log 2>&1; echo rc=$? >> gpurun_out/pytest_$TAG.log
for rep in 1 2; do
  for lib in ref new; do
    for w in $WL; do
      P=""; W=$w
      if [ "${w: -1}" = "p" ]; then P="--packed"; W=${w%p}; fi
      echo "lib=$lib rep=$rep $w" >> $L
      if [ $lib = ref ]; then export ITLUMM_DEV_LIB=$PWD/paper_2207_05808_b200/lib/libitlumm_ref.so; else unset ITLUMM_DEV_LIB; fi
      timeout 300 python tools/kbench.py --workload $W $P --algos tc_pipe --only encode,acc,fused --iters ${ITERS:-100} >> $L 2>&1
    done
  done
done
unset ITLUMM_DEV_LIB
