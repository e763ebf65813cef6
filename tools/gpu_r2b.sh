#!/bin/bash
# Selector removed, SS=2: full GPU suite; sustained cfg5/cfg3 timings with codes tiles vs direct codes.
TAG=${1:-r2b}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider --timeout 600 > gpurun_out/pytest_$TAG.log 2>&1; echo rc=$? >> gpurun_out/pytest_$TAG.log
L=gpurun_out/sus_$TAG.log
for cd in 0 1; do
  for w in cfg5 cfg3_c128; do
    echo "cdirect=$cd $w" >> $L
    ITLUMM_TCP_CDIRECT=$cd timeout 300 python tools/clock_probe.py $w acc >> $L 2>&1
    ITLUMM_TCP_CDIRECT=$cd timeout 300 python tools/clock_probe.py $w fused >> $L 2>&1
  done
done
