#!/bin/bash
TAG=${1:-clk}
mkdir -p gpurun_out
timeout 300 python tools/clock_probe.py cfg5 acc >> gpurun_out/clk_$TAG.log 2>&1
ITLUMM_TCP_DBG=2 timeout 300 python tools/clock_probe.py cfg5 acc >> gpurun_out/clk_$TAG.log 2>&1
timeout 300 python tools/clock_probe.py cfg5 fused >> gpurun_out/clk_$TAG.log 2>&1
