#!/bin/bash
TAG=${1:-gt}
mkdir -p gpurun_out
for d in 0 4 32; do
  echo "== ST=2 dbg=$d" >> gpurun_out/gtrace_$TAG.log
  ITLUMM_TCP_STAGES=2 ITLUMM_TCP_DBG=$d timeout 300 python tools/tcp_gtrace.py cfg5 >> gpurun_out/gtrace_$TAG.log 2>&1
done
