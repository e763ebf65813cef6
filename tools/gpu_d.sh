mkdir -p gpurun_out
timeout 300 ./tools/probes/stream_probe > gpurun_out/stream_probe.jsonl 2>&1
timeout 120 python tools/bwprobe.py > gpurun_out/bwprobe.json 2>&1
bash tools/gpu_check.sh d cfg2 cfg3_c64
